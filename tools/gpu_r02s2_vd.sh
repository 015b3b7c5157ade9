#!/bin/bash
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"
ACCSPMM_LIB=variants timeout 900 python tests/_variants_worker.py > gpurun_out/variants_parity_vd_$TAG.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_vd_$TAG.jsonl; grep "\"ok\": false\|Error" gpurun_out/variants_parity_vd_$TAG.jsonl | cut -c1-300
bash tools/gpu_ab.sh vd reddit 128 3 15 kcfg=-1,reorder=auto,precision=fp16 kcfg=65,reorder=auto,precision=fp16
bash tools/gpu_ab.sh vd reddit 128 3 15 kcfg=-1,reorder=auto kcfg=65,reorder=auto
bash tools/gpu_ab.sh vd reddit 32 3 15 kcfg=-1,reorder=auto kcfg=65,reorder=auto
bash tools/gpu_ab.sh vd reddit 64 3 15 kcfg=-1,reorder=auto kcfg=65,reorder=auto
bash tools/gpu_ab.sh vd webberkstan 128 3 15 kcfg=-1,reorder=auto kcfg=65,reorder=auto
