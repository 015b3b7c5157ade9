#!/bin/bash
cd "$GRAFT_REPO_ROOT"
ACCSPMM_LIB=variants timeout 900 python tests/_variants_worker.py > gpurun_out/variants_parity_pin.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_pin.jsonl; grep "\"ok\": false\|Error" gpurun_out/variants_parity_pin.jsonl | cut -c1-300
bash tools/gpu_ab.sh pin reddit 128 3 15 kcfg=-1,reorder=auto,precision=fp16 kcfg=66,reorder=auto,precision=fp16
bash tools/gpu_ab.sh pin reddit 128 3 15 kcfg=-1,reorder=auto kcfg=66,reorder=auto
bash tools/gpu_ab.sh pin reddit 32 3 15 kcfg=-1,reorder=auto kcfg=66,reorder=auto
bash tools/gpu_ab.sh pin reddit 64 3 15 kcfg=-1,reorder=auto kcfg=66,reorder=auto
bash tools/gpu_ab.sh pin stencil 128 3 15 kcfg=-1 kcfg=66
