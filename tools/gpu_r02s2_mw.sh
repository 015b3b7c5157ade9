#!/bin/bash
cd "$GRAFT_REPO_ROOT"
ACCSPMM_LIB=variants timeout 900 python tests/_variants_worker.py > gpurun_out/variants_parity_mw.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_mw.jsonl; grep "\"ok\": false\|Error" gpurun_out/variants_parity_mw.jsonl | cut -c1-300
bash tools/gpu_ab.sh mw reddit 32 3 15 kcfg=-1,reorder=auto kcfg=68,reorder=auto kcfg=69,reorder=auto
bash tools/gpu_ab.sh mw reddit 64 3 15 kcfg=-1,reorder=auto kcfg=68,reorder=auto kcfg=69,reorder=auto
bash tools/gpu_ab.sh mw reddit 128 3 15 kcfg=-1,reorder=auto,precision=fp16 kcfg=68,reorder=auto,precision=fp16 kcfg=69,reorder=auto,precision=fp16
bash tools/gpu_ab.sh mw reddit 128 3 15 kcfg=-1,reorder=auto kcfg=68,reorder=auto kcfg=69,reorder=auto
