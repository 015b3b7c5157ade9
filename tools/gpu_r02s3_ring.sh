#!/bin/bash
# Deep-ring variants (kcfg 70/71/72: TMA + values 2-3 blocks ahead, run-time stage index):
# parity first, then interleaved A/B against the default on the request/latency-bound regimes
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py 70 71 72 73 74 > gpurun_out/variants_parity_ring.jsonl 2>&1
echo "parity rc=$?"; cat gpurun_out/variants_parity_ring.jsonl | cut -c1-200
if grep -q '"ok": false\|Error' gpurun_out/variants_parity_ring.jsonl; then exit 1; fi
bash tools/gpu_ab.sh ring reddit 128 3 20 kcfg=-1,precision=fp16 kcfg=70,precision=fp16 kcfg=71,precision=fp16 kcfg=73,precision=fp16 kcfg=74,precision=fp16 kcfg=-1 kcfg=70 kcfg=71 kcfg=72 kcfg=73
bash tools/gpu_ab.sh ring reddit 32 3 20 kcfg=-1 kcfg=70 kcfg=71 kcfg=73 kcfg=74
bash tools/gpu_ab.sh ring reddit 64 3 20 kcfg=-1 kcfg=70 kcfg=71 kcfg=73 kcfg=74
