#!/bin/bash
# TF32 m16n8k8 fed by two LDS.64 per tile (L64 layout: rows FW + 4 elements apart, no register
# moves; kcfg 87 at the tuned bound, 88 at 4 more warps): parity, then interleaved A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py 87 88 > gpurun_out/variants_parity_l64.jsonl 2>&1
echo "parity rc=$?"; cat gpurun_out/variants_parity_l64.jsonl | cut -c1-200
if grep -q '"ok": false\|Error' gpurun_out/variants_parity_l64.jsonl; then exit 1; fi
R=reorder=auto
bash tools/gpu_ab.sh l64 reddit 128 5 30 kcfg=-1,$R kcfg=87,$R kcfg=88,$R
bash tools/gpu_ab.sh l64 reddit 64 4 30 kcfg=-1,$R kcfg=87,$R kcfg=88,$R
bash tools/gpu_ab.sh l64 reddit 32 4 30 kcfg=-1,$R kcfg=87,$R kcfg=88,$R
bash tools/gpu_ab.sh l64 reddit 256 3 20 kcfg=-1,$R kcfg=87,$R kcfg=88,$R
bash tools/gpu_ab.sh l64 products 128 3 20 kcfg=-1,$R kcfg=87,$R kcfg=88,$R
bash tools/gpu_ab.sh l64 stencil 128 3 30 kcfg=-1,$R kcfg=87,$R kcfg=88,$R
