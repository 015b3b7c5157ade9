#!/bin/bash
# Stage barriers packed at the head of the warp's shared area (kcfg 85 default ring, 86 deep
# ring) against the default: parity, then interleaved A/B on the reordered Reddit-shaped matrix
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py 85 86 > gpurun_out/variants_parity_head.jsonl 2>&1
echo "parity rc=$?"; cat gpurun_out/variants_parity_head.jsonl | cut -c1-200
if grep -q '"ok": false\|Error' gpurun_out/variants_parity_head.jsonl; then exit 1; fi
R=reorder=auto
bash tools/gpu_ab.sh head reddit 128 5 30 kcfg=-1,$R kcfg=85,$R kcfg=86,$R kcfg=-1,precision=fp16,$R kcfg=85,precision=fp16,$R kcfg=86,precision=fp16,$R
bash tools/gpu_ab.sh head reddit 64 4 30 kcfg=-1,$R kcfg=85,$R kcfg=86,$R
bash tools/gpu_ab.sh head reddit 32 4 30 kcfg=-1,$R kcfg=85,$R kcfg=86,$R
bash tools/gpu_ab.sh head products 128 3 20 kcfg=-1,$R kcfg=85,$R
