#!/bin/bash
# Stage-wait flavour (kcfg 79-84: try_wait without the suspend hint / test_wait spin) on the
# default kernel, on the layout that runs 2.7x slow with the hinted wait (77) and on the deep
# ring (70): parity, then interleaved A/B on the reordered Reddit-shaped matrix
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py 79 80 81 82 83 84 > gpurun_out/variants_parity_wait.jsonl 2>&1
echo "parity rc=$?"; cat gpurun_out/variants_parity_wait.jsonl | cut -c1-200
if grep -q '"ok": false\|Error' gpurun_out/variants_parity_wait.jsonl; then exit 1; fi
R=reorder=auto
bash tools/gpu_ab.sh wait reddit 128 4 30 kcfg=-1,$R kcfg=79,$R kcfg=80,$R kcfg=77,$R kcfg=81,$R kcfg=82,$R kcfg=70,$R kcfg=83,$R kcfg=84,$R
bash tools/gpu_ab.sh wait reddit 128 4 30 kcfg=-1,precision=fp16,$R kcfg=79,precision=fp16,$R kcfg=80,precision=fp16,$R kcfg=70,precision=fp16,$R kcfg=83,precision=fp16,$R kcfg=84,precision=fp16,$R
bash tools/gpu_ab.sh wait reddit 64 4 30 kcfg=-1,$R kcfg=79,$R kcfg=80,$R kcfg=70,$R kcfg=83,$R kcfg=84,$R
bash tools/gpu_ab.sh wait reddit 32 4 30 kcfg=-1,$R kcfg=79,$R kcfg=80,$R kcfg=83,$R kcfg=84,$R
