#!/bin/bash
# Is the 2-4x cliff an address-mapping effect?  The deep ring (70) and the default ring with the
# per-CTA shared-memory footprint padded by 128 B - 1 KB (kcfg 90-94), on the regimes where the
# deep ring collapses (TF32 N = 64, FP16 N = 128) and N = 128 TF32
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py 90 91 92 93 94 > gpurun_out/variants_parity_pad.jsonl 2>&1
echo "parity rc=$?"; cat gpurun_out/variants_parity_pad.jsonl | cut -c1-120
if grep -q '"ok": false\|Error' gpurun_out/variants_parity_pad.jsonl; then exit 1; fi
R=reorder=auto
bash tools/gpu_ab.sh pad reddit 64 4 30 kcfg=-1,$R kcfg=70,$R kcfg=90,$R kcfg=91,$R kcfg=92,$R kcfg=93,$R kcfg=94,$R
bash tools/gpu_ab.sh pad reddit 128 4 30 kcfg=-1,precision=fp16,$R kcfg=70,precision=fp16,$R kcfg=90,precision=fp16,$R kcfg=91,precision=fp16,$R kcfg=92,precision=fp16,$R kcfg=93,precision=fp16,$R kcfg=94,precision=fp16,$R
bash tools/gpu_ab.sh pad reddit 128 3 30 kcfg=-1,$R kcfg=93,$R kcfg=94,$R kcfg=90,$R
