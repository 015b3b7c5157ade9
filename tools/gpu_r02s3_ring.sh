#!/bin/bash
# Deep-ring variants (kcfg 70-72: TMA + values 2-3 blocks ahead, run-time stage index), coalesced
# value loads (73/74) and stage-barrier spacing (75-78): parity first, then interleaved A/B
# against the default on the reordered Reddit-shaped matrix (the bench's plan)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py ${PARITY:-75 76 77 78} > gpurun_out/variants_parity_ring.jsonl 2>&1
echo "parity rc=$?"; cat gpurun_out/variants_parity_ring.jsonl | cut -c1-200
if grep -q '"ok": false\|Error' gpurun_out/variants_parity_ring.jsonl; then exit 1; fi
R=reorder=auto
bash tools/gpu_ab.sh bar reddit 128 3 30 kcfg=-1,precision=fp16,$R kcfg=75,precision=fp16,$R kcfg=76,precision=fp16,$R kcfg=77,precision=fp16,$R kcfg=78,precision=fp16,$R kcfg=70,precision=fp16,$R kcfg=-1,$R kcfg=77,$R kcfg=78,$R kcfg=75,$R
bash tools/gpu_ab.sh bar reddit 64 3 30 kcfg=-1,$R kcfg=70,$R kcfg=75,$R kcfg=76,$R kcfg=77,$R kcfg=78,$R
bash tools/gpu_ab.sh bar reddit 32 3 30 kcfg=-1,$R kcfg=75,$R kcfg=77,$R kcfg=78,$R
