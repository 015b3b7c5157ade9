#!/bin/bash
# 32-bit vs 64-bit value decode (default vs kcfg 62) on the L2- and issue-bound regimes; value
# evict-first (53) on the HBM-bound papers100M-shaped matrix
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
run() { timeout 1500 python tools/sweep.py --config $1 --N $2 --rounds 3 --steps 15 --variants $3 --out gpurun_out/sweep_dec_${TAG}_$1_$2_$4.jsonl > /dev/null 2>gpurun_out/sweep_dec_${TAG}_$1_$2_$4.err; echo "$1 $2 $4 rc=$?"
  python -c "
import json
for l in open('gpurun_out/sweep_dec_${TAG}_$1_$2_$4.jsonl'): r=json.loads(l); print('  %-40s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"; }
run reddit 128 "kcfg=-1,reorder=auto kcfg=62,reorder=auto" tf32
run reddit 128 "kcfg=-1,reorder=auto,precision=fp16 kcfg=62,reorder=auto,precision=fp16" fp16
run reddit 32 "kcfg=-1,reorder=auto kcfg=62,reorder=auto" tf32
run papers100m 64 "kcfg=-1 kcfg=62 kcfg=53" tf32
