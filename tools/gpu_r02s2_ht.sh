#!/bin/bash
# default kernel without tag handling for untagged plans (HT = false) + parity of the touched tests
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_hotcols.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/ht_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ht_tests_$TAG.log
run() { timeout 1500 python tools/sweep.py --config $1 --N $2 --rounds 3 --steps 15 --variants $3 --out gpurun_out/sweep_ht_${TAG}_$1_$2_$4.jsonl > /dev/null 2>gpurun_out/sweep_ht_${TAG}_$1_$2_$4.err; echo "$1 $2 $4 rc=$?"
  python -c "
import json
for l in open('gpurun_out/sweep_ht_${TAG}_$1_$2_$4.jsonl'): r=json.loads(l); print('  %-40s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"; }
run reddit 128 "kcfg=-1,reorder=auto kcfg=62,reorder=auto kcfg=63,reorder=auto" tf32
run reddit 128 "kcfg=-1,reorder=auto,precision=fp16 kcfg=63,reorder=auto,precision=fp16" fp16
run reddit 32 "kcfg=-1,reorder=auto kcfg=62,reorder=auto kcfg=63,reorder=auto" tf32
run reddit 64 "kcfg=-1,reorder=auto kcfg=63,reorder=auto" tf32
run papers100m 64 "hot=on hot=off" tf32
