#!/bin/bash
# Hot columns (R22): parity + A/B on the B >> L2 configs (papers100M-shaped N=64, products-shaped N=128)
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hotcols.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/hot_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/hot_tests_$TAG.log
ACCSPMM_LIB=variants timeout 900 python tests/_variants_worker.py > gpurun_out/variants_parity_hot_$TAG.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_hot_$TAG.jsonl; grep "\"ok\": false\|Error" gpurun_out/variants_parity_hot_$TAG.jsonl | cut -c1-300
run() { timeout 1800 python tools/sweep.py --config $1 --N $2 --rounds 3 --steps 10 --variants $3 --out gpurun_out/sweep_hot_${TAG}_$1_$2.jsonl > /dev/null 2>gpurun_out/sweep_hot_${TAG}_$1_$2.err; echo "$1 $2 rc=$?"
  python -c "
import json
for l in open('gpurun_out/sweep_hot_${TAG}_$1_$2.jsonl'): r=json.loads(l); print('  %-40s %.3f ms (min %.3f) hot=%s'%(r['variant'],r['ms'],r['ms_min'],r['hot_cols']))"; }
run papers100m 64 "hot=off hot=on hot=on,hmb=32 hot=on,hmb=96"
run products 128 "hot=off,reorder=auto hot=on,reorder=auto hot=on,reorder=auto,hmb=32"
