#!/bin/bash
# B3 parity (after the pack fix) + A/B: FP32 rows vs B3 vs B3 with values 2 blocks ahead (58) vs B3 at 24 warps (59)
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_b3.py -q -p no:cacheprovider > gpurun_out/b3b_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/b3b_tests_$TAG.log
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py > gpurun_out/variants_parity_b3_$TAG.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_b3_$TAG.jsonl; grep "\"ok\": false" gpurun_out/variants_parity_b3_$TAG.jsonl | cut -c1-300
for cfg in "reddit 128" "reddit 64" "products 128"; do set -- $cfg
  timeout 900 python tools/sweep.py --config $1 --N $2 --rounds 3 --steps 20 --variants b3=0,reorder=auto b3=1,reorder=auto kcfg=58,reorder=auto kcfg=59,reorder=auto \
    --out gpurun_out/sweep_b3b_${TAG}_$1_$2.jsonl > /dev/null 2>gpurun_out/sweep_b3b_${TAG}_$1_$2.err; echo "$cfg rc=$?"
  python -c "
import json
for l in open('gpurun_out/sweep_b3b_${TAG}_$1_$2.jsonl'): r=json.loads(l); print('  %-30s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"
done
