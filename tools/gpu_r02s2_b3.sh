#!/bin/bash
# B3 (3-byte TF32 image of B): parity + interleaved A/B against FP32 rows (ACCSPMM_B3=0).
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_b3.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/b3_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/b3_tests_$TAG.log
for cfg in "reddit 128" "reddit 64" "reddit 256" "products 128"; do set -- $cfg
  timeout 900 python tools/sweep.py --config $1 --N $2 --rounds 3 --steps 20 --variants b3=1,reorder=auto b3=0,reorder=auto \
    --out gpurun_out/sweep_b3_${TAG}_$1_$2.jsonl > /dev/null 2>gpurun_out/sweep_b3_${TAG}_$1_$2.err; echo "$cfg rc=$?"
  python -c "
import json
for l in open('gpurun_out/sweep_b3_${TAG}_$1_$2.jsonl'): r=json.loads(l); print('  %-30s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"
done
timeout 900 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --json-out gpurun_out/bench_b3_$TAG.json > gpurun_out/bench_b3_$TAG.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_b3_$TAG.json')); r=d['roofline']
print(d['ms_per_step'], d['value'], r['bound'], r['frac'], r.get('traffic'), r['l2']['frac'], d['clocks']['sm_mhz'])"
