#!/bin/bash
# Hot columns (R22) on papers100M-shaped N=64: bench lines (in-job ncu DRAM bytes) hot on vs off, reorder off
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hotcols.py -q -p no:cacheprovider > gpurun_out/hot2_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/hot2_tests_$TAG.log
for h in on off; do
  timeout 1800 python bench.py --config papers100m --N 64 --steps 10 --warmup 3 --reorder off --hot-cols $h --no-e2e --no-cpu-baseline --ncu-timeout 900 \
    --json-out gpurun_out/bench_p100m_hot${h}_$TAG.json > gpurun_out/bench_p100m_hot${h}_$TAG.log 2>&1; echo "p100m hot=$h rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_p100m_hot${h}_$TAG.json')); r=d['roofline']
print(d['ms_per_step'], d['step_ms_min'], r['bound'], r['frac'], r.get('traffic'), (r['hbm'] or {}).get('frac'), d['clocks']['sm_mhz'], d['plan']['hot_cols'], r['traffic_detail'].get('l2_tex_read_bytes'))"
done
