#!/bin/bash
# papers100M-shaped (configs[4], N=64 TF32) bench lines with the in-job ncu DRAM traffic: reorder auto (R21) and off
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for ro in auto off; do
  timeout 1800 python bench.py --config papers100m --N 64 --steps 20 --warmup 3 --reorder $ro --no-e2e --cpu-seconds 5 --ncu-timeout 900 \
    --json-out gpurun_out/bench_p100m_${ro}_$TAG.json > gpurun_out/bench_p100m_${ro}_$TAG.log 2>&1; echo "p100m $ro rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_p100m_${ro}_$TAG.json')); r=d['roofline']
print(d['ms_per_step'], d['value'], r['bound'], r['frac'], r.get('traffic'), r['l2']['frac'], (r['hbm'] or {}).get('frac'), d['clocks']['sm_mhz'], d['plan']['ms_reorder'], d['plan']['NB'], d['plan_create_s'])"
done
