#!/bin/bash
# Bench lines (20 steps, in-job ncu DRAM traffic) for the other configs and widths of DESIGN.md §7
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
line() { name=$1; shift
  timeout 1200 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline "$@" --json-out gpurun_out/line_${TAG}_$name.json > gpurun_out/line_${TAG}_$name.log 2>&1; echo "$name rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/line_${TAG}_$name.json')); r=d['roofline']
print('   %.3f ms (min %.3f) %.0f GFLOP/s  bound=%s frac=%.3f l2=%.3f hbm=%s dram=%s MHz=%s hot=%s' % (d['ms_per_step'], d['step_ms_min'], d['value'], r['bound'], r['frac'], r['l2']['frac'], (r['hbm'] or {}).get('frac'), r.get('traffic'), d['clocks']['sm_mhz'], d['plan'].get('hot_cols')))"
}
line reddit_fp16 --precision fp16
line reddit_n64 --N 64
line reddit_n32 --N 32
line reddit_n256 --N 256
line reddit_fp16_n256 --precision fp16 --N 256
line products --config products
line products_hubs --config products_hubs
line stencil --config stencil
line banded --config banded
line roadnet --config roadnet
line webberkstan --config webberkstan
