#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "products_hub" > gpurun_out/gpu_tests_s32.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s32.log
for v in "--config products_hubs" "--config products_hubs --balance off"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 900 python bench.py $v --steps 30 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_s32_$t.json > gpurun_out/bench_s32_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s32_$t.json')); r=d['roofline']; p=d['plan']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  min', round(d['step_ms_min'],3), 'l2frac', round(r['l2']['frac'],3), 'units', p['n_units'], 'split', p['n_split_windows'], 'ibd', round(p['ibd'],1))" 2>&1 | tail -1
done
