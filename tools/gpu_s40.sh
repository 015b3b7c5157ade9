#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "full_size_config_sampled" > gpurun_out/gpu_tests_s40.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s40.log
for v in "--config banded" "--config banded --reorder off" "--precision fp16 --N 64" "--precision fp16 --N 32"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 50 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_s40_$t.json > gpurun_out/bench_s40_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s40_$t.json')); r=d['roofline']; p=d['plan']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  min', round(d['step_ms_min'],3), 'l2frac', round(r['l2']['frac'],3), 'NB', p['NB'], 'reorder', p['reorder_applied'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
