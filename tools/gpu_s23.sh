#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s23.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s23.log
for v in "--config papers100m_small --N 64" "--config stencil" "--config roadnet" "--config yeasth" "--config dd" "--config webberkstan"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 50 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_s23_$t.json > gpurun_out/bench_s23_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s23_$t.json')); r=d['roofline']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  min', round(d['step_ms_min'],3), 'units', d['plan']['n_units'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
timeout 2400 python bench.py --config papers100m --N 64 --reorder off --steps 10 --warmup 3 --no-e2e --cpu-seconds 10 --json-out gpurun_out/bench_x3.json > gpurun_out/bench_x3.log 2>&1; echo "x rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_x3.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], r['l2']['frac'], d['plan']['n_units'], d['plan_create_s'], d['clocks'], d['cpu_baseline'])"
