#!/bin/bash
# Run-to-run spread of the driver's bench command (5 fresh processes) and one default-length
# (300-step) line on the final tree
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-ncu --no-cpu-baseline --json-out gpurun_out/rep_$i.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/rep_$i.json')); r=d['roofline']
print('run $i', round(d['value']), 'GFLOP/s', round(d['ms_per_step'],4), 'ms', 'l2 frac', round(r['l2']['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', round(d['e2e']['value']))"
done
timeout 900 python bench.py --json-out gpurun_out/rep_default300.json > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/rep_default300.json')); r=d['roofline']
print('default 300 steps', round(d['value']), 'GFLOP/s', round(d['ms_per_step'],4), 'ms', 'bound', r['bound'], round(r['frac'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', round(d['e2e']['value']))"
