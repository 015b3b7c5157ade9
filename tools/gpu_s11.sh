#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in products reddit stencil papers100m_small; do for m in 1 2; do
  ACCSPMM_ROUND_B=$m timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline --no-e2e --build device --json-out gpurun_out/bench_s11_${c}_$m.json > gpurun_out/bench_s11_${c}_$m.log 2>&1
  echo "$c round=$m rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s11_${c}_$m.json')); r=d['roofline']; p=d['plan']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  kernel', round(r['launch_ms'],3), 'reuse', round(p['sum_U']/d['config']['K'],1))" 2>&1 | tail -1
done; done
