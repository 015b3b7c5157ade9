#!/bin/bash
# Round-1 final evidence with the final binary: GPU suite, smoke, official bench line, other
# workloads, launch list, ncu full TF32/FP16.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final2.log
timeout 900 python bench.py --json-out gpurun_out/bench_final2.json > gpurun_out/bench_final2.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final2.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r['l2']['frac'], d['clocks'], d['e2e']['value'], d['e2e']['sync_per_step']['value'], d['cpu_baseline']['value'])"
for v in "--precision fp16" "--N 64" "--N 256" "--config products" "--config stencil" "--config roadnet" "--config papers100m_small --N 64"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 50 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_final2_$t.json > gpurun_out/bench_final2_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_final2_$t.json')); r=d['roofline']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  min', round(d['step_ms_min'],3), 'l2frac', round(r['l2']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_final2.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_final2_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_final2.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_final2_reddit_fp16 python bench.py --profile --steps 1 --warmup 3 --no-flush --precision fp16 > gpurun_out/ncu_full_final2_fp16.log 2>&1; echo "ncu fp16 rc=$?"
