#!/bin/bash
# End-of-round evidence with the final binary (GPU suite, smoke, default bench, wide N, launch list, ncu)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_final3.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final3.log
timeout 900 python bench.py --json-out gpurun_out/bench_final3.json > gpurun_out/bench_final3.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final3.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r['l2']['frac'], d['clocks'], d['e2e']['value'], d['e2e']['sync_per_step']['value'], d['cpu_baseline']['value'], r['bytes_model_per_launch'].get('B_compulsory'))"
for v in "--N 256" "--N 512" "--precision fp16 --N 256" "--N 602"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 30 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_final3_$t.json > gpurun_out/bench_final3_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_final3_$t.json')); r=d['roofline']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  min', round(d['step_ms_min'],3), 'l2frac', round(r['l2']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_final3.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_final3_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_final3.log 2>&1; echo "ncu full rc=$?"
