#!/bin/bash
# Round-1 final evidence (1 GPU): GPU suite + smoke, official bench line, other workloads,
# launch list, ncu --set full TF32/FP16, papers100M-shaped full size.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py --json-out gpurun_out/bench_final.json > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r['l2']['frac'], d['clocks'], d['e2e']['value'], d['e2e']['sync_per_step']['value'], d['cpu_baseline']['value'])"
for v in "--precision fp16" "--N 64" "--N 32" "--N 256" "--N 512" "--config products" "--config stencil" "--config roadnet" "--config yeasth" "--config dd" "--config webberkstan" "--config papers100m_small --N 64" "--precision fp16 --N 256"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 50 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_final_$t.json > gpurun_out/bench_final_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_final_$t.json')); r=d['roofline']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  min', round(d['step_ms_min'],3), 'l2frac', round(r['l2']['frac'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_final.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_final_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_final.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_final_reddit_fp16 python bench.py --profile --steps 1 --warmup 3 --no-flush --precision fp16 > gpurun_out/ncu_full_final_fp16.log 2>&1; echo "ncu fp16 rc=$?"
timeout 2400 python bench.py --config papers100m --N 64 --reorder off --steps 10 --warmup 3 --no-e2e --cpu-seconds 10 --json-out gpurun_out/bench_final_papers100m.json > gpurun_out/bench_final_papers100m.log 2>&1; echo "x rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final_papers100m.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['frac'], r['l2']['frac'], d['plan']['n_units'], d['plan_create_s'], d['clocks'])"
