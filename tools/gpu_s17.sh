#!/bin/bash
# full GPU suite on the new defaults, official-length bench, launch list, ncu full TF32 + FP16
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s17.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s17.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s17.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_s17.log
timeout 900 python bench.py --json-out gpurun_out/bench_r01s3.json > gpurun_out/bench_r01s3.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_r01s3.json')); r=d['roofline']
print(d['value'], d['ms_per_step'], r['launch_ms'], r['frac'], r['l2']['frac'], d['clocks'], d['e2e']['value'], d['e2e']['sync_per_step']['value'])"
for v in "--precision fp16" "--N 64" "--N 32" "--N 256" "--N 512" "--config products" "--config stencil" "--config roadnet" "--config papers100m_small --N 64"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 50 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_r01s3_$t.json > gpurun_out/bench_r01s3_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_r01s3_$t.json')); r=d['roofline']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  kernel', round(r['launch_ms'],3), 'l2frac', round(r['l2']['frac'],3))" 2>&1 | tail -1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01s3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_r01s3.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_r01s3_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_r01s3.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_r01s3_reddit_fp16 python bench.py --profile --steps 1 --warmup 3 --no-flush --precision fp16 > gpurun_out/ncu_full_r01s3_fp16.log 2>&1; echo "ncu fp16 rc=$?"
