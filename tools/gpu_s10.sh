#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_autograd.py -q -x -p no:cacheprovider -k "permute or autograd or forward or input_checks" > gpurun_out/gpu_tests_s10.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests_s10.log
for v in "" "--permute-cols" "--N 256" "--N 256 --permute-cols" "--N 512" "--N 512 --permute-cols" "--config products" "--config products --permute-cols" "--precision fp16 --permute-cols" "--config roadnet --permute-cols"; do
  t=$(echo "x$v" | tr -d ' -')
  timeout 600 python bench.py $v --steps 30 --no-cpu-baseline --no-e2e --build device --json-out gpurun_out/bench_s10_$t.json > gpurun_out/bench_s10_$t.log 2>&1
  echo "$v rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s10_$t.json')); r=d['roofline']
print('  ', round(d['value']), 'GF/s', round(d['ms_per_step'],3), 'ms  kernel', round(r['launch_ms'],3), 'l2frac', round(r['l2']['frac'],3), 'plan_s', round(d['plan_create_s'],2))" 2>&1 | tail -1
done
