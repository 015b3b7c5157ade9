#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_autograd.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s34.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s34.log
for n in 602 608 96 48 100; do
timeout 600 python bench.py --N $n --steps 20 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_s34_N$n.json > gpurun_out/bench_s34_N$n.log 2>&1; echo "N$n rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s34_N$n.json')); print('  ', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['launch_ms'],3))"
done
