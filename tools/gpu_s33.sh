#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s33.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s33.log
timeout 600 python bench.py --N 602 --steps 30 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_s33_N602.json > gpurun_out/bench_s33_N602.log 2>&1; echo "N602 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_s33_N602.json')); print(round(d['value']), d['ms_per_step'], d['roofline']['launch_ms'])"
