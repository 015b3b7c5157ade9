#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s9.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests_s9.log
timeout 600 python bench.py --steps 100 --warmup 5 --cpu-seconds 5 --json-out gpurun_out/bench_s9.json > gpurun_out/bench_s9.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_s9.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['l2'], d['e2e'], d['plan_create_s'])"
for c in roadnet yeasth dd webberkstan; do
  timeout 600 python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_s9_$c.json > gpurun_out/bench_s9_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_s9_$c.log | cut -c1-400
done
