#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
free -g | tee gpurun_out/free.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null
true
true
timeout 1500 python bench.py --config papers100m --N 64 --reorder off --steps 10 --warmup 3 --no-e2e --cpu-seconds 10 --json-out gpurun_out/bench_x.json > gpurun_out/bench_x.log 2>&1; echo "x rc=$?"; tail -25 gpurun_out/bench_x.log | cut -c1-300
