#!/bin/bash
# configs[4] full size (papers100M-shaped, 111M rows, ~1.6B nnz), N = 64, one GPU, current kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
free -g | tee gpurun_out/free_x2.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 2400 python bench.py --config papers100m --N 64 --reorder off --steps 10 --warmup 3 --no-e2e --cpu-seconds 10 --build device --json-out gpurun_out/bench_x2.json > gpurun_out/bench_x2.log 2>&1; echo "x rc=$?"; tail -3 gpurun_out/bench_x2.log | cut -c1-600
