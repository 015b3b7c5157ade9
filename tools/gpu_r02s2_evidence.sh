#!/bin/bash
# Evidence for the fixed default kernel: the driver's bench line (default args), ncu --set full of
# the SpMM launch (TF32 and FP16, Reddit-shaped N=128), the launch list of the bench command.
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
TAG=$TAG bash tools/gpu_r02_ncu.sh
