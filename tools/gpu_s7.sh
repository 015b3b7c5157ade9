#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or build" > gpurun_out/gpu_tests_s7.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s7.log
V="reorder=on reorder=on,precision=fp16 kcfg=31,reorder=on,precision=fp16 reorder=on kcfg=24,reorder=on reorder=on,precision=fp16 reorder=on,N=256 kcfg=24,reorder=on,N=256 reorder=on,N=256,precision=fp16 reorder=on,N=512"
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 30 --out gpurun_out/sweep_s7.jsonl --variants $V > gpurun_out/sweep_s7.log 2>&1
echo "sweep rc=$?"; cut -c1-110 gpurun_out/sweep_s7.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --json-out gpurun_out/bench_s7.json > gpurun_out/bench_s7.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_s7.log | cut -c1-1500
