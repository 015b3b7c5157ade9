#!/bin/bash
# End-of-session check of the committed tree: build, full GPU suite, smoke, the driver's bench
# command, compute-sanitizer tier (incl. the 16-row-window kernel), ncu launch list + one full
# capture of the default kernel (TF32 Reddit-shaped N = 128)
TAG=${TAG:-r02s3}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hotcols.py tests/test_gpu_tall_mma.py -q -x -p no:cacheprovider \
    -k "tiny_config or split_window_hub or padding_lanes or single_bit or empty_windows or concatenated_windows or fused_allgather or integer_bit_exact_and_balance_invariant and 64 or hot_cols_integer_bit_exact or every_tile_position or tall_mma_integer_bit_exact_split_windows and 64" \
    > gpurun_out/sanitizer_${tool}_$TAG.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -2 gpurun_out/sanitizer_${tool}_$TAG.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 3 -c 1 \
  -o gpurun_out/prof_${TAG}_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 > gpurun_out/ncu_${TAG}_tf32.log 2>&1
echo "ncu full rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ncu --no-e2e > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
