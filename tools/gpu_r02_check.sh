#!/bin/bash
# Round-2 check of the tree: build, GPU suite, smoke, default bench line, sanitizer tier
# (memcheck / racecheck / synccheck / initcheck on the split-window, padding, empty-window and
# fused all-gather fixtures).  TAG env = file tag.
TAG=${TAG:-r02}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
if [ "${SANITIZE:-1}" = "1" ]; then
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hotcols.py -q -x -p no:cacheprovider \
    -k "tiny_config or split_window_hub or padding_lanes or single_bit or empty_windows or concatenated_windows or fused_allgather or integer_bit_exact_and_balance_invariant and 64 or hot_cols_integer_bit_exact" \
    > gpurun_out/sanitizer_${tool}_$TAG.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 gpurun_out/sanitizer_${tool}_$TAG.log
done
fi
