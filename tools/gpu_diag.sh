#!/bin/bash
# ncu captures of the weak configs + compute-sanitizer on small parity cases.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for cfg in "fp16:--precision fp16" "n32:--N 32" "products:--config products"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
    -o gpurun_out/prof_diag_$tag python bench.py --profile --steps 1 --warmup 3 --no-flush $args > gpurun_out/ncu_diag_$tag.log 2>&1
  echo "ncu $tag rc=$?"
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "tiny_config or split_window_hub or padding or single_bit or empty_windows or rho_b" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
