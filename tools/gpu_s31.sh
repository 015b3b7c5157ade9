#!/bin/bash
# values two blocks ahead (kcfg 49), now that the LDGSTS miscompile is gone
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ACCSPMM_KCFG=49 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or split_window or single_bit or empty_windows or full_size_config_sampled" > gpurun_out/gpu_tests_s31.log 2>&1; echo "tests kcfg49 rc=$?"; tail -2 gpurun_out/gpu_tests_s31.log
timeout 2000 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 5 --out gpurun_out/sweep_s31.jsonl --variants \
  reorder=on kcfg=49,reorder=on reorder=on,precision=fp16 kcfg=49,reorder=on,precision=fp16 reorder=on,N=64 kcfg=49,reorder=on,N=64 > gpurun_out/sweep_s31.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s31.log
timeout 900 python tools/sweep.py --config products --N 128 --steps 10 --rounds 4 --out gpurun_out/sweep_s31_products.jsonl --variants reorder=on kcfg=49,reorder=on > gpurun_out/sweep_s31_products.log 2>&1
echo "products rc=$?"; cut -c1-130 gpurun_out/sweep_s31_products.log
