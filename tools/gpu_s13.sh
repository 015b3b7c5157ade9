#!/bin/bash
# value staging through shared memory (kcfg 40 = tuned MINB + VST, 41 = MINB 1 + VST)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ACCSPMM_KCFG=40 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or split_window or single_bit or dense_band or empty_windows or full_size_config_sampled" > gpurun_out/gpu_tests_s13.log 2>&1; echo "tests kcfg40 rc=$?"; tail -3 gpurun_out/gpu_tests_s13.log
V="reorder=on kcfg=40,reorder=on kcfg=41,reorder=on reorder=on,precision=fp16 kcfg=40,reorder=on,precision=fp16 reorder=on,N=64 kcfg=40,reorder=on,N=64 reorder=on kcfg=40,reorder=on"
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 30 --out gpurun_out/sweep_s13.jsonl --variants $V > gpurun_out/sweep_s13.log 2>&1
echo "sweep rc=$?"; cut -c1-120 gpurun_out/sweep_s13.log
timeout 900 python tools/sweep.py --config products --N 128 --steps 20 --out gpurun_out/sweep_s13_products.jsonl --variants reorder=on kcfg=40,reorder=on > gpurun_out/sweep_s13_products.log 2>&1
echo "products rc=$?"; cut -c1-120 gpurun_out/sweep_s13_products.log
