#!/bin/bash
# one warp per CTA (uniform smem addresses: fewer R2UR in the TMA issue, kcfg 42) and TMA without L2 hint (43)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ACCSPMM_KCFG=42 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or split_window or full_size_config_sampled" > gpurun_out/gpu_tests_s14.log 2>&1; echo "tests kcfg42 rc=$?"; tail -3 gpurun_out/gpu_tests_s14.log
V="reorder=on kcfg=42,reorder=on kcfg=43,reorder=on reorder=on,precision=fp16 kcfg=42,reorder=on,precision=fp16 kcfg=43,reorder=on,precision=fp16 reorder=on,N=64 kcfg=42,reorder=on,N=64 reorder=on kcfg=42,reorder=on"
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 30 --out gpurun_out/sweep_s14.jsonl --variants $V > gpurun_out/sweep_s14.log 2>&1
echo "sweep rc=$?"; cut -c1-120 gpurun_out/sweep_s14.log
timeout 900 python tools/sweep.py --config products --N 128 --steps 20 --out gpurun_out/sweep_s14_products.jsonl --variants reorder=on kcfg=42,reorder=on > gpurun_out/sweep_s14_products.log 2>&1
echo "products rc=$?"; cut -c1-120 gpurun_out/sweep_s14_products.log
