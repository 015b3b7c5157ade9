#!/bin/bash
# one warp per CTA as the default; FP16 ldmatrix fragments (kcfg 44)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s16.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s16.log
ACCSPMM_KCFG=44 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fp16 and (ragged_float or integer_bit_exact or split_window or single_bit or dense_band or empty_windows or full_size or permute)" > gpurun_out/gpu_tests_s16_ldsm.log 2>&1; echo "tests kcfg44 rc=$?"; tail -3 gpurun_out/gpu_tests_s16_ldsm.log
timeout 1500 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 5 --out gpurun_out/sweep_s16.jsonl --variants \
  reorder=on kcfg=46,reorder=on reorder=on,precision=fp16 kcfg=44,reorder=on,precision=fp16 kcfg=46,reorder=on,precision=fp16 reorder=on,N=256 kcfg=46,reorder=on,N=256 reorder=on,N=32 kcfg=46,reorder=on,N=32 reorder=on,N=16 kcfg=46,reorder=on,N=16 > gpurun_out/sweep_s16.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s16.log
