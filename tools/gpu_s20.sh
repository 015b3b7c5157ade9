#!/bin/bash
# after_block sentinel (default) + TF32 m16n8k8 variant (kcfg 48)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s20.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s20.log
ACCSPMM_KCFG=48 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tf32 and (ragged_float or integer_bit_exact or split_window or full_size)" > gpurun_out/gpu_tests_s20_k8.log 2>&1; echo "tests kcfg48 rc=$?"; tail -2 gpurun_out/gpu_tests_s20_k8.log
timeout 1500 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 5 --out gpurun_out/sweep_s20.jsonl --variants \
  reorder=on kcfg=48,reorder=on reorder=on,N=64 kcfg=48,reorder=on,N=64 > gpurun_out/sweep_s20.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s20.log
