#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ACCSPMM_SLICE_MAJOR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or split_window" > gpurun_out/gpu_tests_s35.log 2>&1; echo "tests sm rc=$?"; tail -2 gpurun_out/gpu_tests_s35.log
timeout 2000 python tools/sweep.py --config reddit --N 256 --steps 10 --rounds 4 --out gpurun_out/sweep_s35.jsonl --variants \
  reorder=on sm=1,reorder=on reorder=on,N=512 sm=1,reorder=on,N=512 reorder=on,N=256,precision=fp16 sm=1,reorder=on,N=256,precision=fp16 > gpurun_out/sweep_s35.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s35.log
timeout 900 python tools/sweep.py --config products --N 256 --steps 10 --rounds 3 --out gpurun_out/sweep_s35_p.jsonl --variants reorder=on sm=1,reorder=on > gpurun_out/sweep_s35_p.log 2>&1
echo "products rc=$?"; cut -c1-130 gpurun_out/sweep_s35_p.log
