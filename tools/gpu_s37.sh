#!/bin/bash
# 3/4-stage TMA ring (kcfg 50/51) vs 2 stages: correctness, then interleaved A/B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for k in 50 51; do
ACCSPMM_KCFG=$k timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or split_window or single_bit or empty_windows or dense_band or full_size_config_sampled" > gpurun_out/gpu_tests_s37_$k.log 2>&1; echo "tests kcfg$k rc=$?"; tail -1 gpurun_out/gpu_tests_s37_$k.log
done
timeout 2000 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 4 --out gpurun_out/sweep_s37.jsonl --variants \
  reorder=on,precision=fp16 kcfg=50,reorder=on,precision=fp16 kcfg=51,reorder=on,precision=fp16 reorder=on,N=64 kcfg=50,reorder=on,N=64 kcfg=51,reorder=on,N=64 reorder=on kcfg=50,reorder=on reorder=on,N=32 kcfg=51,reorder=on,N=32 > gpurun_out/sweep_s37.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s37.log
timeout 900 python tools/sweep.py --config papers100m_small --N 64 --steps 20 --rounds 3 --out gpurun_out/sweep_s37_p.jsonl --variants x=1 kcfg=51 > gpurun_out/sweep_s37_p.log 2>&1
echo "papers rc=$?"; cut -c1-130 gpurun_out/sweep_s37_p.log
