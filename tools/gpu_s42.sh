#!/bin/bash
# value loads with ld.global.nc.L2::256B (kcfg 52)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ACCSPMM_KCFG=52 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ragged_float or integer_bit_exact or split_window or single_bit or full_size_config_sampled" > gpurun_out/gpu_tests_s42.log 2>&1; echo "tests kcfg52 rc=$?"; tail -1 gpurun_out/gpu_tests_s42.log
timeout 2000 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 5 --out gpurun_out/sweep_s42.jsonl --variants \
  reorder=on kcfg=52,reorder=on reorder=on,precision=fp16 kcfg=52,reorder=on,precision=fp16 reorder=on,N=64 kcfg=52,reorder=on,N=64 > gpurun_out/sweep_s42.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s42.log
for c in papers100m_small stencil; do timeout 900 python tools/sweep.py --config $c --N 64 --steps 20 --rounds 3 --out gpurun_out/sweep_s42_$c.jsonl --variants x=1 kcfg=52 > gpurun_out/sweep_s42_$c.log 2>&1; echo "$c rc=$?"; cut -c1-130 gpurun_out/sweep_s42_$c.log; done
timeout 900 python tools/sweep.py --config products --N 128 --steps 10 --rounds 3 --out gpurun_out/sweep_s42_pr.jsonl --variants reorder=on kcfg=52,reorder=on > gpurun_out/sweep_s42_pr.log 2>&1
echo "products rc=$?"; cut -c1-130 gpurun_out/sweep_s42_pr.log
