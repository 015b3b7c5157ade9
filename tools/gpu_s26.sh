#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s26.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s26.log
timeout 1500 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 4 --out gpurun_out/sweep_s26.jsonl --variants \
  reorder=on reorder=on,N=64 kcfg=48,reorder=on,N=64 reorder=on,precision=fp16 > gpurun_out/sweep_s26.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s26.log
timeout 900 python tools/sweep.py --config papers100m_small --N 64 --steps 20 --rounds 4 --out gpurun_out/sweep_s26_p.jsonl --variants x=1 kcfg=48 > gpurun_out/sweep_s26_p.log 2>&1
echo "papers rc=$?"; cut -c1-130 gpurun_out/sweep_s26_p.log
