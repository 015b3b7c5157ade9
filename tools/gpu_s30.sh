#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python tools/repro_illegal.py reddit 20 2>&1 | tail -1
timeout 300 python tools/repro_illegal.py dcsbm:100000:30000000 20 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s30.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s30.log
timeout 1500 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 4 --out gpurun_out/sweep_s30.jsonl --variants reorder=on reorder=on,precision=fp16 reorder=on,N=64 > gpurun_out/sweep_s30.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s30.log
for c in products stencil papers100m_small; do timeout 900 python tools/sweep.py --config $c --N 128 --steps 20 --rounds 3 --out gpurun_out/sweep_s30_$c.jsonl --variants reorder=on > gpurun_out/sweep_s30_$c.log 2>&1; echo "$c rc=$?"; cut -c1-130 gpurun_out/sweep_s30_$c.log; done
