#!/bin/bash
# Session-2 check: full GPU suite with the tuned launch bounds + per-slice tensor maps; wide-N sweep.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_s5.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests_s5.log
V=""
for n in 128 256 512; do for p in tf32 fp16; do V="$V reorder=on,N=$n,precision=$p"; done; done
V="$V kcfg=20,reorder=on,N=256 reorder=on,N=64 reorder=on,N=32 reorder=on,N=16 reorder=on,N=64,precision=fp16"
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 20 --out gpurun_out/sweep_s5.jsonl --variants $V > gpurun_out/sweep_s5.log 2>&1
echo "sweep rc=$?"; cut -c1-110 gpurun_out/sweep_s5.log
