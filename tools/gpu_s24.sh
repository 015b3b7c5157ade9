#!/bin/bash
# TF32 m16n8k4 (default) vs m16n8k8 (kcfg 48), interleaved, more rounds
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 2000 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 8 --out gpurun_out/sweep_s24.jsonl --variants \
  reorder=on kcfg=48,reorder=on reorder=on,N=64 kcfg=48,reorder=on,N=64 reorder=on,N=32 kcfg=48,reorder=on,N=32 > gpurun_out/sweep_s24.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s24.log
