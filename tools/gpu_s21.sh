#!/bin/bash
# HBM-bound papers100M-shaped: grouping (AUTO) vs one window per unit; 1 vs 2 warps per CTA
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python tools/sweep.py --config papers100m_small --N 64 --steps 20 --rounds 4 --out gpurun_out/sweep_s21.jsonl --variants \
  balance=off balance=auto kcfg=46,balance=off kcfg=46,balance=auto kcfg=20,balance=off balance=on,cap=32 > gpurun_out/sweep_s21.log 2>&1
echo "sweep rc=$?"; cut -c1-150 gpurun_out/sweep_s21.log
bash tools/gpu_s20.sh
