#!/bin/bash
# TMA L2 sector promotion of the gathered rows: none / 64 / 128 / 256 B
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 2000 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 4 --out gpurun_out/sweep_s38.jsonl --variants \
  reorder=on promo=0,reorder=on promo=2,reorder=on reorder=on,precision=fp16 promo=0,reorder=on,precision=fp16 promo=2,reorder=on,precision=fp16 > gpurun_out/sweep_s38.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s38.log
timeout 900 python tools/sweep.py --config papers100m_small --N 64 --steps 20 --rounds 3 --out gpurun_out/sweep_s38_p.jsonl --variants x=1 promo=0 promo=2 > gpurun_out/sweep_s38_p.log 2>&1
echo "papers rc=$?"; cut -c1-130 gpurun_out/sweep_s38_p.log
timeout 900 python tools/sweep.py --config products --N 128 --steps 10 --rounds 3 --out gpurun_out/sweep_s38_pr.jsonl --variants reorder=on promo=0,reorder=on promo=2,reorder=on > gpurun_out/sweep_s38_pr.log 2>&1
echo "products rc=$?"; cut -c1-130 gpurun_out/sweep_s38_pr.log
