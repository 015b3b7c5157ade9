#!/bin/bash
# interleaved A/B (5 rounds): 2 warps/CTA (default) vs 1 warp/CTA (kcfg 42)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 5 --out gpurun_out/sweep_s15.jsonl --variants \
  reorder=on kcfg=42,reorder=on reorder=on,precision=fp16 kcfg=42,reorder=on,precision=fp16 reorder=on,N=64 kcfg=42,reorder=on,N=64 reorder=on,N=256 kcfg=42,reorder=on,N=256 > gpurun_out/sweep_s15.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s15.log
timeout 900 python tools/sweep.py --config products --N 128 --steps 10 --rounds 4 --out gpurun_out/sweep_s15_products.jsonl --variants reorder=on kcfg=42,reorder=on > gpurun_out/sweep_s15_products.log 2>&1
echo "products rc=$?"; cut -c1-130 gpurun_out/sweep_s15_products.log
timeout 900 python tools/sweep.py --config stencil --N 128 --steps 20 --rounds 4 --out gpurun_out/sweep_s15_stencil.jsonl --variants x=1 kcfg=42 > gpurun_out/sweep_s15_stencil.log 2>&1
echo "stencil rc=$?"; cut -c1-130 gpurun_out/sweep_s15_stencil.log
