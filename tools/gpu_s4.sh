#!/bin/bash
# Session-2 probe 3: device BitTCF builder tests, launch-bounds sweep (MINB) across widths/precisions/configs.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_build.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_build.log 2>&1; echo "build tests rc=$?"; tail -15 gpurun_out/gpu_tests_build.log
V=""
for p in tf32 fp16; do for k in 24 31 32 33; do V="$V kcfg=$k,reorder=on,precision=$p"; done; done
for n in 64 32 16; do for k in 20 24 31 33; do V="$V kcfg=$k,reorder=on,N=$n"; done; done
for k in 20 24 31 33; do V="$V kcfg=$k,reorder=on,N=64,precision=fp16"; done
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 20 --out gpurun_out/sweep_s4.jsonl --variants $V > gpurun_out/sweep_s4.log 2>&1
echo "sweep rc=$?"; cut -c1-110 gpurun_out/sweep_s4.log
timeout 900 python tools/sweep.py --config stencil --N 128 --steps 20 --out gpurun_out/sweep_s4_stencil.jsonl --variants kcfg=20 kcfg=24 kcfg=31 kcfg=33 > gpurun_out/sweep_s4_stencil.log 2>&1
echo "sweep stencil rc=$?"; cut -c1-110 gpurun_out/sweep_s4_stencil.log | tail -4
timeout 900 python tools/sweep.py --config products --N 128 --steps 20 --out gpurun_out/sweep_s4_products.jsonl --variants kcfg=20,reorder=on kcfg=24,reorder=on > gpurun_out/sweep_s4_products.log 2>&1
echo "sweep products rc=$?"; cut -c1-110 gpurun_out/sweep_s4_products.log | tail -4
