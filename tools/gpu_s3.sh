#!/bin/bash
# Session-2 probe 2: value L2 prefetch (kcfg 26-28), FP16 conflict-free box, carveout, FW=64 at N=128.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not exhaustive" > gpurun_out/gpu_tests_s3.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s3.log
V=""
for p in tf32 fp16; do for k in 20 24 26 27 28; do V="$V kcfg=$k,reorder=on,precision=$p"; done; done
V="$V kcfg=24,reorder=on,fw=64 kcfg=27,reorder=on,fw=64 kcfg=27,reorder=on,N=64 kcfg=20,reorder=on,N=64 kcfg=27,reorder=on,N=32 kcfg=20,reorder=on,N=32"
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 20 --out gpurun_out/sweep_s3.jsonl --variants $V > gpurun_out/sweep_s3.log 2>&1
echo "sweep rc=$?"; cut -c1-120 gpurun_out/sweep_s3.log | tail -20
timeout 900 python tools/sweep.py --config stencil --N 128 --steps 20 --out gpurun_out/sweep_s3_stencil.jsonl --variants kcfg=20 kcfg=24 kcfg=26 kcfg=27 > gpurun_out/sweep_s3_stencil.log 2>&1
echo "sweep stencil rc=$?"; cut -c1-120 gpurun_out/sweep_s3_stencil.log | tail -4
