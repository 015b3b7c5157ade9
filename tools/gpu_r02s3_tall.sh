#!/bin/bash
# 16-row windows on the mma.sync kernel (reading R20): parity, then interleaved A/B against the
# 8-row default on the reordered Reddit-shaped matrix (TF32 / FP16, N = 128 / 64 / 32)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tall_mma.py -q -x -p no:cacheprovider > gpurun_out/tall_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/tall_tests.log
grep -q "passed" gpurun_out/tall_tests.log && ! grep -q "failed\|error" gpurun_out/tall_tests.log || exit 1
R=reorder=auto
T=wh=16,kernel=mma_sync
bash tools/gpu_ab.sh tall reddit 128 4 30 $R $T,$R precision=fp16,$R precision=fp16,$T,$R
bash tools/gpu_ab.sh tall reddit 64 3 30 $R $T,$R precision=fp16,$R precision=fp16,$T,$R
bash tools/gpu_ab.sh tall reddit 32 3 30 $R $T,$R
bash tools/gpu_ab.sh tall products 128 3 20 $R $T,$R
bash tools/gpu_ab.sh tall stencil 128 3 30 $R $T,$R
