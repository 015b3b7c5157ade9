#!/bin/bash
# papers100M-shaped N=64 (HBM-bound): B3 (3-byte TF32 image, needs the rho(B) pre-pass) vs FP32 rows
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python tools/sweep.py --config papers100m --N 64 --rounds 3 --steps 10 --variants "rb=2" "rb=1" "rb=1,b3=1" \
  --out gpurun_out/sweep_p100m_b3_$TAG.jsonl > /dev/null 2>gpurun_out/sweep_p100m_b3_$TAG.err; echo "rc=$?"
python -c "
import json
for l in open('gpurun_out/sweep_p100m_b3_$TAG.jsonl'): r=json.loads(l); print('  %-30s %.3f ms (min %.3f) hot=%s'%(r['variant'],r['ms'],r['ms_min'],r['hot_cols']))"
timeout 1200 python -m pytest tests/test_gpu_hotcols.py -q -p no:cacheprovider 2>&1 | tail -2
