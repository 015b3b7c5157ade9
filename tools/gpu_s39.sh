#!/bin/bash
# L2 persisting access-policy window on B (ACCSPMM_L2_PERSIST MiB)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('persisting max', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)"
timeout 2000 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 4 --out gpurun_out/sweep_s39.jsonl --variants \
  reorder=on persist=48,reorder=on persist=80,reorder=on persist=120,reorder=on reorder=on,precision=fp16 persist=80,reorder=on,precision=fp16 > gpurun_out/sweep_s39.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s39.log
timeout 900 python tools/sweep.py --config products --N 128 --steps 10 --rounds 3 --out gpurun_out/sweep_s39_pr.jsonl --variants reorder=on persist=80,reorder=on > gpurun_out/sweep_s39_pr.log 2>&1
echo "products rc=$?"; cut -c1-130 gpurun_out/sweep_s39_pr.log
