"""GPU-box probe: can torch symmetric memory rendezvous two ranks sharing one GPU (gloo group)?
If so the fused all-gather path runs end to end here (tests/test_gpu_distributed_fused.py)."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group(os.environ.get("PG", "gloo"))
try:
    from paper_2501_09251_b200 import distributed as D
    fa = D.FusedAllGather(64, 16, torch.device("cuda", 0))
    print("rank", rank, "symmetric memory OK", flush=True)
except Exception as e:
    print("rank", rank, "symmetric memory unavailable:", repr(e)[:300], flush=True)
dist.destroy_process_group()
