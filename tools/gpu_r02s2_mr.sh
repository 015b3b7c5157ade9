#!/bin/bash
# multi-rank path on one GPU (gloo, every rank on cuda:0): torchrun 2 ranks, Reddit-shaped and papers100M 1/64
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
export ACCSPMM_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/mr_reddit.log 2>&1; echo "reddit rc=$?"; tail -1 gpurun_out/mr_reddit.log | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 10 --warmup 3 --config papers100m_small --N 64 > gpurun_out/mr_p100s.log 2>&1; echo "p100m_small rc=$?"; tail -1 gpurun_out/mr_p100s.log | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/mr_ref.log | cut -c1-200
