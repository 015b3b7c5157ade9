#!/bin/bash
# multi-rank bench path on one GPU (2 and 4 ranks sharing cuda:0 over gloo) + reference arm
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for n in 2 4; do
  ACCSPMM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $n --steps 20 --warmup 3 --json-out gpurun_out/bench_shared_p$n.json > gpurun_out/bench_shared_p$n.log 2>&1
  echo "shared p$n rc=$?"; tail -1 gpurun_out/bench_shared_p$n.log | cut -c1-400
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
