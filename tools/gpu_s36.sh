#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "zero_width or fused_allgather or any_feature" > gpurun_out/gpu_tests_s36.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s36.log
ACCSPMM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 20 --warmup 3 --allgather nccl --json-out gpurun_out/bench_shared2_p2.json > gpurun_out/bench_shared2_p2.log 2>&1
echo "shared p2 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_shared2_p2.json')); print(d['value'], d['ms_per_step'], d['n_gpus'], d['allgather'], d['e2e']['value'])"
