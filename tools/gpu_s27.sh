#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fused_allgather or cuda_graph or partitions or unpermute" > gpurun_out/gpu_tests_s27.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_s27.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tools/probe_symm_shared.py > gpurun_out/probe_symm.log 2>&1; echo "probe rc=$?"; grep -v "^W1\|warn" gpurun_out/probe_symm.log | tail -6
PG=nccl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tools/probe_symm_shared.py > gpurun_out/probe_symm_nccl.log 2>&1; echo "probe nccl rc=$?"; grep -v "^W1\|warn" gpurun_out/probe_symm_nccl.log | tail -6
timeout 1500 python tools/sweep.py --config reddit --N 128 --steps 20 --rounds 3 --out gpurun_out/sweep_s27.jsonl --variants reorder=on reorder=on,precision=fp16 > gpurun_out/sweep_s27.log 2>&1
echo "sweep rc=$?"; cut -c1-130 gpurun_out/sweep_s27.log
