#!/bin/bash
# L2 probe through both request engines (LDG / TMA bulk), the default bench line with the new
# peak, and the multi-rank bench path on one GPU (gloo, 2 ranks) after the e2e byte change
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_build.py -q -k "l2_probe" -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "
import paper_2501_09251_b200 as acc
for mb in (32, 64, 96):
    print(mb, 'MiB', 'ldg %.0f' % acc.accspmm_probe_l2_bandwidth_ex(mb << 20, 100, mode=1),
          'tma %.0f' % acc.accspmm_probe_l2_bandwidth_ex(mb << 20, 100, mode=2))
" 2>&1 | tee gpurun_out/l2_probe_engines.txt
timeout 900 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench_probe.json > gpurun_out/bench_probe.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_probe.json')); r=d['roofline']
print('value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'bound', r['bound'], 'frac', round(r['frac'],3), 'peak', round(r['peak']), r['l2']['peak_before'], r['l2']['peak_after'])"
export ACCSPMM_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/mr_reddit.log 2>&1; echo "mr reddit rc=$?"; tail -1 gpurun_out/mr_reddit.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
