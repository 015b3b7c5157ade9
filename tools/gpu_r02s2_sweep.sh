#!/bin/bash
# Round 2 session 2: TMA gather4 throughput probe + interleaved A/B of the unmeasured mma.sync
# variants (53 value evict-first, 54/55 chunk values by bulk copy, 56 hybrid TMA + cp.async gather)
# on the request-bound (FP16 N=128, TF32 N=32) and L2-bound (TF32 N=128) regimes.
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py > gpurun_out/variants_parity_$TAG.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_$TAG.jsonl; grep "\"ok\": false" gpurun_out/variants_parity_$TAG.jsonl | cut -c1-300
timeout 300 ./build/tma_gather_probe > gpurun_out/tma_probe3_$TAG.txt 2>&1; echo "probe rc=$?"
timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-ncu 2>&1 | tail -1 | cut -c 1-300
V="kcfg=-1,reorder=auto kcfg=53,reorder=auto kcfg=54,reorder=auto kcfg=55,reorder=auto kcfg=56,reorder=auto kcfg=57,reorder=auto"
timeout 900 python tools/sweep.py --config reddit --N 128 --rounds 3 --steps 20 --variants $V --out gpurun_out/sweep_${TAG}_tf32.jsonl > /dev/null 2>gpurun_out/sweep_${TAG}_tf32.err; echo "tf32 rc=$?"
VF=$(for v in $V; do printf "%s,precision=fp16 " $v; done)
timeout 900 python tools/sweep.py --config reddit --N 128 --rounds 3 --steps 20 --variants $VF --out gpurun_out/sweep_${TAG}_fp16.jsonl > /dev/null 2>gpurun_out/sweep_${TAG}_fp16.err; echo "fp16 rc=$?"
timeout 900 python tools/sweep.py --config reddit --N 32 --rounds 3 --steps 20 --variants $V --out gpurun_out/sweep_${TAG}_n32.jsonl > /dev/null 2>gpurun_out/sweep_${TAG}_n32.err; echo "n32 rc=$?"
for f in gpurun_out/sweep_${TAG}_*.jsonl; do echo $f; python -c "
import json,sys
for l in open('$f'): r=json.loads(l); print('  %-40s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"; done
