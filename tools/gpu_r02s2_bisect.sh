#!/bin/bash
# Bisect of the default-kernel slowdown (Reddit-shaped N=128 TF32: 2.5 ms at round 1, 5.5 ms at HEAD)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for t in build/bs_e737541 build/bs_54e9b09 build/bs_7a0b6f6 build/bs_209b66c build/r1tree .; do
  (cd $t && timeout 400 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-ncu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step'],3), d['step_ms_min'], d['plan']['n_units'])")
done
timeout 300 ./build/tma_gather_probe > gpurun_out/tma_probe2_r02s2.txt 2>&1; echo "probe rc=$?"
