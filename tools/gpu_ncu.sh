#!/bin/bash
# ncu full capture of the SpMM kernel for one configuration (env: TAG, BENCHARGS, KCFG)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
export ACCSPMM_KCFG=${KCFG:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 2 -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py --profile --steps 1 --warmup 2 --no-flush $BENCHARGS > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
