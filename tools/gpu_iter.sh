#!/bin/bash
# Iteration script: GPU parity tests + tuning sweep + short bench.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider -k "not exhaustive" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 900 python tools/sweep.py --config reddit --N 128 --out gpurun_out/sweep.jsonl --variants $SWEEP > gpurun_out/sweep.log 2>&1
echo "sweep rc=$?"; cut -c1-200 gpurun_out/sweep.log | tail -20
