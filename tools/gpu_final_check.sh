#!/bin/bash
# final check of the committed tree: build, GPU suite, smoke, default bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_finalcheck.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_finalcheck.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_finalcheck.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_finalcheck.log
timeout 900 python bench.py --json-out gpurun_out/bench_finalcheck.json > gpurun_out/bench_finalcheck.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_finalcheck.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_finalcheck.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_finalcheck.log | cut -c1-200
