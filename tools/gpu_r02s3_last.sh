#!/bin/bash
# Last check of the final tree: full GPU suite (incl. the variant parity worker), smoke, bench line
TAG=${TAG:-r02s3z}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
