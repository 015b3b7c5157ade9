#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "measurement_variants" > gpurun_out/gpu_tests_s43.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_s43.log
