#!/bin/bash
# Full GPU suite + variant parity (incl. the B3 variants) + smoke on the current tree
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_$TAG.log
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py > gpurun_out/variants_parity_$TAG.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_$TAG.jsonl; grep "\"ok\": false\|Error" gpurun_out/variants_parity_$TAG.jsonl | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
