#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python tools/partition_scaling.py reddit 128 10 > gpurun_out/scaling_reddit.log 2>&1; echo "reddit rc=$?"; tail -1 gpurun_out/scaling_reddit.log | cut -c1-300; grep "^[1248] " gpurun_out/scaling_reddit.log | cut -c1-200
REORDER=off timeout 2400 python tools/partition_scaling.py papers100m 64 5 > gpurun_out/scaling_papers.log 2>&1; echo "papers rc=$?"; grep "^[1248] " gpurun_out/scaling_papers.log | cut -c1-200
