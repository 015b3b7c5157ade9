#!/bin/bash
# concatenation limit (reading R7c): ACCSPMM_GROUP_CAP sweep on HBM- and L2-bound matrices
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { c=$1; N=$2; shift 2; timeout 1500 python tools/sweep.py --config $c --N $N --steps 20 --rounds 4 --out gpurun_out/sweep_s22_$c.jsonl --variants "$@" > gpurun_out/sweep_s22_$c.log 2>&1; echo "$c rc=$?"; cut -c1-120 gpurun_out/sweep_s22_$c.log; }
run papers100m_small 64 gcap=16 gcap=32 gcap=64 gcap=128 balance=off
run reddit 128 reorder=on,gcap=32 reorder=on,gcap=64 reorder=on,gcap=128 reorder=on,gcap=4096
run products 128 reorder=on,gcap=32 reorder=on,gcap=64 reorder=on,gcap=4096
run stencil 128 gcap=32 gcap=64 gcap=4096
run roadnet 128 reorder=on,gcap=16 reorder=on,gcap=32 reorder=on,balance=off
