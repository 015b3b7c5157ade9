#!/bin/bash
# type-1 matrices: balance (window grouping) on/off, reorder on/off, N = 128/512; L2 probe
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python -c "
import sys; sys.path.insert(0,'.')
import paper_2501_09251_b200 as acc
for b in (16<<20, 64<<20, 96<<20): print('l2 probe', b>>20, 'MiB', round(acc.accspmm_probe_l2_bandwidth(b, 40)), 'GB/s')
" 2>&1 | tee gpurun_out/l2probe.log
for c in roadnet yeasth dd webberkstan; do
  timeout 900 python tools/sweep.py --config $c --N 128 --steps 30 --out gpurun_out/sweep_s8_$c.jsonl --variants \
    balance=off balance=on balance=auto,reorder=on balance=on,reorder=on balance=on,N=512 balance=off,N=512 balance=on,reorder=on,N=512 > gpurun_out/sweep_s8_$c.log 2>&1
  echo "$c rc=$?"; cut -c1-150 gpurun_out/sweep_s8_$c.log
done
timeout 900 python tools/sweep.py --config stencil --N 128 --steps 30 --out gpurun_out/sweep_s8_stencil.jsonl --variants balance=off balance=on > gpurun_out/sweep_s8_stencil.log 2>&1
echo "stencil rc=$?"; cut -c1-150 gpurun_out/sweep_s8_stencil.log
