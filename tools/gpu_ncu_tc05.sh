#!/bin/bash
# ncu full capture of the tcgen05 kernel (and the mma.sync one) on the Reddit-shaped workload
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "tc05_w32:--kernel tcgen05 --window-rows 32" "tc05_w8:--kernel tcgen05 --window-rows 8"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 2 -c 1 \
    -o gpurun_out/prof_$tag python bench.py --profile --steps 1 --warmup 2 --no-flush $args > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
done
