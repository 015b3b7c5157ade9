#!/bin/bash
# ncu full captures of the default SpMM launch in the request/latency-bound regimes
# (Reddit-shaped: TF32 N = 32 and 64, FP16 N = 128)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "tf32_N32:--N 32" "tf32_N64:--N 64" "fp16_N128:--precision fp16"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 3 -c 1 \
    -o gpurun_out/prof_narrow_$tag python bench.py --profile --steps 1 --warmup 3 $args > gpurun_out/ncu_narrow_$tag.log 2>&1
  echo "ncu $tag rc=$?"
done
