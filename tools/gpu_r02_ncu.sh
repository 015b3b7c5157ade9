#!/bin/bash
# ncu full captures of the default SpMM kernel (TF32 and FP16, Reddit-shaped N=128) + launch list
TAG=${TAG:-r02}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "tf32:" "fp16:--precision fp16"; do
  tag=${cfg%%:*}; args=${cfg#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_reddit_$tag python bench.py --profile --steps 1 --warmup 3 $args > gpurun_out/ncu_${TAG}_$tag.log 2>&1
  echo "ncu $tag rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-ncu > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
