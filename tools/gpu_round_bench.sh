#!/bin/bash
# Official round bench + ncu evidence (1 GPU).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py --json-out gpurun_out/bench_r01.json > gpurun_out/bench_r01.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r01.log | cut -c1-600
for v in "--reorder off" "--precision fp16" "--N 64" "--N 32" "--config stencil" "--config products" "--config products --reorder off" "--config stencil --reorder off"; do
  tag=$(echo $v | tr -d ' -')
  timeout 600 python bench.py $v --steps 30 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_r01_$tag.json > gpurun_out/bench_r01_$tag.log 2>&1; echo "$v rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --json-out gpurun_out/bench_r01_reference.json > gpurun_out/bench_r01_reference.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_r01_reference.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_r01.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_r01_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_r01.log 2>&1; echo "ncu full rc=$?"
