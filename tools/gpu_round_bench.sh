#!/bin/bash
# Official round bench + ncu evidence (1 GPU).  TAG env = file tag (default r01).
TAG=${TAG:-r01}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
for v in "--reorder off" "--precision fp16" "--N 64" "--N 32" "--config stencil" "--config products" "--config papers100m_small --N 64 --reorder off"; do
  t=$(echo $v | tr -d ' -')
  timeout 600 python bench.py $v --steps 30 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_${TAG}_$t.json > gpurun_out/bench_${TAG}_$t.log 2>&1; echo "$v rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_${TAG}_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
