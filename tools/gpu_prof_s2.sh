#!/bin/bash
# Round-1 (session 2) evidence: launch list of the default bench command, ncu --set full of the
# SpMM kernel (TF32 default, FP16), official-length bench line.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01s2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_r01s2.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_r01s2_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_full_r01s2.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_r01s2_reddit_fp16 python bench.py --profile --steps 1 --warmup 3 --no-flush --precision fp16 > gpurun_out/ncu_full_r01s2_fp16.log 2>&1; echo "ncu fp16 rc=$?"
timeout 900 python bench.py --json-out gpurun_out/bench_r01s2.json > gpurun_out/bench_r01s2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r01s2.log | cut -c1-300
