#!/bin/bash
# Round-1 profiling + tuning sweep on one B200.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python tools/sweep.py --config reddit --N 128 --out gpurun_out/sweep_reddit.jsonl --variants \
  kcfg=0 kcfg=1 kcfg=2 kcfg=3 kcfg=0,cap=32 kcfg=0,cap=128 kcfg=0,cap=512 kcfg=0,balance=off \
  kcfg=0,precision=fp16 kcfg=1,precision=fp16 kcfg=0,N=64 kcfg=0,N=32 kcfg=0,N=256 > gpurun_out/sweep_reddit.log 2>&1
echo "sweep rc=$?"; cat gpurun_out/sweep_reddit.log | tail -16
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r01.csv \
  python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_launches_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 2 -c 1 \
  -o gpurun_out/prof_reddit_tf32_r01 python bench.py --profile --steps 1 --warmup 2 --no-flush > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout 900 python tools/sweep.py --config reddit --N 128 --steps 10 --out gpurun_out/sweep_reorder.jsonl --variants \
  kcfg=0,reorder=on > gpurun_out/sweep_reorder.log 2>&1; echo "reorder rc=$?"; tail -3 gpurun_out/sweep_reorder.log
