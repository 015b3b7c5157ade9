#!/bin/bash
# Session-2 probe: gather4 template variants (kcfg 20/23/24/25) at TF32/FP16, wide N, and an ncu full capture of FP16.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 20 --out gpurun_out/sweep_s2.jsonl --variants \
  kcfg=20,reorder=on kcfg=23,reorder=on kcfg=24,reorder=on kcfg=25,reorder=on kcfg=21,reorder=on \
  kcfg=20,reorder=on,precision=fp16 kcfg=23,reorder=on,precision=fp16 kcfg=24,reorder=on,precision=fp16 kcfg=25,reorder=on,precision=fp16 \
  kcfg=20,reorder=on,N=256 kcfg=20,reorder=on,N=512 kcfg=20,reorder=on,N=256,precision=fp16 > gpurun_out/sweep_s2.log 2>&1
echo "sweep rc=$?"; cut -c1-160 gpurun_out/sweep_s2.log | tail -14
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_s2_reddit_fp16 python bench.py --profile --steps 1 --warmup 3 --no-flush --precision fp16 > gpurun_out/ncu_fp16.log 2>&1; echo "ncu fp16 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_bittcf -s 3 -c 1 \
  -o gpurun_out/prof_s2_reddit_tf32 python bench.py --profile --steps 1 --warmup 3 --no-flush > gpurun_out/ncu_tf32.log 2>&1; echo "ncu tf32 rc=$?"
