cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi; nvidia-smi -q -d CLOCK,PERFORMANCE | head -60
(cd build/r1tree && timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400) > gpurun_out/diag_r1tree.txt; echo r1 done
timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-ncu 2>&1 | tail -1 | cut -c1-400 > gpurun_out/diag_head.txt; echo head done
timeout 600 python tools/sweep.py --config reddit --N 128 --rounds 2 --steps 20 --variants kcfg=-1,reorder=auto > gpurun_out/diag_sweep.txt 2>&1; echo sweep done
cat gpurun_out/diag_*.txt
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
