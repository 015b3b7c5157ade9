#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
V="reorder=on reorder=on,precision=fp16 kcfg=24,reorder=on,precision=fp16 kcfg=31,reorder=on,precision=fp16 kcfg=20,reorder=on,precision=fp16 reorder=on,N=256 reorder=on,N=256,precision=fp16 kcfg=24,reorder=on,N=256,precision=fp16"
timeout 1200 python tools/sweep.py --config reddit --N 128 --steps 30 --out gpurun_out/sweep_s6.jsonl --variants $V > gpurun_out/sweep_s6.log 2>&1
echo "sweep rc=$?"; cut -c1-110 gpurun_out/sweep_s6.log
ACCSPMM_TRACE=1 timeout 600 python -c "
import sys,time; sys.path.insert(0,'.')
import gen, paper_2501_09251_b200 as acc
cfg,A=gen.make_config('reddit'); v=gen.values_uniform(A.nnz,cfg.seed_A+1)
for b in ('host','device'):
    t=time.perf_counter(); p=acc.Plan(A.M,A.K,A.rowptr,A.colidx,v,reorder='on',build=b); dt=time.perf_counter()-t
    print(b, round(dt,2), {k: round(p.info[k],1) for k in ('ms_reorder','ms_build','ms_schedule','ms_upload')})
" > gpurun_out/plan_times.log 2>&1; cat gpurun_out/plan_times.log
