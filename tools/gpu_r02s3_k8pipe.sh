#!/bin/bash
# Tensor-pipe cost of the TF32 MMA shape: m16n8k4 (default at FW 128) vs m16n8k8 (kcfg 48)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__inst_executed_pipe_tensor.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  -k regex:g4_kernel --clock-control none --csv --log-file gpurun_out/k8pipe.csv \
  python tools/sweep.py --config reddit --N 128 --steps 1 --variants kcfg=-1,reorder=auto kcfg=48,reorder=auto > gpurun_out/k8pipe.log 2>&1
echo "rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/k8pipe.csv')) if len(r)>10]
h=rows[0]; iN=h.index('Metric Name'); iV=h.index('Metric Value'); iid=h.index('ID')
for r in rows[1:]:
    print(r[iid], r[iN], r[iV])
PY
