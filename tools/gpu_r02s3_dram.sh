#!/bin/bash
# DRAM bytes of one SpMM launch (Reddit-shaped TF32 N = 128, cold L2): the default against value
# loads with an L2 evict-first policy (kcfg 53)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:g4_kernel --clock-control none --csv --log-file gpurun_out/dram.csv \
  python tools/sweep.py --config reddit --N 128 --steps 1 --variants kcfg=-1,reorder=auto kcfg=53,reorder=auto > gpurun_out/dram.log 2>&1
echo "rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/dram.csv')) if len(r)>10]
h=rows[0]; iN=h.index('Metric Name'); iV=h.index('Metric Value'); iid=h.index('ID')
for r in rows[1:]:
    print(r[iid], r[iN], r[iV])
PY
