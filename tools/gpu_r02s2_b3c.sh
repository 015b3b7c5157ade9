#!/bin/bash
# B3 with deeper TMA rings (60: 3 stages / 18 warps, 61: 4 stages / 14 warps) vs B3 and FP32 rows (+ FP32 3-stage, 50)
TAG=${TAG:-r02s2}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
ACCSPMM_LIB=variants timeout 600 python tests/_variants_worker.py > gpurun_out/variants_parity_b3c_$TAG.jsonl 2>&1; echo "variants parity rc=$?"; grep -c "\"ok\": true" gpurun_out/variants_parity_b3c_$TAG.jsonl; grep "\"ok\": false" gpurun_out/variants_parity_b3c_$TAG.jsonl | cut -c1-300
for cfg in "reddit 128" "products 128" "reddit 256"; do set -- $cfg
  timeout 900 python tools/sweep.py --config $1 --N $2 --rounds 3 --steps 20 --variants b3=0,reorder=auto b3=1,reorder=auto kcfg=50,b3=0,reorder=auto kcfg=60,reorder=auto kcfg=61,reorder=auto \
    --out gpurun_out/sweep_b3c_${TAG}_$1_$2.jsonl > /dev/null 2>gpurun_out/sweep_b3c_${TAG}_$1_$2.err; echo "$cfg rc=$?"
  python -c "
import json
for l in open('gpurun_out/sweep_b3c_${TAG}_$1_$2.jsonl'): r=json.loads(l); print('  %-30s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"
done
