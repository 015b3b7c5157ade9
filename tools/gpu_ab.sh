#!/bin/bash
# Interleaved A/B of plan/kernel variants on one matrix (GPU box), one JSON line per variant.
# usage: bash tools/gpu_ab.sh TAG CONFIG N ROUNDS STEPS VARIANT...
#   VARIANT = comma-separated tools/sweep.py keys, e.g. kcfg=62,reorder=auto  hot=on,hmb=32
#   (kcfg variants and ACCSPMM_* knobs exist only in libaccspmm_variants.so, which sweep.py loads)
TAG=$1; CFG=$2; N=$3; ROUNDS=$4; STEPS=$5; shift 5
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
OUT=gpurun_out/sweep_${TAG}_${CFG}_${N}.jsonl
timeout 2400 python tools/sweep.py --config "$CFG" --N "$N" --rounds "$ROUNDS" --steps "$STEPS" --variants "$@" \
  --out "$OUT" > /dev/null 2> "${OUT%.jsonl}.err"; echo "$CFG N=$N rc=$?"
python -c "
import json
for l in open('$OUT'): r=json.loads(l); print('  %-44s %.3f ms (min %.3f)'%(r['variant'],r['ms'],r['ms_min']))"
