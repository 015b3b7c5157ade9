cd "$GRAFT_REPO_ROOT"
for st in 20 30 60; do timeout 600 python bench.py --steps $st --warmup 5 --no-ncu --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print($st, 'dev', round(d['ms_per_step'],3), 'e2e', round(e['ms_per_step'],3), e['steps'], 'sync', round(e['sync_per_step']['ms_per_step'],3))"; done
