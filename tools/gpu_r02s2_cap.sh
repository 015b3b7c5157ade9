#!/bin/bash
# products-shaped (HBM-bound, B = 1.25 GB): unit cap vs the rows in flight (L2 working set)
cd "$GRAFT_REPO_ROOT"
bash tools/gpu_ab.sh cap products 128 2 10 reorder=auto reorder=auto,cap=64 reorder=auto,cap=128 reorder=auto,cap=256 reorder=auto,cap=1024
bash tools/gpu_ab.sh cap reddit 128 2 10 reorder=auto reorder=auto,cap=128 reorder=auto,cap=256
