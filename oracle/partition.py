"""nnz-balanced contiguous RowWindow ranges across ranks (TEST INFRASTRUCTURE ONLY).

BASELINE.json north_star: "Row windows are partitioned by nnz-balanced ranges
across the GPUs of one 8xB200 box."  Reading (SURVEY §8(c) C-2 "Partition"):
pre(w) = nnz in windows [0, w); b_0 = 0, b_P = W and, in exact integers,
b_k = min{ w : P*pre(w) >= k*nnz } for k = 1..P-1.  Rank k owns [b_k, b_{k+1}).
"""
from __future__ import annotations

import numpy as np


def window_nnz(M: int, rowptr) -> np.ndarray:
    rowptr = np.asarray(rowptr, dtype=np.int64)
    W = (M + 7) // 8
    ends = np.minimum(np.arange(1, W + 1) * 8, M)
    starts = np.arange(W) * 8
    return rowptr[ends] - rowptr[starts]


def bounds(M: int, rowptr, nparts: int) -> list:
    """[b_0, ..., b_P] by the literal min{} definition (O(P*W) brute force)."""
    wn = window_nnz(M, rowptr)
    W = wn.size
    pre = [0]
    for x in wn:
        pre.append(pre[-1] + int(x))
    nnz = pre[-1]
    out = [0]
    for k in range(1, nparts):
        b = next(w for w in range(W + 1) if nparts * pre[w] >= k * nnz)
        out.append(b)
    out.append(W)
    return out
