"""IBD, the Eq. (4) cost model and the work-unit schedule (TEST INFRASTRUCTURE ONLY).

PAPER.md §3.5:
  * Eq. (3): IBD = sum_w |TCBlockPerRowWindow_w - AvgTCBlock| / NumOfRowWindow;
    balancing applies when IBD "exceeds 8" -- strict >.
  * Eq. (4): T = LoadDenseTime + MMATime + WBTime, M=K=8, N=16;
    element counts x 4 bytes for the bandwidth terms.
  * TC blocks are redistributed so TBs take "nearly uniform computation
    time", with "a maximum threshold of 32 TC blocks per TB".

The unit builder is the reading of SURVEY Q16 / DESIGN.md "Schedule": contiguous
greedy packing along window order.  A window with more blocks than the cap is
split evenly into ceil(nb/cap) segments (cross-row write-back); shorter
windows are concatenated while sum(blocks + wb) <= cap + wb and at most WMAX
windows per unit, where wb is the C write-back of one window expressed in
TC-block loads (8 rows x N x 4 B over 8 rows x N x es_B: 1 for TF32, 2 for FP16).
"""
from __future__ import annotations

import math

import numpy as np

PROFILES = {  # PAPER.md Table 3; B200 per BASELINE.md §2 (spec, not measured)
    "RTX4090": {"bw": 1008e9, "tf32": 82.6e12},
    "A800": {"bw": 1935e9, "tf32": 156e12},
    "H100": {"bw": 3.35e12, "tf32": 494.7e12},
    "B200": {"bw": 8.0e12, "tf32": 1.1e15},
}

IBD_THRESHOLD = 8.0
PAPER_CAP = 32
WMAX = 31             # windows per concatenated unit (bounds the per-unit C write-back)
NO_SPLIT = 0xFFFFFFFF


def ibd(blocks_per_window) -> float:
    """Eq. (3): mean absolute deviation of TC blocks per RowWindow."""
    x = np.asarray(blocks_per_window, dtype=np.float64)
    if x.size == 0:
        raise ValueError("IBD of an empty window list")
    avg = x.sum() / x.size
    return float(np.abs(x - avg).sum() / x.size)


def eq4_time(profile: str, feature_dim: int, tc_blocks_per_tb: int, elem_bytes: int = 4) -> float:
    """Eq. (4) exactly as printed (WBTime == LoadDenseTime), M=K=8, 4-byte elements."""
    bw, flops = PROFILES[profile]["bw"], PROFILES[profile]["tf32"]
    Mt, Kt = 8, 8
    load = Kt * feature_dim * tc_blocks_per_tb * elem_bytes / bw
    mma = Mt * (2 * Kt - 1) * feature_dim / flops
    wb = Kt * feature_dim * tc_blocks_per_tb * elem_bytes / bw
    return load + mma + wb


def wb_cost(precision: str) -> int:
    """C write-back of one 8-row window in units of one TC block's B-row loads (Q15 corrected form)."""
    return {"tf32": 1, "fp16": 2}[precision]


GROUP_CAP = 32  # reading R7c: concatenation limit of grouped plans under the automatic cap


def auto_group_cap(cap: int) -> int:
    return max(1, min(cap, GROUP_CAP))


def auto_cap(NB: int) -> int:
    """B200 default cap when unit_cap == 0 (reading R7): ~192 units per SM, in [32, 4096], multiple of 32."""
    c = -(-NB // (148 * 192))
    c = -(-c // 32) * 32
    return max(PAPER_CAP, min(4096, c))


def build_units(rwo, cap: int, balance: bool, precision: str = "tf32", group: bool = False,
                group_cap: int | None = None, wh: int = 8):
    """Work units (w0, nw, b0, b1, split_id, seg, nseg, slot) covering every block once.

    Not balanced: one unit per RowWindow, or with ``group`` (the B200 reading R7b,
    DESIGN.md: balance AUTO below the IBD threshold) consecutive WHOLE windows packed into
    one unit by the same concatenation rule, never split.  ``group_cap`` (reading R7c) bounds
    the concatenation separately from the split cap (default: cap)."""
    rwo = np.asarray(rwo, dtype=np.int64)
    W = rwo.size - 1
    units = []
    if not balance and not group:
        for w in range(W):
            units.append((w, 1, int(rwo[w]), int(rwo[w + 1]), NO_SPLIT, 0, 1, 0))
        return units
    wb = wb_cost(precision) * (wh // 8)   # a window of wh rows writes wh/8 tiles' worth of C
    split_id = 0
    slot = 0
    cur = None  # [w0, nw, b0, b1, cost]
    for w in range(W):
        nb = int(rwo[w + 1] - rwo[w])
        if nb > cap and balance:
            if cur is not None:
                units.append((cur[0], cur[1], cur[2], cur[3], NO_SPLIT, 0, 1, 0))
                cur = None
            nseg = -(-nb // cap)
            for k in range(nseg):
                s0 = int(rwo[w]) + (k * nb) // nseg
                s1 = int(rwo[w]) + ((k + 1) * nb) // nseg
                units.append((w, 1, s0, s1, split_id, k, nseg, slot + k))
            split_id += 1
            slot += nseg
        else:
            c = nb + wb
            if cur is not None and cur[1] < WMAX and cur[4] + c <= (group_cap or cap) + wb:
                cur[1] += 1
                cur[3] = int(rwo[w + 1])
                cur[4] += c
            else:
                if cur is not None:
                    units.append((cur[0], cur[1], cur[2], cur[3], NO_SPLIT, 0, 1, 0))
                cur = [w, 1, int(rwo[w]), int(rwo[w + 1]), c]
    if cur is not None:
        units.append((cur[0], cur[1], cur[2], cur[3], NO_SPLIT, 0, 1, 0))
    return units


def check_coverage(units, rwo) -> None:
    """Every TC block covered exactly once; windows covered in order; segments contiguous."""
    rwo = np.asarray(rwo, dtype=np.int64)
    W = rwo.size - 1
    nextb = 0
    nextw = 0
    for (w0, nw, b0, b1, split, seg, nseg, slot) in units:
        assert b0 == nextb, "blocks not contiguous"
        if split == NO_SPLIT:
            assert w0 == nextw and b0 == rwo[w0] and b1 == rwo[w0 + nw]
            nextw = w0 + nw
        else:
            assert nw == 1 and rwo[w0] <= b0 < b1 <= rwo[w0 + 1]
            if seg == nseg - 1:
                assert b1 == rwo[w0 + 1]
                nextw = w0 + 1
        nextb = b1
    assert nextb == rwo[-1] and nextw == W


def unit_times(units, rwo, profile="A800", feature_dim=128):
    """Literal Eq. (4) time per unit (one segment per window in the unit)."""
    return [eq4_time(profile, feature_dim, b1 - b0) for (_, _, b0, b1, *_rest) in units]


def mean_ratio(times) -> float:
    t = np.asarray(times, dtype=np.float64)
    return float(t.max() / t.mean()) if t.size else 0.0


__all__ = ["ibd", "eq4_time", "build_units", "auto_cap", "check_coverage", "PROFILES",
           "IBD_THRESHOLD", "PAPER_CAP", "WMAX", "NO_SPLIT", "math"]
