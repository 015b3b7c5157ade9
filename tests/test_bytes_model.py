"""Pins the roofline accounting (bench.py `roofline.achieved`) to SURVEY §8(d)'s per-unit
algorithmic bytes, recomputed here from the oracle's BitTCF encoding -- not from the library."""
import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from oracle import bittcf as bt


@pytest.mark.parametrize("precision,N", [("tf32", 128), ("fp16", 64), ("tf32", 32)])
def test_bytes_model_matches_per_unit_figures(precision, N):
    A = gen.dcsbm(2000, 80_000, 5, 2.2, 0.2, 1500, seed=2, oversample=1.3)
    v = gen.values_uniform(A.nnz, 1)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, device=-1, reorder="off")
    F = bt.encode(A.M, A.K, A.rowptr, A.colidx)
    es = 2 if precision == "fp16" else 4
    W, NB, nnz = F["W"], F["NB"], A.nnz
    # per nnz: es_A bytes of value; per TC block: 8 B mask + 32 B SparseAToB + 4 B TCOffset
    # + es_B*N per valid lane; per window: 4 B RowWindowOffset + 8 rows*N*4 B of C (ragged: M rows)
    valid_lanes = int(F["U"].sum())
    expect_A = es * nnz + NB * (8 + 32 + 4) + 4 + 4 * (W + 1) + 32 * p.info["n_units"]
    expect_B = es * N * valid_lanes
    expect_C = 4 * A.M * N
    bm = acc.bytes_model(p.info, N)
    assert bm["B_model"] == expect_B
    assert bm["C"] == expect_C
    assert bm["A_fmt"] == expect_A
    assert bm["flops"] == 2 * nnz * N
