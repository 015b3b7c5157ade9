"""Pins for the FP64 SpMM oracle (oracle/spmm_oracle.c) -- P:650, SURVEY §8(c) C-2."""
import numpy as np
import pytest

import gen
from oracle import spmm as osp
from oracle.rounding import rho


def _dense(A: gen.Csr, vals):
    D = np.zeros((A.M, A.K), dtype=np.float64)
    D[A.row_ids(), A.colidx] = vals
    return D


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
def test_matches_dense_gemm_brute_force(precision):
    A = gen.uniform_random(512, 512, 5120, seed=1)
    a = rho(gen.values_uniform(A.nnz, 2), precision)
    B = rho(gen.dense_normal(512, 16, 3), precision)
    C, S = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, B)
    ref = _dense(A, a.astype(np.float64)) @ B.astype(np.float64)
    assert np.all(np.abs(C - ref) <= 1e-12 * S + 1e-300)
    Sref = np.abs(_dense(A, a.astype(np.float64))) @ np.abs(B.astype(np.float64))
    assert np.allclose(S, Sref, rtol=1e-12, atol=0)


def test_spec_examples():
    # S:86 identity A -> C == B exactly
    I = gen.identity(6)
    B = gen.dense_normal(6, 4, 0)
    C, _ = osp.spmm_fp64(6, 6, I.rowptr, I.colidx, np.ones(6, np.float32), B)
    assert np.array_equal(C, B.astype(np.float64))
    # S:87 zero A -> all zeros
    Z = gen.Csr(4, 4, np.zeros(5, np.int64), np.zeros(0, np.int32))
    C, _ = osp.spmm_fp64(4, 4, Z.rowptr, Z.colidx, np.zeros(0, np.float32), np.ones((4, 2), np.float32))
    assert np.array_equal(C, np.zeros((4, 2)))
    # S:88 single entry (1,2) = 3, B = ones(4x2) -> row 1 = [3, 3], others 0
    E = gen.csr_from_pairs([1], [2], 4, 4)
    C, _ = osp.spmm_fp64(4, 4, E.rowptr, E.colidx, np.float32([3.0]), np.ones((4, 2), np.float32))
    assert C.tolist() == [[0, 0], [3, 3], [0, 0], [0, 0]]


def test_integer_inputs_exact():
    A = gen.uniform_random(200, 150, 3000, seed=5)
    a = gen.values_int(A.nnz, 6)
    B = gen.dense_int(150, 8, 7)
    C, _ = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, B)
    # exact brute force with Python integers
    ai = a.astype(np.int64)
    Bi = B.astype(np.int64)
    ref = np.zeros((A.M, 8), dtype=np.int64)
    for i in range(A.M):
        for p in range(A.rowptr[i], A.rowptr[i + 1]):
            ref[i] += ai[p] * Bi[A.colidx[p]]
    assert np.array_equal(C, ref.astype(np.float64))


def test_row_subset_and_thread_independence():
    A = gen.uniform_random(300, 300, 4000, seed=8)
    a = rho(gen.values_uniform(A.nnz, 9), "tf32")
    B = rho(gen.dense_normal(300, 32, 10), "tf32")
    C1, S1 = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, B, nthreads=1)
    C8, S8 = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, B, nthreads=8)
    assert np.array_equal(C1, C8) and np.array_equal(S1, S8)
    rows = np.array([299, 0, 17, 17, 150])
    Cr, Sr = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, B, rows=rows)
    assert np.array_equal(Cr, C1[rows]) and np.array_equal(Sr, S1[rows])


def test_dimension_mismatch_and_bad_index():
    A = gen.identity(4)
    with pytest.raises(ValueError):
        osp.spmm_fp64(4, 4, A.rowptr, A.colidx, np.ones(4, np.float32), np.ones((5, 2), np.float32))
    bad = np.array([0, 1, 2, 3], np.int32)
    bad[2] = 9
    with pytest.raises(ValueError):
        osp.spmm_fp64(4, 4, A.rowptr, bad, np.ones(4, np.float32), np.ones((4, 2), np.float32))


def test_check_detects_violations():
    C_ref = np.array([[1.0, 2.0]])
    S = np.array([[1.0, 2.0]])
    assert osp.check(C_ref + 0.5e-3, C_ref, S, "tf32")["ok"]
    assert not osp.check(C_ref + 2e-3, C_ref, S, "tf32")["ok"]
    assert not osp.check(np.array([[np.nan, 2.0]]), C_ref, S, "tf32")["ok"]
    assert osp.check(C_ref + 3e-3, C_ref, S, "fp16")["ok"]
