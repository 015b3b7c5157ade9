"""GPU parity of the pre-rounded-B path: with high B-row reuse (sum_w|U_w| >= 32 K) rho(B) is
applied once per execute by a pre-pass and the kernel gathers the rounded rows.
Every fixture here has high reuse; integer data must be bit-exact, floats within tau, and the
RNA carries / ties of rho must survive the gather bit for bit.  (The variants build's 3-byte
image of the rounded B, "B3", is covered by tests/_variants_worker.py.)
"""
import numpy as np
import pytest

import gen
from gpu_util import assert_bit_exact, assert_within, run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()


def _high_reuse(seed=0, M=4003, K=211, nnz=80000):
    A = gen.uniform_random(M, K, nnz, seed=seed)
    return A


def test_fixture_has_high_reuse():
    A = _high_reuse()
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 128, 2)
    _, p = run(A, v, B, "tf32")
    assert p.info["sum_U"] >= 32 * A.K


@pytest.mark.parametrize("N", [16, 32, 64, 128, 192, 256, 384, 1152])
def test_prepass_integer_bit_exact(N):
    A = _high_reuse(seed=N)
    v = gen.values_int(A.nnz, 3)
    B = gen.dense_int(A.K, N, 4)
    for kw in ({}, {"balance": "on", "unit_cap": 32}, {"reorder": "on"}):
        C, p = run(A, v, B, "tf32", **kw)
        assert_bit_exact(C, A, v, B, "tf32")


@pytest.mark.parametrize("N", [64, 128, 256])
def test_prepass_float_within_tolerance(N):
    A = _high_reuse(seed=7 + N)
    v = gen.values_uniform(A.nnz, 5)
    B = gen.dense_normal(A.K, N, 6)
    C, _ = run(A, v, B, "tf32")
    assert_within(C, A, v, B, "tf32")


def test_prepass_rho_b_bits_survive():
    """A = 8-row selector pattern with unit values: C rows are rho(B) rows bit for bit, over B
    values spanning the exponent range (tiny normals to 1e38) and both signs, with mantissa bits
    that exercise the RNA carry into bits 15..8 and into the exponent."""
    K = 64
    A = gen.csr_from_pairs(np.arange(4096), np.arange(4096) % K, 4096, K)
    v = np.ones(A.nnz, np.float32)
    rng = np.random.default_rng(11)
    mant = rng.integers(0, 1 << 23, size=(K, 128), dtype=np.uint32)
    mant[:, :8] = 0x7FF000 | np.arange(8, dtype=np.uint32)[None, :]      # RNA carries into the exponent
    mant[:, 8:16] = 0x000FFF                                             # just below a tie
    mant[:, 16:24] = 0x001000                                            # exact ties (round away)
    expo = rng.integers(2, 253, size=(K, 128), dtype=np.uint32)
    sign = rng.integers(0, 2, size=(K, 128), dtype=np.uint32)
    B = ((sign << 31) | (expo << 23) | mant).view(np.float32)
    C, p = run(A, v, B, "tf32")
    assert p.info["sum_U"] >= 32 * K
    assert_bit_exact(C, A, v, B, "tf32")


def test_prepass_permute_cols_and_split_windows():
    A = _high_reuse(seed=21, M=2048, K=2048, nnz=200000)
    v = gen.values_int(A.nnz, 8)
    B = gen.dense_int(A.K, 128, 9)
    C, p = run(A, v, B, "tf32", reorder="on", permute_cols=True, balance="on", unit_cap=32)
    assert p.info["sum_U"] >= 32 * A.K
    assert_bit_exact(C, A, v, B, "tf32")
