"""Pins for the reference BitTCF encoder/decoder (oracle/bittcf.py) -- P:250-273."""
import json
import os

import numpy as np
import pytest

import gen
from oracle import bittcf as bt

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _enc(A, vals=None):
    return bt.encode(A.M, A.K, A.rowptr, A.colidx, vals)


def _brute_encode(A):
    """Pure-Python, window-by-window encoder (small inputs) for cross-checking the vectorised one."""
    W = (A.M + 7) // 8
    rwo, tco, a2b, bits = [0], [0], [], []
    for w in range(W):
        rows = range(8 * w, min(8 * w + 8, A.M))
        U = sorted({int(A.colidx[p]) for i in rows for p in range(A.rowptr[i], A.rowptr[i + 1])})
        nb = (len(U) + 7) // 8
        for t in range(nb):
            lanes = U[8 * t:8 * t + 8]
            a2b += lanes + [0] * (8 - len(lanes))
            m = 0
            for i in rows:
                for p in range(A.rowptr[i], A.rowptr[i + 1]):
                    c = int(A.colidx[p])
                    if c in lanes:
                        m |= 1 << ((i - 8 * w) * 8 + lanes.index(c))
            bits.append(m)
            tco.append(tco[-1] + bin(m).count("1"))
        rwo.append(rwo[-1] + nb)
    return rwo, tco, a2b, bits


def test_golden_fixtures():
    with open(os.path.join(GOLDEN, "bittcf_fixtures.json")) as f:
        fx = json.load(f)
    for case in fx["cases"]:
        A = gen.csr_from_pairs(case["rows"], case["cols"], case["M"], case["K"])
        F = _enc(A)
        assert F["RowWindowOffset"].tolist() == case["RowWindowOffset"], case["name"]
        assert F["TCOffset"].tolist() == case["TCOffset"], case["name"]
        assert F["SparseAToB"].tolist() == case["SparseAToB"], case["name"]
        assert [int(x) for x in F["TCLocalBit"]] == [int(x, 16) for x in case["TCLocalBit"]], case["name"]
        assert bt.bittcf_index_bytes(case["M"], F["NB"]) == case["index_bytes"], case["name"]


def test_byte_formula_worked_values():
    # substitution into P:253
    assert bt.bittcf_index_bytes(8, 1) == 56
    assert bt.bittcf_index_bytes(16, 3) == 148
    assert bt.bittcf_index_bytes(8, 0) == 12
    # S:309-312 ME-TCF: tie at 8 nnz, BitTCF wins at 64, ME-TCF wins at 1
    assert bt.metcf_index_bytes(8, 1, 8) == 56
    assert bt.metcf_index_bytes(8, 1, 64) == 112
    assert bt.metcf_index_bytes(8, 1, 1) == 49


def test_single_bit_probes_pin_bit_order():
    """64 probes: target nnz at (r, lane c); lanes 0..c-1 filled in row r'=(r+1)%8 (SURVEY C-4 a8(ii))."""
    for r in range(8):
        for c in range(8):
            rp = (r + 1) % 8
            rows = [rp] * c + [r]
            cols = list(range(c)) + [c]
            A = gen.csr_from_pairs(rows, cols, 8, 8)
            F = _enc(A)
            expect = (((1 << c) - 1) << (8 * rp)) | (1 << (8 * r + c))
            assert int(F["TCLocalBit"][0]) == expect


def test_value_order_and_decode_offset():
    # mask bits {0,5,9} -> offset of bit 9 = 2
    assert bt.value_index((1 << 0) | (1 << 5) | (1 << 9), 9) == 2
    A = gen.csr_from_pairs([0, 0, 1], [10, 20, 10], 8, 32)
    F = _enc(A, np.float32([1.0, 2.0, 3.0]))
    # bits: (r0,l0)=0, (r0,l1)=1, (r1,l0)=8 -> values ascending by bit
    assert int(F["TCLocalBit"][0]) == 0x103
    assert F["values"].tolist() == [1.0, 2.0, 3.0]


@pytest.mark.parametrize("seed", range(200))
def test_roundtrip_random(seed):
    """S:568 acceptance 1: decode(encode(A)) == A bit-exactly on 200 random matrices."""
    rng = np.random.default_rng(1000 + seed)
    M = int(rng.integers(1, 513))
    K = int(rng.integers(1, 513))
    dens = float(10 ** rng.uniform(-3, np.log10(0.3)))
    nnz = max(0, min(M * K, int(dens * M * K)))
    A = gen.uniform_random(M, K, nnz, seed=seed)
    v = gen.values_uniform(A.nnz, seed)
    F = _enc(A, v)
    rp, ci, vv = bt.decode(F)
    assert np.array_equal(rp, A.rowptr) and np.array_equal(ci, A.colidx) and np.array_equal(vv, v)
    # invariants S:275
    tco = F["TCOffset"].astype(np.int64)
    assert np.array_equal(np.diff(tco), np.bitwise_count(F["TCLocalBit"]).astype(np.int64))
    assert int(tco[-1]) == A.nnz
    assert bt.array_bytes(F) == bt.bittcf_index_bytes(M, F["NB"])
    assert bt.bittcf_index_bytes(M, F["NB"]) - bt.metcf_index_bytes(M, F["NB"], A.nnz) == 8 * F["NB"] - A.nnz
    # padding lanes never carry bits
    lanes_used = np.zeros((F["NB"], 8), bool)
    for k in range(64):
        lanes_used[:, k % 8] |= ((F["TCLocalBit"] >> np.uint64(k)) & np.uint64(1)).astype(bool)
    U = F["U"]
    valid = np.zeros((F["NB"], 8), bool)
    b = 0
    for u in U:
        for t in range((int(u) + 7) // 8):
            valid[b, :min(8, int(u) - 8 * t)] = True
            b += 1
    assert np.array_equal(lanes_used, valid)


@pytest.mark.parametrize("seed", range(20))
def test_vectorised_equals_brute_force(seed):
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 70)), int(rng.integers(1, 90))
    A = gen.uniform_random(M, K, int(rng.integers(0, M * K // 3 + 1)), seed=seed)
    F = _enc(A)
    rwo, tco, a2b, bits = _brute_encode(A)
    assert F["RowWindowOffset"].tolist() == rwo and F["TCOffset"].tolist() == tco
    assert F["SparseAToB"].tolist() == a2b and [int(x) for x in F["TCLocalBit"]] == bits


def test_mean_nnz_tc():
    dense = gen.csr_from_pairs(np.repeat(np.arange(8), 8), np.tile(np.arange(8), 8), 8, 8)
    assert bt.mean_nnz_tc(_enc(dense)) == 64.0
    assert bt.mean_nnz_tc(_enc(gen.identity(16))) == 8.0


def test_empty_and_ragged():
    E = gen.Csr(13, 9, np.zeros(14, np.int64), np.zeros(0, np.int32))
    F = _enc(E)
    assert F["NB"] == 0 and F["RowWindowOffset"].tolist() == [0, 0, 0]
    assert bt.decode(F)[0].tolist() == [0] * 14
    R = gen.csr_from_pairs([12, 12], [0, 8], 13, 9)   # last window holds only rows 8..12
    F = _enc(R)
    assert F["RowWindowOffset"].tolist() == [0, 0, 1]
    assert int(F["TCLocalBit"][0]) == (1 << 32) | (1 << 33)


def test_permute_rows():
    A = gen.uniform_random(40, 30, 200, seed=3)
    v = gen.values_uniform(A.nnz, 4)
    perm = np.random.default_rng(5).permutation(40)
    rp, ci, vv = bt.permute_rows(40, A.rowptr, A.colidx, v, perm)
    for r in range(40):
        o = perm[r]
        assert np.array_equal(ci[rp[r]:rp[r + 1]], A.colidx[A.rowptr[o]:A.rowptr[o + 1]])
        assert np.array_equal(vv[rp[r]:rp[r + 1]], v[A.rowptr[o]:A.rowptr[o + 1]])


# ----------------------------------------------------------------------- tall windows (R20)

def _brute_encode_tall(A, wh):
    """Per-window dense construction for windows of wh rows, written independently of
    bt.encode: dense 0/1 tile of the window, condensed columns, wh/8 words per block with the
    paper's bit rule inside each 8-row word, values in row-major tile order."""
    nw = wh // 8
    dense = np.zeros((A.M, A.K), bool)
    val = np.zeros((A.M, A.K))
    for r in range(A.M):
        for p in range(A.rowptr[r], A.rowptr[r + 1]):
            dense[r, A.colidx[p]] = True
            val[r, A.colidx[p]] = p + 1.0          # value = 1 + CSR position (identifies the nnz)
    rwo, tco, a2b, bits, vals = [0], [0], [], [], []
    for w0 in range(0, A.M, wh):
        win = dense[w0:w0 + wh]
        cols = [c for c in range(A.K) if win[:, c].any()]
        for t in range(0, len(cols), 8):
            lane_cols = cols[t:t + 8]
            a2b += lane_cols + [0] * (8 - len(lane_cols))
            words = [0] * nw
            for r in range(win.shape[0]):
                for l, c in enumerate(lane_cols):
                    if win[r, c]:
                        words[r // 8] |= 1 << ((r % 8) * 8 + l)
                        vals.append(val[w0 + r, c])
            bits += words
            tco.append(len(vals))
        rwo.append(len(tco) - 1)
    return rwo, tco, a2b, bits, vals


@pytest.mark.parametrize("wh", [16, 32])
@pytest.mark.parametrize("seed", range(12))
def test_tall_windows_vectorised_equals_brute_force(wh, seed):
    rng = np.random.default_rng(100 + seed)
    M, K = int(rng.integers(1, 90)), int(rng.integers(1, 70))
    A = gen.uniform_random(M, K, int(rng.integers(0, M * K // 3 + 1)), seed=seed)
    v = np.arange(1, A.nnz + 1, dtype=np.float64)
    F = bt.encode(A.M, A.K, A.rowptr, A.colidx, v, wh=wh)
    rwo, tco, a2b, bits, vals = _brute_encode_tall(A, wh)
    assert F["RowWindowOffset"].tolist() == rwo and F["TCOffset"].tolist() == tco
    assert F["SparseAToB"].tolist() == a2b and [int(x) for x in F["TCLocalBit"]] == bits
    assert F["values"].tolist() == vals


@pytest.mark.parametrize("wh", [16, 32])
@pytest.mark.parametrize("seed", range(8))
def test_tall_windows_roundtrip_and_invariants(wh, seed):
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 300)), int(rng.integers(1, 200))
    A = gen.uniform_random(M, K, int(rng.integers(0, M * K // 4 + 1)), seed=seed)
    v = gen.values_uniform(A.nnz, seed)
    F = bt.encode(A.M, A.K, A.rowptr, A.colidx, v, wh=wh)
    rp, ci, vv = bt.decode(F)                                   # S:324 round trip
    assert np.array_equal(rp, A.rowptr) and np.array_equal(ci, A.colidx) and np.array_equal(vv, v)
    words = F["TCLocalBit"].reshape(-1, wh // 8)
    assert np.array_equal(np.diff(F["TCOffset"].astype(np.int64)), np.bitwise_count(words).sum(axis=1))
    assert F["W"] == (M + wh - 1) // wh and F["NB"] == int(((F["U"] + 7) // 8).sum())
    # a tall window's condensed columns are the union of its 8-row windows' (P:250 per 8 rows)
    F8 = bt.encode(A.M, A.K, A.rowptr, A.colidx, wh=8)
    for w in range(F["W"]):
        cols = set(F["SparseAToB"][8 * F["RowWindowOffset"][w]: 8 * F["RowWindowOffset"][w + 1]][
            : F["U"][w]].tolist())
        sub = set()
        for w8 in range(w * wh // 8, min(F8["W"], (w + 1) * wh // 8)):
            sub |= set(F8["SparseAToB"][8 * F8["RowWindowOffset"][w8]: 8 * F8["RowWindowOffset"][w8 + 1]][
                : F8["U"][w8]].tolist())
        assert cols == sub


def test_tall_window_worked_example():
    """Hand-derived 16-row window: row 0 has columns {3, 5}, row 9 has {5, 7}.  Condensed
    columns [3, 5, 7] -> one block, SparseAToB [3, 5, 7, 0, 0, 0, 0, 0]; word 0 (rows 0-7): row 0
    lanes 0, 1 -> 0x3; word 1 (rows 8-15): row 9 is local row 1 there, lanes 1, 2 -> bits 9, 10
    -> 0x600; values in tile order (0,3) (0,5) (9,5) (9,7); the value of (9,7) sits at
    TCOffset + popc(word 0) + popc(word 1 below bit 10) = 0 + 2 + 1 = 3 (P:273 over the words)."""
    A = gen.csr_from_pairs(np.array([0, 0, 9, 9]), np.array([3, 5, 5, 7]), 16, 8)
    v = np.array([10.0, 20.0, 30.0, 40.0])
    F = bt.encode(A.M, A.K, A.rowptr, A.colidx, v, wh=16)
    assert F["NB"] == 1 and F["RowWindowOffset"].tolist() == [0, 1] and F["TCOffset"].tolist() == [0, 4]
    assert F["SparseAToB"].tolist() == [3, 5, 7, 0, 0, 0, 0, 0]
    assert [int(x) for x in F["TCLocalBit"]] == [0x3, 0x600]
    assert F["values"].tolist() == [10.0, 20.0, 30.0, 40.0]
    with pytest.raises(ValueError):
        bt.encode(A.M, A.K, A.rowptr, A.colidx, v, wh=24)
