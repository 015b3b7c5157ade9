"""CPU tests of libaccspmm through its C ABI (host-only plans, device = -1): symbols,
error paths, and BitTCF / schedule / partition / reorder bit-exact against the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from oracle import balance as ob
from oracle import bittcf as bt
from oracle import partition as op
from oracle import reorder as orr
from oracle.rounding import fp16_rne, tf32_rna

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2501_09251_b200 import _build
    _build.build()


def host_plan(A, vals, **kw):
    kw.setdefault("device", -1)
    kw.setdefault("reorder", "off")   # fixtures pin the un-reordered format unless they ask
    return acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, **kw)


def test_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "accspmm.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(accspmm_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(acc.EXPORTED)
    lib = ctypes.CDLL(acc.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert acc.accspmm_abi_version() == 1


def test_status_strings():
    assert acc.accspmm_status_string(0) == "ACCSPMM_OK"
    assert acc.accspmm_status_string(2) == "ACCSPMM_ERR_INVALID_CSR"


@pytest.mark.parametrize("case", ["unsorted", "duplicate", "range", "rowptr", "rowptr0"])
def test_invalid_csr_rejected(case):
    rowptr = np.array([0, 2, 3], np.int64)
    colidx = np.array([1, 3, 0], np.int32)
    if case == "unsorted":
        colidx = np.array([3, 1, 0], np.int32)
    elif case == "duplicate":
        colidx = np.array([1, 1, 0], np.int32)
    elif case == "range":
        colidx = np.array([1, 9, 0], np.int32)
    elif case == "rowptr":
        rowptr = np.array([0, 3, 2], np.int64)
    elif case == "rowptr0":
        rowptr = np.array([1, 2, 3], np.int64)
    opt = acc.accspmm_options_default()
    opt.device = -1
    with pytest.raises(acc.AccSpmmError) as ei:
        acc.accspmm_plan_create_ex(2, 4, rowptr, colidx, np.ones(3, np.float32), opt)
    assert ei.value.status == 2


def test_bad_options_and_host_only_execute():
    A = gen.identity(8)
    opt = acc.accspmm_options_default()
    opt.device = -1
    opt.nparts, opt.part = 2, 2
    with pytest.raises(acc.AccSpmmError) as ei:
        acc.accspmm_plan_create_ex(8, 8, A.rowptr, A.colidx, np.ones(8, np.float32), opt)
    assert ei.value.status == 1
    p = host_plan(A, np.ones(8, np.float32))
    with pytest.raises(acc.AccSpmmError) as ei:   # no CPU fallback: host-only plans cannot execute
        acc.accspmm_execute(p.handle, 16, 16, 16)
    assert ei.value.status == 3


@pytest.mark.parametrize("args", [(0, 1, 0), (1 << 20, 0, 0), (1 << 20, 1, 3), (1 << 20, 1, -1)])
def test_l2_probe_rejects_bad_arguments(args):
    """The measurement hook validates before touching the device (header: bytes >= 1 MiB,
    iters >= 1, mode 0/1/2)."""
    with pytest.raises(acc.AccSpmmError) as ei:
        acc.accspmm_probe_l2_bandwidth_ex(*args)
    assert ei.value.status == 1


def _check_format(F, ref, precision):
    assert np.array_equal(F["RowWindowOffset"], ref["RowWindowOffset"])
    assert np.array_equal(F["TCOffset"], ref["TCOffset"])
    assert np.array_equal(F["SparseAToB"], ref["SparseAToB"])
    assert np.array_equal(F["TCLocalBit"], ref["TCLocalBit"])
    if precision == "tf32":
        assert np.array_equal(F["values"].view(np.uint32), ref["values"].view(np.uint32))
    else:
        assert np.array_equal(F["values"].view(np.uint16), ref["values"].view(np.uint16))


def _rho_vals(v, precision):
    return tf32_rna(v) if precision == "tf32" else fp16_rne(v)


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("seed", range(30))
def test_format_bit_exact_vs_oracle(seed, precision):
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 700)), int(rng.integers(1, 700))
    dens = float(10 ** rng.uniform(-3, np.log10(0.2)))
    A = gen.uniform_random(M, K, int(dens * M * K), seed=seed)
    v = gen.values_uniform(A.nnz, seed + 1)
    p = host_plan(A, v, precision=precision)
    ref = bt.encode(A.M, A.K, A.rowptr, A.colidx, _rho_vals(v, precision))
    _check_format(p.export_format(), ref, precision)
    I = p.info
    assert I["NB"] == ref["NB"] and I["W"] == ref["W"] and I["sum_U"] == int(ref["U"].sum())
    assert I["index_bytes"] == bt.bittcf_index_bytes(M, ref["NB"])
    assert I["metcf_index_bytes"] == bt.metcf_index_bytes(M, ref["NB"], A.nnz)
    assert I["mean_nnz_tc"] == pytest.approx(bt.mean_nnz_tc(ref), rel=1e-12)


def test_golden_fixtures_through_library():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "bittcf_fixtures.json")) as f:
        fx = json.load(f)
    for case in fx["cases"]:
        A = gen.csr_from_pairs(case["rows"], case["cols"], case["M"], case["K"])
        F = host_plan(A, np.ones(A.nnz, np.float32)).export_format()
        assert F["RowWindowOffset"].tolist() == case["RowWindowOffset"], case["name"]
        assert F["TCOffset"].tolist() == case["TCOffset"], case["name"]
        assert F["SparseAToB"].tolist() == case["SparseAToB"], case["name"]
        assert [int(x) for x in F["TCLocalBit"]] == [int(x, 16) for x in case["TCLocalBit"]], case["name"]


def test_empty_matrices():
    for M, K in [(0, 0), (0, 5), (13, 9)]:
        A = gen.Csr(M, K, np.zeros(M + 1, np.int64), np.zeros(0, np.int32))
        p = host_plan(A, np.zeros(0, np.float32))
        assert p.info["NB"] == 0 and p.info["W"] == (M + 7) // 8
        u = p.export_units()
        assert u.shape[0] == (0 if M == 0 else 1)  # AUTO groups the empty windows into one unit
        ob.check_coverage([tuple(int(x) for x in r) for r in u], np.zeros(p.info["W"] + 1, np.int64))
        off = host_plan(A, np.zeros(0, np.float32), balance="off")
        assert off.export_units().shape[0] == p.info["W"]


@pytest.mark.parametrize("balance", ["off", "on", "auto"])
@pytest.mark.parametrize("cap", [0, 32, 100])
@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("shape", ["powerlaw", "road"])
def test_schedule_bit_exact_vs_oracle(balance, cap, precision, shape):
    """Units equal the oracle's, for a high-IBD graph (AUTO balances) and a low-IBD road grid
    (AUTO keeps windows whole but groups them, reading R7b)."""
    if shape == "powerlaw":
        A = gen.dcsbm(4000, 160_000, 7, 2.3, 0.25, 2500, seed=11, oversample=1.3)
    else:
        A = gen.road_grid(120, 0.7, seed=2)
    p = host_plan(A, gen.values_uniform(A.nnz, 1), balance=balance, unit_cap=cap, precision=precision)
    I = p.info
    F = p.export_format()
    rwo = F["RowWindowOffset"].astype(np.int64)
    ibd = ob.ibd(np.diff(rwo))
    assert I["ibd"] == pytest.approx(ibd, rel=1e-12)
    on = balance == "on" or (balance == "auto" and ibd > ob.IBD_THRESHOLD)
    assert I["balanced"] == int(on)
    expect_cap = cap if cap > 0 else ob.auto_cap(I["NB"])
    assert I["unit_cap"] == expect_cap
    group = balance == "auto" and not on
    assert I["grouped"] == int(group)
    if shape == "road":
        assert not on or balance == "on"
    expect_gcap = expect_cap if (cap > 0 or on) else ob.auto_group_cap(expect_cap)
    assert I["group_cap"] == expect_gcap
    ref = np.array(ob.build_units(rwo, expect_cap, on, precision, group=group, group_cap=expect_gcap),
                   dtype=np.uint64).astype(np.uint32)
    got = p.export_units()
    assert got.shape == ref.shape and np.array_equal(got, ref)
    ob.check_coverage([tuple(int(x) for x in u) for u in got], rwo)
    assert I["n_split_windows"] == len({int(u[4]) for u in got if u[4] != ob.NO_SPLIT})


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partition_bounds_and_slabs(P):
    A = gen.dcsbm(3000, 60_000, 5, 2.2, 0.2, 1500, seed=3, oversample=1.3)
    v = gen.values_uniform(A.nnz, 2)
    b = acc.accspmm_partition_bounds(A.M, A.rowptr, P)
    assert b.tolist() == op.bounds(A.M, A.rowptr, P)
    rows = []
    for k in range(P):
        p = host_plan(A, v, part=k, nparts=P)
        I = p.info
        assert I["window_begin"] == b[k] and I["row_begin"] == 8 * b[k]
        r0, r1 = 8 * b[k], min(A.M, 8 * b[k + 1])
        assert I["rows"] == max(0, r1 - r0)
        sub_ptr = A.rowptr[r0:r1 + 1] - A.rowptr[r0] if r1 > r0 else np.zeros(1, np.int64)
        sub_col = A.colidx[A.rowptr[r0]:A.rowptr[r1]] if r1 > r0 else np.zeros(0, np.int32)
        ref = bt.encode(max(0, r1 - r0), A.K, sub_ptr, sub_col, tf32_rna(v[A.rowptr[r0]:A.rowptr[max(r0, r1)]]))
        _check_format(p.export_format(), ref, "tf32")
        rows.append(p.export_rows())
    assert np.array_equal(np.concatenate(rows), np.arange(A.M, dtype=np.uint32))


def _graphs():
    out = []
    for seed in range(6):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(20, 200))
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < 0.05
        out.append(gen.csr_from_pairs(iu[keep], ju[keep], n, n, symmetric=True))
    out.append(gen.sbm(256, 8, 0.3, 0.01, seed=1))
    out.append(gen.two_cliques(6, seed=2))
    out.append(gen.star(9))
    out.append(gen.uniform_random(150, 150, 900, seed=4))   # asymmetric pattern
    out.append(gen.identity(10))
    return out


@pytest.mark.parametrize("idx", range(11))
def test_reorder_matches_oracle_algorithm1(idx):
    """No community list outgrows the R6b cap on these graphs: the library equals the literal
    Alg. 1 of the oracle, and the oracle's bounded variant is a no-op there."""
    A = _graphs()[idx]
    got = acc.accspmm_reorder(A.M, A.rowptr, A.colidx)
    st = {}
    ref = orr.reorder(A.M, A.K, A.rowptr, A.colidx)
    assert np.array_equal(orr.reorder(A.M, A.K, A.rowptr, A.colidx, edge_cap=orr.EDGE_CAP, stats=st), ref)
    assert st.get("truncations", 0) == 0
    assert np.array_equal(got.astype(np.int64), ref)


def _shuffled(A, seed):
    """Symmetric relabelling P A P^T (random P): hides any structure the ids carry."""
    n = A.M
    lab = np.random.default_rng(seed).permutation(n)
    r = lab[A.row_ids()]
    c = lab[A.colidx.astype(np.int64)]
    return gen.csr_from_pairs(r, c, n, n)


@pytest.mark.parametrize("nx", [14, 16])
def test_reorder_edge_cap_branch_matches_oracle(nx):
    """Reading R6b: a community carries on only its 256 heaviest community
    edges after a visit.  On 27-point stencils of 14^3 / 16^3 vertices a community list
    outgrows 256 (the branch triggers 1 / 3 times and changes the ordering against the literal
    Alg. 1), and the library's permutation equals the oracle's bounded variant exactly."""
    A = gen.stencil27(nx)
    st = {}
    ref = orr.reorder(A.M, A.K, A.rowptr, A.colidx, edge_cap=orr.EDGE_CAP, stats=st)
    assert st["truncations"] >= 1
    assert not np.array_equal(ref, orr.reorder(A.M, A.K, A.rowptr, A.colidx))   # the branch matters
    got = acc.accspmm_reorder(A.M, A.rowptr, A.colidx).astype(np.int64)
    assert np.array_equal(got, ref)


def test_reorder_edge_cap_invariants_on_large_graph():
    """Where R6b triggers, the bounded reordering is still a valid Alg. 1 ordering (the
    invariants S:194-199 / S:572 pin both variants): a bijection, deterministic, a shuffled
    stencil (18^3) plus a shuffled two-clique component keeps each clique contiguous, and the
    TC-block count of the reordered shuffled stencil drops below the shuffled one."""
    from oracle import bittcf as bt
    S = _shuffled(gen.stencil27(18), 1)
    k = 12
    T = gen.two_cliques(k, seed=4)
    n = S.M + T.M
    r = np.concatenate([S.row_ids(), T.row_ids() + S.M])
    c = np.concatenate([S.colidx.astype(np.int64), T.colidx.astype(np.int64) + S.M])
    A = gen.csr_from_pairs(r, c, n, n)
    lab = np.random.default_rng(4).permutation(2 * k)   # two_cliques(seed=4) labelling
    clique_of = {S.M + int(lab[i]): (0 if i < k else 1) for i in range(2 * k)}
    for cap in (None, orr.EDGE_CAP):
        st = {}
        perm = orr.reorder(A.M, A.K, A.rowptr, A.colidx, edge_cap=cap, stats=st)
        assert sorted(perm.tolist()) == list(range(n))
        assert np.array_equal(perm, orr.reorder(A.M, A.K, A.rowptr, A.colidx, edge_cap=cap))
        seq = [clique_of[int(v)] for v in perm if int(v) in clique_of]
        pos = [i for i, v in enumerate(perm) if int(v) in clique_of]
        first = [p for p, q in zip(pos, seq) if q == 0]
        second = [p for p, q in zip(pos, seq) if q == 1]
        assert max(first) - min(first) == k - 1 and max(second) - min(second) == k - 1
        if cap is not None:
            assert st["truncations"] >= 1
            assert np.array_equal(acc.accspmm_reorder(A.M, A.rowptr, A.colidx).astype(np.int64), perm)
    pS = orr.reorder(S.M, S.K, S.rowptr, S.colidx, edge_cap=orr.EDGE_CAP)
    inv = np.empty_like(pS)
    inv[pS] = np.arange(S.M)
    R = gen.csr_from_pairs(inv[S.row_ids()], S.colidx.astype(np.int64), S.M, S.M)
    assert bt.encode(R.M, R.K, R.rowptr, R.colidx)["NB"] < bt.encode(S.M, S.K, S.rowptr, S.colidx)["NB"]


@pytest.mark.parametrize("mode", ["on", "auto"])
def test_reordered_plan_format(mode):
    A = gen.sbm(512, 16, 0.3, 0.005, seed=5)
    v = gen.values_uniform(A.nnz, 6)
    p = host_plan(A, v, reorder=mode)
    perm = p.export_rows().astype(np.int64)
    assert sorted(perm.tolist()) == list(range(A.M))
    rp, ci, vv = bt.permute_rows(A.M, A.rowptr, A.colidx, v, perm)
    ref = bt.encode(A.M, A.K, rp, ci, tf32_rna(vv))
    _check_format(p.export_format(), ref, "tf32")
    base = bt.encode(A.M, A.K, A.rowptr, A.colidx)
    if mode == "auto":
        assert p.info["nb_unreordered"] == base["NB"]
        assert (p.info["reorder_applied"] == 1) == (ref["NB"] < base["NB"]) or p.info["reorder_applied"] == 0
    assert p.info["NB"] <= base["NB"] or mode == "on"


@pytest.mark.parametrize("shape", [(300, 170, 4000), (1, 9, 3), (40, 1, 12), (0, 5, 0), (13, 9, 0)])
def test_csr_transpose_vs_scipy(shape):
    """accspmm_csr_transpose (the backward-pass operand A^T) equals scipy's transpose exactly."""
    import scipy.sparse as sp
    M, K, nnz = shape
    A = gen.uniform_random(M, K, nnz, seed=M + K) if nnz else gen.Csr(M, K, np.zeros(M + 1, np.int64),
                                                                      np.zeros(0, np.int32))
    v = gen.values_uniform(A.nnz, 3)
    tr, tc, tv = acc.accspmm_csr_transpose(A.M, A.K, A.rowptr, A.colidx, v)
    ref = sp.csr_matrix((v, A.colidx, A.rowptr), shape=(M, K)).T.tocsr()
    ref.sort_indices()
    assert np.array_equal(tr, ref.indptr.astype(np.int64))
    assert np.array_equal(tc, ref.indices.astype(np.int32))
    assert np.array_equal(tv, ref.data.astype(np.float32))
    if A.nnz:
        t2 = acc.accspmm_csr_transpose(K, M, tr, tc, tv)
        assert np.array_equal(t2[0], A.rowptr) and np.array_equal(t2[1], A.colidx) and np.array_equal(t2[2], v)


def test_csr_transpose_rejects_invalid():
    with pytest.raises(acc.AccSpmmError) as ei:
        acc.accspmm_csr_transpose(2, 4, np.array([0, 2, 3]), np.array([3, 1, 0]), np.ones(3, np.float32))
    assert ei.value.status == 2


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("nparts", [1, 3])
def test_permute_cols_format_is_symmetric_permutation(precision, nparts):
    """permute_cols: the plan holds BitTCF of A' = P A P^T (rows and columns relabelled by the
    same Alg. 1 permutation) -- encoded independently by the oracle."""
    A = gen.dcsbm(2000, 60_000, 6, 2.2, 0.1, 800, seed=5, oversample=1.3)
    v = gen.values_uniform(A.nnz, 2)
    full = host_plan(A, v, precision=precision, reorder="on", permute_cols=True)
    assert full.info["cols_permuted"] == 1 and full.info["reorder_applied"] == 1
    perm = full.export_rows().astype(np.int64)            # new -> old
    inv = np.empty_like(perm)
    inv[perm] = np.arange(A.M)
    r, c = inv[A.row_ids()], inv[A.colidx.astype(np.int64)]
    order = np.lexsort((c, r))
    Ap = gen.csr_from_pairs(r[order], c[order], A.M, A.K)
    vp = v[order]
    rows_seen = 0
    for part in range(nparts):
        p = host_plan(A, v, precision=precision, reorder="on", permute_cols=True, part=part, nparts=nparts)
        I = p.info
        lo, hi = I["row_begin"], I["row_begin"] + I["rows"]
        sl = gen.csr_from_pairs(Ap.row_ids()[(Ap.row_ids() >= lo) & (Ap.row_ids() < hi)] - lo,
                                Ap.colidx[(Ap.row_ids() >= lo) & (Ap.row_ids() < hi)], hi - lo, A.K)
        vs = vp[(Ap.row_ids() >= lo) & (Ap.row_ids() < hi)]
        ref = bt.encode(sl.M, sl.K, sl.rowptr, sl.colidx, _rho_vals(vs, precision))
        _check_format(p.export_format(), ref, precision)
        rows_seen += I["rows"]
    assert rows_seen == A.M
    # without a permutation (reorder off) the option changes nothing
    off = host_plan(A, v, precision=precision, reorder="off", permute_cols=True)
    assert off.info["cols_permuted"] == 0


def test_sass_reads_no_unwritten_uniform_registers():
    """Guard against a ptxas (12.9) miscompile seen in this kernel: an LDGSTS whose cache-policy
    descriptor sat in a uniform register that no instruction wrote ('illegal instruction' at
    run time on large units).  Every kernel of the built library is scanned (tools/check_sass_ur.py)."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "check_sass_ur.py"), acc.LIB_PATH],
                       capture_output=True, text=True, check=True)
    assert r.stdout.strip().endswith("kernels with unwritten uniform reads: 0"), r.stdout[-2000:]


def test_binding_rejects_malformed_operands():
    """Plan.execute* check shape, dtype, layout and device before handing raw pointers to the C
    ABI (which cannot see them): a half-precision B on a TF32 plan, a transposed B or a CPU
    tensor must raise instead of reading out of bounds or computing garbage."""
    import torch
    A = gen.uniform_random(40, 24, 200, seed=1)
    v = gen.values_uniform(A.nnz, 1)
    p = host_plan(A, v)
    with pytest.raises(TypeError):
        p.execute(torch.zeros((24, 16), dtype=torch.float16))
    with pytest.raises(ValueError):
        p.execute(torch.zeros((23, 16), dtype=torch.float32))
    with pytest.raises(ValueError):
        p.execute(torch.zeros((16, 24), dtype=torch.float32).t())       # not contiguous
    with pytest.raises(ValueError):
        p.execute(torch.zeros((24,), dtype=torch.float32))              # not 2-D
    with pytest.raises(ValueError):
        p.execute(torch.zeros((24, 16), dtype=torch.float32))           # host memory
    with pytest.raises(ValueError):
        p.execute_host(np.zeros((24, 16), np.float32), np.zeros((40, 8), np.float32))
    with pytest.raises(TypeError):
        p.execute_host(np.zeros((24, 16), np.float32), np.zeros((40, 16), np.float64))
    with pytest.raises(ValueError):
        p.execute_host_batch([np.zeros((24, 16), np.float32)], [])
    ph = host_plan(A, v, precision="fp16")
    with pytest.raises(TypeError):
        ph.execute_host(np.zeros((24, 16), np.float32), np.zeros((40, 16), np.float32))


def test_default_options_follow_the_abi_contract():
    """plan_create defaults are TF32, reorder auto, balance auto."""
    opt = acc.accspmm_options_default()
    assert opt.precision == acc.TF32
    assert opt.reorder == acc.REORDER["auto"]
    assert opt.balance == acc.BALANCE["auto"]
    assert opt.nparts == 1 and opt.unit_cap == 0


def test_product_library_has_no_measurement_knobs():
    """The product library never reads ACCSPMM_* knobs (they live in libaccspmm_variants.so)."""
    import subprocess
    lib = acc.LIB_PATH
    assert lib.endswith("libaccspmm.so")
    strings = subprocess.run(["strings", lib], capture_output=True, text=True).stdout
    for knob in ("ACCSPMM_KCFG", "ACCSPMM_FW", "ACCSPMM_ROUND_B", "ACCSPMM_L2_PERSIST", "ACCSPMM_L2PROMO",
                 "ACCSPMM_SLICE_MAJOR", "ACCSPMM_GROUP_CAP"):
        assert knob not in strings, knob


def test_library_schedule_equals_hand_written_paper_schedule():
    """The library's units for unit_cap = 32 on a matrix whose windows hold
    3, 70, 5, 40, 2, 1, 30, 64, 0, 4 TC blocks equal the units written out by hand in
    tests/test_oracle_balance.py (row 8w of window w has 8*nb consecutive columns)."""
    from test_oracle_balance import HAND_RWO, HAND_UNITS
    blocks = np.diff(HAND_RWO)
    rows, cols = [], []
    for w, nb in enumerate(blocks):
        for c in range(8 * int(nb)):
            rows.append(8 * w)
            cols.append(c)
    A = gen.csr_from_pairs(np.array(rows), np.array(cols), 8 * len(blocks), 8 * int(blocks.max()))
    p = host_plan(A, np.ones(A.nnz, np.float32), balance="on", unit_cap=32)
    assert p.export_format()["RowWindowOffset"].tolist() == HAND_RWO
    assert p.info["ibd"] == pytest.approx(23.28, abs=1e-12) and p.info["balanced"] == 1
    assert [tuple(int(x) for x in u) for u in p.export_units()] == HAND_UNITS


@pytest.mark.parametrize("wh", [16, 32])
@pytest.mark.parametrize("reorder", ["off", "on"])
@pytest.mark.parametrize("precision", ["tf32"])
def test_tall_window_format_and_units_bit_exact_vs_oracle(wh, reorder, precision):
    """Reading R20: the library's tall-window plan (host builder) exports exactly the oracle's
    wh-row encoding of the (row-permuted) matrix, and its units equal the oracle schedule with
    the wh/8-scaled window write-back (balanced, cap 32, and grouped)."""
    from oracle import balance as ob
    from oracle import bittcf as bt
    from oracle.rounding import rho
    A = gen.dcsbm(2000, 60_000, 5, 2.2, 0.2, 1500, seed=wh, oversample=1.3)
    v = gen.values_uniform(A.nnz, 3)
    for balance, cap in (("on", 32), ("auto", 0)):
        p = host_plan(A, v, precision=precision, reorder=reorder, window_rows=wh, balance=balance, unit_cap=cap)
        assert p.info["window_rows"] == wh and p.info["kernel"] == acc.KERNEL["tcgen05"]
        perm = p.export_rows().astype(np.int64)
        rp, ci, vv = bt.permute_rows(A.M, A.rowptr, A.colidx, v, perm)
        ref = bt.encode(A.M, A.K, rp, ci, rho(vv, precision), wh=wh)
        F = p.export_format()
        for k in ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit"):
            assert np.array_equal(F[k], ref[k].astype(F[k].dtype)), k
        assert np.array_equal(F["values"], ref["values"])
        assert p.info["sum_U"] == int(ref["U"].sum())
        rwo = ref["RowWindowOffset"]
        if p.info["balanced"]:
            units = ob.build_units(rwo, p.info["unit_cap"], True, precision, wh=wh)
        else:
            units = ob.build_units(rwo, p.info["unit_cap"], False, precision, group=bool(p.info["grouped"]),
                                   group_cap=p.info["group_cap"], wh=wh)
        assert [tuple(int(x) for x in u) for u in p.export_units()] == [tuple(u) for u in units]


def test_window_rows_and_kernel_option_validation():
    A = gen.uniform_random(64, 64, 400, seed=2)
    v = gen.values_uniform(A.nnz, 1)
    with pytest.raises(acc.AccSpmmError) as e:
        host_plan(A, v, window_rows=24)
    assert e.value.status == 1                                   # INVALID_VALUE
    with pytest.raises(acc.AccSpmmError) as e:
        host_plan(A, v, window_rows=16, precision="fp16")        # tcgen05 path is TF32 only
    assert e.value.status == 3
    with pytest.raises(acc.AccSpmmError) as e:
        host_plan(A, v, window_rows=32, kernel="mma_sync")       # mma.sync runs 8- or 16-row windows
    assert e.value.status == 3
    for precision in ("tf32", "fp16"):                           # 16-row windows on mma.sync (R20)
        p = host_plan(A, v, window_rows=16, kernel="mma_sync", precision=precision)
        assert p.info["window_rows"] == 16 and p.info["kernel"] == acc.KERNEL["mma_sync"]
    p = host_plan(A, v, window_rows=16)                           # tall windows default to tcgen05
    assert p.info["kernel"] == acc.KERNEL["tcgen05"]
    p = host_plan(A, v)
    assert p.info["window_rows"] == 8 and p.info["kernel"] == acc.KERNEL["mma_sync"]
    p = host_plan(A, v, kernel="tcgen05")
    assert p.info["window_rows"] == 8 and p.info["kernel"] == acc.KERNEL["tcgen05"]


def _r21_graphs():
    return [("sbm", gen.sbm(512, 16, 0.3, 0.005, seed=1)),
            ("dcsbm", gen.dcsbm(2000, 60_000, 5, 2.2, 0.2, 1500, seed=2, oversample=1.3)),
            ("directed", gen.powerlaw_directed(3000, 8.0, seed=3)),
            ("stencil", gen.stencil27(12)),
            ("cliques", gen.two_cliques(20, seed=5))]


@pytest.mark.parametrize("idx", range(5))
@pytest.mark.parametrize("params", [(64, 4, 8), (1, 1, 64), (500, 7, 16), (100_000, 1, 8)])
def test_parallel_reorder_equals_oracle_r21(idx, params):
    """Reading R21 (the parallel Alg. 1 of plan creation above 8M vertices): the library equals
    the oracle's literal restatement (rounds of Step I, segments of Step II) exactly."""
    name, A = _r21_graphs()[idx]
    rs, sg, L = params
    ref = orr.reorder_parallel(A.M, A.K, A.rowptr, A.colidx, rs, sg, L)
    got = acc.accspmm_reorder_parallel(A.M, A.rowptr, A.colidx, rs, sg, L).astype(np.int64)
    assert np.array_equal(got, ref), name


def test_parallel_reorder_thread_count_independent():
    """R21 is a function of the input and (round, segments, L) only: 1 thread == all threads."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import numpy as np, gen, paper_2501_09251_b200 as acc; "
            "A = gen.dcsbm(20000, 600_000, 8, 2.2, 0.2, 3000, seed=9, oversample=1.3); "
            "p = acc.accspmm_reorder_parallel(A.M, A.rowptr, A.colidx, 1024, 16, 8); "
            "sys.stdout.write(str(int(np.uint64(np.sum(p.astype(np.uint64) * np.arange(A.M, dtype=np.uint64))))))") % ROOT
    outs = []
    for t in ("1", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                   timeout=300).stdout)
    assert outs[0] and outs[0] == outs[1]


def test_parallel_reorder_invariants():
    """R21 keeps Alg. 1's invariants: bijection, determinism, a shuffled
    two-clique fixture comes out as two contiguous ranges, and on the S:572 SBM (n = 512, 16
    blocks, p_in 0.3, p_out 0.005) the reordered matrix has more nnz per TC block than the
    shuffled one for 10 seeds."""
    from oracle import bittcf as bt
    for seed in range(5):
        k = 8
        A = gen.two_cliques(k, seed=seed)
        lab = np.random.default_rng(seed).permutation(2 * k)
        clique_of = {int(lab[i]): (0 if i < k else 1) for i in range(2 * k)}
        perm = acc.accspmm_reorder_parallel(A.M, A.rowptr, A.colidx, 4, 1, 8).astype(np.int64)
        assert sorted(perm.tolist()) == list(range(2 * k))
        seq = [clique_of[int(v)] for v in perm]
        assert seq == sorted(seq) or seq == sorted(seq, reverse=True)
    for seed in range(10):
        A = gen.sbm(512, 16, 0.3, 0.005, seed=seed)
        p1 = acc.accspmm_reorder_parallel(A.M, A.rowptr, A.colidx, 64, 1, 8).astype(np.int64)
        p2 = acc.accspmm_reorder_parallel(A.M, A.rowptr, A.colidx, 64, 1, 8).astype(np.int64)
        assert np.array_equal(p1, p2) and sorted(p1.tolist()) == list(range(512))
        inv = np.empty_like(p1)
        inv[p1] = np.arange(512)
        R = gen.csr_from_pairs(inv[A.row_ids()], A.colidx.astype(np.int64), 512, 512)
        assert bt.mean_nnz_tc(bt.encode(R.M, R.K, R.rowptr, R.colidx)) > \
            bt.mean_nnz_tc(bt.encode(A.M, A.K, A.rowptr, A.colidx))


def test_plan_create_with_supplied_permutation():
    """accspmm_plan_create_perm: a permutation computed elsewhere gives the same plan as running
    Alg. 1 inside plan creation; non-bijections and non-square A are rejected."""
    A = gen.sbm(600, 12, 0.2, 0.01, seed=3)
    v = gen.values_uniform(A.nnz, 4)
    perm = acc.accspmm_reorder(A.M, A.rowptr, A.colidx)
    for mode in ("on", "auto"):
        p0 = host_plan(A, v, reorder=mode)
        p1 = host_plan(A, v, reorder=mode, perm=perm)
        assert np.array_equal(p0.export_rows(), p1.export_rows())
        for k in ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit", "values"):
            assert np.array_equal(p0.export_format()[k], p1.export_format()[k])
    bad = perm.copy()
    bad[0] = bad[1]
    with pytest.raises(acc.AccSpmmError):
        host_plan(A, v, reorder="on", perm=bad)
    R = gen.uniform_random(10, 12, 30, seed=1)
    with pytest.raises(acc.AccSpmmError):
        host_plan(R, gen.values_uniform(R.nnz, 1), reorder="on", perm=np.arange(10, dtype=np.uint32))


def test_plan_b_bytes_reports_stored_b_element_size():
    """accspmm_plan_b_bytes (the es_B of the bytes model): the product library gathers FP32 rows
    for TF32 (the 3-byte image B3 is a variants-build measurement) and FP16 rows for FP16."""
    A = gen.uniform_random(300, 40, 3000, seed=2)       # high B-row reuse: the pre-round pass runs
    v = gen.values_uniform(A.nnz, 3)
    for prec, es in (("tf32", 4), ("fp16", 2)):
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=prec, device=-1)
        assert p.info["sum_U"] >= 32 * A.K
        for N in (16, 64, 128, 602):
            assert p.b_bytes(N) == es
        with pytest.raises(acc.AccSpmmError):
            p.b_bytes(0)
        p.close()


def _hot_order(A, rows_old):
    """Reading R22 written out: columns by descending in-degree over the given (original) rows,
    ties by ascending id -> colorig (new -> original)."""
    sel = np.concatenate([np.arange(A.rowptr[o], A.rowptr[o + 1]) for o in rows_old]) if len(rows_old) else \
        np.zeros(0, np.int64)
    deg = np.bincount(A.colidx[sel], minlength=A.K)
    return np.lexsort((np.arange(A.K), -deg))


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("reorder,nparts", [("off", 1), ("on", 1), ("on", 3)])
def test_hot_cols_format_is_column_relabelling(precision, reorder, nparts):
    """hot_cols (reading R22): each plan holds the paper's BitTCF of its slab with the columns
    relabelled by descending in-degree over the slab's rows (ties by id) -- encoded
    independently by the oracle on the explicitly relabelled matrix; windows then condense their
    hottest columns first."""
    A = gen.powerlaw_directed(3000, 12.0, seed=3)
    v = gen.values_uniform(A.nnz, 5)
    full = host_plan(A, v, precision=precision, reorder=reorder, hot_cols="on")
    perm = full.export_rows().astype(np.int64)              # slab row -> original row
    rows_seen = 0
    for part in range(nparts):
        p = host_plan(A, v, precision=precision, reorder=reorder, hot_cols="on", part=part, nparts=nparts)
        I = p.info
        assert I["hot_cols"] == 1 and I["cols_permuted"] == 0
        rows_old = p.export_rows().astype(np.int64)
        colorig = _hot_order(A, rows_old)
        newid = np.empty(A.K, np.int64)
        newid[colorig] = np.arange(A.K)
        r, c, vv = [], [], []
        for i, o in enumerate(rows_old):
            lo, hi = A.rowptr[o], A.rowptr[o + 1]
            cc = newid[A.colidx[lo:hi]]
            k = np.argsort(cc, kind="stable")
            r.append(np.full(hi - lo, i))
            c.append(cc[k])
            vv.append(v[lo:hi][k])
        r, c, vv = np.concatenate(r), np.concatenate(c), np.concatenate(vv)
        sl = gen.csr_from_pairs(r, c, len(rows_old), A.K)
        ref = bt.encode(sl.M, sl.K, sl.rowptr, sl.colidx, _rho_vals(vv, precision))
        _check_format(p.export_format(), ref, precision)
        rows_seen += I["rows"]
    assert rows_seen == A.M and len(perm) == A.M


def test_hot_cols_auto_rule_and_validation():
    """AUTO applies R22 only for K >= 2^20 with a skewed reference distribution (the 1% most
    referenced of the referenced columns carry >= 10% of nnz); ON is refused where the tags
    cannot be used."""
    K = 1 << 20
    rng = np.random.default_rng(1)
    rows = np.repeat(np.arange(2000), 10)
    skew = gen.csr_from_pairs(rows, np.where(rng.random(rows.size) < 0.5, rng.integers(0, 50, rows.size),
                                             rng.integers(0, K, rows.size)), 2000, K)
    flat = gen.csr_from_pairs(rows, rng.integers(0, K, rows.size), 2000, K)
    assert host_plan(skew, np.ones(skew.nnz, np.float32)).info["hot_cols"] == 1
    assert host_plan(flat, np.ones(flat.nnz, np.float32)).info["hot_cols"] == 0
    assert host_plan(skew, np.ones(skew.nnz, np.float32), hot_cols="off").info["hot_cols"] == 0
    small = gen.uniform_random(300, 300, 3000, seed=2)
    sv = np.ones(small.nnz, np.float32)
    assert host_plan(small, sv).info["hot_cols"] == 0                       # K < 2^20
    assert host_plan(small, sv, hot_cols="on").info["hot_cols"] == 1
    for kw in ({"window_rows": 16}, {"permute_cols": True, "reorder": "on"}):
        with pytest.raises(acc.AccSpmmError):
            host_plan(small, sv, hot_cols="on", **kw)
