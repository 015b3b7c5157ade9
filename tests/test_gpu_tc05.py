"""GPU parity of the tcgen05/TMEM kernel and of tall RowWindows (reading R20)
against the FP64 oracle, through the C ABI.  Same bar as test_gpu_parity.py: floats within
tau*S + 1e-6 (TF32), integer-valued inputs bit-exact (split windows, reordering, partitions
included), every output starts as a NaN canary."""
import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from gpu_util import assert_bit_exact, assert_within, oracle, run, to_dev_B

pytestmark = pytest.mark.gpu
WH = [8, 16, 32]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()
    from paper_2501_09251_b200 import _build
    _build.build()


def tc(**kw):
    kw.setdefault("kernel", "tcgen05")
    return kw


@pytest.mark.parametrize("wh", WH)
@pytest.mark.parametrize("N", [128, 256, 384, 64, 100])
@pytest.mark.parametrize("balance", ["off", "on"])
def test_tc05_random_ragged_float(wh, N, balance):
    """Ragged M, K; N = 64 / 100 run through the padded path (128-feature slices)."""
    A = gen.uniform_random(1003, 777, 20000, seed=N + wh)
    v = gen.values_uniform(A.nnz, 5)
    B = gen.dense_normal(A.K, N, 6)
    C, p = run(A, v, B, "tf32", **tc(window_rows=wh, balance=balance, unit_cap=8))
    assert p.info["kernel"] == acc.KERNEL["tcgen05"] and p.info["window_rows"] == wh
    assert_within(C, A, v, B, "tf32")


@pytest.mark.parametrize("wh", WH)
@pytest.mark.parametrize("N", [128, 256])
def test_tc05_integer_bit_exact_split_windows(wh, N):
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=N + wh, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, N, 2)
    C_off, _ = run(A, v, B, "tf32", **tc(window_rows=wh, balance="off"))
    C_on, p = run(A, v, B, "tf32", **tc(window_rows=wh, balance="on", unit_cap=32))
    assert p.info["n_split_windows"] > 0
    assert_bit_exact(C_off, A, v, B, "tf32")
    assert np.array_equal(C_on, C_off)
    C_mma, _ = run(A, v, B, "tf32", balance="on", unit_cap=32)          # the mma.sync kernel agrees
    assert np.array_equal(C_mma, C_off)


@pytest.mark.parametrize("wh", WH)
def test_tc05_reordered_and_partitions(wh):
    """Reordering (rows scattered through perm) and nparts = 3 slabs concatenate to the product."""
    import torch
    A = gen.dcsbm(2500, 100_000, 5, 2.2, 0.2, 1500, seed=wh, oversample=1.3)
    v = gen.values_int(A.nnz, 2)
    B = gen.dense_int(A.K, 128, 3)
    C, _ = run(A, v, B, "tf32", **tc(window_rows=wh, reorder="on"))
    assert_bit_exact(C, A, v, B, "tf32")
    out = torch.full((A.M, 128), float("nan"), device="cuda")
    for part in range(3):
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="on", part=part, nparts=3, **tc(window_rows=wh))
        G = p.execute(to_dev_B(B, "tf32"))
        rows = torch.from_numpy(p.export_rows().astype(np.int64)).cuda()
        out[rows] = G
    torch.cuda.synchronize()
    assert_bit_exact(out.cpu().numpy(), A, v, B, "tf32")


@pytest.mark.parametrize("wh", WH)
def test_tc05_empty_windows_ragged_and_degenerate(wh):
    """M = 8k+3 with empty leading rows, windows without blocks inside grouped units, nnz = 0,
    K = 0: every row is written (no canary left)."""
    rows = np.concatenate([np.arange(64, 70), np.arange(200, 203), np.arange(700, 1003, 7)])
    A = gen.csr_from_pairs(rows, (rows * 13) % 500, 1003, 500)
    v = gen.values_int(A.nnz, 4)
    B = gen.dense_int(500, 128, 5)
    for balance in ("auto", "off", "on"):
        C, _ = run(A, v, B, "tf32", **tc(window_rows=wh, balance=balance))
        assert_bit_exact(C, A, v, B, "tf32")
    E = gen.Csr(37, 50, np.zeros(38, np.int64), np.zeros(0, np.int32))
    C, _ = run(E, np.zeros(0, np.float32), gen.dense_int(50, 128, 1), "tf32", **tc(window_rows=wh))
    assert np.array_equal(C, np.zeros((37, 128), np.float32))
    Z = gen.Csr(21, 0, np.zeros(22, np.int64), np.zeros(0, np.int32))
    C, _ = run(Z, np.zeros(0, np.float32), np.zeros((0, 128), np.float32), "tf32", **tc(window_rows=wh))
    assert np.array_equal(C, np.zeros((21, 128), np.float32))


@pytest.mark.parametrize("wh", [16, 32])
def test_tall_window_device_build_equals_host_build(wh):
    A = gen.dcsbm(3000, 120_000, 5, 2.2, 0.2, 2000, seed=wh, oversample=1.3)
    v = gen.values_uniform(A.nnz, 1)
    ph = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="on", window_rows=wh, build="host")
    pd = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="on", window_rows=wh, build="device")
    Fh, Fd = ph.export_format(), pd.export_format()
    for k in ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit", "values"):
        assert np.array_equal(Fh[k], Fd[k]), k
    assert np.array_equal(ph.export_units(), pd.export_units())


@pytest.mark.parametrize("wh", [16, 32])
def test_tall_window_device_decode_matches_oracle_tiles(wh):
    from oracle import bittcf as bt
    from oracle.rounding import rho
    A = gen.uniform_random(300, 200, 6000, seed=wh)
    v = gen.values_uniform(A.nnz, 1)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="off", window_rows=wh)
    tiles = p.debug_decode().cpu().numpy()
    F = bt.encode(A.M, A.K, A.rowptr, A.colidx, rho(v, "tf32"), wh=wh)
    rp, ci, vv = bt.decode(F)
    ref = np.zeros((F["NB"], 8 * wh), np.float32)
    blk_of_window = F["RowWindowOffset"]
    for r in range(A.M):
        w, lr = divmod(r, wh)
        for q in range(rp[r], rp[r + 1]):
            U = F["SparseAToB"][8 * blk_of_window[w]: 8 * blk_of_window[w + 1]]
            pos = int(np.nonzero(U == ci[q])[0][0])
            ref[blk_of_window[w] + pos // 8, lr * 8 + pos % 8] = vv[q]
    assert np.array_equal(tiles, ref)


def test_tc05_full_size_reddit_sampled():
    """The Reddit-shaped configuration (configs[2], 115M nnz, N = 128) on the tcgen05 kernel
    with 32-row windows: 3,000 sampled rows within tolerance, no NaN anywhere."""
    import torch
    cfg, A = gen.make_config("reddit")
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, 128, cfg.seed_B)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="auto", build="device", **tc(window_rows=32))
    C = torch.full((A.M, 128), float("nan"), device="cuda")
    p.execute(to_dev_B(B, "tf32"), C)
    torch.cuda.synchronize()
    Cg = C.cpu().numpy()
    assert np.isfinite(Cg).all()
    rows = np.sort(np.random.default_rng(0).choice(A.M, 3000, replace=False))
    assert_within(Cg, A, v, B, "tf32", rows=rows)


def test_tc05_cuda_graph_capture():
    import torch
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=7, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B0 = gen.dense_int(A.K, 128, 2)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="on", balance="on", unit_cap=32, **tc(window_rows=16))
    Bd = to_dev_B(B0, "tf32")
    C = torch.full((A.M, 128), float("nan"), device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        p.execute(Bd, C, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    C.fill_(float("nan"))
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        p.execute(Bd, C, torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    assert_bit_exact(C.cpu().numpy(), A, v, B0, "tf32")
    _ = oracle
