"""GPU parity of 16-row RowWindows (reading R20) on the mma.sync kernel (kernel="mma_sync",
window_rows=16: every gathered row feeds two accumulator halves) against the FP64 oracle,
through the C ABI.  Same bar as test_gpu_parity.py: floats within tau*S + 1e-6 (TF32) /
4e-3 (FP16), integer-valued inputs bit-exact (split windows, reordering, partitions, every
feature width), every output starts as a NaN canary."""
import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from gpu_util import assert_bit_exact, assert_within, run, to_dev_B

pytestmark = pytest.mark.gpu
PREC = ["tf32", "fp16"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()
    from paper_2501_09251_b200 import _build
    _build.build()


def tall(**kw):
    kw.setdefault("kernel", "mma_sync")
    kw.setdefault("window_rows", 16)
    return kw


@pytest.mark.parametrize("precision", PREC)
@pytest.mark.parametrize("N", [16, 32, 64, 128, 256, 100])
@pytest.mark.parametrize("balance", ["off", "on"])
def test_tall_mma_random_ragged_float(precision, N, balance):
    """Ragged M, K; every feature width (16/32/64/128 slices, N = 100 through the padded path)."""
    A = gen.uniform_random(1003, 777, 20000, seed=N + 3)
    v = gen.values_uniform(A.nnz, 5)
    B = gen.dense_normal(A.K, N, 6)
    C, p = run(A, v, B, precision, **tall(balance=balance, unit_cap=8))
    assert p.info["kernel"] == acc.KERNEL["mma_sync"] and p.info["window_rows"] == 16
    assert_within(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PREC)
@pytest.mark.parametrize("N", [32, 64, 128, 256])
def test_tall_mma_integer_bit_exact_split_windows(precision, N):
    """Split windows (balance on, small cap) sum their partial 16 x N tiles in segment order:
    bit-identical to balance off, to the oracle, and to the 8-row-window kernel."""
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=N + 1, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, N, 2)
    C_off, _ = run(A, v, B, precision, **tall(balance="off"))
    C_on, p = run(A, v, B, precision, **tall(balance="on", unit_cap=32))
    assert p.info["n_split_windows"] > 0
    assert_bit_exact(C_off, A, v, B, precision)
    assert np.array_equal(C_on, C_off)
    C8, _ = run(A, v, B, precision, balance="on", unit_cap=32)
    assert np.array_equal(C8, C_off)


@pytest.mark.parametrize("precision", PREC)
def test_tall_mma_every_tile_position(precision):
    """Window 8r + c holds the probe entry (row r, column c) plus the other seven columns in row
    (r + 8) % 16, i.e. in the other occupancy word, so its one block condenses columns 0..7 onto
    lanes 0..7 and the probe sits at tile position (r, c): all 128 positions of a 16 x 8 block,
    both words, distinct values, bit-exact."""
    rows, cols = [], []
    for r in range(16):
        for c in range(8):
            w = 8 * r + c
            rows.append(16 * w + r)
            cols.append(c)
            for j in range(8):
                if j != c:
                    rows.append(16 * w + (r + 8) % 16)
                    cols.append(j)
    A = gen.csr_from_pairs(np.array(rows), np.array(cols), 16 * 128, 8)
    v = (np.arange(A.nnz) % 7 + 1).astype(np.float32) * np.where(np.arange(A.nnz) % 3 == 0, -1, 1)
    B = gen.dense_int(8, 64, 3)
    C, p = run(A, v, B, precision, **tall(reorder="off"))
    assert p.info["NB"] == 128
    assert_bit_exact(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PREC)
def test_tall_mma_reordered_and_partitions(precision):
    """Reordering (rows scattered through perm) and nparts = 3 slabs concatenate to the product."""
    import torch
    A = gen.dcsbm(2500, 100_000, 5, 2.2, 0.2, 1500, seed=16, oversample=1.3)
    v = gen.values_int(A.nnz, 2)
    B = gen.dense_int(A.K, 128, 3)
    C, _ = run(A, v, B, precision, **tall(reorder="on"))
    assert_bit_exact(C, A, v, B, precision)
    out = torch.full((A.M, 128), float("nan"), device="cuda")
    for part in range(3):
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", part=part, nparts=3,
                     **tall())
        G = p.execute(to_dev_B(B, precision))
        rows = torch.from_numpy(p.export_rows().astype(np.int64)).cuda()
        out[rows] = G
    torch.cuda.synchronize()
    assert_bit_exact(out.cpu().numpy(), A, v, B, precision)


@pytest.mark.parametrize("precision", PREC)
def test_tall_mma_empty_windows_ragged_and_degenerate(precision):
    """M = 16k+3 with empty leading rows, windows without blocks inside grouped units, nnz = 0,
    K = 0: every row is written (no canary left)."""
    rows = np.concatenate([np.arange(64, 70), np.arange(200, 203), np.arange(700, 1003, 7)])
    A = gen.csr_from_pairs(rows, (rows * 13) % 500, 1003, 500)
    v = gen.values_int(A.nnz, 4)
    B = gen.dense_int(500, 128, 5)
    for balance in ("auto", "off", "on"):
        C, _ = run(A, v, B, precision, **tall(balance=balance))
        assert_bit_exact(C, A, v, B, precision)
    E = gen.Csr(37, 50, np.zeros(38, np.int64), np.zeros(0, np.int32))
    C, _ = run(E, np.zeros(0, np.float32), gen.dense_int(50, 128, 1), precision, **tall())
    assert np.array_equal(C, np.zeros((37, 128), np.float32))


@pytest.mark.parametrize("precision", PREC)
def test_tall_mma_full_size_reddit_sampled(precision):
    """The Reddit-shaped configuration (configs[2], 115M nnz, N = 128) with 16-row windows on the
    mma.sync kernel: 3,000 sampled rows within tolerance, no NaN anywhere."""
    import torch
    cfg, A = gen.make_config("reddit")
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, 128, cfg.seed_B)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="auto", build="device", **tall())
    C = torch.full((A.M, 128), float("nan"), device="cuda")
    p.execute(to_dev_B(B, precision), C)
    torch.cuda.synchronize()
    Cg = C.cpu().numpy()
    assert np.isfinite(Cg).all()
    rows = np.sort(np.random.default_rng(0).choice(A.M, 3000, replace=False))
    assert_within(Cg, A, v, B, precision, rows=rows)


@pytest.mark.parametrize("precision", PREC)
def test_tall_mma_fused_allgather_epilogue(precision):
    """accspmm_execute_allgather with 16-row windows: both accumulator halves of every window go
    to every destination in original row order (3 parts, 3 local destinations, split windows,
    reordering; integer data bit-exact)."""
    import torch
    A = gen.dcsbm(4000, 200_000, 6, 2.2, 0.2, 2500, seed=3, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 128, 2)
    Bd = to_dev_B(B, precision)
    dsts = [torch.full((A.M, 128), float("nan"), device="cuda") for _ in range(3)]
    for part in range(3):
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", balance="on",
                     unit_cap=32, part=part, nparts=3, **tall())
        p.execute_allgather(Bd, dsts)
    torch.cuda.synchronize()
    for d in dsts:
        assert_bit_exact(d.cpu().numpy(), A, v, B, precision)


@pytest.mark.parametrize("precision", PREC)
def test_tall_mma_cuda_graph_and_host_batch(precision):
    """The plan replays under CUDA-graph capture and through the pipelined host batch API with
    the same bits as a plain execute."""
    import torch
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=9, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B0 = gen.dense_int(A.K, 64, 2)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", balance="on", unit_cap=32,
                 **tall())
    Bd = to_dev_B(B0, precision)
    ref = p.execute(Bd).cpu().numpy()
    assert_bit_exact(ref, A, v, B0, precision)
    C = torch.full((A.M, 64), float("nan"), device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        p.execute(Bd, C, s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    C.fill_(float("nan"))
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        p.execute(Bd, C, s)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), ref)
    Bh = [Bd.cpu().pin_memory() for _ in range(3)]
    Ch = [torch.full((A.M, 64), float("nan")).pin_memory() for _ in range(3)]
    p.execute_host_batch(Bh, Ch)
    for c in Ch:
        assert np.array_equal(c.numpy(), ref)
