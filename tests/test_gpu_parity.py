"""GPU parity: the sm_100a CUDA path (through the C ABI) vs the FP64 oracle.

Tolerance (BASELINE north_star): |C_gpu - C_ref| <= tau*S + 1e-6, tau = 1e-3 TF32 / 4e-3 FP16.
Integer-valued inputs (A in {-3..3}\\{0}, B in {-8..8}) must be bit-exact.
Fixtures follow SURVEY §8(c) C-4; every output starts as a NaN canary.
"""
import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from gpu_util import assert_bit_exact, assert_within, oracle, run, to_dev_B

pytestmark = pytest.mark.gpu

PRECISIONS = ["tf32", "fp16"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()
    from paper_2501_09251_b200 import _build
    _build.build()


def _ragged(seed=0, M=1003, K=777, nnz=20000):
    return gen.uniform_random(M, K, nnz, seed=seed)


def test_tiny_config():
    cfg, A = gen.make_config("tiny")
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, 16, cfg.seed_B)
    C, _ = run(A, v, B, "tf32")
    assert_within(C, A, v, B, "tf32")


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("N", [16, 32, 48, 64, 96, 128, 256, 384, 512, 1152])
@pytest.mark.parametrize("balance", ["off", "on"])
def test_random_ragged_float(precision, N, balance):
    """N up to 512 (the paper's widest feature dimension) uses one TMA map per 128-wide
    slice; N = 1152 (9 slices) exercises the single full-width map."""
    A = _ragged(seed=N)
    v = gen.values_uniform(A.nnz, 5)
    B = gen.dense_normal(A.K, N, 6)
    C, p = run(A, v, B, precision, balance=balance, unit_cap=8)
    assert_within(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("N", [16, 32, 64, 128, 256, 512])
def test_integer_bit_exact_and_balance_invariant(precision, N):
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=N, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, N, 2)
    C_off, _ = run(A, v, B, precision, balance="off")
    C_on, p = run(A, v, B, precision, balance="on", unit_cap=32)
    assert p.info["n_split_windows"] > 0
    assert_bit_exact(C_off, A, v, B, precision)
    assert np.array_equal(C_on, C_off)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_permutation_matrix_exact(precision):
    A = gen.permutation_matrix(1000, seed=3)
    v = np.ones(A.nnz, np.float32)
    B = gen.dense_normal(1000, 64, 4)
    C, _ = run(A, v, B, precision)
    assert_bit_exact(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_rho_b_bit_exact_both_rounding_paths(precision):
    """C = A.rho(B) with one unit nnz per row is rho(B) itself: pins the B rounding on the
    in-kernel path (low B-row reuse) and on the pre-round pass (high reuse) bit-exactly."""
    low = gen.permutation_matrix(2048, seed=5)                        # reuse 1
    high = gen.csr_from_pairs(np.arange(4096), np.arange(4096) % 8, 4096, 8)   # reuse 512
    for A in (low, high):
        v = np.ones(A.nnz, np.float32)
        B = gen.dense_normal(A.K, 128, 9)
        C, p = run(A, v, B, precision)
        assert_bit_exact(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_padding_lanes_do_not_leak_inf(precision):
    # windows with 1..7 unique columns (partial last block), column 0 unused, B[0,:] = +Inf
    rows, cols = [], []
    for w in range(7):
        for u in range(1, w + 2):
            rows.append(8 * w + (u % 8))
            cols.append(10 * w + u)
    A = gen.csr_from_pairs(rows, cols, 64, 128)
    v = gen.values_int(A.nnz, 0)
    B = gen.dense_int(128, 32, 1)
    B[0, :] = np.inf
    C, _ = run(A, v, B, precision)
    assert np.isfinite(C).all()
    assert_bit_exact(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_single_bit_probes(precision):
    # 64 windows, window (8r+c) holds the probe for position (r, c) (SURVEY C-4 a8(ii))
    rows, cols = [], []
    for r in range(8):
        for c in range(8):
            w = 8 * r + c
            rp = (r + 1) % 8
            for l in range(c):
                rows.append(8 * w + rp)
                cols.append(l)
            rows.append(8 * w + r)
            cols.append(c)
    A = gen.csr_from_pairs(rows, cols, 512, 8)
    v = gen.values_int(A.nnz, 3)
    B = gen.dense_int(8, 16, 4)
    C, _ = run(A, v, B, precision)
    assert_bit_exact(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_dense_band_and_dense_windows(precision):
    r = np.repeat(np.arange(64), 40)
    c = np.tile(np.arange(40), 64) + (np.repeat(np.arange(64), 40) // 8) * 3
    A = gen.csr_from_pairs(r, c, 64, 300)
    v = gen.values_int(A.nnz, 5)
    B = gen.dense_int(300, 128, 6)
    C, _ = run(A, v, B, precision)
    assert_bit_exact(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_empty_windows_ragged_and_degenerate(precision):
    # M = 8k+3, rows 0..63 empty, K not a multiple of 8
    base = gen.uniform_random(8 * 50 + 3, 45, 600, seed=9)
    keep = base.row_ids() >= 64
    A = gen.csr_from_pairs(base.row_ids()[keep], base.colidx[keep], base.M, base.K)
    v = gen.values_int(A.nnz, 7)
    B = gen.dense_int(45, 32, 8)
    for bal in ("off", "on"):
        C, _ = run(A, v, B, precision, balance=bal, unit_cap=4)
        assert_bit_exact(C, A, v, B, precision)
        assert np.all(C[:64] == 0)
    # nnz = 0
    Z = gen.Csr(37, 20, np.zeros(38, np.int64), np.zeros(0, np.int32))
    C, _ = run(Z, np.zeros(0, np.float32), gen.dense_int(20, 16, 1), precision)
    assert np.all(C == 0)
    # M = 0
    E = gen.Csr(0, 20, np.zeros(1, np.int64), np.zeros(0, np.int32))
    C, _ = run(E, np.zeros(0, np.float32), gen.dense_int(20, 16, 1), precision)
    assert C.shape == (0, 16)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_split_window_hub(precision):
    # one window of 8 rows x 4000 distinct columns = 500 blocks > cap 32
    rng = np.random.default_rng(1)
    rows = np.repeat(np.arange(8), 1500)
    cols = np.concatenate([rng.choice(4000, 1500, replace=False) for _ in range(8)])
    A = gen.csr_from_pairs(np.concatenate([rows, [20]]), np.concatenate([cols, [5]]), 24, 4000)
    v = gen.values_int(A.nnz, 2)
    B = gen.dense_int(4000, 64, 3)
    C_on, p = run(A, v, B, precision, balance="on", unit_cap=32)
    assert p.info["n_split_windows"] == 1 and p.info["n_segments"] >= 16
    C_off, _ = run(A, v, B, precision, balance="off")
    assert_bit_exact(C_on, A, v, B, precision)
    assert np.array_equal(C_on, C_off)
    vf = gen.values_uniform(A.nnz, 4)
    Bf = gen.dense_normal(4000, 64, 5)
    C, _ = run(A, vf, Bf, precision, balance="on", unit_cap=32)
    assert_within(C, A, vf, Bf, precision)


def test_concatenated_windows_exact():
    # 1000 windows with one block each, balance forced on (concatenation) vs off
    A = gen.uniform_random(8000, 8000, 8000, seed=12)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(8000, 32, 2)
    C_on, p = run(A, v, B, "tf32", balance="on", unit_cap=32)
    assert p.info["n_units"] < 1000
    C_off, _ = run(A, v, B, "tf32", balance="off")
    assert np.array_equal(C_on, C_off)
    assert_bit_exact(C_on, A, v, B, "tf32")


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partitions_concatenate_to_whole(P):
    A = gen.dcsbm(5000, 200_000, 6, 2.2, 0.2, 3000, seed=4, oversample=1.3)
    v = gen.values_uniform(A.nnz, 3)
    B = gen.dense_normal(A.K, 64, 4)
    C1, _ = run(A, v, B, "tf32", balance="on", unit_cap=32)
    slabs = []
    for k in range(P):
        Ck, pk = run(A, v, B, "tf32", balance="on", unit_cap=32, part=k, nparts=P)
        assert np.array_equal(pk.export_rows(), np.arange(pk.info["row_begin"], pk.info["row_begin"] + pk.info["rows"]))
        slabs.append(Ck)
    assert np.array_equal(np.concatenate(slabs), C1)


@pytest.mark.parametrize("mode", ["on", "auto"])
@pytest.mark.parametrize("precision", PRECISIONS)
def test_reordered_product_equals_unreordered_oracle(mode, precision):
    A = gen.sbm(2048, 32, 0.1, 0.002, seed=7)
    vi = gen.values_int(A.nnz, 1)
    Bi = gen.dense_int(A.K, 32, 2)
    C, p = run(A, vi, Bi, precision, reorder=mode)
    if mode == "on":
        assert p.info["reorder_applied"] == 1
    assert_bit_exact(C, A, vi, Bi, precision)
    vf = gen.values_uniform(A.nnz, 3)
    Bf = gen.dense_normal(A.K, 64, 4)
    C, _ = run(A, vf, Bf, precision, reorder=mode)
    assert_within(C, A, vf, Bf, precision)


def test_reordered_partitions_and_unpermute():
    import torch
    A = gen.sbm(1024, 16, 0.1, 0.004, seed=8)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 32, 2)
    C1, _ = run(A, v, B, "tf32", reorder="on")
    P = 3
    slabs, ids = [], []
    for k in range(P):
        Ck, pk = run(A, v, B, "tf32", reorder="on", part=k, nparts=P)
        slabs.append(Ck)
        ids.append(pk.export_rows())
    # emulate the all-gather of padded slabs + device un-permute (K6)
    mx = max(s.shape[0] for s in slabs)
    G = np.zeros((P * mx, 32), np.float32)
    rid = np.full(P * mx, 0xFFFFFFFF, np.uint32)
    for k in range(P):
        G[k * mx:k * mx + slabs[k].shape[0]] = slabs[k]
        rid[k * mx:k * mx + slabs[k].shape[0]] = ids[k]
    Gd = torch.from_numpy(G).cuda()
    rd = torch.from_numpy(rid.view(np.int32)).cuda()
    Cd = torch.full((A.M, 32), float("nan"), device="cuda")
    acc.accspmm_unpermute(Gd.data_ptr(), rd.data_ptr(), P * mx, 32, Cd.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(Cd.cpu().numpy(), C1)


def test_repeat_runs_bitwise_deterministic():
    import torch
    A = gen.dcsbm(4000, 300_000, 5, 2.2, 0.2, 3000, seed=5, oversample=1.3)
    v = gen.values_uniform(A.nnz, 1)
    B = gen.dense_normal(A.K, 128, 2)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, balance="on", unit_cap=32)
    Bd = to_dev_B(B, "tf32")
    outs = [p.execute(Bd).cpu().numpy() for _ in range(3)]
    torch.cuda.synchronize()
    assert p.info["n_split_windows"] > 0
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("precision", PRECISIONS)
def test_device_decode_matches_oracle_tiles(precision):
    from oracle import bittcf as bt
    from oracle.rounding import rho
    A = _ragged(seed=2, M=300, K=200, nnz=6000)
    v = gen.values_uniform(A.nnz, 1)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="off")
    tiles = p.debug_decode().cpu().numpy()
    F = bt.encode(A.M, A.K, A.rowptr, A.colidx, rho(v, precision))
    ref = np.zeros((F["NB"], 64), np.float32)
    tco = F["TCOffset"].astype(np.int64)
    for b in range(F["NB"]):
        m = int(F["TCLocalBit"][b])
        for k in range(64):
            if (m >> k) & 1:
                ref[b, k] = F["values"][tco[b] + bin(m & ((1 << k) - 1)).count("1")]
    assert np.array_equal(tiles, ref)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_device_plan_exports_paper_format(precision):
    """The device copy of the format (padding lanes re-marked for the TMA) exports as BitTCF."""
    from oracle import bittcf as bt
    from oracle.rounding import rho
    A = _ragged(seed=6, M=700, K=900, nnz=9000)
    v = gen.values_uniform(A.nnz, 2)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="off")
    F = p.export_format()
    ref = bt.encode(A.M, A.K, A.rowptr, A.colidx, rho(v, precision))
    for k in ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit"):
        assert np.array_equal(F[k], ref[k]), k
    assert np.array_equal(F["values"].astype(np.float32), ref["values"].astype(np.float32))


def test_e2e_host_path_matches_device_path():
    A = _ragged(seed=3)
    v = gen.values_uniform(A.nnz, 1)
    B = gen.dense_normal(A.K, 128, 2)
    C, p = run(A, v, B, "tf32")
    Ch = np.full((A.M, 128), np.nan, np.float32)
    p.execute_host(np.ascontiguousarray(B), Ch)
    assert np.array_equal(Ch, C)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_e2e_host_batch_pipeline_matches_device_path(precision):
    """accspmm_execute_host_batch: 5 different B (pinned and pageable) through the two-slot
    pipeline; every C equals the device-path C of its own B bitwise."""
    import torch
    A = _ragged(seed=4)
    v = gen.values_uniform(A.nnz, 1)
    Bs = [gen.dense_normal(A.K, 64, 10 + i) for i in range(5)]
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision)
    ref = []
    for B in Bs:
        C = torch.full((A.M, 64), float("nan"), device="cuda")
        p.execute(to_dev_B(B, precision), C)
        ref.append(C.cpu().numpy())
    hdt = torch.float16 if precision == "fp16" else torch.float32
    Bh = [torch.from_numpy(B).to(hdt).pin_memory() if i % 2 == 0 else torch.from_numpy(B).to(hdt)
          for i, B in enumerate(Bs)]
    Ch = [torch.full((A.M, 64), float("nan")).pin_memory() for _ in Bs]
    p.execute_host_batch(Bh, Ch)
    for c, r in zip(Ch, ref):
        assert np.array_equal(c.numpy(), r)
    acc.accspmm_execute_host_batch(p.handle, [], [], 64)  # empty batch is a no-op


def test_e2e_mixed_host_calls_with_growing_N():
    """ADVICE r1 repro: execute_host_batch(N=16), execute_host(N=128), execute_host_batch(N=128)
    must regrow the second staging slots too (each slot carries its own size); every C equals
    the oracle product of its own B."""
    A = _ragged(seed=9)
    v = gen.values_int(A.nnz, 1)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="off")
    for kind, N in (("batch", 16), ("single", 128), ("batch", 128), ("single", 256), ("batch", 256)):
        Bs = [gen.dense_int(A.K, N, 30 + N + i) for i in range(3)]
        Cs = [np.full((A.M, N), np.nan, np.float32) for _ in Bs]
        if kind == "batch":
            p.execute_host_batch(Bs, Cs)
        else:
            for B, C in zip(Bs, Cs):
                p.execute_host(B, C)
        for B, C in zip(Bs, Cs):
            assert_bit_exact(C, A, v, B, "tf32")


def test_execute_errors():
    import torch
    A = _ragged(seed=4, M=100, K=100, nnz=500)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, gen.values_uniform(A.nnz, 1))
    B = torch.zeros((100, 24), device="cuda")
    C = torch.zeros((100, 24), device="cuda")
    with pytest.raises(acc.AccSpmmError) as ei:   # N % 16 != 0 is padded, but not in the fused all-gather
        acc.accspmm_execute_allgather(p.handle, B.data_ptr(), 24, [C.data_ptr()])
    assert ei.value.status == 3
    with pytest.raises(acc.AccSpmmError) as ei:
        acc.accspmm_execute(p.handle, B.data_ptr(), 0, C.data_ptr())
    assert ei.value.status == 1
    B = torch.zeros((100, 32), device="cuda")
    with pytest.raises(acc.AccSpmmError) as ei:
        acc.accspmm_execute(p.handle, B.data_ptr() + 4, 32, C.data_ptr())
    assert ei.value.status == 1


def test_tf32_rounding_exhaustive_vs_oracle():
    """Pins oracle/rounding.tf32_rna to the hardware cvt.rna.tf32.f32 over all 2^32 patterns."""
    import torch
    from oracle.rounding import tf32_rna
    chunk = 1 << 28
    inp = torch.empty(chunk, dtype=torch.int32, device="cuda")
    out = torch.empty(chunk, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for c in range(1 << 32 >> 28):
        base = c * chunk
        host = (np.arange(chunk, dtype=np.uint64) + base).astype(np.uint32)
        inp.copy_(torch.from_numpy(host.view(np.int32)))
        acc.accspmm_debug_round_tf32(inp.data_ptr(), out.data_ptr(), chunk, s)
        dev = out.cpu().numpy().view(np.uint32)
        ref = tf32_rna(host.view(np.float32)).view(np.uint32)
        assert np.array_equal(dev, ref), f"chunk {c}"


# --------------------------------------------------------------- full-size configs, sampled rows

def _sample_rows(M, n, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([rng.integers(0, M, n), [0, M - 1]]))


@pytest.mark.parametrize("name,N,precision", [
    ("reddit", 128, "tf32"), ("reddit", 128, "fp16"), ("reddit", 32, "tf32"), ("reddit", 64, "tf32"),
    ("stencil", 128, "tf32"), ("products", 128, "tf32"), ("papers100m_small", 64, "tf32"),
    ("reddit", 256, "tf32"), ("reddit", 512, "fp16"), ("reddit", 64, "fp16"), ("reddit", 32, "fp16"),
    ("banded", 128, "tf32"),
    ("roadnet", 128, "tf32"), ("yeasth", 512, "tf32"), ("dd", 256, "fp16"), ("webberkstan", 128, "tf32"),
])
def test_full_size_config_sampled(name, N, precision):
    cfg, A = gen.make_config(name)
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, N, cfg.seed_B)
    C, p = run(A, v, B, precision)
    rows = _sample_rows(A.M, 3000, 1)
    assert np.isfinite(C).all()
    assert_within(C, A, v, B, precision, rows=rows)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_grouped_whole_windows_equal_one_window_per_unit(precision):
    """Balance AUTO below the IBD threshold groups whole windows per unit (reading R7b); on
    integer data the result equals the paper's one-window-per-unit schedule bitwise."""
    A = gen.road_grid(300, 0.7, seed=4)
    v = gen.values_int(A.nnz, 3)
    B = gen.dense_int(A.K, 128, 4)
    C_auto, pa = run(A, v, B, precision, balance="auto")
    C_off, po = run(A, v, B, precision, balance="off")
    assert pa.info["grouped"] == 1 and pa.info["n_units"] < po.info["n_units"] == po.info["W"]
    assert_bit_exact(C_auto, A, v, B, precision)
    assert np.array_equal(C_auto, C_off)


@pytest.mark.parametrize("name,N,reorder", [("reddit", 128, "auto"), ("papers100m_small", 64, "off")])
def test_bench_configuration_sampled(name, N, reorder):
    """The launch configuration bench.py times (reorder/balance auto), sampled rows vs the oracle."""
    cfg, A = gen.make_config(name)
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, N, cfg.seed_B)
    C, p = run(A, v, B, "tf32", reorder=reorder, balance="auto")
    assert np.isfinite(C).all()
    assert_within(C, A, v, B, "tf32", rows=_sample_rows(A.M, 3000, 3))


def test_full_size_reddit_integer_sampled_bit_exact():
    cfg, A = gen.make_config("reddit")
    v = gen.values_int(A.nnz, cfg.seed_A + 1)
    B = gen.dense_int(A.K, 128, cfg.seed_B)
    C, p = run(A, v, B, "tf32")
    assert p.info["balanced"] == 1
    rows = _sample_rows(A.M, 2000, 2)
    Cr, _ = oracle(A, v, B, "tf32", rows=rows)
    assert np.array_equal(C[rows].astype(np.float64), Cr)


# --------------------------------------------------------------- randomized sweep

@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_and_options(seed):
    """Seeded random shapes, densities, N, precision and plan options vs the oracle."""
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
    nnz = int(min(M * K, 10 ** rng.uniform(0, 5)))
    A = gen.uniform_random(M, K, nnz, seed=seed)
    N = int(rng.choice([16, 32, 48, 64, 80, 128, 192, 256, 384]))
    precision = PRECISIONS[seed % 2]
    balance = ["off", "on", "auto"][seed % 3]
    cap = int(rng.choice([0, 8, 32, 100]))
    reorder = "on" if (M == K and seed % 4 == 0) else "off"
    if seed % 5 == 0:
        v = gen.values_int(A.nnz, seed)
        B = gen.dense_int(K, N, seed + 1)
        C, _ = run(A, v, B, precision, balance=balance, unit_cap=cap, reorder=reorder)
        assert_bit_exact(C, A, v, B, precision)
    else:
        v = gen.values_uniform(A.nnz, seed)
        B = gen.dense_normal(K, N, seed + 1)
        C, _ = run(A, v, B, precision, balance=balance, unit_cap=cap, reorder=reorder)
        assert_within(C, A, v, B, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("shape", ["graph", "road"])
def test_permute_cols_exact(precision, shape):
    """Symmetric reordering (permute_cols): the columns are relabelled with the
    rows, the device SparseAToB keeps original ids, so no B' = B[perm] pass runs (only the TF32
    pre-round at high reuse); integer data bit-exact, floats within tolerance."""
    if shape == "graph":
        A = gen.dcsbm(5000, 250_000, 6, 2.2, 0.15, 3000, seed=8, oversample=1.3)
    else:
        A = gen.road_grid(200, 0.7, seed=8)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 128, 2)
    C, p = run(A, v, B, precision, reorder="on", permute_cols=True)
    pre = precision == "tf32" and p.info["sum_U"] >= 32 * A.K
    assert p.info["cols_permuted"] == 1 and p.launches_per_execute == (2 if pre else 1)
    assert_bit_exact(C, A, v, B, precision)
    vf = gen.values_uniform(A.nnz, 3)
    Bf = gen.dense_normal(A.K, 256, 4)
    Cf, _ = run(A, vf, Bf, precision, reorder="on", permute_cols=True)
    assert_within(Cf, A, vf, Bf, precision)


def test_permute_cols_partitions_and_device_build():
    import torch
    A = gen.dcsbm(4000, 200_000, 6, 2.2, 0.2, 2500, seed=6, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 64, 2)
    Cfull, _ = run(A, v, B, "tf32", reorder="on", permute_cols=True)
    out = torch.full((A.M, 64), float("nan"), device="cuda")
    for part in range(3):
        for build in ("host", "device"):
            p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, reorder="on", permute_cols=True, part=part, nparts=3,
                         build=build)
            G = p.execute(to_dev_B(B, "tf32"))
            rows = torch.from_numpy(p.export_rows().astype(np.int64)).cuda()
            out[rows] = G
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), Cfull)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_execute_is_cuda_graph_capturable(precision):
    """After one warm-up call (workspace / scratch allocation, kernel attributes), execute
    issues only kernel launches on the given stream: it can be captured into a CUDA graph and
    replayed (launch overhead matters for small matrices, e.g. the DD shape at ~80 us)."""
    import torch
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=7, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B0 = gen.dense_int(A.K, 128, 2)
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", balance="on", unit_cap=32)
    Bd = to_dev_B(B0, precision)
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
    assert_bit_exact(C.cpu().numpy(), A, v, B0, precision)
    B1 = gen.dense_int(A.K, 128, 3)
    Bd.copy_(to_dev_B(B1, precision))
    g.replay()
    torch.cuda.synchronize()
    assert_bit_exact(C.cpu().numpy(), A, v, B1, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("P", [1, 3])
def test_fused_allgather_epilogue(precision, P):
    """accspmm_execute_allgather on one GPU with several local destinations standing in for
    the ranks' C: every part's rows land in every destination in original row order, so after
    all P parts each destination is the whole product (integer data: bit-exact)."""
    import torch
    A = gen.dcsbm(4000, 200_000, 6, 2.2, 0.2, 2500, seed=2, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 256, 2)
    Bd = to_dev_B(B, precision)
    dsts = [torch.full((A.M, 256), float("nan"), device="cuda") for _ in range(3)]
    for part in range(P):
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", balance="on",
                     unit_cap=32, part=part, nparts=P)
        p.execute_allgather(Bd, dsts)
    torch.cuda.synchronize()
    for d in dsts:
        assert_bit_exact(d.cpu().numpy(), A, v, B, precision)
    with pytest.raises(acc.AccSpmmError):
        acc.accspmm_execute_allgather(p.handle, Bd.data_ptr(), 256, [])


def test_products_hub_rows_balancer_stress():
    """SURVEY §8(d) P adversarial variant (8 rows of 200K nnz on the products shape): the hub
    windows are split into many segments and reduced by the deterministic fixup; the hub rows
    and a random row sample match the oracle, and balance on = balance off bitwise on the hubs
    (integer data)."""
    cfg, A = gen.make_config("products_hubs")
    nnz_row = np.diff(A.rowptr)
    hubs = np.nonzero(nnz_row >= 200_000)[0]
    assert hubs.size == 8
    rows = np.union1d(hubs, _sample_rows(A.M, 2000, 3))
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, 128, cfg.seed_B)
    C, p = run(A, v, B, "tf32", reorder="auto", build="device")
    assert p.info["balanced"] == 1 and p.info["n_split_windows"] > 0
    assert_within(C, A, v, B, "tf32", rows=rows)
    vi = gen.values_int(A.nnz, 2)
    Bi = gen.dense_int(A.K, 64, 3)
    Con, _ = run(A, vi, Bi, "tf32", balance="on", build="device")
    Coff, _ = run(A, vi, Bi, "tf32", balance="off", build="device")
    assert np.array_equal(Con[hubs], Coff[hubs])
    Cr, _ = oracle(A, vi, Bi, "tf32", rows=hubs)
    assert np.array_equal(Con[hubs].astype(np.float64), Cr)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("N", [1, 7, 24, 100, 602])
def test_any_feature_width_padded(precision, N):
    """N % 16 != 0 (e.g. Reddit's 602 input features) goes through the padded copies; integer
    data bit-exact, split windows and reordering included, through the device and host APIs."""
    import torch
    A = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=N, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, N, 2)
    C, p = run(A, v, B, precision, reorder="on", balance="on", unit_cap=32)
    assert C.shape == (A.M, N)
    assert_bit_exact(C, A, v, B, precision)
    hdt = np.float16 if precision == "fp16" else np.float32
    Ch = np.full((A.M, N), np.nan, np.float32)
    p.execute_host(np.ascontiguousarray(B.astype(hdt)), Ch)
    assert np.array_equal(Ch, C)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_zero_width_inner_dimension(precision):
    """K = 0 (B has no rows): no TC block exists, C is all zeros, including the fused all-gather."""
    import torch
    A = gen.Csr(21, 0, np.zeros(22, np.int64), np.zeros(0, np.int32))
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, np.zeros(0, np.float32), precision=precision)
    dt = torch.float16 if precision == "fp16" else torch.float32
    B = torch.zeros((0, 32), dtype=dt, device="cuda")
    C = torch.full((21, 32), float("nan"), device="cuda")
    p.execute(B, C)
    D = torch.full((21, 32), float("nan"), device="cuda")
    p.execute_allgather(B, [D])
    torch.cuda.synchronize()
    assert torch.all(C == 0) and torch.all(D == 0)
