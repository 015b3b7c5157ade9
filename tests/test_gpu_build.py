"""GPU: the device-side BitTCF builder (build="device", kernels/build_sm100.cu).

The device builder must produce the paper's BitTCF bit for bit: every exported
array equals the oracle's independent encoder (oracle/bittcf.py) and the host builder, for
both precisions, with reordering, partitions, ragged/empty windows and special values; the
SpMM through a device-built plan is then bitwise identical to the host-built plan's.
"""
import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from gpu_util import assert_bit_exact, assert_within, to_dev_B
from oracle import bittcf as bt
from oracle.rounding import rho

pytestmark = pytest.mark.gpu

KEYS = ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()
    from paper_2501_09251_b200 import _build
    _build.build()


def _pair(A, v, precision, **kw):
    kw.setdefault("reorder", "off")
    ph = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, build="host", **kw)
    pd = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, build="device", **kw)
    return ph, pd


def _same_format(ph, pd):
    Fh, Fd = ph.export_format(), pd.export_format()
    for k in KEYS:
        assert np.array_equal(Fh[k], Fd[k]), k
    assert Fh["values"].view(np.uint8).tobytes() == Fd["values"].view(np.uint8).tobytes()
    for k in ("W", "NB", "plan_nnz", "sum_U", "n_units", "n_split_windows", "rows", "ibd"):
        assert ph.info[k] == pd.info[k], k
    assert np.array_equal(ph.export_units(), pd.export_units())
    return Fd


def _run(p, B, precision):
    import torch
    C = torch.full((p.out_rows, B.shape[1]), float("nan"), device="cuda")
    p.execute(to_dev_B(B, precision), C)
    torch.cuda.synchronize()
    return C.cpu().numpy()


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("shape", [(1003, 777, 20000), (8, 8, 64), (700, 900, 9000), (5, 3, 7), (4096, 100, 30000)])
def test_device_build_equals_oracle_encoder(precision, shape):
    M, K, nnz = shape
    A = gen.uniform_random(M, K, nnz, seed=M + K)
    v = gen.values_uniform(A.nnz, 3)
    ph, pd = _pair(A, v, precision)
    Fd = _same_format(ph, pd)
    ref = bt.encode(A.M, A.K, A.rowptr, A.colidx, rho(v, precision))
    for k in KEYS:
        assert np.array_equal(Fd[k], ref[k]), k
    assert np.array_equal(Fd["values"].astype(np.float32), ref["values"].astype(np.float32))


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
def test_device_build_special_values_bit_exact(precision):
    """rho on the device follows the host rule on NaN payloads, Inf, ties and overflow."""
    A = gen.uniform_random(64, 64, 600, seed=1)
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 32, A.nnz, dtype=np.uint64).astype(np.uint32)
    special = np.array([0x7F800000, 0xFF800000, 0x7FC00001, 0x7F800001, 0xFFFFFFFF, 0x7F7FFFFF, 0x00001000,
                        0x3F801000, 0x47800000, 0x477FF000, 0x33000000, 0x80000000], np.uint32)
    bits[:len(special)] = special
    v = bits.view(np.float32)
    ph, pd = _pair(A, v, precision)
    _same_format(ph, pd)


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
def test_device_build_empty_and_degenerate(precision):
    for A in (gen.csr_from_pairs(np.array([], np.int64), np.array([], np.int64), 19, 5),
              gen.csr_from_pairs(np.array([3, 3, 17]), np.array([0, 4, 2]), 21, 5),
              gen.identity(8), gen.star(300)):
        v = gen.values_uniform(A.nnz, 1)
        ph, pd = _pair(A, v, precision)
        _same_format(ph, pd)
        if A.M:
            B = gen.dense_normal(A.K, 32, 2)
            assert np.array_equal(_run(ph, B, precision), _run(pd, B, precision))


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("reorder,nparts", [("on", 1), ("off", 3), ("on", 4)])
def test_device_build_reorder_partitions(precision, reorder, nparts):
    A = gen.dcsbm(4000, 200_000, 6, 2.2, 0.2, 2500, seed=5, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 64, 2)
    for part in range(nparts):
        ph, pd = _pair(A, v, precision, reorder=reorder, part=part, nparts=nparts)
        _same_format(ph, pd)
        assert np.array_equal(ph.export_rows(), pd.export_rows())
        assert np.array_equal(_run(ph, B, precision), _run(pd, B, precision))
    if nparts == 1:
        assert_bit_exact(_run(pd, B, precision), A, v, B, precision)


def test_device_build_parity_vs_oracle_float():
    A = gen.dcsbm(6000, 400_000, 8, 2.3, 0.25, 3000, seed=9, oversample=1.3)
    v = gen.values_uniform(A.nnz, 4)
    B = gen.dense_normal(A.K, 128, 5)
    pd = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision="tf32", build="device", reorder="on")
    assert_within(_run(pd, B, "tf32"), A, v, B, "tf32")


def test_device_build_reddit_shaped_equals_host():
    """The Reddit-shaped benchmark matrix (configs[2]): device and host builds are identical."""
    cfg, A = gen.make_config("reddit")
    v = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    ph, pd = _pair(A, v, "tf32")
    _same_format(ph, pd)
    assert pd.info["ms_build"] < ph.info["ms_build"]


def test_device_build_requires_device():
    A = gen.identity(16)
    with pytest.raises(acc.AccSpmmError):
        acc.Plan(A.M, A.K, A.rowptr, A.colidx, np.ones(16, np.float32), build="device", device=-1)


@pytest.mark.gpu
def test_l2_probe_both_engines():
    """L2 read-bandwidth probe (the roofline denominator of bench.py): both request engines give
    a bandwidth above the HBM copy bandwidth and below the L2's physical ceiling (a 96 MiB buffer
    is L2-resident on the B200's 126 MB L2), and mode 0 is the larger of the two."""
    ldg = acc.accspmm_probe_l2_bandwidth_ex(96 << 20, 20, mode=1)
    tma = acc.accspmm_probe_l2_bandwidth_ex(96 << 20, 20, mode=2)
    best = acc.accspmm_probe_l2_bandwidth_ex(96 << 20, 20, mode=0)
    for g in (ldg, tma, best):
        assert 7000.0 < g < 60000.0, (ldg, tma, best)
    assert best >= 0.9 * max(ldg, tma), (ldg, tma, best)
