"""GPU parity of hot-column plans (reading R22, DESIGN.md §3/§6): the format is built on the
columns relabelled by in-degree, the device SparseAToB holds original column ids with a hotness
tag on every block's lane 0, and the kernel picks each block's L2 policy from the tag.  The
product must stay exactly C = A . rho(B): integer data bit-exact (split windows, reordering,
partitions, FP16), floats within tau, and the device plan exports the same paper-format arrays
as the host builder."""
import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from gpu_util import assert_bit_exact, assert_within, run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()


def _skewed(seed=0, n=6000):
    return gen.powerlaw_directed(n, 14.0, seed=seed)


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("kw", [{}, {"reorder": "on"}, {"balance": "on", "unit_cap": 32}, {"build": "device"}])
def test_hot_cols_integer_bit_exact(precision, kw):
    A = _skewed(seed=1)
    v = gen.values_int(A.nnz, 2)
    for N in (64, 256):
        B = gen.dense_int(A.K, N, 3)
        C, p = run(A, v, B, precision, hot_cols="on", **kw)
        assert p.info["hot_cols"] == 1
        assert_bit_exact(C, A, v, B, precision)


def test_hot_cols_float_and_partitions():
    import torch
    A = _skewed(seed=4)
    v = gen.values_uniform(A.nnz, 5)
    B = gen.dense_normal(A.K, 128, 6)
    C, _ = run(A, v, B, "tf32", hot_cols="on", reorder="on")
    assert_within(C, A, v, B, "tf32")
    Bd = torch.from_numpy(B).cuda()
    whole = torch.from_numpy(C).cuda()
    for nparts in (2, 3):
        for part in range(nparts):
            p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision="tf32", reorder="on", hot_cols="on",
                         part=part, nparts=nparts, device=0)
            Cs = p.execute(Bd)
            rows = torch.from_numpy(p.export_rows().astype(np.int64)).cuda()
            assert torch.equal(Cs, whole[rows]) or torch.allclose(Cs, whole[rows], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
def test_hot_cols_device_plan_exports_paper_format(precision):
    """The device SparseAToB holds original ids + tags; the export maps them back, so a device
    plan (either builder) exports exactly the host plan's format of the relabelled matrix."""
    A = _skewed(seed=7)
    v = gen.values_uniform(A.nnz, 8)
    ref = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", hot_cols="on",
                   device=-1).export_format()
    for build in ("host", "device"):
        F = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder="on", hot_cols="on",
                     device=0, build=build).export_format()
        for k, r in ref.items():
            if isinstance(r, np.ndarray) and r.ndim:
                assert np.array_equal(np.asarray(F[k]).view(np.uint8), r.view(np.uint8)), (build, k)
            else:
                assert F[k] == r, (build, k)


def test_permute_cols_gathers_original_rows():
    """permute_cols now keeps original ids in the device SparseAToB: no B' = P B pass runs
    (one launch per execute at low reuse), and the product is unchanged."""
    A = gen.dcsbm(3000, 80_000, 6, 2.2, 0.1, 800, seed=5, oversample=1.3)
    v = gen.values_int(A.nnz, 1)
    B = gen.dense_int(A.K, 64, 2)
    C, p = run(A, v, B, "tf32", reorder="on", permute_cols=True, balance="on", unit_cap=32)
    assert p.info["cols_permuted"] == 1
    assert_bit_exact(C, A, v, B, "tf32")
