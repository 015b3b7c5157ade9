"""Full-size parity on BASELINE configs[4] (papers100M-shaped: 111,059,956 rows, 1.61B nnz,
N = 64, TF32), streamed against the FP64 oracle -- for reorder off and
auto (Alg. 1 at this scale runs the parallel variant of reading R21).

The product is C = A . B exactly; the oracle recomputes C and the bound S for a
sample of rows: 1,000,000 uniformly drawn rows, every row with out-degree >= 500 and the
first and last rows, and each sampled GPU row must satisfy |C_gpu - C_ref| <= 1e-3*S + 1e-6.
Every other row is checked for finiteness (no NaN canary left, no Inf)."""
import os

import numpy as np
import pytest

import gen
import paper_2501_09251_b200 as acc
from oracle import spmm as osp
from oracle.rounding import rho

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
N = 64


@pytest.fixture(scope="module")
def config4():
    import torch
    torch.cuda.init()
    cfg, A = gen.make_config("papers100m")
    vals = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = rho(gen.dense_normal(A.K, N, cfg.seed_B), "tf32")   # rho is idempotent: the kernel re-rounds
    a = rho(vals, "tf32")
    rng = np.random.default_rng(4)
    deg = np.diff(A.rowptr)
    rows = np.unique(np.concatenate([rng.choice(A.M, 1_000_000, replace=False), np.nonzero(deg >= 500)[0],
                                     [0, A.M - 1]])).astype(np.int64)
    Cr, S = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, B, rows=rows)
    yield A, vals, B, rows, Cr, S
    del A, vals, B


@pytest.mark.parametrize("reorder", ["off", "auto"])
def test_config4_full_size_streamed(config4, reorder):
    import torch
    A, vals, B, rows, Cr, S = config4
    assert A.M == 111_059_956 and A.nnz > 1_600_000_000
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, precision="tf32", reorder=reorder, build="device")
    info = p.info
    if reorder == "auto":
        assert info["nb_unreordered"] > 0 and info["ms_reorder"] > 0
    Bd = torch.from_numpy(B).cuda()
    C = torch.full((A.M, N), float("nan"), device="cuda")
    p.execute(Bd, C)
    torch.cuda.synchronize()
    # finiteness of every row, chunked on the device
    for r0 in range(0, A.M, 8_000_000):
        assert bool(torch.isfinite(C[r0:r0 + 8_000_000]).all())
    got = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    rep = osp.check(got, Cr, S, "tf32")
    assert rep["ok"], rep
    print(f"\nconfigs[4] reorder={reorder}: {rows.size} rows checked, max err/tol {rep['max_err_over_tol']:.3g}, "
          f"reorder_applied={info['reorder_applied']} ms_reorder={info['ms_reorder']:.0f} NB={info['NB']} "
          f"NB_unreordered={info['nb_unreordered']}")
    del C, Bd, p
    torch.cuda.empty_cache()
    _ = os
