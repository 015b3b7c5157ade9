"""GPU: the autograd operator (paper_2501_09251_b200.autograd) -- forward C = A.B and
backward dB = A^T.dC both run the sm_100a kernel; checked against the FP64 oracle of A and
of A^T (A^T built here with scipy, independently of the library)."""
import numpy as np
import pytest
import scipy.sparse as sp

import gen
from gpu_util import assert_within, to_dev_B

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    torch.cuda.init()
    from paper_2501_09251_b200 import _build
    _build.build()


def _transpose(A, v):
    t = sp.csr_matrix((v, A.colidx, A.rowptr), shape=(A.M, A.K)).T.tocsr()
    t.sort_indices()
    return gen.Csr(A.K, A.M, t.indptr.astype(np.int64), t.indices.astype(np.int32)), t.data.astype(np.float32)


@pytest.mark.parametrize("precision", ["tf32", "fp16"])
@pytest.mark.parametrize("reorder", ["off", "on"])
def test_forward_backward_vs_oracle(precision, reorder):
    import torch
    from paper_2501_09251_b200.autograd import SparseOperator
    A = gen.dcsbm(3000, 120_000, 5, 2.2, 0.2, 1500, seed=2, oversample=1.3)
    A = gen.csr_from_pairs(A.row_ids()[A.colidx < 2500], A.colidx[A.colidx < 2500], A.M, 2500)  # non-square
    v = gen.values_uniform(A.nnz, 1)
    op = SparseOperator(A.M, A.K, A.rowptr, A.colidx, v, precision=precision, reorder=reorder)
    B0 = gen.dense_normal(A.K, 64, 2)
    W = gen.dense_normal(A.M, 64, 3)
    B = to_dev_B(B0, precision).requires_grad_(True)
    C = op @ B
    assert_within(C.detach().cpu().numpy(), A, v, B0, precision)
    (C * torch.from_numpy(W).cuda()).sum().backward()
    At, vt = _transpose(A, v)
    W_in = W.astype(np.float16).astype(np.float32) if precision == "fp16" else W
    g = B.grad.float().cpu().numpy()
    if precision == "fp16":  # the FP16 gradient is stored in B's dtype: compare with its rounding
        from oracle import spmm as osp
        from oracle.rounding import rho
        Cr, S = osp.spmm_fp64(At.M, At.K, At.rowptr, At.colidx, rho(vt, "fp16"), rho(W_in, "fp16"))
        assert np.all(np.abs(g - Cr) <= 4e-3 * S + 1e-6 + np.abs(Cr) * 2 ** -11)
    else:
        assert_within(g, At, vt, W_in, precision)


def test_input_checks():
    import torch
    from paper_2501_09251_b200.autograd import SparseOperator, spmm
    A = gen.identity(32)
    op = SparseOperator(32, 32, A.rowptr, A.colidx, np.ones(32, np.float32))
    with pytest.raises(ValueError):
        spmm(op, torch.zeros(31, 16, device="cuda"))
    with pytest.raises(TypeError):
        spmm(op, torch.zeros(32, 16, device="cuda", dtype=torch.float16))
    with pytest.raises(ValueError):
        spmm(op, torch.zeros(32, 16))
    x = torch.randn(32, 16, device="cuda")
    assert torch.equal(op @ x, x.float().contiguous()) or torch.allclose(op @ x, x, rtol=1e-3, atol=1e-6)
