"""Helpers for the GPU parity tests: run the CUDA path through the C ABI, compute the oracle."""
import numpy as np

import paper_2501_09251_b200 as acc
from oracle import spmm as osp
from oracle.rounding import rho

NAN_BITS = 0x7FC00000


def to_dev_B(B, precision):
    import torch
    if precision == "fp16":
        return torch.from_numpy(np.ascontiguousarray(B.astype(np.float16))).cuda()
    return torch.from_numpy(np.ascontiguousarray(B, dtype=np.float32)).cuda()


def run(A, vals, B, precision="tf32", **kw):
    """C from the CUDA path (canary-filled output, so unwritten elements show up as NaN)."""
    import torch
    kw.setdefault("reorder", "off")   # fixtures pin the un-reordered format unless they ask
    p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, precision=precision, **kw)
    Bd = to_dev_B(B, precision)
    rows = p.out_rows
    C = torch.full((rows, B.shape[1]), float("nan"), dtype=torch.float32, device="cuda")
    p.execute(Bd, C)
    torch.cuda.synchronize()
    out = C.cpu().numpy()
    return out, p


def oracle(A, vals, B, precision, rows=None):
    return osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, rho(vals, precision), rho(B, precision), rows=rows)


def assert_within(Cg, A, vals, B, precision, rows=None):
    Cr, S = oracle(A, vals, B, precision, rows=rows)
    got = Cg if rows is None else Cg[rows]
    rep = osp.check(got, Cr, S, precision)
    assert rep["ok"], rep
    return rep


def assert_bit_exact(Cg, A, vals, B, precision):
    Cr, _ = oracle(A, vals, B, precision)
    assert np.isfinite(Cg).all()
    assert np.array_equal(Cg.astype(np.float64), Cr), np.argwhere(Cg.astype(np.float64) != Cr)[:5]
