"""PyTorch autograd integration of the Acc-SpMM path (the paper's
future work "integrate ... into DGL").

``SparseOperator`` holds two plans of the library: one of A (forward C = A . B) and one of
A^T (backward dB = A^T . dC), the transpose built by ``accspmm_csr_transpose`` in the
library's C++.  ``op @ B`` (or ``spmm(op, B)``) is differentiable in B; A is a fixed
operator (a graph adjacency), so no gradient flows to its values.  Both directions run
the sm_100a SpMM kernel through the C ABI; this module only marshals arguments (shape
checks and, for FP16 plans, the cast of the incoming gradient to the plan's input type).
"""
from __future__ import annotations

import numpy as np
import torch

from . import Plan, accspmm_csr_transpose


class SparseOperator:
    """A fixed sparse M x K matrix usable as a differentiable left operand."""

    def __init__(self, M, K, rowptr, colidx, vals, precision="tf32", reorder="auto", balance="auto",
                 device=None, build="host"):
        kw = dict(precision=precision, reorder=reorder, balance=balance, build=build)
        if device is not None:
            kw["device"] = int(device)
        self.M, self.K, self.precision = int(M), int(K), precision
        self.fwd = Plan(M, K, rowptr, colidx, np.asarray(vals, np.float32), **kw)
        t_rowptr, t_colidx, t_vals = accspmm_csr_transpose(M, K, rowptr, colidx, vals)
        self.bwd = Plan(K, M, t_rowptr, t_colidx, t_vals, **kw)
        self.in_dtype = torch.float16 if precision == "fp16" else torch.float32

    def close(self):
        self.fwd.close()
        self.bwd.close()

    def __matmul__(self, B: torch.Tensor) -> torch.Tensor:
        return spmm(self, B)


class _SpMM(torch.autograd.Function):
    @staticmethod
    def forward(ctx, B, op):
        ctx.op = op
        ctx.b_dtype = B.dtype
        return op.fwd.execute(B.contiguous())

    @staticmethod
    def backward(ctx, dC):
        op = ctx.op
        if not ctx.needs_input_grad[0]:
            return None, None
        dB = op.bwd.execute(dC.to(op.in_dtype).contiguous())
        return dB.to(ctx.b_dtype), None


def spmm(op: SparseOperator, B: torch.Tensor) -> torch.Tensor:
    """C = A . B (float32 C); B is K x N on the plan's device, float32 (TF32 plans) or
    float16 (FP16 plans), any N >= 1 (N % 16 != 0 is padded inside the library)."""
    if B.dim() != 2 or B.shape[0] != op.K:
        raise ValueError(f"B must be {op.K} x N, got {tuple(B.shape)}")
    if B.dtype != op.in_dtype:
        raise TypeError(f"B must be {op.in_dtype} for a {op.precision} plan")
    if not B.is_cuda:
        raise ValueError("B must be a CUDA tensor (there is no CPU fallback)")
    return _SpMM.apply(B, op)
