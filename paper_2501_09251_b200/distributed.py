"""Multi-GPU plumbing for the SpMM path: one process per GPU, torch.distributed for collectives.

Row windows are independent, so the path shards without a reduction:
rank k builds a sub-plan of the nnz-balanced RowWindow range [b_k, b_{k+1})
(``accspmm_plan_create_ex`` with part = k, nparts = P; BASELINE north_star), B is
broadcast once from rank 0 (NCCL over NVLink on the GPU box), each rank writes its
C slab in reordered-row order, and the optional all-gather of padded slabs plus
``accspmm_unpermute`` (a device kernel) restores C in original row order.

The fused alternative to that all-gather (``spmm_allgather_fused``): C lives in symmetric
memory (torch.distributed._symmetric_memory, peer-mapped over NVLink), and every rank's SpMM
epilogue writes its rows straight into every rank's C in original row order
(``accspmm_execute_allgather``) -- the exchange overlaps the compute window by window, with
no collective and no un-permute pass; a device-side barrier closes the step.

This module only moves data between ranks and calls the C ABI; the SpMM and the
un-permute run in libaccspmm's CUDA kernels.
"""
from __future__ import annotations

import numpy as np

from . import Plan, accspmm_reorder, accspmm_unpermute

PAD = -1  # row id of a padding row in a gathered slab (0xFFFFFFFF as uint32)


def rank_plan(M, K, rowptr, colidx, vals, rank: int, world: int, **plan_kw) -> Plan:
    """This rank's sub-plan: RowWindows [b_rank, b_rank+1) of the nnz-balanced partition."""
    return Plan(M, K, rowptr, colidx, vals, part=rank, nparts=world, **plan_kw)


def broadcast_perm(M: int, rowptr, colidx, src: int = 0, group=None, device=None):
    """Alg. 1 once: rank ``src`` computes the permutation (accspmm_reorder; the parallel variant
    of reading R21 above 8M vertices) and broadcasts it, so preprocessing does not replicate the
    reordering on every rank.  Returns u32[M] new -> old on every rank."""
    import torch
    import torch.distributed as dist
    if dist.get_rank(group) == src:
        t = torch.from_numpy(accspmm_reorder(M, rowptr, colidx).astype(np.int64))
    else:
        t = torch.empty(M, dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    dist.broadcast(t, src=src, group=group)
    return t.cpu().numpy().astype(np.uint32)


def broadcast_B(B, src: int = 0, group=None):
    """B is needed on every rank; broadcast it once (outside any timed step)."""
    import torch.distributed as dist
    dist.broadcast(B, src=src, group=group)
    return B


def gather_slabs(C_slab, orig_rows, group=None):
    """All-gather every rank's C slab (rows x N) and its original row ids.

    Slabs are padded to the largest slab (``all_gather_into_tensor`` needs equal chunks);
    padding rows carry id PAD.  Returns (G[P*max_rows, N], ids[P*max_rows]) on C_slab's device.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rows, N = C_slab.shape
    mx = torch.tensor([rows], dtype=torch.int64, device=C_slab.device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    mx = int(mx.item())
    padded = torch.zeros((mx, N), dtype=C_slab.dtype, device=C_slab.device)
    padded[:rows] = C_slab
    ids = torch.full((mx,), PAD, dtype=torch.int32, device=C_slab.device)
    ids[:rows] = torch.as_tensor(np.asarray(orig_rows, dtype=np.uint32).view(np.int32), device=C_slab.device)
    G = torch.empty((world * mx, N), dtype=C_slab.dtype, device=C_slab.device)
    I = torch.empty((world * mx,), dtype=torch.int32, device=C_slab.device)
    dist.all_gather_into_tensor(G, padded, group=group)
    dist.all_gather_into_tensor(I, ids, group=group)
    return G, I


def unpermute(G, ids, M: int, stream=None):
    """C[ids[i]] = G[i] on the device (K6 kernel); padding rows skipped.  CUDA tensors only."""
    import torch
    if not G.is_cuda:
        raise RuntimeError("accspmm unpermute runs on the GPU only (no CPU fallback)")
    C = torch.empty((M, G.shape[1]), dtype=torch.float32, device=G.device)
    s = torch.cuda.current_stream(G.device).cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)
    accspmm_unpermute(G.data_ptr(), ids.data_ptr(), G.shape[0], G.shape[1], C.data_ptr(), s)
    return C


def _stream_ctx(stream):
    """Runs the enclosed collectives on ``stream`` (NCCL and symmetric-memory barriers are issued
    on the current stream), so they are ordered after the SpMM launched there."""
    import contextlib

    import torch
    if stream is None or not hasattr(stream, "cuda_stream"):
        return contextlib.nullcontext()
    return torch.cuda.stream(stream)


def spmm_all(plan: Plan, B, M: int, stream=None):
    """Execute this rank's slab and assemble the full C on every rank (all-gather + un-permute),
    everything ordered on ``stream`` (default: the current stream)."""
    with _stream_ctx(stream):
        C_slab = plan.execute(B, stream=stream)
        G, I = gather_slabs(C_slab, plan.export_rows())
        return unpermute(G, I, M, stream)


class FusedAllGather:
    """Symmetric-memory C (M x N float32) shared by the ranks of ``group`` and the peer views
    the fused epilogue writes into.  Allocate once, reuse for every step."""

    def __init__(self, M: int, N: int, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.group = group or dist.group.WORLD
        self.C = symm.empty(M, N, dtype=torch.float32, device=device)
        self.hdl = symm.rendezvous(self.C, self.group)
        world = dist.get_world_size(self.group)
        self.views = [self.hdl.get_buffer(r, (M, N), torch.float32) for r in range(world)]
        self.hdl.barrier()

    def step(self, plan: Plan, B, stream=None):
        """C = A . B on every rank: this rank's rows are written into all ranks' C, then a
        device barrier waits for every rank's rows.  A barrier before the epilogue writes
        keeps a fast rank's step t+1 from overwriting a peer's C while that peer is still
        consuming step t (write-after-read across ranks).  Both barriers and the SpMM are
        ordered on ``stream`` (default: the current stream)."""
        with _stream_ctx(stream):
            self.hdl.barrier()
            plan.execute_allgather(B, self.views, stream)
            self.hdl.barrier()
        return self.C


def spmm_allgather_fused(plan: Plan, B, M: int, group=None, stream=None):
    """One-shot fused all-gather (allocates the symmetric C; use FusedAllGather to reuse it)."""
    return FusedAllGather(M, B.shape[1], B.device, group).step(plan, B, stream)
