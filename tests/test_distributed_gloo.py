"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing: per-rank sub-plans, B broadcast,
padded all-gather of slabs + row ids, reconstruction of C (reading R9).

The slab products here come from the FP64 oracle (the CUDA path cannot run on CPU);
what is tested is the host/collective logic around it.  The device un-permute kernel
is covered by tests/test_gpu_parity.py::test_reordered_partitions_and_unpermute.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, reorder, result_q):
    import torch
    import torch.distributed as dist

    import gen
    from oracle import spmm as osp
    from oracle.rounding import rho
    from paper_2501_09251_b200 import distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        A = gen.sbm(600, 12, 0.2, 0.01, seed=3)
        vals = gen.values_uniform(A.nnz, 4)
        N = 32
        B = torch.from_numpy(gen.dense_normal(A.K, N, 5)) if rank == 0 else torch.zeros((A.K, N))
        D.broadcast_B(B, src=0)
        plan = D.rank_plan(A.M, A.K, A.rowptr, A.colidx, vals, rank, world, reorder=reorder, device=-1)
        if reorder != "off":
            # Alg. 1 once on rank 0, broadcast: the same sub-plan as reordering on every rank
            perm = D.broadcast_perm(A.M, A.rowptr, A.colidx)
            plan_b = D.rank_plan(A.M, A.K, A.rowptr, A.colidx, vals, rank, world, reorder=reorder, device=-1,
                                 perm=perm)
            assert np.array_equal(plan_b.export_rows(), plan.export_rows())
            for k in ("RowWindowOffset", "TCOffset", "SparseAToB", "TCLocalBit"):
                assert np.array_equal(plan_b.export_format()[k], plan.export_format()[k])
        info = plan.info
        rows = plan.export_rows()
        assert info["nparts"] == world and info["part"] == rank and len(rows) == info["rows"]
        # this rank's slab via the oracle (stand-in for the device execute)
        a = rho(vals, "tf32")
        b = rho(B.numpy(), "tf32")
        slab, _ = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows.astype(np.int64))
        G, I = D.gather_slabs(torch.from_numpy(slab.astype(np.float32)), rows)
        C = np.zeros((A.M, N), np.float32)
        ids = I.numpy()
        keep = ids != D.PAD
        C[ids[keep].view(np.uint32)] = G.numpy()[keep]
        full, _ = osp.spmm_fp64(A.M, A.K, A.rowptr, A.colidx, a, b)
        ok = np.array_equal(C, full.astype(np.float32)) and int(keep.sum()) == A.M
        seen = np.sort(ids[keep].view(np.uint32))
        ok = ok and np.array_equal(seen, np.arange(A.M, dtype=np.uint32))
        result_q.put((rank, bool(ok), int(info["rows"]), int(info["plan_nnz"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("reorder", ["off", "on"])
def test_two_rank_gloo_partition_broadcast_gather(reorder):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, reorder, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [r[1] for r in res] == [True, True], res
    total_rows = sum(r[2] for r in res)
    assert total_rows == 600
    # nnz-balanced: neither rank holds more than half the nnz plus one window's worth
    assert abs(res[0][3] - res[1][3]) < 0.2 * (res[0][3] + res[1][3])
    for p in procs:
        assert p.exitcode == 0


def test_unpermute_refuses_cpu_tensors():
    import torch
    from paper_2501_09251_b200 import distributed as D
    with pytest.raises(RuntimeError):
        D.unpermute(torch.zeros((4, 4)), torch.zeros(4, dtype=torch.int32), 4)


_ = os
