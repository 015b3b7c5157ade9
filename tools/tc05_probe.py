"""Quick GPU probe of the tcgen05 kernel: parity vs the FP64 oracle on small cases + Reddit timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import gen
import paper_2501_09251_b200 as acc
from gpu_util import oracle, to_dev_B
from oracle import spmm as osp


def case(name, A, v, B, **kw):
    try:
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, v, **kw)
        C = torch.full((p.out_rows, B.shape[1]), float("nan"), device="cuda")
        p.execute(to_dev_B(B, "tf32"), C)
        torch.cuda.synchronize()
        Cg = C.cpu().numpy()
        Cr, S = oracle(A, v, B, "tf32")
        rep = osp.check(Cg, Cr, S, "tf32")
        exact = np.array_equal(Cg.astype(np.float64), Cr)
        print(name, kw, "ok" if rep["ok"] else "FAIL", "exact" if exact else "", rep["max_err_over_tol"],
              rep["violations"], "nan", int(np.isnan(Cg).sum()), flush=True)
    except Exception as e:
        print(name, kw, "EXC", repr(e)[:300], flush=True)


def main():
    A = gen.uniform_random(1003, 777, 20000, seed=1)
    v = gen.values_uniform(A.nnz, 5)
    B = gen.dense_normal(A.K, 128, 6)
    for wh in (8, 16, 32):
        case("ragged", A, v, B, window_rows=wh, kernel="tcgen05", reorder="off", balance="off")
    Ai = gen.dcsbm(3000, 150_000, 5, 2.2, 0.2, 2000, seed=3, oversample=1.3)
    vi = gen.values_int(Ai.nnz, 1)
    Bi = gen.dense_int(Ai.K, 256, 2)
    for wh in (8, 16, 32):
        case("int", Ai, vi, Bi, window_rows=wh, kernel="tcgen05", reorder="off", balance="off")
        case("int-bal", Ai, vi, Bi, window_rows=wh, kernel="tcgen05", reorder="off", balance="on", unit_cap=32)
        case("int-reorder", Ai, vi, Bi, window_rows=wh, kernel="tcgen05", reorder="on")
    if len(sys.argv) > 1:
        cfg, R = gen.make_config("reddit")
        vals = gen.values_uniform(R.nnz, cfg.seed_A + 1)
        Bd = torch.from_numpy(gen.dense_normal(R.K, 128, cfg.seed_B)).cuda()
        flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
        perm = None
        for wh, kern in ((8, "mma_sync"), (8, "tcgen05"), (16, "tcgen05"), (32, "tcgen05")):
            t0 = time.time()
            p = acc.Plan(R.M, R.K, R.rowptr, R.colidx, vals, window_rows=wh, kernel=kern, reorder="auto",
                         build="device")
            C = torch.empty((R.M, 128), device="cuda")
            for _ in range(3):
                p.execute(Bd, C)
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                p.execute(Bd, C)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            i = p.info
            rows = np.random.default_rng(0).choice(R.M, 2000, replace=False)
            Cr, S = oracle(R, vals, gen.dense_normal(R.K, 128, cfg.seed_B), "tf32", rows=np.sort(rows))
            rep = osp.check(C.cpu().numpy()[np.sort(rows)], Cr, S, "tf32")
            print("reddit", wh, kern, "ms %.3f" % np.median(ts), "min %.3f" % min(ts), "NB", i["NB"], "sumU", i["sum_U"],
                  "units", i["n_units"], "plan %.1fs" % (time.time() - t0), "ok", rep["ok"], rep["max_err_over_tol"],
                  flush=True)
            del p


if __name__ == "__main__":
    main()
