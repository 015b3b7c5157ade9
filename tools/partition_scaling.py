"""Per-partition execute times on ONE GPU -> projected multi-GPU strong scaling.

For P in {1, 2, 4, 8}: build the nnz-balanced sub-plans (part k of P, exactly what rank k of a
P-GPU run builds), time each part's execute alone (CUDA events, L2 flushed between reps,
median of R), and report max_k t_k -- the step time of a P-GPU run if the GPUs do not interfere
(B broadcast excluded: it is once per B) -- and t_1 / max_k t_k.  Evidence for the partition's
balance, not a multi-GPU measurement.
usage: python tools/partition_scaling.py <config> <N> [reps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_2501_09251_b200 as acc

name, N = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfg, A = gen.make_config(name)
vals = gen.values_uniform(A.nnz, cfg.seed_A + 1)
reorder = os.environ.get("REORDER", "auto")
B = torch.from_numpy(gen.dense_normal(A.K, N, cfg.seed_B)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
out = {"config": name, "N": N, "nnz": A.nnz, "reorder": reorder, "parts": {}}
t1 = None
for P in (1, 2, 4, 8):
    times, nnzs = [], []
    for k in range(P):
        p = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, reorder=reorder, part=k, nparts=P, build="device")
        C = torch.empty((p.out_rows, N), device="cuda")
        for _ in range(2):
            p.execute(B, C)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(B, C)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        times.append(float(np.median(ts)))
        nnzs.append(int(p.info["plan_nnz"]))
        del p, C
        torch.cuda.empty_cache()
    tmax = max(times)
    if P == 1:
        t1 = tmax
    out["parts"][P] = {"ms_per_part": [round(t, 4) for t in times], "nnz_per_part": nnzs, "max_ms": round(tmax, 4),
                       "projected_speedup": round(t1 / tmax, 3), "projected_GFLOPs": 2.0 * A.nnz * N / (tmax * 1e-3) / 1e9}
    print(P, out["parts"][P], flush=True)
print(json.dumps(out))
