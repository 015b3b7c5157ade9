"""Tuning sweep (GPU box): one matrix, many plan/kernel variants, CUDA-event timing per variant.

usage: python tools/sweep.py --config reddit --N 128 --variants 'kcfg=0' 'kcfg=1,cap=256' ...
variant keys: kcfg (ACCSPMM_KCFG), fw (ACCSPMM_FW), b3 (ACCSPMM_B3), hot (hot_cols plan option),
hmb / hl2 (ACCSPMM_HOT_MB / ACCSPMM_HOT_L2_MB), rb (ACCSPMM_ROUND_B: 1 pass, 2 in-kernel), cap, balance, reorder, precision, N
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the A/B knobs and kernel variants exist only in the measurement build
os.environ.setdefault("ACCSPMM_LIB", "variants")
import numpy as np
import torch

import gen
import paper_2501_09251_b200 as acc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--N", type=int, default=128)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--variants", nargs="+", default=["kcfg=0"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--rounds", type=int, default=1,
                    help="interleave the variants this many times (A B A B ...) and pool the samples: "
                         "clock/power drift over the run then hits every variant alike")
    a = ap.parse_args()
    cfg, A = gen.make_config(a.config)
    vals = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    Bs = {}
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    plans = {}
    res = []
    samples = {}
    for rnd, v in [(r, v) for r in range(a.rounds) for v in a.variants]:
        kv = dict(x.split("=") for x in v.split(",") if x)
        N = int(kv.get("N", a.N))
        prec = kv.get("precision", "tf32")
        os.environ["ACCSPMM_KCFG"] = kv.get("kcfg", "-1")
        os.environ["ACCSPMM_FW"] = kv.get("fw", "0")
        os.environ["ACCSPMM_SLICE_MAJOR"] = kv.get("sm", "1")
        os.environ["ACCSPMM_L2PROMO"] = kv.get("promo", "3")
        os.environ["ACCSPMM_L2_PERSIST"] = kv.get("persist", "0")
        os.environ["ACCSPMM_B3"] = kv.get("b3", "0")
        os.environ["ACCSPMM_HOT_MB"] = kv.get("hmb", "64")
        os.environ["ACCSPMM_ROUND_B"] = kv.get("rb", "0")
        os.environ["ACCSPMM_HOT_L2_MB"] = kv.get("hl2", "96")
        if "gcap" in kv:
            os.environ["ACCSPMM_GROUP_CAP"] = kv["gcap"]
        else:
            os.environ.pop("ACCSPMM_GROUP_CAP", None)
        key = (prec, kv.get("balance", "auto"), int(kv.get("cap", 0)), kv.get("reorder", "off"), kv.get("gcap"),
               int(kv.get("wh", 0)), kv.get("kernel", "auto"), kv.get("hot", "auto"))
        if key not in plans:
            t0 = time.perf_counter()
            plans[key] = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, precision=prec, balance=key[1],
                                  unit_cap=key[2], reorder=key[3], window_rows=key[5], kernel=key[6], hot_cols=key[7],
                                  build="device")
            plans[key].create_s = time.perf_counter() - t0
        p = plans[key]
        if (prec, N) not in Bs:
            B = gen.dense_normal(A.K, N, cfg.seed_B)
            Bs[(prec, N)] = torch.from_numpy(B).cuda().to(torch.float16 if prec == "fp16" else torch.float32)
        Bd = Bs[(prec, N)]
        C = torch.empty((A.M, N), device="cuda")
        for _ in range(3):
            p.execute(Bd, C)
        ts = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(Bd, C)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        samples.setdefault(v, []).extend(ts)
        if rnd < a.rounds - 1:
            continue
        ts = samples[v]
        ms = float(np.median(ts))
        bm = acc.bytes_model(p.info, N)
        r = {"variant": v, "ms": ms, "ms_min": float(min(ts)), "samples": len(ts), "GFLOPs": bm["flops"] / ms / 1e6,
             "model_GBs": bm["total"] / ms / 1e6, "NB": p.info["NB"], "sum_U": p.info["sum_U"],
             "units": p.info["n_units"], "cap": p.info["unit_cap"], "balanced": p.info["balanced"],
             "split": p.info["n_split_windows"], "reorder_ms": p.info["ms_reorder"],
             "create_s": round(p.create_s, 2), "reorder_applied": p.info["reorder_applied"],
             "hot_cols": p.info["hot_cols"]}
        print(json.dumps(r), flush=True)
        res.append(r)
    if a.out:
        with open(a.out, "w") as f:
            for r in res:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
