#!/usr/bin/env python
"""bench.py -- SpMM GFLOP/s (2*nnz*N/t) and achieved bytes/s vs the B200 HBM roofline.

Default workload (BASELINE.json north_star target): the Reddit-shaped graph
(configs[2], 232,965 nodes, ~115M nnz, DC-SBM, labels shuffled) at N = 128, TF32.
One "step" = one accspmm_execute over the whole matrix (all §8(a) execute rows:
work fetch, A-stream load, B-row gather, bitmap decode, MMA, epilogue, split-window
fixup) with B and the plan resident in HBM; L2 is flushed (256 MiB write) between
timed steps.  Multi-GPU (torchrun): RowWindows are split into nnz-balanced ranges,
B is broadcast once over NCCL (outside the timed region), each rank computes its
C slab; time = max over ranks.  ``--impl reference`` times the FP64 oracle on the
host cores on a bounded row sample instead (the only other place oracle/ runs).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 256 << 20
METRIC = "SpMM GFLOP/s (2\u00b7nnz\u00b7N/t) and achieved HBM GB/s vs peak at N=128, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--N", type=int, default=128)
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp16"])
    ap.add_argument("--reorder", default="auto", choices=["off", "on", "auto"])
    ap.add_argument("--balance", default="auto", choices=["off", "on", "auto"])
    ap.add_argument("--unit-cap", type=int, default=0)
    ap.add_argument("--permute-cols", action="store_true", help="symmetric reordering: relabel columns too")
    ap.add_argument("--build", default="device", choices=["host", "device"], help="BitTCF builder")
    ap.add_argument("--allgather", default="none", choices=["none", "nccl", "fused"],
                    help="N > 1: also time assembling the full C on every rank (NCCL all-gather + "
                         "un-permute, or the fused epilogue into symmetric memory); reported as "
                         "'allgather', the headline value stays the slab step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu: warmup + steps, no extras")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(key):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(key)
    return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(args):
    import gen
    cfg, A = gen.make_config(args.config)
    vals = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, args.N, cfg.seed_B)
    return cfg, A, vals, B


def cpu_oracle_sample(A, vals, B, precision, seconds, seed=0, rounded=None):
    """The FP64 oracle as it stands, on the host cores, over a bounded random row sample
    (rho(A), rho(B) are computed once, outside the timed sample)."""
    from oracle import spmm as osp
    from oracle.rounding import rho
    a, b = rounded if rounded is not None else (rho(vals, precision), rho(B, precision))
    rng = np.random.default_rng(seed)
    nnz_row = np.diff(A.rowptr)
    N = B.shape[1]
    rows = np.sort(rng.choice(A.M, size=min(A.M, 256), replace=False))
    _, t = osp.timed_spmm(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows)
    rate = 2.0 * nnz_row[rows].sum() * N / max(t, 1e-9)
    target_flops = rate * seconds
    avg = 2.0 * nnz_row.mean() * N
    n = int(min(A.M, max(256, target_flops / max(avg, 1.0))))
    rows = np.sort(rng.choice(A.M, size=n, replace=False))
    _, t = osp.timed_spmm(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows)
    flops = 2.0 * nnz_row[rows].sum() * N
    return {"value": flops / t / 1e9, "unit": "GFLOP/s", "cores": osp.num_threads(), "kind": "oracle",
            "sample": f"{n} of {A.M} rows (random, seed {seed}), {int(nnz_row[rows].sum())} nnz, N={N}, "
                      f"FP64 CSR triple loop, {t:.2f} s"}, t


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle.rounding import rho
    cfg, A, vals, B = make_inputs(args)
    rounded = (rho(vals, args.precision), rho(B, args.precision))
    steps = []
    info = None
    per_step_seconds = max(0.25, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        cb, t = cpu_oracle_sample(A, vals, B, args.precision, per_step_seconds, seed=i, rounded=rounded)
        if i >= args.warmup:
            steps.append(cb["value"])
            info = cb
    value = statistics.median(steps)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, cfg, A, world),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": info["cores"], "kind": "oracle",
                         "sample": info["sample"]},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out, args)


def workload_config(args, cfg, A, world):
    return {"workload": f"{cfg.name}: {cfg.note}; N={args.N}, {args.precision}",
            "matrix": cfg.name, "baseline_config_index": cfg.baseline_index, "M": A.M, "K": A.K, "nnz": A.nnz,
            "N": args.N, "precision": args.precision, "reorder": args.reorder, "balance": args.balance,
            "permute_cols": bool(getattr(args, "permute_cols", False)),
            "l2": "none" if args.no_flush else f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
            "parallelism": f"rowwindow-nnz-partition x{world}"}


def kernel_name(args):
    """The SpMM kernel flavour the library's default dispatch picks."""
    kcfg = int(os.environ.get("ACCSPMM_KCFG", "-1"))
    g4 = kcfg < 0 or kcfg >= 20
    if not g4:
        return "spmm_bittcf_kernel (register-direct gather)"
    return "spmm_bittcf_g4_kernel (TMA gather4, " + ("1 warp/CTA)" if kcfg < 0 else "variant %d)" % kcfg)


def emit(out, args):
    line = json.dumps(out)
    print(line, flush=True)
    if args.json_out:
        with open(args.json_out, "w") as f:
            f.write(line + "\n")


def time_allgather(args, plan, Bd, A, stream, world, shared):
    """N > 1 extra: full C on every rank per step, NCCL (execute + all-gather + un-permute) or
    fused (epilogue writes into every rank's symmetric-memory C + device barrier).  Device
    time, max over ranks; failures are reported, not raised (the slab step is the headline)."""
    import torch
    import torch.distributed as dist
    from paper_2501_09251_b200 import distributed as D
    out = {"mode": args.allgather}
    try:
        steps = max(3, min(args.steps, 20))
        if args.allgather == "fused":
            fa = D.FusedAllGather(A.M, args.N, Bd.device)
            run = lambda: fa.step(plan, Bd, stream)  # noqa: E731
        else:
            run = lambda: D.spmm_all(plan, Bd, A.M, stream)  # noqa: E731
        for _ in range(2):
            run()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t = float(t.item())
        out.update({"ms_per_step": t / steps * 1e3, "value": 2.0 * A.nnz * args.N * steps / t / 1e9,
                    "unit": "GFLOP/s", "steps": steps})
    except Exception as e:  # reported beside the headline, never a silent substitute for it
        out["unavailable"] = repr(e)[:300]
    return out


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import paper_2501_09251_b200 as acc

    # ACCSPMM_BENCH_SHARED_GPU=1: every rank on cuda:0 over gloo (exercises the multi-rank
    # path on a one-GPU box; NCCL refuses two ranks per device).  Default: one GPU per rank, NCCL.
    shared = os.environ.get("ACCSPMM_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg, A, vals, B = make_inputs(args)
    t0 = time.perf_counter()
    plan = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, precision=args.precision, reorder=args.reorder,
                    balance=args.balance, unit_cap=args.unit_cap, part=rank, nparts=world, device=local,
                    permute_cols=args.permute_cols, build=args.build)
    plan_s = time.perf_counter() - t0
    info = plan.info
    tdt = torch.float16 if args.precision == "fp16" else torch.float32
    stream = torch.cuda.current_stream()
    # B lives on every GPU: rank 0's copy is broadcast once over NCCL (not timed as a step)
    Bd = torch.from_numpy(B).to(device="cuda", dtype=tdt) if rank == 0 or world == 1 else \
        torch.empty((A.K, args.N), dtype=tdt, device="cuda")
    bcast_ms = None
    if world > 1:
        torch.cuda.synchronize()
        tb = time.perf_counter()
        if shared:
            Bh = Bd.cpu()
            dist.broadcast(Bh, src=0)
            Bd.copy_(Bh)
        else:
            dist.broadcast(Bd, src=0)
        torch.cuda.synchronize()
        bcast_ms = (time.perf_counter() - tb) * 1e3
    C = torch.empty((plan.out_rows, args.N), dtype=torch.float32, device="cuda")
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        plan.execute(Bd, C, stream)
        if not args.no_flush:
            flush.zero_()
    torch.cuda.synchronize()

    l2_peak_before = acc.accspmm_probe_l2_bandwidth(96 << 20, 100)  # again after the loop: max of both
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    plan.set_timing(True)   # in-library CUDA events around the SpMM kernel launch (dominant kernel)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    tw = time.perf_counter()
    for i in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        ev[i][0].record(stream)
        plan.execute(Bd, C, stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - tw
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    kernel_ms = plan.kernel_times()
    plan.set_timing(False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_local = sum(step_ms) / 1e3
    t_max = t_local
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    flops_total = 2.0 * A.nnz * args.N * args.steps
    value = flops_total / t_max / 1e9
    ms_per_step = t_max / args.steps * 1e3

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_per_step, "value": value}))
        return

    allgather = None
    if world > 1 and args.allgather != "none":
        allgather = time_allgather(args, plan, Bd, A, stream, world, shared)

    # warm regime: the same steps back to back, no L2 flush in between
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0.record(stream)
    for _ in range(args.steps):
        plan.execute(Bd, C, stream)
    w1.record(stream)
    torch.cuda.synchronize()
    warm_ms = w0.elapsed_time(w1) / args.steps

    bm = acc.bytes_model(info, args.N)
    # the HBM lower bound of the gather -- every distinct column's B row once
    es_b = 2 if args.precision == "fp16" else 4
    bm["B_compulsory"] = int(es_b * args.N * np.count_nonzero(np.bincount(A.colidx, minlength=A.K)))
    avg_s = float(np.mean(kernel_ms)) / 1e3 if len(kernel_ms) else t_local / args.steps
    peak, peak_kind = load_peaks()
    achieved = bm["total"] / avg_s / 1e9
    traffic = load_traffic(f"{args.config}-N{args.N}-{args.precision}-{args.reorder}-{args.balance}-p{world}")
    # L2 roofline: every model byte (gathered B rows, A stream, C) passes through L2, and on
    # graphs whose B fits L2 the gather is served from there -- the binding resource
    l2_peak = max(acc.accspmm_probe_l2_bandwidth(96 << 20, 100), l2_peak_before)

    # ---- end to end through the public API with pinned host buffers (H2D B + execute + D2H C)
    # Every step copies its own B from pinned host memory and its C back (separate host buffers
    # per ring slot).  Headline: accspmm_execute_host_batch, which overlaps H2D(i+1) and D2H(i-1)
    # with the SpMM of step i; beside it the one-call-per-step synchronous accspmm_execute_host.
    e2e = None
    if not args.no_e2e:
        ring = 3
        Bh = [torch.from_numpy(B).to(tdt).pin_memory() for _ in range(ring)]
        Ch = [torch.empty((plan.out_rows, args.N), dtype=torch.float32).pin_memory() for _ in range(ring)]
        e_steps = max(3, min(args.steps, 30))
        Bb = [Bh[i % ring] for i in range(e_steps)]
        Cb = [Ch[i % ring] for i in range(e_steps)]

        def timed(fn):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            fn()
            s1.record(stream)
            torch.cuda.synchronize()
            te = s0.elapsed_time(s1) / 1e3
            if world > 1:
                tt = torch.tensor([te], dtype=torch.float64, device="cpu" if shared else "cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                te = float(tt.item())
            return te

        plan.execute_host_batch(Bb[:4], Cb[:4], stream)  # warm-up (staging buffers, streams)
        te = timed(lambda: plan.execute_host_batch(Bb, Cb, stream))
        for _ in range(2):
            plan.execute_host(Bh[0], Ch[0], stream)

        def sync_steps():
            for i in range(e_steps):
                plan.execute_host(Bb[i], Cb[i], stream)
        ts = timed(sync_steps)
        e2e = {"value": 2.0 * A.nnz * args.N * e_steps / te / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(Bh[0].numel() * Bh[0].element_size()),
               "d2h_bytes_per_step": int(Ch[0].numel() * Ch[0].element_size()), "steps": e_steps,
               "ms_per_step": te / e_steps * 1e3,
               "api": "accspmm_execute_host_batch (H2D/SpMM/D2H pipelined over 2 device slots)",
               "sync_per_step": {"value": 2.0 * A.nnz * args.N * e_steps / ts / 1e9,
                                 "ms_per_step": ts / e_steps * 1e3, "api": "accspmm_execute_host"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = cpu_oracle_sample(A, vals, B, args.precision, args.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": workload_config(args, cfg, A, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_model_per_launch": bm, "frac_of_8TBps_spec": achieved / 8000.0,
                         "kernel": kernel_name(args), "launch_ms": avg_s * 1e3,
                         "kernel_share_of_step": avg_s * args.steps / t_local,
                         "l2": {"achieved": achieved, "peak": l2_peak, "unit": "GB/s", "frac": achieved / l2_peak,
                                "peak_kind": "measured live: accspmm_probe_l2_bandwidth (96 MiB, ld.global.cg, best "
                                             "of 4 launch shapes, before and after the timed loop)"}},
            "cpu_baseline": cpu,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": args.steps * plan.launches_per_execute,
            "plan": {k: info[k] for k in ("W", "NB", "sum_U", "mean_nnz_tc", "ibd", "balanced", "grouped", "unit_cap",
                                          "n_units", "n_split_windows", "n_segments", "reorder_applied",
                                          "cols_permuted", "ms_reorder", "ms_build", "ms_schedule", "ms_upload",
                                          "device_bytes")},
            "plan_build": args.build,
            "warm": {"ms_per_step": warm_ms, "value": 2.0 * A.nnz * args.N / (warm_ms / 1e3) / 1e9,
                     "note": "back-to-back steps without the L2 flush (rank-local)"},
            "plan_create_s": plan_s, "broadcast_ms": bcast_ms, "allgather": allgather, "wall_s_timed_loop": wall,
            "step_ms_min": min(step_ms), "step_ms_max": max(step_ms),
        }
        emit(out, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
