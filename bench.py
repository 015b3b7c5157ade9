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
    ap.add_argument("--window-rows", type=int, default=0, help="rows per RowWindow: 0/8 = paper, 16/32 = tall (R20)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "mma_sync", "tcgen05"])
    ap.add_argument("--hot-cols", default="auto", choices=["auto", "on", "off"],
                    help="columns relabelled by in-degree with per-block L2 hotness tags (reading R22)")
    ap.add_argument("--allgather", default="none", choices=["none", "nccl", "fused"],
                    help="N > 1: also time assembling the full C on every rank (NCCL all-gather + "
                         "un-permute, or the fused epilogue into symmetric memory); reported as "
                         "'allgather', the headline value stays the slab step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu: warmup + steps, no extras")
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-job ncu capture of the DRAM traffic")
    ap.add_argument("--ncu-timeout", type=float, default=300.0)
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons of the bench GPU sampled through NVML every
    5 ms during the timed region, plus one sample right before and one right after it, so even
    a 50 ms region carries its own record (the recipe's nvidia-smi clocks line, B200_PROFILING.md)."""
    PERIOD_S = 0.005

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.h = None
        self.nv = None
        self.error = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            prop = torch.cuda.get_device_properties(device_index)
            bus = "%08X:%02X:%02X.0" % (prop.pci_domain_id, prop.pci_bus_id, prop.pci_device_id)
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            self.nv = nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # reported in the record, never fatal
            self.error = repr(e)[:200]

    def _sample(self):
        nv = self.nv
        try:
            self.samples.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        except Exception as e:
            self.error = repr(e)[:200]

    def _run(self):
        while not self.stop_flag.is_set():
            self._sample()
            time.sleep(self.PERIOD_S)

    def start(self):
        if self.h is None:
            return
        self.stop_flag = threading.Event()
        self._sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self):
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "error": self.error or "NVML unavailable"}
        self.stop_flag.set()
        self.t.join(timeout=2)
        self._sample()
        nv = self.nv
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                "hw_power_brake_slowdown": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        reasons = sorted({n for _, r in self.samples for n, b in bits.items() if r & b})
        sm = [float(c) for c, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.max_mhz),
                "sm_mhz_min": min(sm) if sm else None, "reasons": reasons, "samples": len(sm),
                "source": "NVML, every 5 ms + before/after the timed loop"}


NCU = "/usr/local/cuda/bin/ncu"
NCU_METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
               "gpu__time_duration.sum")


def ncu_traffic(args, world):
    """DRAM / L2 traffic of one SpMM launch of THIS workload, captured in this job: a child
    bench process (same matrix, plan options, N) runs under ncu, which profiles its 3rd SpMM
    launch (cache-control all: caches flushed before the launch, as in the timed loop).
    Returns bytes per launch, or {"unavailable": why}."""
    if not os.path.exists(NCU):
        return {"unavailable": "ncu not found"}
    cmd = [NCU, "--metrics", ",".join(NCU_METRICS), "--clock-control", "none", "--print-units", "base",
           "-k", "regex:spmm_", "-s", "2", "-c", "1", "--csv",
           sys.executable, os.path.abspath(__file__), "--ncu-child", "--config", args.config, "--N", str(args.N),
           "--precision", args.precision, "--reorder", args.reorder, "--balance", args.balance,
           "--unit-cap", str(args.unit_cap), "--build", args.build, "--window-rows", str(args.window_rows),
           "--kernel", args.kernel, "--hot-cols", args.hot_cols]
    if args.permute_cols:
        cmd.append("--permute-cols")
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK=os.environ.get("LOCAL_RANK", "0"))
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=args.ncu_timeout, env=env)
    except Exception as e:
        return {"unavailable": repr(e)[:200]}
    import csv
    import io
    vals = {}
    kernel = None
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    for row in csv.DictReader(io.StringIO("\n".join(lines))):
        name = row.get("Metric Name")
        if name in NCU_METRICS:
            try:
                vals[name] = float(row["Metric Value"].replace(",", ""))
                kernel = row.get("Kernel Name", kernel)
            except ValueError:
                pass
    if "dram__bytes_read.sum" not in vals:
        return {"unavailable": f"ncu rc={r.returncode}: " + (r.stderr or r.stdout)[-300:]}
    out = {"dram_bytes": vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0.0),
           "dram_read_bytes": vals["dram__bytes_read.sum"], "dram_write_bytes": vals.get("dram__bytes_write.sum"),
           "l2_tex_read_bytes": 32.0 * vals["lts__t_sectors_srcunit_tex_op_read.sum"]
           if "lts__t_sectors_srcunit_tex_op_read.sum" in vals else None,
           "ncu_kernel_ns": vals.get("gpu__time_duration.sum"), "kernel": (kernel or "")[:120],
           "how": "ncu --metrics " + ",".join(NCU_METRICS) + " on the 3rd SpMM launch of a child run of this "
                  "workload in this job (cache-control all = cold L2, like the flushed timed loop)"}
    return out


def run_ncu_child(args):
    """--ncu-child: build the same plan and execute it 3 times (ncu captures the 3rd launch)."""
    import torch

    import paper_2501_09251_b200 as acc
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    cfg, A, vals, B = make_inputs(args)
    plan = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, precision=args.precision, reorder=args.reorder,
                    balance=args.balance, unit_cap=args.unit_cap, device=torch.cuda.current_device(),
                    permute_cols=args.permute_cols, build=args.build, window_rows=args.window_rows,
                    kernel=args.kernel, hot_cols=args.hot_cols)
    Bd = torch.from_numpy(B).to(device="cuda", dtype=torch.float16 if args.precision == "fp16" else torch.float32)
    C = torch.empty((plan.out_rows, args.N), dtype=torch.float32, device="cuda")
    for _ in range(3):
        plan.execute(Bd, C)
    torch.cuda.synchronize()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def single_thread_baselines(seconds: float = 2.0) -> dict:
    """the oracle on ONE host thread for configs T (tiny, whole) and S (stencil,
    bounded row sample), GFLOP/s = 2*nnz*N/t."""
    import gen
    from oracle import spmm as osp
    from oracle.rounding import rho
    out = {}
    for name, N in (("tiny", 16), ("stencil", 128)):
        cfg, A = gen.make_config(name)
        a = rho(gen.values_uniform(A.nnz, cfg.seed_A + 1), "tf32")
        b = rho(gen.dense_normal(A.K, N, cfg.seed_B), "tf32")
        nnz_row = np.diff(A.rowptr)
        rng = np.random.default_rng(0)
        rows = np.sort(rng.choice(A.M, size=min(A.M, 2048), replace=False))
        _, t = osp.timed_spmm(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows, nthreads=1)
        rate = 2.0 * nnz_row[rows].sum() * N / max(t, 1e-9)
        n = int(min(A.M, max(2048, rate * seconds / max(2.0 * nnz_row.mean() * N, 1.0))))
        rows = np.arange(A.M) if n >= A.M else np.sort(rng.choice(A.M, size=n, replace=False))
        _, t = osp.timed_spmm(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows, nthreads=1)
        out[name] = {"value": 2.0 * nnz_row[rows].sum() * N / t / 1e9, "unit": "GFLOP/s", "N": N,
                     "rows": int(rows.size), "of_rows": int(A.M), "seconds": t}
    return out


def make_inputs(args):
    import gen
    cfg, A = gen.make_config(args.config)
    vals = gen.values_uniform(A.nnz, cfg.seed_A + 1)
    B = gen.dense_normal(A.K, args.N, cfg.seed_B)
    return cfg, A, vals, B


def host_threads() -> int:
    """Every host core this process may run on.  torchrun exports OMP_NUM_THREADS=1 to its
    workers, so the oracle's OpenMP default would time one thread under --gpus N > 1."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def cpu_oracle_sample(A, vals, B, precision, seconds, seed=0, rounded=None):
    """The FP64 oracle as it stands, on the host cores, over a bounded random row sample
    (rho(A), rho(B) are computed once, outside the timed sample)."""
    from oracle import spmm as osp
    nt = host_threads()
    from oracle.rounding import rho
    a, b = rounded if rounded is not None else (rho(vals, precision), rho(B, precision))
    rng = np.random.default_rng(seed)
    nnz_row = np.diff(A.rowptr)
    N = B.shape[1]
    rows = np.sort(rng.choice(A.M, size=min(A.M, 256), replace=False))
    _, t = osp.timed_spmm(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows, nthreads=nt)
    rate = 2.0 * nnz_row[rows].sum() * N / max(t, 1e-9)
    target_flops = rate * seconds
    avg = 2.0 * nnz_row.mean() * N
    n = int(min(A.M, max(256, target_flops / max(avg, 1.0))))
    rows = np.sort(rng.choice(A.M, size=n, replace=False))
    _, t = osp.timed_spmm(A.M, A.K, A.rowptr, A.colidx, a, b, rows=rows, nthreads=nt)
    flops = 2.0 * nnz_row[rows].sum() * N
    return {"value": flops / t / 1e9, "unit": "GFLOP/s", "cores": osp.num_threads(nt), "kind": "oracle",
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
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # one whole-workload SpMM at the sampled rate (each timed step computes a bounded row sample)
        "ms_per_step": 2.0 * A.nnz * args.N / (value * 1e9) * 1e3 if value > 0 else None,
        "ms_per_step_is": "2*nnz*N / value: the full product at the rate measured on the row samples",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, cfg, A, world),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": info["cores"], "kind": "oracle",
                         "sample": info["sample"], "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out, args)


def workload_config(args, cfg, A, world):
    return {"workload": f"{cfg.name}: {cfg.note}; N={args.N}, {args.precision}",
            "matrix": cfg.name, "baseline_config_index": cfg.baseline_index, "M": A.M, "K": A.K, "nnz": A.nnz,
            "N": args.N, "precision": args.precision, "reorder": args.reorder, "balance": args.balance,
            "permute_cols": bool(getattr(args, "permute_cols", False)),
            "l2": "none" if args.no_flush else f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
            "window_rows": args.window_rows or 8, "kernel": args.kernel, "hot_cols": args.hot_cols,
            "parallelism": f"rowwindow-nnz-partition x{world}"}


def kernel_name(plan):
    """The SpMM kernel the library's dispatch picks for this plan."""
    if plan.info["kernel"] == 2:
        return ("spmm_tc05_kernel (TMA gather4 -> TMEM, tcgen05.mma kind::tf32, accumulators in TMEM; "
                f"{plan.info['window_rows']}-row windows)")
    return "spmm_bittcf_g4_kernel (TMA gather4 + mma.sync, 1 warp/CTA)"


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
    if args.ncu_child:
        run_ncu_child(args)
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
    perm = None
    perm_s = None
    if world > 1 and args.reorder != "off" and A.M == A.K:
        # Alg. 1 once on rank 0, broadcast to the other ranks (not replicated per rank)
        from paper_2501_09251_b200 import distributed as D
        perm = D.broadcast_perm(A.M, A.rowptr, A.colidx, device=None if shared else torch.device("cuda", local))
        perm_s = time.perf_counter() - t0
    plan = acc.Plan(A.M, A.K, A.rowptr, A.colidx, vals, precision=args.precision, reorder=args.reorder,
                    balance=args.balance, unit_cap=args.unit_cap, part=rank, nparts=world, device=local,
                    permute_cols=args.permute_cols, build=args.build, window_rows=args.window_rows,
                    kernel=args.kernel, perm=perm, hot_cols=args.hot_cols)
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

    # L2 read bandwidth through both request engines (LDG and TMA bulk copies); again after the
    # loop, the peak is the largest of the four
    l2_before = {m: acc.accspmm_probe_l2_bandwidth_ex(96 << 20, 100, mode=i) for m, i in (("ldg", 1), ("tma", 2))}
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

    # bytes per B element as stored for this execute (TF32 with a pre-rounded B: the 3-byte
    # image B3) -- the algorithmic B bytes of the bytes model
    es_b = plan.b_bytes(args.N)
    bm = acc.bytes_model(info, args.N, es_b)
    bm["es_b"] = es_b
    # the HBM lower bound of the gather -- every distinct column's B row once
    bm["B_compulsory"] = int(es_b * args.N * np.count_nonzero(np.bincount(A.colidx, minlength=A.K)))
    avg_s = float(np.mean(kernel_ms)) / 1e3 if len(kernel_ms) else t_local / args.steps
    hbm_peak, peak_kind = load_peaks()
    model_gbs = bm["total"] / avg_s / 1e9
    # L2 roofline: every model byte (gathered B rows, A stream, C) passes through L2, and on
    # graphs whose B fits L2 the gather is served from there
    l2_after = {m: acc.accspmm_probe_l2_bandwidth_ex(96 << 20, 100, mode=i) for m, i in (("ldg", 1), ("tma", 2))}
    l2_peak = max(max(l2_before.values()), max(l2_after.values()))
    # ---- end to end through the public API with pinned host buffers (H2D B + execute + D2H C)
    # Every step copies its own B from pinned host memory and its C back (separate host buffers
    # per ring slot).  Headline: accspmm_execute_host_batch, which overlaps H2D(i+1) and D2H(i-1)
    # with the SpMM of step i; beside it the one-call-per-step synchronous accspmm_execute_host.
    e2e = None
    if not args.no_e2e:
        ring = 3
        Bh = [torch.from_numpy(B).to(tdt).pin_memory() for _ in range(ring)]
        Ch = [torch.empty((plan.out_rows, args.N), dtype=torch.float32).pin_memory() for _ in range(ring)]
        e_steps = 40   # fixed: the pipeline's fill and drain amortised alike whatever --steps is
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
        io_bytes = [int(Bh[0].numel() * Bh[0].element_size()), int(Ch[0].numel() * Ch[0].element_size())]
        if world > 1:
            tb = torch.tensor(io_bytes, dtype=torch.int64, device="cpu" if shared else "cuda")
            dist.all_reduce(tb)
            io_bytes = [int(x) for x in tb.tolist()]
        e2e = {"value": 2.0 * A.nnz * args.N * e_steps / te / 1e9, "unit": "GFLOP/s",
               # whole job: every rank copies its own B in and its C slab out each step
               "h2d_bytes_per_step": io_bytes[0], "d2h_bytes_per_step": io_bytes[1], "ranks": world,
               "steps": e_steps,
               "ms_per_step": te / e_steps * 1e3,
               "api": "accspmm_execute_host_batch (H2D/SpMM/D2H pipelined over 2 device slots)",
               "sync_per_step": {"value": 2.0 * A.nnz * args.N * e_steps / ts / 1e9,
                                 "ms_per_step": ts / e_steps * 1e3, "api": "accspmm_execute_host"}}

    # (after the e2e loop: the ncu child process must not precede any timed region)
    # HBM roofline: the DRAM bytes ncu counts for one launch of this workload, captured in
    # this job, over the same in-library launch time
    if rank == 0 and world == 1 and not args.no_ncu:
        traffic = ncu_traffic(args, world)
    else:
        traffic = {"unavailable": "--no-ncu" if args.no_ncu else "captured on single-GPU runs only (ncu replays "
                   "kernels; never under a multi-rank command)"}
    l2 = {"achieved": model_gbs, "peak": l2_peak, "unit": "GB/s", "frac": model_gbs / l2_peak,
          "achieved_is": "stated bytes model (SURVEY §8(d): A_fmt + es*N*sum_w|U_w| + C) / SpMM launch time",
          "peak_kind": "measured live in this job by accspmm_probe_l2_bandwidth_ex over a 96 MiB L2-resident "
                       "buffer: 128-bit ld.global.cg from every SM (best of 4 launch shapes) and TMA bulk copies "
                       "into shared memory (best of 4 ring/chunk shapes), before and after the timed loop; the max",
          "peak_before": l2_before, "peak_after": l2_after}
    hbm = None
    if "dram_bytes" in traffic:
        dram_gbs = traffic["dram_bytes"] / avg_s / 1e9
        compulsory = bm["A_fmt"] + bm["B_compulsory"] + bm["C"]
        hbm = {"achieved": dram_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": dram_gbs / hbm_peak,
               "peak_kind": peak_kind + " (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)",
               "achieved_is": "ncu dram__bytes_read+write of one launch (this job) / SpMM launch time",
               "bytes_per_launch": traffic["dram_bytes"], "compulsory_bytes": compulsory,
               "bytes_over_compulsory": traffic["dram_bytes"] / max(compulsory, 1)}
    # the binding resource is the one closer to its peak
    bound = "hbm" if hbm is not None and hbm["frac"] > l2["frac"] else "l2"
    rec = hbm if bound == "hbm" else l2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = cpu_oracle_sample(A, vals, B, args.precision, args.cpu_seconds)
        cpu["cpu_model"] = cpu_model()
        cpu["single_thread"] = single_thread_baselines()

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": workload_config(args, cfg, A, world),
            "roofline": {"bound": bound, "achieved": rec["achieved"], "peak": rec["peak"], "unit": "GB/s",
                         "frac": rec["frac"], "traffic": traffic.get("dram_bytes"), "traffic_detail": traffic,
                         "l2": l2, "hbm": hbm, "bytes_model_per_launch": bm,
                         "model_bytes_over_hbm_peak": model_gbs / hbm_peak,
                         "kernel": kernel_name(plan), "launch_ms": avg_s * 1e3,
                         "kernel_share_of_step": avg_s * args.steps / t_local},
            "cpu_baseline": cpu,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": args.steps * plan.launches_per_execute,
            "plan": {k: info[k] for k in ("W", "NB", "sum_U", "mean_nnz_tc", "ibd", "balanced", "grouped", "unit_cap",
                                          "n_units", "n_split_windows", "n_segments", "reorder_applied",
                                          "cols_permuted", "hot_cols", "ms_reorder", "ms_build", "ms_schedule", "ms_upload",
                                          "device_bytes")},
            "plan_build": args.build,
            "warm": {"ms_per_step": warm_ms, "value": 2.0 * A.nnz * args.N / (warm_ms / 1e3) / 1e9,
                     "note": "back-to-back steps without the L2 flush (rank-local)"},
            "plan_create_s": plan_s, "reorder_broadcast_s": perm_s, "broadcast_ms": bcast_ms, "allgather": allgather, "wall_s_timed_loop": wall,
            "step_ms_min": min(step_ms), "step_ms_max": max(step_ms),
        }
        emit(out, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
