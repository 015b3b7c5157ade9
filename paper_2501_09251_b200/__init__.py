"""paper_2501_09251_b200 -- B200-native Acc-SpMM (arXiv 2501.09251) hot path.

Thin ctypes binding of ``libaccspmm.so`` (C ABI declared in include/accspmm.h).
Every function here only marshals arguments: all of the SpMM path (format
build, schedule, decode, MMA, epilogue) runs in the library's C++ and CUDA code.
There is no CPU fallback -- if the library is missing, importing the binding
raises, and a host-only plan refuses to execute.

The functions keep the C names (``accspmm_plan_create`` ...); ``Plan`` is a
small convenience wrapper taking numpy arrays and torch CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ACCSPMM_LIB=variants selects the measurement build (same ABI, plus the rejected kernel variants
# and the ACCSPMM_* A/B knobs; tools/sweep.py); the product library is libaccspmm.so
LIB_PATH = os.path.join(_HERE, "libaccspmm_variants.so" if os.environ.get("ACCSPMM_LIB") == "variants"
                        else "libaccspmm.so")

TF32, FP16 = 0, 1
REORDER = {"off": 0, "on": 1, "auto": 2}
BALANCE = {"off": 0, "on": 1, "auto": 2}
PRECISION = {"tf32": TF32, "fp16": FP16}
BUILD = {"host": 0, "device": 1}
KERNEL = {"auto": 0, "mma_sync": 1, "tcgen05": 2}
KERNEL_NAME = {v: k for k, v in KERNEL.items()}
HOT = {"auto": 0, "on": 1, "off": 2}
NO_SPLIT = 0xFFFFFFFF


class AccSpmmError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_status_name(status)}: {message}")
        self.status = status


class accspmm_options(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int32), ("reorder", ctypes.c_int32), ("balance", ctypes.c_int32),
                ("unit_cap", ctypes.c_int32), ("part", ctypes.c_int32), ("nparts", ctypes.c_int32),
                ("device", ctypes.c_int32), ("build", ctypes.c_int32), ("permute_cols", ctypes.c_int32),
                ("window_rows", ctypes.c_int32), ("kernel", ctypes.c_int32), ("hot_cols", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 4)]


_I64 = ["M", "K", "nnz", "rows", "row_begin", "window_begin", "W", "NB", "plan_nnz", "sum_U", "n_units",
        "n_split_windows", "n_segments", "nb_unreordered"]
_I32 = ["precision", "reorder_applied", "balanced", "unit_cap", "perm_present", "part", "nparts", "device"]


class accspmm_plan_info(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_int64) for n in _I64] + [(n, ctypes.c_int32) for n in _I32]
                + [("mean_nnz_tc", ctypes.c_double), ("ibd", ctypes.c_double)]
                + [(n, ctypes.c_int64) for n in ("index_bytes", "metcf_index_bytes", "csr_index_bytes",
                                                  "value_bytes", "device_bytes")]
                + [(n, ctypes.c_double) for n in ("ms_validate", "ms_reorder", "ms_build", "ms_schedule",
                                                   "ms_upload")]
                + [("grouped", ctypes.c_int64), ("cols_permuted", ctypes.c_int64), ("group_cap", ctypes.c_int64),
                   ("window_rows", ctypes.c_int64), ("kernel", ctypes.c_int64), ("hot_cols", ctypes.c_int64),
                   ("reserved", ctypes.c_int64 * 2)])

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "reserved"}


_lib = None
EXPORTED = [
    "accspmm_options_default", "accspmm_plan_create", "accspmm_plan_create_ex", "accspmm_execute",
    "accspmm_execute_host", "accspmm_plan_destroy", "accspmm_plan_get_info", "accspmm_plan_export_format",
    "accspmm_plan_export_units", "accspmm_plan_export_rows", "accspmm_reorder", "accspmm_partition_bounds",
    "accspmm_unpermute", "accspmm_debug_round_tf32", "accspmm_debug_decode", "accspmm_status_string",
    "accspmm_last_error", "accspmm_abi_version", "accspmm_plan_set_timing", "accspmm_plan_kernel_times",
    "accspmm_probe_l2_bandwidth", "accspmm_probe_l2_bandwidth_ex", "accspmm_execute_host_batch", "accspmm_csr_transpose",
    "accspmm_execute_allgather", "accspmm_reorder_parallel", "accspmm_plan_create_perm", "accspmm_plan_b_bytes",
]


def load_library(path: str = LIB_PATH):
    """Loads libaccspmm.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2501_09251_b200._build` "
                          "(the CUDA path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    S = ctypes.c_int
    sig = {
        "accspmm_options_default": ([ctypes.POINTER(accspmm_options)], S),
        "accspmm_plan_create": ([I64, I64, P, P, P, ctypes.POINTER(P)], S),
        "accspmm_plan_create_ex": ([I64, I64, P, P, P, ctypes.POINTER(accspmm_options), ctypes.POINTER(P)], S),
        "accspmm_plan_create_perm": ([I64, I64, P, P, P, ctypes.POINTER(accspmm_options), P, ctypes.POINTER(P)], S),
        "accspmm_execute": ([P, P, I64, P, P], S),
        "accspmm_execute_host": ([P, P, I64, P, P], S),
        "accspmm_plan_destroy": ([P], None),
        "accspmm_plan_get_info": ([P, ctypes.POINTER(accspmm_plan_info)], S),
        "accspmm_plan_b_bytes": ([P, I64, P], S),
        "accspmm_plan_export_format": ([P, P, P, P, P, P], S),
        "accspmm_plan_export_units": ([P, P], S),
        "accspmm_plan_export_rows": ([P, P], S),
        "accspmm_reorder": ([I64, P, P, P], S),
        "accspmm_reorder_parallel": ([I64, P, P, I64, I64, I32, P], S),
        "accspmm_partition_bounds": ([I64, P, I32, P], S),
        "accspmm_unpermute": ([P, P, I64, I64, P, P], S),
        "accspmm_debug_round_tf32": ([P, P, I64, P], S),
        "accspmm_debug_decode": ([P, P, P], S),
        "accspmm_status_string": ([S], ctypes.c_char_p),
        "accspmm_last_error": ([], ctypes.c_char_p),
        "accspmm_abi_version": ([], I32),
        "accspmm_plan_set_timing": ([P, I32], S),
        "accspmm_plan_kernel_times": ([P, P, I32, ctypes.POINTER(I32)], S),
        "accspmm_probe_l2_bandwidth": ([I64, I32, ctypes.POINTER(ctypes.c_double)], S),
        "accspmm_probe_l2_bandwidth_ex": ([I64, I32, I32, ctypes.POINTER(ctypes.c_double)], S),
        "accspmm_execute_host_batch": ([P, P, P, I32, I64, P], S),
        "accspmm_csr_transpose": ([I64, I64, P, P, P, P, P, P], S),
        "accspmm_execute_allgather": ([P, P, I64, P, I32, P], S),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _status_name(s: int) -> str:
    try:
        return load_library().accspmm_status_string(s).decode()
    except Exception:  # pragma: no cover
        return f"status {s}"


def _check(status: int):
    if status != 0:
        raise AccSpmmError(status, load_library().accspmm_last_error().decode())


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return int(a)


# ------------------------------------------------------------------ C-named functions

def accspmm_options_default() -> accspmm_options:
    opt = accspmm_options()
    _check(load_library().accspmm_options_default(ctypes.byref(opt)))
    return opt


def accspmm_plan_create(M, K, rowptr, colidx, vals):
    return accspmm_plan_create_ex(M, K, rowptr, colidx, vals, None)


def accspmm_plan_create_ex(M, K, rowptr, colidx, vals, opt: accspmm_options | None):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    out = ctypes.c_void_p()
    _check(load_library().accspmm_plan_create_ex(int(M), int(K), _ptr(rowptr), _ptr(colidx), _ptr(vals),
                                                 ctypes.byref(opt) if opt is not None else None, ctypes.byref(out)))
    return out.value


def accspmm_plan_create_perm(M, K, rowptr, colidx, vals, opt: accspmm_options | None, perm):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    out = ctypes.c_void_p()
    _check(load_library().accspmm_plan_create_perm(int(M), int(K), _ptr(rowptr), _ptr(colidx), _ptr(vals),
                                                   ctypes.byref(opt) if opt is not None else None, _ptr(perm),
                                                   ctypes.byref(out)))
    return out.value


def accspmm_execute(plan, B_ptr, N, C_ptr, stream_ptr=None):
    _check(load_library().accspmm_execute(plan, B_ptr, int(N), C_ptr, stream_ptr))


def accspmm_execute_host(plan, B_host_ptr, N, C_host_ptr, stream_ptr=None):
    _check(load_library().accspmm_execute_host(plan, B_host_ptr, int(N), C_host_ptr, stream_ptr))


def accspmm_execute_host_batch(plan, B_host_ptrs, C_host_ptrs, N, stream_ptr=None):
    n = len(B_host_ptrs)
    if len(C_host_ptrs) != n:
        raise ValueError("B and C batches differ in length")
    Bs = (ctypes.c_void_p * max(n, 1))(*B_host_ptrs)
    Cs = (ctypes.c_void_p * max(n, 1))(*C_host_ptrs)
    _check(load_library().accspmm_execute_host_batch(plan, Bs, Cs, n, int(N), stream_ptr))


def accspmm_execute_allgather(plan, B_ptr, N, C_ptrs, stream_ptr=None):
    arr = (ctypes.c_void_p * max(len(C_ptrs), 1))(*C_ptrs)
    _check(load_library().accspmm_execute_allgather(plan, B_ptr, int(N), arr, len(C_ptrs), stream_ptr))


def accspmm_plan_destroy(plan):
    if plan:
        load_library().accspmm_plan_destroy(plan)


def accspmm_plan_b_bytes(plan, N) -> int:
    """Bytes per element of B an execute at width N gathers (4 FP32 rows, 3 the TF32 image B3, 2 FP16)."""
    out = ctypes.c_int32()
    _check(load_library().accspmm_plan_b_bytes(plan, int(N), ctypes.byref(out)))
    return out.value


def accspmm_plan_get_info(plan) -> dict:
    info = accspmm_plan_info()
    _check(load_library().accspmm_plan_get_info(plan, ctypes.byref(info)))
    return info.as_dict()


def accspmm_plan_export_format(plan) -> dict:
    info = accspmm_plan_get_info(plan)
    W, NB, nnz = info["W"], info["NB"], info["plan_nnz"]
    nw = info["window_rows"] // 8   # occupancy words per block (1 for the paper's 8-row windows)
    rwo = np.empty(W + 1, np.uint32)
    tco = np.empty(NB + 1, np.uint32)
    a2b = np.empty(8 * NB, np.uint32)
    bits = np.empty(NB * nw, np.uint64)
    vals = np.empty(nnz, np.uint16 if info["precision"] == FP16 else np.float32)
    _check(load_library().accspmm_plan_export_format(plan, _ptr(rwo), _ptr(tco), _ptr(a2b), _ptr(bits), _ptr(vals)))
    if info["precision"] == FP16:
        vals = vals.view(np.float16)
    return {"RowWindowOffset": rwo, "TCOffset": tco, "SparseAToB": a2b, "TCLocalBit": bits, "values": vals,
            "W": W, "NB": NB, "nnz": nnz, "window_rows": info["window_rows"]}


def accspmm_plan_export_units(plan) -> np.ndarray:
    n = accspmm_plan_get_info(plan)["n_units"]
    u = np.empty((n, 8), np.uint32)
    _check(load_library().accspmm_plan_export_units(plan, _ptr(u)))
    return u


def accspmm_plan_export_rows(plan) -> np.ndarray:
    n = accspmm_plan_get_info(plan)["rows"]
    r = np.empty(n, np.uint32)
    if n:
        _check(load_library().accspmm_plan_export_rows(plan, _ptr(r)))
    return r


def accspmm_reorder(n, rowptr, colidx) -> np.ndarray:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    perm = np.empty(n, np.uint32)
    _check(load_library().accspmm_reorder(int(n), _ptr(rowptr), _ptr(colidx), _ptr(perm)))
    return perm


def accspmm_reorder_parallel(n, rowptr, colidx, round=0, segments=0, L=0) -> np.ndarray:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    perm = np.empty(n, np.uint32)
    _check(load_library().accspmm_reorder_parallel(int(n), _ptr(rowptr), _ptr(colidx), int(round), int(segments),
                                                   int(L), _ptr(perm)))
    return perm


def accspmm_csr_transpose(M, K, rowptr, colidx, vals=None):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    nnz = int(rowptr[-1]) if M > 0 else 0
    t_rowptr = np.empty(K + 1, np.int64)
    t_colidx = np.empty(nnz, np.int32)
    t_vals = None
    if vals is not None:
        vals = np.ascontiguousarray(vals, dtype=np.float32)
        t_vals = np.empty(nnz, np.float32)
    _check(load_library().accspmm_csr_transpose(int(M), int(K), _ptr(rowptr), _ptr(colidx), _ptr(vals),
                                                _ptr(t_rowptr), _ptr(t_colidx), _ptr(t_vals)))
    return t_rowptr, t_colidx, t_vals


def accspmm_partition_bounds(M, rowptr, nparts) -> np.ndarray:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    b = np.empty(nparts + 1, np.int64)
    _check(load_library().accspmm_partition_bounds(int(M), _ptr(rowptr), int(nparts), _ptr(b)))
    return b


def accspmm_unpermute(G_ptr, orig_row_ptr, n_rows, N, C_ptr, stream_ptr=None):
    _check(load_library().accspmm_unpermute(G_ptr, orig_row_ptr, int(n_rows), int(N), C_ptr, stream_ptr))


def accspmm_debug_round_tf32(in_ptr, out_ptr, n, stream_ptr=None):
    _check(load_library().accspmm_debug_round_tf32(in_ptr, out_ptr, int(n), stream_ptr))


def accspmm_debug_decode(plan, tiles_ptr, stream_ptr=None):
    _check(load_library().accspmm_debug_decode(plan, tiles_ptr, stream_ptr))


def accspmm_plan_set_timing(plan, enable: bool):
    _check(load_library().accspmm_plan_set_timing(plan, int(bool(enable))))


def accspmm_plan_kernel_times(plan, max_n: int = 4096) -> np.ndarray:
    out = np.empty(max_n, np.float32)
    n = ctypes.c_int32()
    _check(load_library().accspmm_plan_kernel_times(plan, _ptr(out), int(max_n), ctypes.byref(n)))
    return out[:n.value].copy()


def accspmm_probe_l2_bandwidth(nbytes: int = 64 << 20, iters: int = 50) -> float:
    g = ctypes.c_double()
    _check(load_library().accspmm_probe_l2_bandwidth(int(nbytes), int(iters), ctypes.byref(g)))
    return g.value


def accspmm_probe_l2_bandwidth_ex(nbytes: int = 64 << 20, iters: int = 50, mode: int = 0) -> float:
    """mode 1: ld.global.cg loads, 2: TMA bulk copies, 0: the larger of the two."""
    g = ctypes.c_double()
    _check(load_library().accspmm_probe_l2_bandwidth_ex(int(nbytes), int(iters), int(mode), ctypes.byref(g)))
    return g.value


def accspmm_status_string(s: int) -> str:
    return load_library().accspmm_status_string(s).decode()


def accspmm_last_error() -> str:
    return load_library().accspmm_last_error().decode()


def accspmm_abi_version() -> int:
    return load_library().accspmm_abi_version()


# ------------------------------------------------------------------ convenience wrapper

def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _check_2d(name, X, rows, dtypes, N=None):
    """Shape / dtype / layout checks the C ABI cannot do (it only sees pointers)."""
    if X.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(X.shape)}")
    if X.shape[0] != rows:
        raise ValueError(f"{name} must have {rows} rows, got {X.shape[0]}")
    if N is not None and X.shape[1] != N:
        raise ValueError(f"{name} must have {N} columns, got {X.shape[1]}")
    dt = str(X.dtype).replace("torch.", "")
    if dt not in dtypes:
        raise TypeError(f"{name} dtype must be {dtypes[0]}, got {dt}")
    contiguous = X.is_contiguous() if hasattr(X, "is_contiguous") else X.flags["C_CONTIGUOUS"]
    if not contiguous:
        raise ValueError(f"{name} must be contiguous (row-major, leading dimension = number of columns)")


class Plan:
    """Owns one accspmm_plan.  ``execute`` takes torch CUDA tensors (B: K x N, float32 for
    TF32 / float16 for FP16) and returns / fills C (float32)."""

    def __init__(self, M, K, rowptr, colidx, vals, precision="tf32", reorder="auto", balance="auto",
                 unit_cap=0, part=0, nparts=1, device=None, build="host", permute_cols=False, window_rows=0,
                 kernel="auto", perm=None, hot_cols="auto"):
        """perm (optional, u32[M] new -> old): an Alg. 1 permutation computed elsewhere (e.g. once
        on rank 0 and broadcast), used instead of running the reordering again.  hot_cols:
        auto / on / off -- columns relabelled by in-degree with per-block L2 hotness tags (R22)."""
        opt = accspmm_options_default()
        opt.hot_cols = HOT[hot_cols]
        opt.window_rows = int(window_rows)
        opt.kernel = KERNEL[kernel]
        opt.build = BUILD[build]
        opt.permute_cols = int(bool(permute_cols))
        opt.precision = PRECISION[precision]
        opt.reorder = REORDER[reorder]
        opt.balance = BALANCE[balance]
        opt.unit_cap = int(unit_cap)
        opt.part, opt.nparts = int(part), int(nparts)
        if device is not None:
            opt.device = int(device)
        self.precision = precision
        if perm is not None:
            self.handle = accspmm_plan_create_perm(M, K, rowptr, colidx, vals, opt, perm)
        else:
            self.handle = accspmm_plan_create_ex(M, K, rowptr, colidx, vals, opt)
        self.info = accspmm_plan_get_info(self.handle)

    def close(self):
        if getattr(self, "handle", None):
            accspmm_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def out_rows(self) -> int:
        return self.info["M"] if self.info["nparts"] == 1 else self.info["rows"]

    @property
    def _b_dtypes(self):
        return ("float16",) if self.precision == "fp16" else ("float32",)

    def _check_device(self, name, X):
        if not getattr(X, "is_cuda", False):
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback; use execute_host for host buffers)")
        if X.device.index != self.info["device"]:
            raise ValueError(f"{name} is on cuda:{X.device.index}, the plan on cuda:{self.info['device']}")

    def _check_B(self, B):
        _check_2d("B", B, self.info["K"], self._b_dtypes)
        self._check_device("B", B)

    def execute(self, B, C=None, stream=None):
        import torch
        self._check_B(B)
        N = B.shape[1]
        if C is None:
            C = torch.empty((self.out_rows, N), dtype=torch.float32, device=B.device)
        else:
            _check_2d("C", C, self.out_rows, ("float32",), N)
            self._check_device("C", C)
        accspmm_execute(self.handle, B.data_ptr(), N, C.data_ptr(), _stream_ptr(stream))
        return C

    def execute_allgather(self, B, C_all, stream=None):
        """Fused all-gather: this plan's rows go to every matrix of C_all (full M x N float32
        CUDA tensors, local or peer-mapped) in original row order."""
        self._check_B(B)
        for k, c in enumerate(C_all):
            _check_2d(f"C_all[{k}]", c, self.info["M"], ("float32",), B.shape[1])
        accspmm_execute_allgather(self.handle, B.data_ptr(), B.shape[1], [c.data_ptr() for c in C_all],
                                  _stream_ptr(stream))
        return C_all

    def _check_host(self, B_host, C_host, N=None):
        _check_2d("B_host", B_host, self.info["K"], self._b_dtypes, N)
        _check_2d("C_host", C_host, self.info["rows"], ("float32",), B_host.shape[1])
        for name, X in (("B_host", B_host), ("C_host", C_host)):
            if getattr(X, "is_cuda", False):
                raise ValueError(f"{name} must be host memory (numpy or CPU tensor)")

    def execute_host(self, B_host, C_host, stream=None):
        """End to end with host buffers (numpy or pinned torch CPU tensors)."""
        self._check_host(B_host, C_host)
        N = B_host.shape[1]
        accspmm_execute_host(self.handle, _ptr(B_host), N, _ptr(C_host), _stream_ptr(stream))
        return C_host

    def execute_host_batch(self, B_hosts, C_hosts, stream=None):
        """Pipelined end to end over a batch of host B / C buffers (pinned for overlap)."""
        if len(B_hosts) != len(C_hosts):
            raise ValueError("B and C batches differ in length")
        if not B_hosts:
            return C_hosts
        N = B_hosts[0].shape[1]
        for b, c in zip(B_hosts, C_hosts):
            self._check_host(b, c, N)
        accspmm_execute_host_batch(self.handle, [_ptr(b) for b in B_hosts], [_ptr(c) for c in C_hosts], N,
                                   _stream_ptr(stream))
        return C_hosts

    def export_format(self) -> dict:
        return accspmm_plan_export_format(self.handle)

    def export_units(self) -> np.ndarray:
        return accspmm_plan_export_units(self.handle)

    def export_rows(self) -> np.ndarray:
        return accspmm_plan_export_rows(self.handle)

    def set_timing(self, enable=True):
        accspmm_plan_set_timing(self.handle, enable)

    def kernel_times(self) -> np.ndarray:
        return accspmm_plan_kernel_times(self.handle)

    def b_bytes(self, N: int) -> int:
        return accspmm_plan_b_bytes(self.handle, N)

    @property
    def launches_per_execute(self) -> int:
        """SpMM kernel + (TF32 with high B-row reuse) the rho(B) pre-pass -- mirrors
        accspmm_execute (relabelled columns gather B's original rows: no pass)."""
        i = self.info
        pre = self.precision == "tf32" and i["K"] > 0 and i["sum_U"] >= 32 * i["K"]
        return 2 if pre else 1

    def debug_decode(self, stream=None):
        import torch
        tiles = torch.empty((self.info["NB"], 8 * self.info["window_rows"]), dtype=torch.float32, device="cuda")
        accspmm_debug_decode(self.handle, tiles.data_ptr(), _stream_ptr(stream))
        return tiles


def bytes_model(info: dict, N: int, es_b: int | None = None) -> dict:
    """SURVEY §8(d) stated bytes model for one execute: A-format + unique B rows per window + C.
    es_b = bytes per stored B element as the execute gathers it (Plan.b_bytes(N): 3 for the TF32
    image B3); default the precision's element size."""
    es_a = 2 if info["precision"] == FP16 else 4
    es_b = es_a if es_b is None else es_b
    W, NB = info["W"], info["NB"]
    nw = info.get("window_rows", 8) // 8   # u64 occupancy words per block
    a_fmt = (4 * (W + 1) + 4 * (NB + 1) + 32 * NB + 8 * nw * NB + es_a * info["plan_nnz"]
             + 32 * info["n_units"] + (4 * info["rows"] if info["perm_present"] and info["nparts"] == 1 else 0))
    b_model = es_b * N * info["sum_U"]
    c = 4 * info["rows"] * N
    return {"A_fmt": a_fmt, "B_model": b_model, "C": c, "total": a_fmt + b_model + c,
            "flops": 2 * info["plan_nnz"] * N}
