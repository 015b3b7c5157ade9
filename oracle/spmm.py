"""FP64 SpMM oracle wrapper + the elementwise pass criterion (TEST INFRASTRUCTURE ONLY).

Definition: C = rho(A) . rho(B) in IEEE
binary64, sequential CSR-order accumulation per row; bound S = |rho(A)|.|rho(B)|.
Pass iff |C_gpu - C_ref| <= tau*S + 1e-6 elementwise, tau = 1e-3 (TF32) or
4e-3 (FP16) -- BASELINE.json north_star.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "spmm_oracle.c")
_lib = None

TAU = {"tf32": 1e-3, "fp16": 4e-3}
ATOL = 1e-6


def build(force: bool = False) -> str:
    """Compile spmm_oracle.c with gcc + OpenMP (building the checker is not using it)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        lib.oracle_spmm_fp64.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P, P, ctypes.c_int64,
                                         P, ctypes.c_int64, P, P, ctypes.c_int]
        lib.oracle_spmm_fp64.restype = ctypes.c_int
        lib.oracle_num_threads.argtypes = [ctypes.c_int]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def num_threads(nthreads: int = 0) -> int:
    return _load().oracle_num_threads(nthreads)


def spmm_fp64(M, K, rowptr, colidx, a_rounded, B_rounded, rows=None, nthreads: int = 0,
              with_bound: bool = True):
    """C_ref (and S) for all rows or the row subset ``rows``; inputs already rho-rounded."""
    lib = _load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    a = np.ascontiguousarray(a_rounded, dtype=np.float32)
    B = np.ascontiguousarray(B_rounded, dtype=np.float32)
    if B.ndim != 2 or B.shape[0] != K:
        raise ValueError("dimension mismatch: B must be K x N")
    N = B.shape[1]
    rows_arr = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    R = M if rows_arr is None else rows_arr.size
    C = np.empty((R, N), dtype=np.float64)
    S = np.empty((R, N), dtype=np.float64) if with_bound else None
    rc = lib.oracle_spmm_fp64(M, K, _ptr(rowptr), _ptr(colidx), _ptr(a), _ptr(B), N,
                              _ptr(rows_arr), R, _ptr(C), _ptr(S), nthreads)
    if rc != 0:
        raise ValueError("oracle: bad row or column index")
    return (C, S) if with_bound else C


def timed_spmm(M, K, rowptr, colidx, a_rounded, B_rounded, rows=None, nthreads: int = 0):
    t0 = time.perf_counter()
    C = spmm_fp64(M, K, rowptr, colidx, a_rounded, B_rounded, rows=rows, nthreads=nthreads,
                  with_bound=False)
    return C, time.perf_counter() - t0


def check(C_gpu, C_ref, S, precision: str):
    """SURVEY §8(c) C-5 comparison: returns a report dict; ``ok`` iff zero violations, all finite."""
    tau = TAU[precision]
    C_gpu = np.asarray(C_gpu, dtype=np.float64)
    tol = tau * S + ATOL
    err = np.abs(C_gpu - C_ref)
    finite = bool(np.isfinite(C_gpu).all())
    viol = ~(err <= tol)
    nviol = int(viol.sum())
    ratio = err / tol
    worst = np.unravel_index(int(np.nanargmax(np.where(np.isfinite(ratio), ratio, np.inf))), err.shape) \
        if err.size else None
    denom = np.maximum(np.abs(C_ref), 1e-30)
    return {
        "ok": finite and nviol == 0,
        "violations": nviol,
        "finite": finite,
        "max_err_over_tol": float(np.nanmax(ratio)) if err.size else 0.0,
        "worst": tuple(int(x) for x in worst) if worst is not None else None,
        "max_rel": float(np.nanmax(err / denom)) if err.size else 0.0,
        "tau": tau,
    }
