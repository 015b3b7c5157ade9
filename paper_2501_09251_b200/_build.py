"""Builds libaccspmm.so in-tree: C++17 host code (g++ -fopenmp) + CUDA kernels for sm_100a (nvcc).

The library travels to the GPU box with the repo snapshot (it is git-ignored,
not gpurun-ignored).  Rebuilds only when a source or header is newer than the .so.

``build(variants=True)`` builds libaccspmm_variants.so instead: the same sources with
-DACCSPMM_VARIANTS, i.e. the measured-and-rejected kernel variants and the ACCSPMM_* A/B
knobs (tools/sweep.py).  The product library contains neither.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "accspmm")
LIB = os.path.join(PKG, "libaccspmm.so")
BUILD_VARIANTS = os.path.join(ROOT, "build", "accspmm_variants")
LIB_VARIANTS = os.path.join(PKG, "libaccspmm_variants.so")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")) + glob.glob(os.path.join(CSRC, "capi", "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    hdr = glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return cpp, cu, hdr


def _obj(src, bdir=BUILD):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(bdir, rel + ".o")


def _compile(src, verbose=False, variants=False):
    obj = _obj(src, BUILD_VARIANTS if variants else BUILD)
    inc = ["-I", INCLUDE, "-I", CSRC]
    defs = ["-DACCSPMM_VARIANTS"] if variants else []
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
               *defs, *inc, "-c", src, "-o", obj]
    else:
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-Wall",
               *defs, "-I", os.path.join(CUDA_HOME, "include"), *inc, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, variants: bool = False) -> str:
    lib, bdir = (LIB_VARIANTS, BUILD_VARIANTS) if variants else (LIB, BUILD)
    cpp, cu, hdr = _sources()
    # largest translation units first: the pool then finishes them in parallel with the rest
    srcs = sorted(cpp + cu, key=lambda f: -os.path.getsize(f))
    newest = max(os.path.getmtime(f) for f in srcs + hdr + [__file__])
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
        return lib
    os.makedirs(bdir, exist_ok=True)
    hdr_time = max(os.path.getmtime(f) for f in hdr + [__file__])
    todo = [s for s in srcs if force or not os.path.exists(_obj(s, bdir))
            or os.path.getmtime(_obj(s, bdir)) < max(os.path.getmtime(s), hdr_time)]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for obj, log in ex.map(lambda s: _compile(s, verbose, variants), todo):
            if verbose and log:
                sys.stderr.write(log)
    objs = [_obj(s, bdir) for s in srcs]
    LIBX = lib
    tmp = LIBX + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIBX)
    return LIBX


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, variants="--variants" in sys.argv))
