"""Sparse-pattern, value and dense-operand generators (seeded, synthetic).

Every generator returns CSR in the boundary layout of include/accspmm.h:
``rowptr`` int64[M+1], ``colidx`` int32[nnz] strictly ascending within a row.
Recipes follow SURVEY.md §8(d) "Generator recipes"; shapes follow PAPER.md
Table 1 and BASELINE.json ``configs``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_native.so")
_SRC = os.path.join(_HERE, "_native.c")
_lib = None


def build(force: bool = False) -> str:
    """gcc -fopenmp the plumbing helpers (pairs -> CSR, DC-SBM draws)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11", _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


def _native():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P, I = ctypes.c_void_p, ctypes.c_int64
        lib.gen_pairs_to_csr.argtypes = [I, P, P, I, I, ctypes.c_int, ctypes.c_int, P, P]
        lib.gen_pairs_to_csr.restype = I
        lib.gen_dcsbm_draw.argtypes = [I, I, P, P, P, P, P, P, P, P, ctypes.c_double, ctypes.c_uint64, P, P]
        lib.gen_dcsbm_draw.restype = None
        D = ctypes.c_double
        lib.gen_x_degrees.argtypes = [I, D, D, D, I, ctypes.c_uint64, P]
        lib.gen_x_degrees.restype = None
        lib.gen_alias_build.argtypes = [I, P, P, P]
        lib.gen_alias_build.restype = None
        lib.gen_x_fill.argtypes = [I, I, P, P, P, ctypes.c_uint64, P, P]
        lib.gen_x_fill.restype = I
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Csr:
    M: int
    K: int
    rowptr: np.ndarray  # int64[M+1]
    colidx: np.ndarray  # int32[nnz]

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1]) if self.M > 0 else 0

    def row_ids(self) -> np.ndarray:
        return np.repeat(np.arange(self.M, dtype=np.int64), np.diff(self.rowptr))


def csr_from_pairs(rows, cols, M: int, K: int, symmetric: bool = False, drop_diag: bool = False) -> Csr:
    """Canonical CSR (sorted, unique columns per row) from (row, col) pairs.

    ``symmetric`` also inserts (col, row); ``drop_diag`` drops (i, i)."""
    rows = np.ascontiguousarray(rows, dtype=np.int64).ravel()
    cols = np.ascontiguousarray(cols, dtype=np.int64).ravel()
    rowptr = np.zeros(M + 1, dtype=np.int64)
    colidx = np.empty(rows.size * (2 if symmetric else 1), dtype=np.int32)
    nnz = _native().gen_pairs_to_csr(rows.size, _p(rows), _p(cols), M, K, int(symmetric),
                                     int(drop_diag), _p(rowptr), _p(colidx))
    if nnz < 0:
        raise ValueError("pair index out of range")
    return Csr(M, K, rowptr, colidx[:nnz].copy())


# --------------------------------------------------------------------------- patterns

def uniform_random(M: int, K: int, nnz: int, seed: int) -> Csr:
    """Config T: nnz distinct positions sampled without replacement."""
    rng = np.random.default_rng(seed)
    k = rng.choice(M * K, size=nnz, replace=False)
    r, c = np.divmod(np.sort(k), K)
    return csr_from_pairs(r, c, M, K)


def stencil27(nx: int) -> Csr:
    """Config S(i): 27-point stencil on an nx^3 grid, row id = x + nx*y + nx^2*z."""
    n = nx ** 3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % nx, idx // (nx * nx)
    rows, cols = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < nx)
                      & (z + dz >= 0) & (z + dz < nx))
                rows.append(idx[ok])
                cols.append(idx[ok] + dx + nx * dy + nx * nx * dz)
    return csr_from_pairs(np.concatenate(rows), np.concatenate(cols), n, n)


def banded_random(M: int, per_row: int, halfwidth: int, seed: int) -> Csr:
    """Config S(ii): per_row uniform draws within +-halfwidth of the diagonal, deduplicated."""
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(M, dtype=np.int64), per_row)
    c = np.clip(r + rng.integers(-halfwidth, halfwidth + 1, size=r.size), 0, M - 1)
    return csr_from_pairs(r, c, M, M)


def dcsbm(n: int, target_nnz: int, communities: int, alpha: float, mu: float,
          dmax: float, seed: int, oversample: float = 1.0) -> Csr:
    """Configs R / P: symmetric degree-corrected SBM, labels uncorrelated with ids.

    1. comm ~ U{0..C-1}; 2. theta = 1 + Lomax(alpha-1), rescaled to mean
    target_nnz/n and capped at dmax; 3. E = oversample*target_nnz/2 edges,
    src ~ Cat(theta), dst ~ Cat(theta) with prob. mu else Cat(theta | comm[src]);
    4. drop self-loops, symmetrise, deduplicate.
    """
    rng = np.random.default_rng(seed)
    comm = rng.integers(0, communities, size=n)
    theta = 1.0 + rng.pareto(alpha - 1.0, size=n)
    theta *= (target_nnz / n) / theta.mean()
    theta = np.minimum(theta, dmax)
    E = int(oversample * target_nnz / 2)
    cum = np.cumsum(theta)
    # within-community draws: vertices sorted by community, per-community cumulative weights
    order = np.argsort(comm, kind="stable").astype(np.int64)
    cum_sorted = np.cumsum(theta[order])
    starts = np.searchsorted(comm[order], np.arange(communities), side="left").astype(np.int64)
    ends = np.searchsorted(comm[order], np.arange(communities), side="right").astype(np.int64)
    base = np.where(starts > 0, cum_sorted[np.maximum(starts - 1, 0)], 0.0)
    tot = np.where(ends > starts, cum_sorted[np.maximum(ends - 1, 0)] - base, 0.0)
    comm32 = comm.astype(np.int32)
    src = np.empty(E, dtype=np.int64)
    dst = np.empty(E, dtype=np.int64)
    _native().gen_dcsbm_draw(E, n, _p(cum), _p(comm32), _p(order), _p(cum_sorted), _p(starts), _p(ends),
                             _p(base), _p(tot), float(mu), int(seed) & 0xFFFFFFFFFFFFFFFF, _p(src), _p(dst))
    return csr_from_pairs(src, dst, n, n, symmetric=True, drop_diag=True)


def powerlaw_directed(n: int, mean_deg: float, seed: int, mu: float = 2.3, sigma: float = 0.8,
                      dmax: int = 2000, alpha: float = 1.2) -> Csr:
    """Config X (papers100M-shaped): out-degree round(lognormal(mu, sigma)) rescaled to mean
    ``mean_deg``, capped at dmax; columns ~ Cat(p), p_j = 1 + Lomax(alpha); dedup per row."""
    lib = _native()
    rng = np.random.default_rng(seed)
    w = 1.0 + rng.pareto(alpha, size=n)
    prob = np.empty(n, dtype=np.float64)
    alias = np.empty(n, dtype=np.int64)
    lib.gen_alias_build(n, _p(w), _p(prob), _p(alias))
    del w
    deg = np.empty(n, dtype=np.int64)
    lib.gen_x_degrees(n, float(mean_deg), float(mu), float(sigma), int(dmax), int(seed) & 0xFFFFFFFFFFFFFFFF, _p(deg))
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=off[1:])
    del deg
    colidx = np.empty(int(off[-1]), dtype=np.int32)
    rowptr = np.empty(n + 1, dtype=np.int64)
    nnz = lib.gen_x_fill(n, n, _p(off), _p(prob), _p(alias), (int(seed) * 7919 + 1) & 0xFFFFFFFFFFFFFFFF,
                         _p(colidx), _p(rowptr))
    del off, prob, alias
    if nnz < colidx.size:
        colidx = colidx[:nnz].copy()
    return Csr(n, n, rowptr, colidx)


def road_grid(side: int, keep: float, seed: int, shuffle: bool = True) -> Csr:
    """roadNet-shaped (PAPER Table 1 type-1, rCA/rPA, AvgL ~2.8): the side x side 4-neighbour
    grid, each undirected edge kept with probability ``keep`` (grid degree 4 -> AvgL ~4*keep),
    symmetric, no self-loops; labels shuffled unless ``shuffle`` is False."""
    rng = np.random.default_rng(seed)
    n = side * side
    idx = np.arange(n, dtype=np.int64)
    x, y = idx % side, idx // side
    right = idx[x + 1 < side]
    down = idx[y + 1 < side]
    src = np.concatenate([right, down])
    dst = np.concatenate([right + 1, down + side])
    k = rng.random(src.size) < keep
    src, dst = src[k], dst[k]
    if shuffle:
        lab = rng.permutation(n).astype(np.int64)
        src, dst = lab[src], lab[dst]
    return csr_from_pairs(src, dst, n, n, symmetric=True, drop_diag=True)


def molecules(n_graphs: int, mean_nodes: float, extra_edge_frac: float, seed: int, window: int = 0) -> Csr:
    """Graph-classification-shaped (PAPER Table 1 type-1: YeastH/OVCAR-8H/Yeast AvgL ~2.1, DD
    AvgL ~5): a block-diagonal union of ``n_graphs`` small graphs with consecutive ids (as in
    the TU datasets).  Each graph: a random recursive tree (node i joins a random earlier node,
    within the previous ``window`` nodes if window > 0) plus extra_edge_frac * size random
    chords (rings / contacts); symmetric, no self-loops."""
    rng = np.random.default_rng(seed)
    sizes = np.maximum(2, rng.poisson(mean_nodes - 2, n_graphs) + 2).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)])
    n = int(off[-1])
    g = np.repeat(np.arange(n_graphs), sizes)
    local = np.arange(n, dtype=np.int64) - off[g]
    child = np.nonzero(local > 0)[0]
    lo = np.zeros(child.size, np.int64) if window <= 0 else np.maximum(0, local[child] - window)
    parent_local = lo + np.floor(rng.random(child.size) * (local[child] - lo)).astype(np.int64)
    src = [child, off[g[child]] + parent_local]
    n_extra = int(extra_edge_frac * n)
    eg = rng.integers(0, n_graphs, n_extra)
    a = off[eg] + np.floor(rng.random(n_extra) * sizes[eg]).astype(np.int64)
    if window > 0:
        b = np.clip(a + rng.integers(-window, window + 1, n_extra), off[eg], off[eg + 1] - 1)
    else:
        b = off[eg] + np.floor(rng.random(n_extra) * sizes[eg]).astype(np.int64)
    rows = np.concatenate([src[0], a])
    cols = np.concatenate([src[1], b])
    return csr_from_pairs(rows, cols, n, n, symmetric=True, drop_diag=True)


def web_hosts(n: int, mean_deg: float, local_frac: float, seed: int, mean_host: float = 2000.0) -> Csr:
    """web-BerkStan-shaped (PAPER Table 1 type-1, AvgL 11.09): directed; pages in host blocks of
    consecutive ids (sizes 1 + Lomax(1.5) scaled to ``mean_host``); out-degree lognormal
    rescaled to ``mean_deg``; a link stays in its host with probability ``local_frac``
    (uniform there), else goes to a global page ~ Cat(1 + Lomax(1.2)); dedup per row."""
    rng = np.random.default_rng(seed)
    hs = 1.0 + rng.pareto(1.5, size=max(1, int(2 * n / mean_host)))
    hs = np.maximum(1, np.round(hs * mean_host / hs.mean())).astype(np.int64)
    hs = hs[np.cumsum(hs) <= n]
    hs = np.append(hs, n - hs.sum()) if hs.sum() < n else hs
    hoff = np.concatenate([[0], np.cumsum(hs)])
    host = np.repeat(np.arange(hs.size), hs)
    d = rng.lognormal(1.8, 1.0, n)
    deg = np.minimum(np.round(d * mean_deg / d.mean()).astype(np.int64), 5000)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    loc = rng.random(src.size) < local_frac
    h = host[src]
    dst = np.empty(src.size, np.int64)
    dst[loc] = hoff[h[loc]] + np.floor(rng.random(int(loc.sum())) * hs[h[loc]]).astype(np.int64)
    pop = 1.0 + rng.pareto(1.2, size=n)
    cdf = np.cumsum(pop)
    cdf /= cdf[-1]
    dst[~loc] = np.minimum(np.searchsorted(cdf, rng.random(int((~loc).sum()))), n - 1)
    return csr_from_pairs(src, dst, n, n)


def add_hub_rows(A: Csr, hubs: int, nnz_per_hub: int, seed: int) -> Csr:
    """SURVEY §8(d) P adversarial variant: ``hubs`` rows (spread over the matrix) replaced by rows
    of ``nnz_per_hub`` distinct uniformly drawn columns (not symmetrised: the load balancer's
    worst case is one window with ~nnz_per_hub / 8 * hubs-in-window blocks)."""
    rng = np.random.default_rng(seed)
    hub_rows = np.sort(rng.choice(A.M, size=hubs, replace=False))
    keep = ~np.isin(A.row_ids(), hub_rows)
    rows = [A.row_ids()[keep]]
    cols = [A.colidx[keep].astype(np.int64)]
    for h in hub_rows:
        rows.append(np.full(nnz_per_hub, h, np.int64))
        cols.append(rng.choice(A.K, size=nnz_per_hub, replace=False).astype(np.int64))
    return csr_from_pairs(np.concatenate(rows), np.concatenate(cols), A.M, A.K)


def sbm(n: int, blocks: int, p_in: float, p_out: float, seed: int, shuffle: bool = True) -> Csr:
    """Symmetric 0/1 stochastic block model, no self-loops, optional label shuffle."""
    rng = np.random.default_rng(seed)
    b = np.arange(n) // (n // blocks)
    iu, ju = np.triu_indices(n, 1)
    p = np.where(b[iu] == b[ju], p_in, p_out)
    keep = rng.random(iu.size) < p
    r, c = iu[keep], ju[keep]
    if shuffle:
        lab = rng.permutation(n)
        r, c = lab[r], lab[c]
    return csr_from_pairs(r, c, n, n, symmetric=True)


def identity(n: int) -> Csr:
    i = np.arange(n)
    return csr_from_pairs(i, i, n, n)


def permutation_matrix(n: int, seed: int) -> Csr:
    """A = P with one 1 per row at column sigma(i) (SURVEY §8(c) C-4, a7/a10 fixture)."""
    rng = np.random.default_rng(seed)
    return csr_from_pairs(np.arange(n), rng.permutation(n), n, n)


def two_cliques(k: int, seed: int | None = None, bridge: bool = True) -> Csr:
    """Two k-cliques (optionally joined by one edge), labels optionally shuffled."""
    rows, cols = [], []
    for off in (0, k):
        for i in range(k):
            for j in range(k):
                if i != j:
                    rows.append(off + i)
                    cols.append(off + j)
    if bridge:
        rows += [k - 1, k]
        cols += [k, k - 1]
    rows, cols = np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)
    if seed is not None:
        lab = np.random.default_rng(seed).permutation(2 * k)
        rows, cols = lab[rows], lab[cols]
    return csr_from_pairs(rows, cols, 2 * k, 2 * k)


def star(leaves: int) -> Csr:
    """K_{1,leaves}: centre 0 joined to 1..leaves."""
    r = np.concatenate([np.zeros(leaves, int), np.arange(1, leaves + 1)])
    c = np.concatenate([np.arange(1, leaves + 1), np.zeros(leaves, int)])
    return csr_from_pairs(r, c, leaves + 1, leaves + 1)


# --------------------------------------------------------------------------- values

def values_uniform(nnz: int, seed: int, chunk: int = 1 << 24) -> np.ndarray:
    """A values ~ U[-1, 1) float32 (SURVEY §8(d) 'Values and B'); drawn in chunks from one
    stream (identical to a single draw) so 1.6B values need no float64 temporary."""
    rng = np.random.default_rng(seed)
    out = np.empty(nnz, dtype=np.float32)
    for a in range(0, nnz, chunk):
        n = min(chunk, nnz - a)
        out[a:a + n] = rng.uniform(-1.0, 1.0, n)
    return out


def values_int(nnz: int, seed: int) -> np.ndarray:
    """Integer variant: A in {-3..3} \\ {0} (bit-exact in TF32/FP16 x FP32 accumulate)."""
    rng = np.random.default_rng(seed)
    mag = rng.integers(1, 4, size=nnz)
    sgn = np.where(rng.random(nnz) < 0.5, -1, 1)
    return (mag * sgn).astype(np.float32)


def dense_normal(K: int, N: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((K, N), dtype=np.float32)


def dense_int(K: int, N: int, seed: int) -> np.ndarray:
    """Integer variant: B in {-8..8}."""
    return np.random.default_rng(seed).integers(-8, 9, size=(K, N)).astype(np.float32)
