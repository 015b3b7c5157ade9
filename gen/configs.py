"""Named synthetic workloads = BASELINE.json ``configs`` made concrete.

| name      | BASELINE.json config                          | shape template        |
|-----------|-----------------------------------------------|----------------------------------|
| tiny      | configs[0] 512x512 ~5K nnz, N=16              | -                                |
| stencil   | configs[1] SuiteSparse-shaped banded/FEM 1M   | SuiteSparse FEM          |
| banded    | configs[1] variant (ii), banded-random        | -                                |
| reddit    | configs[2] Reddit-shaped, N=32/64/128         | reddit 232,965 / 114.8M  |
| products  | configs[3] ogbn-products-shaped, N=128        | -                                |
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from . import matrices as mx


@dataclass(frozen=True)
class Config:
    name: str
    baseline_index: int
    Ns: tuple
    seed_A: int
    seed_B: int
    build: Callable[[], "mx.Csr"]
    note: str


def _tiny():
    return mx.uniform_random(512, 512, 5120, seed=1)


def _stencil():
    return mx.stencil27(100)


def _banded():
    return mx.banded_random(1_000_000, 30, 256, seed=3)


def _reddit():
    # DC-SBM, 41 communities, Pareto(2.3) weights, mean ~493, cap 21,657, mu=0.25
    return mx.dcsbm(232_965, 114_848_857, 41, 2.3, 0.25, 21_657, seed=7, oversample=1.36)


def _products():
    return mx.dcsbm(2_449_029, 123_718_280, 47, 2.1, 0.10, 17_481, seed=9, oversample=1.22)


def _papers100m():
    # directed, out-degree lognormal(2.3, 0.8) rescaled to mean 14.55, popularity Pareto(1.2)
    return mx.powerlaw_directed(111_059_956, 14.55, seed=11)


def _papers100m_small():
    # 1/64 scale of config X with the same per-row statistics (CPU-checkable, multi-GPU tests)
    return mx.powerlaw_directed(111_059_956 // 64, 14.55, seed=11)


CONFIGS = {
    "tiny": Config("tiny", 0, (16,), 1, 2, _tiny, "uniform random 512x512, 5120 nnz"),
    "stencil": Config("stencil", 1, (128,), 3, 4, _stencil, "27-point stencil on 100^3 grid, 26.46M nnz"),
    "banded": Config("banded", 1, (128,), 3, 4, _banded, "banded-random 1M rows, 30 draws/row within +-256"),
    "reddit": Config("reddit", 2, (32, 64, 128), 7, 8, _reddit,
                     "Reddit-shaped DC-SBM 232,965 nodes ~115M nnz, labels shuffled"),
    "products": Config("products", 3, (128,), 9, 10, _products,
                       "ogbn-products-shaped DC-SBM 2,449,029 nodes ~124M nnz"),
    "papers100m": Config("papers100m", 4, (64,), 11, 12, _papers100m,
                         "ogbn-papers100M-shaped directed power-law 111,059,956 nodes ~1.6B nnz"),
    "papers100m_small": Config("papers100m_small", 4, (64,), 11, 12, _papers100m_small,
                               "papers100M-shaped at 1/64 scale (1,735,311 nodes ~25M nnz)"),
}


def make_config(name: str):
    cfg = CONFIGS[name]
    return cfg, cfg.build()
