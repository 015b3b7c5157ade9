"""Named synthetic workloads = BASELINE.json ``configs`` made concrete.

| name      | BASELINE.json config                          | shape template        |
|-----------|-----------------------------------------------|----------------------------------|
| tiny      | configs[0] 512x512 ~5K nnz, N=16              | -                                |
| stencil   | configs[1] SuiteSparse-shaped banded/FEM 1M   | SuiteSparse FEM          |
| banded    | configs[1] variant (ii), banded-random        | -                                |
| reddit    | configs[2] Reddit-shaped, N=32/64/128         | reddit 232,965 / 114.8M  |
| products  | configs[3] ogbn-products-shaped, N=128        | -                                |
| roadnet, yeasth, dd, webberkstan | not a BASELINE config: PAPER Table 1 type-1 shapes (NEXT-3) | P:469-475 |
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


def _products_hubs():
    # SURVEY §8(d) P adversarial variant: products-shaped plus 8 hub rows of 200K nnz each
    return mx.add_hub_rows(_products(), 8, 200_000, seed=21)


def _papers100m():
    # directed, out-degree lognormal(2.3, 0.8), popularity Pareto(1.2).  The drawn mean is 15.37
    # so that after per-row deduplication (hot columns collide at this scale) the matrix holds
    # 1,613,461,269 nnz = 14.53 per row, ogbn-papers100M's ~1.616B (BASELINE configs[4]); a
    # drawn mean of 14.55 gave 1.53B
    return mx.powerlaw_directed(111_059_956, 15.37, seed=11)


def _papers100m_small():
    # 1/64 scale of config X with the same per-row statistics (CPU-checkable, multi-GPU tests)
    return mx.powerlaw_directed(111_059_956 // 64, 14.55, seed=11)


# PAPER Table 1 type-1 matrices (small AvgL), for NEXT-3's narrow-window workloads
def _roadnet():
    # roadNet-CA: 1,971,281 rows, 5,533,214 nnz, AvgL 2.81 -> 1404^2 grid, edge keep 0.7025
    return mx.road_grid(1404, 0.7025, seed=13)


def _yeasth():
    # YeastH: 3,138,114 rows, 6,487,230 nnz, AvgL 2.07 -> ~39-node molecules, 3.5% ring chords
    return mx.molecules(80_464, 39.0, 0.063, seed=15)


def _dd():
    # DD: 334,926 rows, 1,686,092 nnz, AvgL 5.03 -> ~284-node protein graphs, local contacts
    return mx.molecules(1_178, 284.3, 1.85, seed=17, window=12)


def _webberkstan():
    # web-BerkStan: 685,230 rows, 7,600,595 nnz, AvgL 11.09 -> host blocks, 80% local links
    return mx.web_hosts(685_230, 11.15, 0.8, seed=19)


CONFIGS = {
    "tiny": Config("tiny", 0, (16,), 1, 2, _tiny, "uniform random 512x512, 5120 nnz"),
    "stencil": Config("stencil", 1, (128,), 3, 4, _stencil, "27-point stencil on 100^3 grid, 26.46M nnz"),
    "banded": Config("banded", 1, (128,), 3, 4, _banded, "banded-random 1M rows, 30 draws/row within +-256"),
    "reddit": Config("reddit", 2, (32, 64, 128), 7, 8, _reddit,
                     "Reddit-shaped DC-SBM 232,965 nodes ~115M nnz, labels shuffled"),
    "products": Config("products", 3, (128,), 9, 10, _products,
                       "ogbn-products-shaped DC-SBM 2,449,029 nodes ~124M nnz"),
    "roadnet": Config("roadnet", -1, (128, 256, 512), 13, 14, _roadnet,
                      "roadNet-CA-shaped grid road graph 1,971,216 nodes ~5.5M nnz (type-1), labels shuffled"),
    "yeasth": Config("yeasth", -1, (128, 256, 512), 15, 16, _yeasth,
                     "YeastH-shaped union of ~39-node molecules ~3.1M nodes ~6.5M nnz (type-1)"),
    "dd": Config("dd", -1, (128, 256, 512), 17, 18, _dd,
                 "DD-shaped union of ~284-node protein graphs ~335K nodes ~1.7M nnz (type-1)"),
    "webberkstan": Config("webberkstan", -1, (128, 256, 512), 19, 20, _webberkstan,
                          "web-BerkStan-shaped directed host-block web graph 685,230 nodes ~7.6M nnz (type-1)"),
    "products_hubs": Config("products_hubs", 3, (128,), 9, 10, _products_hubs,
                            "ogbn-products-shaped DC-SBM plus 8 hub rows of 200K nnz (balancer stress)"),
    "papers100m": Config("papers100m", 4, (64,), 11, 12, _papers100m,
                         "ogbn-papers100M-shaped directed power-law 111,059,956 nodes ~1.6B nnz"),
    "papers100m_small": Config("papers100m_small", 4, (64,), 11, 12, _papers100m_small,
                               "papers100M-shaped at 1/64 scale (1,735,311 nodes ~25M nnz)"),
}


def make_config(name: str):
    cfg = CONFIGS[name]
    return cfg, cfg.build()
