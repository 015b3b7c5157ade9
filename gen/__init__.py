"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the SpMM method (no rounding, no tiling, no
encoding, no product): it only draws sparse patterns, values and dense operands
with the shapes and distributions of the paper's workloads (SURVEY.md §8(d),
"Configs as concrete synthetic inputs"; Table 1).
"""
from .matrices import (  # noqa: F401
    Csr,
    csr_from_pairs,
    uniform_random,
    stencil27,
    banded_random,
    dcsbm,
    powerlaw_directed,
    road_grid,
    molecules,
    web_hosts,
    add_hub_rows,
    sbm,
    identity,
    permutation_matrix,
    two_cliques,
    star,
    values_uniform,
    values_int,
    dense_normal,
    dense_int,
)
from .configs import CONFIGS, make_config  # noqa: F401
