"""Pins for oracle/rounding.py (rho) against closed forms, not against itself.

TF32 RNA: round to the nearest multiple of the TF32 quantum,
ties away from zero.  The closed form below is written in fp64 arithmetic
(quantum = 2^(e-11) for |x| in [2^(e-1), 2^e), 2^-136 below 2^-126), which is
independent of the bit trick the oracle uses.
"""
import math

import numpy as np

from oracle.rounding import fp16_rne, rho, tf32_rna


def _rna_closed_form(x: float) -> float:
    if x == 0.0 or not math.isfinite(x):
        return x
    ax = abs(x)
    if ax < 2.0 ** -126:
        q = 2.0 ** -136
    else:
        _, e = math.frexp(ax)          # ax in [2^(e-1), 2^e)
        q = 2.0 ** (e - 11)
    y = math.floor(ax / q + 0.5) * q
    if y >= 2.0 ** 128:
        y = math.inf
    return math.copysign(y, x)


def test_tf32_worked_values():
    one = 1.0
    cases = {
        one: one,
        one + 2 ** -10: one + 2 ** -10,          # representable: unchanged
        one + 2 ** -11: one + 2 ** -10,          # tie -> away from zero
        one + 2 ** -11 - 2 ** -23: one,          # below the tie -> down
        -(one + 2 ** -11): -(one + 2 ** -10),    # sign-symmetric
        3.0: 3.0,
        0.0: 0.0,
    }
    x = np.array(list(cases.keys()), dtype=np.float32)
    y = tf32_rna(x)
    assert y.tolist() == [np.float32(v) for v in cases.values()]


def test_tf32_matches_closed_form_random():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 32, size=200_000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x) & (np.abs(x) < 3.0e38)]
    y = tf32_rna(x)
    ref = np.array([_rna_closed_form(float(v)) for v in x], dtype=np.float64)
    assert np.array_equal(y.astype(np.float64), ref)


def test_tf32_low_bits_cleared_and_specials():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(10_000).astype(np.float32)
    assert np.all((tf32_rna(x).view(np.uint32) & 0x1FFF) == 0)
    sp = np.array([np.inf, -np.inf, np.nan, np.finfo(np.float32).max], dtype=np.float32)
    y = tf32_rna(sp)
    assert y[0] == np.inf and y[1] == -np.inf and np.isnan(y[2]) and y[3] == np.inf


def test_tf32_nan_truncated_not_rounded():
    """DESIGN.md reading R1: NaNs keep their sign and top payload bits, low 13 bits cleared."""
    u = np.array([0x7FC00000, 0x7FFFFFFF, 0x7F801FFF, 0x7F800001, 0xFFFFF000], dtype=np.uint32)
    y = tf32_rna(u.view(np.float32)).view(np.uint32)
    assert y.tolist() == [0x7FC00000, 0x7FFFE000, 0x7F800000, 0x7F800000, 0xFFFFE000]


def test_fp16_rne_ties_to_even():
    x = np.array([1 + 2 ** -11, 1 + 3 * 2 ** -11, 65520.0, 2 ** -25, -2.5], dtype=np.float32)
    y = fp16_rne(x).astype(np.float64)
    assert y.tolist() == [1.0, 1 + 2 ** -9, math.inf, 0.0, -2.5]


def test_rho_dispatch():
    x = np.float32([1 + 2 ** -11])
    assert rho(x, "tf32")[0] == np.float32(1 + 2 ** -10)
    assert rho(x, "fp16")[0] == np.float32(1.0)
