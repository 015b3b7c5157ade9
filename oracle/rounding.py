"""rho: the input rounding both sides apply before the product (TEST INFRASTRUCTURE ONLY).

PAPER.md P:308 fixes the arithmetic type ("we mainly focus on tf32 datatype")
but never the rounding mode; SURVEY §8(c) Q1 adopts round-to-nearest, ties
away from zero (the semantics of PTX ``cvt.rna.tf32.f32``), applied
unconditionally on the float32 bit pattern:

    u = bits(x);  u = (u + 0x1000) & 0xFFFFE000

This is written out here as that definition for every non-NaN input: Inf stays
Inf and values with |bits| >= 0x7F7FF000 overflow to +-Inf.  NaN inputs are not
rounded but truncated, u & 0xFFFFE000 (so a NaN whose payload lives only in the
low 13 bits becomes +-Inf): that is what cvt.rna.tf32.f32 does on sm_100a, as
pinned by the exhaustive 2^32-pattern test (tests/test_gpu_parity.py) and
recorded as DESIGN.md reading R1.  The bit trick alone would wrap large NaN
payloads into the sign bit, which no hardware does.

FP16 path: IEEE round-to-nearest-even, i.e. numpy's
float32 -> float16 cast.
"""
from __future__ import annotations

import numpy as np


def tf32_rna(x, chunk: int = 1 << 24) -> np.ndarray:
    """TF32 round-to-nearest, ties away from zero, kept in float32 bits.

    Computed in uint32, chunk by chunk (the bench's papers100M-shaped B is 28 GB): for a
    non-NaN input u + 0x1000 cannot wrap (|bits| <= 0x7F800000), NaNs take the truncation."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    src = x.reshape(-1).view(np.uint32)
    out = np.empty(src.size, dtype=np.uint32)
    mask = np.uint32(0xFFFFE000)
    for a in range(0, src.size, chunk):
        u = src[a:a + chunk]
        r = (u + np.uint32(0x1000)) & mask
        nan = (u & np.uint32(0x7FFFFFFF)) > np.uint32(0x7F800000)
        if nan.any():
            r[nan] = u[nan] & mask
        out[a:a + chunk] = r
    return out.view(np.float32).reshape(x.shape)


def fp16_rne(x) -> np.ndarray:
    """IEEE binary16 round-to-nearest-even."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float32).astype(np.float16)


def rho(x, precision: str) -> np.ndarray:
    """Rounded operand as float32 (exactly representable), for the FP64 oracle."""
    if precision == "tf32":
        return tf32_rna(x)
    if precision == "fp16":
        return fp16_rne(x).astype(np.float32)
    raise ValueError(precision)
