"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO AllReduce or policy arithmetic: it only draws numbers.  It
is the one module both sides (oracle/ and the CUDA path's tests) may import
(DESIGN.md "Input recipe").

Every array is a pure function of (cfg, rank, count, dtype, dist), drawn with
numpy ``PCG64(SeedSequence([2603, cfg, rank, count, dist_id, dtype_id]))``
(SURVEY.md §8(d) "Synthetic inputs per config").  bf16 values are returned as
their uint16 bit patterns; they are made by TRUNCATING a float32 draw to its top
16 bits (round-toward-zero), so the generator never performs the bf16
round-to-nearest-even that the oracle and the kernels implement.

Distributions (BASELINE.json configs):

=========  =====================================================================
dist       meaning
=========  =====================================================================
``ints``   integer values: i32 in [-2^20, 2^20), i64 in [-2^40, 2^40),
           f32 in [-2^12, 2^12] (every rank-order sum exact in f32 for n<=8),
           bf16 in [-16, 16] (every sum of <=8 terms exact in bf16)
``full``   i32 / i64 over the full two's-complement range (exercises wrap)
``unif``   f32 / bf16 uniform(-1, 1)
``logu``   f32 / bf16 random sign x 2^U(-20, 20)  (wide dynamic range)
``normal`` f32 / bf16 N(0, 1)
``small``  i32 / i64 in [-8, 8)  (tiny domain for brute force)
=========  =====================================================================
"""
from __future__ import annotations

import numpy as np

DTYPES = ("i32", "i64", "f32", "bf16")
DISTS = ("ints", "full", "unif", "logu", "normal", "small")
_DTYPE_ID = {d: i for i, d in enumerate(DTYPES)}
_DIST_ID = {d: i for i, d in enumerate(DISTS)}

#: numpy storage dtype of each logical dtype (bf16 travels as raw uint16 bits)
NP_STORAGE = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "bf16": np.uint16}
ESIZE = {"i32": 4, "i64": 8, "f32": 4, "bf16": 2}


def rng(cfg: int, rank: int, count: int, dtype: str, dist: str) -> np.random.Generator:
    ss = np.random.SeedSequence([2603, int(cfg), int(rank), int(count),
                                 _DIST_ID[dist], _DTYPE_ID[dtype]])
    return np.random.Generator(np.random.PCG64(ss))


def _f32_to_bf16_bits_truncate(x: np.ndarray) -> np.ndarray:
    """Top 16 bits of each float32: a bf16 value (round toward zero)."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def gen(dtype: str, count: int, rank: int, cfg: int = 0, dist: str = "ints") -> np.ndarray:
    """One rank's input vector of ``count`` elements (numpy storage dtype)."""
    if dtype not in NP_STORAGE:
        raise ValueError(f"unknown dtype {dtype!r}")
    g = rng(cfg, rank, count, dtype, dist)
    n = int(count)
    if dtype == "i32":
        if dist == "full":
            return g.integers(-(2**31), 2**31, size=n, dtype=np.int64).astype(np.int32)
        if dist == "small":
            return g.integers(-8, 8, size=n, dtype=np.int32)
        return g.integers(-(2**20), 2**20, size=n, dtype=np.int32)
    if dtype == "i64":
        if dist == "full":
            return g.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, size=n,
                              dtype=np.int64, endpoint=True)
        if dist == "small":
            return g.integers(-8, 8, size=n, dtype=np.int64)
        return g.integers(-(2**40), 2**40, size=n, dtype=np.int64)
    # floating point
    if dist == "ints":
        lim = 2**12 if dtype == "f32" else 16
        x = g.integers(-lim, lim, size=n, dtype=np.int32, endpoint=True).astype(np.float32)
    elif dist == "unif":
        x = g.uniform(-1.0, 1.0, size=n).astype(np.float32)
    elif dist == "logu":
        mag = np.exp2(g.uniform(-20.0, 20.0, size=n))
        sign = np.where(g.integers(0, 2, size=n) == 0, -1.0, 1.0)
        x = (sign * mag).astype(np.float32)
    elif dist == "normal":
        x = g.standard_normal(size=n, dtype=np.float32)
    else:
        raise ValueError(f"dist {dist!r} not defined for {dtype}")
    if dtype == "f32":
        return x
    return _f32_to_bf16_bits_truncate(x)


def gen_ranks(dtype: str, count: int, nranks: int, cfg: int = 0, dist: str = "ints") -> list:
    """Inputs of all ranks, rank order."""
    return [gen(dtype, count, r, cfg, dist) for r in range(nranks)]
