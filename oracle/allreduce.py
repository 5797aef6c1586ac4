"""Oracle: the AllReduce result by its plain definition — TEST INFRASTRUCTURE ONLY.

Definition followed (SURVEY.md §8(c) "Definition of the result"; PAPER.md
L106-107 names AllReduce as the collective the policy selects algorithms for;
SPEC.md L622 glossary "Collective"): an AllReduce of x_0 .. x_{n-1}, each of
``count`` elements, leaves on EVERY rank

    y[i] = op( ... op( op(x_0[i], x_1[i]), x_2[i]) ..., x_{n-1}[i])

evaluated left to right in rank order.  Precision per dtype (DESIGN.md readings
R2, R3, R5):

* i32 / i64: two's-complement wrap-around (computed in uint32 / uint64 so the
  wrap is defined); max / min on the signed values.
* f32: one IEEE-754 binary32 round-to-nearest-even add per rank, in rank order
  (numpy elementwise float32 add: no FMA, no pairwise summation).
* bf16: each input widened exactly to f32 (bits << 16), accumulated in f32 in
  rank order, rounded ONCE to bf16 with round-to-nearest-even
  (R3: "every bf16 kernel accumulates in f32 and rounds once").
* float max / min: fmax / fmin (inputs carry no NaN; the result is one of the
  inputs, so it is exact).

Arrays use the storage dtypes of ``synth.NP_STORAGE``; bf16 is uint16 bits.
Parity: pinned by tests/test_oracle_allreduce.py (pure-Python brute force with
exact rational arithmetic, closed forms, a library routine for the bf16
rounding special case, invariants).
"""
from __future__ import annotations

import numpy as np

OPS = ("sum", "max", "min")


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float32 values."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_bits_rne(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 bits, round-to-nearest, ties-to-even.

    With b the uint32 pattern of x: (b + 0x7FFF + ((b >> 16) & 1)) >> 16.
    (No NaN reaches this function: inputs are finite and sums of <= 8 finite
    bf16 values stay finite in f32.)
    """
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def allreduce(xs, dtype: str, op: str) -> np.ndarray:
    """Rank-ordered AllReduce of the per-rank arrays ``xs`` (list, rank order).

    Returns the single vector every rank must hold afterwards.
    """
    if op not in OPS:
        raise ValueError(f"unknown op {op!r}")
    n = len(xs)
    if n == 0:
        raise ValueError("need at least one rank")
    count = len(xs[0])
    for x in xs:
        if len(x) != count:
            raise ValueError("ranks disagree on count")
    if dtype in ("i32", "i64"):
        st = np.int32 if dtype == "i32" else np.int64
        ut = np.uint32 if dtype == "i32" else np.uint64
        if op == "sum":
            acc = np.array(xs[0], dtype=st).view(ut).copy()
            for r in range(1, n):
                np.add(acc, np.asarray(xs[r], dtype=st).view(ut), out=acc)
            return acc.view(st)
        acc = np.array(xs[0], dtype=st, copy=True)
        f = np.maximum if op == "max" else np.minimum
        for r in range(1, n):
            f(acc, np.asarray(xs[r], dtype=st), out=acc)
        return acc
    if dtype == "f32":
        acc = np.array(xs[0], dtype=np.float32, copy=True)
        f = {"sum": np.add, "max": np.fmax, "min": np.fmin}[op]
        for r in range(1, n):
            f(acc, np.asarray(xs[r], dtype=np.float32), out=acc)
        return acc
    if dtype == "bf16":
        acc = bf16_bits_to_f32(xs[0]).copy()
        f = {"sum": np.add, "max": np.fmax, "min": np.fmin}[op]
        for r in range(1, n):
            f(acc, bf16_bits_to_f32(xs[r]), out=acc)
        return f32_to_bf16_bits_rne(acc)
    raise ValueError(f"unknown dtype {dtype!r}")


def allreduce_window(gen_rank, nranks: int, count: int, dtype: str, op: str,
                     lo: int, hi: int) -> np.ndarray:
    """Oracle over the element window [lo, hi) only.

    ``gen_rank(r)`` returns rank r's full input (the caller may cache it);
    used to check sampled outputs at full bench sizes without materialising
    the whole result.
    """
    return allreduce([np.asarray(gen_rank(r))[lo:hi] for r in range(nranks)], dtype, op)
