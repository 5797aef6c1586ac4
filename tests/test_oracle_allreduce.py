"""Pins for oracle/allreduce.py against things other than itself (CPU only).

* brute force on tiny inputs in pure Python: integers with explicit masking,
  floating point with EXACT rational arithmetic (fractions.Fraction) and an
  independent round-to-nearest-even onto the binary32 / bfloat16 grids;
* closed forms (SURVEY.md §8(c) "What pins each part");
* a library routine for the bf16 rounding special case (torch's float32 ->
  bfloat16 cast, round-to-nearest-even);
* the textbook recursive-summation error bound (Higham) for random f32;
* invariants: rank permutation (order-free ops), n = 1 identity, idempotence.
"""
from fractions import Fraction
import math
import struct

import numpy as np
import pytest

import synth
from oracle import allreduce as orc

# ---------------------------------------------------------------- brute force


def _round_to_grid(x: Fraction, p: int, emin: int) -> Fraction:
    """Round x to the binary floating-point grid with p significand bits and
    minimum normal exponent emin, ties to even (no overflow handling needed:
    test values stay far below the largest finite value)."""
    if x == 0:
        return Fraction(0)
    sign = -1 if x < 0 else 1
    a = abs(x)
    # e = floor(log2(a))
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, emin)
    ulp = Fraction(2) ** (e - p + 1)
    q = a / ulp
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * fl * ulp


def rf32(x: Fraction) -> Fraction:
    return _round_to_grid(x, 24, -126)


def rbf16(x: Fraction) -> Fraction:
    return _round_to_grid(x, 8, -126)


def f32_frac(v) -> Fraction:
    return Fraction(float(np.float32(v)))


def bf16_bits_frac(b) -> Fraction:
    f = struct.unpack("<f", struct.pack("<I", int(b) << 16))[0]
    return Fraction(f)


def frac_to_bf16_bits(x: Fraction) -> int:
    return struct.unpack("<I", struct.pack("<f", float(x)))[0] >> 16


def brute_int(xs, bits, op):
    mask = (1 << bits) - 1
    out = []
    for i in range(len(xs[0])):
        if op == "sum":
            acc = 0
            for x in xs:
                acc = (acc + (int(x[i]) & mask)) & mask
            if acc >= 1 << (bits - 1):
                acc -= 1 << bits
        elif op == "max":
            acc = int(xs[0][i])
            for x in xs[1:]:
                if int(x[i]) > acc:
                    acc = int(x[i])
        else:
            acc = int(xs[0][i])
            for x in xs[1:]:
                if int(x[i]) < acc:
                    acc = int(x[i])
        out.append(acc)
    return out


def brute_f32(xs, op):
    out = []
    for i in range(len(xs[0])):
        acc = f32_frac(xs[0][i])
        for x in xs[1:]:
            v = f32_frac(x[i])
            if op == "sum":
                acc = rf32(acc + v)
            elif op == "max":
                acc = v if v > acc else acc
            else:
                acc = v if v < acc else acc
        out.append(acc)
    return out


def brute_bf16(xs, op):
    out = []
    for i in range(len(xs[0])):
        acc = bf16_bits_frac(xs[0][i])
        for x in xs[1:]:
            v = bf16_bits_frac(x[i])
            if op == "sum":
                acc = rf32(acc + v)          # f32 accumulation, one RNE per add
            elif op == "max":
                acc = v if v > acc else acc
            else:
                acc = v if v < acc else acc
        out.append(frac_to_bf16_bits(rbf16(acc)))   # single final rounding
    return out


@pytest.mark.parametrize("op", ["sum", "max", "min"])
@pytest.mark.parametrize("dtype", ["i32", "i64"])
@pytest.mark.parametrize("dist", ["small", "full"])
def test_brute_force_int(dtype, op, dist):
    bits = 32 if dtype == "i32" else 64
    for n in range(1, 9):
        for count in (0, 1, 2, 3, 7, 16, 33):
            xs = synth.gen_ranks(dtype, count, n, cfg=90 + n, dist=dist)
            got = orc.allreduce(xs, dtype, op)
            assert got.dtype == synth.NP_STORAGE[dtype]
            assert [int(v) for v in got] == brute_int(xs, bits, op)


@pytest.mark.parametrize("op", ["sum", "max", "min"])
@pytest.mark.parametrize("dist", ["unif", "logu", "normal"])
def test_brute_force_f32(op, dist):
    for n in range(1, 9):
        for count in (0, 1, 5, 24):
            xs = synth.gen_ranks("f32", count, n, cfg=70 + n, dist=dist)
            got = orc.allreduce(xs, "f32", op)
            exp = brute_f32(xs, op)
            assert [Fraction(float(v)) for v in got] == exp


@pytest.mark.parametrize("op", ["sum", "max", "min"])
@pytest.mark.parametrize("dist", ["unif", "logu", "normal", "ints"])
def test_brute_force_bf16(op, dist):
    for n in range(1, 9):
        for count in (0, 1, 5, 24):
            xs = synth.gen_ranks("bf16", count, n, cfg=50 + n, dist=dist)
            got = orc.allreduce(xs, "bf16", op)
            assert got.dtype == np.uint16
            assert [int(v) for v in got] == brute_bf16(xs, op)


def test_f32_rounding_steps_matter():
    """A case where left-to-right RNE differs from the exact sum: guards
    against an oracle that sums in higher precision or in another order."""
    big, small = np.float32(2.0 ** 24), np.float32(1.0)
    xs = [np.array([big]), np.array([small]), np.array([small])]
    got = orc.allreduce(xs, "f32", "sum")
    # (2^24 + 1) rounds to 2^24 (tie, even), twice
    assert float(got[0]) == 2.0 ** 24
    xs2 = [np.array([small]), np.array([small]), np.array([big])]
    assert float(orc.allreduce(xs2, "f32", "sum")[0]) == 2.0 ** 24 + 2


# ---------------------------------------------------------------- closed forms


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_closed_form_triangular(n):
    count = 1024
    i = np.arange(count, dtype=np.int64)
    xs = [((r + 1) * (i + 1)).astype(np.int32) for r in range(n)]
    got = orc.allreduce(xs, "i32", "sum")
    np.testing.assert_array_equal(got.astype(np.int64), (i + 1) * n * (n + 1) // 2)


def test_closed_form_wrap_i32():
    x = np.full(16, 0x7FFFFFFF, dtype=np.int32)
    assert (orc.allreduce([x, x], "i32", "sum") == -2).all()
    got8 = orc.allreduce([x] * 8, "i32", "sum")
    assert (got8.astype(np.int64) == ((8 * 0x7FFFFFFF) % 2**32) - 2**32).all()


def test_closed_form_wrap_i64():
    x = np.full(4, 2**62, dtype=np.int64)
    assert (orc.allreduce([x] * 4, "i64", "sum") == 0).all()
    assert (orc.allreduce([x] * 2, "i64", "sum") == np.iinfo(np.int64).min).all()


@pytest.mark.parametrize("dtype", ["i32", "i64", "f32"])
def test_closed_form_max_min(dtype):
    st = synth.NP_STORAGE[dtype]
    for n in range(1, 9):
        xs = [np.full(9, r, dtype=st) for r in range(n)]
        assert (orc.allreduce(xs, dtype, "max") == n - 1).all()
        assert (orc.allreduce(xs, dtype, "min") == 0).all()


def test_closed_form_integer_valued_floats_exact():
    """Integer-valued inputs make every f32/bf16 sum exact (SURVEY §8(c) point 3)."""
    for n in range(1, 9):
        xs = synth.gen_ranks("f32", 4096, n, cfg=1, dist="ints")
        exact = sum(x.astype(np.int64) for x in xs)
        np.testing.assert_array_equal(orc.allreduce(xs, "f32", "sum").astype(np.int64), exact)
        xb = synth.gen_ranks("bf16", 4096, n, cfg=3, dist="ints")
        vals = [orc.bf16_bits_to_f32(x).astype(np.int64) for x in xb]
        exact_b = sum(vals)
        got = orc.bf16_bits_to_f32(orc.allreduce(xb, "bf16", "sum")).astype(np.int64)
        np.testing.assert_array_equal(got, exact_b)


# ------------------------------------------------- library routine (bf16 RNE)


def test_bf16_rounding_matches_torch_cast():
    torch = pytest.importorskip("torch")
    g = np.random.default_rng(7)
    x = g.standard_normal(200000).astype(np.float32) * np.float32(1000)
    # force many exact ties: low 16 bits = 0x8000
    ties = (x.view(np.uint32) & np.uint32(0xFFFF0000)) | np.uint32(0x8000)
    x = np.concatenate([x, ties.view(np.float32), np.array([0.0, -0.0, 1.0, -1.0], np.float32)])
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(orc.f32_to_bf16_bits_rne(x), ref)


# ------------------------------------------------------- textbook error bound


@pytest.mark.parametrize("n", [2, 4, 8])
def test_f32_recursive_summation_bound(n):
    """|fl(sum) - sum| <= (n-1) u sum|x| + O(u^2), u = 2^-24 (Higham, recursive
    summation).  Exact reference with Fractions."""
    xs = synth.gen_ranks("f32", 600, n, cfg=11, dist="unif")
    got = orc.allreduce(xs, "f32", "sum")
    u = Fraction(1, 2**24)
    for i in range(600):
        exact = sum(Fraction(float(x[i])) for x in xs)
        abssum = sum(abs(Fraction(float(x[i]))) for x in xs)
        err = abs(Fraction(float(got[i])) - exact)
        assert err <= (n - 1) * u * abssum * (1 + n * u)


# ------------------------------------------------------------------ invariants


@pytest.mark.parametrize("dtype,op", [("i32", "sum"), ("i64", "sum"), ("i32", "max"),
                                      ("i64", "min"), ("f32", "max"), ("f32", "min"),
                                      ("bf16", "max"), ("bf16", "min")])
def test_rank_permutation_invariance(dtype, op):
    xs = synth.gen_ranks(dtype, 777, 8, cfg=5, dist="full" if dtype[0] == "i" else "normal")
    ref = orc.allreduce(xs, dtype, op)
    g = np.random.default_rng(3)
    for _ in range(4):
        perm = g.permutation(8)
        np.testing.assert_array_equal(orc.allreduce([xs[p] for p in perm], dtype, op), ref)


@pytest.mark.parametrize("dtype", synth.DTYPES)
def test_single_rank_identity(dtype):
    x = synth.gen(dtype, 1000, 0, cfg=2, dist="full" if dtype[0] == "i" else "normal")
    for op in orc.OPS:
        np.testing.assert_array_equal(orc.allreduce([x], dtype, op), x)


@pytest.mark.parametrize("dtype", synth.DTYPES)
def test_max_min_idempotent(dtype):
    x = synth.gen(dtype, 500, 0, cfg=4, dist="full" if dtype[0] == "i" else "normal")
    for op in ("max", "min"):
        np.testing.assert_array_equal(orc.allreduce([x] * 5, dtype, op), x)


def test_rejects_bad_args():
    with pytest.raises(ValueError):
        orc.allreduce([], "f32", "sum")
    with pytest.raises(ValueError):
        orc.allreduce([np.zeros(3, np.float32)], "f32", "prod")
    with pytest.raises(ValueError):
        orc.allreduce([np.zeros(3, np.float32), np.zeros(2, np.float32)], "f32", "sum")


def test_window_matches_full():
    xs = synth.gen_ranks("bf16", 5000, 4, cfg=9, dist="normal")
    full = orc.allreduce(xs, "bf16", "sum")
    w = orc.allreduce_window(lambda r: xs[r], 4, 5000, "bf16", "sum", 1234, 2345)
    np.testing.assert_array_equal(w, full[1234:2345])
    assert math.isfinite(float(orc.bf16_bits_to_f32(full).max()))
