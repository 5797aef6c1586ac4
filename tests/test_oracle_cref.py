"""Pins for the threaded C oracle (oracle/c/allreduce_ref.c): bit-exact against
oracle/allreduce.py (itself pinned by brute force and closed forms) for every
dtype x op, rank counts 1-8, ragged counts and thread counts, plus the closed
forms of SURVEY.md §8(c) directly."""
import numpy as np
import pytest

import synth
from oracle import allreduce as orc
from oracle import cref


@pytest.mark.parametrize("dtype", ["i32", "i64", "f32", "bf16"])
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_matches_numpy_oracle(dtype, op):
    for n in (1, 2, 3, 8):
        for count, threads in ((0, 1), (1, 4), (7, 3), (10_007, 1), (100_003, 8)):
            for dist in ({"i32": "full", "i64": "full", "f32": "logu", "bf16": "normal"}[dtype], "ints"):
                xs = synth.gen_ranks(dtype, count, n, cfg=9, dist=dist)
                exp = orc.allreduce(xs, dtype, op)
                got = cref.allreduce(xs, dtype, op, threads)
                assert np.array_equal(got.view(np.uint8), exp.view(np.uint8)), (n, count, threads, dist)


def test_closed_forms():
    n, count = 2, 1024
    xs = [np.array([(r + 1) * (i + 1) for i in range(count)], dtype=np.int32) for r in range(n)]
    assert np.array_equal(cref.allreduce(xs, "i32", "sum", 3), 3 * np.arange(1, count + 1, dtype=np.int32))
    xs = [np.full(5, 0x7FFFFFFF, dtype=np.int32) for _ in range(2)]
    assert np.all(cref.allreduce(xs, "i32", "sum") == -2)
    xs = [np.full(9, r, dtype=np.int64) for r in range(8)]
    assert np.all(cref.allreduce(xs, "i64", "max", 2) == 7)
    assert np.all(cref.allreduce(xs, "i64", "min", 2) == 0)
    # bf16: 1 + 2^-8 (a tie at bf16 precision) rounds to even (1.0); 1 + 3*2^-8 rounds up to 1 + 2^-6
    one, tiny = np.uint16(0x3F80), np.uint16(0x3B80)   # 1.0 and 2^-8
    assert cref.allreduce([np.array([one]), np.array([tiny])], "bf16", "sum")[0] == 0x3F80
    three_tiny = np.uint16(0x3C40)                     # 3 * 2^-8 = 0.01171875
    assert cref.allreduce([np.array([one]), np.array([three_tiny])], "bf16", "sum")[0] == 0x3F82


def test_rejects_bad_arguments():
    with pytest.raises(ValueError):
        cref.allreduce([np.zeros(3, np.float32)], "f32", "sum", 0)
