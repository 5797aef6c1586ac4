"""Pins for oracle/collectives.py (CPU): pure-Python brute force on tiny inputs,
closed forms, and the identity ReduceScatter blocks == AllReduce slices for the
order-free integer ops (checked against the brute force, not the oracle)."""
import numpy as np
import pytest

import synth
from oracle import collectives as OC


def brute_rs_int(xs, bits, op):
    n, c = len(xs), len(xs[0]) // len(xs)
    mask = (1 << bits) - 1
    out = []
    for r in range(n):
        blk = []
        for i in range(c):
            vals = [int(x[r * c + i]) for x in xs]
            if op == "sum":
                acc = 0
                for v in vals:
                    acc = (acc + (v & mask)) & mask
                if acc >= 1 << (bits - 1):
                    acc -= 1 << bits
            else:
                acc = max(vals) if op == "max" else min(vals)
            blk.append(acc)
        out.append(blk)
    return out


@pytest.mark.parametrize("op", ["sum", "max", "min"])
@pytest.mark.parametrize("dtype,bits", [("i32", 32), ("i64", 64)])
def test_reduce_scatter_brute_force(dtype, bits, op):
    for n in range(1, 9):
        for c in (0, 1, 3, 10):
            xs = synth.gen_ranks(dtype, n * c, n, cfg=60, dist="full")
            got = OC.reduce_scatter(xs, dtype, op)
            assert [[int(v) for v in g] for g in got] == brute_rs_int(xs, bits, op)


def test_reduce_scatter_closed_form():
    n, c = 4, 256
    i = np.arange(n * c, dtype=np.int64)
    xs = [((r + 1) * (i + 1)).astype(np.int32) for r in range(n)]
    got = OC.reduce_scatter(xs, "i32", "sum")
    for r in range(n):
        np.testing.assert_array_equal(got[r].astype(np.int64), (i[r * c:(r + 1) * c] + 1) * n * (n + 1) // 2)


def test_all_gather_brute_force():
    for n in range(1, 9):
        for c in (0, 1, 7):
            xs = synth.gen_ranks("bf16", c, n, cfg=61, dist="normal")
            got = OC.all_gather(xs)
            exp = [int(v) for x in xs for v in x]
            assert [int(v) for v in got] == exp
            assert got.dtype == np.uint16 or c == 0


def test_broadcast_identity():
    xs = synth.gen_ranks("f32", 100, 5, cfg=62, dist="unif")
    for root in range(5):
        np.testing.assert_array_equal(OC.broadcast(xs, root), xs[root])
    with pytest.raises(ValueError):
        OC.broadcast(xs, 5)


def test_reduce_scatter_rejects_ragged():
    with pytest.raises(ValueError):
        OC.reduce_scatter([np.zeros(5, np.int32), np.zeros(5, np.int32)], "i32", "sum")
