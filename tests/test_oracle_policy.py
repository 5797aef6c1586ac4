"""Pins for oracle/policy.py and oracle/metrics.py (CPU only).

The decision mapping is pinned to the paper's worked examples (Listing 1,
nvlink_ring_mid_v2, bad_channels) and SPEC.md's invoke_tuner examples, stored
as cited fixtures in tests/golden/; the metric arithmetic to PAPER.md's
"~394 us" for 128 MiB at Table 2's 596.9 GB/s.
"""
import pytest

from oracle import metrics, policy as P
from tests.golden_io import blocks, rows_and_cases, table

MiB = 1 << 20


def test_listing1_threshold_cases():
    rows, cases, _ = rows_and_cases("listing1_size_aware.txt")
    assert P.validate(rows) == "ok"
    for nranks, nbytes, algo, proto, nch in cases:
        assert P.decide(rows, P.COLL_ALLREDUCE, nranks, nbytes) == (algo, proto, nch)


def test_nvlink_ring_mid_v2_cases():
    rows, cases, status = rows_and_cases("nvlink_ring_mid_v2.txt")
    assert P.validate(rows) == status == "ok"
    for case in cases:
        nranks, nbytes = case[0], case[1]
        got = P.decide(rows, P.COLL_ALLREDUCE, nranks, nbytes)
        dflt = P.decide([], P.COLL_ALLREDUCE, nranks, nbytes)
        if case[2] == "default":
            assert got == dflt
        else:
            assert got[:2] == (case[2], case[3])
            assert got[2] == dflt[2]          # channels deferred (row nch = 0)


def test_spec_invoke_tuner_blocks():
    for name, (rows, cases) in blocks("spec_invoke_tuner.txt").items():
        assert P.validate(rows) == "ok", name
        for nranks, nbytes, nch in cases:
            got = P.decide(rows, P.COLL_ALLREDUCE, nranks, nbytes)
            if nch == "default":
                assert got[2] == P.decide([], P.COLL_ALLREDUCE, nranks, nbytes)[2]
            else:
                assert got[2] == nch, name


def test_noop_equivalence_sweep():
    """with noop (empty table) every decision is the default."""
    for n in range(1, 9):
        for k in range(0, 41):
            for d in (-1, 0, 1):
                b = max(0, (1 << k) + d)
                assert P.decide([], 0, n, b) == P.decide([(0, 0, P.U64_MAX, P.UNSET, P.UNSET, 0)], 0, n, b)


def test_default_table_is_total_and_clamped():
    for n in range(1, 9):
        for k in range(0, 64):
            a, p, c = P.decide([], 0, n, 1 << k)
            assert a in (P.TREE, P.RING, P.ONESHOT, P.TWOSHOT)
            assert p in (P.LL, P.SIMPLE)
            assert 1 <= c <= P.MAXCH
    assert P.decide([], 7, 8, 1024) is None               # no default row for an unknown collective
    assert P.decide([], P.COLL_ALLGATHER, 8, 1024) == (P.ONESHOT, P.SIMPLE, 32)


def test_first_match_and_nranks_filter():
    rows = [(0, 2, 1000, P.RING, P.LL, 3), (0, 0, 1000, P.TREE, P.SIMPLE, 5)]
    assert P.decide(rows, 0, 2, 1000) == (P.RING, P.LL, 3)
    assert P.decide(rows, 0, 4, 1000) == (P.TREE, P.SIMPLE, 5)
    assert P.decide(rows, 0, 4, 1001) == P.decide([], 0, 4, 1001)


def test_validation_rules():
    ok = (0, 0, 100, P.RING, P.SIMPLE, 4)
    assert P.validate([ok]) == "ok"
    assert P.validate([]) == "ok"
    assert P.validate([ok] * 1 + [(0, 0, 200, P.TREE, P.LL, 0)]) == "ok"
    assert P.validate([ok, ok]) == "einval"                       # not ascending
    assert P.validate([(0, 0, 100, 9, P.SIMPLE, 4)]) == "einval"  # unknown algo
    assert P.validate([(0, 0, 100, P.RING, 7, 4)]) == "einval"    # unknown proto
    assert P.validate([(9, 0, 100, P.RING, P.LL, 4)]) == "einval" # unknown coll
    assert P.validate([(0, 9, 100, P.RING, P.LL, 4)]) == "einval" # nranks > 8
    assert P.validate([(0, 0, 100, P.NVLS, P.SIMPLE, 4)]) == "eunsupported"
    assert P.validate([(0, 0, 100, P.RING, P.LL128, 4)]) == "ok"            # LL128 built (f2)
    assert P.validate([(0, 0, 100, P.NVLS, P.SIMPLE, 4), ok]) == "einval"
    assert P.validate([(0, 0, i, P.RING, P.LL, 1) for i in range(65)]) == "einval"
    assert P.validate([(0, 0, i, P.RING, P.LL, 1) for i in range(64)]) == "ok"
    # different (coll, nranks) groups are ordered independently
    assert P.validate([(0, 8, 100, P.RING, P.LL, 1), (0, 0, 50, P.RING, P.LL, 1)]) == "ok"


# ----------------------------------------------------------------- metrics


def test_busbw_394us_pin():
    rows = table("table2_busbw.txt")
    size, default_bw = int(rows[5][0]), rows[5][1]
    assert size == 128 * MiB
    t = metrics.latency_from_busbw(size, 8, default_bw)
    assert t == pytest.approx(394e-6, rel=0.01)        # PAPER.md L447-448 "~394 us"
    assert metrics.busbw_gbs(size, 8, t) == pytest.approx(default_bw)


def test_table2_deltas_reproduce():
    for size, dflt, ring, delta in table("table2_busbw.txt"):
        assert 100.0 * (ring / dflt - 1.0) == pytest.approx(delta, abs=0.06)


def test_busbytes_convention():
    assert metrics.busbytes_allreduce(800, 8) == 1400.0
    assert metrics.busbytes_allreduce(800, 2) == 800.0
    assert metrics.busbytes_allreduce(800, 1) == 0.0
    assert metrics.algbw_gbs(10**9, 1.0) == 1.0
