"""scripts/tune_policy.py's table construction (CPU): per-size winners merged
into first-match rows that reproduce every winner under polar_decide and the
oracle, and the best single global choice (E10)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import tune_policy as T  # noqa: E402
from oracle import policy as OP  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402

CODES = (L.ALGO_CODES, L.PROTO_CODES)


def test_merge_rows_reproduces_winners():
    sizes = [8, 64, 4096, 65536, 1 << 20, 4 << 20, 32 << 20, 128 << 20]
    winners = ["oneshot/ll/2", "oneshot/ll/2", "oneshot/ll/4", "twoshot/ll128/8", "twoshot/simple/16",
               "ring/ll128/32", "ring/ll128/32", "twoshot/simple/32"]
    best = {}
    for s, w in zip(sizes, winners):
        a, p, c = w.split("/")
        best[s] = (1e-6, a, p, int(c))
    rows = T.merge_rows(best, sizes, 8, CODES)
    assert rows[-1][2] == T.U64_MAX and len(rows) == 6          # runs of equal winners share a row
    assert L.STATUS_NAMES[L.set_policy_status(rows)[0]] == OP.validate(rows) == "ok"
    try:
        for s, w in zip(sizes, winners):
            a, p, c = w.split("/")
            exp = (L.ALGO_CODES[a], L.PROTO_CODES[p], int(c))
            assert L.decide(8, s).as_tuple() == OP.decide(rows, 0, 8, s) == exp
        # between measured sizes the next larger measured size's winner applies (inclusive bounds)
        assert L.decide(8, 65) .as_tuple() == OP.decide(rows, 0, 8, 4096)
        # other rank counts are untouched (rows carry nranks = 8)
        assert L.decide(4, 8).as_tuple() == OP.decide([], 0, 4, 8)
    finally:
        L.set_policy([])


def test_best_single_global_choice():
    sizes = [1, 2, 3]
    meas = {("a", "x", 1): {1: 1.0, 2: 1.0, 3: 9.0},     # total 11
            ("b", "y", 2): {1: 3.0, 2: 3.0, 3: 3.0},     # total 9  <- best single
            ("c", "z", 4): {1: 0.1, 2: 0.1}}             # not measured at every size
    r = T.best_single(meas, sizes)
    assert r["choice"] == ["b", "y", 2] and r["us"]["3"] == 3e6
    assert T.best_single({}, sizes) is None
