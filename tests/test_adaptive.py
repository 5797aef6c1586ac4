"""Profiler -> tuner closed loop on CPU: the controller rule
(R15) in the library vs the oracle transcription, pinned to the
paper's three-phase behaviour (§5.3), and the row flag
plumbing through set_policy / decide."""
import math
import random

import pytest

from oracle import adaptive as OA
from oracle import policy as OP
from paper_2603_11438_b200 import polar as L

PERIOD = 10_000   # calls per window: the paper's 100,000-call ramp = 10 windows


def model(c, base=400e3):
    """Latency (ns) of one call at c channels: decreasing with c (more channels,
    more bandwidth) — the shape of Fig. 3's bad_channels vs default gap."""
    return base * (0.2 + 1.6 / c)


def table(nwin, contended=(), scale=10.0, silent=()):
    out = []
    for w in range(nwin):
        if w in silent:
            out.append([math.nan] * 33)
            continue
        k = scale if w in contended else 1.0
        out.append([0.0] + [model(c) * k for c in range(1, 33)])
    return out


def test_three_phase_matches_paper():
    """Ramp 2 -> 12 within 100k calls, back off to <= 3 under a 10x spike,
    ramp back to 12 within 100k calls after recovery."""
    contention = set(range(10, 20))
    lat = table(30, contended=contention)
    p = L.adaptive_params(enabled=True, period=PERIOD, c_min=2, contention_factor=4.0)
    tr = L.adaptive_simulate(p, 12, lat)
    assert tr == OA.simulate(12, lat)
    assert tr[9] == 12 and all(a <= b for a, b in zip(tr[:10], tr[1:10]))       # baseline ramp
    assert (10 + 1) * PERIOD <= 110_000 and tr[9] == 12                           # within 100k calls
    assert all(c <= 3 for c in tr[10:20])                                          # contention
    assert tr[29] == 12 and max(tr[20:30]) == 12                                   # recovery
    assert tr.index(12, 20) - 19 <= 10                                             # within 100k calls


def test_without_profiler_stays_at_two():
    """"Without the profiler, the tuner receives no samples and remains at 2
    channels": windows without samples change nothing."""
    lat = table(40, silent=set(range(40)))
    p = L.adaptive_params(enabled=False, period=PERIOD)
    tr = L.adaptive_simulate(p, 12, lat)
    assert tr == [2] * 40 == OA.simulate(12, lat)


@pytest.mark.parametrize("seed", range(40))
def test_random_tables_match_oracle(seed):
    rnd = random.Random(seed)
    nwin = rnd.randrange(1, 60)
    cap = rnd.randrange(1, 33)
    c_min = rnd.randrange(1, 9)
    factor = rnd.choice([1.5, 2.0, 4.0, 8.0])
    scale = rnd.choice([1.0, 0.5, 3.0])
    lat = []
    for _ in range(nwin):
        if rnd.random() < 0.1:
            lat.append([math.nan] * 33)
        else:
            k = rnd.choice([1.0, 1.0, 1.0, 10.0, 0.3])
            lat.append([0.0] + [model(c) * k * rnd.uniform(0.9, 1.1) for c in range(1, 33)])
    p = L.adaptive_params(enabled=True, period=100, c_min=c_min, contention_factor=factor, latency_scale=scale)
    assert L.adaptive_simulate(p, cap, lat) == OA.simulate(cap, lat, c_min=c_min, factor=factor, scale=scale)


def test_param_validation():
    lat = table(2)
    for bad in (dict(period=0), dict(c_min=0), dict(c_min=33), dict(contention_factor=1.0),
                dict(latency_scale=0.0)):
        with pytest.raises(L.PolarError) as e:
            L.adaptive_simulate(L.adaptive_params(**bad), 12, lat)
        assert e.value.name == "einval"


def test_row_flag_validation_and_decision():
    L.set_policy([])
    try:
        rows = [(0, 0, 1 << 20, OP.ONESHOT, OP.LL, 4), (0, 0, 2**64 - 1, OP.TWOSHOT, OP.SIMPLE, 12, OP.ROW_ADAPTIVE_NCH)]
        assert OP.validate(rows) == "ok"
        L.set_policy(rows)
        got = L.decide_batch([(8, 4 << 20), (8, 1024)])
        assert got[0][:3] == OP.decide(rows, 0, 8, 4 << 20) and got[0][4] == OP.decide_full(rows, 0, 8, 4 << 20)[3] == 1
        assert got[1][4] == 0
        bad = [(0, 0, 100, OP.RING, OP.LL, 4, 0x2)]
        assert OP.validate(bad) == "einval"
        st, _ = L.set_policy_status(bad)
        assert L.STATUS_NAMES[st] == "einval"
        assert L.get_policy()[0] == [rows[0], rows[1]]
    finally:
        L.set_policy([])
