"""The C-ABI library on CPU: symbols, the decision hook vs the oracle, set_policy
validation, the zero-loss swap stress and the decision-cost bench (BASELINE
config 5).  No GPU needed: the policy half of libpolar is pure host code.
"""
import random
import re

import pytest

from oracle import policy as OP
from paper_2603_11438_b200 import polar as L
from tests.golden_io import blocks, rows_and_cases

HEADER = "include/polar.h"


@pytest.fixture(autouse=True)
def _reset_policy():
    L.set_policy([])
    yield
    L.set_policy([])


def test_library_exports_every_header_symbol():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, HEADER)).read()
    declared = set(re.findall(r"^\s*(?:polar_status|uint32_t|uint64_t|int|const char\*)\s+(polar_\w+)\s*\(", text, re.M))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L.lib, name), name
    assert set(L.EXPORTED) == declared
    assert "sm_100a" in L.version()


def test_enums_match_oracle_numbering():
    # two independent transcriptions of SPEC.md L306 + DESIGN.md "Action space"
    assert (L.TREE, L.RING, L.NVLS, L.ONESHOT, L.TWOSHOT) == (OP.TREE, OP.RING, OP.NVLS, OP.ONESHOT, OP.TWOSHOT)
    assert (L.LL, L.LL128, L.SIMPLE, L.UNSET, L.MAXCH) == (OP.LL, OP.LL128, OP.SIMPLE, OP.UNSET, OP.MAXCH)


def _sweep_bytes():
    out = set(range(0, 4097))
    for k in range(0, 41):
        for d in (-1, 0, 1):
            out.add(max(0, (1 << k) + d))
    rnd = random.Random(7)
    out.update(rnd.randrange(0, 1 << 40) for _ in range(3000))
    return sorted(out)


def _rows_thresholds(rows):
    s = set()
    for r in rows + OP.DEFAULT_ROWS:
        m = r[2]
        for d in (-1, 0, 1):
            if 0 <= m + d < 2**64:
                s.add(m + d)
    return s


def _compare(rows):
    sizes = sorted(set(_sweep_bytes()) | _rows_thresholds(rows))
    ctxs = [(n, b) for n in range(1, 9) for b in sizes]
    got = L.decide_batch(ctxs)
    for (n, b), g in zip(ctxs, got):
        assert g[:3] == OP.decide(rows, OP.COLL_ALLREDUCE, n, b), (n, b, rows)


def test_default_table_matches_oracle():
    _compare([])


def test_other_collectives_decisions_match_oracle():
    """f4: the same hook decides ReduceScatter / AllGather / Broadcast (ctx.coll)."""
    rows = [(OP.COLL_ALLGATHER, 0, 1 << 20, OP.ONESHOT, OP.SIMPLE, 4),
            (OP.COLL_REDUCESCATTER, 8, 1 << 24, OP.UNSET, OP.UNSET, 7), (0, 0, 100, OP.RING, OP.LL, 2)]
    L.set_policy(rows)
    for coll in (OP.COLL_ALLGATHER, OP.COLL_BROADCAST, OP.COLL_REDUCESCATTER, OP.COLL_ALLREDUCE):
        ctxs = [(n, b) for n in (1, 2, 8) for b in sorted(_rows_thresholds(rows))[:300]]
        for (n, b), g in zip(ctxs, L.decide_batch(ctxs, coll=coll)):
            assert g[:3] == OP.decide(rows, coll, n, b), (coll, n, b)


def test_listing1_matches_oracle():
    rows, cases, _ = rows_and_cases("listing1_size_aware.txt")
    L.set_policy(rows)
    _compare(rows)
    for nranks, nbytes, a, p, c in cases:
        assert L.decide(nranks, nbytes).as_tuple() == (a, p, c)


def test_spec_blocks_match_oracle():
    for name, (rows, _) in blocks("spec_invoke_tuner.txt").items():
        L.set_policy(rows)
        _compare(rows)


def test_nvlink_ring_mid_v2_accepted():
    rows, _, status = rows_and_cases("nvlink_ring_mid_v2.txt")
    g0 = L.generation()
    st, gen = L.set_policy_status(rows)
    assert L.STATUS_NAMES[st] == status == "ok"
    assert gen == g0 + 1
    _compare(rows)


def test_nvls_rejected_and_old_kept():
    rows = [(0, 0, 1 << 20, OP.RING, OP.LL128, 4), (0, 0, 1 << 30, OP.NVLS, OP.SIMPLE, 0)]
    L.set_policy([])
    g0 = L.generation()
    st, _ = L.set_policy_status(rows)
    assert L.STATUS_NAMES[st] == "eunsupported"
    assert L.generation() == g0
    _compare([])


def _random_rows(rnd, valid_bias=0.8):
    n = rnd.randrange(0, 10)
    rows = []
    maxb = 0
    for _ in range(n):
        maxb += rnd.choice([1, 7, 1000, 1 << 20, 1 << 30])
        algo = rnd.choice([OP.TREE, OP.RING, OP.ONESHOT, OP.TWOSHOT, OP.UNSET] + ([OP.NVLS, 9] if rnd.random() > valid_bias else []))
        proto = rnd.choice([OP.LL, OP.SIMPLE, OP.UNSET] + ([OP.LL128, 5] if rnd.random() > valid_bias else []))
        nch = rnd.choice([0, 1, 2, 16, 32, 33, 64, 2**31, 2**32 - 1])
        nr = rnd.choice([0, 0, 0, 2, 4, 8] + ([9] if rnd.random() > valid_bias else []))
        rows.append((0, nr, maxb if rnd.random() < 0.95 else max(0, maxb - 5), algo, proto, nch))
    return rows


def test_random_tables_validation_and_decisions():
    rnd = random.Random(2603)
    for _ in range(300):
        rows = _random_rows(rnd)
        g0 = L.generation()
        st, gen = L.set_policy_status(rows)
        exp = OP.validate(rows)
        assert L.STATUS_NAMES[st] == exp, rows
        if exp == "ok":
            assert gen == g0 + 1
            ctxs = [(n, b) for n in (1, 2, 3, 8) for b in sorted(_rows_thresholds(rows))[:200]]
            for (n, b), g in zip(ctxs, L.decide_batch(ctxs)):
                assert g[:3] == OP.decide(rows, 0, n, b)
                assert g[3] == gen
        else:
            assert L.generation() == g0


def test_get_policy_roundtrip_and_copy_semantics():
    rows = [(0, 0, 100, OP.RING, OP.LL, 3), (0, 8, 5000, OP.TREE, OP.SIMPLE, 0)]
    g = L.set_policy(rows)
    got, gen = L.get_policy()
    assert got == rows and gen == g


def test_decide_argument_errors():
    with pytest.raises(L.PolarError) as e:
        L.decide(0, 10)
    assert e.value.name == "einval"
    with pytest.raises(L.PolarError) as e:
        L.decide(9, 10)
    assert e.value.name == "einval"
    with pytest.raises(L.PolarError) as e:
        L.decide(8, 10, coll=7)
    assert e.value.name == "eunsupported"


def test_swap_stress_zero_loss():
    """SPEC.md L444-446 / PAPER.md L483-487: 4 invokers, 1 reloader, 1000 swaps,
    400,000 calls; every call returns a decision of its own generation's table."""
    a = [(0, 0, 32768, OP.TREE, OP.SIMPLE, 4), (0, 0, 2**64 - 1, OP.RING, OP.SIMPLE, 4)]
    b = [(0, 0, 4 << 20, OP.ONESHOT, OP.LL, 2), (0, 0, 2**64 - 1, OP.TWOSHOT, OP.SIMPLE, 32)]
    s = L.bench_swap(a, b, nthreads=4, calls_per_thread=100_000, nswaps=1000)
    assert s["issued"] == 400_000
    assert s["calls"] == s["issued"]
    assert s["invalid"] == 0
    assert s["nonmonotonic"] == 0
    assert s["swaps"] == 1000
    assert s["rejected"] == 100 and s["rejected_changed"] == 0
    assert s["swap_p50_ns"] > 0


def test_decision_cost_bench_sane():
    ctxs = [(n, 1 << k) for k in range(3, 31) for n in (2, 4, 8)]
    s = L.bench_decide(ctxs, nwarm=10_000, ncalls=100_000)
    assert s["calls"] == 100_000
    assert 0 < s["batched_mean_ns"] < 2000
    assert s["p50_ns"] <= s["p99_ns"]


def test_committed_policy_files_validate():
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pdir = os.path.join(root, "policies")
    for name in sorted(os.listdir(pdir)):
        rows = [tuple(r) for r in json.load(open(os.path.join(pdir, name)))["rows"]]
        exp = OP.validate(rows)
        st, _ = L.set_policy_status(rows)
        assert L.STATUS_NAMES[st] == exp, name
        assert exp == "ok", name
        if exp == "ok":
            _compare(rows)


def test_collective_rows_without_kernel_rejected():
    """ReduceScatter / AllGather / Broadcast have one kernel (the direct step,
    ONESHOT / SIMPLE): a row naming anything else is refused at install time,
    the old table stays, and the oracle agrees."""
    L.set_policy([])
    for coll in (OP.COLL_ALLGATHER, OP.COLL_BROADCAST, OP.COLL_REDUCESCATTER):
        g0 = L.generation()
        for algo, proto in ((OP.RING, OP.SIMPLE), (OP.TWOSHOT, OP.UNSET), (OP.UNSET, OP.LL), (OP.ONESHOT, OP.LL128)):
            rows = [(coll, 0, 1 << 20, algo, proto, 4)]
            st, _ = L.set_policy_status(rows)
            assert L.STATUS_NAMES[st] == OP.validate(rows) == "eunsupported", (coll, algo, proto)
            assert L.generation() == g0
        ok_rows = [(coll, 0, 1 << 20, OP.ONESHOT, OP.UNSET, 4), (coll, 0, 1 << 30, OP.UNSET, OP.SIMPLE, 0)]
        st, _ = L.set_policy_status(ok_rows)
        assert L.STATUS_NAMES[st] == OP.validate(ok_rows) == "ok"
    L.set_policy([])
