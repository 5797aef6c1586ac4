"""Generative cases (hypothesis): random policy tables —
valid and malformed — through the C ABI's set_policy/decide against the oracle's
validation and linear-scan decision, at random and threshold-adjacent sizes."""
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import policy as OP
from paper_2603_11438_b200 import polar as L

ALGOS = [OP.TREE, OP.RING, OP.NVLS, OP.ONESHOT, OP.TWOSHOT, OP.UNSET, 7]
PROTOS = [OP.LL, OP.LL128, OP.SIMPLE, OP.UNSET, 4]
COLLS = [OP.COLL_ALLREDUCE, OP.COLL_ALLGATHER, OP.COLL_BROADCAST, OP.COLL_REDUCESCATTER]

row = st.tuples(st.sampled_from(COLLS + [9]), st.sampled_from([0, 0, 1, 2, 4, 8, 9]),
                st.one_of(st.integers(0, 1 << 30), st.sampled_from([2**64 - 1, (1 << 40) + 3])),
                st.sampled_from(ALGOS), st.sampled_from(PROTOS),
                st.sampled_from([0, 1, 2, 4, 16, 32, 33, 64, 2**31, 2**32 - 1]))


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(rows=st.lists(row, max_size=12), sizes=st.lists(st.integers(0, 1 << 41), min_size=1, max_size=20),
       sorted_rows=st.booleans())
def test_random_tables(rows, sizes, sorted_rows):
    if sorted_rows:   # make most tables valid: ascending max_bytes within each (coll, nranks) group
        rows = sorted(rows, key=lambda r: r[2])
    exp = OP.validate(rows)
    g0 = L.generation()
    st_, gen = L.set_policy_status(rows)
    assert L.STATUS_NAMES[st_] == exp
    active = rows if exp == "ok" else None
    if exp == "ok":
        assert gen == g0 + 1
    else:
        assert L.generation() == g0
    if active is None:
        active, _ = L.get_policy()
    probes = set(sizes)
    for r in active:
        for d in (-1, 0, 1):
            if 0 <= r[2] + d < 2**64:
                probes.add(r[2] + d)
    ctxs = [(n, b) for n in (1, 2, 3, 8) for b in sorted(probes)]
    for (n, b), g in zip(ctxs, L.decide_batch(ctxs)):
        assert g[:3] == OP.decide(active, OP.COLL_ALLREDUCE, n, b), (n, b)
    L.set_policy([])
