"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element
(virtual ranks on one B200).  Every algorithm x
protocol x dtype x op, sizes spanning several tiles/chunks and ragged tails,
edge cases (count 0/1, count < nranks, unaligned buffers, back-to-back calls
alternating algorithms without a host sync), and the policy-selected path whose
recorded decision must equal the oracle's decision mapping.
"""
import itertools

import numpy as np
import pytest

import synth
from oracle import policy as OP
from tests.gpu_common import check_result, default_dist, to_device, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_11438_b200 import polar as L  # noqa: E402

ALGOS = ["oneshot", "twoshot", "ring", "tree"]
PROTOS = ["ll", "ll128", "simple"]
_COMMS = {}


def comm(n):
    """Cached virtual comm; a comm with a latched error is unusable by design
    (polar.h), so it is replaced rather than letting one failure cascade."""
    c = _COMMS.get(n)
    if c is not None:
        try:
            c.check()
        except L.PolarError:
            c = None
    if c is None:
        torch.cuda.synchronize()
        c = _COMMS[n] = L.Comm.virtual(n, 0)
    return c


def run(n, dtype, op, count, algo, proto, nch, dist=None, cfg=1, offset=0):
    xs = synth.gen_ranks(dtype, count, n, cfg=cfg, dist=dist or default_dist(dtype))
    ts = [to_device(x, dtype, offset) for x in xs]
    c = comm(n)
    c.allreduce_forced(ts, algo, proto, nch, op=op)
    torch.cuda.synchronize()
    c.check()
    got = [to_host(t, dtype) for t in ts]
    check_result(got, xs, dtype, op, algo, n)
    d = c.last_decision()
    assert (L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto]) == (algo, proto)


@pytest.mark.parametrize("algo,proto", list(itertools.product(ALGOS, PROTOS)))
@pytest.mark.parametrize("dtype", synth.DTYPES)
def test_matrix_sum(algo, proto, dtype):
    for n in (2, 3, 4, 8):
        for count, nch in ((1, 1), (7, 2), (1000, 3), (40_003, 4), (300_001, 8)):
            run(n, dtype, "sum", count, algo, proto, nch)


@pytest.mark.parametrize("algo,proto", list(itertools.product(ALGOS, PROTOS)))
@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("dtype", synth.DTYPES)
def test_matrix_max_min(algo, proto, op, dtype):
    for n, count, nch in ((4, 12_345, 3), (8, 999, 1)):
        run(n, dtype, op, count, algo, proto, nch)


@pytest.mark.parametrize("algo,proto", list(itertools.product(ALGOS, PROTOS)))
def test_exact_integer_valued_floats(algo, proto):
    """Integer-valued inputs: every algorithm must match bit for bit."""
    for dtype in ("f32", "bf16"):
        xs = synth.gen_ranks(dtype, 77_777, 8, cfg=4, dist="ints")
        ts = [to_device(x, dtype) for x in xs]
        c = comm(8)
        c.allreduce_forced(ts, algo, proto, 5)
        torch.cuda.synchronize()
        from oracle import allreduce as orc
        exp = orc.allreduce(xs, dtype, "sum")
        for t in ts:
            assert np.array_equal(to_host(t, dtype), exp)


@pytest.mark.parametrize("algo,proto", list(itertools.product(ALGOS, PROTOS)))
def test_edges(algo, proto):
    for n in (2, 8):
        run(n, "f32", "sum", 0, algo, proto, 1)           # no-op
        run(n, "f32", "sum", 1, algo, proto, 32)          # count < nranks, more channels than packs
        run(n, "i32", "sum", n - 1, algo, proto, 2)
        run(n, "bf16", "sum", 9, algo, proto, 3)          # one full pack + 1
        run(n, "i64", "sum", 4097, algo, proto, 7, offset=1)    # unaligned buffers
        run(n, "bf16", "sum", 5000, algo, proto, 2, offset=3)


@pytest.mark.parametrize("algo,proto", list(itertools.product(ALGOS, PROTOS)))
def test_multi_chunk(algo, proto):
    """Sizes beyond one staging chunk / FIFO loop chunk, max channels."""
    run(8, "f32", "sum", (3 << 20) + 17, algo, proto, 32)
    run(2, "bf16", "sum", (5 << 20) + 3, algo, proto, 16)


def test_back_to_back_alternating_no_sync():
    """Consecutive calls of different algorithms/protocols/channel counts on one
    stream, without host synchronisation (epochs, FIFO counters, parities)."""
    n, dtype = 8, "f32"
    c = comm(n)
    rng = np.random.default_rng(11)
    combos = list(itertools.product(ALGOS, PROTOS))
    xs_list, ts_list = [], []
    for it in range(24):
        algo, proto = combos[rng.integers(len(combos))]
        count = int(rng.integers(1, 200_000))
        xs = synth.gen_ranks(dtype, count, n, cfg=100 + it, dist="ints")
        ts = [to_device(x, dtype) for x in xs]
        c.allreduce_forced(ts, algo, proto, int(rng.integers(1, 33)))
        xs_list.append((xs, algo))
        ts_list.append(ts)
    torch.cuda.synchronize()
    c.check()
    for (xs, algo), ts in zip(xs_list, ts_list):
        check_result([to_host(t, dtype) for t in ts], xs, dtype, "sum", algo, n)


@pytest.mark.parametrize("algo", ["tree", "ring"])
def test_simple_fifo_unit_sizes_back_to_back(algo, monkeypatch):
    """Warp-specialised ring/tree Simple (kernels.cuh ring_simple_ws /
    tree_simple_ws): back-to-back calls whose channels hold 1 tiny slot, a few
    slots (tree: half-slot units) and many slots (tree: whole-slot units) on one
    stream without host sync, mixed with LL calls that advance the same FIFO
    counters: the half-slot tail encoding must keep every wait exact.  On a
    POLAR_CLUSTER=0 comm: the FIFO kernels for every size."""
    n, dtype = 8, "f32"
    monkeypatch.setenv("POLAR_CLUSTER", "0")
    c = L.Comm.virtual(n, 0)
    plan = [(1000, "simple", 4), ((1 << 20) // 4, "simple", 18), ((24 << 20) // 4, "simple", 18),
            (777, "ll", 4), ((3 << 20) // 4 + 5, "simple", 8), (5, "simple", 2), ((40 << 20) // 4, "simple", 32),
            ((1 << 20) // 4, "ll128", 18), ((2 << 20) // 4, "simple", 18)]
    pending = []
    for it, (count, proto, nch) in enumerate(plan * 2):
        xs = synth.gen_ranks(dtype, count, n, cfg=300 + it, dist="ints")
        ts = [to_device(x, dtype) for x in xs]
        c.allreduce_forced(ts, algo, proto, nch)
        pending.append((xs, ts))
    torch.cuda.synchronize()
    c.check()
    for xs, ts in pending:
        check_result([to_host(t, dtype) for t in ts], xs, dtype, "sum", algo, n)
    c.destroy()


def test_policy_selected_decision_matches_oracle():
    """polar_allreduce (policy-selected): recorded decision == oracle mapping."""
    rows = [(0, 0, 16 << 10, OP.ONESHOT, OP.LL, 2), (0, 0, 256 << 10, OP.TWOSHOT, OP.LL, 4),
            (0, 8, 2 << 20, OP.RING, OP.SIMPLE, 6), (0, 0, 4 << 20, OP.TREE, OP.UNSET, 0)]
    L.set_policy(rows)
    try:
        for n in (2, 8):
            c = comm(n)
            for count in (2, 4096, 65_536, 300_000, 1 << 20, 3 << 20):
                xs = synth.gen_ranks("f32", count, n, cfg=7, dist="ints")
                ts = [to_device(x, "f32") for x in xs]
                c.allreduce(ts)
                torch.cuda.synchronize()
                d = c.last_decision()
                exp = OP.decide(rows, 0, n, count * 4)
                assert d.as_tuple() == exp
                from oracle import allreduce as orc
                ref = orc.allreduce(xs, "f32", "sum")
                for t in ts:
                    assert np.array_equal(to_host(t, "f32"), ref)
    finally:
        L.set_policy([])


def test_default_policy_bench_size_sampled():
    """Full bench size (C2: 8 ranks x 128 MiB f32, the launch config bench.py
    times): sampled windows checked against the oracle one by one."""
    from oracle import allreduce as orc
    n, count = 8, 32 << 20
    xs = synth.gen_ranks("f32", count, n, cfg=2, dist="unif")
    c = comm(n)
    ts = [to_device(x, "f32") for x in xs]
    c.allreduce(ts)
    torch.cuda.synchronize()
    c.check()
    rng = np.random.default_rng(5)
    windows = [(0, 4096), (count - 4099, count)] + [(int(s), int(s) + 2048) for s in rng.integers(0, count - 2048, 16)]
    for lo, hi in windows:
        exp = orc.allreduce([x[lo:hi] for x in xs], "f32", "sum")
        for t in ts:
            got = to_host(t[lo:hi], "f32")
            assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), (lo, hi)


@pytest.mark.parametrize("n", [2, 3, 8])
def test_twoshot_tma_forced(n, monkeypatch):
    """The TMA-staged two-shot (cp.async.bulk + mbarrier pipeline), forced on a
    dedicated comm: every dtype/op, ragged sizes spanning many tiles and chunks,
    the partial last pack, and an unaligned buffer (falls back to the LDG path)."""
    monkeypatch.setenv("POLAR_TWOSHOT_TMA", "1")
    c = L.Comm.virtual(n, 0)
    try:
        for dtype in synth.DTYPES:
            for op in ("sum", "max"):
                for count, nch, off in ((1, 1, 0), (4097, 3, 0), (300_001, 8, 0), (1_234_567, 32, 0), (5000, 2, 1)):
                    xs = synth.gen_ranks(dtype, count, n, cfg=12, dist=default_dist(dtype))
                    ts = [to_device(x, dtype, off) for x in xs]
                    c.allreduce_forced(ts, "twoshot", "simple", nch, op=op)
                    torch.cuda.synchronize()
                    c.check()
                    check_result([to_host(t, dtype) for t in ts], xs, dtype, op, "twoshot", n)
    finally:
        c.destroy()


def test_twoshot_tma_auto_large_n2():
    """Auto selection takes the TMA path for n = 2 and >= 64 MiB: sampled parity."""
    from oracle import allreduce as orc
    n, count = 2, (96 << 20) // 4 + 5
    xs = synth.gen_ranks("f32", count, n, cfg=13, dist="unif")
    c = comm(n)
    ts = [to_device(x, "f32") for x in xs]
    c.allreduce_forced(ts, "twoshot", "simple", 32)
    torch.cuda.synchronize()
    c.check()
    for lo, hi in ((0, 8192), (count // 2, count // 2 + 8192), (count - 9000, count)):
        exp = orc.allreduce([x[lo:hi] for x in xs], "f32", "sum")
        for t in ts:
            assert np.array_equal(to_host(t[lo:hi], "f32").view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("algo", ALGOS)
def test_ll128_stress_back_to_back(algo):
    """LL128 relies on a warp's 128-B line store landing as one unit (device.cuh
    "LL128"): many back-to-back calls of one size, no host sync in between,
    integer-valued inputs so every algorithm must be bit-exact; a torn line
    (flag seen before its data) would show up as a wrong element."""
    from oracle import allreduce as orc
    n, dtype, count = 8, "f32", 1_000_003
    c = comm(n)
    cases = []
    for it in range(12):
        xs = synth.gen_ranks(dtype, count, n, cfg=300 + it, dist="ints")
        ts = [to_device(x, dtype) for x in xs]
        c.allreduce_forced(ts, algo, "ll128", 1 + (it * 5) % 32)
        cases.append((xs, ts))
    torch.cuda.synchronize()
    c.check()
    for xs, ts in cases:
        exp = orc.allreduce(xs, dtype, "sum")
        for t in ts:
            assert np.array_equal(to_host(t, dtype), exp)


def test_paper_policy_nvlink_ring_mid_v2():
    """The paper's case-study policy as a table: Ring/LL128 at
    4-32 MiB, Ring/Simple at 64-192 MiB, default otherwise; 8 ranks, f32 sum."""
    from oracle import allreduce as orc
    from tests.golden_io import rows_and_cases
    rows, _, _ = rows_and_cases("nvlink_ring_mid_v2.txt")
    L.set_policy(rows)
    try:
        n = 8
        c = comm(n)
        for nbytes in (2 << 20, 4 << 20, 8 << 20, 32 << 20, 48 << 20, 64 << 20):
            count = nbytes // 4
            xs = synth.gen_ranks("f32", count, n, cfg=21, dist="ints")
            ts = [to_device(x, "f32") for x in xs]
            c.allreduce(ts)
            torch.cuda.synchronize()
            c.check()
            assert c.last_decision().as_tuple() == OP.decide(rows, 0, n, nbytes)
            exp = orc.allreduce(xs, "f32", "sum")
            for t in ts:
                assert np.array_equal(to_host(t, "f32"), exp)
    finally:
        L.set_policy([])


@pytest.mark.parametrize("chunk", ["65536", "8388608"])
def test_allreduce_host_chunk_pipeline(chunk, monkeypatch):
    """polar_allreduce_host (the e2e path): host buffers in, host buffers out,
    processed as overlapping chunks; ragged counts spanning many chunks, pinned
    and pageable host memory, and the policy-selected kernels per chunk."""
    from oracle import allreduce as orc
    monkeypatch.setenv("POLAR_HOST_CHUNK", chunk)
    for n, dtype, count in ((8, "f32", 3_000_017), (3, "bf16", 1_000_001), (2, "i64", 70_001)):
        xs = synth.gen_ranks(dtype, count, n, cfg=41, dist=default_dist(dtype))
        c = comm(n)
        for pinned in (True, False):
            host = [torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16) if dtype == "bf16"
                    else torch.from_numpy(x.copy()) for x in xs]
            if pinned:
                host = [h.pin_memory() for h in host]
            dev = [torch.empty_like(h, device="cuda") for h in host]
            c.allreduce_host(host, dev)
            c.check()
            exp = orc.allreduce(xs, dtype, "sum")
            for h in host:
                got = h.view(torch.int16).numpy() if dtype == "bf16" else h.numpy()
                assert np.array_equal(got.view(np.uint8), exp.view(np.uint8))


@pytest.mark.parametrize("algo,proto", [("twoshot", "simple"), ("ring", "simple"), ("twoshot", "ll128")])
def test_beyond_2pow31_elements(algo, proto):
    """Maximum sizes: 2^31 + 1003 f32 elements per rank (8 GiB, the paper's largest
    Table-2 size) — every index past 2^31 must be 64-bit.  Inputs are a
    formula evaluated on the device; sampled windows (including the ragged end)
    are checked against the oracle on the same formula evaluated on the host."""
    from oracle import allreduce as orc
    n, count = 2, (1 << 31) + 1003

    def host(r, lo, hi):
        i = np.arange(lo, hi, dtype=np.int64)
        return (((i * 2654435761 + 977 * r) % 1021) - 510).astype(np.float32)

    ts = []
    for r in range(n):
        t = torch.empty(count, dtype=torch.float32, device="cuda")
        step = 1 << 28
        for lo in range(0, count, step):
            hi = min(count, lo + step)
            i = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
            t[lo:hi] = (((i * 2654435761 + 977 * r) % 1021) - 510).to(torch.float32)
            del i
        ts.append(t)
    c = comm(n)
    try:
        c.allreduce_forced(ts, algo, proto, 32)
        torch.cuda.synchronize()
        c.check()
        for lo, hi in ((0, 4096), ((1 << 31) - 2048, (1 << 31) + 1000), (count - 5000, count), (1 << 30, (1 << 30) + 999)):
            exp = orc.allreduce([host(r, lo, hi) for r in range(n)], "f32", "sum")
            for t in ts:
                assert np.array_equal(t[lo:hi].cpu().numpy(), exp), (lo, hi)
    finally:
        del ts
        torch.cuda.empty_cache()


def test_single_rank_is_identity_without_launch():
    """n = 1 (SURVEY.md §8(c) reading 10): every call is an in-place identity,
    decided (the decision is recorded) but not launched."""
    c = L.Comm.virtual(1, 0)
    try:
        x = torch.arange(1000, dtype=torch.float32, device="cuda")
        before = c.launches()
        c.allreduce([x])
        assert c.last_decision().as_tuple() == OP.decide([], 0, 1, 4000)
        for algo in ALGOS:
            for proto in PROTOS:
                c.allreduce_forced([x], algo, proto, 4)
        torch.cuda.synchronize()
        c.check()
        assert c.launches() == before
        assert torch.equal(x, torch.arange(1000, dtype=torch.float32, device="cuda"))
    finally:
        c.destroy()


@pytest.mark.parametrize("case", ["policy", "ring/simple", "tree/simple", "twoshot/ll128", "ring/ll128"])
def test_c3_bf16_1gib_n4_sampled(case):
    """BASELINE config 3 at its largest size: bf16 sum, 1 GiB per rank (512 Mi
    elements), n = 4.  Inputs N(0,1) rounded to bf16 (the C3
    tolerance distribution), drawn on the device from a seeded generator; the
    sampled windows of every rank's input are kept on the host BEFORE the call,
    and the results there are compared with the oracle: one-/two-shot bit-exact,
    ring / tree within 1e-2 * |y*| (R3; f32 partials make them exact in practice)
    and every rank bitwise identical.  `policy` = the default table's decision
    for 1 GiB (two-shot Simple, TMA-staged at n <= 4)."""
    from oracle import allreduce as orc
    n, count = 4, (1 << 30) // 2
    rng = np.random.default_rng(3)
    windows = [(0, 8192), (count - 8195, count), ((1 << 28) - 3000, (1 << 28) + 3000)] + \
        [(int(s), int(s) + 4096) for s in rng.integers(0, count - 4096, 8)]
    ts, win = [], []
    for r in range(n):
        g = torch.Generator(device="cuda")
        g.manual_seed(2603_03 * 10 + r)
        t = torch.randn(count, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16)
        win.append([to_host(t[lo:hi], "bf16") for lo, hi in windows])
        ts.append(t)
    c = comm(n)
    try:
        if case == "policy":
            c.allreduce(ts)
            algo = L.ALGO_NAMES[c.last_decision().algo]
            assert c.last_decision().as_tuple() == OP.decide([], 0, n, count * 2)
        else:
            algo, proto = case.split("/")
            c.allreduce_forced(ts, algo, proto, 32)
        torch.cuda.synchronize()
        c.check()
        for k, (lo, hi) in enumerate(windows):
            got = [to_host(t[lo:hi], "bf16") for t in ts]
            check_result(got, [win[r][k] for r in range(n)], "bf16", "sum", algo, n)
    finally:
        del ts
        torch.cuda.empty_cache()


@pytest.mark.parametrize("flags", ["0", "1", "3"])
def test_ring_tma_forced(flags, monkeypatch):
    """The TMA-staged ring Simple (kernels.cuh ring_simple_tma; opt-in with
    POLAR_RING_TMA=1): every dtype / op, several laps and tiles, bf16 f32
    partials through the FIFO, ragged (non-TMA-eligible) counts falling back to
    the LDG ring on the same FIFOs, back to back without host sync.  flags: bit 0
    L2 eviction hints, bit 1 discard of consumed FIFO lines."""
    monkeypatch.setenv("POLAR_RING_TMA", "1")
    monkeypatch.setenv("POLAR_RING_TMA_FLAGS", flags)
    monkeypatch.setenv("POLAR_CLUSTER", "0")   # the FIFO kernels (aligned sizes would run as clusters)
    for n in (2, 3, 8):
        c = L.Comm.virtual(n, 0)
        try:
            pending = []
            for dtype in synth.DTYPES:
                for op in ("sum", "max"):
                    for count, nch in ((4096, 1), (3 << 20, 8), (1_000_003, 5), (777_216, 32)):
                        xs = synth.gen_ranks(dtype, count, n, cfg=14, dist=default_dist(dtype))
                        ts = [to_device(x, dtype) for x in xs]
                        c.allreduce_forced(ts, "ring", "simple", nch, op=op)
                        pending.append((xs, ts, dtype, op))
                torch.cuda.synchronize()
                c.check()
                for xs, ts, dt, op in pending:
                    check_result([to_host(t, dt) for t in ts], xs, dt, op, "ring", n)
                pending = []
        finally:
            c.destroy()
