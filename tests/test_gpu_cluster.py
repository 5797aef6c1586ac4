"""GPU parity of the cluster transport (csrc/cluster.cuh; DESIGN.md §8 "Cluster
transport"): on virtual comms, ring / tree Simple on whole 16-B packs of
16-B aligned buffers run as one thread-block cluster per channel, every hop a
distributed-shared-memory store.  Checked against the oracle element by
element, against the peer-memory FIFO kernels (POLAR_CLUSTER=0 comm) where the
reduction order is the same, at the bench size on sampled windows, under CUDA
graph replay and under fault injection; and the dispatch rule (which calls run
as clusters) through polar_comm_transport.
"""
import numpy as np
import pytest

import synth
from tests.gpu_common import check_result, default_dist, to_device, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402

ES = {"i32": 4, "i64": 8, "f32": 4, "bf16": 2}


def _comm(n, monkeypatch, cluster=True, **env):
    monkeypatch.setenv("POLAR_CLUSTER", "1" if cluster else "0")
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    return L.Comm.virtual(n, 0)


def _aligned(count, dtype):
    """Round a count down to whole 16-B packs (the cluster path's condition)."""
    per = 16 // ES[dtype]
    return max(per, count // per * per)


@pytest.mark.parametrize("algo", ["ring", "tree"])
@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_cluster_matrix(algo, n, monkeypatch):
    """Every dtype x op, sizes from one pack to many laps / tiles with ragged
    tails, channel counts 1..32: the cluster path vs the oracle (the tree's size
    bound lifted so that every size runs as clusters)."""
    c = _comm(n, monkeypatch, POLAR_CLUSTER_TREE_MAX=1 << 40)
    try:
        for dtype in synth.DTYPES:
            for op in ("sum", "max", "min"):
                for count, nch in ((16, 1), (1000, 3), (40_000, 4), (300_000, 7), ((3 << 20) + 64, 32)):
                    count = _aligned(count, dtype)
                    if op != "sum" and count > 400_000:
                        continue
                    xs = synth.gen_ranks(dtype, count, n, cfg=21, dist=default_dist(dtype))
                    ts = [to_device(x, dtype) for x in xs]
                    c.allreduce_forced(ts, algo, "simple", nch, op=op)
                    assert c.transport() == "cluster", (dtype, count)
                    torch.cuda.synchronize()
                    c.check()
                    check_result([to_host(t, dtype) for t in ts], xs, dtype, op, algo, n)
    finally:
        c.destroy()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cluster_tree_vs_fifo_tree(dtype, monkeypatch):
    """The cluster tree (a double binary tree: the second half of each channel
    through the tree with positions shifted by ceil(n/2)) against the FIFO
    tree: every element is reduced up one binary tree in both, so integer-valued
    inputs give identical results, and real data stays within the tree's bound
    (R2 / R3); sizes from one tile to many, channel counts 1..15."""
    n = 8
    a = _comm(n, monkeypatch, cluster=True)
    b = _comm(n, monkeypatch, cluster=False)
    try:
        for count, nch in ((4096, 1), (123_456, 5), (2_000_000, 15), (9_000_000, 15)):
            count = _aligned(count, dtype)
            for dist in ("ints", default_dist(dtype)):
                xs = synth.gen_ranks(dtype, count, n, cfg=33, dist=dist)
                ta = [to_device(x, dtype) for x in xs]
                tb = [to_device(x, dtype) for x in xs]
                a.allreduce_forced(ta, "tree", "simple", nch)
                b.allreduce_forced(tb, "tree", "simple", nch)
                assert a.transport() == "cluster" and b.transport() == "peer"
                assert a.launched_channels() == b.launched_channels() == nch
                torch.cuda.synchronize()
                a.check()
                got = [to_host(t, dtype) for t in ta]
                check_result(got, xs, dtype, "sum", "tree", n)
                if dist == "ints":
                    fifo = to_host(tb[0], dtype)
                    for g in got:
                        assert np.array_equal(g, fifo), count
    finally:
        a.destroy()
        b.destroy()


def test_fifo_ring_tree_aligned_matrix(monkeypatch):
    """The peer-memory FIFO ring / tree Simple (what real comms run) keeps its
    own coverage at aligned sizes on a POLAR_CLUSTER=0 comm."""
    for n in (2, 8):
        c = _comm(n, monkeypatch, cluster=False)
        try:
            for algo in ("ring", "tree"):
                for dtype in synth.DTYPES:
                    for count, nch in ((1000, 3), (300_000, 8), ((3 << 20), 32)):
                        count = _aligned(count, dtype)
                        xs = synth.gen_ranks(dtype, count, n, cfg=44, dist=default_dist(dtype))
                        ts = [to_device(x, dtype) for x in xs]
                        c.allreduce_forced(ts, algo, "simple", nch)
                        assert c.transport() == "peer"
                        torch.cuda.synchronize()
                        c.check()
                        check_result([to_host(t, dtype) for t in ts], xs, dtype, "sum", algo, n)
        finally:
            c.destroy()


@pytest.mark.parametrize("algo", ["ring", "tree"])
def test_cluster_empty_channels_and_tiny(algo, monkeypatch):
    """More channels than packs (most clusters get an empty slice and go
    straight to the rendezvous), one pack, one tile plus one pack, and a
    ragged last tile, back to back without host sync."""
    for n in (2, 8):
        c = _comm(n, monkeypatch)
        try:
            pending = []
            for dtype, count, nch in (("f32", 4, 15), ("bf16", 8, 15), ("i64", 64, 15), ("f32", 4100, 9),
                                      ("bf16", 8200, 3), ("i32", 1024 * 4 + 4, 1)):
                xs = synth.gen_ranks(dtype, count, n, cfg=71, dist=default_dist(dtype))
                ts = [to_device(x, dtype) for x in xs]
                c.allreduce_forced(ts, algo, "simple", nch)
                assert c.transport() == "cluster"
                pending.append((xs, ts, dtype))
            torch.cuda.synchronize()
            c.check()
            for xs, ts, dtype in pending:
                check_result([to_host(t, dtype) for t in ts], xs, dtype, "sum", algo, n)
        finally:
            c.destroy()


def test_cluster_dispatch_rule(monkeypatch):
    """Which calls run as clusters (polar.h polar_comm_transport): ring / tree
    Simple on aligned whole packs; not LL / LL128, not a partial last pack, not
    an unaligned buffer, not the tree above POLAR_CLUSTER_TREE_MAX."""
    n = 4
    c = _comm(n, monkeypatch, POLAR_CLUSTER_TREE_MAX=1 << 20)
    try:
        def run(count, algo, proto, offset=0, dtype="f32"):
            xs = synth.gen_ranks(dtype, count, n, cfg=5, dist="ints")
            ts = [to_device(x, dtype, offset) for x in xs]
            c.allreduce_forced(ts, algo, proto, 4)
            torch.cuda.synchronize()
            c.check()
            check_result([to_host(t, dtype) for t in ts], xs, dtype, "sum", algo, n)
            return c.transport()
        assert run(4096, "ring", "simple") == "cluster"
        assert run(4096, "tree", "simple") == "cluster"
        assert run(4097, "ring", "simple") == "peer"           # partial last pack
        assert run(4096, "ring", "simple", offset=1) == "peer"  # unaligned buffers
        assert run(4096, "ring", "ll") == "peer"
        assert run(4096, "twoshot", "simple") == "peer"
        assert run((1 << 20) // 4, "tree", "simple") == "cluster"        # 1 MiB = the bound
        assert run((1 << 20) // 4 + 4, "tree", "simple") == "peer"       # above it
        assert run((4 << 20) // 4, "ring", "simple") == "cluster"        # the ring has no bound
    finally:
        c.destroy()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cluster_ring_bench_size_sampled(dtype, monkeypatch):
    """The C2 size (8 ranks x 128 MiB) through the cluster ring, in the launch
    configuration the bench's algorithm record times (32 channels requested,
    clamped to the clusters that fit): sampled windows vs the oracle."""
    n, count = 8, (128 << 20) // ES[dtype]
    c = _comm(n, monkeypatch)
    try:
        xs = synth.gen_ranks(dtype, count, n, cfg=2, dist=default_dist(dtype))
        ts = [to_device(x, dtype) for x in xs]
        c.allreduce_forced(ts, "ring", "simple", 32)
        assert c.transport() == "cluster"
        torch.cuda.synchronize()
        c.check()
        rng = np.random.default_rng(7)
        windows = [(0, 4096), (count - 4096, count)] + [(int(s), int(s) + 2048)
                                                        for s in rng.integers(0, count - 2048, 16)]
        for lo, hi in windows:
            got = [to_host(t[lo:hi], dtype) for t in ts]
            check_result(got, [x[lo:hi] for x in xs], dtype, "sum", "ring", n)
    finally:
        del ts
        c.destroy()
        torch.cuda.empty_cache()


def test_cluster_graph_replay(monkeypatch):
    """Cluster ring and tree captured in one CUDA graph with a peer-transport
    call between them, replayed with new inputs: exact on integer-valued data."""
    n = 8
    c = _comm(n, monkeypatch)
    try:
        counts = [262_144, 4_099, 65_536]
        algos = [("ring", "simple"), ("ring", "simple"), ("tree", "simple")]   # 4_099: partial pack -> peer
        bufs = [[torch.empty(k, dtype=torch.float32, device="cuda") for _ in range(n)] for k in counts]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for (algo, proto), b in zip(algos, bufs):
                c.allreduce_forced(b, algo, proto, 6)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for (algo, proto), b in zip(algos, bufs):
                c.allreduce_forced(b, algo, proto, 6)
        for rep in range(3):
            xs_all = []
            for k, b in zip(counts, bufs):
                xs = synth.gen_ranks("f32", k, n, cfg=500 + rep, dist="ints")
                for r in range(n):
                    b[r].copy_(torch.from_numpy(xs[r]))
                xs_all.append(xs)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            c.check()
            for xs, b in zip(xs_all, bufs):
                exp = orc.allreduce(xs, "f32", "sum")
                for t in b:
                    assert np.array_equal(to_host(t, "f32"), exp), rep
    finally:
        c.destroy()


def test_cluster_jitter_back_to_back(monkeypatch):
    """Random warp delays before the DSMEM sends (POLAR_JITTER_NS), cluster and
    peer calls back to back without host sync: exact on integer-valued data."""
    n = 8
    c = _comm(n, monkeypatch, POLAR_JITTER_NS=20000, POLAR_TIMEOUT_MS=30000)
    try:
        rng = np.random.default_rng(3)
        pending = []
        for it in range(24):
            algo = ("ring", "tree")[it % 2]
            count = int(rng.integers(1, 400_000)) * 4
            if it % 3 == 2:
                count += 1                                  # a peer-transport call in between
            xs = synth.gen_ranks("f32", count, n, cfg=600 + it, dist="ints")
            ts = [to_device(x, "f32") for x in xs]
            c.allreduce_forced(ts, algo, "simple", int(rng.integers(1, 16)))
            pending.append((xs, ts, algo))
        torch.cuda.synchronize()
        c.check()
        for xs, ts, algo in pending:
            check_result([to_host(t, "f32") for t in ts], xs, "f32", "sum", algo, n)
    finally:
        c.destroy()


def test_cluster_random_sweep(monkeypatch):
    """Seeded random configurations through the cluster transport — n, dtype,
    op, whole-pack count (up to ~4 MiB per rank), channel count — each checked
    against the oracle; ring and tree alternate, back to back per comm."""
    rng = np.random.default_rng(2026)
    for n in (2, 3, 4, 6, 7, 8):
        c = _comm(n, monkeypatch)
        try:
            pending = []
            for it in range(12):
                dtype = synth.DTYPES[int(rng.integers(len(synth.DTYPES)))]
                op = ("sum", "max", "min")[int(rng.integers(3))]
                per = 16 // ES[dtype]
                count = per * int(rng.integers(1, (4 << 20) // 16))
                algo = ("ring", "tree")[it % 2]
                nch = int(rng.integers(1, 33))
                xs = synth.gen_ranks(dtype, count, n, cfg=900 + it, dist=default_dist(dtype))
                ts = [to_device(x, dtype) for x in xs]
                c.allreduce_forced(ts, algo, "simple", nch, op=op)
                assert c.transport() == "cluster"
                pending.append((xs, ts, dtype, op, algo))
            torch.cuda.synchronize()
            c.check()
            for xs, ts, dtype, op, algo in pending:
                check_result([to_host(t, dtype) for t in ts], xs, dtype, op, algo, n)
        finally:
            c.destroy()
