"""Time-bounded random stress of every AllReduce kernel on virtual comms
(POLAR_STRESS_S seconds, default 45): random n, dtype, op, algorithm x
protocol (ring / tree Simple run as clusters where eligible, the peer-memory
FIFO kernels otherwise), element counts (whole packs and ragged), channel
counts and buffer offsets, issued in back-to-back batches of 6 calls (a fifth of them direct ReduceScatter /
AllGather / Broadcast) on one
stream with no host synchronisation in between, half of the comms with
random fault-injection delays.  Integer-valued inputs make every algorithm's
result exact, so each call is compared bitwise with the oracle.  A rare race
(a late remote write, a stage reused early) shows up here as a mismatch or a
timeout, which no fixed-size parity case would hit."""
import os
import time

import numpy as np
import pytest

import synth
from tests.gpu_common import to_device, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle import allreduce as orc  # noqa: E402
from oracle import collectives as ocol  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402

ALGOS = ("oneshot", "twoshot", "ring", "tree")
PROTOS = ("ll", "ll128", "simple")
ES = {"i32": 4, "i64": 8, "f32": 4, "bf16": 2}


def test_random_back_to_back_stress(monkeypatch):
    budget = float(os.environ.get("POLAR_STRESS_S", "45"))
    debug = os.environ.get("POLAR_STRESS_DEBUG") == "1"   # print every call, synchronise after it
    rng = np.random.default_rng(int(os.environ.get("POLAR_STRESS_SEED", "2603")))
    t_end = time.monotonic() + budget
    calls = clusters = 0
    stats = {}
    monkeypatch.setenv("POLAR_CLUSTER_TREE_MAX", str(1 << 40))
    while time.monotonic() < t_end:
        n = int(rng.integers(2, 9))
        jitter = int(rng.integers(2)) * 3000
        monkeypatch.setenv("POLAR_JITTER_NS", str(jitter))
        c = L.Comm.virtual(n, 0)
        try:
            for _batch in range(4):
                pending = []
                for _ in range(6):
                    dtype = synth.DTYPES[int(rng.integers(len(synth.DTYPES)))]
                    op = ("sum", "max", "min")[int(rng.integers(3))]
                    algo = ALGOS[int(rng.integers(4))]
                    proto = PROTOS[int(rng.integers(3))]
                    per = 16 // ES[dtype]
                    big = int(rng.integers(2)) == 1
                    count = int(rng.integers(1, (1 << 21) if big else 5000))
                    if int(rng.integers(2)):
                        count = max(per, count // per * per)     # whole packs (cluster-eligible)
                    off = int(rng.integers(2)) * int(rng.integers(1, per))   # element offset: unaligned start
                    nch = int(rng.integers(1, 33))
                    xs = synth.gen_ranks(dtype, count, n, cfg=int(rng.integers(1 << 30)), dist="ints")
                    if int(rng.integers(5)) == 0 and count >= n:
                        # a direct ReduceScatter / AllGather / Broadcast in the same stream
                        coll = ("rs", "ag", "bc")[int(rng.integers(3))]
                        blk = max(1, count // n)
                        if coll == "rs":
                            xr = [x[:blk * n] for x in xs]
                            snd = [to_device(x, dtype) for x in xr]
                            rcv = [to_device(np.zeros(blk, dtype=x.dtype), dtype) for x in xr]
                            c.reduce_scatter(snd, rcv, op=op)
                            pending.append(("rs", xr, rcv, dtype, op, None))
                        elif coll == "ag":
                            xa = [x[:blk] for x in xs]
                            snd = [to_device(x, dtype) for x in xa]
                            rcv = [to_device(np.zeros(blk * n, dtype=x.dtype), dtype) for x in xa]
                            c.all_gather(snd, rcv)
                            pending.append(("ag", xa, rcv, dtype, op, None))
                        else:
                            root = int(rng.integers(n))
                            bts = [to_device(x, dtype) for x in xs]
                            c.broadcast(bts, root=root)
                            pending.append(("bc", xs, bts, dtype, op, root))
                        stats[(coll,)] = stats.get((coll,), 0) + 1
                        continue
                    ts = [to_device(x, dtype, offset=off) for x in xs]
                    if debug:
                        print("call", n, jitter, dtype, op, algo, proto, count, nch, off, flush=True)
                    c.allreduce_forced(ts, algo, proto, nch, op=op)
                    if debug:
                        torch.cuda.synchronize()
                    key = (algo, proto, c.transport())
                    stats[key] = stats.get(key, 0) + 1
                    clusters += c.transport() == "cluster"
                    pending.append((xs, ts, dtype, op, key, count, nch, off))
                torch.cuda.synchronize()
                c.check()
                for item in pending:
                    if isinstance(item[0], str):
                        coll, xs, outs, dtype, op, root = item
                        if coll == "rs":
                            exps = ocol.reduce_scatter(xs, dtype, op)
                        elif coll == "ag":
                            exps = [ocol.all_gather(xs)] * n
                        else:
                            exps = [ocol.broadcast(xs, root)] * n
                        for r, (t, e) in enumerate(zip(outs, exps)):
                            got = to_host(t, dtype)
                            ok = np.array_equal(got, e) if (dtype == "f32" and op != "sum" and coll == "rs") else \
                                np.array_equal(got.view(np.uint8), np.asarray(e).view(np.uint8))
                            assert ok, (n, coll, dtype, op, len(xs[0]), r)
                        calls += 1
                        continue
                    xs, ts, dtype, op, key, count, nch, off = item
                    exp = orc.allreduce(xs, dtype, op)
                    for r, t in enumerate(ts):
                        got = to_host(t, dtype)
                        ok = np.array_equal(got, exp) if (dtype == "f32" and op != "sum") else \
                            np.array_equal(got.view(np.uint8), exp.view(np.uint8))
                        assert ok, (n, dtype, op, key, count, nch, off, jitter, r)
                    calls += 1
        finally:
            c.destroy()
    print(f"stress: {calls} calls checked in {budget:.0f} s, {clusters} as clusters; "
          f"{sorted(stats.items(), key=str)}")
    assert calls > 0
