"""Hot reload under load on the GPU path (BASELINE config 5 x the hot path;
PAPER.md L390-397, L483-487: the policy is swapped while collectives run and no
call is lost): one thread issues 300 policy-selected AllReduces on a virtual comm
while another swaps between two tables every 0.5 ms.  Every call must complete
with the oracle's result, record a decision that belongs to one of the two
tables at the generation it reports, and generations must never go backwards."""
import threading
import time

import numpy as np
import pytest

import synth
from oracle import allreduce as orc
from oracle import policy as OP
from tests.gpu_common import to_device, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_11438_b200 import polar as L  # noqa: E402


def test_swap_while_allreducing():
    n, count = 4, 30_001
    table_a = [(0, 0, 2**64 - 1, OP.TWOSHOT, OP.SIMPLE, 8)]
    table_b = [(0, 0, 64 << 10, OP.ONESHOT, OP.LL128, 4), (0, 0, 2**64 - 1, OP.RING, OP.LL, 6)]
    g0 = L.set_policy(table_a)
    gens = {}
    stop = threading.Event()

    def reloader():
        k = 0
        while not stop.is_set():
            rows = table_b if k % 2 == 0 else table_a
            g = L.set_policy(rows)
            gens[g] = rows
            k += 1
            time.sleep(0.0005)

    gens[g0] = table_a
    c = L.Comm.virtual(n, 0)
    t = threading.Thread(target=reloader)
    xs = synth.gen_ranks("f32", count, n, cfg=77, dist="ints")
    exp = orc.allreduce(xs, "f32", "sum")
    last_gen, calls, seen = g0, 0, []
    try:
        t.start()
        while calls < 300:
            ts = [to_device(x, "f32") for x in xs]
            c.allreduce(ts)
            torch.cuda.synchronize()
            c.check()
            d = c.last_decision()
            assert d.generation >= last_gen
            last_gen = d.generation
            seen.append((d.generation, d.as_tuple()))
            calls += 1
            for tt in ts:
                assert np.array_equal(to_host(tt, "f32"), exp)
        stop.set()
        t.join()
        # every call's decision is the oracle's mapping under the table of the
        # generation it reports (the table published with that generation)
        for g, dec in seen:
            assert dec == OP.decide(gens[g], 0, n, count * 4), (g, dec)
        assert len({g for g, _ in seen}) > 10
    finally:
        stop.set()
        t.join()
        c.destroy()
        L.set_policy([])
