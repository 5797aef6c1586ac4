"""CUDA-graph capture of polar calls (epochs and FIFO counters live
in device memory, so replaying a captured sequence stays correct).  Three
AllReduces with different algorithms/protocols and a ReduceScatter are captured
once and replayed several times with fresh inputs copied in between."""
import numpy as np
import pytest

import synth
from oracle import allreduce as orc
from oracle import collectives as OC
from tests.gpu_common import to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_11438_b200 import polar as L  # noqa: E402


@pytest.mark.parametrize("n", [2, 8])
def test_graph_replay(n):
    comm = L.Comm.virtual(n, 0)
    try:
        counts = [70_001, 4_099, 300_007]
        algos = [("ring", "ll"), ("twoshot", "simple"), ("tree", "simple")]
        bufs = [[torch.empty(c, dtype=torch.float32, device="cuda") for _ in range(n)] for c in counts]
        rc = 9_999
        rs_in = [torch.empty(n * rc, dtype=torch.int32, device="cuda") for _ in range(n)]
        rs_out = [torch.empty(rc, dtype=torch.int32, device="cuda") for _ in range(n)]
        s = torch.cuda.Stream()
        # warm up on the capture stream (first use of each path outside capture)
        with torch.cuda.stream(s):
            for (algo, proto), b in zip(algos, bufs):
                comm.allreduce_forced(b, algo, proto, 3)
            comm.reduce_scatter(rs_in, rs_out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for (algo, proto), b in zip(algos, bufs):
                comm.allreduce_forced(b, algo, proto, 3)
            comm.reduce_scatter(rs_in, rs_out)
        for rep in range(4):
            xs_all = []
            for c, b in zip(counts, bufs):
                xs = synth.gen_ranks("f32", c, n, cfg=300 + rep, dist="ints")
                for r in range(n):
                    b[r].copy_(torch.from_numpy(xs[r]))
                xs_all.append(xs)
            xr = synth.gen_ranks("i32", n * rc, n, cfg=400 + rep, dist="full")
            for r in range(n):
                rs_in[r].copy_(torch.from_numpy(xr[r]))
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            comm.check()
            for xs, b in zip(xs_all, bufs):
                exp = orc.allreduce(xs, "f32", "sum")
                for t in b:
                    assert np.array_equal(to_host(t, "f32"), exp), rep
            exp = OC.reduce_scatter(xr, "i32", "sum")
            for r in range(n):
                assert np.array_equal(to_host(rs_out[r], "i32"), exp[r])
    finally:
        comm.destroy()
