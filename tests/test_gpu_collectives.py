"""ReduceScatter / AllGather / Broadcast through the same hook vs
oracle/collectives.py on virtual ranks: dtypes, ops, ragged and 16-B-unaligned
blocks, in-place forms, every root, n = 1 identity, and the recorded decision."""
import numpy as np
import pytest

import synth
from oracle import collectives as OC
from oracle import policy as OP
from tests.gpu_common import default_dist, to_device, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_11438_b200 import polar as L  # noqa: E402

_C = {}


def comm(n):
    if n not in _C:
        _C[n] = L.Comm.virtual(n, 0)
    return _C[n]


def _eq(got, exp, dtype, op):
    if dtype == "f32" and op != "sum":
        return np.array_equal(got, exp)
    return np.array_equal(got.view(np.uint8), exp.view(np.uint8))


@pytest.mark.parametrize("dtype", synth.DTYPES)
@pytest.mark.parametrize("op", ["sum", "max", "min"])
def test_reduce_scatter(dtype, op):
    for n in (1, 2, 3, 8):
        c = comm(n)
        for rc in (1, 4, 1001, 65_539):
            xs = synth.gen_ranks(dtype, n * rc, n, cfg=70, dist=default_dist(dtype))
            sends = [to_device(x, dtype) for x in xs]
            recvs = [torch.empty(rc, dtype=sends[0].dtype, device="cuda") for _ in range(n)]
            c.reduce_scatter(sends, recvs, op=op)
            torch.cuda.synchronize()
            c.check()
            exp = OC.reduce_scatter(xs, dtype, op)
            for r in range(n):
                assert _eq(to_host(recvs[r], dtype), exp[r], dtype, op), (n, rc, r)
            d = c.last_decision()
            assert d.as_tuple() == OP.decide([], OP.COLL_REDUCESCATTER, n, n * rc * synth.ESIZE[dtype])


def test_reduce_scatter_in_place():
    n, rc = 4, 33_333
    xs = synth.gen_ranks("bf16", n * rc, n, cfg=71, dist="normal")
    bufs = [to_device(x, "bf16") for x in xs]
    comm(n).reduce_scatter(bufs, [bufs[r][r * rc:(r + 1) * rc] for r in range(n)])
    torch.cuda.synchronize()
    exp = OC.reduce_scatter(xs, "bf16", "sum")
    for r in range(n):
        assert np.array_equal(to_host(bufs[r][r * rc:(r + 1) * rc], "bf16"), exp[r])


@pytest.mark.parametrize("dtype", synth.DTYPES)
def test_all_gather(dtype):
    for n in (1, 2, 3, 8):
        c = comm(n)
        for sc in (1, 5, 1001, 70_001):
            xs = synth.gen_ranks(dtype, sc, n, cfg=72, dist=default_dist(dtype))
            sends = [to_device(x, dtype) for x in xs]
            recvs = [torch.zeros(n * sc, dtype=sends[0].dtype, device="cuda") for _ in range(n)]
            c.all_gather(sends, recvs)
            torch.cuda.synchronize()
            c.check()
            exp = OC.all_gather(xs)
            for r in range(n):
                assert np.array_equal(to_host(recvs[r], dtype).view(np.uint8), exp.view(np.uint8)), (n, sc, r)


def test_all_gather_in_place():
    n, sc = 8, 12_345
    xs = synth.gen_ranks("i64", sc, n, cfg=73, dist="full")
    recvs = [torch.zeros(n * sc, dtype=torch.int64, device="cuda") for _ in range(n)]
    for r in range(n):
        recvs[r][r * sc:(r + 1) * sc] = torch.from_numpy(xs[r]).cuda()
    comm(n).all_gather([recvs[r][r * sc:(r + 1) * sc] for r in range(n)], recvs)
    torch.cuda.synchronize()
    exp = OC.all_gather(xs)
    for r in range(n):
        assert np.array_equal(to_host(recvs[r], "i64"), exp)


@pytest.mark.parametrize("dtype", synth.DTYPES)
def test_broadcast_every_root(dtype):
    for n in (1, 3, 8):
        c = comm(n)
        for root in range(n):
            xs = synth.gen_ranks(dtype, 40_003, n, cfg=74 + root, dist=default_dist(dtype))
            bufs = [to_device(x, dtype) for x in xs]
            c.broadcast(bufs, root=root)
            torch.cuda.synchronize()
            c.check()
            exp = OC.broadcast(xs, root)
            for r in range(n):
                assert np.array_equal(to_host(bufs[r], dtype).view(np.uint8), exp.view(np.uint8))


def test_unsupported_decision_and_bad_root():
    n = 2
    c = comm(n)
    b = [torch.ones(100, device="cuda") for _ in range(n)]
    with pytest.raises(L.PolarError) as e:
        c.broadcast(b, root=2)
    assert e.value.name == "einval"
    L.set_policy([(OP.COLL_ALLGATHER, 0, 2**64 - 1, OP.RING, OP.SIMPLE, 4)])
    try:
        with pytest.raises(L.PolarError) as e:
            c.all_gather(b, [torch.ones(200, device="cuda") for _ in range(n)])
        assert e.value.name == "eunsupported"
    finally:
        L.set_policy([])
