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
    # a collective row naming an algorithm with no kernel is refused at install
    # time (the old table stays), not at call time
    g0 = L.generation()
    st, _ = L.set_policy_status([(OP.COLL_ALLGATHER, 0, 2**64 - 1, OP.RING, OP.SIMPLE, 4)])
    assert L.STATUS_NAMES[st] == "eunsupported" and L.generation() == g0
    recv = [torch.zeros(200, device="cuda") for _ in range(n)]
    c.all_gather(b, recv)
    torch.cuda.synchronize()
    assert all(bool((r == 1).all()) for r in recv)


def _fold_xor(arr_u32):
    w = arr_u32.reshape(-1, 4).astype(np.uint64)
    return int(np.bitwise_xor.reduce(((w[:, 0] ^ w[:, 2]) << np.uint64(32)) | (w[:, 1] ^ w[:, 3])))


def _pattern(npacks, writer):
    i = np.arange(npacks, dtype=np.uint64)
    p = np.empty((npacks, 4), dtype=np.uint32)
    p[:, 0] = (i & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    p[:, 1] = ((i >> np.uint64(32)).astype(np.uint32)) ^ np.uint32(0x9E3779B9)
    p[:, 2] = writer
    p[:, 3] = ~p[:, 0]
    return p.reshape(-1)


@pytest.mark.parametrize("n", [2, 3, 8])
def test_p2p_probe_virtual(n):
    """polar_p2p_probe: every rank reads peer (r+1)%n (checked by the
    XOR of the packs it loaded), writes the pattern into it (checked in the peer
    buffer afterwards) and bounces a flag with r^1; rates and latencies are > 0."""
    nbytes = (1 << 20) + 4096
    c = comm(n)
    bufs = [torch.randint(-2**31, 2**31 - 1, (nbytes // 4,), dtype=torch.int32, device="cuda") for _ in range(n)]
    before = [b.cpu().numpy().view(np.uint32).copy() for b in bufs]
    res = c.p2p_probe(bufs, iters=3)
    for r in range(n):
        peer = (r + 1) % n
        assert res[r]["load_xor"] == _fold_xor(before[peer]), r
        assert res[r]["load_gbs"] > 0 and res[r]["store_gbs"] > 0
        assert (res[r]["pingpong_us"] > 0) == ((r ^ 1) < n)
        got = bufs[peer].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, _pattern(nbytes // 16, r)), r


def test_binding_rejects_bad_tensors():
    """polar.py passes only a pointer and one count per call: a strided view, a
    buffer shorter than its peers', mixed dtypes, host tensors or a wrong RS/AG
    size ratio would make a kernel read or write past a buffer's end — the
    binding refuses them with EINVAL before anything is launched."""
    n = 2
    c = comm(n)
    before = c.launches()
    good = [torch.zeros(1000, device="cuda") for _ in range(n)]
    cases = [
        [torch.zeros(2000, device="cuda")[::2], good[1]],                 # strided view
        [good[0], torch.zeros(999, device="cuda")],                        # shorter peer
        [good[0], torch.zeros(1000, device="cuda", dtype=torch.int32)],    # mixed dtype
        [torch.zeros(1000), good[1]],                                      # host tensor
    ]
    for ts in cases:
        with pytest.raises(L.PolarError) as e:
            c.allreduce(ts)
        assert e.value.name == "einval"
    with pytest.raises(L.PolarError) as e:     # RS: numel(send) must be n * numel(recv)
        c.reduce_scatter([torch.zeros(1999, device="cuda") for _ in range(n)], good)
    assert e.value.name == "einval"
    with pytest.raises(L.PolarError) as e:     # AG: numel(recv) must be n * numel(send)
        c.all_gather(good, [torch.zeros(1000, device="cuda") for _ in range(n)])
    assert e.value.name == "einval"
    assert c.launches() == before
