"""NCCL tuner-plugin shim: dlopen
libpolar_nccl_tuner.so, drive its ncclTunerPlugin_v3 / _v4 getCollInfo with a
fake cost table, and check the paper's translation rule — the preferred cell 0,
every other available cell the 1e9 sentinel, unavailable (-1) cells untouched,
no change when the preferred cell is unavailable or no row matches, and the
channel request clamped to NCCL's maximum — on the paper's worked policies
(nvlink_ring_mid_v2; bad_channels, L581).  CPU only."""
import ctypes as C
import os
import subprocess
import sys

import pytest

from oracle import policy as OP
from paper_2603_11438_b200 import polar as L
from tests.golden_io import rows_and_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TUNER = os.path.join(ROOT, "paper_2603_11438_b200", "libpolar_nccl_tuner.so")
NUM_ALGO, NUM_PROTO = 7, 3          # NCCL 2.28: TREE RING COLLNET_DIRECT COLLNET_CHAIN NVLS NVLS_TREE PAT
FUNC_ALLREDUCE, FUNC_SEND = 4, 6
IGNORE, SENTINEL = -1.0, 1e9
INIT = C.CFUNCTYPE(C.c_int, C.c_size_t, C.c_size_t, C.c_void_p, C.POINTER(C.c_void_p))
GET3 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_size_t, C.c_int, C.c_void_p, C.c_int, C.c_int,
                   C.POINTER(C.c_int))
GET4 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_size_t, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                   C.POINTER(C.c_int))
DESTROY = C.CFUNCTYPE(C.c_int, C.c_void_p)


class V3(C.Structure):
    _fields_ = [("name", C.c_char_p), ("init", INIT), ("getCollInfo", GET3), ("destroy", DESTROY)]


class V4(C.Structure):
    _fields_ = [("name", C.c_char_p), ("init", INIT), ("getCollInfo", GET4), ("destroy", DESTROY)]


@pytest.fixture(scope="module")
def plugin():
    if not os.path.exists(TUNER):
        pytest.skip("libpolar_nccl_tuner.so not built")
    lib = C.CDLL(TUNER)
    return V3.in_dll(lib, "ncclTunerPlugin_v3"), V4.in_dll(lib, "ncclTunerPlugin_v4")


@pytest.fixture(autouse=True)
def _reset():
    L.set_policy([])
    yield
    L.set_policy([])


def fake_table(ignored=((2, 0), (2, 1), (2, 2), (3, 0), (3, 1), (3, 2), (6, 0), (6, 1))):
    t = (C.c_float * (NUM_ALGO * NUM_PROTO))()
    for a in range(NUM_ALGO):
        for p in range(NUM_PROTO):
            t[a * NUM_PROTO + p] = IGNORE if (a, p) in ignored else 10.0 + 3 * a + p
    return t


def call(pl, nbytes, nranks=8, func=FUNC_ALLREDUCE, table=None, max_ch=32, v4=False):
    ctx = C.c_void_p()
    assert pl.init(nranks, 1, None, C.byref(ctx)) == 0
    t = table if table is not None else fake_table()
    nch = C.c_int(max_ch)
    if v4:
        st = pl.getCollInfo(ctx, func, nbytes, 1, C.cast(t, C.c_void_p), NUM_ALGO, NUM_PROTO, 0, C.byref(nch))
    else:
        st = pl.getCollInfo(ctx, func, nbytes, 1, C.cast(t, C.c_void_p), NUM_ALGO, NUM_PROTO, C.byref(nch))
    assert st == 0 and pl.destroy(ctx) == 0
    return [[t[a * NUM_PROTO + p] for p in range(NUM_PROTO)] for a in range(NUM_ALGO)], nch.value


def expect_preferred(tab, algo, proto):
    base = fake_table()
    for a in range(NUM_ALGO):
        for p in range(NUM_PROTO):
            b = base[a * NUM_PROTO + p]
            if b == IGNORE:
                assert tab[a][p] == IGNORE, (a, p)
            elif (a, p) == (algo, proto):
                assert tab[a][p] == 0.0, (a, p)
            else:
                assert tab[a][p] == pytest.approx(SENTINEL), (a, p)


def untouched(tab):
    base = fake_table()
    return all(tab[a][p] == base[a * NUM_PROTO + p] for a in range(NUM_ALGO) for p in range(NUM_PROTO))


@pytest.mark.parametrize("v4", [False, True])
def test_nvlink_ring_mid_v2_cost_tables(plugin, v4):
    pl = plugin[1] if v4 else plugin[0]
    assert pl.name == b"polar"
    rows, cases, _ = rows_and_cases("nvlink_ring_mid_v2.txt")
    L.set_policy(rows)
    for nranks, nbytes, a, p, *rest in [c + (None,) * (5 - len(c)) for c in cases]:
        tab, nch = call(pl, nbytes, nranks, v4=v4)
        if a == "default":
            assert untouched(tab) and nch == 32, nbytes        # defers to NCCL's own choice
        else:
            # the paper's RING (1) / LL128 (1) / SIMPLE (2): NCCL's own numbering
            expect_preferred(tab, a, p)
            assert nch == 32                                     # nch UNSET: NCCL's value kept
            assert OP.decide(rows, 0, nranks, nbytes)[:2] == (a, p)


def test_bad_channels_sets_one_channel_only(plugin):
    L.set_policy([(0, 0, 2**64 - 1, L.UNSET, L.UNSET, 1)])   # 1 channel, algorithm left to NCCL
    for nbytes in (4 << 20, 128 << 20, 8 << 30):
        tab, nch = call(plugin[0], nbytes)
        assert untouched(tab) and nch == 1


def test_channel_clamp_and_unavailable_cells(plugin):
    pl = plugin[0]
    L.set_policy([(0, 0, 1 << 20, L.TREE, L.LL, 64), (0, 0, 1 << 30, L.RING, L.LL128, 12)])
    tab, nch = call(pl, 1 << 20, max_ch=16)          # request 64 -> MAXCH 32 -> NCCL's max 16
    expect_preferred(tab, 0, 0)
    assert nch == 16
    tab, nch = call(pl, 1 << 20, max_ch=0)           # no maximum passed: clamp to [1, 32]
    assert nch == 32
    # preferred cell unavailable (-1): table left alone, NCCL falls back
    t = fake_table(ignored=((1, 1), (2, 0)))
    before = list(t)
    tab, nch = call(pl, 1 << 25, table=t)
    assert [x for row in tab for x in row] == before and nch == 12


def test_partial_rows_and_polar_only_algorithms(plugin):
    pl = plugin[0]
    # algo set, proto UNSET: NCCL keeps its protocol costs within RING; others sentinel
    L.set_policy([(0, 0, 1 << 20, L.RING, L.UNSET, 0), (0, 0, 1 << 24, L.UNSET, L.SIMPLE, 0),
                  (0, 0, 1 << 30, L.TWOSHOT, L.SIMPLE, 8)])
    tab, _ = call(pl, 1000)
    base = fake_table()
    for a in range(NUM_ALGO):
        for p in range(NUM_PROTO):
            b = base[a * NUM_PROTO + p]
            assert tab[a][p] == (IGNORE if b == IGNORE else (b if a == 1 else pytest.approx(SENTINEL)))
    tab, _ = call(pl, 1 << 22)                       # proto SIMPLE only: every algo's SIMPLE keeps its cost
    for a in range(NUM_ALGO):
        for p in range(NUM_PROTO):
            b = base[a * NUM_PROTO + p]
            assert tab[a][p] == (IGNORE if b == IGNORE else (b if p == 2 else pytest.approx(SENTINEL)))
    # polar's own two-shot has no NCCL kernel: only the protocol and channels carry over
    tab, nch = call(pl, 1 << 28)
    assert nch == 8 and all(tab[a][2] == base[a * NUM_PROTO + 2] for a in range(NUM_ALGO))
    # other NCCL functions (Send) and no matching row: nothing changes
    tab, nch = call(pl, 1 << 20, func=FUNC_SEND)
    assert untouched(tab) and nch == 32
    L.set_policy([])
    tab, nch = call(pl, 1 << 20)
    assert untouched(tab) and nch == 32


def test_policy_file_at_init(tmp_path):
    """POLAR_POLICY=file.json is read (and validated) at plugin init, as NCCL
    would load the plugin in a process that never imports polar."""
    code = f"""
import ctypes as C
INIT = C.CFUNCTYPE(C.c_int, C.c_size_t, C.c_size_t, C.c_void_p, C.POINTER(C.c_void_p))
GET3 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_size_t, C.c_int, C.c_void_p, C.c_int, C.c_int,
                   C.POINTER(C.c_int))
DESTROY = C.CFUNCTYPE(C.c_int, C.c_void_p)
class V3(C.Structure):
    _fields_ = [("name", C.c_char_p), ("init", INIT), ("getCollInfo", GET3), ("destroy", DESTROY)]
pl = V3.in_dll(C.CDLL({TUNER!r}), "ncclTunerPlugin_v3")   # no polar import: the plugin reads the file
def best(nbytes):
    ctx = C.c_void_p()
    assert pl.init(8, 1, None, C.byref(ctx)) == 0
    t = (C.c_float * 21)(*[10.0 + i for i in range(21)])
    nch = C.c_int(32)
    assert pl.getCollInfo(ctx, 4, nbytes, 1, C.cast(t, C.c_void_p), 7, 3, C.byref(nch)) == 0
    zeros = [i for i in range(21) if t[i] == 0.0]
    return [(i // 3, i % 3) for i in zeros], sorted(set(t))
assert best(8 << 20)[0] == [(1, 1)]
assert best(64 << 20)[0] == [(1, 2)]
assert best(48 << 20) == ([], [10.0 + i for i in range(21)])
print("ok")
"""
    env = dict(os.environ, POLAR_POLICY=os.path.join(ROOT, "policies", "nvlink_ring_mid_v2.json"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.gpu
def test_nccl_loads_the_shim():
    """NCCL 2.28.9 itself (torch's libnccl.so.2, through ctypes) loads the shim
    as a tuner plugin and calls its init on a one-rank communicator (the pool has
    one GPU; NCCL asks a tuner for decisions only on multi-rank communicators)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "experiments", "nccl_tuner_load.py")], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "TUNER/Plugin: Using polar" in r.stdout and "polar tuner: init nRanks 1" in r.stdout
    assert r.stdout.strip().endswith("LOADED")
