"""Host logic of the measurement path (CPU): bench.py's parity checker of the
timed buffers (it must accept the oracle's result and refuse a single flipped
bit, a rank that differs, or a ring result outside R2's bound), its sampled
windows, the NCCL TUNING-log parser, and the binding's tensor checks."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import bench  # noqa: E402
import nccl_ctypes  # noqa: E402
import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402

torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True)
def _no_device_sync(monkeypatch):
    monkeypatch.setattr(torch.cuda, "synchronize", lambda *a, **k: None)   # CPU stand-in


class _Dec:
    def __init__(self, algo):
        self.algo = algo


class _FakeL:
    ALGO_NAMES = {3: "oneshot", 4: "twoshot", 1: "ring"}


class _FakeComm:
    def __init__(self, algo):
        self.algo = algo

    def check(self):
        pass

    def last_decision(self):
        return _Dec(self.algo)


def _run(n, count, algo, corrupt=None):
    """n 'ranks' of CPU tensors; step() writes the oracle's result (optionally corrupted)."""
    xs = synth.gen_ranks("f32", count, n, cfg=2, dist="unif")
    bufs = [torch.zeros(count, dtype=torch.float32) for _ in range(n)]
    exp = orc.allreduce(xs, "f32", "sum")

    def step():
        for r, b in enumerate(bufs):
            y = exp.copy()
            if corrupt:
                corrupt(r, y)
            b.copy_(torch.from_numpy(y))
    return bench.check_parity(_FakeL, _FakeComm(algo), bufs, xs, list(range(n)), n, count, step, lambda o: [o])


def test_parity_accepts_the_oracle_result():
    p = _run(8, 100_003, 4)
    assert p["ok"] and p["ranks_identical"] and p["rule"].startswith("bit-exact")
    assert p["windows"] == 18 and p["elements_per_rank"] == 17 * 2048 + 2051   # the tail window runs to the last element


def test_parity_refuses_one_flipped_bit_in_a_window():
    lo = bench.parity_windows(100_003)[3][0]

    def flip(r, y):
        v = y.view(np.uint32)
        v[lo + 7] ^= 1
    p = _run(4, 100_003, 4, corrupt=flip)
    assert not p["ok"]


def test_parity_refuses_ranks_that_differ():
    def one_rank(r, y):
        if r == 2:
            y[-1] = np.nextafter(y[-1], np.float32(np.inf))
    p = _run(4, 50_000, 1, corrupt=one_rank)     # within R2's bound, but not identical
    assert not p["ok"] and not p["ranks_identical"]


def test_parity_ring_bound():
    ok = _run(8, 60_000, 1)
    assert ok["ok"] and ok["rule"].startswith("|y - y*|") and ok["max_err_over_bound"] == 0.0

    def far(r, y):
        y[0] += 1.0                                 # far outside 1e-6 * n * sum|x|
    assert not _run(8, 60_000, 1, corrupt=far)["ok"]


def test_parity_windows_cover_both_ends():
    w = bench.parity_windows(1 << 20)
    assert w[0] == (0, 2048) and w[1][1] == 1 << 20
    assert all(0 <= a < b <= 1 << 20 for a, b in w)


def test_nccl_tuning_log_parser(tmp_path):
    log = tmp_path / "nccl.log"
    log.write_text("host:1:1 [0] NCCL INFO 4194304 Bytes -> Algo 4 proto 2 time 10.0\n"
                   "host:1:1 [0] NCCL INFO something else\n"
                   "host:1:1 [0] NCCL INFO 8192 Bytes -> Algo 1 proto 0 time 3.1\n"
                   "host:1:1 [0] NCCL INFO 4194304 Bytes -> Algo 1 proto 1 time 9.0\n")
    got = nccl_ctypes.parse_tuning(str(log))
    assert got == {4194304: ("ring", "ll128"), 8192: ("ring", "ll")}     # last decision per size wins
    assert nccl_ctypes.parse_tuning(str(tmp_path / "missing")) == {}


def test_binding_tensor_checks_on_cpu():
    from paper_2603_11438_b200 import polar as L
    L._check_tensor(torch.zeros(4), "x", cuda=False)                      # host tensor where host expected
    for bad, cuda in ((torch.zeros(4), True), (torch.zeros(8)[::2], False), ([1, 2], False)):
        with pytest.raises(L.PolarError) as e:
            L._check_tensor(bad, "x", cuda=cuda)
        assert e.value.name == "einval"
