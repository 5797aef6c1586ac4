"""Fault injection and failure detection on the GPU.

* jitter: random __nanosleep before 1/8 of all signalling / LL stores
  (POLAR_JITTER_NS) — every algorithm x protocol must stay exact under skewed
  arrival orders, including back-to-back calls without host sync;
* timeout: a rank that never joins makes its peer's wait expire after
  POLAR_TIMEOUT_MS: ETIMEOUT latched, control returned, later calls refused.
"""
import itertools
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from tests.gpu_common import check_result, to_device, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_11438_b200 import polar as L  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMBOS = list(itertools.product(["oneshot", "twoshot", "ring", "tree"], ["ll", "ll128", "simple"]))


@pytest.mark.parametrize("n", [3, 8])
def test_jitter_all_protocols(n, monkeypatch):
    monkeypatch.setenv("POLAR_JITTER_NS", "20000")
    monkeypatch.setenv("POLAR_TIMEOUT_MS", "30000")
    c = L.Comm.virtual(n, 0)
    try:
        rng = np.random.default_rng(n)
        pending = []
        for it in range(3 * len(COMBOS)):
            algo, proto = COMBOS[it % len(COMBOS)]
            count = int(rng.integers(1, 150_000))
            dtype = ("f32", "i32", "bf16")[it % 3]
            xs = synth.gen_ranks(dtype, count, n, cfg=200 + it, dist="ints")
            ts = [to_device(x, dtype) for x in xs]
            c.allreduce_forced(ts, algo, proto, int(rng.integers(1, 9)))
            pending.append((xs, ts, dtype, algo))
        torch.cuda.synchronize()
        c.check()
        for xs, ts, dtype, algo in pending:
            check_result([to_host(t, dtype) for t in ts], xs, dtype, "sum", algo, n)
    finally:
        c.destroy()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("algo,proto", [("twoshot", "simple"), ("oneshot", "ll"), ("ring", "simple")])
def test_missing_rank_times_out(tmp_path, algo, proto):
    out = tmp_path / "to.json"
    env = dict(os.environ)
    env["POLAR_TIMEOUT_MS"] = "1500"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "mp_timeout_worker.py"), str(out), algo, proto]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert all(x["first_ok"] for x in rep)
    r0 = [x for x in rep if x["rank"] == 0][0]
    assert r0["status"] == "etimeout"
    assert r0["next_call"] == "etimeout"
    assert r0["seconds"] < 60


@pytest.mark.parametrize("mode", [1, 2])
def test_ll128_line_atomicity_probe(mode):
    """The LL128 premise on this GPU (polar_probe_ll128): a reader that sees a
    line's flag sees that line's payload, with readers spinning while writers
    are delayed warp-uniformly (mode 1, the LL128 fault injection) or by
    per-lane divergent busy waits (mode 2).  Per-lane NANOSLEEP before the store
    (mode 0) is known to tear (profiles/r01_probe_ll128.jsonl) and is not used."""
    torn, reads = L.probe_ll128(0, pairs=32, iters=20000, jitter_ns=2000, jitter_mode=mode)
    assert reads == 32 * 20000 * 32
    assert torn == 0
