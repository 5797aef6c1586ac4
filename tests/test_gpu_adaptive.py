"""Profiler -> tuner closed loop live on the GPU (PAPER.md
§5.3): device-timed telemetry feeds the controller, the launched
channel count ramps 2 -> cap, backs off under injected contention (10x latency,
SPEC.md L366-368 style) and recovers; with the profiler off it stays at 2.
Real comms (2 processes) must follow identical channel traces on every rank."""
import json
import os
import socket
import subprocess
import sys

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

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CAP, PERIOD = 12, 8
ROWS = [(0, 0, 2**64 - 1, OP.TWOSHOT, OP.SIMPLE, CAP, OP.ROW_ADAPTIVE_NCH)]


def _run_windows(c, ts, nwin):
    trace = []
    for _ in range(nwin * PERIOD):
        c.allreduce(ts)
        torch.cuda.synchronize()      # every call's telemetry completes before the next window closes
        trace.append(c.launched_channels())
    c.check()
    return trace[PERIOD - 1::PERIOD]  # channels launched at the last call of each window


def test_closed_loop_three_phases():
    L.set_policy(ROWS)
    c = L.Comm.virtual(8, 0)
    try:
        c.adaptive_config(enabled=True, period=PERIOD, c_min=2, contention_factor=4.0)
        xs = synth.gen_ranks("f32", 1 << 20, 8, cfg=21, dist="ints")
        ts = [to_device(x, "f32") for x in xs]
        ramp = _run_windows(c, ts, 12)
        assert ramp[0] <= 3 and ramp[-1] == CAP and ramp == sorted(ramp)
        c.adaptive_inject(10.0)                         # contention: 10x latency
        cont = _run_windows(c, ts, 6)
        assert all(x <= 3 for x in cont[1:]), cont
        assert c.adaptive_state()["contended"] == 1
        c.adaptive_inject(1.0)                          # recovery
        rec = _run_windows(c, ts, 12)
        assert rec[-1] == CAP, rec
        st = c.adaptive_state()
        assert st["samples"] >= 20 * PERIOD and st["windows"] >= 25
        # the data path stayed exact throughout (each call doubles... check one fresh call)
        ts2 = [to_device(x, "f32") for x in xs]
        c.allreduce(ts2)
        torch.cuda.synchronize()
        exp = orc.allreduce(xs, "f32", "sum")
        assert all(np.array_equal(to_host(t, "f32"), exp) for t in ts2)
    finally:
        c.destroy()
        L.set_policy([])


def test_profiler_off_stays_at_cmin():
    L.set_policy(ROWS)
    c = L.Comm.virtual(4, 0)
    try:
        c.adaptive_config(enabled=False, period=PERIOD, c_min=2)
        ts = [torch.ones(1 << 18, device="cuda") for _ in range(4)]
        tr = _run_windows(c, ts, 6)
        assert tr == [2] * 6
        assert c.adaptive_state()["samples"] == 0
    finally:
        c.destroy()
        L.set_policy([])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_real_comm_ranks_follow_identical_traces(tmp_path):
    out = tmp_path / "ad.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "mp_adaptive_worker.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert rep[0]["trace"] == rep[1]["trace"]
    assert rep[0]["trace"][-1] == rep[0]["cap"] and all(x["ok"] for x in rep)
