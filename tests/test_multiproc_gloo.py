"""N>1 host logic on CPU: world_size-2 (and 3) gloo process groups launched by
torchrun on 127.0.0.1 (no GPU): bootstrap all-gather through the C callback,
layout-mismatch detection, rank-consistent decisions."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, nranks, mode, env_extra=None):
    out = tmp_path / f"{mode}.json"
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "gloo_worker.py"), str(out), mode]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(out.read_text())


@pytest.mark.parametrize("nranks", [2, 3])
def test_bootstrap_and_consistent_decisions(tmp_path, nranks):
    rep = _run(tmp_path, nranks, "consistency")
    assert len(rep) == nranks
    for r in rep:
        assert r["bootstrap"] == "ok" and r["bootstrap_tensor_ag"] == "ok"
        assert r["decisions_identical"] and r["gens_identical"]
        assert r["gens"] == sorted(r["gens"]) and len(set(r["gens"])) == len(r["gens"])


def test_bootstrap_detects_layout_mismatch(tmp_path):
    """One rank with a different POLAR_OS_CHUNK would corrupt staging offsets:
    the check must fail on every rank (torchrun passes env to all ranks, so the
    mismatch is injected through a per-rank variable the worker maps)."""
    rep = _run(tmp_path, 2, "mismatch", {"POLAR_TEST_SKEW_RANK": "1"})
    assert all(r["bootstrap"] == "estate" for r in rep)
