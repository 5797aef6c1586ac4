"""Real multi-process comms (polar_comm_init + CUDA IPC), one process per rank,
launched with torchrun on 127.0.0.1.  On a 1-GPU box every rank shares GPU 0
(IPC between processes on one device; kernels time-slice), which exercises the
whole real-comm path — bootstrap all-gather, IPC mapping, per-process launches,
flags across contexts — except NVLink itself."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nranks,tma,jitter", [(2, "0", "0"), (3, "0", "0"), (2, "1", "0"), (3, "0", "20000")])
def test_multiprocess_ipc_all_algorithms(tmp_path, nranks, tma, jitter):
    """tma=1: the TMA-staged two-shot (cp.async.bulk) on CUDA-IPC-mapped peer memory.
    jitter: random __nanosleep (< 20 us) before 1/8 of all signal / LL stores in
    every process (sys-scope flags, the warp-specialised ring/tree publishers
    included): every result must stay exact under skewed arrival orders."""
    out = tmp_path / "mp.json"
    env = dict(os.environ)
    env["POLAR_TWOSHOT_TMA"] = tma
    env["POLAR_JITTER_NS"] = jitter
    env.setdefault("POLAR_TIMEOUT_MS", "60000")
    env["POLAR_BOUNCE"] = str(1 << 20)   # small bounce buffer: exercise the chunked bounce path
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "mp_worker.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    res = json.loads(out.read_text())
    bad = [x for x in res if not (x["ok"] and x["identical"])]
    assert not bad, bad
    assert len(res) == nranks * (1 + 4 * 3 * 3 + 3 + 4 + 1 + 1 + 6 + 3 * 5 + 1 + 1)


def test_multiprocess_north_star_size_c2(tmp_path):
    """the north_star call at its own size — polar_allreduce on
    128 MiB f32 per rank (C2's largest), 3 processes on CUDA IPC: registered
    (zero-copy two-shot) and unregistered (bounce) buffers under the default
    table, forced ring / tree Simple at 32 channels, back-to-back mixes, a
    stale (freed) registration, deregistration, auto-registration (rank-dependent
    and unaligned offsets, mapping cache, a freed allocation, CUDA-graph
    capture, a refused mismatched configuration), and a path mismatch that must
    latch ESTATE before any data moves (tests/mp_worker_c2.py)."""
    out = tmp_path / "c2.json"
    env = dict(os.environ)
    env.setdefault("POLAR_TIMEOUT_MS", "120000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "mp_worker_c2.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-4000:]
    res = json.loads(out.read_text())
    bad = [x for x in res if not (x["ok"] and x["identical"])]
    assert not bad, bad
    tags = {x["tag"] for x in res}
    assert {"c2/registered/policy", "c2/unregistered/policy", "c2/ring/simple/32ch", "c2/tree/simple/32ch",
            "c2/after-free", "c2/deregistered", "path-mismatch-latched-before-data",
            "autoreg/mismatch-refused", "autoreg/first", "autoreg/again", "autoreg/b2b-other", "autoreg/stats",
            "autoreg/unaligned", "autoreg/after-free", "autoreg/graph-replay0", "autoreg/graph-replay1",
            "autoreg/graph-captured"} <= tags
    dec = {x["tag"]: x["decision"] for x in res if "decision" in x}
    assert dec["c2/registered/policy"][:2] == ["twoshot", "simple"]
    assert dec["c2/unregistered/policy"][:2] == ["twoshot", "simple"]
    assert dec["autoreg/first"][:2] == ["twoshot", "simple"]
    # R2 headroom of the f32 ring / tree results (reported, asserted <= 1 above)
    print({x["tag"]: round(x["max_err_over_bound"], 4) for x in res if x["rank"] == 0 and "max_err_over_bound" in x})


def test_tune_policy_real_ranks(tmp_path):
    """scripts/tune_policy.py --real: one process per rank,
    device time max over ranks, identical call counts on every rank; writes a
    table polar_set_policy accepts, with the best single choice (E10)."""
    out = tmp_path / "tuned.json"
    env = dict(os.environ, POLAR_TIMEOUT_MS="60000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "scripts", "tune_policy.py"),
           "--real", "--sizes", "4096,262144", "--nch", "2,4", "--combos", "oneshot/ll,twoshot/simple,ring/ll128",
           "--out", str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    doc = json.loads(out.read_text())
    assert doc["set_policy_status"] == "ok" and doc["rows"][-1][2] == 2**64 - 1
    assert doc["best_single"] and doc["ll128_probe"]["torn_lanes"] == 0
    assert set(doc["winners"]) == {"4096", "262144"}


@pytest.mark.parametrize("vmm_rank", [None, "1"])
def test_multiprocess_autoreg_cache_and_agreement(tmp_path, vmm_rank):
    """polar_comm_autoreg beyond the C2 test: 40 live buffers in separate
    allocations (the 32-per-peer mapping cache evicts, re-opens on reuse), and
    one rank allocating from VMM memory (expandable segments: not
    IPC-exportable) so that every rank bounces those calls; results bit-exact
    against the oracle (tests/mp_worker_autoreg.py)."""
    out = tmp_path / "ar.json"
    env = dict(os.environ)
    env.setdefault("POLAR_TIMEOUT_MS", "60000")
    if vmm_rank is not None:
        env["POLAR_TEST_VMM_RANK"] = vmm_rank
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "mp_worker_autoreg.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    res = json.loads(out.read_text())
    bad = [x for x in res if not x["ok"]]
    assert not bad, bad
    tags = {x["tag"] for x in res}
    assert ({"cache/stats", "mixed-registration/auto", "decision-mismatch/estate"} <= tags) if vmm_rank is None \
        else ("vmm/stats" in tags)


@pytest.mark.parametrize("jitter", ["0", "3000"])
def test_multiprocess_random_stress(tmp_path, jitter):
    """Time-bounded random stress of the real-comm path (3 processes, CUDA IPC):
    forced algorithm x protocol or policy-selected, registered / unregistered /
    auto-registered buffers, back-to-back batches; every result bit-exact
    (tests/mp_worker_stress.py)."""
    out = tmp_path / "stress.json"
    env = dict(os.environ)
    env.setdefault("POLAR_TIMEOUT_MS", "60000")
    env.setdefault("POLAR_STRESS_S", "40")
    env["POLAR_JITTER_NS"] = jitter
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "mp_worker_stress.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-4000:]
    rep = json.loads(out.read_text())
    assert all(x["calls"] == rep[0]["calls"] and x["calls"] > 0 for x in rep)
    bad = [b for x in rep for b in x["bad"]]
    assert not bad, bad[:20]
    print({"calls": rep[0]["calls"], "kinds": len(rep[0]["kinds"])})
