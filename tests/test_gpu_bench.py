"""The bench contract end to end on the GPU box: the N=1 line and the N>1
torchrun path (one process per rank, CUDA-IPC peers, device timing max over
ranks) — the latter with every rank on GPU 0 (POLAR_BENCH_SHARE_GPU=1; NCCL's
baseline is skipped because NCCL refuses two ranks on one GPU)."""
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
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_torchrun_two_ranks_shared_gpu():
    env = dict(os.environ, POLAR_BENCH_SHARE_GPU="1", POLAR_TIMEOUT_MS="20000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "5", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    d = _line(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 2 and d["config"]["nranks"] == 2 and d["config"]["shared_gpu_test"]
    assert d["value"] > 0 and d["gpu_launches"] == 5
    assert d["decision"]["algo"] == "twoshot"
    assert d["roofline"]["bound"] == "nvlink" and d["roofline"]["hbm"]["bound"] == "hbm"
    assert d["e2e"]["h2d_bytes_per_step"] == d["config"]["bytes_per_rank"]
    # the timed buffers were re-filled and checked against the oracle
    assert d["parity"]["ok"] and d["parity"]["ranks_identical"], d["parity"]
    # N > 1 sweep schema (NCCL cleanly skipped on a shared GPU)
    sw = d["nvlink_sweep"]
    assert "nccl_default" not in sw["variants"] and "bad_channels" in sw["variants"]
    assert str(4 << 10) in sw["sizes"] and str(16 << 20) in sw["sizes"]
    for rec in sw["sizes"].values():
        # (time-sliced ranks on one GPU: tiny sizes take ~ms, so only positivity is checked)
        assert rec["polar_us"] > 0 and rec["polar_busbw_gbs"] >= 0 and rec["bad_channels_decision"][2] == 1
        assert "nccl_busbw_gbs" not in rec and 0 <= rec["nvlink_frac"]
    assert "speedup_vs_nccl" not in d and "cpu_model" in d["cpu_baseline"]
    assert d["e2e"]["pcie"]["floor_ms"] > 0


def test_bench_single_gpu_line():
    """N = 1 (the driver's default run): the line carries parity, the L2-labelled
    C2 sweep, the 4 KiB - 1 GiB size sweep (active and tuned tables), the
    PCIe-bounded e2e and the CPU model."""
    env = dict(os.environ, POLAR_TIMEOUT_MS="20000")
    r = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    d = _line(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["parity"]["ok"] and d["parity"]["ranks_identical"]
    assert d["roofline"]["bound"] == "hbm" and d["gpu_launches"] == 5
    for sz, rec in d["c2_sweep"].items():
        assert rec["l2"].startswith("flushed") == (8 * int(sz) <= 2 * (126 << 20))
    # north_star's size range at N = 1: 4 KiB - 1 GiB, active table and the tuned virtual table
    for series in (d["size_sweep"]["sizes"], d["size_sweep"]["tuned_virtual"]["sizes"]):
        assert [int(k) for k in series] == [(4 << 10) << (2 * k) for k in range(10)]
        for sz, rec in series.items():
            bus = 2 * 7 / 8 * int(sz) / (rec["us"] * 1e-6) / 1e9      # busBW = S * 2(n-1)/n / t
            assert rec["us"] > 0 and abs(rec["busbw_gbs"] - bus) <= 0.01 + 1e-3 * bus, (sz, rec)
            assert abs(rec["algbw_gbs"] - bus / 1.75) <= 0.01 + 1e-3 * bus, (sz, rec)
            assert rec["l2"].startswith("flushed") == (8 * int(sz) <= 2 * (126 << 20))


def test_nccl_variants_script():
    """scripts/nccl_variants.py: every rank on one GPU -> each variant reports a
    clean skip; one rank -> the ctypes NCCL path runs end to end (its TUNING
    log parsed) on this box."""
    r = subprocess.run([sys.executable, "scripts/nccl_variants.py", "--gpus", "2", "--variants", "default,Ring/LL",
                        "--sizes", "4096,1048576"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    recs = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert [x["variant"] for x in recs] == ["default", "Ring/LL"] and all("share a GPU" in x["skipped"] for x in recs)
    r = subprocess.run([sys.executable, "scripts/nccl_variants.py", "--gpus", "1", "--variants", "default",
                        "--sizes", "4096,1048576"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    recs = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(recs) == 2 and all(x["us"] > 0 and x["nccl_version"].startswith("2.") for x in recs), recs
