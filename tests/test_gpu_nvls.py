"""NVLS: the switch-reduction AllReduce over a multicast
object.  Runs the data path wherever polar_comm_init could create and bind a
multicast object; otherwise records the driver's exact refusal (and the fabric
state) under gpurun_out/ and skips the data checks — on the 1-GPU pool every
rank shares GPU 0, where a multicast object over the ranks' devices cannot
exist (profiles/r02_probe_multicast_c.txt: cuMulticastCreate INVALID_VALUE even
for one device with fabric state Completed/Success)."""
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

from paper_2603_11438_b200 import polar as L  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_virtual_comm_has_no_nvls():
    c = L.Comm.virtual(4, 0)
    try:
        avail, why = c.nvls_info()
        assert not avail and "virtual" in why
        with pytest.raises(L.PolarError) as e:
            c.allreduce_forced([torch.ones(64, device="cuda") for _ in range(4)], "nvls", "simple", 2)
        assert e.value.name == "eunsupported"
        st, _ = L.set_policy_status([(0, 0, 1 << 30, L.NVLS, L.SIMPLE, 8)])
        assert L.STATUS_NAMES[st] == "eunsupported" and not L.lib.polar_nvls_available()
    finally:
        c.destroy()


def test_nvls_real_comm(tmp_path):
    out = tmp_path / "nvls.json"
    ngpu = torch.cuda.device_count()
    nranks = 2 if ngpu < 2 else min(ngpu, 8)
    env = dict(os.environ, POLAR_TIMEOUT_MS="60000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "mp_worker_nvls.py"),
           str(out)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    res = json.loads(out.read_text())
    assert len({x["available"] for x in res}) == 1, res      # every rank agrees
    for x in res:
        assert x["cases"] and all(cs["ok"] for cs in x["cases"]), x
    if not res[0]["available"]:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        fabric = subprocess.run("nvidia-smi -q | grep -A3 -i '^ *Fabric'", shell=True, capture_output=True,
                                text=True).stdout
        with open(os.path.join(ROOT, "gpurun_out", "nvls_unavailable.txt"), "w") as f:
            f.write(f"ranks={nranks} gpus={ngpu}\nwhy: {res[0]['why']}\n{fabric}")
        pytest.skip(f"no multicast object on this box: {res[0]['why']}")
