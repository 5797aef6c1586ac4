"""Does NCCL 2.28.9 load libpolar_nccl_tuner.so?  One-rank NCCL communicator
(the pool has one GPU) with NCCL_TUNER_PLUGIN pointing at the shim and NCCL's
INFO log captured: the log must show NCCL loading the plugin and, if NCCL asks
the tuner for this communicator, the shim's decisions."""
import ctypes as C
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
log = os.path.join(tempfile.gettempdir(), "nccl_tuner_load.log")
os.environ["NCCL_TUNER_PLUGIN"] = os.path.join(ROOT, "paper_2603_11438_b200", "libpolar_nccl_tuner.so")
os.environ["NCCL_DEBUG"] = "INFO"
os.environ["NCCL_DEBUG_SUBSYS"] = "ALL"
os.environ["NCCL_DEBUG_FILE"] = log
os.environ["POLAR_POLICY"] = os.path.join(ROOT, "policies", "nvlink_ring_mid_v2.json")
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import nccl_ctypes as N  # noqa: E402

torch.cuda.set_device(0)
n = N.Nccl()
comm = n.init(1, n.unique_id(), 0)
buf = torch.ones(1 << 20, device="cuda")
for sz in (4 << 10, 8 << 20, 64 << 20 // 4):
    n.allreduce(comm, buf.data_ptr(), min(sz, buf.numel()), N.NCCL_FLOAT32, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
n.destroy(comm)
text = open(log, errors="replace").read()
lines = [ln for ln in text.splitlines() if "tuner" in ln.lower() or "polar" in ln.lower()]
print("\n".join(lines[:40]))
print("LOADED" if any("polar" in ln for ln in lines) else "NOT LOADED")
