"""Cooperative vs plain launch for virtual comms (POLAR_VIRTUAL_COOP): host
enqueue cost, back-to-back device time per call, inter-kernel gap."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

n = 8
comm = L.Comm.virtual(n, 0)
bufs = [torch.randn((128 << 20) // 4, device="cuda") for _ in range(n)]
s = torch.cuda.current_stream()
out = {"coop": os.environ.get("POLAR_VIRTUAL_COOP", "1")}
for size in (8, 64 << 10, 1 << 20, 4 << 20, 16 << 20, 128 << 20):
    v = [b[: size // 4] for b in bufs]
    for _ in range(20):
        comm.allreduce(v)
    torch.cuda.synchronize()
    it = 200 if size < (16 << 20) else 50
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(it):
        comm.allreduce(v)
    b.record(s)
    b.synchronize()
    comm.check()
    out[str(size)] = {"us": round(a.elapsed_time(b) * 1e3 / it, 2), "enqueue_ns": round(comm.bench_enqueue(v, ncalls=500), 1)}
print(json.dumps(out), flush=True)
