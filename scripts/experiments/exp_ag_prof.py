"""Diagnostic: cluster ring all-gather warp time split (build -DPOLAR_CL_PROF=1):
ns spent [0] issuing / waiting for the predecessor's count, [1] waiting for my
final tiles, [2] waiting for pulled tiles, [3] stalled on the predecessor."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

for n in (2, 8):
    comm = L.Comm.virtual(n, 0)
    for mib in (1, 8):
        cnt = (mib << 20) // 4
        bufs = [torch.randn(cnt, device="cuda") for _ in range(n)]
        tr = torch.zeros(n * 32 * 8, dtype=torch.int64, device="cuda")
        comm.allreduce_forced(bufs, "ring", "simple", 32)
        comm.set_trace(tr)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        comm.allreduce_forced(bufs, "ring", "simple", 32)
        b.record()
        torch.cuda.synchronize()
        comm.set_trace(None)
        nch = comm.launched_channels()
        t = tr.view(-1, 8)[: n * nch].cpu().double() / 1e3
        print(json.dumps({"n": n, "mib": mib, "us": round(a.elapsed_time(b) * 1e3, 1), "nch": nch,
                          "split_us_mean": [round(float(x), 1) for x in t.mean(0)],
                          "split_us_max": [round(float(x), 1) for x in t.max(0).values]}), flush=True)
    comm.destroy()
