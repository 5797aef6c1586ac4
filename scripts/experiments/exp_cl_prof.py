"""Diagnostic: per-CTA cycles of the cluster ring's compute warp 1 spent waiting
for `full` / own / `empty` and working (build with -DPOLAR_CL_PROF=1)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

n = 8
comm = L.Comm.virtual(n, 0)
for mib in (8, 128):
    cnt = (mib << 20) // 4
    bufs = [torch.randn(cnt, device="cuda") for _ in range(n)]
    tr = torch.zeros(n * 32 * 4, dtype=torch.int64, device="cuda")
    for _ in range(3):
        comm.allreduce_forced(bufs, "ring", "simple", 32)
    comm.set_trace(tr)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    comm.allreduce_forced(bufs, "ring", "simple", 32)
    b.record()
    torch.cuda.synchronize()
    comm.set_trace(None)
    nch = comm.launched_channels()
    t = tr.view(-1, 4)[: n * nch].cpu().double() / 1.9e3   # us at ~1.9 GHz
    print(json.dumps({"mib": mib, "us": round(a.elapsed_time(b) * 1e3, 1), "nch": nch,
                      "full_us": [round(float(x), 1) for x in (t[:, 0].min(), t[:, 0].mean(), t[:, 0].max())],
                      "own_us": [round(float(x), 1) for x in (t[:, 1].min(), t[:, 1].mean(), t[:, 1].max())],
                      "empty_us": [round(float(x), 1) for x in (t[:, 2].min(), t[:, 2].mean(), t[:, 2].max())],
                      "work_us": [round(float(x), 1) for x in (t[:, 3].min(), t[:, 3].mean(), t[:, 3].max())]}),
          flush=True)
