"""Why does bench.py time 128 MiB two-shot slower than sweep.py?  Same process,
same comm: (allocator: polar_mem_alloc vs torch) x (NVML clock sampler on/off)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402

n, count = 8, (128 << 20) // 4
comm = L.Comm.virtual(n, 0)
sym = comm.mem_alloc_tensors(count, torch.float32)
tor = [torch.empty(count, device="cuda") for _ in range(n)]
for b in sym + tor:
    b.uniform_(-1, 1)
s = torch.cuda.current_stream()


def timeit(bufs, steps, sampler):
    ptrs = [b.data_ptr() for b in bufs]
    for _ in range(5):
        comm.allreduce_raw(ptrs, count, L.FLOAT32, L.SUM, s.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    a.record(s)
    for _ in range(steps):
        comm.allreduce_raw(ptrs, count, L.FLOAT32, L.SUM, s.cuda_stream)
    b.record(s)
    b.synchronize()
    if ctx:
        ctx.__exit__()
    return a.elapsed_time(b) * 1e3 / steps


for rep in range(2):
    for name, bufs in (("mem_alloc", sym), ("torch", tor)):
        for steps in (50, 200):
            for smp in (False, True):
                print(json.dumps({"rep": rep, "alloc": name, "steps": steps, "sampler": smp,
                                  "us": round(timeit(bufs, steps, smp), 2)}), flush=True)
