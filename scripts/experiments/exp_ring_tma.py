"""A/B: ring / tree Simple on 8 virtual ranks, TMA-staged FIFOs vs the
warp-specialised LDG kernels (env knobs read at comm creation).  Device time
per call, back-to-back events; parity of each variant checked on integer
inputs (exact for every algorithm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

n = int(os.environ.get("AB_N", "8"))
algos = os.environ.get("AB_ALGOS", "ring").split(",")
# a variant = "K=V;K2=V2"; every variant starts from the same environment
variants = [[kv.split("=") for kv in v.split(";")] for v in
            os.environ.get("AB_VARIANTS", "POLAR_RING_TMA=0,POLAR_RING_TMA=1").split(",")]
BASE_ENV = dict(os.environ)
sizes = [int(x) << 20 for x in os.environ.get("AB_SIZES_MIB", "1,8,32,128").split(",")]
dts = os.environ.get("AB_DTYPES", "f32,bf16").split(",")
s = torch.cuda.current_stream()
maxb = max(sizes)
for var in variants:
    os.environ.clear()
    os.environ.update(BASE_ENV)
    for key, val in var:
        os.environ[key] = val
    vname = ";".join(f"{k}={v}" for k, v in var)
    comm = L.Comm.virtual(n, 0)
    bufs = comm.mem_alloc_tensors(maxb // 4, torch.float32)
    for algo in algos:
        for dt in dts:
            tdt = torch.float32 if dt == "f32" else torch.bfloat16
            for sz in sizes:
                cnt = sz // (4 if dt == "f32" else 2)
                views = [b.view(tdt)[:cnt] for b in bufs]
                for r, v in enumerate(views):
                    v.copy_(torch.randint(-8, 9, (cnt,), device="cuda").to(tdt) if dt == "bf16" else
                            torch.randint(-4096, 4097, (cnt,), device="cuda").to(tdt))
                exp = sum(v.double() for v in views)
                comm.allreduce_forced(views, algo, "simple", 32)
                torch.cuda.synchronize()
                comm.check()
                ok = all(bool(torch.equal(v.double(), exp)) for v in views)
                it = max(5, min(100, int(0.2 / max(1e-5, sz * n / 3e12))))
                for _ in range(3):
                    comm.allreduce_forced(views, algo, "simple", 32)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for _ in range(it):
                    comm.allreduce_forced(views, algo, "simple", 32)
                b.record(s)
                b.synchronize()
                comm.check()
                t = a.elapsed_time(b) / 1e3 / it
                print(json.dumps({"variant": vname, "algo": algo, "dtype": dt, "n": n, "bytes": sz,
                                  "us": round(t * 1e6, 1), "busbw_gbs": round(sz * 2 * (n - 1) / n / t / 1e9, 1),
                                  "hbm_frac": round(2 * n * sz / t / 6553.6e9, 3), "parity": ok,
                                  "launched_ch": comm.launched_channels()}), flush=True)
    comm.destroy()
