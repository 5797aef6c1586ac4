"""Forced-decision sweep on virtual ranks: device time per call for every
(algorithm, protocol, channels) at every size; JSON lines to stdout.

python scripts/sweep.py --n 8 --dtype f32 --sizes 4K,64K,1M,4M,16M,128M --nch 4,16,32
Used to derive the tuned policy table (policies/*.json) and for BASELINE
config 3 sweeps.  Timing: CUDA events on the launching stream around K calls
after W warm-ups; inputs are resident (no L2 flush between calls for sizes
whose n buffers exceed L2; smaller sizes are reported as L2-warm).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

ES = {"i32": 4, "i64": 8, "f32": 4, "bf16": 2}
TD = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "bf16": torch.bfloat16}


def parse_size(s):
    s = s.strip().upper()
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    if s[-1] in mult:
        return int(float(s[:-1]) * mult[s[-1]])
    return int(s)


def time_calls(fn, warm, iters):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(iters):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--sizes", default="4K,64K,256K,1M,4M,16M,64M,128M")
    ap.add_argument("--algos", default="oneshot:ll,oneshot:simple,twoshot:ll,twoshot:simple,ring:ll,ring:simple,tree:ll,tree:simple")
    ap.add_argument("--nch", default="1,4,8,16,32")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warm", type=int, default=5)
    ap.add_argument("--max-time", type=float, default=0.05, help="skip configs slower than this (s/call)")
    ap.add_argument("--graph", action="store_true", help="time K calls captured in one CUDA graph (device time, no host launch cost)")
    args = ap.parse_args()
    n, dt = args.n, args.dtype
    comm = L.Comm.virtual(n, 0)
    sizes = [parse_size(x) for x in args.sizes.split(",")]
    bufs = [torch.zeros(max(sizes) // ES[dt], dtype=TD[dt], device="cuda") for _ in range(n)]
    for b in bufs:
        b.normal_() if dt in ("f32", "bf16") else b.random_(-100, 100)
    for size in sizes:
        count = size // ES[dt]
        views = [b[:count] for b in bufs]
        for ap_ in args.algos.split(","):
            algo, proto = ap_.split(":")
            for nch in [int(x) for x in args.nch.split(",")]:
                fn = lambda: comm.allreduce_forced(views, algo, proto, nch)  # noqa: E731
                t1 = time_calls(fn, 1, 1)
                if t1 > args.max_time:
                    print(json.dumps({"n": n, "dtype": dt, "bytes": size, "algo": algo, "proto": proto, "nch": nch,
                                      "skipped": f"{t1*1e6:.0f} us"}), flush=True)
                    continue
                iters = max(3, min(args.iters, int(0.2 / max(t1, 1e-6))))
                if args.graph:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        for _ in range(iters):
                            fn()
                    t = time_calls(g.replay, 2, 3) / iters
                else:
                    t = time_calls(fn, args.warm, iters)
                comm.check()
                bus = size * 2 * (n - 1) / n / t / 1e9
                hbm = 2 * n * size / t / 1e9
                print(json.dumps({"n": n, "dtype": dt, "bytes": size, "algo": algo, "proto": proto,
                                  "nch": comm.launched_channels(), "us": round(t * 1e6, 2),
                                  "busbw_gbs": round(bus, 1), "min_hbm_gbs": round(hbm, 1)}), flush=True)


if __name__ == "__main__":
    main()
