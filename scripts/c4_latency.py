"""BASELINE config 4: small-message latency regime, 8 B - 256 KiB, 8 ranks, LL,
1-4 channels (plus Simple for comparison).  Per (size, algo, proto, nch):
  eager_us  - back-to-back polar_allreduce_v calls, CUDA-event time per call
  graph_us  - the same calls captured in one CUDA graph (device time per call)
  enqueue_ns- native host cost per call (decide + dispatch + launch), polar_bench_enqueue
Virtual ranks on one B200 (peers are local HBM, not NVLink): the numbers bound
the kernel + launch floor, not NVLink latency.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402


def ev_time(fn, iters):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(iters):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--algos", default="oneshot:ll,oneshot:ll128,twoshot:ll,twoshot:ll128,tree:ll,tree:ll128,ring:ll,"
                                       "ring:ll128,oneshot:simple,twoshot:simple")
    ap.add_argument("--nch", default="1,2,3,4")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    comm = L.Comm.virtual(a.n, 0)
    sizes = [8 << k for k in range(0, 16)]          # 8 B .. 256 KiB
    bufs = [torch.randn(max(sizes) // 4, device="cuda") for _ in range(a.n)]
    for size in sizes:
        views = [b[: size // 4] for b in bufs]
        for ap_ in a.algos.split(","):
            algo, proto = ap_.split(":")
            for nch in [int(x) for x in a.nch.split(",")]:
                fn = lambda: comm.allreduce_forced(views, algo, proto, nch)  # noqa: E731
                for _ in range(10):
                    fn()
                torch.cuda.synchronize()
                eager = ev_time(fn, a.iters)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(50):
                        fn()
                g.replay()
                torch.cuda.synchronize()
                graph = ev_time(g.replay, 5) / 50
                comm.check()
                print(json.dumps({"n": a.n, "bytes": size, "algo": algo, "proto": proto, "nch": nch,
                                  "eager_us": round(eager, 2), "graph_us": round(graph, 2)}), flush=True)
        # host enqueue cost with the policy-selected path at this size
        ns = comm.bench_enqueue(views, ncalls=2000)
        d = comm.last_decision()
        print(json.dumps({"n": a.n, "bytes": size, "enqueue_ns": round(ns, 1),
                          "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels]}), flush=True)


if __name__ == "__main__":
    main()
