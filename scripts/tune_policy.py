"""Derive a measured policy table for virtual ranks on this B200 (device time,
CUDA-graph replay): every (algorithm, protocol, channels) at sizes 8 B-256 MiB,
best per size, merged into first-match rows (inclusive max_bytes = the last
measured size of a run of equal winners).  JSON lines: one per measurement,
then {"table": ...} per rank count.

python scripts/tune_policy.py --n 2,4,8 > gpurun_out/tune.jsonl
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

COMBOS = [(a, p) for a in ("oneshot", "twoshot", "ring", "tree") for p in ("ll", "ll128", "simple")]


def graph_time(fn, reps):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(3):
        g.replay()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / (3 * reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="2,4,8")
    ap.add_argument("--sizes", default=",".join(str(8 << (2 * k)) for k in range(13)))   # 8 B .. 128 MiB
    ap.add_argument("--nch", default="1,2,4,8,16,32")
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    sizes = [int(x) for x in a.sizes.split(",")]
    for n in [int(x) for x in a.n.split(",")]:
        comm = L.Comm.virtual(n, 0)
        bufs = [torch.randn(max(sizes) // 4, device="cuda") for _ in range(n)]
        best = {}
        for size in sizes:
            v = [b[: size // 4] for b in bufs]
            for algo, proto in COMBOS:
                for nch in [int(x) for x in a.nch.split(",")]:
                    fn = lambda: comm.allreduce_forced(v, algo, proto, nch)  # noqa: E731
                    fn()
                    torch.cuda.synchronize()
                    comm.check()
                    launched = comm.launched_channels()
                    t1 = graph_time(fn, 1)
                    if t1 > 0.02:
                        continue
                    reps = max(1, min(50, int(0.01 / max(t1, 1e-6))))
                    t = graph_time(fn, reps)
                    print(json.dumps({"n": n, "bytes": size, "algo": algo, "proto": proto, "nch": nch,
                                      "launched": launched, "us": round(t * 1e6, 2),
                                      "busbw_gbs": round(size * 2 * (n - 1) / n / t / 1e9, 2)}), flush=True)
                    if size not in best or t < best[size][0]:
                        best[size] = (t, algo, proto, nch)
        rows = []
        for size in sizes:
            _, algo, proto, nch = best[size]
            code = (L.ALGO_CODES[algo], L.PROTO_CODES[proto], nch)
            if rows and tuple(rows[-1][3:]) == code:
                rows[-1][2] = size
            else:
                rows.append([0, n, size, *code])
        rows[-1][2] = 2**64 - 1
        print(json.dumps({"n": n, "table": rows,
                          "winners": {s: [best[s][1], best[s][2], best[s][3], round(best[s][0] * 1e6, 2)] for s in sizes}}),
              flush=True)
        del bufs
        comm.destroy()


if __name__ == "__main__":
    main()
