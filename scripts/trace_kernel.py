"""Per-CTA timeline of one AllReduce launch (diagnostic; polar_comm_set_trace).

python scripts/trace_kernel.py --n 8 --mib 128 --algo twoshot --proto simple --nch 16
Prints start skew, barrier waits and the loop-time spread across CTAs.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--mib", type=float, default=128)
    ap.add_argument("--algo", default="twoshot")
    ap.add_argument("--proto", default="simple")
    ap.add_argument("--nch", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    comm = L.Comm.virtual(a.n, 0)
    count = int(a.mib * (1 << 20)) // 4
    bufs = [torch.randn(count, device="cuda") for _ in range(a.n)]
    tr = torch.zeros(a.n * 32 * 4, dtype=torch.int64, device="cuda")
    for _ in range(3):
        comm.allreduce_forced(bufs, a.algo, a.proto, a.nch)
    torch.cuda.synchronize()
    comm.set_trace(tr)
    for rep in range(a.reps):
        tr.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        comm.allreduce_forced(bufs, a.algo, a.proto, a.nch)
        e1.record()
        torch.cuda.synchronize()
        nch = comm.launched_channels()
        t = tr.view(-1, 4)[: a.n * nch].cpu().double()
        base = t[:, 0].min()
        t = (t - base) / 1e3   # us
        loop = t[:, 2] - t[:, 1]
        rep_ = {
            "event_us": round(e0.elapsed_time(e1) * 1e3, 1),
            "span_us": round(float(t[:, 3].max()), 1),
            "start_skew_us": round(float(t[:, 0].max()), 2),
            "entry_wait_us_med": round(float((t[:, 1] - t[:, 0]).median()), 2),
            "entry_wait_us_max": round(float((t[:, 1] - t[:, 0]).max()), 2),
            "loop_us_min": round(float(loop.min()), 1), "loop_us_med": round(float(loop.median()), 1),
            "loop_us_max": round(float(loop.max()), 1),
            "loop_end_us_min": round(float(t[:, 2].min()), 1), "loop_end_us_max": round(float(t[:, 2].max()), 1),
            "exit_wait_us_max": round(float((t[:, 3] - t[:, 2]).max()), 1),
            "nch": nch, "mib": a.mib,
            # per rank (owner): earliest and latest loop end of its CTAs (virtual
            # comms: block b = rank b / nch)
            "owner_loop_end_us": [[round(float(t[r * nch:(r + 1) * nch, 2].min()), 1),
                                   round(float(t[r * nch:(r + 1) * nch, 2].max()), 1)] for r in range(a.n)],
        }
        print(json.dumps(rep_), flush=True)
    # inter-kernel gap: two back-to-back launches traced into separate buffers
    tr2 = torch.zeros_like(tr)
    comm.set_trace(tr)
    comm.allreduce_forced(bufs, a.algo, a.proto, a.nch)
    comm.set_trace(tr2)
    comm.allreduce_forced(bufs, a.algo, a.proto, a.nch)
    torch.cuda.synchronize()
    nch = comm.launched_channels()
    t1 = tr.view(-1, 4)[: a.n * nch].cpu().double()
    t2 = tr2.view(-1, 4)[: a.n * nch].cpu().double()
    print(json.dumps({"gap_us": round(float(t2[:, 0].min() - t1[:, 3].max()) / 1e3, 2),
                      "span1_us": round(float(t1[:, 3].max() - t1[:, 0].min()) / 1e3, 1)}), flush=True)
    comm.set_trace(None)


if __name__ == "__main__":
    main()
