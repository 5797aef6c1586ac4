"""Experiment: the ring on 8 virtual ranks split between the cluster transport
(15 clusters = 120 SMs) and the FIFO ring on the SMs the clusters leave idle
(3 channels = 24 CTAs), concurrently on two streams over disjoint slices of the
message.  Device time of the fork/join per size and split; integer inputs, exact."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

n = 8
os.environ["POLAR_CLUSTER"] = "1"
ca = L.Comm.virtual(n, 0)
os.environ["POLAR_CLUSTER"] = "0"
cb = L.Comm.virtual(n, 0)
S = int(os.environ.get("HY_MIB", "128")) << 20
cnt = S // 4
bufs = [torch.randint(-1000, 1000, (cnt,), device="cuda").float() for _ in range(n)]
exp = sum(b.double() for b in bufs)
s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()
fch = int(os.environ.get("HY_FCH", "3"))


def call(f):
    ka = int(cnt * f) // 4 * 4
    ev = torch.cuda.Event()
    ev.record(s0)
    s1.wait_event(ev)
    if ka > 0:
        ca.allreduce_forced([b[:ka] for b in bufs], "ring", "simple", 32, stream=s0)
    if ka < cnt:
        cb.allreduce_forced([b[ka:] for b in bufs], "ring", "simple", fch, stream=s1)
    ev2 = torch.cuda.Event()
    ev2.record(s1)
    s0.wait_event(ev2)


for f in [float(x) for x in os.environ.get("HY_F", "1.0,0.95,0.92,0.9,0.88,0.85").split(",")]:
    for b, x in zip(bufs, [None] * n):
        pass
    src = [b.clone() for b in bufs]
    call(f)
    torch.cuda.synchronize()
    ok = all(torch.equal(b.double(), exp) for b in bufs)
    for b, x in zip(bufs, src):
        b.copy_(x)
    for _ in range(3):
        call(f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    e0.record(s0)
    for _ in range(it):
        call(f)
    e1.record(s0)
    e1.synchronize()
    ca.check()
    cb.check()
    t = e0.elapsed_time(e1) / 1e3 / it
    print(json.dumps({"f_cluster": f, "fifo_ch": fch, "bytes": S, "us": round(t * 1e6, 1),
                      "hbm_frac": round(2 * n * S / t / 6460.5e9, 4), "exact": ok,
                      "launched": [ca.launched_channels(), cb.launched_channels()]}), flush=True)
    for b, x in zip(bufs, src):
        b.copy_(x)
