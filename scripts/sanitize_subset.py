"""Small parity subset for compute-sanitizer (memcheck / racecheck / synccheck):
every algorithm x protocol, f32 + bf16, ragged counts (ring / tree Simple up to
many FIFO slots per channel), 3 virtual ranks, the TMA
two-shot, the direct collectives and the p2p probe; exits non-zero on a mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402
from tests.gpu_common import to_device, to_host  # noqa: E402

n = 3
c = L.Comm.virtual(n, 0)
bad = 0
for dtype in ("f32", "bf16"):
    for algo in ("oneshot", "twoshot", "ring", "tree"):
        for proto in ("ll", "ll128", "simple"):
            # ring / tree Simple also at multi-slot sizes (warp-specialised kernels:
            # half-slot units, and the tree's whole-slot units beyond 4 slots per channel)
            for count in ((7, 5003, 300_001, 1_300_001) if proto == "simple" and algo in ("ring", "tree") else (7, 5003)):
                xs = synth.gen_ranks(dtype, count, n, cfg=5, dist="ints")
                ts = [to_device(x, dtype) for x in xs]
                c.allreduce_forced(ts, algo, proto, 2)
                torch.cuda.synchronize()
                c.check()
                exp = orc.allreduce(xs, dtype, "sum")
                ok = all(np.array_equal(to_host(t, dtype), exp) for t in ts)
                bad += 0 if ok else 1
                print(dtype, algo, proto, count, "ok" if ok else "MISMATCH", flush=True)
os.environ["POLAR_TWOSHOT_TMA"] = "1"
ct = L.Comm.virtual(n, 0)
xs = synth.gen_ranks("f32", 70_001, n, cfg=6, dist="ints")
ts = [to_device(x, "f32") for x in xs]
ct.allreduce_forced(ts, "twoshot", "simple", 2)
torch.cuda.synchronize()
ok = all(np.array_equal(to_host(t, "f32"), orc.allreduce(xs, "f32", "sum")) for t in ts)
bad += 0 if ok else 1
print("tma twoshot", "ok" if ok else "MISMATCH", flush=True)
# TMA-staged ring Simple (opt-in kernel; round 2), with and without L2 hints + discard
for flags in ("1", "3"):
    os.environ["POLAR_RING_TMA"] = "1"
    os.environ["POLAR_CLUSTER"] = "0"      # aligned sizes would run as clusters
    os.environ["POLAR_RING_TMA_FLAGS"] = flags
    cr = L.Comm.virtual(n, 0)
    for dtype in ("f32", "bf16"):
        for count in (300_001 * 4 // 4 * 4, 1_300_000):
            xs = synth.gen_ranks(dtype, count, n, cfg=7, dist="ints")
            ts = [to_device(x, dtype) for x in xs]
            cr.allreduce_forced(ts, "ring", "simple", 2)
            torch.cuda.synchronize()
            cr.check()
            ok = all(np.array_equal(to_host(t, dtype), orc.allreduce(xs, dtype, "sum")) for t in ts)
            bad += 0 if ok else 1
            print("ring tma", flags, dtype, count, "ok" if ok else "MISMATCH", flush=True)
    cr.destroy()
    del os.environ["POLAR_RING_TMA"], os.environ["POLAR_RING_TMA_FLAGS"], os.environ["POLAR_CLUSTER"]
# cluster transport (csrc/cluster.cuh): ring / tree Simple on aligned whole packs,
# DSMEM hops between the CTAs of a cluster; n = 3 and 8, multi-lap sizes
os.environ["POLAR_CLUSTER_TREE_MAX"] = str(1 << 40)
for nc in (3, 8):
    cc = L.Comm.virtual(nc, 0)
    for dtype in ("f32", "bf16"):
        for algo in ("ring", "tree"):
            for count in (5_008, 300_000, 1_300_000):
                xs = synth.gen_ranks(dtype, count, nc, cfg=8, dist="ints")
                ts = [to_device(x, dtype) for x in xs]
                cc.allreduce_forced(ts, algo, "simple", 3)
                assert cc.transport() == "cluster"
                torch.cuda.synchronize()
                cc.check()
                ok = all(np.array_equal(to_host(t, dtype), orc.allreduce(xs, dtype, "sum")) for t in ts)
                bad += 0 if ok else 1
                print("cluster", nc, dtype, algo, count, "ok" if ok else "MISMATCH", flush=True)
    cc.destroy()
del os.environ["POLAR_CLUSTER_TREE_MAX"]
sends = [torch.randn(n * 1000, device="cuda") for _ in range(n)]
recvs = [torch.empty(1000, device="cuda") for _ in range(n)]
c.reduce_scatter(sends, recvs)
c.all_gather(recvs, sends)
c.broadcast(sends, root=1)
probe = c.p2p_probe([torch.zeros(4096, device="cuda") for _ in range(n)], iters=2)
torch.cuda.synchronize()
c.check()
print("direct collectives + probe done", flush=True)
ct.destroy()
c.destroy()
sys.exit(1 if bad else 0)
