"""The cluster section of scripts/sanitize_subset.py alone (triage)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402
from tests.gpu_common import to_device, to_host  # noqa: E402
bad = 0
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
print("bad", bad)
