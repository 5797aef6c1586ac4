"""One cluster-transport case for compute-sanitizer triage: CL_N ranks, CL_DT, CL_ALGO, CL_COUNT."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402
from tests.gpu_common import to_device, to_host  # noqa: E402

n = int(os.environ.get("CL_N", "3"))
dtype = os.environ.get("CL_DT", "bf16")
algo = os.environ.get("CL_ALGO", "ring")
count = int(os.environ.get("CL_COUNT", "1300000"))
c = L.Comm.virtual(n, 0)
xs = synth.gen_ranks(dtype, count, n, cfg=8, dist="ints")
ts = [to_device(x, dtype) for x in xs]
c.allreduce_forced(ts, algo, "simple", 3)
torch.cuda.synchronize()
c.check()
ok = all(np.array_equal(to_host(t, dtype), orc.allreduce(xs, dtype, "sum")) for t in ts)
print("case", n, dtype, algo, count, c.transport(), "ok" if ok else "MISMATCH", flush=True)
