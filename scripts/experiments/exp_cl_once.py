"""Two cluster-ring calls (8 virtual ranks, f32) for an ncu capture of the second."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

n, mib = 8, int(os.environ.get("CL_MIB", "32"))
algo = os.environ.get("CL_ALGO", "ring")
dt = torch.float32 if os.environ.get("CL_DT", "f32") == "f32" else torch.bfloat16
comm = L.Comm.virtual(n, 0)
cnt = (mib << 20) // (4 if dt == torch.float32 else 2)
bufs = [torch.randn(cnt, device="cuda").to(dt) for _ in range(n)]
for _ in range(2):
    comm.allreduce_forced(bufs, algo, "simple", 32)
torch.cuda.synchronize()
comm.check()
print("ok", comm.launched_channels())
