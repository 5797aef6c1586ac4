"""Per-CTA timeline of the REAL-comm two-shot with every rank in its own process
on one GPU under MPS (run with torchrun + POLAR_BENCH-style env; see
scripts/gpu_mps_bench.sh for the MPS setup).  Rank 0 prints per-rank entry wait,
loop and exit wait (us, relative to the earliest CTA start of the call)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

dist.init_process_group("gloo")
ws, rank = dist.get_world_size(), dist.get_rank()
torch.cuda.set_device(0)


def ag(b):
    out = [None] * ws
    dist.all_gather_object(out, b)
    return out


comm = L.Comm.init(ws, rank, 0, ag)
nch = int(os.environ.get("NCH", "16"))
mib = float(os.environ.get("MIB", "128"))
count = int(mib * (1 << 20)) // 4
(buf,) = comm.mem_alloc_tensors(count, torch.float32)
buf.uniform_(-1, 1)
tr = torch.zeros(32 * 4, dtype=torch.int64, device="cuda")
for _ in range(5):
    comm.allreduce_forced(buf, "twoshot", "simple", nch)
torch.cuda.synchronize()
dist.barrier()
comm.set_trace(tr)
comm.allreduce_forced(buf, "twoshot", "simple", nch)
torch.cuda.synchronize()
comm.set_trace(None)
t = tr.view(-1, 4)[:nch].cpu().tolist()
allt = [None] * ws
dist.all_gather_object(allt, t)
if rank == 0:
    base = min(r[0] for tt in allt for r in tt)
    out = []
    for r, tt in enumerate(allt):
        start = [(x[0] - base) / 1e3 for x in tt]
        entry = [(x[1] - x[0]) / 1e3 for x in tt]
        loop = [(x[2] - x[1]) / 1e3 for x in tt]
        exitw = [(x[3] - x[2]) / 1e3 for x in tt]
        out.append({"rank": r, "start_us": [round(min(start), 1), round(max(start), 1)],
                    "entry_wait_us_max": round(max(entry), 1), "loop_us": [round(min(loop), 1), round(max(loop), 1)],
                    "exit_wait_us_max": round(max(exitw), 1), "end_us": round(max((x[3] - base) / 1e3 for x in tt), 1)})
    print(json.dumps({"n": ws, "nch": nch, "mib": mib, "ranks": out}), flush=True)
comm.destroy()
dist.destroy_process_group()
