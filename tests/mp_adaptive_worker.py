"""One rank of a 2-process closed-loop run: each rank's controller closes its
windows at the same call indices, gathers the window means of all ranks through
the bootstrap all-gather and must launch the same channel count every call."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402

CAP, PERIOD, NWIN = 6, 4, 8


def main():
    out_path = sys.argv[1]
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank if torch.cuda.device_count() > rank else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")

    def allgather(b):
        o = [None] * ws
        dist.all_gather_object(o, b)
        return o

    comm = L.Comm.init(ws, rank, dev, allgather)
    L.set_policy([(0, 0, 2**64 - 1, L.TWOSHOT, L.SIMPLE, CAP, L.ROW_ADAPTIVE_NCH)])
    comm.adaptive_config(enabled=True, period=PERIOD, c_min=2, contention_factor=4.0)
    (buf,) = comm.mem_alloc_tensors(1 << 18, torch.float32)
    trace, ok = [], True
    for i in range(PERIOD * NWIN):
        buf.fill_(float(rank + 1))
        comm.allreduce(buf)
        torch.cuda.synchronize()
        ok = ok and bool((buf == ws * (ws + 1) / 2).all())
        trace.append(comm.launched_channels())
    comm.check()
    rep = {"rank": rank, "trace": trace, "ok": ok, "cap": CAP}
    allrep = [None] * ws
    dist.all_gather_object(allrep, rep)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allrep, f)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
