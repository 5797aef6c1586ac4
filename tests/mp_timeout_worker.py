"""Failure detection: rank 1 skips one AllReduce; rank 0's kernel
must stop waiting after POLAR_TIMEOUT_MS, latch POLAR_ETIMEOUT in the comm, and
return control (no hang, no __trap).  Rank 0 writes a JSON report."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402


def main():
    out_path, algo, proto = sys.argv[1], sys.argv[2], sys.argv[3]
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank if torch.cuda.device_count() > rank else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")

    def allgather(b):
        o = [None] * ws
        dist.all_gather_object(o, b)
        return o

    comm = L.Comm.init(ws, rank, dev, allgather)
    t = torch.ones(100_000, device="cuda")
    comm.allreduce_forced(t, algo, proto, 2)          # a healthy call first
    torch.cuda.synchronize()
    comm.check()
    ok_first = bool((t == ws).all())
    rep = {"rank": rank, "first_ok": ok_first}
    dist.barrier()
    if rank == 0:
        t0 = time.time()
        st = None
        comm.allreduce_forced(t, algo, proto, 2)      # rank 1 never joins
        torch.cuda.synchronize()
        try:
            comm.check()
            st = "ok"
        except L.PolarError as e:
            st = e.name
        rep.update({"status": st, "seconds": round(time.time() - t0, 2)})
        # the comm stays latched: the next call reports the error without launching
        try:
            comm.allreduce_forced(t, algo, proto, 2)
            rep["next_call"] = "ok"
        except L.PolarError as e:
            rep["next_call"] = e.name
    dist.barrier()
    allrep = [None] * ws
    dist.all_gather_object(allrep, rep)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allrep, f)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
