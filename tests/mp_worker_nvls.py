"""One rank of a real comm exercising NVLS, launched by
torchrun.  Records whether polar_comm_init could create and bind a multicast
object (and the driver's exact refusal if not); where it could, checks the
switch-reduced AllReduce against the oracle: integers exact, f32 sum within
R2's bound (the switch's summation order is unspecified), bf16 within 1e-2
relative (f32 accumulation, one rounding), f32 max refused.  Rank 0 writes JSON."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402
from tests.gpu_common import to_device, to_host  # noqa: E402


def main():
    out_path = sys.argv[1]
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")

    def allgather(b):
        o = [None] * ws
        dist.all_gather_object(o, b)
        return o

    comm = L.Comm.init(ws, rank, dev, allgather)
    avail, why = comm.nvls_info()
    res = {"rank": rank, "available": avail, "why": why, "process_available": bool(L.lib.polar_nvls_available()),
           "cases": []}
    if avail:
        for dtype, dist_, count, nch in (("i32", "full", 1_000_003, 8), ("i64", "full", 70_001, 4),
                                          ("f32", "unif", (64 << 20) // 4 + 5, 32), ("bf16", "normal", 3_000_001, 16)):
            xs = synth.gen_ranks(dtype, count, ws, cfg=70, dist=dist_)
            t = to_device(xs[rank], dtype)
            comm.allreduce_forced(t, "nvls", "simple", nch)
            torch.cuda.synchronize()
            comm.check()
            got = to_host(t, dtype)
            exp = orc.allreduce(xs, dtype, "sum")
            if dtype in ("i32", "i64"):
                ok = bool(np.array_equal(got, exp))
            elif dtype == "f32":
                bound = 1e-6 * ws * np.sum(np.abs(np.stack(xs).astype(np.float64)), axis=0)
                ok = bool(np.all(np.abs(got.astype(np.float64) - exp) <= bound))
            else:
                y, ys = orc.bf16_bits_to_f32(got).astype(np.float64), orc.bf16_bits_to_f32(exp).astype(np.float64)
                ok = bool(np.all(np.abs(y - ys) <= 1e-2 * np.abs(ys)))
            res["cases"].append({"dtype": dtype, "count": count, "ok": ok})
        # policy row accepted now that a multicast object exists, and used
        gen = L.set_policy([(0, 0, 2**64 - 1, L.NVLS, L.SIMPLE, 16)])
        xs = synth.gen_ranks("i32", 4096, ws, cfg=71, dist="full")
        t = to_device(xs[rank], "i32")
        comm.allreduce(t)
        torch.cuda.synchronize()
        res["cases"].append({"dtype": "i32/policy", "ok": bool(np.array_equal(to_host(t, "i32"),
                                                                             orc.allreduce(xs, "i32", "sum")))
                             and comm.last_decision().algo == L.NVLS and gen > 0})
        L.set_policy([])
        try:
            comm.allreduce_forced(torch.ones(100, device="cuda"), "nvls", "simple", 1, op="max")
            refused = False
        except L.PolarError as e:
            refused = e.name == "eunsupported"
        res["cases"].append({"dtype": "f32/max", "ok": refused})
    else:
        # no multicast object: NVLS decisions are refused, NVLS rows too
        try:
            comm.allreduce_forced(torch.ones(100, device="cuda"), "nvls", "simple", 1)
            refused = False
        except L.PolarError as e:
            refused = e.name == "eunsupported"
        st, _ = L.set_policy_status([(0, 0, 2**64 - 1, L.NVLS, L.SIMPLE, 16)])
        res["cases"].append({"dtype": "refused", "ok": refused and L.STATUS_NAMES[st] == "eunsupported"})
    comm.destroy()
    allres = allgather(res)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allres, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
