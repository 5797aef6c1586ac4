"""One rank of a real (multi-process) comm exercising auto-registration
(polar_comm_autoreg) beyond the north_star-size test (tests/mp_worker_c2.py):

  * the mapping cache bound: 40 live buffers in separate allocations, each
    allreduced once (32 auto-opened mappings per peer are kept, the least
    recently used are closed), then the first ones again (re-opened);
  * agreement when one rank's buffer cannot be exported: the rank named by
    POLAR_TEST_VMM_RANK allocates with PyTorch's expandable segments (cuMem /
    VMM memory, no cudaIpcGetMemHandle), so every rank must take the bounce
    path for those calls (the choice depends on the gathered records only);
  * registrations are not consulted (rank 0 registered, the others not: one path);
  * the exchange as a synchronous decision check: rank 0 decides ring, the
    others two-shot — every rank returns ESTATE before anything is launched.

Every result is compared bitwise with the oracle (two-shot: rank-ordered fold,
bit-exact) on a window at each end and one in the middle.  Rank 0 writes JSON.
"""
import json
import os
import sys

RANK = int(os.environ["RANK"])
if os.environ.get("POLAR_TEST_VMM_RANK") == str(RANK):
    os.environ["PYTORCH_CUDA_ALLOC_CONF"] = "expandable_segments:True"   # before torch initialises CUDA

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402

COUNT = 3 << 20          # 12 MiB of f32: its own caching-allocator segment (> 10 MiB)
NBUF = 40


def main():
    out_path = sys.argv[1]
    ws = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")

    def allgather_obj(b):
        o = [None] * ws
        dist.all_gather_object(o, b)
        return o

    comm = L.Comm.init(ws, RANK, 0, L.torch_allgather(dist, ws))
    comm.autoreg(True, 1 << 20)
    stream = torch.cuda.current_stream()
    windows = [(0, 1024), (COUNT // 2, COUNT // 2 + 1024), (COUNT - 1027, COUNT)]
    results = []

    def ar(t):
        st = L.lib.polar_allreduce(comm.h, L.C.c_void_p(t.data_ptr()), t.numel(), L.FLOAT32, L.SUM,
                                   L.C.c_void_p(stream.cuda_stream))
        if st != L.OK:
            raise L.PolarError(st, "polar_allreduce")

    def inputs(k):
        return synth.gen("f32", COUNT, RANK, cfg=100 + k, dist="unif")

    def check(tag, t, k):
        got = t.cpu().numpy()
        mine = inputs(k)
        wins = allgather_obj([mine[lo:hi].copy() for lo, hi in windows])
        ok = True
        for w, (lo, hi) in enumerate(windows):
            exp = orc.allreduce([wins[p][w] for p in range(ws)], "f32", "sum")
            ok = ok and bool(np.array_equal(got[lo:hi].view(np.uint32), exp.view(np.uint32)))
        results.append({"tag": tag, "rank": RANK, "ok": ok})

    vmm = os.environ.get("POLAR_TEST_VMM_RANK")
    if vmm is None:
        # 1. the mapping cache bound
        bufs = [torch.from_numpy(inputs(k)).cuda() for k in range(NBUF)]
        for k, b in enumerate(bufs):
            ar(b)
        torch.cuda.synchronize()
        comm.check()
        for k in (0, 17, NBUF - 1):
            check(f"cache/first-pass/{k}", bufs[k], k)
        s1 = comm.autoreg_stats()
        for k in (0, 1):                      # closed (least recently used): opened again
            bufs[k].copy_(torch.from_numpy(inputs(k)))
            ar(bufs[k])
        torch.cuda.synchronize()
        comm.check()
        for k in (0, 1):
            check(f"cache/reopened/{k}", bufs[k], k)
        s2 = comm.autoreg_stats()
        results.append({"tag": "cache/stats", "rank": RANK, "s1": s1, "s2": s2,
                        "ok": (s1["zero_copy"] == NBUF and s1["opens"] == NBUF * (ws - 1) and
                               s1["evictions"] == (NBUF - 32) * (ws - 1) and
                               s2["opens"] - s1["opens"] == 2 * (ws - 1) and s2["bounced"] == 0)})
        # 3. registrations are not consulted under auto-registration: rank 0 has
        #    its buffer registered, the others not — one path for all, exact
        b3 = torch.from_numpy(inputs(3)).cuda()
        if RANK == 0:
            L.lib.polar_register(comm.h, L.C.c_void_p(b3.data_ptr()), b3.numel() * 4)
        # (a registration is collective; rank 0 alone registering would block, so
        # the others register a scratch tensor in the same call order)
        else:
            dummy = torch.empty(1 << 20, dtype=torch.float32, device="cuda")
            L.lib.polar_register(comm.h, L.C.c_void_p(dummy.data_ptr()), dummy.numel() * 4)
        ar(b3)
        torch.cuda.synchronize()
        comm.check()
        check("mixed-registration/auto", b3, 3)
        # 4. ranks that decide the call differently (rank 0 forces ring for this
        #    size): the exchange compares the decision tags, every rank returns
        #    ESTATE before anything is launched, every buffer keeps its input
        b4 = torch.from_numpy(inputs(4)).cuda()
        torch.cuda.synchronize()
        if RANK == 0:
            L.set_policy([(0, 0, 2**64 - 1, L.RING, L.SIMPLE, 8)])
        st = L.lib.polar_allreduce(comm.h, L.C.c_void_p(b4.data_ptr()), COUNT, L.FLOAT32, L.SUM,
                                   L.C.c_void_p(stream.cuda_stream))
        torch.cuda.synchronize()
        untouched = bool(np.array_equal(b4.cpu().numpy().view(np.uint32), inputs(4).view(np.uint32)))
        s3 = comm.autoreg_stats()
        results.append({"tag": "decision-mismatch/estate", "rank": RANK, "status": L.STATUS_NAMES[st],
                        "untouched": untouched, "stats": s3,
                        "ok": L.STATUS_NAMES[st] == "estate" and untouched and s3["mismatches"] == 1})
        L.set_policy([])
    else:
        # 2. one rank's buffers live in VMM memory: every rank bounces, results exact
        for k in range(3):
            b = torch.from_numpy(inputs(k)).cuda()
            ar(b)
            torch.cuda.synchronize()
            comm.check()
            check(f"vmm/bounce/{k}", b, k)
        s = comm.autoreg_stats()
        results.append({"tag": "vmm/stats", "rank": RANK, "stats": s,
                        "ok": s["exchanges"] == 3 and s["bounced"] == 3 and s["zero_copy"] == 0})
    comm.destroy()
    allres = allgather_obj(results)
    if RANK == 0:
        with open(out_path, "w") as f:
            json.dump([r for rr in allres for r in rr], f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
