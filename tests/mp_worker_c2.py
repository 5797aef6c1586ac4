"""One rank of a real (multi-process) comm at the north_star size, launched by
torchrun (VERDICT r01 "test the north_star path at its own size").

BASELINE config 2's largest message (32 Mi f32 = 128 MiB per rank) through the
north_star signature polar_allreduce(buf, count, dtype, op, stream) on
  * a registered symmetric buffer (polar_mem_alloc)   -> default table: zero-copy two-shot
  * an unregistered torch tensor                       -> default table: two-shot via the bounce region
  * forced ring / tree Simple (the paper's selected algorithms)
plus stale-registration handling, deregistration, and the synchronous
entry-handshake check (ranks addressing one call differently latch ESTATE
before any data moves).  Every result is checked on sampled windows against the
oracle (two-shot bit-exact; ring / tree within R2's 1e-6 * n * sum|x| bound,
max err/bound reported) and hashed across ranks (bitwise identical, R4).

Each rank generates only its own input and all-gathers its input WINDOWS, so
host memory stays at one message per process.  Rank 0 writes a JSON report.
"""
import hashlib
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

COUNT = 32 << 20   # 128 MiB of f32 per rank (C2's largest size)


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

    comm = L.Comm.init(ws, rank, dev, L.torch_allgather(dist, ws))
    results = []
    rng = np.random.default_rng(77)
    windows = [(0, 4096), (COUNT - 4099, COUNT)] + [(int(s), int(s) + 2048)
                                                     for s in rng.integers(0, COUNT - 2048, 12)]
    x_mine = synth.gen("f32", COUNT, rank, cfg=2, dist="unif")
    # every rank's input windows (the oracle needs all ranks' values there)
    win_all = allgather([x_mine[lo:hi].copy() for lo, hi in windows])

    def check(tag, t, exact):
        got = t.cpu().numpy()
        worst = 0.0
        ok = True
        h = hashlib.sha1()
        for k, (lo, hi) in enumerate(windows):
            xs = [win_all[p][k] for p in range(ws)]
            exp = orc.allreduce(xs, "f32", "sum")
            g = got[lo:hi]
            h.update(g.tobytes())
            if exact:
                ok = ok and bool(np.array_equal(g.view(np.uint32), exp.view(np.uint32)))
            else:
                bound = 1e-6 * ws * np.sum(np.abs(np.stack(xs).astype(np.float64)), axis=0)
                err = np.abs(g.astype(np.float64) - exp.astype(np.float64))
                worst = max(worst, float(np.max(err / np.maximum(bound, 1e-300))))
                ok = ok and bool(np.all(err <= bound))
        hs = allgather(h.hexdigest())
        d = comm.last_decision()
        results.append({"tag": tag, "rank": rank, "ok": ok, "identical": len(set(hs)) == 1,
                        "max_err_over_bound": worst, "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto],
                                                                  d.nchannels]})

    stream = torch.cuda.current_stream()

    def ar(t):
        st = L.lib.polar_allreduce(comm.h, L.C.c_void_p(t.data_ptr()), t.numel(), L.FLOAT32, L.SUM,
                                   L.C.c_void_p(stream.cuda_stream))
        if st != L.OK:
            raise L.PolarError(st, "polar_allreduce")

    # 1. registered symmetric buffer, policy-selected (two-shot zero-copy)
    (sym,) = comm.mem_alloc_tensors(COUNT, torch.float32)
    sym.copy_(torch.from_numpy(x_mine))
    ar(sym)
    torch.cuda.synchronize()
    comm.check()
    check("c2/registered/policy", sym, True)
    # 2. unregistered torch tensor, policy-selected (two-shot through the bounce region)
    plain = torch.from_numpy(x_mine).cuda()
    ar(plain)
    torch.cuda.synchronize()
    comm.check()
    check("c2/unregistered/policy", plain, True)
    # 3. forced ring / tree Simple on the unregistered tensor (32 channels, the paper's
    #    setting; POLAR_TEST_NCH lowers it when every rank shares one GPU: 8 x 32 CTAs
    #    would not be co-resident on 148 SMs)
    fnch = int(os.environ.get("POLAR_TEST_NCH", "32"))
    for algo in ("ring", "tree"):
        plain.copy_(torch.from_numpy(x_mine))
        comm.allreduce_forced(plain, algo, "simple", fnch)
        torch.cuda.synchronize()
        comm.check()
        check(f"c2/{algo}/simple/32ch", plain, False)
    # 4. back to back without host sync: registered, unregistered, registered again
    sym.copy_(torch.from_numpy(x_mine))
    plain.copy_(torch.from_numpy(x_mine))
    sym2 = torch.from_numpy(x_mine).cuda()
    ar(sym)
    ar(plain)
    ar(sym2)
    torch.cuda.synchronize()
    comm.check()
    check("c2/b2b/registered", sym, True)
    check("c2/b2b/unregistered", plain, True)
    check("c2/b2b/unregistered2", sym2, True)
    del sym2
    # 5. a user registration whose allocation is freed is dropped at its next use
    #    (every rank frees; a new allocation may reuse the addresses)
    reg = torch.empty(COUNT, dtype=torch.float32, device="cuda")
    comm.register(reg)
    reg.copy_(torch.from_numpy(x_mine))
    ar(reg)
    torch.cuda.synchronize()
    check("c2/user-registered", reg, True)
    del reg
    torch.cuda.synchronize()
    torch.cuda.empty_cache()          # cudaFree of the segment: the registration is now stale
    fresh = torch.from_numpy(x_mine).cuda()
    ar(fresh)
    torch.cuda.synchronize()
    comm.check()
    check("c2/after-free", fresh, True)
    # 6. deregistration (collective), then the buffer runs the bounce path
    reg2 = torch.from_numpy(x_mine).cuda()
    comm.register(reg2)
    comm.deregister(reg2)
    ar(reg2)
    torch.cuda.synchronize()
    comm.check()
    check("c2/deregistered", reg2, True)
    # 8. auto-registration (polar_comm_autoreg): unregistered tensors run zero-copy
    #    after one IPC-handle exchange per call; offsets differ between ranks
    try:
        comm.autoreg(rank == 0, 1 << 20)      # ranks disagree: refused on every rank
        mism = "accepted"
    except L.PolarError as ex:
        mism = ex.name
    results.append({"tag": "autoreg/mismatch-refused", "rank": rank, "ok": mism == "einval", "identical": True})
    comm.autoreg(True, 1 << 20)
    s0 = comm.autoreg_stats()
    big = torch.empty(COUNT + 4096, dtype=torch.float32, device="cuda")
    v1 = big[1024 * rank:1024 * rank + COUNT]            # 16-B aligned, rank-dependent offset
    v1.copy_(torch.from_numpy(x_mine))
    ar(v1)
    torch.cuda.synchronize()
    comm.check()
    check("autoreg/first", v1, True)
    s1 = comm.autoreg_stats()
    v1.copy_(torch.from_numpy(x_mine))
    ar(v1)                                               # the same allocation: no new open
    v2 = torch.from_numpy(x_mine).cuda()
    ar(v2)                                               # back to back, another allocation
    torch.cuda.synchronize()
    comm.check()
    check("autoreg/again", v1, True)
    check("autoreg/b2b-other", v2, True)
    s2 = comm.autoreg_stats()
    results.append({"tag": "autoreg/stats", "rank": rank, "identical": True,
                    "ok": (s1["zero_copy"] - s0["zero_copy"] == 1 and s1["opens"] - s0["opens"] == ws - 1 and
                           s2["zero_copy"] - s1["zero_copy"] == 2 and s2["opens"] - s1["opens"] == ws - 1),
                    "stats": [s0, s1, s2]})
    # unaligned, rank-dependent offsets (4-B aligned only: the kernel's scalar path)
    v3 = big[1 + rank:1 + rank + COUNT]
    v3.copy_(torch.from_numpy(x_mine))
    ar(v3)
    torch.cuda.synchronize()
    comm.check()
    check("autoreg/unaligned", v3, True)
    # a freed and re-allocated buffer (the peers' old mappings are stale)
    del v1, v2, v3, big
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    v4 = torch.from_numpy(x_mine).cuda()
    ar(v4)
    torch.cuda.synchronize()
    comm.check()
    check("autoreg/after-free", v4, True)
    # CUDA-graph capture: the exchange runs at capture time, replays reuse the pointers
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=gs):
        st = L.lib.polar_allreduce(comm.h, L.C.c_void_p(v4.data_ptr()), COUNT, L.FLOAT32, L.SUM,
                                   L.C.c_void_p(gs.cuda_stream))
    ok_cap = st == L.OK
    for rep in range(2):
        v4.copy_(torch.from_numpy(x_mine))
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        comm.check()
        check(f"autoreg/graph-replay{rep}", v4, True)
    results.append({"tag": "autoreg/graph-captured", "rank": rank, "ok": ok_cap, "identical": True})
    del g
    results.append({"tag": "autoreg/final-stats", "rank": rank, "ok": True, "identical": True,
                    "stats": comm.autoreg_stats()})
    comm.autoreg(False)
    # 7. ranks addressing one call differently: rank 0 registered, the others not.
    #    The entry handshake compares the decision tags (path included) and every
    #    rank latches ESTATE before any data moves: every buffer keeps its input.
    probe_n = 1 << 20
    if rank == 0:
        (buf,) = comm.mem_alloc_tensors(probe_n, torch.float32)
    else:
        comm.mem_alloc_tensors(probe_n, torch.float32)   # collective: every rank allocates
        buf = torch.empty(probe_n, dtype=torch.float32, device="cuda")
    buf.copy_(torch.from_numpy(x_mine[:probe_n]))
    torch.cuda.synchronize()
    dist.barrier()
    st = L.lib.polar_allreduce(comm.h, L.C.c_void_p(buf.data_ptr()), probe_n, L.FLOAT32, L.SUM,
                               L.C.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    try:
        comm.check()
        latched = None
    except L.PolarError as ex:
        latched = ex.name
    untouched = bool(np.array_equal(buf.cpu().numpy().view(np.uint32), x_mine[:probe_n].view(np.uint32)))
    results.append({"tag": "path-mismatch-latched-before-data", "rank": rank, "ok": st == L.OK and
                    latched == "estate" and untouched, "identical": True, "latched": latched,
                    "untouched": untouched})
    comm.destroy()
    allres = allgather(results)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump([r for rr in allres for r in rr], f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
