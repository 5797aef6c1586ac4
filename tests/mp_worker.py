"""One rank of a real (multi-process) polar comm, launched by torchrun.

Each rank: gloo process group for the host bootstrap only, polar_comm_init
(CUDA IPC exchange of the scratch), then every algorithm x protocol on this
rank's seeded input, checked against the oracle (each rank regenerates every
rank's input itself).  Also the registered zero-copy two-shot (polar_mem_alloc)
and the unregistered two-shot bounce path.  Rank 0 writes a JSON report.

Device: LOCAL_RANK if that many GPUs exist, else GPU 0 for every rank (ranks
then share one GPU through CUDA IPC and context time-slicing).
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
    results = []
    # LL128 is refused on a real comm until its premise was probed over this transport
    try:
        comm.allreduce_forced(torch.ones(4096, device="cuda"), "ring", "ll128", 1)
        refused = False
    except L.PolarError as e:
        refused = e.name == "eunsupported"
    torn, reads = comm.probe_ll128(iters=2000)
    results.append({"tag": "ll128-gate", "rank": rank, "ok": refused and torn == 0 and reads == ws * 64 * 2000 * 32,
                    "identical": True, "torn": torn, "reads": reads})

    def check(tag, t, xs, dtype, op, exact):
        got = to_host(t, dtype)
        exp = orc.allreduce(xs, dtype, op)
        if exact:
            ok = np.array_equal(got.view(np.uint8), exp.view(np.uint8))
        else:
            bound = 1e-6 * ws * np.sum(np.abs(np.stack(xs).astype(np.float64)), axis=0)
            ok = bool(np.all(np.abs(got.astype(np.float64) - exp.astype(np.float64)) <= bound))
        # cross-rank bitwise identity: gather a hash of the result
        h = hashlib.sha1(got.tobytes()).hexdigest()
        hs = [None] * ws
        dist.all_gather_object(hs, h)
        results.append({"tag": tag, "rank": rank, "ok": bool(ok), "identical": len(set(hs)) == 1})

    for algo in ("oneshot", "twoshot", "ring", "tree"):
        for proto in ("ll", "ll128", "simple"):
            for dtype, count, nch in (("f32", 70_001, 3), ("bf16", 5_003, 2), ("i32", 1, 1)):
                xs = synth.gen_ranks(dtype, count, ws, cfg=31, dist="ints")
                t = to_device(xs[rank], dtype)
                comm.allreduce_forced(t, algo, proto, nch)
                torch.cuda.synchronize()
                comm.check()
                check(f"{algo}/{proto}/{dtype}/{count}", t, xs, dtype, "sum", True)
    # registered zero-copy two-shot on symmetric memory, random floats: exact (rank order)
    count = 1 << 20
    xs = synth.gen_ranks("f32", count, ws, cfg=32, dist="unif")
    (buf,) = comm.mem_alloc_tensors(count, torch.float32)
    buf.copy_(torch.from_numpy(xs[rank]))
    comm.allreduce_forced(buf, "twoshot", "simple", 8)
    torch.cuda.synchronize()
    check("twoshot/simple/registered", buf, xs, "f32", "sum", True)
    # two registrations inside one torch allocation (caching-allocator pattern):
    # the second must reuse the first IPC mapping; zero-copy two-shot on a view
    big = torch.empty(3 * count, dtype=torch.float32, device="cuda")
    comm.register(big[:count])
    view = big[count:2 * count]
    comm.register(view)
    view.copy_(torch.from_numpy(xs[rank]))
    comm.allreduce_forced(view, "twoshot", "simple", 4)
    torch.cuda.synchronize()
    check("twoshot/simple/registered-view", view, xs, "f32", "sum", True)
    # other collectives (f4) on registered symmetric buffers
    from oracle import collectives as OC
    rc = 10_007
    xs_rs = synth.gen_ranks("f32", ws * rc, ws, cfg=33, dist="unif")
    (sym,) = comm.mem_alloc_tensors(ws * rc, torch.float32)
    sym.copy_(torch.from_numpy(xs_rs[rank]))
    rs_out = torch.empty(rc, device="cuda")
    L.lib.polar_reduce_scatter(comm.h, L.C.c_void_p(sym.data_ptr()), L.C.c_void_p(rs_out.data_ptr()), rc, L.FLOAT32,
                               L.SUM, L.C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    comm.check()
    got = rs_out.cpu().numpy()
    exp = OC.reduce_scatter(xs_rs, "f32", "sum")[rank]
    results.append({"tag": "rs/registered", "rank": rank, "ok": bool(np.array_equal(got.view(np.uint32), exp.view(np.uint32))),
                    "identical": True})
    xs_ag = synth.gen_ranks("i32", rc, ws, cfg=34, dist="full")
    src = torch.from_numpy(xs_ag[rank]).cuda()
    sym_i = sym.view(torch.int32)
    st = L.lib.polar_all_gather(comm.h, L.C.c_void_p(src.data_ptr()), L.C.c_void_p(sym_i.data_ptr()), rc, L.INT32,
                                L.C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    results.append({"tag": "ag/registered", "rank": rank, "ok": st == 0 and bool(np.array_equal(
        sym_i.cpu().numpy(), OC.all_gather(xs_ag))), "identical": True})
    bc = sym[:rc]
    bc.copy_(torch.from_numpy(xs_rs[rank][:rc]))
    st = L.lib.polar_broadcast(comm.h, L.C.c_void_p(bc.data_ptr()), rc, L.FLOAT32, ws - 1,
                               L.C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    results.append({"tag": "bc/registered", "rank": rank, "ok": st == 0 and bool(np.array_equal(
        bc.cpu().numpy(), xs_rs[ws - 1][:rc])), "identical": True})
    plain = torch.ones(rc, device="cuda")
    st = L.lib.polar_broadcast(comm.h, L.C.c_void_p(plain.data_ptr()), rc, L.FLOAT32, 0,
                               L.C.c_void_p(torch.cuda.current_stream().cuda_stream))
    results.append({"tag": "bc/unregistered-einval", "rank": rank, "ok": st == L.EINVAL, "identical": True})
    # p2p probe over the IPC peer mapping: loads of peer (r+1)%n checked by XOR,
    # stores checked in my own buffer (written by rank (r-1)%n)
    (pb,) = comm.mem_alloc_tensors((256 << 10) // 4, torch.int32)
    pb.copy_(torch.from_numpy(synth.gen("i32", (256 << 10) // 4, rank, cfg=35, dist="full")))
    torch.cuda.synchronize()
    peer_before = synth.gen("i32", (256 << 10) // 4, (rank + 1) % ws, cfg=35, dist="full").view(np.uint32)
    w = peer_before.reshape(-1, 4).astype(np.uint64)
    exp_xor = int(np.bitwise_xor.reduce(((w[:, 0] ^ w[:, 2]) << np.uint64(32)) | (w[:, 1] ^ w[:, 3])))
    (pr,) = comm.p2p_probe(pb, iters=3)
    mine = pb.cpu().numpy().view(np.uint32).reshape(-1, 4)
    writer = (rank - 1) % ws
    i = np.arange(mine.shape[0], dtype=np.uint64)
    pat_ok = (np.array_equal(mine[:, 0], (i & np.uint64(0xFFFFFFFF)).astype(np.uint32)) and
              bool((mine[:, 2] == writer).all()) and np.array_equal(mine[:, 3], ~mine[:, 0]))
    results.append({"tag": "p2p_probe", "rank": rank, "identical": True,
                    "ok": bool(pr["load_xor"] == exp_xor and pat_ok and pr["load_gbs"] > 0 and pr["store_gbs"] > 0
                               and (pr["pingpong_us"] > 0) == ((rank ^ 1) < ws))})
    # collective free of a symmetric buffer, then a fresh allocation still works
    sym_ptr = sym.data_ptr()
    del sym, sym_i, bc
    comm.mem_free(sym_ptr)
    (again,) = comm.mem_alloc_tensors(4096, torch.float32)
    again.fill_(float(rank + 1))
    comm.allreduce_forced(again, "twoshot", "simple", 2)
    torch.cuda.synchronize()
    results.append({"tag": "mem_free+realloc", "rank": rank, "ok": bool((again == ws * (ws + 1) / 2).all()),
                    "identical": True})
    # policy-selected on a plain torch tensor (unregistered: bounce path if two-shot)
    t = to_device(xs[rank], "f32")
    comm.allreduce(t)
    torch.cuda.synchronize()
    d = comm.last_decision()
    check(f"policy/{L.ALGO_NAMES[d.algo]}/{L.PROTO_NAMES[d.proto]}", t, xs, "f32", "sum",
          L.ALGO_NAMES[d.algo] in ("oneshot", "twoshot"))
    # back-to-back without host sync, alternating algorithms
    ts, xss = [], []
    for i, (algo, proto) in enumerate([("ring", "ll"), ("twoshot", "simple"), ("tree", "simple"),
                                       ("oneshot", "ll"), ("twoshot", "ll"), ("ring", "simple")]):
        xs = synth.gen_ranks("i32", 30_000 + i, ws, cfg=40 + i, dist="full")
        t = to_device(xs[rank], "i32")
        comm.allreduce_forced(t, algo, proto, 1 + i)
        ts.append(t)
        xss.append((xs, algo))
    torch.cuda.synchronize()
    comm.check()
    for (xs, algo), t in zip(xss, ts):
        check(f"b2b/{algo}", t, xs, "i32", "sum", True)
    # CUDA-graph capture on the real (IPC) comm: registered zero-copy two-shot,
    # warp-specialised ring and tree Simple (multi-slot), ring LL; every replay
    # advances the device-resident epochs / FIFO counters, none is host-synced
    # between the captured calls
    # (the last entry: an UNREGISTERED two-shot, i.e. the bounce pipeline with its
    # two library streams forked into and joined back from the capture, several
    # chunks with the test's 1 MiB bounce region)
    plan = [("twoshot", "simple", 50_003), ("ring", "simple", 400_001), ("tree", "simple", 1_000_003),
            ("ring", "ll", 20_011), ("twoshot", "simple", 700_001)]
    (gsym,) = comm.mem_alloc_tensors(plan[0][2], torch.float32)
    gbufs = [gsym] + [torch.empty(c, dtype=torch.float32, device="cuda") for _, _, c in plan[1:]]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for (algo, proto, _), b in zip(plan, gbufs):
            comm.allreduce_forced(b, algo, proto, 4)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for (algo, proto, _), b in zip(plan, gbufs):
            comm.allreduce_forced(b, algo, proto, 4)
    for rep in range(3):
        xss = [synth.gen_ranks("f32", c, ws, cfg=60 + 10 * rep + i, dist="ints") for i, (_, _, c) in enumerate(plan)]
        for xs, b in zip(xss, gbufs):
            b.copy_(torch.from_numpy(xs[rank]))
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        comm.check()
        for (algo, proto, _), xs, b in zip(plan, xss, gbufs):
            check(f"graph{rep}/{algo}/{proto}", b, xs, "f32", "sum", True)
    del g, gbufs, gsym
    # the e2e host path on unregistered device buffers (host chunks x bounce chunks)
    xs = synth.gen_ranks("f32", 900_001, ws, cfg=95, dist="ints")
    host = torch.from_numpy(xs[rank].copy()).pin_memory()
    devb = torch.empty(900_001, dtype=torch.float32, device="cuda")
    comm.allreduce_host(host, devb)
    comm.check()
    check("host/unregistered", host, xs, "f32", "sum", True)
    # cross-rank decision check (kernels.cuh tag_begin/tag_end):
    # every call above was consistent, so nothing may have latched; then rank 0
    # alone asks for MAX where the others ask for SUM (same algorithm, count and
    # channels, so the exchange completes with silently mixed results) — the next
    # launch must latch POLAR_ESTATE on every rank
    comm.check()
    xs = synth.gen_ranks("f32", 10_001, ws, cfg=90, dist="ints")
    t = to_device(xs[rank], "f32")
    comm.allreduce_forced(t, "twoshot", "ll", 2, op="max" if rank == 0 else "sum")
    comm.allreduce_forced(t, "twoshot", "ll", 2)
    torch.cuda.synchronize()
    try:
        comm.check()
        latched = None
    except L.PolarError as ex:
        latched = ex.name
    results.append({"tag": "decision-mismatch-latched", "rank": rank, "ok": latched == "estate", "identical": True,
                    "latched": latched})
    comm.destroy()
    allres = [None] * ws
    dist.all_gather_object(allres, results)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump([r for rr in allres for r in rr], f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
