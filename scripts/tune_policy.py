"""Derive a measured policy table: every (algorithm, protocol, channels) at each
size, the best per size merged into first-match rows (inclusive max_bytes = the
last measured size of a run of equal winners; the last row open-ended), plus
the paper's comparison points: the best SINGLE global choice (E10, PAPER.md
L566-568) and bad_channels (E11, 1 channel, L581-583).

Virtual ranks (one process, CUDA-graph device time):
    python scripts/tune_policy.py --n 2,4,8 > gpurun_out/tune.jsonl
Real ranks (one process per GPU, torchrun; device time max over ranks; writes
policies/b200_nvlink<n>.json, which bench.py --gpus n then compares with the
default table, the best single choice, bad_channels and NCCL's default):
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        scripts/tune_policy.py --real [--out policies/b200_nvlink8.json]
JSON lines: one per measurement, then {"table": ...} per rank count.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

COMBOS = [(a, p) for a in ("oneshot", "twoshot", "ring", "tree") for p in ("ll", "ll128", "simple")]
U64_MAX = 2**64 - 1


def merge_rows(best, sizes, n, codes):
    """best: {size: (t, algo, proto, nch)} -> first-match rows [coll, nranks,
    max_bytes, algo, proto, nch]; consecutive sizes with the same winner share a
    row whose max_bytes is the last of them; the last row covers every larger size."""
    rows = []
    for size in sorted(sizes):
        _, algo, proto, nch = best[size]
        code = (codes[0][algo], codes[1][proto], nch)
        if rows and tuple(rows[-1][3:]) == code:
            rows[-1][2] = size
        else:
            rows.append([0, n, size, *code])
    if rows:
        rows[-1][2] = U64_MAX
    return rows


def best_single(meas, sizes):
    """E10: the one (algo, proto, nch) with the least total time over every size
    (only choices measured at every size compete).  meas: {(algo, proto, nch): {size: t}}."""
    full = {k: v for k, v in meas.items() if all(s in v for s in sizes)}
    if not full:
        return None
    k = min(full, key=lambda c: sum(full[c][s] for s in sizes))
    return {"choice": list(k), "us": {str(s): round(full[k][s] * 1e6, 2) for s in sizes}}


def graph_time(torch, fn, reps):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(3):
        g.replay()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / (3 * reps)


def event_time(torch, fn, reps):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def tune(L, torch, comm, n, bufs, sizes, nchs, combos, timer, agree, emit):
    """Measure every combo; timer(fn) -> seconds (identical call counts on every rank)."""
    best, meas = {}, {}
    for size in sizes:
        v = [b[: size // 4] for b in bufs]
        for algo, proto in combos:
            for nch in nchs:
                def fn():
                    comm.allreduce_forced(v if len(v) > 1 else v[0], algo, proto, nch)
                try:
                    fn()
                    torch.cuda.synchronize()
                    comm.check()
                except L.PolarError as e:     # e.g. LL128 before its probe passed
                    emit({"n": n, "bytes": size, "algo": algo, "proto": proto, "nch": nch, "skipped": e.name})
                    continue
                t = timer(fn)
                if t is None:
                    continue
                meas.setdefault((algo, proto, nch), {})[size] = t
                emit({"n": n, "bytes": size, "algo": algo, "proto": proto, "nch": nch,
                      "launched": comm.launched_channels(), "us": round(t * 1e6, 2),
                      "busbw_gbs": round(size * 2 * (n - 1) / n / t / 1e9, 2)})
                if size not in best or t < best[size][0]:
                    best[size] = (t, algo, proto, nch)
    return best, meas


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="2,4,8")
    ap.add_argument("--sizes", default=",".join(str(8 << (2 * k)) for k in range(13)))   # 8 B .. 128 MiB
    ap.add_argument("--nch", default="1,2,4,8,16,32")
    ap.add_argument("--combos", default="", help="comma list of algo/proto (default: all 12)")
    ap.add_argument("--real", action="store_true", help="real ranks under torchrun (one process per GPU)")
    ap.add_argument("--out", default="", help="--real: table file (default policies/b200_nvlink<n>.json)")
    a = ap.parse_args()
    import torch

    from paper_2603_11438_b200 import polar as L
    sizes = [int(x) for x in a.sizes.split(",")]
    nchs = [int(x) for x in a.nch.split(",")]
    combos = [tuple(c.split("/")) for c in a.combos.split(",")] if a.combos else COMBOS
    codes = (L.ALGO_CODES, L.PROTO_CODES)

    if a.real:
        import torch.distributed as dist
        ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
        local = int(os.environ.get("LOCAL_RANK", rank))
        dev = local if torch.cuda.device_count() > local else 0
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo")

        def allgather(b):
            o = [None] * ws
            dist.all_gather_object(o, b)
            return o
        comm = L.Comm.init(ws, rank, dev, allgather)
        torn, reads = comm.probe_ll128(iters=2000)   # LL128 is accepted on this transport only if it passed
        (buf,) = comm.mem_alloc_tensors(max(sizes) // 4, torch.float32)
        buf.normal_()

        def timer(fn):
            # identical call counts on every rank: the slowest rank's first call decides
            t1 = max(allgather(event_time(torch, fn, 1)))
            if t1 > 0.05:
                return None
            reps = max(3, min(100, int(0.01 / max(t1, 1e-6))))
            dist.barrier()
            return max(allgather(event_time(torch, fn, reps)))

        def emit(rec):
            if rank == 0:
                print(json.dumps(rec), flush=True)
        best, meas = tune(L, torch, comm, ws, [buf], sizes, nchs, combos, timer, None, emit)
        rows = merge_rows(best, sizes, ws, codes)
        single = best_single(meas, sizes)
        if rank == 0:
            out = a.out or os.path.join(ROOT, "policies", f"b200_nvlink{ws}.json")
            doc = {"name": f"b200_nvlink{ws}", "cite": "measured by scripts/tune_policy.py --real (device time, "
                   "max over ranks); PAPER.md L566-571 (per-size choice), E10 best single L566-568",
                   "rows": rows, "best_single": single["choice"] if single else None,
                   "best_single_us": single["us"] if single else None,
                   "winners": {str(s): [best[s][1], best[s][2], best[s][3], round(best[s][0] * 1e6, 2)] for s in sizes},
                   "ll128_probe": {"torn_lanes": torn, "lane_reads": reads}}
            st, _ = L.set_policy_status(rows)
            doc["set_policy_status"] = L.STATUS_NAMES[st]
            with open(out, "w") as f:
                json.dump(doc, f, indent=1)
            print(json.dumps({"n": ws, "table": rows, "best_single": doc["best_single"], "file": out}), flush=True)
        comm.destroy()
        dist.destroy_process_group()
        return

    for n in [int(x) for x in a.n.split(",")]:
        comm = L.Comm.virtual(n, 0)
        bufs = [torch.randn(max(sizes) // 4, device="cuda") for _ in range(n)]

        def timer(fn):
            t1 = graph_time(torch, fn, 1)
            if t1 > 0.02:
                return None
            return graph_time(torch, fn, max(1, min(50, int(0.01 / max(t1, 1e-6)))))
        best, meas = tune(L, torch, comm, n, bufs, sizes, nchs, combos, timer, None,
                          lambda r: print(json.dumps(r), flush=True))
        rows = merge_rows(best, sizes, n, codes)
        print(json.dumps({"n": n, "table": rows, "best_single": best_single(meas, sizes),
                          "winners": {s: [best[s][1], best[s][2], best[s][3], round(best[s][0] * 1e6, 2)]
                                      for s in sizes}}), flush=True)
        comm.destroy()


if __name__ == "__main__":
    main()
