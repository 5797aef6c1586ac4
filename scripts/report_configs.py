"""Measure BASELINE.json configs 1-5 on one B200 (virtual ranks) -> JSON lines.

python scripts/report_configs.py [--configs 1,2,3,5] > gpurun_out/configs.jsonl
  C1  2-rank int32 sum, 4 KiB-1 MiB, fixed size-threshold table (policies/c1_fixed_threshold.json):
      parity (bit-exact vs oracle, whole vectors), decision == oracle mapping, t, busBW
  C2  8-rank fp32 sum, 4-128 MiB: default policy vs every forced (algo, proto) at its best
      channel count, vs the best single global choice (E10), vs bad_channels (E11)
  C3  bf16 sum, 4 KiB-1 GiB at 2/4/8 ranks: forced {oneshot, twoshot, ring, tree} x {LL, LL128, Simple}
      (16 channels) and policy-selected; sampled parity at every size
  C5  400,000 decisions (p50/p99/batched), swap stress (4 invokers, 1000 swaps)
C4 is scripts/c4_latency.py.  Peers are local HBM (virtual ranks), so these are
kernel/HBM numbers, not NVLink numbers.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from oracle import policy as opol  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402
from tests.gpu_common import to_device, to_host  # noqa: E402

ALGOS = [(a, p) for a in ("oneshot", "twoshot", "ring", "tree") for p in ("ll", "ll128", "simple")]


def emit(d):
    print(json.dumps(d), flush=True)


def ev_time(fn, iters, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(iters):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / iters


def iters_for(fn, budget=0.1):
    t = ev_time(fn, 1, warm=1)
    return max(3, min(100, int(budget / max(t, 1e-6)))), t


def busbw(nbytes, n, t):
    return nbytes * 2 * (n - 1) / n / t / 1e9


def load_rows(name):
    with open(os.path.join(ROOT, "policies", name)) as f:
        return [tuple(r) for r in json.load(f)["rows"]]


def c1():
    rows = load_rows("c1_fixed_threshold.json")
    L.set_policy(rows)
    comm = L.Comm.virtual(2, 0)
    for k in range(9):
        size = 4096 << k
        count = size // 4
        xs = synth.gen_ranks("i32", count, 2, cfg=1, dist="ints")
        ts = [to_device(x, "i32") for x in xs]
        comm.allreduce(ts)
        torch.cuda.synchronize()
        comm.check()
        exp = orc.allreduce(xs, "i32", "sum")
        exact = all(np.array_equal(to_host(t, "i32"), exp) for t in ts)
        d = comm.last_decision()
        dec_ok = d.as_tuple() == opol.decide(rows, 0, 2, size)
        it, _ = iters_for(lambda: comm.allreduce(ts))
        t = ev_time(lambda: comm.allreduce(ts), it)
        emit({"config": "C1", "n": 2, "dtype": "i32", "bytes": size, "bit_exact": exact, "decision_matches_oracle": dec_ok,
              "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels], "us": round(t * 1e6, 2),
              "busbw_gbs": round(busbw(size, 2, t), 2)})
    comm.destroy()
    L.set_policy([])


def c2():
    n = 8
    comm = L.Comm.virtual(n, 0)
    sizes = [(4 << 20) << k for k in range(6)]
    bufs = [torch.empty(max(sizes) // 4, device="cuda").uniform_(-1, 1) for _ in range(n)]
    best_global = {}
    for size in sizes:
        v = [b[: size // 4] for b in bufs]
        L.set_policy([])
        it, _ = iters_for(lambda: comm.allreduce(v))
        t = ev_time(lambda: comm.allreduce(v), it)
        d = comm.last_decision()
        rec = {"config": "C2", "n": n, "dtype": "f32", "bytes": size, "policy": "default",
               "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels],
               "busbw_gbs": round(busbw(size, n, t), 1), "us": round(t * 1e6, 1),
               # back-to-back calls: where the n ranks' buffers fit in the 126 MB L2 the
               # inputs may be L2-resident (bench.py's c2_sweep flushes instead)
               "l2_resident_possible": n * size <= (126 << 20)}
        forced = {}
        for algo, proto in ALGOS:
            best = None
            for nch in (4, 8, 12, 16, 18):
                fn = lambda: comm.allreduce_forced(v, algo, proto, nch)  # noqa: E731
                it, t1 = iters_for(fn, 0.05)
                if t1 > 0.05:
                    continue
                tt = ev_time(fn, it)
                bw = busbw(size, n, tt)
                best_global[(algo, proto, nch)] = best_global.get((algo, proto, nch), []) + [bw]
                if best is None or bw > best[0]:
                    best = (round(bw, 1), nch)
            forced[f"{algo}/{proto}"] = best
        rec["forced_best"] = forced
        # the paper's case-study policy as a table (Ring/LL128 4-32 MiB, Ring/Simple 64-192 MiB)
        L.set_policy(load_rows("nvlink_ring_mid_v2.json"))
        it, _ = iters_for(lambda: comm.allreduce(v), 0.05)
        tp = ev_time(lambda: comm.allreduce(v), it)
        d = comm.last_decision()
        rec["nvlink_ring_mid_v2"] = {"decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels],
                                     "busbw_gbs": round(busbw(size, n, tp), 1)}
        # bad_channels: a policy forcing 1 channel, everything else deferred
        L.set_policy([(0, 0, 2**64 - 1, L.UNSET, L.UNSET, 1)])
        it, _ = iters_for(lambda: comm.allreduce(v), 0.05)
        tb = ev_time(lambda: comm.allreduce(v), it)
        rec["bad_channels_busbw_gbs"] = round(busbw(size, n, tb), 1)
        L.set_policy([])
        emit(rec)
    # E10: best single global choice across the sweep (geomean)
    full = {k: v for k, v in best_global.items() if len(v) == len(sizes)}
    if full:
        g = max(full, key=lambda k: np.exp(np.mean(np.log(full[k]))))
        emit({"config": "C2", "best_single_global": list(g), "busbw_gbs": [round(x, 1) for x in full[g]]})
    comm.destroy()


def c3():
    for n in (2, 4, 8):
        comm = L.Comm.virtual(n, 0)
        sizes = [4096 << k for k in range(0, 19)]      # 4 KiB .. 1 GiB
        maxc = max(sizes) // 2
        bufs = [torch.empty(maxc, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        for size in sizes:
            count = size // 2
            # parity sample: regenerate the first min(count, 1M) elements and check them exactly
            m = min(count, 1 << 20)
            xs = synth.gen_ranks("bf16", m, n, cfg=3, dist="normal")
            rec = {"config": "C3", "n": n, "dtype": "bf16", "bytes": size}
            for algo, proto in ALGOS + [("policy", "")]:
                for r in range(n):
                    bufs[r][:m].copy_(to_device(xs[r], "bf16"))
                v = [b[:count] for b in bufs]
                if algo == "policy":
                    fn = lambda: comm.allreduce(v)  # noqa: E731
                else:
                    fn = lambda: comm.allreduce_forced(v, algo, proto, 16)  # noqa: E731
                fn()
                torch.cuda.synchronize()
                comm.check()
                got = to_host(v[0][:m], "bf16")
                exp = orc.allreduce(xs, "bf16", "sum")
                same = all(np.array_equal(to_host(b[:m], "bf16"), got) for b in v)
                yg = orc.bf16_bits_to_f32(got).astype(np.float64)
                ye = orc.bf16_bits_to_f32(exp).astype(np.float64)
                within = bool(np.all(np.abs(yg - ye) <= 1e-2 * np.abs(ye)))
                it, t1 = iters_for(fn, 0.05)
                key = f"{algo}/{proto}" if proto else "policy"
                if t1 > 0.25:
                    rec[key] = {"skipped_us": round(t1 * 1e6)}
                    continue
                t = ev_time(fn, it, warm=1)
                d = comm.last_decision()
                rec[key] = {"busbw_gbs": round(busbw(size, n, t), 1), "us": round(t * 1e6, 1),
                            "bit_exact_sample": bool(np.array_equal(got, exp)), "within_1e-2": within,
                            "ranks_identical": same}
                if algo == "policy":
                    rec[key]["decision"] = [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels]
            emit(rec)
        del bufs
        comm.destroy()
        torch.cuda.empty_cache()


def f4():
    """ReduceScatter / AllGather / Broadcast, 8 virtual ranks, f32.
    busBW (nccl-tests): RS, AG: S*(n-1)/n / t with S the full buffer; BC: S / t."""
    n = 8
    comm = L.Comm.virtual(n, 0)
    for total in [(64 << 10) << (2 * k) for k in range(0, 7)]:      # 64 KiB .. 256 MiB
        blk = total // n // 4
        sends = [torch.randn(n * blk, device="cuda") for _ in range(n)]
        recvs = [torch.empty(blk, device="cuda") for _ in range(n)]
        agsend = [torch.randn(blk, device="cuda") for _ in range(n)]
        agrecv = [torch.empty(n * blk, device="cuda") for _ in range(n)]
        rec = {"config": "F4", "n": n, "dtype": "f32", "bytes": total}
        for name, fn, bb in (("reduce_scatter", lambda: comm.reduce_scatter(sends, recvs), total * (n - 1) / n),
                             ("all_gather", lambda: comm.all_gather(agsend, agrecv), total * (n - 1) / n),
                             ("broadcast", lambda: comm.broadcast(agrecv, root=3), total)):
            it, _ = iters_for(fn, 0.05)
            t = ev_time(fn, it)
            rec[name] = {"busbw_gbs": round(bb / t / 1e9, 1), "us": round(t * 1e6, 1)}
        emit(rec)
        del sends, recvs, agsend, agrecv
    comm.destroy()


def e12():
    """Stability (PAPER.md L588-595 method): 20 independent runs at 128 MiB, 8 ranks,
    each the mean of 20 timed calls after warm-up; mean +- sd and CV of busBW, for
    the policy-selected AllReduce and for AllGather (the paper's collective)."""
    n, size = 8, 128 << 20
    comm = L.Comm.virtual(n, 0)
    bufs = [torch.empty(size // 4, device="cuda").uniform_(-1, 1) for _ in range(n)]
    ag_s = [torch.randn(size // 4 // n, device="cuda") for _ in range(n)]
    ag_r = [torch.empty(size // 4, device="cuda") for _ in range(n)]
    for name, fn, bb in (("allreduce", lambda: comm.allreduce(bufs), size * 2 * (n - 1) / n),
                         ("all_gather", lambda: comm.all_gather(ag_s, ag_r), size * (n - 1) / n)):
        runs = [bb / ev_time(fn, 20, warm=5) / 1e9 for _ in range(20)]
        m, sd = float(np.mean(runs)), float(np.std(runs, ddof=1))
        emit({"config": "E12", "op": name, "n": n, "bytes": size, "runs": 20,
              "busbw_mean_gbs": round(m, 2), "busbw_sd_gbs": round(sd, 2), "cv_pct": round(100 * sd / m, 3)})
    comm.destroy()


def table2():
    """PAPER.md Table 2 sizes on this box (8 ranks, f32 sum): the policy's choice vs
    ring (the paper's winner in 4-128 MiB) at 256 MiB, 1 GiB and 8 GiB."""
    n = 8
    comm = L.Comm.virtual(n, 0)
    for size in (256 << 20, 1 << 30, 8 << 30):
        bufs = [torch.empty(size // 4, device="cuda").uniform_(-1, 1) for _ in range(n)]
        rec = {"config": "T2", "n": n, "dtype": "f32", "bytes": size}
        t = ev_time(lambda: comm.allreduce(bufs), 3, warm=1)
        d = comm.last_decision()
        rec["policy"] = {"decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels],
                         "busbw_gbs": round(busbw(size, n, t), 1)}
        t = ev_time(lambda: comm.allreduce_forced(bufs, "ring", "simple", 32), 2, warm=1)
        rec["ring_simple"] = {"busbw_gbs": round(busbw(size, n, t), 1)}
        emit(rec)
        del bufs
        torch.cuda.empty_cache()
    comm.destroy()


def c5():
    ctxs = [(nr, 1 << k) for k in range(3, 31) for nr in (2, 4, 8)]
    s = L.bench_decide(ctxs, nwarm=10_000, ncalls=400_000)
    emit({"config": "C5", "kind": "decide_noop", **{k: round(v, 2) if isinstance(v, float) else v for k, v in s.items()}})
    L.set_policy(load_rows("b200_virtual.json"))
    s = L.bench_decide(ctxs, nwarm=10_000, ncalls=400_000)
    emit({"config": "C5", "kind": "decide_tuned_table", **{k: round(v, 2) if isinstance(v, float) else v for k, v in s.items()}})
    a = [(0, 0, 32768, L.TREE, L.SIMPLE, 4), (0, 0, 2**64 - 1, L.RING, L.SIMPLE, 4)]
    b = load_rows("b200_virtual.json")
    sw = L.bench_swap(a, b, nthreads=4, calls_per_thread=100_000, nswaps=1000)
    emit({"config": "C5", "kind": "swap_stress", **{k: round(v, 1) if isinstance(v, float) else v for k, v in sw.items()}})
    L.set_policy([])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,5,f4,e12,t2")
    a = ap.parse_args()
    t0 = time.time()
    for c in a.configs.split(","):
        {"1": c1, "2": c2, "3": c3, "5": c5, "f4": f4, "e12": e12, "t2": table2}[c.strip()]()
    emit({"elapsed_s": round(time.time() - t0, 1), "cpu_cores": len(os.sched_getaffinity(0))})


if __name__ == "__main__":
    main()
