"""bench.py — BASELINE.json metric on B200: AllReduce busBW (GB/s), policy-selected.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl polar|reference]

N = 1 (no torchrun): 8 VIRTUAL ranks on cuda:0,
    BASELINE config 2's largest size: fp32 sum, 128 MiB per rank, the decision
    made by the policy hook each call.  All ranks' traffic shares one HBM, so the
    roofline is HBM: every step must read n x S and write n x S bytes.
N > 1 (torchrun, one rank per GPU): real ranks over NVLink/NVSwitch with CUDA
    IPC peer mappings, same message; NCCL's default AllReduce is timed beside
    it on the same buffers for the "speedup vs NCCL default" half of the metric.

A step = one policy-selected polar AllReduce (decide + one kernel launch) of the
workload.  Timing: W warm-up steps, then K steps between CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.  The
n x 128 MiB inputs exceed the 126 MB L2, so no flush is needed between steps.
--impl reference times the CPU oracle (oracle/) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AllReduce busBW GB/s vs size at 2/4/8 B200; speedup vs NCCL default"
S_BYTES = 128 << 20            # BASELINE config 2 headline size (per rank)
VIRTUAL_RANKS = 8
C2_SIZES = [4 << 20, 8 << 20, 16 << 20, 32 << 20, 64 << 20, 128 << 20]
PAPER_8GPU_128MIB_DEFAULT = 596.9   # PAPER.md Table 2 L559 (8x B300, NCCL NVLS) — context


def busbw(nbytes, n, t):
    return nbytes * 2.0 * (n - 1) / n / t / 1e9


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def env_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


# ------------------------------------------------------------------ reference
def run_reference(args):
    """The CPU oracle, as it stands, timed on the host cores (rank 0 only)."""
    ws, rank, _ = env_dist()
    if rank != 0:
        return
    import synth
    from oracle import cref

    n = VIRTUAL_RANKS if ws == 1 else ws
    cores = len(os.sched_getaffinity(0))
    count_full = S_BYTES // 4
    xs_full = synth.gen_ranks("f32", count_full, n, cfg=2, dist="unif")

    def oracle(xs):
        return cref.allreduce(xs, "f32", "sum", cores)

    t0 = time.perf_counter()
    oracle(xs_full)
    t_full = time.perf_counter() - t0
    budget = 120.0
    frac = min(1.0, budget / max(1, args.steps + args.warmup) / max(t_full, 1e-9))
    count = max(4096, int(count_full * frac)) // 4096 * 4096
    xs = [x[:count] for x in xs_full]
    for _ in range(args.warmup):
        oracle(xs)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle(xs)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    v = busbw(count * 4, n, t)
    sample = (f"{n} ranks x {count} f32 ({count * 4 / 2**20:.1f} MiB/rank) of the {S_BYTES >> 20} MiB workload, "
              f"plain C oracle (oracle/c/allreduce_ref.c) on {cores} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(n, ws > 1),
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def workload_config(n, real):
    return {
        "workload": (f"C2 {n}-rank AllReduce fp32 sum, {S_BYTES >> 20} MiB per rank, policy-selected, "
                     + ("real ranks (1 per GPU, NVLink)" if real else f"{n} virtual ranks on 1 B200")),
        "nranks": n, "bytes_per_rank": S_BYTES, "op": "sum", "dtype": "f32",
        "l2": f"inputs larger than L2 ({n} x {S_BYTES >> 20} MiB resident), no flush",
    }


# ------------------------------------------------------------------ cpu baseline leg
def _time_oracle(fn, budget_s, max_runs=200):
    ts = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(ts) < 3:
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if len(ts) >= max_runs:
            break
    return statistics.median(ts), len(ts)


def cpu_baseline(n, count):
    """The oracle timed on the host: the plain threaded C oracle on every core
    this process may run on, and the numpy oracle on 1 core."""
    import synth
    from oracle import allreduce as orc
    from oracle import cref
    sub = min(count, 8 << 20)
    xs = synth.gen_ranks("f32", sub, n, cfg=2, dist="unif")
    cores = len(os.sched_getaffinity(0))
    t_c, runs_c = _time_oracle(lambda: cref.allreduce(xs, "f32", "sum", cores), 10.0)
    t_np, runs_np = _time_oracle(lambda: orc.allreduce(xs, "f32", "sum"), 5.0)
    return {"value": round(busbw(sub * 4, n, t_c), 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} ranks x {sub} f32 ({sub * 4 >> 20} MiB/rank) of the C2 workload, plain C oracle "
                      f"(oracle/c/allreduce_ref.c) on {cores} threads, median of {runs_c} runs",
            "numpy_1core": {"value": round(busbw(sub * 4, n, t_np), 3), "unit": "GB/s", "cores": 1,
                            "runs": runs_np}}


def decision_cost(L):
    ctxs = [(nr, 1 << k) for k in range(3, 31) for nr in (2, 4, 8)]
    s = L.bench_decide(ctxs, nwarm=10_000, ncalls=400_000)
    return {"calls": s["calls"], "p50_ns": s["p50_ns"], "p99_ns": s["p99_ns"],
            "timer_overhead_ns": s["timer_overhead_ns"], "batched_mean_ns": round(s["batched_mean_ns"], 2)}


# ------------------------------------------------------------------ polar
def run_polar(args):
    import numpy as np
    import torch

    import synth
    from paper_2603_11438_b200 import polar as L

    ws, rank, local = env_dist()
    real = ws > 1
    # test hook (tests/test_gpu_bench.py): every rank on GPU 0, so the N>1 path
    # (one process per rank, CUDA-IPC peers, max over ranks) runs on a 1-GPU box;
    # NCCL refuses two ranks on one GPU, so its baseline is skipped then
    shared = os.environ.get("POLAR_BENCH_SHARE_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    pg = None
    if real:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist

        def allgather(b):
            out = [None] * ws
            dist.all_gather_object(out, b)
            return out

        comm = L.Comm.init(ws, rank, local, allgather)
        n = ws
    else:
        comm = L.Comm.virtual(VIRTUAL_RANKS, local)
        n = VIRTUAL_RANKS
    if args.policy:
        with open(args.policy) as f:
            rows = [tuple(r) for r in json.load(f)["rows"]]
        L.set_policy(rows)
    count = S_BYTES // 4
    # symmetric buffers (zero-copy): nlocal tensors
    bufs = comm.mem_alloc_tensors(count, torch.float32)
    ranks_here = list(range(n)) if not real else [rank]
    host_inputs = [synth.gen("f32", count, r, cfg=2, dist="unif") for r in ranks_here]
    for b, x in zip(bufs, host_inputs):
        b.copy_(torch.from_numpy(x))
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    ptrs = [b.data_ptr() for b in bufs]

    def step():
        st = comm.allreduce_raw(ptrs, count, L.FLOAT32, L.SUM, sptr)
        if st != 0:
            raise L.PolarError(st, "polar_allreduce_v")

    def barrier():
        if pg:
            pg.barrier()

    def max_over_ranks(x):
        if not pg:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    comm.check()
    decision = comm.last_decision()
    launched_nch = comm.launched_channels()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = comm.launches()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    comm.check()
    launches = comm.launches() - launches0
    t_step = max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / args.steps)
    value = busbw(S_BYTES, n, t_step)

    # roofline of the (only) kernel of the step: the dispatched allreduce kernel
    peak, peak_src = load_peaks()
    if real:
        alg_bytes = 2 * S_BYTES   # per rank: read own S + write own S locally (NVLink bytes reported in busBW)
        bound_note = "per-rank local HBM; NVLink fraction = busBW / 900"
    else:
        alg_bytes = 2 * n * S_BYTES   # read every rank's input once, write every rank's output once
        bound_note = "all virtual ranks share one HBM"
    achieved = alg_bytes / t_step / 1e9
    traffic = load_traffic()
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes, "kernel": kernel_name(L, decision), "note": bound_note}
    if traffic and not real and traffic.get("workload") == "virtual8_f32_128MiB":
        roof["traffic"] = traffic.get("dram_bytes_per_launch")
        roof["traffic_source"] = traffic.get("source")

    # per-size sweep (C2 sizes), policy-selected
    sweep = {}
    for sz in C2_SIZES:
        cnt = sz // 4
        it = max(5, min(50, int(0.05 / max(1e-6, t_step * sz / S_BYTES))))
        for _ in range(3):
            comm.allreduce_raw(ptrs, cnt, L.FLOAT32, L.SUM, sptr)
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(it):
            comm.allreduce_raw(ptrs, cnt, L.FLOAT32, L.SUM, sptr)
        b.record(stream)
        b.synchronize()
        t = max_over_ranks(a.elapsed_time(b) / 1e3 / it)
        d = comm.last_decision()
        sweep[str(sz)] = {"busbw_gbs": round(busbw(sz, n, t), 1), "us": round(t * 1e6, 1),
                          "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels],
                          "launched_channels": comm.launched_channels()}
    comm.check()

    # e2e: through the C-ABI with HOST buffers; H2D + allreduce + D2H inside the timed region
    host = [torch.from_numpy(x).pin_memory() for x in host_inputs]
    e2e_steps = max(2, min(args.steps, 5))
    comm.allreduce_host(host, bufs)   # warm
    for hb, x in zip(host, host_inputs):
        hb.copy_(torch.from_numpy(x))
    barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(e2e_steps):
        comm.allreduce_host(host, bufs)
    b.record(stream)
    b.synchronize()
    t_e2e = max_over_ranks(a.elapsed_time(b) / 1e3 / e2e_steps)
    e2e = {"value": round(busbw(S_BYTES, n, t_e2e), 3), "unit": "GB/s",
           "h2d_bytes_per_step": len(bufs) * S_BYTES, "d2h_bytes_per_step": len(bufs) * S_BYTES,
           "ms_per_step": round(t_e2e * 1e3, 3)}

    # p2p probe: the measured peer-path roofline on the same buffers
    # (after the timed regions: the probe overwrites the peer buffers)
    probe = comm.p2p_probe(bufs, iters=3)
    if real:
        loc = probe[0]
        vals = [max_over_ranks(-loc["load_gbs"]), max_over_ranks(-loc["store_gbs"]), max_over_ranks(loc["pingpong_us"])]
        probe_out = {"load_gbs_min_over_ranks": round(-vals[0], 1), "store_gbs_min_over_ranks": round(-vals[1], 1),
                     "pingpong_us_max_over_ranks": round(vals[2], 2),
                     "what": "each rank reads / writes peer (r+1)%n's buffer through the peer mapping, all at once"}
    else:
        probe_out = {"load_gbs_sum": round(sum(p["load_gbs"] for p in probe), 1),
                     "store_gbs_sum": round(sum(p["store_gbs"] for p in probe), 1),
                     "pingpong_us_max": round(max(p["pingpong_us"] for p in probe), 2),
                     "what": "virtual ranks: every peer is local HBM; sums over the 8 concurrent ranks"}

    if real:
        # N > 1: the bound is the per-GPU NVLink path, not HBM.  Algorithmic bytes
        # per launch = each rank's egress 2(n-1)/n S (RS + AG), so achieved = busBW;
        # peak = the p2p probe's measured per-GPU load/store rate (min over ranks),
        # else the nominal 900 GB/s per direction.
        measured = min(probe_out["load_gbs_min_over_ranks"], probe_out["store_gbs_min_over_ranks"])
        use_probe = not shared and measured > 0
        npeak = round(measured, 1) if use_probe else 900.0
        hbm_roof = roof
        roof = {"bound": "nvlink", "achieved": round(value, 1), "peak": npeak, "unit": "GB/s",
                "frac": round(value / npeak, 4), "traffic": None,
                "peak_source": ("measured: p2p probe, min over ranks of peer load/store GB/s" if use_probe
                                else "nominal 900 GB/s per direction per GPU (B200 NVLink 5)"),
                "algorithmic_bytes_per_launch": int(S_BYTES * 2 * (n - 1) / n), "kernel": hbm_roof["kernel"],
                "note": "per-rank NVLink egress; the local-HBM view is in 'hbm'", "hbm": hbm_roof}

    nccl = None
    if real and not shared:
        nccl = time_nccl(args, bufs[0], count, n, stream)

    if rank == 0:
        cpu = cpu_baseline(n, count)
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": round(value / PAPER_8GPU_128MIB_DEFAULT, 4) if (real and n == 8) else None,
            "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(n, real), **({"shared_gpu_test": True} if shared else {})),
            "decision": {"algo": L.ALGO_NAMES[decision.algo], "proto": L.PROTO_NAMES[decision.proto],
                         "nchannels": decision.nchannels, "generation": decision.generation,
                         "launched_channels": launched_nch},
            "algbw_gbs": round(S_BYTES / t_step / 1e9, 2),
            "nvlink_frac": round(value / 900.0, 4) if real else None,
            "nvlink_frac_of_probe": (round(value / min(probe_out["load_gbs_min_over_ranks"],
                                                       probe_out["store_gbs_min_over_ranks"]), 4)
                                     if real and not shared else None),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(), "c2_sweep": sweep, "decision_cost_ns": decision_cost(L),
            "p2p_probe": probe_out,
        }
        if nccl:
            out["nccl_default"] = nccl
            out["speedup_vs_nccl"] = round(value / nccl["busbw_gbs"], 4)
        print(json.dumps(out), flush=True)
    comm.destroy()
    if pg:
        pg.destroy_process_group()


def kernel_name(L, d):
    return f"allreduce_kernel<f32,sum,{L.ALGO_NAMES[d.algo]},{L.PROTO_NAMES[d.proto]}>"


def time_nccl(args, buf, count, n, stream):
    """NCCL's default AllReduce (no NCCL_* overrides) on the same buffer."""
    import torch
    import torch.distributed as dist
    g = dist.new_group(backend="nccl")
    t = buf[:count]
    for _ in range(max(3, args.warmup)):
        dist.all_reduce(t, group=g)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(torch.cuda.current_stream())
    for _ in range(args.steps):
        dist.all_reduce(t, group=g)
    b.record(torch.cuda.current_stream())
    b.synchronize()
    x = torch.tensor([a.elapsed_time(b) / 1e3 / args.steps], dtype=torch.float64)
    dist.all_reduce(x, op=dist.ReduceOp.MAX)
    tt = float(x.item())
    return {"busbw_gbs": round(busbw(count * 4, n, tt), 2), "us": round(tt * 1e6, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="polar", choices=["polar", "reference"])
    ap.add_argument("--policy", default=os.environ.get("POLAR_POLICY", ""),
                    help="policy JSON ({'rows': [[coll,nranks,max_bytes,algo,proto,nch], ...]})")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_polar(args)


if __name__ == "__main__":
    main()
