"""bench.py — BASELINE.json metric on B200: AllReduce busBW (GB/s), policy-selected.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl polar|reference]

N = 1 (no torchrun): 8 VIRTUAL ranks on cuda:0,
    BASELINE config 2's largest size: fp32 sum, 128 MiB per rank, the decision
    made by the policy hook each call.  All ranks' traffic shares one HBM, so the
    roofline is HBM: every step must read n x S and write n x S bytes.
N > 1 (torchrun, one rank per GPU): real ranks over NVLink/NVSwitch with CUDA
    IPC peer mappings, same message; NCCL's default AllReduce (ctypes
    libnccl.so.2, no NCCL_* overrides, its choice read from its TUNING log) is
    timed on the SAME buffers and stream for the "speedup vs NCCL default" half
    of the metric, over the whole 4 KiB - 1 GiB sweep (BASELINE configs 2-3).

A step = one policy-selected polar AllReduce (decide + one kernel launch) of the
workload.  Timing: W warm-up steps, then K steps between CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.  The
n x 128 MiB inputs exceed the 126 MB L2, so no flush is needed between steps.
After the timed region the same buffers are re-filled, one step of the same
launch configuration runs again and sampled windows are checked against the
oracle (`parity`; a busBW is never printed for wrong data without saying so).
--impl reference times the CPU oracle (oracle/) on the host cores instead.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AllReduce busBW GB/s vs size at 2/4/8 B200; speedup vs NCCL default"
S_BYTES = 128 << 20            # BASELINE config 2 headline size (per rank)
VIRTUAL_RANKS = 8
C2_SIZES = [4 << 20, 8 << 20, 16 << 20, 32 << 20, 64 << 20, 128 << 20]
NVLINK_SIZES = [(4 << 10) << k for k in range(19)]    # 4 KiB .. 1 GiB (BASELINE config 3)
L2_BYTES = 126 << 20
NVLINK_GBS = 900.0             # per direction per GPU (PAPER.md L414 / BJ; R11)
PAPER_8GPU_128MIB_DEFAULT = 596.9   # PAPER.md Table 2 L559 (8x B300, NCCL NVLS) — context
U64_MAX = 2**64 - 1


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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


# ------------------------------------------------------------------ CPU oracle legs
def _oracle_workload(n, count):
    import synth
    return synth.gen_ranks("f32", count, n, cfg=2, dist="unif")


def _sample_text(n, count, cores, extra=""):
    return (f"{n} ranks x {count} f32 ({count * 4 / 2**20:.1f} MiB/rank) of the {S_BYTES >> 20} MiB/rank C2 workload, "
            f"plain C oracle (oracle/c/allreduce_ref.c) on {cores} threads of '{cpu_model()}'{extra}")


def run_reference(args):
    """The CPU oracle, as it stands, timed on the host cores (rank 0 only).
    Each step is the FULL C2 workload (n x 128 MiB) when K + W steps fit the
    ~2-minute budget, else the same leading fraction of every rank's input."""
    ws, rank, _ = env_dist()
    if rank != 0:
        return
    from oracle import cref

    n = VIRTUAL_RANKS if ws == 1 else ws
    cores = len(os.sched_getaffinity(0))
    count_full = S_BYTES // 4
    xs_full = _oracle_workload(n, count_full)

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
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(n, ws > 1),
        "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": _sample_text(n, count, cores, f", mean of {args.steps} steps"),
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def workload_config(n, real):
    return {
        "workload": (f"C2 {n}-rank AllReduce fp32 sum, {S_BYTES >> 20} MiB per rank, policy-selected, "
                     + ("real ranks (1 per GPU, NVLink)" if real else f"{n} virtual ranks on 1 B200")),
        "nranks": n, "bytes_per_rank": S_BYTES, "op": "sum", "dtype": "f32",
        "buffers": "symmetric (polar_mem_alloc: registered, zero-copy two-shot)",
        "l2": f"inputs larger than L2 ({n} x {S_BYTES >> 20} MiB resident), no flush",
        "prewarm": "after the W warm-up steps, untimed steps for ~0.25 s (clock ramp out of idle)",
    }


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


def cpu_baseline(n, count, xs=None):
    """The oracle timed on the host on the SAME workload the reference arm times
    (the full n x 128 MiB C2 message): the plain threaded C oracle on every core
    this process may run on, and the numpy oracle on 1 core on
    a 1/16 sample of it (it needs ~0.5 s per MiB of ranks' input)."""
    from oracle import allreduce as orc
    from oracle import cref
    xs = xs if xs is not None else _oracle_workload(n, count)
    cores = len(os.sched_getaffinity(0))
    t_c, runs_c = _time_oracle(lambda: cref.allreduce(xs, "f32", "sum", cores), 10.0, max_runs=20)
    sub = count // 16
    xsub = [x[:sub] for x in xs]
    t_np, runs_np = _time_oracle(lambda: orc.allreduce(xsub, "f32", "sum"), 5.0)
    return {"value": round(busbw(count * 4, n, t_c), 3), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": _sample_text(n, count, cores, f", median of {runs_c} runs"), "cpu_model": cpu_model(),
            "numpy_1core": {"value": round(busbw(sub * 4, n, t_np), 3), "unit": "GB/s", "cores": 1,
                            "runs": runs_np, "sample": f"{n} ranks x {sub} f32 (1/16 of the workload)"}}


def decision_cost(L):
    ctxs = [(nr, 1 << k) for k in range(3, 31) for nr in (2, 4, 8)]
    s = L.bench_decide(ctxs, nwarm=10_000, ncalls=400_000)
    return {"calls": s["calls"], "p50_ns": s["p50_ns"], "p99_ns": s["p99_ns"],
            "timer_overhead_ns": s["timer_overhead_ns"], "batched_mean_ns": round(s["batched_mean_ns"], 2)}


# ------------------------------------------------------------------ parity of the timed buffers
def parity_windows(count, k=16, w=2048, seed=5):
    import numpy as np
    rng = np.random.default_rng(seed)
    return [(0, w), (count - w - 3, count)] + [(int(s), int(s) + w) for s in rng.integers(0, count - w, k)]


def check_parity(L, comm, bufs, host_inputs, ranks_here, n, count, step, gather):
    """Re-fill the timed buffers with their inputs, run ONE step of the same
    launch configuration, and compare sampled windows with the oracle (rank-
    ordered fold, oracle/allreduce.py).  Two-shot / one-shot results must be
    bit-exact (R2); ring / tree within 1e-6 n sum|x|.  gather(obj) -> list over
    processes (identity for one process).  Returns the `parity` object."""
    import numpy as np
    import torch
    from oracle import allreduce as orc
    wins = parity_windows(count)
    for b, x in zip(bufs, host_inputs):
        b.copy_(torch.from_numpy(x))
    torch.cuda.synchronize()
    step()
    torch.cuda.synchronize()
    comm.check()
    d = comm.last_decision()
    exact = L.ALGO_NAMES[d.algo] in ("oneshot", "twoshot")
    # every rank's input windows, rank order
    mine = {r: [x[lo:hi].copy() for lo, hi in wins] for r, x in zip(ranks_here, host_inputs)}
    allwin = {}
    for part in gather(mine):
        allwin.update(part)
    ok, worst, hashes = True, 0.0, []
    for b in bufs:
        got = b.cpu().numpy()
        hb = hashlib.sha1()
        for k, (lo, hi) in enumerate(wins):
            xs = [allwin[r][k] for r in range(n)]
            exp = orc.allreduce(xs, "f32", "sum")
            g = got[lo:hi]
            hb.update(g.tobytes())
            if exact:
                ok = ok and bool(np.array_equal(g.view(np.uint32), exp.view(np.uint32)))
            else:
                bound = 1e-6 * n * np.sum(np.abs(np.stack(xs).astype(np.float64)), axis=0)
                err = np.abs(g.astype(np.float64) - exp.astype(np.float64))
                worst = max(worst, float(np.max(err / np.maximum(bound, 1e-300))))
                ok = ok and bool(np.all(err <= bound))
        hashes.append(hb.hexdigest())
    alls = gather({"ok": ok, "hashes": hashes, "worst": worst})
    identical = len({h for a in alls for h in a["hashes"]}) == 1
    ok_all = all(a["ok"] for a in alls) and identical
    return {"ok": bool(ok_all), "windows": len(wins), "elements_per_rank": sum(hi - lo for lo, hi in wins),
            "rule": "bit-exact vs the rank-ordered oracle" if exact else "|y - y*| <= 1e-6 n sum|x| (R2)",
            "max_err_over_bound": round(max(a["worst"] for a in alls), 6) if not exact else 0.0,
            "ranks_identical": identical,
            "what": "same buffers and launch configuration as the timed steps, re-filled with their inputs"}


# ------------------------------------------------------------------ polar
def run_polar(args):
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
    nccl_log = None
    if real and not shared:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import nccl_ctypes
        nccl_log = nccl_ctypes.enable_tuning_log(os.path.join(tempfile.gettempdir(), f"polar_nccl_tuning.r{rank}"))
    pg = None
    if real:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist

        def allgather(b):
            out = [None] * ws
            dist.all_gather_object(out, b)
            return out

        comm = L.Comm.init(ws, rank, local, L.torch_allgather(dist, ws))
        n = ws
        # LL128's premise over this transport (a real comm refuses LL128 until it passed)
        t0 = time.perf_counter()
        torn, reads = comm.probe_ll128(iters=2000)
        ll128_probe = {"torn_lanes": torn, "lane_reads": reads, "accepted": torn == 0 and reads > 0,
                       "s": round(time.perf_counter() - t0, 3)}
    else:
        comm = L.Comm.virtual(VIRTUAL_RANKS, local)
        n = VIRTUAL_RANKS
        ll128_probe = None

        def allgather(b):
            return [b]
    if args.policy:
        with open(args.policy) as f:
            rows = [tuple(r) for r in json.load(f)["rows"]]
        L.set_policy(rows)
    count = S_BYTES // 4
    max_bytes = S_BYTES if not real else (16 << 20 if shared else max(NVLINK_SIZES))
    # symmetric buffers (zero-copy): nlocal tensors; the timed message is their first 128 MiB
    big = comm.mem_alloc_tensors(max(count, max_bytes // 4), torch.float32)
    bufs = [b[:count] for b in big]
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

    t_w = time.perf_counter()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # clock ramp: the GPU may come out of idle (120 MHz) at the start of the run;
    # after the W warm-up steps keep stepping (untimed) for ~0.25 s so the timed
    # steps run at full clock (measured: with 5 warm-up steps after idle time
    # the timed steps came out ~3 % slow).  The same count on every rank (the
    # steps are collectives).
    t_est = (time.perf_counter() - t_w) / max(1, args.warmup)
    prewarm = int(max_over_ranks(float(min(4000, int(0.25 / max(t_est, 1e-5))))))
    for _ in range(prewarm):
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
        torch.cuda.nvtx.range_push("timed")     # ncu --nvtx --nvtx-include "timed/": the timed launches only
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    barrier()
    comm.check()
    launches = comm.launches() - launches0
    t_step = max_over_ranks(ev0.elapsed_time(ev1) / 1e3 / args.steps)
    value = busbw(S_BYTES, n, t_step)

    # the timed buffers, re-filled, one more step of the same configuration, checked
    parity = check_parity(L, comm, bufs, host_inputs, ranks_here, n, count, step, allgather)

    # real comms: the north_star call on an UNREGISTERED torch tensor of the same
    # size (two-shot through the pipelined bounce region) against the registered
    # buffers timed above
    unreg = None
    if real:
        plain = torch.from_numpy(host_inputs[0]).cuda()
        pp = [plain.data_ptr()]

        def ustep():
            st = comm.allreduce_raw(pp, count, L.FLOAT32, L.SUM, sptr)
            if st != 0:
                raise L.PolarError(st, "polar_allreduce (unregistered)")
        for _ in range(args.warmup):
            ustep()
        torch.cuda.synchronize()
        barrier()
        uk = max(5, min(args.steps, 50))
        tu = max_over_ranks(_time_calls(ustep, uk, stream))
        comm.check()
        unreg = {"busbw_gbs": round(busbw(S_BYTES, n, tu), 2), "us": round(tu * 1e6, 1), "steps": uk,
                 "ratio_vs_registered": round(tu / t_step, 4),
                 "path": "torch tensor, not registered: two-shot via the bounce region, copy-in / kernel / copy-out "
                         "pipelined over 2 x POLAR_BOUNCE/2 halves"}
        # the same tensor with auto-registration (polar_comm_autoreg): one IPC-handle
        # all-gather per call on the host, zero-copy on the device
        comm.autoreg(True, 1 << 20)
        for _ in range(args.warmup):
            ustep()
        torch.cuda.synchronize()
        barrier()
        ta = max_over_ranks(_time_calls(ustep, uk, stream))
        comm.check()
        # one more auto-registered call on the re-filled tensor: bitwise equal to
        # the registered buffer's checked result (same inputs, same kernel), on every rank
        plain.copy_(torch.from_numpy(host_inputs[0]))
        torch.cuda.synchronize()
        barrier()
        ustep()
        torch.cuda.synchronize()
        comm.check()
        ars = comm.autoreg_stats()
        comm.autoreg(False)
        same = bool(torch.equal(plain.view(torch.int32), bufs[0].view(torch.int32)))
        got = allgather(hashlib.sha1(plain.cpu().numpy().tobytes()).hexdigest())
        unreg["autoreg"] = {"busbw_gbs": round(busbw(S_BYTES, n, ta), 2), "us": round(ta * 1e6, 1), "steps": uk,
                            "ratio_vs_registered": round(ta / t_step, 4), "stats": ars,
                            "parity": {"equal_to_checked_registered_result": same,
                                       "ranks_identical": len(set(got)) == 1},
                            "path": "the same tensor, auto-registered: per call one host all-gather of "
                                    "{IPC handle, buffer id, offset}, peer allocations opened once, zero-copy two-shot"}
        del plain

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

    # per-size sweep
    if real:
        sweep = nvlink_sweep(args, L, comm, big, n, rank, stream, barrier, max_over_ranks, allgather, shared,
                             nccl_log)
    else:
        sweep = c2_sweep_virtual(L, comm, big, n, stream, t_step)
        size_sweep = {"policy": "the active table (built-in default unless --policy): NVLink-oriented, "
                                "one-shot below 1 MiB (DESIGN.md §4)",
                      "sizes": size_sweep_virtual(L, comm, n, stream, peak)}
        tuned = os.path.join(ROOT, "policies", "b200_virtual.json")
        if os.path.exists(tuned) and not args.policy:
            with open(tuned) as f:
                rows = [tuple(r) for r in json.load(f)["rows"]]
            size_sweep["tuned_virtual"] = {
                "policy": "policies/b200_virtual.json (per-size choice measured on virtual ranks)",
                "sizes": size_sweep_virtual(L, comm, n, stream, peak, table=rows)}
    comm.check()
    # virtual N=1: every algorithm's Simple kernel at the C2 size against the
    # same HBM roofline (ring / tree on both transports: clusters, and the
    # peer-memory FIFOs that real comms run)
    algos = None if real else algorithm_records(L, big, n, stream, peak_for_records())

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
    e2e["pcie"] = pcie_roofline(torch, len(bufs) * S_BYTES, t_e2e, max_over_ranks)

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
        npeak = round(measured, 1) if use_probe else NVLINK_GBS
        hbm_roof = roof
        roof = {"bound": "nvlink", "achieved": round(value, 1), "peak": npeak, "unit": "GB/s",
                "frac": round(value / npeak, 4), "traffic": None,
                "peak_source": ("measured: p2p probe, min over ranks of peer load/store GB/s" if use_probe
                                else "nominal 900 GB/s per direction per GPU (B200 NVLink 5)"),
                "algorithmic_bytes_per_launch": int(S_BYTES * 2 * (n - 1) / n), "kernel": hbm_roof["kernel"],
                "note": "per-rank NVLink egress; the local-HBM view is in 'hbm'", "hbm": hbm_roof}
        if use_probe:
            for v in sweep["sizes"].values():
                v["frac_of_probe"] = round(v["polar_busbw_gbs"] / npeak, 4)

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
            "parity": parity,
            "algbw_gbs": round(S_BYTES / t_step / 1e9, 2),
            "nvlink_frac": round(value / NVLINK_GBS, 4) if real else None,
            "nvlink_frac_of_probe": (round(value / min(probe_out["load_gbs_min_over_ranks"],
                                                       probe_out["store_gbs_min_over_ranks"]), 4)
                                     if real and not shared else None),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(), ("nvlink_sweep" if real else "c2_sweep"): sweep,
            "decision_cost_ns": decision_cost(L), "p2p_probe": probe_out,
        }
        if algos is not None:
            out["algorithms"] = algos
        if not real:
            out["size_sweep"] = size_sweep
        if ll128_probe is not None:
            out["ll128_probe"] = ll128_probe
        if unreg is not None:
            out["unregistered"] = unreg
        if real and sweep.get("nccl_version"):
            nd = sweep["sizes"].get(str(S_BYTES), {})
            if nd.get("nccl_busbw_gbs"):
                out["nccl_default"] = {"busbw_gbs": nd["nccl_busbw_gbs"], "us": nd["nccl_us"],
                                       "choice": nd.get("nccl_choice"), "version": sweep["nccl_version"]}
                out["speedup_vs_nccl"] = round(value / nd["nccl_busbw_gbs"], 4)
        print(json.dumps(out), flush=True)
    comm.destroy()
    if pg:
        pg.destroy_process_group()


def kernel_name(L, d):
    return f"allreduce_kernel<f32,sum,{L.ALGO_NAMES[d.algo]},{L.PROTO_NAMES[d.proto]}>"


def pcie_roofline(torch, nbytes, t_e2e, max_over_ranks):
    """e2e bound: the step moves nbytes host->device and nbytes back over this
    GPU's PCIe link; measured here with pinned copies (each direction alone, and
    both at once on two streams) so the e2e time has its own floor."""
    n = min(nbytes, 256 << 20)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    t_h2d = timed(lambda: d.copy_(h, non_blocking=True))
    t_d2h = timed(lambda: h.copy_(d, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    t_both = timed(both)
    h2d, d2h, bidir = n / t_h2d / 1e9, n / t_d2h / 1e9, n / t_both / 1e9
    floor = nbytes / (bidir * 1e9)          # both directions overlapped at the measured concurrent rate
    return {"h2d_gbs": round(h2d, 1), "d2h_gbs": round(d2h, 1), "bidir_each_gbs": round(bidir, 1),
            "floor_ms": round(floor * 1e3, 3), "frac": round(floor / t_e2e, 4),
            "what": "e2e floor = bytes each way / concurrent per-direction PCIe rate (pinned copies, this GPU)"}


def _time_calls(fn, iters, stream, flush=None):
    """Mean device time of one call: back to back between two events, or (flush
    given) each call between its own events after an L2 flush."""
    import torch
    if flush is None:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(iters):
            fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / 1e3 / iters
    tot = 0.0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        flush()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    for a, b in evs:
        tot += a.elapsed_time(b) / 1e3
    return tot / iters


def peak_for_records():
    return load_peaks()[0]


def algorithm_records(L, big, n, stream, peak):
    """Each algorithm's Simple kernel, forced, on the bench's own buffers at the
    C2 size (8 virtual ranks x 128 MiB, f32 and bf16), back to back: us, busBW
    and the fraction of the HBM copy peak its algorithmic bytes (2 n S: every
    input read once, every output written once) reach.  Ring and tree run on
    both virtual transports: "cluster" (one thread-block cluster per channel,
    DSMEM hops; the default) and "peer" (the FIFO kernels through global
    memory, POLAR_CLUSTER=0), whatever the size."""
    import torch
    out = {}
    comms = {}
    old = os.environ.get("POLAR_CLUSTER")
    for tr, env in (("cluster", "1"), ("peer", "0")):
        os.environ["POLAR_CLUSTER"] = env
        os.environ["POLAR_CLUSTER_TREE_MAX"] = str(1 << 40) if tr == "cluster" else str(16 << 20)
        comms[tr] = L.Comm.virtual(n, torch.cuda.current_device())
    if old is None:
        os.environ.pop("POLAR_CLUSTER", None)
    else:
        os.environ["POLAR_CLUSTER"] = old
    os.environ.pop("POLAR_CLUSTER_TREE_MAX", None)
    sptr = stream.cuda_stream
    ptrs = [b.data_ptr() for b in big]
    try:
        for dt, code, es in (("f32", L.FLOAT32, 4), ("bf16", L.BFLOAT16, 2)):
            cnt = S_BYTES // es
            for algo, tr in (("twoshot", "peer"), ("ring", "cluster"), ("ring", "peer"),
                             ("tree", "cluster"), ("tree", "peer")):
                c = comms[tr]
                dec = L.Decision(L.ALGO_CODES[algo], L.SIMPLE, 32, 0)

                def call():
                    st = c.allreduce_forced_raw(ptrs, cnt, code, L.SUM, dec, sptr)
                    if st != 0:
                        raise L.PolarError(st, "polar_allreduce_forced")
                for _ in range(3):
                    call()
                torch.cuda.synchronize()
                t = _time_calls(call, 10, stream)
                c.check()
                out[f"{algo}/{tr}/{dt}"] = {
                    "us": round(t * 1e6, 1), "busbw_gbs": round(busbw(S_BYTES, n, t), 1),
                    "hbm_frac": round(2 * n * S_BYTES / t / 1e9 / peak, 4),
                    "transport": c.transport(), "launched_channels": c.launched_channels()}
    finally:
        for c in comms.values():
            c.destroy()
    return out


def c2_sweep_virtual(L, comm, big, n, stream, t_step):
    """C2 sizes (4-128 MiB per rank), policy-selected, 8 virtual ranks.  Where
    the n ranks' buffers fit in twice the L2 (n S <= 252 MB) every call is timed
    alone after an L2 flush (a 256 MiB write), so no point is an L2 number."""
    import torch
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sptr = stream.cuda_stream
    out = {}
    for sz in C2_SIZES:
        cnt = sz // 4
        ptrs = [b.data_ptr() for b in big]
        it = max(5, min(50, int(0.05 / max(1e-6, t_step * sz / S_BYTES))))

        def call():
            st = comm.allreduce_raw(ptrs, cnt, L.FLOAT32, L.SUM, sptr)
            if st != 0:
                raise L.PolarError(st, "polar_allreduce_v")
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        flushed = n * sz <= 2 * L2_BYTES
        t = _time_calls(call, it, stream, flush=(lambda: flush_buf.zero_()) if flushed else None)
        d = comm.last_decision()
        out[str(sz)] = {"busbw_gbs": round(busbw(sz, n, t), 1), "us": round(t * 1e6, 1),
                        "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels],
                        "launched_channels": comm.launched_channels(),
                        "l2": "flushed before every call" if flushed else "n x S > 2 x L2, back to back"}
    return out


def size_sweep_virtual(L, comm, n, stream, peak, table=None):
    """north_star's size range at N = 1: 4 KiB - 1 GiB per rank (x4 steps), 8
    virtual ranks, f32 sum, policy-selected; algBW, busBW and the fraction of
    the HBM copy peak by the 2 n S yardstick.  Points with n S <= 2 x L2 are
    timed one call at a time after an L2 flush (no L2-resident number);
    larger ones back to back."""
    import torch
    sizes = [(4 << 10) << (2 * k) for k in range(10)]
    top = max(sizes)
    saved = None
    if table is not None:
        saved = L.get_policy()[0]
        L.set_policy(table)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    big = torch.zeros(n * (top // 4), dtype=torch.float32, device="cuda")
    sptr = stream.cuda_stream
    out = {}
    for sz in sizes:
        cnt = sz // 4
        ptrs = [big[r * (top // 4):].data_ptr() for r in range(n)]

        def call():
            st = comm.allreduce_raw(ptrs, cnt, L.FLOAT32, L.SUM, sptr)
            if st != 0:
                raise L.PolarError(st, "polar_allreduce_v")
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        flushed = n * sz <= 2 * L2_BYTES
        it = 20 if flushed else max(5, min(20, int(0.05 / (2 * n * sz / 6e12))))
        t = _time_calls(call, it, stream, flush=(lambda: flush_buf.zero_()) if flushed else None)
        d = comm.last_decision()
        out[str(sz)] = {"algbw_gbs": round(sz / t / 1e9, 2), "busbw_gbs": round(busbw(sz, n, t), 2),
                        "us": round(t * 1e6, 2), "hbm_frac": round(2 * n * sz / t / 1e9 / peak, 4),
                        "decision": [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels],
                        "l2": "flushed before every call" if flushed else "n x S > 2 x L2, back to back"}
    del big, flush_buf
    torch.cuda.empty_cache()
    if saved is not None:
        L.set_policy(saved)
    return out


def nvlink_sweep(args, L, comm, big, n, rank, stream, barrier, max_over_ranks, allgather, shared, nccl_log):
    """N > 1: busBW per size, 4 KiB - 1 GiB, on the same symmetric buffers and
    stream: polar with the active table, polar with `bad_channels` (PAPER.md
    L581: every size at 1 channel, algorithm / protocol deferred), polar with a
    tuned table if policies/b200_nvlink<n>.json exists, and NCCL's default
    (ctypes libnccl, no overrides; its algorithm / protocol from its TUNING
    log).  Back-to-back calls like nccl-tests; sizes with S <= L2 are labelled."""
    import torch
    sptr = stream.cuda_stream
    ptr = big[0].data_ptr()
    sizes = [s for s in NVLINK_SIZES if s <= (16 << 20 if shared else max(NVLINK_SIZES))]
    nccl = ncomm = None
    version = None
    if not shared:
        try:
            import nccl_ctypes
            nccl = nccl_ctypes.Nccl()
            version = nccl.version()
            uid = allgather(nccl.unique_id() if rank == 0 else None)[0]
            ncomm = nccl.init(n, uid, rank)
        except Exception as e:  # noqa: BLE001
            nccl, version = None, f"unavailable: {e}"
    prev_rows, _ = L.get_policy()
    tuned_path = os.path.join(ROOT, "policies", f"b200_nvlink{n}.json")
    tuned = single = None
    if os.path.exists(tuned_path):
        with open(tuned_path) as f:
            doc = json.load(f)
        tuned = [tuple(r) for r in doc["rows"]]
        if doc.get("best_single"):
            a_, p_, c_ = doc["best_single"]
            single = [(0, 0, U64_MAX, L.ALGO_CODES[a_], L.PROTO_CODES[p_], int(c_))]
    # the paper's comparison points: the active table, bad_channels (E11, PAPER.md
    # L581-583), the measured per-size table and the best single global choice (E10, L566-568)
    variants = [("polar", prev_rows), ("bad_channels", [(0, 0, U64_MAX, L.UNSET, L.UNSET, 1)])]
    if tuned:
        variants.append(("tuned", tuned))
    if single:
        variants.append(("best_single", single))
    if comm.nvls_info()[0] and os.environ.get("POLAR_BENCH_NVLS") == "1":
        # the switch reduction, where the node grants a multicast object (f1; NCCL's
        # own default on the paper's node).  Opt-in: the NVLS
        # kernels have never run on this pool (no multicast object), and a failing
        # variant must not cost the rest of the bench line.
        variants.append(("nvls", [(0, 0, U64_MAX, L.NVLS, L.SIMPLE, 32)]))

    def polar_call(cnt):
        st = comm.allreduce_raw([ptr], cnt, L.FLOAT32, L.SUM, sptr)
        if st != 0:
            raise L.PolarError(st, "polar_allreduce")

    out = {}
    for sz in sizes:
        cnt = sz // 4
        rec = {"l2_resident_possible": sz <= L2_BYTES}
        for name, rows in variants:
            L.set_policy(rows)
            for _ in range(3):
                polar_call(cnt)
            torch.cuda.synchronize()
            # the iteration count must be identical on every rank (collective calls)
            t1 = max_over_ranks(_time_calls(lambda: polar_call(cnt), 1, stream))
            it = int(max(5, min(200, 2e-3 / max(t1, 1e-7))))
            barrier()
            t = max_over_ranks(_time_calls(lambda: polar_call(cnt), it, stream))
            d = comm.last_decision()
            rec[f"{name}_busbw_gbs"] = round(busbw(sz, n, t), 4)
            rec[f"{name}_us"] = round(t * 1e6, 2)
            rec[f"{name}_decision"] = [L.ALGO_NAMES[d.algo], L.PROTO_NAMES[d.proto], d.nchannels]
        L.set_policy(prev_rows)
        if nccl is not None:
            def nccl_call():
                nccl.allreduce(ncomm, ptr, cnt, 7, sptr)
            for _ in range(3):
                nccl_call()
            torch.cuda.synchronize()
            t1 = max_over_ranks(_time_calls(nccl_call, 1, stream))
            it = int(max(5, min(200, 2e-3 / max(t1, 1e-7))))
            barrier()
            t = max_over_ranks(_time_calls(nccl_call, it, stream))
            rec["nccl_busbw_gbs"] = round(busbw(sz, n, t), 4)
            rec["nccl_us"] = round(t * 1e6, 2)
            rec["speedup_vs_nccl"] = round(rec["polar_busbw_gbs"] / rec["nccl_busbw_gbs"], 4)
        rec["nvlink_frac"] = round(rec["polar_busbw_gbs"] / NVLINK_GBS, 6)
        out[str(sz)] = rec
    comm.check()
    if nccl is not None:
        torch.cuda.synchronize()
        choices = nccl_ctypes.parse_tuning(nccl_log) if nccl_log else {}
        for sz in sizes:
            if sz in choices:
                out[str(sz)]["nccl_choice"] = list(choices[sz])
        nccl.destroy(ncomm)
    # the paper's E10 (best single global choice) needs the full grid: scripts/tune_policy.py --real
    best = None
    if out:
        wins = [s for s, r in out.items() if "speedup_vs_nccl" in r and r["speedup_vs_nccl"] > 1.0
                and (4 << 20) <= int(s) <= (128 << 20)]
        best = {"beats_nccl_in_4_128MiB_at": wins}
    return {"sizes": out, "nccl_version": version, "summary": best,
            "variants": [v[0] for v in variants] + (["nccl_default"] if nccl is not None else [])}


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
