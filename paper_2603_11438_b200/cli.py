"""polar operator CLI (host side; SPEC.md cli module L560-592 analog).

    python -m paper_2603_11438_b200.cli validate policies/b200_virtual.json
    python -m paper_2603_11438_b200.cli explain  policies/listing1_size_aware.json --nranks 8
    python -m paper_2603_11438_b200.cli decide   policies/c1_fixed_threshold.json --nranks 2 --bytes 65536
    python -m paper_2603_11438_b200.cli bench-decide [--calls 400000]
    python -m paper_2603_11438_b200.cli reload-test [--threads 4 --calls 400000 --swaps 1000]
    python -m paper_2603_11438_b200.cli adaptive-sim [--windows 30 --contention 10:20]

Every command goes through libpolar's C ABI (validation, decisions, benches and
the controller all run in the library).  Exit status: 0 ok, 1 usage, 3 rejected
policy, 4 runtime error.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

from paper_2603_11438_b200 import polar as L

SIZES = [8 << k for k in range(0, 28)]   # 8 B .. 1 GiB


def load_rows(path):
    with open(path) as f:
        d = json.load(f)
    rows = d["rows"] if isinstance(d, dict) else d
    return [tuple(int(x) for x in r) for r in rows]


def fmt_size(b):
    for unit, sh in (("GiB", 30), ("MiB", 20), ("KiB", 10)):
        if b >= 1 << sh and b % (1 << sh) == 0:
            return f"{b >> sh} {unit}"
    return f"{b} B"


def cmd_validate(a):
    rows = load_rows(a.policy)
    st, gen = L.set_policy_status(rows)
    name = L.STATUS_NAMES[st]
    print(f"{a.policy}: {len(rows)} rows -> {name}" + (f" (generation {gen})" if st == L.OK else ""))
    return 0 if st == L.OK else 3


def cmd_explain(a):
    rows = load_rows(a.policy) if a.policy != "noop" else []
    st, _ = L.set_policy_status(rows)
    if st != L.OK:
        print(f"rejected: {L.STATUS_NAMES[st]}")
        return 3
    coll = {"allreduce": 0, "allgather": 1, "broadcast": 2, "reducescatter": 3}[a.coll]
    out = L.decide_batch([(a.nranks, s) for s in SIZES], coll=coll)
    print(f"# {a.policy}, {a.coll}, nranks={a.nranks}")
    print(f"{'bytes':>10}  algo      proto   nch  flags")
    for s, (algo, proto, nch, gen, flags) in zip(SIZES, out):
        print(f"{fmt_size(s):>10}  {L.ALGO_NAMES[algo]:8s}  {L.PROTO_NAMES[proto]:6s}  {nch:3d}  {flags}")
    return 0


def cmd_decide(a):
    rows = load_rows(a.policy) if a.policy != "noop" else []
    st, _ = L.set_policy_status(rows)
    if st != L.OK:
        print(f"rejected: {L.STATUS_NAMES[st]}")
        return 3
    d = L.decide(a.nranks, a.bytes)
    print(json.dumps({"algo": L.ALGO_NAMES[d.algo], "proto": L.PROTO_NAMES[d.proto], "nchannels": d.nchannels,
                      "generation": d.generation, "flags": d.flags}))
    return 0


def cmd_bench_decide(a):
    if a.policy:
        L.set_policy(load_rows(a.policy))
    ctxs = [(nr, 1 << k) for k in range(3, 31) for nr in (2, 4, 8)]
    s = L.bench_decide(ctxs, nwarm=10_000, ncalls=a.calls)
    print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in s.items()}))
    return 0


def cmd_reload_test(a):
    A = [(0, 0, 32768, L.TREE, L.SIMPLE, 4), (0, 0, 2**64 - 1, L.RING, L.SIMPLE, 4)]
    B = [(0, 0, 4 << 20, L.ONESHOT, L.LL, 2), (0, 0, 2**64 - 1, L.TWOSHOT, L.SIMPLE, 32)]
    s = L.bench_swap(A, B, nthreads=a.threads, calls_per_thread=a.calls // a.threads, nswaps=a.swaps)
    print(json.dumps({k: round(v, 1) if isinstance(v, float) else v for k, v in s.items()}))
    ok = s["calls"] == s["issued"] and s["invalid"] == 0 and s["nonmonotonic"] == 0 and s["rejected_changed"] == 0
    print("zero-loss:", "PASS" if ok else "FAIL")
    return 0 if ok else 4


def cmd_adaptive_sim(a):
    lo, hi = (int(x) for x in a.contention.split(":")) if a.contention else (0, 0)
    table = []
    for w in range(a.windows):
        k = a.spike if lo <= w < hi else 1.0
        table.append([0.0] + [a.base_ns * (0.2 + 1.6 / c) * k for c in range(1, 33)])
    if a.no_profiler:
        table = [[math.nan] * 33 for _ in range(a.windows)]
    p = L.adaptive_params(enabled=not a.no_profiler, period=a.period, c_min=a.c_min,
                          contention_factor=a.factor)
    tr = L.adaptive_simulate(p, a.cap, table)
    print(json.dumps({"period_calls": a.period, "channels_after_each_window": tr}))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="polar-cli", description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("validate")
    v.add_argument("policy")
    e = sub.add_parser("explain")
    e.add_argument("policy", help="policy JSON or 'noop'")
    e.add_argument("--nranks", type=int, default=8)
    e.add_argument("--coll", default="allreduce", choices=["allreduce", "allgather", "broadcast", "reducescatter"])
    d = sub.add_parser("decide")
    d.add_argument("policy")
    d.add_argument("--nranks", type=int, required=True)
    d.add_argument("--bytes", type=int, required=True)
    b = sub.add_parser("bench-decide")
    b.add_argument("--calls", type=int, default=400_000)
    b.add_argument("--policy", default="")
    r = sub.add_parser("reload-test")
    r.add_argument("--threads", type=int, default=4)
    r.add_argument("--calls", type=int, default=400_000)
    r.add_argument("--swaps", type=int, default=1000)
    s = sub.add_parser("adaptive-sim")
    s.add_argument("--windows", type=int, default=30)
    s.add_argument("--contention", default="10:20", help="window range [lo:hi) with a latency spike")
    s.add_argument("--spike", type=float, default=10.0)
    s.add_argument("--cap", type=int, default=12)
    s.add_argument("--c-min", type=int, default=2)
    s.add_argument("--period", type=int, default=10_000)
    s.add_argument("--factor", type=float, default=4.0)
    s.add_argument("--base-ns", type=float, default=400e3)
    s.add_argument("--no-profiler", action="store_true")
    a = ap.parse_args(argv)
    try:
        return {"validate": cmd_validate, "explain": cmd_explain, "decide": cmd_decide,
                "bench-decide": cmd_bench_decide, "reload-test": cmd_reload_test,
                "adaptive-sim": cmd_adaptive_sim}[a.cmd](a)
    except (OSError, ValueError, KeyError) as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 1
    except L.PolarError as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
