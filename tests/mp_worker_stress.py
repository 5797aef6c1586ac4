"""One rank of a time-bounded random stress of the REAL-comm path (one process
per rank, CUDA IPC, sys-scope flags, entry / exit handshakes), launched by
torchrun; the multi-process counterpart of tests/test_gpu_stress.py.

Every rank draws the same configuration sequence from a shared seed (the calls
are collective): algorithm x protocol forced or policy-selected, dtype, op,
element count (whole packs and ragged), channel count, and the buffer kind —
the registered symmetric buffer at a random offset (zero-copy), an unregistered
tensor (bounce), or an unregistered tensor under auto-registration — issued in
back-to-back batches of 4 calls with no host synchronisation in between.
Integer-valued inputs make every result exact; each rank regenerates every
rank's input and compares its own result bitwise with the oracle.  Rank 0
decides when the time budget (POLAR_STRESS_S) is spent.  Rank 0 writes JSON.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import allreduce as orc  # noqa: E402
from paper_2603_11438_b200 import polar as L  # noqa: E402
from tests.gpu_common import to_device, to_host  # noqa: E402

ES = {"i32": 4, "i64": 8, "f32": 4, "bf16": 2}
SYM_BYTES = 8 << 20


def main():
    out_path = sys.argv[1]
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")

    def allgather_obj(b):
        o = [None] * ws
        dist.all_gather_object(o, b)
        return o

    comm = L.Comm.init(ws, rank, dev, L.torch_allgather(dist, ws))
    if os.environ.get("POLAR_STRESS_POLICY"):
        # ranks sharing one GPU under MPS: a table that caps the channels so every
        # rank's CTAs stay co-resident (policies/mps_cap16.json)
        with open(os.environ["POLAR_STRESS_POLICY"]) as f:
            L.set_policy([tuple(r) for r in json.load(f)["rows"]])
    torn, reads = comm.probe_ll128(iters=500)      # real comms accept LL128 once probed
    (sym,) = comm.mem_alloc_tensors(SYM_BYTES // 4, torch.float32)
    rng = np.random.default_rng(int(os.environ.get("POLAR_STRESS_SEED", "2603")))
    budget = float(os.environ.get("POLAR_STRESS_S", "60"))
    t_end = time.monotonic() + budget
    calls, bad, kinds = 0, [], {}
    autoreg = False
    while True:
        go = allgather_obj(time.monotonic() < t_end if rank == 0 else None)[0]
        if not go:
            break
        want_ar = bool(rng.integers(2))
        if want_ar != autoreg:
            comm.autoreg(want_ar, 1 << 20)
            autoreg = want_ar
        pending = []
        for _ in range(4):
            dtype = synth.DTYPES[int(rng.integers(len(synth.DTYPES)))]
            op = ("sum", "max", "min")[int(rng.integers(3))]
            per = 16 // ES[dtype]
            count = int(rng.integers(1, 400_000 if rng.integers(3) else 4000))
            if rng.integers(2):
                count = max(per, count // per * per)
            kind = ("sym", "plain", "plain")[int(rng.integers(3))]
            mode = int(rng.integers(3))          # 0 policy-selected, else forced
            algo = ("oneshot", "twoshot", "ring", "tree")[int(rng.integers(4))]
            proto = ("ll", "ll128", "simple")[int(rng.integers(3))]
            nch = int(rng.integers(1, 5))
            cfg = int(rng.integers(1 << 30))
            xs = synth.gen_ranks(dtype, count, ws, cfg=cfg, dist="ints")
            if kind == "sym":
                span = SYM_BYTES // ES[dtype]
                off = int(rng.integers(0, max(1, span - count)))
                off = min(off, span - count) if count <= span else 0
                if count > span:
                    kind = "plain"
            if kind == "sym":
                t = sym.view(torch.uint8).view({"i32": torch.int32, "i64": torch.int64, "f32": torch.float32,
                                                "bf16": torch.bfloat16}[dtype])[off:off + count]
                t.copy_(to_device(xs[rank], dtype))
            else:
                t = to_device(xs[rank], dtype)
            if mode == 0:
                comm.allreduce(t, op=op)
                key = ("policy", kind, autoreg)
            else:
                comm.allreduce_forced(t, algo, proto, nch, op=op)
                key = (algo, proto, kind, autoreg)
            kinds[str(key)] = kinds.get(str(key), 0) + 1
            # the registered buffer is re-filled by the next call that uses it: a
            # copy of the result is taken in stream order, still without a host sync
            pending.append((t.clone() if kind == "sym" else t, xs, dtype, op, key, count, kind))
        torch.cuda.synchronize()
        comm.check()
        for t, xs, dtype, op, key, count, kind in pending:
            got = to_host(t, dtype)
            exp = orc.allreduce(xs, dtype, op)
            ok = np.array_equal(got, exp) if (dtype == "f32" and op != "sum") else \
                np.array_equal(got.view(np.uint8), exp.view(np.uint8))
            if not ok:
                bad.append([str(key), dtype, op, count])
            calls += 1
    comm.destroy()
    rep = {"rank": rank, "calls": calls, "bad": bad, "kinds": kinds, "ll128_probe": [torn, reads]}
    allrep = allgather_obj(rep)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allrep, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
