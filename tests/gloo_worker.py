"""One rank of the CPU-only multi-process test (gloo, world_size >= 2).

Host logic of the N>1 path that runs without a GPU:
  * polar_bootstrap_check through the ctypes all-gather callback (the exact
    callback polar_comm_init uses) — must pass when ranks agree, and fail on
    EVERY rank when one rank's scratch layout differs (POLAR_* env);
  * rank-consistent decisions: every rank decides the same (algo, proto, nch)
    for a sweep, with a policy installed collectively between calls
    (R12), generations advancing in lock-step.
Writes a JSON report (rank 0).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch.distributed as dist  # noqa: E402

from paper_2603_11438_b200 import polar as L  # noqa: E402


def main():
    out_path, mode = sys.argv[1], sys.argv[2]
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")

    def allgather(b):
        o = [None] * ws
        dist.all_gather_object(o, b)
        return o

    rep = {"rank": rank}
    if os.environ.get("POLAR_TEST_SKEW_RANK") == str(rank):
        os.environ["POLAR_OS_CHUNK"] = str(2 << 20)   # this rank's scratch layout differs
    rep["bootstrap"] = L.STATUS_NAMES[L.bootstrap_check(ws, rank, allgather)]
    if mode == "consistency":
        # the same check through the pickle-free byte all-gather (polar.torch_allgather)
        rep["bootstrap_tensor_ag"] = L.STATUS_NAMES[L.bootstrap_check(ws, rank, L.torch_allgather(dist, ws))]
        sizes = [1 << k for k in range(3, 31)] + [(1 << k) + 1 for k in range(3, 31)]
        tables = [[], [(0, 0, 32768, L.TREE, L.SIMPLE, 4), (0, 0, 2**64 - 1, L.RING, L.SIMPLE, 4)],
                  [(0, ws, 1 << 20, L.ONESHOT, L.LL, 2), (0, 0, 2**64 - 1, L.UNSET, L.UNSET, 64)]]
        decisions, gens = [], []
        for t in tables:
            dist.barrier()                 # collective swap between calls (R12)
            gens.append(L.set_policy(t))
            decisions.append(L.decide_batch([(ws, s) for s in sizes]))
        allrep = [None] * ws
        dist.all_gather_object(allrep, {"dec": decisions, "gens": gens})
        rep["decisions_identical"] = all(a["dec"] == allrep[0]["dec"] for a in allrep)
        rep["gens_identical"] = all(a["gens"] == allrep[0]["gens"] for a in allrep)
        rep["gens"] = gens
    allrep = [None] * ws
    dist.all_gather_object(allrep, rep)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allrep, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
