"""NCCL's own algorithms on B200, the shape of the paper's Table 2 (PAPER.md
L538-564) and SURVEY.md §8(d)'s context variants: AllReduce busBW per size for
NCCL's default selection and for every NCCL_ALGO x NCCL_PROTO override, each a
separate torchrun job (NCCL reads the overrides at communicator creation).
ctypes libnccl.so.2 (scripts/nccl_ctypes.py), device time max over ranks, the
choice NCCL made per size read from its TUNING log.

    python scripts/nccl_variants.py --gpus 8 [--sizes 4096,...] > gpurun_out/nccl_variants.jsonl

Where NCCL cannot run (one GPU shared by every rank: NCCL refuses duplicate
GPUs) each variant prints {"variant": ..., "skipped": why} and the script
still exits 0.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SIZES = [(4 << 10) << k for k in range(19)]          # 4 KiB .. 1 GiB
VARIANTS = [("default", None, None)] + [(f"{a}/{p}", a, p) for a in ("Ring", "Tree", "NVLS")
                                         for p in ("LL", "LL128", "Simple")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(args):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, HERE)
    import nccl_ctypes as N
    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    log = N.enable_tuning_log(os.path.join(tempfile.gettempdir(), f"nccl_variants.r{rank}"))
    dev = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")

    def allgather(o):
        out = [None] * ws
        dist.all_gather_object(out, o)
        return out
    variant = os.environ.get("POLAR_NCCL_VARIANT", "default")
    uuids = allgather(str(torch.cuda.get_device_properties(dev).uuid))
    why = None
    if len(set(uuids)) < ws:
        why = "ranks share a GPU: NCCL refuses duplicate GPUs (run on a node with one GPU per rank)"
    nccl = comm = None
    if why is None:
        try:
            nccl = N.Nccl()
            uid = allgather(nccl.unique_id() if rank == 0 else None)[0]
            comm = nccl.init(ws, uid, rank)
        except Exception as e:  # noqa: BLE001
            why = f"NCCL init failed: {e}"
    whys = allgather(why)
    why = next((w for w in whys if w), None)
    if why:
        if rank == 0:
            print(json.dumps({"variant": variant, "n": ws, "skipped": why}), flush=True)
        dist.destroy_process_group()
        return
    sizes = [int(x) for x in args.sizes.split(",")] if args.sizes else SIZES
    buf = torch.empty(max(sizes) // 4, dtype=torch.float32, device="cuda").normal_()
    s = torch.cuda.current_stream()
    recs = []
    for sz in sizes:
        cnt = sz // 4

        def call():
            nccl.allreduce(comm, buf.data_ptr(), cnt, N.NCCL_FLOAT32, s.cuda_stream)

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        call()
        b.record(s)
        b.synchronize()
        t1 = max(allgather(a.elapsed_time(b) / 1e3))
        it = int(max(5, min(200, 2e-3 / max(t1, 1e-7))))
        dist.barrier()
        a.record(s)
        for _ in range(it):
            call()
        b.record(s)
        b.synchronize()
        t = max(allgather(a.elapsed_time(b) / 1e3 / it))
        recs.append({"variant": variant, "n": ws, "bytes": sz, "us": round(t * 1e6, 2),
                     "busbw_gbs": round(sz * 2 * (ws - 1) / ws / t / 1e9, 2)})
    torch.cuda.synchronize()
    choices = N.parse_tuning(log)
    if rank == 0:
        for r in recs:
            if r["bytes"] in choices:
                r["nccl_choice"] = list(choices[r["bytes"]])
            r["nccl_version"] = nccl.version()
            print(json.dumps(r), flush=True)
    nccl.destroy(comm)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--sizes", default="")
    ap.add_argument("--variants", default="", help="comma list of names (default: all)")
    ap.add_argument("--worker", action="store_true")
    args = ap.parse_args()
    if args.worker:
        return worker(args)
    want = set(args.variants.split(",")) if args.variants else None
    for name, algo, proto in VARIANTS:
        if want and name not in want:
            continue
        env = dict(os.environ, POLAR_NCCL_VARIANT=name)
        for k in ("NCCL_ALGO", "NCCL_PROTO"):
            env.pop(k, None)
        if algo:
            env["NCCL_ALGO"], env["NCCL_PROTO"] = algo, proto
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(HERE, "nccl_variants.py"),
               "--worker"] + (["--sizes", args.sizes] if args.sizes else [])
        r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=3600)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 and not lines:
            lines = [json.dumps({"variant": name, "n": args.gpus, "skipped": f"rc={r.returncode}: "
                                 + (r.stderr.strip().splitlines() or [""])[-1][-300:]})]
        for ln in lines:
            print(ln, flush=True)


if __name__ == "__main__":
    main()
