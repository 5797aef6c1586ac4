"""PCIe ceilings for the e2e leg: pinned H2D / D2H alone and concurrent, 1 GiB."""
import json
import torch

GB = 1 << 30
h = torch.empty(GB, dtype=torch.uint8).pin_memory()
h2 = torch.empty(GB, dtype=torch.uint8).pin_memory()
d = torch.empty(GB, dtype=torch.uint8, device="cuda")
d2 = torch.empty(GB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()


def h2d_chunks(nstreams):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    ch = GB // 64

    def f():
        for k in range(64):
            with torch.cuda.stream(ss[k % nstreams]):
                d[k * ch:(k + 1) * ch].copy_(h[k * ch:(k + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()
    return f


out = {"h2d_gbs": GB / t(lambda: d.copy_(h, non_blocking=True)) / 1e9,
       "d2h_gbs": GB / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9,
       "both_each_gbs": GB / t(both) / 1e9}
for ns in (1, 2, 4):
    out[f"h2d_16MiB_chunks_{ns}streams_gbs"] = GB / t(h2d_chunks(ns)) / 1e9
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
