"""Helpers for the -m gpu parity tests: upload seeded inputs, run through the
C-ABI, compare with the oracle element by element."""
import numpy as np

import synth
from oracle import allreduce as orc

TORCH_DTYPES = None


def torch_dtype(dtype):
    import torch
    return {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]


def to_device(x: np.ndarray, dtype: str, offset: int = 0):
    """Upload a numpy array (bf16 as uint16 bits); `offset` elements of padding
    in front make the tensor start unaligned."""
    import torch
    if dtype == "bf16":
        t = torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if offset:
        pad = torch.zeros(offset + t.numel(), dtype=t.dtype)
        pad[offset:] = t
        return pad.cuda()[offset:]
    return t.cuda()


def to_host(t, dtype: str) -> np.ndarray:
    import torch
    c = t.detach().cpu()
    if dtype == "bf16":
        return c.view(torch.int16).numpy().view(np.uint16).copy()
    return c.numpy().copy()


def default_dist(dtype):
    return {"i32": "full", "i64": "full", "f32": "unif", "bf16": "normal"}[dtype]


def check_result(got_per_rank, xs, dtype, op, algo, n):
    """Parity bar: ints bit-exact; f32 one-/two-shot bit-exact, ring/
    tree within 1e-6*n*sum|x| (R2); bf16 within 1e-2*|y*| (R3, expected exact);
    and every rank bitwise identical (R4)."""
    exp = orc.allreduce(xs, dtype, op)
    first = got_per_rank[0]
    for r, g in enumerate(got_per_rank):
        assert np.array_equal(g.view(np.uint8), first.view(np.uint8)), f"rank {r} differs from rank 0"
    exact = dtype in ("i32", "i64") or op != "sum" or algo in ("oneshot", "twoshot")
    if exact:
        if dtype == "f32" and op != "sum":
            ok = np.array_equal(first, exp)          # value compare: +0 == -0 for fmax/fmin
        else:
            ok = np.array_equal(first, exp)          # same storage dtype: bitwise for ints / bf16 bits
            if dtype == "f32":
                ok = np.array_equal(first.view(np.uint32), exp.view(np.uint32))
        if not ok:
            idx = np.flatnonzero(first != exp)[:10]
            raise AssertionError(f"mismatch at {idx.tolist()}: got {first[idx]} exp {exp[idx]}")
        return
    if dtype == "f32":
        abssum = np.sum(np.abs(np.stack(xs).astype(np.float64)), axis=0)
        err = np.abs(first.astype(np.float64) - exp.astype(np.float64))
        assert np.all(err <= 1e-6 * n * abssum), f"max err/bound {np.max(err / np.maximum(1e-300, 1e-6 * n * abssum))}"
        return
    # bf16 sum, ring / tree
    y = orc.bf16_bits_to_f32(first).astype(np.float64)
    ys = orc.bf16_bits_to_f32(exp).astype(np.float64)
    assert np.all(np.abs(y - ys) <= 1e-2 * np.abs(ys)), "bf16 outside 1e-2 relative"
