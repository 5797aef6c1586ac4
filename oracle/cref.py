"""ctypes wrapper of oracle/c/allreduce_ref.c — TEST INFRASTRUCTURE ONLY.

The plain threaded C oracle (SURVEY.md §8(d) "a plain threaded C++ variant (no
intrinsics) on all cores, cross-checked bit-exactly against numpy"): the CPU
baseline bench.py times beside the GPU.  Built by ``build()`` (gcc, no nvcc)
into oracle/c/liboracle_ref.so; the product path never loads it.
Pinned by tests/test_oracle_cref.py against oracle/allreduce.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "allreduce_ref.c")
LIB = os.path.join(HERE, "c", "liboracle_ref.so")
DT = {"i32": 2, "i64": 4, "f32": 7, "bf16": 9}
OPS = {"sum": 0, "max": 2, "min": 3}
STORAGE = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "bf16": np.uint16}


def build() -> str:
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-ffp-contract=off", "-fno-fast-math",
               "-Wall", SRC, "-o", LIB, "-lm"]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_allreduce.restype = C.c_int
        _lib.oracle_allreduce.argtypes = [C.POINTER(C.c_void_p), C.c_void_p, C.c_size_t, C.c_int, C.c_int,
                                          C.c_int, C.c_int]
    return _lib


def allreduce(xs, dtype: str, op: str, nthreads: int = 1) -> np.ndarray:
    """Rank-ordered AllReduce of ``xs`` (same storage dtypes as oracle/allreduce.py)."""
    lib = _load()
    st = STORAGE[dtype]
    arrs = [np.ascontiguousarray(x, dtype=st) for x in xs]
    count = len(arrs[0]) if arrs else 0
    y = np.empty(count, dtype=st)
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    rc = lib.oracle_allreduce(ptrs, y.ctypes.data, count, len(arrs), DT[dtype], OPS[op], int(nthreads))
    if rc != 0:
        raise ValueError("oracle_allreduce rejected its arguments")
    return y
