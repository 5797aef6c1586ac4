"""NCCL (the timed baseline) through ctypes on libnccl.so.2.

The paper's "default" is NCCL's own selection (R13); bench.py times
it on the SAME device buffers and streams as polar, with no NCCL_* overrides
(the NCCL_ALGO x NCCL_PROTO variants are separate processes:
scripts/nccl_variants.py).  NCCL's choice per call is read back from its
TUNING log (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=TUNING) written to a per-rank
file, which `enable_tuning_log` must set up before the first NCCL call of the
process.  Nothing here is on polar's path; it is measurement tooling.
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import re

NCCL_FLOAT32, NCCL_BFLOAT16, NCCL_INT32 = 7, 9, 2
NCCL_SUM = 0
ALGO_NAMES = {0: "tree", 1: "ring", 2: "collnet_direct", 3: "collnet_chain", 4: "nvls", 5: "nvls_tree", 6: "pat"}
PROTO_NAMES = {0: "ll", 1: "ll128", 2: "simple"}


class UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


def lib_path() -> str:
    """The torch-bundled NCCL (2.28.9 in this image), else the system one."""
    import torch
    here = os.path.dirname(torch.__file__)
    cands = glob.glob(os.path.join(os.path.dirname(here), "nvidia", "nccl", "lib", "libnccl.so.2"))
    return cands[0] if cands else "libnccl.so.2"


def enable_tuning_log(path_prefix: str):
    """Ask NCCL to log its per-collective decisions (TUNING) into path_prefix.<pid>."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,TUNING")
    os.environ["NCCL_DEBUG_FILE"] = path_prefix + ".%p"
    return path_prefix + f".{os.getpid()}"


_TUNE = re.compile(r"(\d+) Bytes -> Algo (\d+) proto (\d+)")


def parse_tuning(path: str):
    """{bytes: (algo, proto)} from NCCL's TUNING log lines (last one per size)."""
    out = {}
    try:
        with open(path, errors="replace") as f:
            for line in f:
                m = _TUNE.search(line)
                if m:
                    out[int(m.group(1))] = (ALGO_NAMES.get(int(m.group(2)), m.group(2)),
                                            PROTO_NAMES.get(int(m.group(3)), m.group(3)))
    except OSError:
        pass
    return out


class Nccl:
    def __init__(self):
        self.lib = C.CDLL(lib_path())
        L = self.lib
        L.ncclGetErrorString.restype = C.c_char_p
        L.ncclGetUniqueId.argtypes = [C.POINTER(UniqueId)]
        L.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
        L.ncclAllReduce.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ncclCommDestroy.argtypes = [C.c_void_p]
        L.ncclGetVersion.argtypes = [C.POINTER(C.c_int)]

    def _ck(self, r, what):
        if r != 0:
            raise RuntimeError(f"{what}: {self.lib.ncclGetErrorString(r).decode()} ({r})")

    def version(self) -> str:
        v = C.c_int(0)
        self._ck(self.lib.ncclGetVersion(C.byref(v)), "ncclGetVersion")
        x = v.value
        return f"{x // 10000}.{(x // 100) % 100}.{x % 100}"

    def unique_id(self) -> bytes:
        u = UniqueId()
        self._ck(self.lib.ncclGetUniqueId(C.byref(u)), "ncclGetUniqueId")
        return C.string_at(C.addressof(u), 128)   # (u.internal would stop at the first NUL)

    def init(self, nranks: int, uid: bytes, rank: int):
        u = UniqueId()
        C.memmove(C.addressof(u), uid, 128)
        comm = C.c_void_p()
        self._ck(self.lib.ncclCommInitRank(C.byref(comm), nranks, u, rank), "ncclCommInitRank")
        return comm

    def allreduce(self, comm, ptr: int, count: int, dtype: int, stream_ptr: int, op: int = NCCL_SUM):
        self._ck(self.lib.ncclAllReduce(C.c_void_p(ptr), C.c_void_p(ptr), count, dtype, op, comm,
                                        C.c_void_p(stream_ptr)), "ncclAllReduce")

    def destroy(self, comm):
        self._ck(self.lib.ncclCommDestroy(comm), "ncclCommDestroy")
