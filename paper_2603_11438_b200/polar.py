"""Thin ctypes binding of libpolar (include/polar.h) — argument marshalling only.

Every step of the hot path (decision, dispatch, the kernels) runs inside
libpolar.so; this module only converts Python/torch arguments to the C ABI.
If the library is missing it raises at import: there is no Python or CPU
fallback for any operation.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("POLAR_LIB", os.path.join(_HERE, "libpolar.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libpolar.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no fallback implementation)")
lib = C.CDLL(LIB_PATH)

# ----------------------------------------------------------------- enums
OK, EINVAL, ECUDA, EUNSUPPORTED, ETIMEOUT, EBUSY, ESTATE, ENOMEM = range(8)
STATUS_NAMES = {OK: "ok", EINVAL: "einval", ECUDA: "ecuda", EUNSUPPORTED: "eunsupported",
                ETIMEOUT: "etimeout", EBUSY: "ebusy", ESTATE: "estate", ENOMEM: "enomem"}
INT32, INT64, FLOAT32, BFLOAT16 = 2, 4, 7, 9
SUM, MAX, MIN = 0, 2, 3
COLL_ALLREDUCE, COLL_ALLGATHER, COLL_BROADCAST, COLL_REDUCESCATTER = 0, 1, 2, 3
TREE, RING, NVLS, ONESHOT, TWOSHOT = 0, 1, 2, 3, 4
LL, LL128, SIMPLE = 0, 1, 2
UNSET = 0xFFFFFFFF
MAXCH, MAXRANKS, MAXROWS = 32, 8, 64
ROW_ADAPTIVE_NCH = 0x1

DTYPE_CODES = {"i32": INT32, "i64": INT64, "f32": FLOAT32, "bf16": BFLOAT16}
OP_CODES = {"sum": SUM, "max": MAX, "min": MIN}
ALGO_CODES = {"tree": TREE, "ring": RING, "nvls": NVLS, "oneshot": ONESHOT, "twoshot": TWOSHOT}
PROTO_CODES = {"ll": LL, "ll128": LL128, "simple": SIMPLE}
ALGO_NAMES = {v: k for k, v in ALGO_CODES.items()}
PROTO_NAMES = {v: k for k, v in PROTO_CODES.items()}
TRANSPORT_NAMES = {0: "peer", 1: "cluster"}


class PolarError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))
        super().__init__(f"{what}: {lib.polar_status_string(status).decode()}")


# --------------------------------------------------------------- structs
class Ctx(C.Structure):
    _fields_ = [("coll", C.c_uint32), ("nranks", C.c_uint32), ("bytes", C.c_uint64)]


class Decision(C.Structure):
    _fields_ = [("algo", C.c_uint32), ("proto", C.c_uint32), ("nchannels", C.c_uint32),
                ("generation", C.c_uint32), ("flags", C.c_uint32), ("_pad", C.c_uint32)]

    def as_tuple(self):
        return (self.algo, self.proto, self.nchannels)

    def __repr__(self):
        return (f"Decision({ALGO_NAMES.get(self.algo, self.algo)}, {PROTO_NAMES.get(self.proto, self.proto)}, "
                f"nch={self.nchannels}, gen={self.generation})")


class PolicyRow(C.Structure):
    _fields_ = [("coll", C.c_uint32), ("nranks", C.c_uint32), ("max_bytes", C.c_uint64),
                ("algo", C.c_uint32), ("proto", C.c_uint32), ("nchannels", C.c_uint32), ("flags", C.c_uint32)]


class BenchStats(C.Structure):
    _fields_ = [("calls", C.c_uint64), ("p50_ns", C.c_double), ("p99_ns", C.c_double),
                ("mean_ns", C.c_double), ("min_ns", C.c_double), ("max_ns", C.c_double),
                ("timer_overhead_ns", C.c_double), ("batched_mean_ns", C.c_double)]


class SwapStats(C.Structure):
    _fields_ = [("calls", C.c_uint64), ("issued", C.c_uint64), ("invalid", C.c_uint64),
                ("nonmonotonic", C.c_uint64), ("swaps", C.c_uint64), ("rejected", C.c_uint64),
                ("rejected_changed", C.c_uint64), ("swap_p50_ns", C.c_double), ("swap_p99_ns", C.c_double),
                ("swap_max_ns", C.c_double), ("final_generation", C.c_uint32)]


class AdaptiveParams(C.Structure):
    _fields_ = [("enabled", C.c_uint32), ("period", C.c_uint32), ("c_min", C.c_uint32), ("_pad", C.c_uint32),
                ("contention_factor", C.c_double), ("latency_scale", C.c_double)]


class AdaptiveState(C.Structure):
    _fields_ = [("channels", C.c_uint32), ("contended", C.c_uint32), ("windows", C.c_uint64),
                ("samples", C.c_uint64), ("last_mean_ns", C.c_double)]


class AutoregStats(C.Structure):
    _fields_ = [("exchanges", C.c_uint64), ("zero_copy", C.c_uint64), ("bounced", C.c_uint64),
                ("opens", C.c_uint64), ("evictions", C.c_uint64), ("mismatches", C.c_uint64)]


AG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

_P = C.c_void_p
_sigs = {
    "polar_set_policy": (C.c_int, [C.POINTER(PolicyRow), C.c_uint32, C.POINTER(C.c_uint32)]),
    "polar_decide": (C.c_int, [C.POINTER(Ctx), C.POINTER(Decision)]),
    "polar_decide_batch": (C.c_int, [C.POINTER(Ctx), C.POINTER(Decision), C.c_size_t]),
    "polar_policy_generation": (C.c_uint32, []),
    "polar_get_policy": (C.c_int, [C.POINTER(PolicyRow), C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "polar_bench_decide": (C.c_int, [C.POINTER(Ctx), C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.POINTER(BenchStats)]),
    "polar_bench_swap": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint32, C.POINTER(PolicyRow), C.c_uint32,
                                   C.POINTER(PolicyRow), C.c_uint32, C.POINTER(SwapStats)]),
    "polar_comm_init": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int, C.c_int, AG_FN, _P]),
    "polar_comm_init_virtual": (C.c_int, [C.POINTER(_P), C.c_int, C.c_int]),
    "polar_bootstrap_check": (C.c_int, [C.c_int, C.c_int, AG_FN, _P]),
    "polar_comm_destroy": (C.c_int, [_P]),
    "polar_comm_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "polar_mem_alloc": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "polar_mem_free": (C.c_int, [_P, _P]),
    "polar_register": (C.c_int, [_P, _P, C.c_size_t]),
    "polar_deregister": (C.c_int, [_P, _P]),
    "polar_comm_autoreg": (C.c_int, [_P, C.c_int, C.c_size_t]),
    "polar_comm_autoreg_stats": (C.c_int, [_P, C.POINTER(AutoregStats)]),
    "polar_allreduce": (C.c_int, [_P, _P, C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_allreduce_v": (C.c_int, [_P, C.POINTER(_P), C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_allreduce_forced": (C.c_int, [_P, C.POINTER(_P), C.c_size_t, C.c_int, C.c_int, C.POINTER(Decision), _P]),
    "polar_allreduce_host": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_reduce_scatter": (C.c_int, [_P, _P, _P, C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_reduce_scatter_v": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_all_gather": (C.c_int, [_P, _P, _P, C.c_size_t, C.c_int, _P]),
    "polar_all_gather_v": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.c_size_t, C.c_int, _P]),
    "polar_broadcast": (C.c_int, [_P, _P, C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_broadcast_v": (C.c_int, [_P, C.POINTER(_P), C.c_size_t, C.c_int, C.c_int, _P]),
    "polar_comm_last_decision": (C.c_int, [_P, C.POINTER(Decision)]),
    "polar_comm_launches": (C.c_uint64, [_P]),
    "polar_comm_launch_info": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "polar_comm_transport": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "polar_comm_check": (C.c_int, [_P]),
    "polar_comm_set_trace": (C.c_int, [_P, _P, C.c_size_t]),
    "polar_p2p_probe": (C.c_int, [_P, C.POINTER(_P), C.c_size_t, C.c_int, _P]),
    "polar_bench_enqueue": (C.c_int, [_P, C.POINTER(_P), C.c_size_t, C.c_int, C.c_int, _P, C.c_uint64,
                                      C.POINTER(C.c_double)]),
    "polar_adaptive_config": (C.c_int, [_P, C.POINTER(AdaptiveParams)]),
    "polar_adaptive_get_state": (C.c_int, [_P, C.POINTER(AdaptiveState)]),
    "polar_adaptive_inject": (C.c_int, [_P, C.c_double]),
    "polar_adaptive_simulate": (C.c_int, [C.POINTER(AdaptiveParams), C.c_uint32, C.POINTER(C.c_double), C.c_uint32,
                                          C.POINTER(C.c_uint32)]),
    "polar_nvls_available": (C.c_int, []),
    "polar_comm_probe_ll128": (C.c_int, [_P, C.c_ulonglong, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "polar_comm_nvls_info": (C.c_int, [_P, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
    "polar_status_string": (C.c_char_p, [C.c_int]),
    "polar_version": (C.c_char_p, []),

}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs) + ("polar_probe_ll128",)   # + diagnostics bound on first use


def _check(st, what):
    if st != OK:
        raise PolarError(st, what)


# ---------------------------------------------------------------- policy
def rows_array(rows):
    arr = (PolicyRow * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i] = PolicyRow(*[int(x) for x in r[:6]], int(r[6]) if len(r) > 6 else 0)
    return arr


def set_policy_status(rows):
    """Raw status of polar_set_policy (no raise) and the generation."""
    arr = rows_array(rows)
    gen = C.c_uint32(0)
    st = lib.polar_set_policy(arr, len(rows), C.byref(gen))
    return st, gen.value


def set_policy(rows) -> int:
    st, gen = set_policy_status(rows)
    _check(st, "polar_set_policy")
    return gen


def decide(nranks: int, nbytes: int, coll: int = COLL_ALLREDUCE) -> Decision:
    d = Decision()
    _check(lib.polar_decide(C.byref(Ctx(coll, nranks, nbytes)), C.byref(d)), "polar_decide")
    return d


def decide_batch(ctxs, coll: int = COLL_ALLREDUCE):
    """ctxs: list of (nranks, nbytes) -> list of (algo, proto, nch, generation, flags)."""
    n = len(ctxs)
    a = (Ctx * max(1, n))()
    for i, (nr, b) in enumerate(ctxs):
        a[i] = Ctx(coll, nr, b)
    out = (Decision * max(1, n))()
    _check(lib.polar_decide_batch(a, out, n), "polar_decide_batch")
    return [(d.algo, d.proto, d.nchannels, d.generation, d.flags) for d in out[:n]]


def generation() -> int:
    return lib.polar_policy_generation()


def get_policy():
    arr = (PolicyRow * MAXROWS)()
    n, g = C.c_uint32(0), C.c_uint32(0)
    _check(lib.polar_get_policy(arr, MAXROWS, C.byref(n), C.byref(g)), "polar_get_policy")
    return [(r.coll, r.nranks, r.max_bytes, r.algo, r.proto, r.nchannels) + ((r.flags,) if r.flags else ())
            for r in arr[:n.value]], g.value


def bench_decide(ctxs, nwarm=10_000, ncalls=400_000):
    a = (Ctx * len(ctxs))()
    for i, (nr, b) in enumerate(ctxs):
        a[i] = Ctx(COLL_ALLREDUCE, nr, b)
    s = BenchStats()
    _check(lib.polar_bench_decide(a, len(ctxs), nwarm, ncalls, None, C.byref(s)), "polar_bench_decide")
    return {k: getattr(s, k) for k, _ in BenchStats._fields_}


def bench_swap(rows_a, rows_b, nthreads=4, calls_per_thread=100_000, nswaps=1000):
    s = SwapStats()
    _check(lib.polar_bench_swap(nthreads, calls_per_thread, nswaps, rows_array(rows_a), len(rows_a),
                                rows_array(rows_b), len(rows_b), C.byref(s)), "polar_bench_swap")
    return {k: getattr(s, k) for k, _ in SwapStats._fields_}


def adaptive_params(enabled=True, period=1000, c_min=2, contention_factor=4.0, latency_scale=1.0):
    return AdaptiveParams(int(enabled), int(period), int(c_min), 0, float(contention_factor), float(latency_scale))


def adaptive_simulate(params: AdaptiveParams, cap: int, lat_table):
    """lat_table: list of windows, each a list of 33 latencies (index = channel count)."""
    nw = len(lat_table)
    flat = (C.c_double * max(1, nw * (MAXCH + 1)))()
    for w, row in enumerate(lat_table):
        for c in range(MAXCH + 1):
            flat[w * (MAXCH + 1) + c] = float(row[c])
    out = (C.c_uint32 * max(1, nw))()
    _check(lib.polar_adaptive_simulate(C.byref(params), cap, flat, nw, out), "polar_adaptive_simulate")
    return list(out[:nw])


# ---------------------------------------------------------------- comms
def _torch_dtype_code(t):
    import torch
    m = {torch.int32: INT32, torch.int64: INT64, torch.float32: FLOAT32, torch.bfloat16: BFLOAT16}
    if t.dtype not in m:
        raise PolarError(EINVAL, f"dtype {t.dtype} not supported")
    return m[t.dtype]


def _check_tensor(t, what, cuda=True):
    if not hasattr(t, "data_ptr") or not hasattr(t, "is_contiguous"):
        raise PolarError(EINVAL, f"{what}: expected a torch tensor, got {type(t).__name__}")
    if t.is_cuda != cuda:
        raise PolarError(EINVAL, f"{what}: expected a {'CUDA' if cuda else 'host'} tensor")
    if not t.is_contiguous():
        raise PolarError(EINVAL, f"{what}: tensor must be contiguous (a strided view would be read past its end)")


def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper so torch can view library memory."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def torch_allgather(dist, world_size: int, group=None):
    """allgather(bytes) -> list[bytes] over a torch.distributed (CPU / gloo)
    group, for Comm.init: every payload of one call has the same size (the C
    ABI's fixed-size records), so it moves as one uint8 tensor per rank without
    pickling (all_gather_object costs ~10x more per call — it matters for
    polar_comm_autoreg, which all-gathers once per call)."""
    import torch

    def ag(b: bytes):
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(world_size)]
        dist.all_gather(out, t, group=group)
        return [o.numpy().tobytes() for o in out]

    return ag


def _make_ag(allgather):
    """Wrap allgather(bytes) -> list[bytes] as the C callback polar_allgather_fn."""

    def _cb(send, recv, nbytes, _user):
        try:
            allb = allgather(C.string_at(send, nbytes))
            C.memmove(recv, b"".join(allb), nbytes * len(allb))
            return 0
        except Exception:  # noqa: BLE001 - must not unwind through C
            return 1

    return AG_FN(_cb)


def bootstrap_check(nranks: int, rank: int, allgather) -> int:
    """Raw status of polar_bootstrap_check (collective, host only)."""
    cb = _make_ag(allgather)
    return lib.polar_bootstrap_check(nranks, rank, cb, None)


class _P2PResult(C.Structure):
    _fields_ = [("load_gbs", C.c_double), ("store_gbs", C.c_double), ("pingpong_us", C.c_double),
                ("load_xor", C.c_ulonglong)]


class Comm:
    """A communicator: ``Comm.virtual(n)`` (n ranks on one GPU) or
    ``Comm.init(n, rank, device, allgather)`` (one rank per process)."""

    def __init__(self, handle, keep=None):
        self.h = C.c_void_p(handle)
        self._keep = keep
        nr, rk, nl = C.c_int(), C.c_int(), C.c_int()
        _check(lib.polar_comm_info(self.h, C.byref(nr), C.byref(rk), C.byref(nl)), "polar_comm_info")
        self.nranks, self.rank, self.nlocal = nr.value, rk.value, nl.value

    @classmethod
    def virtual(cls, nranks: int, device: int = 0):
        h = C.c_void_p()
        _check(lib.polar_comm_init_virtual(C.byref(h), nranks, device), "polar_comm_init_virtual")
        return cls(h.value)

    @classmethod
    def init(cls, nranks: int, rank: int, device: int, allgather):
        """allgather(bytes) -> list[bytes] of every rank's payload (rank order)."""

        cb = _make_ag(allgather)
        h = C.c_void_p()
        _check(lib.polar_comm_init(C.byref(h), nranks, rank, device, cb, None), "polar_comm_init")
        return cls(h.value, keep=cb)

    def destroy(self):
        if self.h:
            _check(lib.polar_comm_destroy(self.h), "polar_comm_destroy")
            self.h = C.c_void_p()

    def mem_alloc(self, nbytes: int):
        """Symmetric device memory: list of nlocal raw pointers."""
        ptrs = (C.c_void_p * self.nlocal)()
        _check(lib.polar_mem_alloc(self.h, nbytes, ptrs), "polar_mem_alloc")
        return [int(p) for p in ptrs]

    def mem_alloc_tensors(self, numel: int, dtype):
        """Symmetric allocation viewed as torch tensors (one per local rank)."""
        import torch
        es = torch.empty(0, dtype=dtype).element_size()
        out = []
        for p in self.mem_alloc(numel * es):
            t = torch.as_tensor(_CudaArray(p, numel * es), device="cuda").view(dtype)
            out.append(t)
        return out

    def mem_free(self, ptr: int):
        _check(lib.polar_mem_free(self.h, C.c_void_p(ptr)), "polar_mem_free")

    def register(self, tensor):
        _check_tensor(tensor, "polar_register")
        _check(lib.polar_register(self.h, C.c_void_p(tensor.data_ptr()), tensor.numel() * tensor.element_size()),
               "polar_register")

    def deregister(self, tensor_or_ptr):
        """Collective: drop the registration starting at this tensor's (or raw pointer's) address."""
        ptr = tensor_or_ptr if isinstance(tensor_or_ptr, int) else tensor_or_ptr.data_ptr()
        _check(lib.polar_deregister(self.h, C.c_void_p(ptr)), "polar_deregister")

    def autoreg(self, enable: bool = True, min_bytes: int = 0):
        """Collective: unregistered two-shot calls of >= min_bytes exchange IPC
        handles and run zero-copy (polar_comm_autoreg)."""
        _check(lib.polar_comm_autoreg(self.h, 1 if enable else 0, int(min_bytes)), "polar_comm_autoreg")

    def autoreg_stats(self) -> dict:
        s = AutoregStats()
        _check(lib.polar_comm_autoreg_stats(self.h, C.byref(s)), "polar_comm_autoreg_stats")
        return {k: int(getattr(s, k)) for k, _ in AutoregStats._fields_}

    def _list(self, tensors, what, cuda=True):
        """nlocal tensors, each a contiguous CUDA tensor, all of one dtype and numel:
        the C ABI sees only a pointer and one count, so a strided view or a
        shorter tensor would make a kernel read or write past its end."""
        if not isinstance(tensors, (list, tuple)):
            tensors = [tensors]
        if len(tensors) != self.nlocal:
            raise PolarError(EINVAL, f"{what}: need {self.nlocal} buffers, got {len(tensors)}")
        t0 = tensors[0]
        for t in tensors:
            _check_tensor(t, what, cuda)
            if t.dtype != t0.dtype or t.numel() != t0.numel():
                raise PolarError(EINVAL, f"{what}: every buffer must have the dtype and numel of the first "
                                         f"({t0.dtype}, {t0.numel()}), got ({t.dtype}, {t.numel()})")
        return list(tensors)

    def _bufs(self, tensors, what="allreduce", cuda=True):
        tensors = self._list(tensors, what, cuda)
        arr = (C.c_void_p * self.nlocal)(*[t.data_ptr() for t in tensors])
        t0 = tensors[0]
        return arr, t0.numel(), _torch_dtype_code(t0)

    def allreduce(self, tensors, op="sum", stream=None):
        """In-place policy-selected AllReduce (one kernel launch)."""
        arr, n, dt = self._bufs(tensors)
        _check(lib.polar_allreduce_v(self.h, arr, n, dt, OP_CODES[op], _stream_ptr(stream)), "polar_allreduce_v")

    def allreduce_raw(self, ptrs, count, dtype_code, op_code, stream_ptr):
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        return lib.polar_allreduce_v(self.h, arr, count, dtype_code, op_code, C.c_void_p(stream_ptr))

    def allreduce_forced(self, tensors, algo, proto, nch, op="sum", stream=None):
        arr, n, dt = self._bufs(tensors)
        d = Decision(ALGO_CODES[algo] if isinstance(algo, str) else algo,
                     PROTO_CODES[proto] if isinstance(proto, str) else proto, nch, 0)
        _check(lib.polar_allreduce_forced(self.h, arr, n, dt, OP_CODES[op], C.byref(d), _stream_ptr(stream)),
               "polar_allreduce_forced")

    def allreduce_forced_raw(self, ptrs, count, dtype_code, op_code, decision, stream_ptr):
        """polar_allreduce_forced on raw device pointers (bench loops); returns the status."""
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        return lib.polar_allreduce_forced(self.h, arr, count, dtype_code, op_code, C.byref(decision),
                                          C.c_void_p(stream_ptr))

    def _ptrs(self, tensors, what):
        tensors = self._list(tensors, what)
        return (C.c_void_p * self.nlocal)(*[t.data_ptr() for t in tensors]), tensors[0]

    def _ratio(self, big, small, what):
        if big.dtype != small.dtype or big.numel() != self.nranks * small.numel():
            raise PolarError(EINVAL, f"{what}: need numel {self.nranks} x {small.numel()} = "
                                     f"{self.nranks * small.numel()} of {small.dtype}, got {big.numel()} of {big.dtype}")

    def reduce_scatter(self, sends, recvs, op="sum", stream=None):
        """recv_r = block r of the rank-ordered reduction of the sends (numel(send) = n * numel(recv))."""
        s, s0 = self._ptrs(sends, "reduce_scatter send")
        r, r0 = self._ptrs(recvs, "reduce_scatter recv")
        self._ratio(s0, r0, "reduce_scatter")
        _check(lib.polar_reduce_scatter_v(self.h, s, r, r0.numel(), _torch_dtype_code(r0), OP_CODES[op],
                                          _stream_ptr(stream)), "polar_reduce_scatter_v")

    def all_gather(self, sends, recvs, stream=None):
        """recv = concatenation of every rank's send (numel(recv) = n * numel(send))."""
        s, s0 = self._ptrs(sends, "all_gather send")
        r, r0 = self._ptrs(recvs, "all_gather recv")
        self._ratio(r0, s0, "all_gather")
        _check(lib.polar_all_gather_v(self.h, s, r, s0.numel(), _torch_dtype_code(s0), _stream_ptr(stream)),
               "polar_all_gather_v")

    def broadcast(self, bufs, root=0, stream=None):
        b, b0 = self._ptrs(bufs, "broadcast")
        _check(lib.polar_broadcast_v(self.h, b, b0.numel(), _torch_dtype_code(b0), int(root), _stream_ptr(stream)),
               "polar_broadcast_v")

    def allreduce_host(self, host_tensors, dev_tensors, op="sum", stream=None):
        harr, n, dt = self._bufs(host_tensors, "allreduce_host host", cuda=False)
        darr, n2, dt2 = self._bufs(dev_tensors, "allreduce_host device")
        if (n2, dt2) != (n, dt):
            raise PolarError(EINVAL, "allreduce_host: host and device buffers differ in numel or dtype")
        _check(lib.polar_allreduce_host(self.h, harr, darr, n, dt, OP_CODES[op], _stream_ptr(stream)),
               "polar_allreduce_host")

    def p2p_probe(self, tensors, iters=5):
        """Collective peer-path probe (polar.h polar_p2p_probe): per local rank a dict
        {load_gbs, store_gbs, pingpong_us, load_xor}; tensors are the symmetric
        buffers (whole tensors, 16-B multiple)."""
        arr, _, _ = self._bufs(tensors)
        nbytes = tensors[0].numel() * tensors[0].element_size() if isinstance(tensors, (list, tuple)) else \
            tensors.numel() * tensors.element_size()
        res = (_P2PResult * self.nlocal)()
        _check(lib.polar_p2p_probe(self.h, arr, nbytes, int(iters), C.cast(res, C.c_void_p)), "polar_p2p_probe")
        return [{"load_gbs": r.load_gbs, "store_gbs": r.store_gbs, "pingpong_us": r.pingpong_us,
                 "load_xor": r.load_xor} for r in res]

    def bench_enqueue(self, tensors, ncalls=2000, op="sum", stream=None) -> float:
        """Host ns per polar_allreduce_v call (decide + dispatch + launch), native loop."""
        arr, n, dt = self._bufs(tensors)
        ns = C.c_double(0)
        _check(lib.polar_bench_enqueue(self.h, arr, n, dt, OP_CODES[op], _stream_ptr(stream), ncalls, C.byref(ns)),
               "polar_bench_enqueue")
        return ns.value

    def last_decision(self) -> Decision:
        d = Decision()
        _check(lib.polar_comm_last_decision(self.h, C.byref(d)), "polar_comm_last_decision")
        return d

    def adaptive_config(self, **kw):
        p = adaptive_params(**kw)
        _check(lib.polar_adaptive_config(self.h, C.byref(p)), "polar_adaptive_config")

    def adaptive_inject(self, latency_scale: float):
        _check(lib.polar_adaptive_inject(self.h, float(latency_scale)), "polar_adaptive_inject")

    def adaptive_state(self):
        s = AdaptiveState()
        _check(lib.polar_adaptive_get_state(self.h, C.byref(s)), "polar_adaptive_get_state")
        return {k: getattr(s, k) for k, _ in AdaptiveState._fields_}

    def launched_channels(self) -> int:
        nch = C.c_uint32(0)
        _check(lib.polar_comm_launch_info(self.h, C.byref(nch), None), "polar_comm_launch_info")
        return nch.value

    def transport(self) -> str:
        """Transport of the most recent AllReduce: "peer" or "cluster" (polar.h)."""
        t = C.c_int(0)
        _check(lib.polar_comm_transport(self.h, C.byref(t)), "polar_comm_transport")
        return TRANSPORT_NAMES[t.value]

    def launches(self) -> int:
        return lib.polar_comm_launches(self.h)

    def set_trace(self, tensor=None):
        """Diagnostics: per-CTA %globaltimer stamps into a uint64/int64 device tensor (None = off)."""
        if tensor is None:
            _check(lib.polar_comm_set_trace(self.h, None, 0), "polar_comm_set_trace")
        else:
            _check(lib.polar_comm_set_trace(self.h, C.c_void_p(tensor.data_ptr()),
                                            tensor.numel() * tensor.element_size()), "polar_comm_set_trace")

    def check(self):
        _check(lib.polar_comm_check(self.h), "polar_comm_check")

    def probe_ll128(self, iters=2000):
        """Collective LL128 premise probe over this comm's transport: (torn, reads)
        summed over ranks; a real comm accepts LL128 only after 0 torn lanes."""
        torn, reads = C.c_ulonglong(0), C.c_ulonglong(0)
        _check(lib.polar_comm_probe_ll128(self.h, int(iters), C.byref(torn), C.byref(reads)),
               "polar_comm_probe_ll128")
        return torn.value, reads.value

    def nvls_info(self):
        """(available, why): does this comm hold a multicast object (NVLS), and
        the object's description or the driver call that refused it."""
        av = C.c_int(0)
        buf = C.create_string_buffer(256)
        _check(lib.polar_comm_nvls_info(self.h, C.byref(av), buf, 256), "polar_comm_nvls_info")
        return bool(av.value), buf.value.decode()


def probe_ll128(device=0, pairs=64, iters=20000, jitter_ns=0, jitter_mode=0):
    """(torn lanes, lanes read) of the LL128 hardware probe (polar.h)."""
    fn = lib.polar_probe_ll128   # diagnostic: bound on first use
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_int, C.c_ulonglong, C.c_uint, C.c_int, C.POINTER(C.c_ulonglong),
                   C.POINTER(C.c_ulonglong)]
    torn, reads = C.c_ulonglong(0), C.c_ulonglong(0)
    _check(fn(int(device), int(pairs), int(iters), int(jitter_ns), int(jitter_mode),
                                 C.byref(torn), C.byref(reads)),
           "polar_probe_ll128")
    return torn.value, reads.value


def version() -> str:
    return lib.polar_version().decode()


def _load_env_policy():
    """POLAR_POLICY=path.json installs that policy table at import (SURVEY.md §5
    "Config / flags"); a rejected table raises (the library keeps noop)."""
    path = os.environ.get("POLAR_POLICY", "")
    if not path:
        return
    import json
    with open(path) as f:
        d = json.load(f)
    rows = d["rows"] if isinstance(d, dict) else d
    set_policy([tuple(int(x) for x in r) for r in rows])


_load_env_policy()
