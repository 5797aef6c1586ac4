"""Oracle: the tuner policy's size -> decision mapping — TEST INFRASTRUCTURE ONLY.

Follows, step by step:

* PAPER.md L108-112 (§2 "NCCL and its plugin system"): per collective the
  tuner receives (collective type, message size, rank topology) and selects an
  algorithm, a protocol and a channel count.
* PAPER.md L304-309 (§3.3 "Policy programming model"): the policy reads the
  context and writes algorithm / protocol / channel-count outputs.
* SPEC.md L306 / L339 (host-sim ContextLayout, invoke_tuner): outputs start
  UNSET (algorithm/protocol 0xFFFFFFFF, channels 0); UNSET outputs defer to the
  host default; channels are clamped to [1, max_channels].
* PAPER.md L384-385 (§4 "NCCL integration challenges"): "our native baseline
  layer clamps the policy's request"; MAXCH = 32 (R8).
* PAPER.md L334 (Listing 1 ``msg_size <= 32*1024``): thresholds are inclusive
  upper bounds; the key is the total message bytes (R6).

A policy here is DATA: an ordered list of rows
``(coll, nranks, max_bytes, algo, proto, nchannels[, flags])``; the first row whose
``coll`` equals the context's, whose ``nranks`` is 0 (any) or equal, and whose
``max_bytes`` >= the message bytes, wins.

The built-in default table (what an empty policy, i.e. the paper's ``noop``,
defers to) is transcribed below from DESIGN.md "Default table" — written here
independently of the library's C++ copy; the decision parity tests compare the
two.

Parity: pinned by tests/test_oracle_policy.py against the paper's worked
examples (Listing 1, ``nvlink_ring_mid_v2``, ``bad_channels``) and SPEC.md's
invoke_tuner examples (tests/golden/*.txt).
"""
from __future__ import annotations

# SPEC.md L306 enum values (TREE=0, RING=1, NVLS=2; LL=0, LL128=1, SIMPLE=2) plus
# the two direct algorithms this build adds.
COLL_ALLREDUCE, COLL_ALLGATHER, COLL_BROADCAST, COLL_REDUCESCATTER = 0, 1, 2, 3
TREE, RING, NVLS, ONESHOT, TWOSHOT = 0, 1, 2, 3, 4
LL, LL128, SIMPLE = 0, 1, 2
UNSET = 0xFFFFFFFF
ROW_ADAPTIVE_NCH = 0x1   # row flag: channels from the closed loop, nchannels = cap (R15)
MAXCH = 32          # DESIGN.md R8
MAXROWS = 64        # DESIGN.md "Policy table" bound
MAXRANKS = 8
U64_MAX = 2**64 - 1

ALGO_NAMES = {TREE: "tree", RING: "ring", NVLS: "nvls", ONESHOT: "oneshot", TWOSHOT: "twoshot"}
PROTO_NAMES = {LL: "ll", LL128: "ll128", SIMPLE: "simple"}

KiB, MiB = 1024, 1024 * 1024

#: DESIGN.md "Default table" (the library's built-in defaults; what ``noop`` defers to).
DEFAULT_ROWS = [
    (COLL_ALLREDUCE, 0, 64 * KiB, ONESHOT, LL, 4),
    (COLL_ALLREDUCE, 0, 1 * MiB, ONESHOT, SIMPLE, 8),
    (COLL_ALLREDUCE, 0, U64_MAX, TWOSHOT, SIMPLE, 32),
    (COLL_ALLGATHER, 0, U64_MAX, ONESHOT, SIMPLE, 32),
    (COLL_BROADCAST, 0, U64_MAX, ONESHOT, SIMPLE, 32),
    (COLL_REDUCESCATTER, 0, U64_MAX, ONESHOT, SIMPLE, 32),
]


def _first_match(rows, coll: int, nranks: int, nbytes: int):
    for row in rows:
        r_coll, r_nranks, r_max = row[0], row[1], row[2]
        if r_coll == coll and (r_nranks == 0 or r_nranks == nranks) and nbytes <= r_max:
            return row
    return None


def decide_full(rows, coll: int, nranks: int, nbytes: int):
    """(algo, proto, nchannels, flags) for one call, or None if the collective has no default.

    Per-field deferral: a matching row's UNSET algo/proto or 0 channels take the
    default table's value for the same context; then channels are clamped to
    [1, MAXCH].  flags are the matching row's (0 if none matched).
    """
    d = _first_match(DEFAULT_ROWS, coll, nranks, nbytes)
    if d is None:
        return None
    m = _first_match(rows, coll, nranks, nbytes)
    algo, proto, nch, flags = d[3], d[4], d[5], 0
    if m is not None:
        if m[3] != UNSET:
            algo = m[3]
        if m[4] != UNSET:
            proto = m[4]
        if m[5] != 0:
            nch = m[5]
        flags = m[6] if len(m) > 6 else 0
    nch = min(max(nch, 1), MAXCH)
    return algo, proto, nch, flags


def decide(rows, coll: int, nranks: int, nbytes: int):
    """(algo, proto, nchannels) — decide_full without the flags."""
    r = decide_full(rows, coll, nranks, nbytes)
    return None if r is None else r[:3]


def validate(rows, nvls_available: bool = False) -> str:
    """Status name set_policy must return for ``rows``.

    "ok", or "einval" (malformed: too many rows, unknown enum, nranks > 8,
    rows of one (coll, nranks) group not strictly ascending in max_bytes), or
    "eunsupported" (well-formed but names a decision no kernel implements:
    NVLS without a multicast object — none can be created on the 1-GPU pool,
    DESIGN.md §1 f1 — or a ReduceScatter / AllGather / Broadcast row naming
    anything but ONESHOT / SIMPLE, the only kernel those collectives have,
    DESIGN.md §4).  LL128 is accepted: the protocol exists (
    PAPER.md L111, L569-571).
    """
    if len(rows) > MAXROWS:
        return "einval"
    unsupported = False
    last = {}
    for row in rows:
        coll, nranks, max_bytes, algo, proto, nch = row[:6]
        flags = row[6] if len(row) > 6 else 0
        if flags & ~ROW_ADAPTIVE_NCH:
            return "einval"
        if coll not in (COLL_ALLREDUCE, COLL_ALLGATHER, COLL_BROADCAST, COLL_REDUCESCATTER):
            return "einval"
        if nranks > MAXRANKS:
            return "einval"
        if algo not in (TREE, RING, NVLS, ONESHOT, TWOSHOT, UNSET):
            return "einval"
        if proto not in (LL, LL128, SIMPLE, UNSET):
            return "einval"
        if not (0 <= max_bytes <= U64_MAX) or not (0 <= nch < 2**32):
            return "einval"
        key = (coll, nranks)
        if key in last and max_bytes <= last[key]:
            return "einval"
        last[key] = max_bytes
        if algo == NVLS and (not nvls_available or coll != COLL_ALLREDUCE):
            unsupported = True
        if coll != COLL_ALLREDUCE and (algo not in (ONESHOT, UNSET) or proto not in (SIMPLE, UNSET)):
            unsupported = True
    return "eunsupported" if unsupported else "ok"
