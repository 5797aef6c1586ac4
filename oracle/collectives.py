"""Oracle: ReduceScatter, AllGather, Broadcast by their plain definitions —
TEST INFRASTRUCTURE ONLY.

SPEC.md L306 enumerates the collectives the tuner context carries (ALLREDUCE,
ALLGATHER, BROADCAST, REDUCESCATTER); PAPER.md L106-107 names AllReduce and
AllGather as NCCL primitives; SURVEY.md §8(f) f4 routes them through the same
decision hook.  Definitions (NCCL semantics; R16):

* ReduceScatter: rank r's input holds n blocks of `recvcount` elements; rank r
  receives block r of the rank-ordered reduction:
      recv_r[i] = op(... op(x_0[r*c + i], x_1[r*c + i]) ..., x_{n-1}[r*c + i])
  with the same per-dtype arithmetic as oracle.allreduce (wrap-around ints,
  RNE f32, bf16 accumulated in f32 and rounded once).
* AllGather: recv[r*c + i] = x_r[i] on every rank (rank-order concatenation).
* Broadcast: every rank ends with root's vector.

Parity: pinned by tests/test_oracle_collectives.py (pure-Python brute force on
tiny inputs, closed forms).
"""
from __future__ import annotations

import numpy as np

from oracle import allreduce as _ar


def reduce_scatter(xs, dtype: str, op: str):
    """List of n per-rank result blocks."""
    n = len(xs)
    total = len(xs[0])
    if total % n:
        raise ValueError("input length must be nranks * recvcount")
    c = total // n
    return [_ar.allreduce([x[r * c:(r + 1) * c] for x in xs], dtype, op) for r in range(n)]


def all_gather(xs):
    """The single vector every rank receives."""
    if any(len(x) != len(xs[0]) for x in xs):
        raise ValueError("ranks disagree on sendcount")
    return np.concatenate([np.asarray(x) for x in xs]) if xs else np.zeros(0)


def broadcast(xs, root: int):
    if not 0 <= root < len(xs):
        raise ValueError("bad root")
    return np.array(xs[root], copy=True)
