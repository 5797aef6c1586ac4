"""Oracle: bandwidth arithmetic of the metric — TEST INFRASTRUCTURE ONLY.

SPEC.md L359 / L623 (GLOSSARY "Bus bandwidth"): for AllReduce,
busbytes = S * 2(n-1)/n, busBW = busbytes / t; algBW = S / t.
PAPER.md L447-449 (§5.1): "a 128 MiB 8-GPU AllReduce on NVLink (~394 us)" at
the 596.9 GB/s default bus bandwidth of Table 2 (L559) pins the convention
(tests/test_oracle_metrics.py).
"""
from __future__ import annotations


def busbytes_allreduce(nbytes: int, nranks: int) -> float:
    if nranks <= 1:
        return 0.0
    return nbytes * 2.0 * (nranks - 1) / nranks


def busbw_gbs(nbytes: int, nranks: int, seconds: float) -> float:
    """Bus bandwidth in GB/s (1e9 bytes/s)."""
    return busbytes_allreduce(nbytes, nranks) / seconds / 1e9


def algbw_gbs(nbytes: int, seconds: float) -> float:
    return nbytes / seconds / 1e9


def latency_from_busbw(nbytes: int, nranks: int, busbw_gbs_: float) -> float:
    """Seconds an AllReduce of ``nbytes`` takes at the given bus bandwidth."""
    return busbytes_allreduce(nbytes, nranks) / (busbw_gbs_ * 1e9)
