"""Oracle: the adaptive-channels controller (profiler -> tuner closed loop) —
TEST INFRASTRUCTURE ONLY.

PAPER.md §5.3 L597-611 describes the behaviour of the paper's
``adaptive_channels`` policy fed by a profiler program through a shared map:
"starts with a conservative channel count (nChannels = 2) ... Without the
profiler, the tuner receives no samples and remains at 2 channels ... ramps from
2 to 12 channels over 100,000 calls.  Under injected contention (10x latency
spike), the policy reduces channels from 12 to 2; upon recovery, it ramps back
to 12 within 100,000 calls."  The logic itself is not shown; R15 fixes
it, and this file transcribes R15 step by step:

    per closed window with mean latency m (no samples: nothing changes)
        ref = ref[c] if known else ref[c-1]
        if ref known and m > factor * ref:  c = c_min                 (back off)
        else:                               ref[c] = m; c = min(c+1, cap)

Parity: pinned by tests/test_adaptive.py against the paper's three-phase
behaviour (ramp 2 -> 12 within 100,000 calls, <= 3 channels under a 10x
contention window, back to 12 within 100,000 calls; no profiler -> stays at 2).
"""
from __future__ import annotations

import math

MAXCH = 32


def simulate(cap, lat_table, c_min=2, factor=4.0, scale=1.0):
    """Channel count after each window; window w is observed at the current c and
    its mean latency is lat_table[w][c] (NaN / <= 0: the window had no samples)."""
    cap = max(1, min(MAXCH, cap))
    c = min(c_min, cap)
    ref = [0.0] * (MAXCH + 1)
    trace = []
    for row in lat_table:
        m = row[c]
        m = 0.0 if (m is None or math.isnan(m)) else m * scale
        if m > 0.0:
            r = ref[c] if ref[c] > 0.0 else (ref[c - 1] if c > 1 else 0.0)
            if r > 0.0 and m > factor * r:
                c = min(c_min, cap)
            else:
                ref[c] = m
                if c < cap:
                    c += 1
        trace.append(c)
    return trace
