"""Run the LL128 hardware probe (polar_probe_ll128) at several jitter levels."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11438_b200 import polar as L  # noqa: E402

for mode in (0, 1, 2):
    for pairs in (8, 64):
        for jit in (0, 500, 2000, 20000):
            iters = 20000 if jit < 20000 else 2000
            torn, reads = L.probe_ll128(0, pairs, iters, jit, mode)
            print(json.dumps({"jitter_mode": mode, "pairs": pairs, "iters": iters, "jitter_ns": jit,
                              "torn_lanes": torn, "lane_reads": reads}), flush=True)
