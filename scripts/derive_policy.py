"""Turn tune_policy.py measurements into one first-match policy table.

python scripts/derive_policy.py gpurun_out/tune_TAG.jsonl [--tol 0.03] > policies/b200_virtual.json
Per rank count: at each measured size take the fastest (algo, proto, nch); keep
the previous row's choice while it is within `tol` of the fastest (fewer rows,
no noise-driven flips); rows are inclusive upper bounds at the last measured
size of a run; the last row per rank count is open-ended.
"""
import argparse
import collections
import json
import sys

CODES_A = {"tree": 0, "ring": 1, "oneshot": 3, "twoshot": 4}
CODES_P = {"ll": 0, "ll128": 1, "simple": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--tol", type=float, default=0.03)
    a = ap.parse_args()
    meas = collections.defaultdict(dict)   # (n, bytes) -> {(algo, proto, nch): us}
    for line in open(a.path):
        if not line.startswith("{"):
            continue
        r = json.loads(line)
        if "us" in r:
            meas[(r["n"], r["bytes"])][(r["algo"], r["proto"], r["nch"])] = r["us"]
    rows, detail = [], {}
    for n in sorted({k[0] for k in meas}):
        sizes = sorted(b for (m, b) in meas if m == n)
        cur, group = None, []
        for size in sizes:
            m = meas[(n, size)]
            best = min(m, key=m.get)
            if cur is not None and cur in m and m[cur] <= (1 + a.tol) * m[best]:
                choice = cur
            else:
                choice = best
            if choice != cur:
                group.append([size, choice])
                cur = choice
            else:
                group[-1][0] = size
            detail[f"{n}:{size}"] = {"choice": list(choice), "us": m[choice], "best": list(best), "best_us": m[best]}
        for i, (upto, (algo, proto, nch)) in enumerate(group):
            mb = upto if i + 1 < len(group) else 2**64 - 1
            rows.append([0, n, mb, CODES_A[algo], CODES_P[proto], nch])
    print(json.dumps({"name": "b200_virtual",
                      "cite": f"measured on one B200, virtual ranks, CUDA-graph device time: {a.path} "
                              f"(scripts/tune_policy.py, scripts/derive_policy.py --tol {a.tol})",
                      "note": "per rank count: fastest (algo, proto, nch) per size, kept while within tol",
                      "rows": rows, "detail": detail}, indent=1))


if __name__ == "__main__":
    main()
