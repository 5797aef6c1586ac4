"""Top CUDA source lines of an ncu report by warp-stall samples, with the main
stall reasons (ncu --page source --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr) if h not in ("Source",)}
i_s = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = [r for r in rows[hi + 1:] if len(r) > i_s and r[0] not in ("", "-")]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0



tot = sum(f(r[i_s]) for r in lines)
print("total samples", tot)
for r in sorted(lines, key=lambda r: -f(r[i_s]))[:ntop]:
    s = f(r[i_s])
    rs = sorted(((f(r[hdr.index(k)]), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{s / tot * 100:5.1f}% L{r[0]:>4} {' '.join(f'{k}={v / max(s, 1) * 100:.0f}%' for v, k in rs):40s} {r[1].strip()[:80]}")
