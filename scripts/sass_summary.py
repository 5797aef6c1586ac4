"""SASS evidence per kernel of libpolar.so (cuobjdump), written to profiles/.

python scripts/sass_summary.py [--dtype f32] > profiles/sass_summary.txt
Counts the instructions that evidence the design choices (B200_PROFILING.md
"What proves a Blackwell-native kernel"; SURVEY.md §0 PTX->SASS table):
  LDG.E.128 / STG.E.128      16-byte vector loads/stores (Simple data path)
  .STRONG.SYS / .STRONG.GPU  flag polls / LL lines / .cg loads
  UBLKCP.S.G / UBLKCP.G.S    TMA bulk copies global->smem / smem->global
  SYNCS.*                    mbarrier (transaction-count) operations
  MEMBAR.ALL.SYS / .GPU      release fences before flags
  BAR.ARV / BAR.SYNC         named-barrier hand-offs (warp-specialised ring / tree Simple)
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_11438_b200", "libpolar.so")
DT = {"i32": 2, "i64": 4, "f32": 7, "bf16": 9}
ALGO = {0: "tree", 1: "ring", 3: "oneshot", 4: "twoshot"}
PROTO = {0: "ll", 1: "ll128", 2: "simple"}
OP = {0: "sum", 2: "max", 3: "min"}
PATS = ["LDG.E.128", "STG.E.128", "STRONG.SYS", "STRONG.GPU", "UBLKCP.S.G", "UBLKCP.G.S", "SYNCS", "SHFL", "VOTE",
        "MEMBAR.ALL.SYS", "MEMBAR.ALL.GPU", "FADD", "NANOSLEEP", "BAR.ARV", "BAR.SYNC"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--op", default="sum")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    rows = []
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        m = re.match(r"_ZN5polar3dev16allreduce_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)EEEvNS0_6ParamsE", name)
        if not m:
            continue
        dt, op, algo, proto = (int(x) for x in m.groups())
        if dt != DT[a.dtype] or op != {v: k for k, v in OP.items()}[a.op]:
            continue
        c = collections.Counter()
        ninstr = 0
        for line in f.split("\n"):
            if re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
                ninstr += 1
                for p in PATS:
                    if p in line:
                        c[p] += 1
        rows.append((ALGO[algo], PROTO[proto], ninstr, c))
    print(f"# SASS evidence, libpolar.so, allreduce_kernel<{a.dtype},{a.op},algo,proto> (cuobjdump -sass, static counts)")
    print("# kernel               instrs  " + "  ".join(PATS))
    for algo, proto, ninstr, c in sorted(rows):
        print(f"{algo + '/' + proto:20s} {ninstr:7d}  " + "  ".join(f"{c[p]:{len(p)}d}" for p in PATS))


if __name__ == "__main__":
    main()
