"""Summarise ncu captures from gpurun_out/ into profiles/ (tracked).

python scripts/ncu_summary.py TAG [--workload virtual8_f32_128MiB]
  reads gpurun_out/launches_TAG.csv (launch list, gpu__time_duration.sum) and
  gpurun_out/prof_TAG.ncu-rep (--set full of the top kernel); writes
  profiles/TAG_launches.csv, profiles/TAG_launch_shares.txt,
  profiles/TAG_ncu_full_metrics.txt and profiles/traffic.json.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "sm__maximum_warps_per_active_cycle_pct", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__cycles_active.avg",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum"]


def launch_shares(tag, kind=""):
    """kind "" = the whole bench run; "timed" = the NVTX "timed" range only."""
    src = os.path.join(OUT, f"launches_{kind + '_' if kind else ''}{tag}.csv")
    if not os.path.exists(src):
        return
    rows = list(csv.reader(open(src)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            recs.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in recs:
        k = (d["Kernel Name"], d["Grid Size"], d["Block Size"])
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values()) or 1.0
    what = "the timed region only (NVTX range 'timed')" if kind else "the whole bench.py run"
    lines = [f"# ncu launch list of {what} ({os.path.basename(src)}), gpu__time_duration.sum, "
             "--clock-control none (cold, serialised)",
             "# launches  total_us  share  mean_us  kernel grid block"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[0]:8d} {v[1] / 1e3:10.1f} {100 * v[1] / tot:6.1f}% {v[1] / v[0] / 1e3:9.2f}  {k[0]} {k[1]} {k[2]}")
    suffix = f"_{kind}" if kind else ""
    shutil.copy(src, os.path.join(PROF, f"{tag}_launches{suffix}.csv"))
    with open(os.path.join(PROF, f"{tag}_launch_shares{suffix}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines[:8]))


def full_metrics(tag, workload):
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = r[0], r[1], r[2:]
    lines = [f"# ncu --set full --clock-control none capture ({os.path.basename(rep)})"]
    traffic = None
    for v in vals:
        name = v[hdr.index("Kernel Name")]
        lines.append(f"kernel: {name}")
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k} = {v[i]} {units[i]}")
                d[k] = (v[i], units[i])
        for op in ("ld", "st"):   # 16 sectors per request = full-warp 16-B accesses
            ks, kr = f"l1tex__t_sectors_pipe_lsu_mem_global_op_{op}.sum", f"l1tex__t_requests_pipe_lsu_mem_global_op_{op}.sum"
            if ks in d and kr in d and float(d[kr][0]) > 0:
                lines.append(f"  global {op} sectors/request = {float(d[ks][0]) / float(d[kr][0]):.2f}")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if "dram__bytes_read.sum" in d:
            rb = float(d["dram__bytes_read.sum"][0]) * scale[d["dram__bytes_read.sum"][1]]
            wb = float(d["dram__bytes_write.sum"][0]) * scale[d["dram__bytes_write.sum"][1]]
            traffic = {"workload": workload, "kernel": name, "dram_bytes_per_launch": int(rb + wb),
                       "dram_read": int(rb), "dram_write": int(wb), "source": f"profiles/{tag}_ncu_full_metrics.txt"}
    with open(os.path.join(PROF, f"{tag}_ncu_full_metrics.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic:
        with open(os.path.join(PROF, "traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--workload", default="virtual8_f32_128MiB")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    launch_shares(a.tag)
    launch_shares(a.tag, "timed")
    full_metrics(a.tag, a.workload)


if __name__ == "__main__":
    main()
