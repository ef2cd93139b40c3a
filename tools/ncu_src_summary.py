#!/usr/bin/env python3
"""Warp-state samples of an ncu --set full --import-source capture, summed by
source line (all launches of the report).  Usage: ncu_src_summary.py rep [top] [column]
(column: a source-page column to sum instead, e.g. "Instructions Executed")."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
COL = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"  # or "Instructions Executed"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur, hdr, si = None, None, None
agg, src, tot = collections.Counter(), {}, 0.0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index(COL)
        continue
    if r[0] == "Function Name" or hdr is None or len(r) <= si or not r[0]:
        continue
    try:
        v = float(r[si])
    except ValueError:
        continue
    key = (cur, int(r[0]))
    agg[key] += v
    src[key] = r[1][:100]
    tot += v
print(f"{rep}: {tot:.0f} {COL}")
for k, v in agg.most_common(top):
    print(f"{v:7.0f} {100 * v / tot:5.1f}%  {k[0]}:{k[1]}  {src[k]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ni, vi, ui, ii = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
want = ("Duration", "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "L2 Hit Rate", "Memory Throughput")
for r in rows[1:]:
    if r[ni] in want:
        print(f"  launch {r[ii]} {r[ni]:36s} {r[vi]:>10s} {r[ui]}")
