#!/usr/bin/env python3
"""Per-kernel summary of an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum[,...] --csv` launch list: launches, total / median time,
DRAM bytes and the achieved DRAM throughput (bytes / duration) of the launches
that move more than 1 MB (tiny launches are latency-bound).
Usage: ncu_metric_summary.py launches.csv [peak_GBps]"""
import collections
import csv
import statistics
import sys

path = sys.argv[1]
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
h = rows[0]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
launch = collections.defaultdict(dict)
name = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    launch[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    name[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
per = collections.defaultdict(list)
for i, m in launch.items():
    per[name[i]].append(m)
print(f"{'kernel':28s} {'n':>5s} {'total ms':>9s} {'med us':>8s} {'DRAM MB':>9s} "
      f"{'GB/s all':>9s} {'GB/s >1MB':>10s} {'n>1MB':>6s}" + ("  frac>1MB" if peak else ""))
for k, ls in sorted(per.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
    t = [m.get("gpu__time_duration.sum", 0.0) for m in ls]  # ns
    b = [m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in ls]
    big = [(bb, tt) for bb, tt in zip(b, t) if bb > 1e6]
    gbs_all = sum(b) / sum(t) if sum(t) else 0.0
    gbs_big = sum(x for x, _ in big) / sum(y for _, y in big) if big else 0.0
    line = (f"{k:28s} {len(ls):5d} {sum(t)/1e6:9.3f} {statistics.median(t)/1e3:8.1f} {sum(b)/1e6:9.1f} "
            f"{gbs_all:9.1f} {gbs_big:10.1f} {len(big):6d}")
    if peak:
        line += f"  {gbs_big/peak:8.3f}"
    print(line)
