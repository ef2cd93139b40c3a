#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel totals of the second half of the launches (the warm repetition)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if "Kernel Name" in r][0]
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and "Kernel Name" not in r]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
part = data[int(len(data) * (1 - frac)):]
by = collections.defaultdict(list)
for d in part:
    by[re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")].append(float(d["Metric Value"]))
T = sum(sum(v) for v in by.values())
for k, v in sorted(by.items(), key=lambda x: -sum(x[1])):
    ts = sorted(v)
    print(f"{sum(v)/1e6:8.2f} ms {100*sum(v)/T:5.1f}%  n={len(v):5d}  med={ts[len(ts)//2]/1e3:7.1f}us  "
          f"max={ts[-1]/1e3:8.1f}us  {k[:60]}")
print(f"total {T/1e6:.2f} ms over {len(part)} launches")
