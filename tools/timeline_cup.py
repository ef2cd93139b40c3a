#!/usr/bin/env python3
"""Device timeline of one warm CUP (CUPTI kernel records via torch.profiler):
per-kernel busy time, and the idle gaps between consecutive kernels.
Usage: timeline_cup.py [n|c2] [p] [out.json]"""
import collections
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "16384"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 65521
out = sys.argv[3] if len(sys.argv) > 3 else None
if arg == "c2":  # config 2: 4096 x 8192, rank 2048, shuffled zero rows
    from paper_1112_5717_b200 import workloads as WL
    m, n = 4096, 8192
    src = WL.c2_dev(m, n, 2048, 2, p)
else:
    m = n = int(arg)
    src = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(src, n, n, 3, p)
work = src.clone()
G.cup_dev(work, m, n, p)
work.copy_(src)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    G.cup_dev(work, m, n, p)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = []
for e in evs:
    name = e.name.replace("rl::(anonymous namespace)::", "").replace("void ", "")
    name = re.sub(r"\(.*", "", name)
    ks.append((e.time_range.start, e.time_range.end, name))
ks.sort()
ks = [k for k in ks if "copy" not in k[2].lower() and "Memcpy" not in k[2]]
t0, t1 = ks[0][0], max(k[1] for k in ks)
busy = collections.defaultdict(float)
cnt = collections.Counter()
gaps = collections.defaultdict(float)
for i, (s, e, nm) in enumerate(ks):
    busy[nm] += e - s
    cnt[nm] += 1
    if i:
        gaps[(ks[i - 1][2], nm)] += s - ks[i - 1][1]
span = t1 - t0
print(f"span {span/1e3:.2f} ms, kernels {len(ks)}, busy {sum(busy.values())/1e3:.2f} ms, "
      f"gaps {sum(gaps.values())/1e3:.2f} ms")
for nm, b in sorted(busy.items(), key=lambda x: -x[1]):
    print(f"  {b/1e3:8.2f} ms  n={cnt[nm]:5d}  avg {b/cnt[nm]:7.1f} us  {nm[:60]}")
print("largest gap totals (prev -> next):")
for (a, b), g in sorted(gaps.items(), key=lambda x: -x[1])[:10]:
    print(f"  {g/1e3:8.2f} ms  {a[:40]} -> {b[:40]}")
if out:
    json.dump([(s - t0, e - t0, nm) for s, e, nm in ks], open(out, "w"))
# overlap of each panel_window with other kernels (concurrency achieved)
wins = [k for k in ks if "panel_window" in k[2]]
ov = 0.0
for s0, e0, _ in wins:
    for s1, e1, nm in ks:
        if "panel_window" in nm:
            continue
        o = min(e0, e1) - max(s0, s1)
        if o > 0:
            ov += o
print(f"window time overlapped by other kernels: {ov/1e3:.2f} ms of {sum(e-s for s,e,_ in wins)/1e3:.2f} ms")
