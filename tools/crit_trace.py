#!/usr/bin/env python3
"""Raw device timeline of one warm CUP (CUPTI kernel records via torch.profiler,
with the stream of every kernel) for critical-path analysis offline.
Usage: crit_trace.py n p out.json  ->  [[start_us, end_us, stream, name], ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

n, p, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
src = torch.empty((n, n), dtype=torch.int32, device="cuda")
G.random_matrix_dev(src, n, n, 3, p)
work = src.clone()
G.cup_dev(work, n, n, p)
work.copy_(src)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    G.cup_dev(work, n, n, p)
    torch.cuda.synchronize()
tmp = out + ".chrome.json"
prof.export_chrome_trace(tmp)
ev = json.load(open(tmp))
ev = ev["traceEvents"] if isinstance(ev, dict) else ev
ks = []
for e in ev:
    if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy"):
        ks.append([float(e["ts"]), float(e["ts"]) + float(e["dur"]), int(e.get("tid", 0)),
                   e["name"].replace("rl::(anonymous namespace)::", "").replace("void ", "").split("(")[0]])
os.remove(tmp)
ks.sort()
t0 = ks[0][0]
for k in ks:
    k[0] -= t0
    k[1] -= t0
json.dump(ks, open(out, "w"))
print(f"{len(ks)} records, span {max(k[1] for k in ks)/1e3:.2f} ms")
