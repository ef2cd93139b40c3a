#!/usr/bin/env python3
"""Host-buffer CUP (rl_cup_u32, pinned memory) of C3: link rates alone, then a
device timeline (CUPTI via torch.profiler: copies and kernels with streams) of
one warm call.  Usage: e2e_trace.py [n] [out.json]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
out = sys.argv[2] if len(sys.argv) > 2 else "e2e_trace.json"
p = 65521
host = torch.empty((n, n), dtype=torch.int32, pin_memory=True)
dev = torch.empty((n, n), dtype=torch.int32, device="cuda")
G.random_matrix_dev(dev, n, n, 3, p)
src = dev.cpu().numpy().view(np.uint32).copy()
for name, fn in (("H2D", lambda: dev.copy_(host, non_blocking=True)),
                 ("D2H", lambda: host.copy_(dev, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name} 1 matrix ({n * n * 4 / 2**30:.2f} GiB): {dt * 1e3:.2f} ms = {n * n * 4 / dt / 1e9:.1f} GB/s")
hv = host.numpy().view(np.uint32)
for i in range(3):
    hv[...] = src
    t0 = time.perf_counter()
    G.cup(hv, p)
    print(f"rl_cup_u32 call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms")
hv[...] = src
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    G.cup(hv, p)
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
cp = [k for k in ks if "emcpy" in k[3] or "Memcpy" in k[3]]
print(f"{len(ks)} records, span {max(k[1] for k in ks) / 1e3:.2f} ms; copies:")
for k in cp:
    print(f"  {k[0] / 1e3:8.2f} -> {k[1] / 1e3:8.2f} ms  stream {k[2]}  {k[3]}")
wins = [k for k in ks if k[3].startswith("panel_window")]
for i in range(0, len(wins), 16):
    print(f"  window {i:3d} starts at {wins[i][0] / 1e3:7.2f} ms")
print(f"  last window ends at {wins[-1][1] / 1e3:7.2f} ms")
