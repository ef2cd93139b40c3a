#!/usr/bin/env python3
"""Leaf-chain breakdown of one warm C3 factorization from a -DRL_LEAFTRACE build
(tools/build_variant.sh lt "-DRL_LEAFTRACE"): window kernel time (after its
pdl_wait) and the gap from one window's exit to the next window's start, summed
by the level of the transition.  Usage: leaftrace.py lib.so [n] [p]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    import paper_1112_5717_b200 as G
    G.LIB_PATH = os.path.abspath(sys.argv[2])
    n, p = int(sys.argv[3]), int(sys.argv[4])
    src = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(src, n, n, 3, p)
    work = src.clone()
    G.cup_dev(work, n, n, p)
    torch.cuda.synchronize()
    work.copy_(src)
    torch.cuda.synchronize()
    G.cup_dev(work, n, n, p)
    torch.cuda.synchronize()
    import ctypes
    import numpy as np
    lib = G.lib()
    print("=== timed rep", flush=True)
    for tag, fn in (("W", "rl_lt_dump_window"), ("B", "rl_lt_dump_bridge")):
        h = np.zeros((1024, 8), np.uint64)
        if getattr(lib, fn)(h.ctypes.data_as(ctypes.c_void_p)) != 0:
            continue
        for k in range(1024):
            if h[k, 0]:
                print(f"LT {tag} {k * 64} {h[k, 0]} {h[k, 1]}" + "".join(f" {int(x)}" for x in h[k, 2:]))
    sys.exit(0)

lib = sys.argv[1]
n = sys.argv[2] if len(sys.argv) > 2 else "16384"
p = sys.argv[3] if len(sys.argv) > 3 else "65521"
out = subprocess.run([sys.executable, __file__, "--child", lib, n, p], capture_output=True, text=True).stdout
out = out.split("=== timed rep", 1)[-1]
ev = collections.defaultdict(dict)
for l in out.splitlines():
    m = re.match(r"LT (\w+) (-?\d+) (\d+) (\d+)(.*)", l)
    if m:
        ev[m.group(1)][int(m.group(2))] = (int(m.group(3)), int(m.group(4))) + tuple(int(x) for x in m.group(5).split())
W = sorted(ev["W"].items())
print(f"{lib}: windows {len(W)}, bridges {len(ev.get('B', {}))}")
t0 = W[0][1][0]
dur = collections.defaultdict(list)
gap = collections.defaultdict(list)
PB = 64
for k in range(1, len(W)):
    lvl = (k & -k).bit_length() - 1
    gap[lvl].append(W[k][1][0] - W[k - 1][1][1])
    dur[lvl].append(W[k][1][1] - W[k][1][0])
tg = td = 0
for lvl in sorted(gap):
    g, d = gap[lvl], dur[lvl]
    tg += sum(g)
    td += sum(d)
    print(f"  level {lvl}: {len(g):3d} transitions, gap sum {sum(g)/1e6:6.2f} ms (avg {sum(g)/len(g)/1e3:6.1f} us), "
          f"window avg {sum(d)/len(d)/1e3:5.1f} us")
print(f"  total: windows {td/1e6:.2f} ms + gaps {tg/1e6:.2f} ms; first window start -> last window end "
      f"{(W[-1][1][1] - t0)/1e6:.2f} ms")
if os.environ.get("LT_ALL"):  # every gap, 16 leaves (one 1024-row tile) per line
    for k0 in range(0, len(W), 16):
        print(f"  gaps before leaves {k0:3d}..: " + " ".join(
            f"{(W[k][1][0] - W[k - 1][1][1]) / 1e3:5.0f}" if k else "    -" for k in range(k0, min(k0 + 16, len(W)))))
    med = collections.defaultdict(list)
    for k in range(1, len(W)):
        med[k % 16].append((W[k][1][0] - W[k - 1][1][1]) / 1e3)
    import statistics as _st
    print("  median gap by position in the tile: " + " ".join(f"{_st.median(med[q]):.0f}" for q in range(16)))
    print("  mean   gap by position in the tile: " + " ".join(f"{sum(med[q]) / len(med[q]):.0f}" for q in range(16)))
slow = sorted(((W[k][1][0] - W[k - 1][1][1], k) for k in range(1, len(W))), reverse=True)[:24]
print("  slowest transitions (us, leaf index: level): " +
      ", ".join(f"{g/1e3:.0f} @{k}:{(k & -k).bit_length() - 1}" for g, k in slow))
wph = [v for _, v in W if len(v) > 5 and v[2] and v[3] and v[5]]
if wph:
    import statistics
    names = ("loaded", "LU done", "A written", "Minv written", "exit")
    cols = (2, 3, 4, 5, 1)
    print("  window phases (us from its pdl_wait, median over leaves): " + ", ".join(
        f"{nm} {statistics.median([(v[c] - v[0]) / 1e3 for v in wph if v[c]]):.2f}" for nm, c in zip(names, cols)))
if "B" in ev:
    bd = [v[1] - v[0] for v in ev["B"].values()]
    print(f"  bridge avg {sum(bd)/len(bd)/1e3:.1f} us")
    import statistics
    ph = [[(v[i] - v[0]) / 1e3 for v in ev["B"].values() if v[i]] for i in (2, 3, 4)]
    print("  bridge phases (us from begin, median): " + ", ".join(f"{statistics.median(x):.2f}" for x in ph if x))
if "B" in ev:
    import statistics
    rel = collections.defaultdict(list)
    Wd = dict(W)
    for row0, v in ev["B"].items():
        top = row0 - 64
        if top not in Wd or row0 not in Wd:
            continue
        wend = Wd[top][1]
        rel["bridge begin"].append(v[0] - wend)
        for i, nm in ((2, "mark2"), (3, "operands"), (4, "G stored")):
            if v[i]:
                rel[nm].append(v[i] - wend)
        rel["bridge end"].append(v[1] - wend)
        rel["next window begin"].append(Wd[row0][0] - wend)
    print("  level-0 transition, us after the top window's exit (median): " +
          ", ".join(f"{k} {statistics.median(x)/1e3:.2f}" for k, x in rel.items()))
