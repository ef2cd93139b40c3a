#!/usr/bin/env python3
"""Per-CTA timelines of the leaf at row RL_TRACE_I0 (8192) from the -DRL_TRACE
build (make -C paper_1112_5717_b200/csrc trace).  Usage: trace_cup.py [n] [p]
Prints kernel phases relative to the window kernel's entry, in microseconds."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ROOT)
    import torch
    import paper_1112_5717_b200 as G
    G.LIB_PATH = os.path.join(ROOT, "paper_1112_5717_b200", "libranklab_gpu_trace.so")
    n, p = int(sys.argv[2]), int(sys.argv[3])
    src = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(src, n, n, 3, p)
    work = src.clone()
    G.cup_dev(work, n, n, p)  # warm (plans, graph)
    torch.cuda.synchronize()
    print("=== timed rep", flush=True)
    work.copy_(src)
    torch.cuda.synchronize()
    G.cup_dev(work, n, n, p)
    torch.cuda.synchronize()
    sys.exit(0)

n = sys.argv[1] if len(sys.argv) > 1 else "16384"
p = sys.argv[2] if len(sys.argv) > 2 else "65521"
out = subprocess.run([sys.executable, __file__, "--child", n, p], capture_output=True, text=True).stdout
out = out.split("=== timed rep", 1)[-1]
lines = [l for l in out.splitlines() if l.startswith("TRACE")]
t0 = None
for l in lines:
    if l.startswith("TRACE window") or l.startswith("TRACE trsm"):
        t0 = int(re.search(r"enter (\d+)", l).group(1))
        break
if t0 is None:
    print(out[-2000:])
    sys.exit(1)
rel = lambda m: f"{(int(m.group(0)) - t0) / 1e3:8.2f}"
tails = []
for l in lines:
    if l.startswith(("TRACE window", "TRACE spec", "TRACE trsm", "TRACE tailw", "TRACE wblk", "TRACE solo")):
        print(re.sub(r"\b(\d{12,})\b", lambda m: rel(m), l))
    elif not l.startswith("TRACE tail"):
        print(l)
    else:
        tails.append([int(x) for x in re.findall(r"\b(\d{12,})\b", l)] + [l])
tails.sort(key=lambda t: t[2])
for t in tails[:2] + tails[-4:]:
    print(re.sub(r"\b(\d{12,})\b", lambda m: rel(m), t[-1]))
if tails:
    print(f"tail CTAs {len(tails)}: enter {min(t[0] for t in tails) - t0:.0f}..{max(t[0] for t in tails) - t0:.0f} ns, "
          f"exit max {max(t[2] for t in tails) - t0:.0f} ns")
