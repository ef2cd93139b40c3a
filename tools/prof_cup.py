#!/usr/bin/env python3
"""One warm CUP factorization of random_matrix(n, n) over GF(p) for profiling
(ncu launch lists / --set full captures).  Usage: prof_cup.py [n] [p] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
p = int(sys.argv[2]) if len(sys.argv) > 2 else 65521
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
s = torch.cuda.current_stream()
src = torch.empty((n, n), dtype=torch.int32, device="cuda")
G.random_matrix_dev(src, n, n, 3, p, stream=s)
work = torch.empty_like(src)
for i in range(reps + 1):
    work.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = G.cup_dev(work, n, n, p, stream=s)
    dt = time.perf_counter() - t0
    print(f"rep {i}: rank {r.rank}  {dt*1e3:.2f} ms  "
          f"{G.model_ops(n, n, r.rank)/dt/1e12:.3f} Tops/s", flush=True)
print(G.plan_stats(n, n, p))
