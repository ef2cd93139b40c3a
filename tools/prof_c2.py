#!/usr/bin/env python3
"""One warm CUP of the config-2 matrix (4096 x 8192, rank 2048, shuffled zero
rows) for ncu launch lists.  Usage: prof_c2.py [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402
from paper_1112_5717_b200 import workloads as WL  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
m, n, p = 4096, 8192, 65521
src = WL.c2_dev(m, n, 2048, 2, p)
work = torch.empty_like(src)
for i in range(reps + 1):
    work.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = G.cup_dev(work, m, n, p)
    dt = time.perf_counter() - t0
    print(f"rep {i}: rank {r.rank}  {dt*1e3:.2f} ms", flush=True)
