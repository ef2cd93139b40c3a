#!/usr/bin/env python3
"""One warm CUP of the swap-heavy case s1 (8192^2 over GF(3), rank <= 6144, first
40 columns zero: transpositions in most leaves, U-row moves) for ncu captures of
the permutation kernels.  Usage: prof_s1.py [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n, inner, p = 8192, 6144, 3
L = torch.empty((n, inner), dtype=torch.int32, device="cuda")
R = torch.empty((inner, n), dtype=torch.int32, device="cuda")
src = torch.empty((n, n), dtype=torch.int32, device="cuda")
G.random_matrix_dev(L, n, inner, 11, p)
G.random_matrix_dev(R, inner, n, 12, p)
G.mm_dev(L, R, src, n, inner, n, 1, 0, p)
del L, R
src[:, :40] = 0
work = torch.empty_like(src)
for i in range(reps + 1):
    work.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = G.cup_dev(work, n, n, p)
    dt = time.perf_counter() - t0
    print(f"rep {i}: rank {r.rank}  {dt*1e3:.2f} ms  {G.model_ops(n, n, r.rank)/dt/1e12:.3f} Tops/s", flush=True)
