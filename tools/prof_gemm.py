#!/usr/bin/env python3
"""One mod-p GEMM C <- C - A*B (m x l x n) on device buffers, for ncu captures
of gemm_tc_kernel.  Usage: prof_gemm.py [m] [l] [n] [p]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

G.LIB_PATH = os.environ.get("RL_LIB", G.LIB_PATH)  # (variant builds)

m, l, n = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 8192, 8192)))
p = int(sys.argv[4]) if len(sys.argv) > 4 else 65521
a = torch.empty((m, l), dtype=torch.int32, device="cuda")
b = torch.empty((l, n), dtype=torch.int32, device="cuda")
c = torch.empty((m, n), dtype=torch.int32, device="cuda")
G.random_matrix_dev(a, m, l, 11, p)
G.random_matrix_dev(b, l, n, 12, p)
G.random_matrix_dev(c, m, n, 13, p)
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 3
mp, mg = G.profile_gemm_dev(a, b, c, m, l, n, p, iters=iters)
L = max(1, ((p - 1).bit_length() + 7) // 8)
print(f"{m}x{l}x{n} p={p}: pack {mp*1e3:.1f} us  gemm {mg*1e3:.1f} us  ({2*m*n*l*L*L/mg/1e9:.1f} int8 TOPS)")
