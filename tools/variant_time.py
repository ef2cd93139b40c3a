#!/usr/bin/env python3
"""Time C3 (16384^2, p = 65521) with an alternative build of the library
(variant_time.py path/to/libranklab_gpu.so [n]): engine tuning experiments;
n = 65536 times config 5 instead."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

G.LIB_PATH = os.path.abspath(sys.argv[1])
n, p = (int(sys.argv[2]) if len(sys.argv) > 2 else 16384), 65521
src = torch.empty((n, n), dtype=torch.int32, device="cuda")
G.random_matrix_dev(src, n, n, 3, p)
work = torch.empty_like(src)
ts = []
nrep = 6 if n <= 16384 else 4
for i in range(nrep):
    work.copy_(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.cup_dev(work, n, n, p, sync=False)
    e1.record()
    e1.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
print(f"{sys.argv[1]}: {min(ts):.2f} ms (min of {len(ts)}), mean {sum(ts)/len(ts):.2f}")
