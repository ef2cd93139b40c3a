#!/usr/bin/env python3
"""Config-4 batched CUP timing: 4096 (or argv[1]) matrices of 256x256 over GF(8388593)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402
from paper_1112_5717_b200 import workloads as W  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = 8388593
t0 = time.perf_counter()
mats, ranks = W.c4_dev(count, p=p)
torch.cuda.synchronize()
print(f"generated {count} matrices in {time.perf_counter() - t0:.2f} s")
work = mats.clone()
for it in range(4):
    work.copy_(mats)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    G.cup_batched_dev(work, count, 256, 256, p, want_meta=False)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"rep {it}: {ms:.2f} ms  {count / ms * 1e3:.0f} matrices/s")
rk, _, _ = G.cup_batched_dev(work.copy_(mats), count, 256, 256, p)
print("ranks ok:", all(int(a) == b for a, b in zip(rk, ranks)))
