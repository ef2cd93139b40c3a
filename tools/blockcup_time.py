#!/usr/bin/env python3
"""Standalone time of the distributed driver's row-block CUP (1024 x w over
GF(65521)) through DeviceOps.cup, on the current stream and on a side stream,
warm engines, no concurrent work.  Usage: blockcup_time.py [w ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402
from paper_1112_5717_b200 import dist as D  # noqa: E402

ops = D.DeviceOps(65521)
side = torch.cuda.Stream(priority=-1)
for w in [int(x) for x in sys.argv[1:]] or [2048, 65536]:
    src = torch.empty((1024, w), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(src, 1024, w, 7, 65521)
    R = torch.empty_like(src)
    for name, st in (("current", torch.cuda.current_stream()), ("side", side)):
        ts = []
        for i in range(6):
            R.copy_(src)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(st):
                ops.cup(R)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"1024 x {w} on {name}: min {min(ts[2:])*1e3:.3f} ms, first {ts[0]*1e3:.1f} ms", flush=True)
