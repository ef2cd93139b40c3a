#!/usr/bin/env python3
"""Per-phase device time of the distributed CUP driver at world 1
(python tools/prof_dist.py M P [block] [tile]): CUDA events around every
phase of dist_cup (row-block gather, block CUP, trsm, Schur GEMM, ...)."""
import os
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1112_5717_b200 import dist as D  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
p = int(sys.argv[2]) if len(sys.argv) > 2 else 65521
block = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
tile = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
sb = int(sys.argv[5]) if len(sys.argv) > 5 else 4096
window = int(sys.argv[6]) if len(sys.argv) > 6 else 0  # > 0: window mode (the N > 1 default, 2 x block)
torch.cuda.set_device(0)
tiles = D.ColumnTiles(m, 1, tile)
pristine = D.random_matrix_local(m, m, 5, p, tiles, 0, "cuda")
x = torch.empty_like(pristine)

acc = defaultdict(float)
cnt = defaultdict(int)
pending = []


def timed(name, fn):
    def w(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn(*a, **k)
        e1.record()
        pending.append((name, e0, e1))
        return out
    return w


ops = D.DeviceOps(p)
ops.cup = timed("block_cup", ops.cup)
ops.trsm_right_upper_unit = timed("trsm", ops.trsm_right_upper_unit)
ops.trsm_left_lower_nonunit = timed("trsm_beyond_window", ops.trsm_left_lower_nonunit)
ops.mm_sub = timed("schur_mm", ops.mm_sub)
E = D._Engine
orig = {k: getattr(E, k) for k in ("gather_cols", "put_cols", "permute_cols", "shift_u_rows",
                                   "solve_rows")}
for k, f in orig.items():
    setattr(E, k, timed(k, f))

for it in range(3):
    x.copy_(pristine)
    pending.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = D.dist_cup(x, m, m, p, tiles, block=block, superblock=sb, ops=ops, window=window)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
acc.clear()
cnt.clear()
for name, a, b in pending:
    acc[name] += a.elapsed_time(b)
    cnt[name] += 1
print(f"m={m} p={p} block={block} tile={tile} sb={sb} window={window} rank={res.rank} steps={res.steps}")
print(f"total device {e0.elapsed_time(e1):.2f} ms, host wall {wall * 1e3:.2f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:14s} {v:9.2f} ms  n={cnt[k]}")
