#!/usr/bin/env python3
"""Small CUP factorizations for compute-sanitizer (racecheck / memcheck /
synccheck): a generic leaf (speculative window path), a GF(3) rank-deficient
matrix with zero leading columns (exact lockstep path, transpositions, U-row
moves), a 31-bit prime (64-bit reduction path) and a small batched call, each
checked bit-exactly against the oracle port.  Usage: sanitize_cup.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_1112_5717_b200 as G  # noqa: E402

rng = np.random.default_rng(7)
cases = []
cases.append((rng.integers(0, 65521, (192, 256), dtype=np.uint64).astype(np.uint32), 65521))
b = rng.integers(0, 3, (160, 200), dtype=np.uint64).astype(np.uint32)
b[:, :40] = 0
b[::5, :] = 0
cases.append((b, 3))
cases.append((rng.integers(0, 2**31 - 1, (130, 150), dtype=np.uint64).astype(np.uint32), 2**31 - 1))
bad = 0
for a, p in cases:
    g_body, o_body = a.copy(), a.copy()
    g = G.cup(g_body, p)
    o = O.port_cup(o_body, p)
    ok = (g.rank == o.rank and np.array_equal(g.row_profile, o.rrp)
          and np.array_equal(g.col_perm, o.sigma) and np.array_equal(g_body, o_body))
    print(f"cup {a.shape} p={p}: rank {g.rank} {'OK' if ok else 'MISMATCH'}", flush=True)
    bad += not ok
bt = rng.integers(0, 8388593, (3, 256, 256), dtype=np.uint64).astype(np.uint32)
gb = bt.copy()
ranks, _, _ = G.cup_batched(gb, 8388593)
for t in range(bt.shape[0]):
    ob = bt[t].copy()
    o = O.port_cup(ob, 8388593)
    ok = ranks[t] == o.rank and np.array_equal(gb[t], ob)
    print(f"batched[{t}]: rank {ranks[t]} {'OK' if ok else 'MISMATCH'}", flush=True)
    bad += not ok
sys.exit(1 if bad else 0)
