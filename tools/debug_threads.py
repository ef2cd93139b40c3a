#!/usr/bin/env python3
"""Concurrency probe for the host-buffer entry point: pairs of job kinds run in
two host threads (cudaStreamPerThread each), N rounds; prints every error.
Usage: debug_threads.py [rounds]"""
import itertools
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rng = np.random.default_rng(4)
KINDS = {
    "mid65521": ((300, 400), 65521),
    "tiny3": ((3, 3), 3),
    "graph31": ((1100, 700), 2**31 - 1),
    "batch23": ((64, 256), 8388593),
}
mats = {k: rng.integers(0, p, s, dtype=np.uint64).astype(np.uint32) for k, (s, p) in KINDS.items()}


def run_pair(ka, kb):
    errs = []

    def work(k):
        try:
            for _ in range(rounds):
                b = mats[k].copy()
                G.cup(b, KINDS[k][1])
        except Exception as e:  # noqa: BLE001
            errs.append((k, repr(e)[:300]))

    th = [threading.Thread(target=work, args=(k,)) for k in (ka, kb)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return errs


for ka, kb in itertools.combinations_with_replacement(sorted(KINDS), 2):
    e = run_pair(ka, kb)
    print(f"{ka:10s} + {kb:10s}: {'OK' if not e else e}", flush=True)
