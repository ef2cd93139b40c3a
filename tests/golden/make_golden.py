#!/usr/bin/env python3
"""Generate the golden fixtures of tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libranklab_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run in the container that has /root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed):
  cup_small.npz   ~300 small matrices (inputs, p, packed body, rank, rrp, sigma,
                  op counts) over p in {2,3,5,7,11,251,257,65521,8388593,2^31-1},
                  random / rank-deficient (random_rank_matrix, spread and generic) /
                  zero-leading-column / zero-row / m>n / empty shapes.
  mm_small.npz    mm(alpha, beta) cases with the reference's results.
  digests.json    sha256 digests of the reference cup output on the seeded
                  configs (C1 1024^2; a C2-style 1024x2048 rank-deficient
                  instance; 16 config-4 matrices) plus their ranks/profiles.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def c2_style(m, n, inner, seed, p):
    """BASELINE config 2 recipe at a given size: A = L*R mod p, rows i = 2 (mod 3)
    zeroed, rows shuffled by Fisher-Yates with SplitMix64(seed+2)."""
    L = O.ref_random_matrix(m, inner, seed, p)
    R = O.ref_random_matrix(inner, n, seed + 1, p)
    A = np.zeros((m, n), np.uint32)
    O.ref_mm(L, R, A, 1, 0, p)
    A[2::3, :] = 0
    s = np.arange(m, dtype=np.int64)
    rnd = O.ref_splitmix64(seed + 2, m)
    t = 0
    for i in range(m, 1, -1):
        j = int(rnd[t] % np.uint64(i))
        t += 1
        s[i - 1], s[j] = s[j], s[i - 1]
    return np.ascontiguousarray(A[s, :])  # new row i = old row s[i] (perm.cpp:103-113)


def c4_matrix(meta_rng, p):
    """BASELINE config 4 recipe for one matrix: r = 128 + below(129); L 256 x r,
    R r x 256 from random_matrix with seeds from the meta stream; A = L*R."""
    r = 128 + int(meta_rng[0] % np.uint64(129))
    L = O.ref_random_matrix(256, r, int(meta_rng[1]), p)
    R = O.ref_random_matrix(r, 256, int(meta_rng[2]), p)
    A = np.zeros((256, 256), np.uint32)
    O.ref_mm(L, R, A, 1, 0, p)
    return A, r


def main():
    assert O.have_ref(), "build oracle/_ref first (make -C oracle ref)"
    rng = np.random.default_rng(20261020)
    primes = [2, 3, 5, 7, 11, 251, 257, 65521, 8388593, 2147483647]
    cases = []
    for t in range(320):
        p = int(primes[t % len(primes)])
        kind = t % 8
        m = int(rng.integers(0, 40))
        n = int(rng.integers(0, 40))
        if kind == 7:
            m, n = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        if kind in (1, 2) and m and n:
            r = int(rng.integers(0, min(m, n) + 1))
            a = O.ref_random_rank_matrix(m, n, r, int(rng.integers(0, 2**62)), p, generic=(kind == 2))
        else:
            a = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
            if kind == 3 and n > 2:
                a[:, : n // 2] = 0
            if kind == 4 and m > 2:
                a[::2, :] = 0
            if kind == 5:  # tall: exercises the r1 == n early return (factor.cpp:47)
                a = rng.integers(0, p, (m + 12, max(1, n // 3)), dtype=np.uint64).astype(np.uint32)
        a = np.ascontiguousarray(a)
        body = a.copy()
        res = O.ref_cup(body, p)
        cases.append((p, a, body, res))
    np.savez_compressed(
        os.path.join(HERE, "cup_small.npz"),
        count=len(cases),
        **{f"p_{i}": np.uint64(c[0]) for i, c in enumerate(cases)},
        **{f"a_{i}": c[1] for i, c in enumerate(cases)},
        **{f"body_{i}": c[2] for i, c in enumerate(cases)},
        **{f"rank_{i}": np.int64(c[3].rank) for i, c in enumerate(cases)},
        **{f"rrp_{i}": c[3].rrp for i, c in enumerate(cases)},
        **{f"sigma_{i}": c[3].sigma for i, c in enumerate(cases)},
        **{f"ops_{i}": c[3].ops for i, c in enumerate(cases)},
    )

    mms = []
    for t in range(60):
        p = int(primes[t % len(primes)])
        m, l, n = (int(x) for x in rng.integers(0, 30, 3))
        a = rng.integers(0, p, (m, l), dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, p, (l, n), dtype=np.uint64).astype(np.uint32)
        c = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        alpha = int([1, p - 1, 0, int(rng.integers(0, p))][t % 4])
        beta = int([1, 0, int(rng.integers(0, p)), 1][t % 4])
        out = c.copy()
        O.ref_mm(a, b, out, alpha, beta, p)
        mms.append((p, a, b, c, alpha, beta, out))
    np.savez_compressed(
        os.path.join(HERE, "mm_small.npz"), count=len(mms),
        **{f"p_{i}": np.uint64(x[0]) for i, x in enumerate(mms)},
        **{f"a_{i}": x[1] for i, x in enumerate(mms)},
        **{f"b_{i}": x[2] for i, x in enumerate(mms)},
        **{f"c_{i}": x[3] for i, x in enumerate(mms)},
        **{f"alpha_{i}": np.uint64(x[4]) for i, x in enumerate(mms)},
        **{f"beta_{i}": np.uint64(x[5]) for i, x in enumerate(mms)},
        **{f"out_{i}": x[6] for i, x in enumerate(mms)},
    )

    dig = {}
    # C1
    a = O.ref_random_matrix(1024, 1024, 1, 65521)
    dig["c1_input"] = digest(a)
    res = O.ref_cup(a, 65521)
    dig["c1"] = dict(m=1024, n=1024, p=65521, seed=1, rank=res.rank,
                     rrp_identity=bool(np.array_equal(res.rrp, np.arange(res.rank))),
                     sigma=digest(res.sigma), body=digest(a), ops=[int(x) for x in res.ops])
    # C2-style at reduced size
    a = c2_style(1024, 2048, 512, 2, 65521)
    dig["c2s_input"] = digest(a)
    res = O.ref_cup(a, 65521)
    dig["c2s"] = dict(m=1024, n=2048, inner=512, p=65521, seed=2, rank=res.rank,
                      rrp=[int(x) for x in res.rrp], sigma=digest(res.sigma), body=digest(a),
                      ops=[int(x) for x in res.ops])
    # C4: first 16 matrices of the batch
    p4 = 8388593
    meta = O.ref_splitmix64(4, 3 * 16)
    c4 = []
    for t in range(16):
        A, r = c4_matrix(meta[3 * t: 3 * t + 3], p4)
        inp = digest(A)
        res = O.ref_cup(A, p4)
        c4.append(dict(r_gen=r, input=inp, rank=res.rank, rrp=digest(res.rrp),
                       sigma=digest(res.sigma), body=digest(A)))
    dig["c4"] = dict(p=p4, seed=4, mats=c4)
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(dig, f, indent=1)
    print("wrote", len(cases), "cup cases,", len(mms), "mm cases, digests")


if __name__ == "__main__":
    main()
