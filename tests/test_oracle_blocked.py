"""Pins the blocked, multithreaded CPU restatement (oracle/blocked.py) -- the
checker behind the config-3 / config-5 digests -- against the compiled
reference: every output (rank, row profile, sigma, packed body, exact op
counts) over random shapes, primes, ranks and leaf sizes, including the
early-return (r1 = n) and zero-row / zero-column structures, and the config
generators against the device recipes' host halves."""
import numpy as np
import pytest

import oracle as O
from oracle import blocked as B
from oracle import configs as CF

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")

PRIMES = [2, 3, 5, 7, 251, 65521, 1000003, 8388593, 67108859, 2**31 - 1]


def _case(rng, p, kind, m, n):
    if kind == 0:
        return rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
    if kind == 1:
        r = int(rng.integers(0, max(1, min(m, n)) + 1))
        if m * n == 0:
            return np.zeros((m, n), np.uint32)
        return O.ref_random_rank_matrix(m, n, r, int(rng.integers(0, 2**63)), p)
    if kind == 2:
        a = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        a[:, : n // 3] = 0
        a[::3] = 0
        return a
    return (rng.integers(0, p, (m, n), dtype=np.uint64) * (rng.random((m, n)) < 0.1)).astype(np.uint32)


@needs_ref
@pytest.mark.parametrize("p", PRIMES)
def test_blocked_equals_reference(p):
    rng = np.random.default_rng(p)
    for trial in range(24):
        m, n = int(rng.integers(0, 100)), int(rng.integers(0, 100))
        a = _case(rng, p, trial % 4, m, n)
        leaf = int(rng.choice([1, 2, 3, 5, 8, 32, 64]))
        x, y = a.copy(), a.copy()
        rr = O.ref_cup(x, p)
        bb = B.cup(y, p, leaf=leaf)
        ctx = f"p={p} {m}x{n} kind={trial % 4} leaf={leaf}"
        assert rr.rank == bb.rank, ctx
        assert np.array_equal(rr.rrp, bb.rrp), ctx
        assert np.array_equal(rr.sigma, bb.sigma), ctx
        assert np.array_equal(x, y), ctx
        assert tuple(int(v) for v in rr.ops) == B.opcount(m, n, bb.rrp, bb.ipiv), ctx


@needs_ref
def test_blocked_tall_and_wide_extremes():
    rng = np.random.default_rng(5)
    for m, n, p in [(300, 7, 65521), (7, 300, 65521), (1, 500, 3), (500, 1, 3), (257, 255, 2)]:
        a = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        x, y = a.copy(), a.copy()
        rr = O.ref_cup(x, p)
        bb = B.cup(y, p, leaf=16)
        assert rr.rank == bb.rank and np.array_equal(x, y) and np.array_equal(rr.sigma, bb.sigma)


def test_digest_matches_definition():
    rng = np.random.default_rng(3)
    a = rng.integers(0, 2**31, (37, 53), dtype=np.uint64).astype(np.uint32)
    M = (1 << 64) - 1

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    h = 0
    for i in range(37):
        for j in range(53):
            h = (h + mix((((i * 53 + j) << 32 | int(a[i, j])) + 0x9E3779B97F4A7C15) & M)) & M
    assert B.digest(a) == h
    # strided view digests its own logical entries
    big = np.zeros((37, 80), np.uint32)
    big[:, 10:63] = a
    assert B.digest(big[:, 10:63]) == h


def test_config_generators_match_the_device_recipes():
    from paper_1112_5717_b200 import workloads as WL
    assert np.array_equal(CF.c2_row_shuffle(4096, 4), WL.c2_row_shuffle(4096, 4))
    r1, l1, s1 = CF.c4_recipe(64, 4)
    r2, l2, s2 = WL.c4_recipe(64, 4)
    assert r1 == r2 and l1 == l2 and s1 == s2


def test_exact_float_gemm_limb_split():
    """p >= 2^26 goes through the 16-bit limb split of the blocked GEMM."""
    rng = np.random.default_rng(9)
    for p in (67108859, 2**31 - 1):
        A = rng.integers(0, p, (40, 300), dtype=np.uint64).astype(np.uint32)
        Bm = rng.integers(0, p, (300, 30), dtype=np.uint64).astype(np.uint32)
        Cm = rng.integers(0, p, (40, 30), dtype=np.uint64).astype(np.uint32)
        want = (Cm.astype(object) - A.astype(object).dot(Bm.astype(object))) % p
        got = Cm.copy()
        B.mm_sub(got, A, Bm, p)
        assert np.array_equal(got.astype(object), want)
