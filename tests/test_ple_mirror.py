"""The identity the GPU ple is built on, pinned against the reference itself:
ranklab::ple(A) (factor.cpp:87-156) == transpose of ranklab::cup(A^T)
(factor.cpp:30-81) -- body, rank, col_profile = row_profile, row_perm =
col_perm^{-1}, and all four op-count buckets.  CPU only (oracle/_ref)."""
import itertools

import numpy as np
import pytest

import oracle as O

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def _mat(m, n, r, seed, p):
    if r >= min(m, n):
        return O.port_random_matrix(m, n, seed, p)
    return O.ref_random_rank_matrix(m, n, r, seed, p, generic=(seed % 2 == 0))


def _check_mirror(a, p):
    ple_body = a.copy()
    r1, prof, perm, ops1 = O.ref_ple(ple_body, p)
    cup_body = np.ascontiguousarray(a.T)
    res = O.ref_cup(cup_body, p)
    assert r1 == res.rank
    assert np.array_equal(prof, res.rrp)
    # A^T = E^T L^T P^T: cup's column permutation is P^T, so as index arrays
    # row_perm is the inverse of cup's sigma
    inv = np.empty_like(res.sigma)
    inv[res.sigma] = np.arange(len(res.sigma), dtype=np.uint32)
    assert np.array_equal(perm, inv)
    assert np.array_equal(ple_body, cup_body.T)
    assert [int(x) for x in ops1] == [int(x) for x in res.ops]


@needs_ref
@pytest.mark.parametrize("m,n", [(1, 1), (1, 6), (6, 1), (9, 4), (4, 9), (8, 8), (33, 17),
                                 (17, 33), (64, 64), (100, 70)])
def test_ple_is_transposed_cup(m, n):
    for p, seed in itertools.product([2, 3, 7, 65521], [1, 2]):
        for r in sorted({0, 1, min(m, n) // 2, min(m, n)}):
            _check_mirror(_mat(m, n, r, seed + 10 * r, p), p)


@needs_ref
def test_ple_mirror_structured():
    # zero columns, duplicated columns, zero rows: non-trivial row permutations
    rng = np.random.default_rng(3)
    for p in (3, 65521):
        a = rng.integers(0, p, (40, 30), dtype=np.uint64).astype(np.uint32)
        a[:, ::4] = 0
        a[:, 5] = a[:, 7]
        a[::3, :] = 0
        _check_mirror(a, p)


@needs_ref
def test_ple_known_answer_gf5():
    # the transpose of the cup golden GF(5) [[2,4],[1,2]] (test_factor.cpp:27-61)
    a = np.array([[2, 1], [4, 2]], np.uint32)
    r, prof, perm, _ = O.ref_ple(a, 5)
    assert r == 1 and prof.tolist() == [0] and perm.tolist() == [0, 1]
    assert a.tolist() == [[2, 1], [2, 0]]
