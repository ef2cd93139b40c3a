"""GPU parity of ple (factor.cpp:87-156) through the C ABI against the
reference compiled from its own sources: body, rank, col_profile, row_perm and
op counts bit-exact.  The GPU computes ple as cup(A^T)^T (the identity itself
is pinned on the CPU in test_ple_mirror.py)."""
import itertools

import numpy as np
import pytest

import oracle as O
import paper_1112_5717_b200 as G
from tests.helpers import c2_style

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def _mat(m, n, r, seed, p):
    if r >= min(m, n):
        return O.port_random_matrix(m, n, seed, p)
    return O.ref_random_rank_matrix(m, n, r, seed, p, generic=(seed % 2 == 0))


def _check(a, p):
    ref = a.copy()
    r, prof, perm, ops = O.ref_ple(ref, p)
    mine = a.copy()
    ctr = G.OpCounter()
    pp = G.ple(mine, p, ctr)
    assert pp.rank == r
    assert np.array_equal(pp.col_profile, prof)
    assert np.array_equal(pp.row_perm, perm)
    assert np.array_equal(mine, ref), f"body differs {a.shape} p={p}"
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == [int(x) for x in ops]


@needs_ref
@pytest.mark.parametrize("m,n", [(1, 1), (1, 7), (7, 1), (9, 4), (4, 9), (64, 64), (65, 130),
                                 (130, 65), (257, 300), (300, 257)])
def test_ple_shapes(m, n):
    for p, seed in itertools.product([3, 65521], [1, 2]):
        for r in sorted({0, 1, min(m, n) // 3, min(m, n)}):
            _check(_mat(m, n, r, seed + r, p), p)


@needs_ref
@pytest.mark.parametrize("p", [2, 251, 8388593, 2147483647])
def test_ple_primes(p):
    _check(O.port_random_matrix(120, 90, 4, p), p)
    _check(O.port_random_matrix(90, 120, 5, p), p)


@needs_ref
def test_ple_structured_and_strided():
    a = c2_style(200, 160, 60, 3, 65521)
    _check(np.ascontiguousarray(a.T), 65521)
    # strided view (stride = parent cols, matrix.hpp:46)
    big = O.port_random_matrix(100, 150, 8, 7)
    view = big[:, 20:120]
    ref = np.ascontiguousarray(view)
    r, prof, perm, _ = O.ref_ple(ref, 7)
    keep = big.copy()
    pp = G.ple(view, 7)
    assert pp.rank == r and np.array_equal(pp.row_perm, perm)
    assert np.array_equal(big[:, 20:120], ref)
    assert np.array_equal(big[:, :20], keep[:, :20]) and np.array_equal(big[:, 120:], keep[:, 120:])


@needs_ref
def test_ple_device_entry_large():
    import torch
    p, m, n = 65521, 1500, 1100
    a = O.port_random_matrix(m, n, 12, p)
    ref = a.copy()
    r, prof, perm, ops = O.ref_ple(ref, p)
    d = torch.from_numpy(a.view(np.int32).copy()).cuda()
    ctr = G.OpCounter()
    pp = G.ple_dev(d, m, n, p, ctr=ctr)
    assert pp.rank == r and np.array_equal(pp.col_profile, prof) and np.array_equal(pp.row_perm, perm)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), ref)
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == [int(x) for x in ops]
