"""GPU parity of the reductions after cup -- col_ech_trans, red_col_ech_trans
(echelon.cpp:5-47), invert_in_place (solvers.cpp:24-31) -- and of the trsm
seam (kernels.cpp:135-154), through the C ABI, against the reference compiled
from its own sources (oracle/_ref).  Bit-exact bodies, metadata and op counts."""
import itertools

import numpy as np
import pytest

import oracle as O
import paper_1112_5717_b200 as G
from tests.helpers import c2_style, matmul_mod

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def _rank_matrix(m, n, r, seed, p):
    if r >= min(m, n):
        return O.port_random_matrix(m, n, seed, p)
    return O.ref_random_rank_matrix(m, n, r, seed, p, generic=False)


def _check_echelon(a, p, reduced):
    ref_body = a.copy()
    ref, ref_ops = O.ref_col_ech_trans(ref_body, p, reduced, return_ops=True)
    body = a.copy()
    ctr = G.OpCounter()
    fn = G.red_col_ech_trans if reduced else G.col_ech_trans
    t = fn(body, p, ctr)
    assert t.rank == ref.rank
    assert np.array_equal(t.row_profile, ref.rrp)
    assert np.array_equal(t.col_perm, ref.sigma)
    assert np.array_equal(body, ref_body), f"body differs ({a.shape}, p={p}, reduced={reduced})"
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == [int(x) for x in ref_ops]


@needs_ref
@pytest.mark.parametrize("reduced", [False, True])
@pytest.mark.parametrize("m,n,r", [(1, 1, 1), (3, 5, 2), (8, 8, 8), (9, 4, 4), (4, 9, 4),
                                   (40, 25, 25), (25, 40, 25), (64, 64, 30), (65, 65, 65),
                                   (130, 100, 100), (100, 130, 57), (200, 200, 200),
                                   (300, 257, 190), (257, 300, 257), (513, 513, 513)])
def test_echelon_shapes(m, n, r, reduced):
    for p in (7, 65521):
        _check_echelon(_rank_matrix(m, n, r, 11 + m + n, p), p, reduced)


@needs_ref
@pytest.mark.parametrize("p", [2, 3, 251, 257, 8388593, 2147483647])
def test_echelon_primes(p):
    for reduced in (False, True):
        _check_echelon(O.port_random_matrix(150, 170, 5, p), p, reduced)
        _check_echelon(O.port_random_matrix(170, 150, 6, p), p, reduced)


@needs_ref
def test_echelon_rank_profile_shifts():
    # C2-style: zero rows and a shuffled row profile (U-row shifts, pivot-row
    # compression over columns [0, j])
    a = c2_style(240, 300, 90, 7, 65521)
    for reduced in (False, True):
        _check_echelon(a, 65521, reduced)


@needs_ref
def test_echelon_device_entry():
    import torch
    p = 65521
    a = O.port_random_matrix(300, 280, 9, p)
    ref_body = a.copy()
    ref = O.ref_col_ech_trans(ref_body, p, True)
    d = torch.from_numpy(a.view(np.int32).copy()).cuda()
    t = G.col_ech_trans_dev(d, 300, 280, p, reduced=True)
    assert t.rank == ref.rank and np.array_equal(t.col_perm, ref.sigma)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), ref_body)


def test_inverse_known_answer():
    # test_solvers.cpp:130-134: GF(7) [[2,1],[0,3]]^{-1} = [[4,1],[0,5]]
    a = np.array([[2, 1], [0, 3]], np.uint32)
    G.invert_in_place(a, 7)
    assert a.tolist() == [[4, 1], [0, 5]]


@needs_ref
@pytest.mark.parametrize("n,p", [(1, 7), (2, 2), (5, 3), (64, 65521), (65, 7), (129, 251),
                                 (300, 65521), (400, 8388593), (257, 2147483647)])
def test_invert_matches_reference(n, p):
    a = O.port_random_matrix(n, n, 21 + n, p)
    ref = a.copy()
    st, ref_ops = O.ref_invert(ref, p, return_ops=True)
    mine = a.copy()
    ctr = G.OpCounter()
    if st == 0:
        G.invert_in_place(mine, p, ctr)
        assert np.array_equal(mine, ref)
        eye = matmul_mod(a, mine, p)
        assert np.array_equal(eye, np.eye(n, dtype=np.uint32))
    else:
        with pytest.raises(G.SingularMatrix):
            G.invert_in_place(mine, p, ctr)
        assert np.array_equal(mine, ref)
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == [int(x) for x in ref_ops]


@needs_ref
def test_invert_singular_leaves_reduced_body():
    p = 65521
    a = _rank_matrix(120, 120, 77, 3, p)
    ref = a.copy()
    st, ref_ops = O.ref_invert(ref, p, return_ops=True)
    assert st == 3
    mine = a.copy()
    ctr = G.OpCounter()
    with pytest.raises(G.SingularMatrix):
        G.invert_in_place(mine, p, ctr)
    assert np.array_equal(mine, ref)
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == [int(x) for x in ref_ops]


def test_invert_large_round_trip():
    import torch
    p, n = 65521, 2048
    d = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(d, n, n, 17, p)
    a = d.clone()
    G.invert_dev(d, n, p)
    eye = torch.zeros((n, n), dtype=torch.int32, device="cuda")
    G.mm_dev(a, d, eye, n, n, n, 1, 0, p)
    assert torch.equal(eye.cpu(), torch.eye(n, dtype=torch.int32))


def test_trsm_known_answer():
    # test_kernels.cpp:90-94: GF(7) Right/Upper/Unit [[1,2],[0,1]], B=[[3,4]] -> [[3,5]]
    t = np.array([[1, 2], [0, 1]], np.uint32)
    b = np.array([[3, 4]], np.uint32)
    G.trsm(G.Side.Right, G.UpLo.Upper, G.Diag.Unit, t, b, 7)
    assert b.tolist() == [[3, 5]]


@needs_ref
@pytest.mark.parametrize("side,uplo,diag", list(itertools.product(
    ["left", "right"], ["upper", "lower"], ["unit", "nonunit"])))
def test_trsm_variants(side, uplo, diag):
    rng = np.random.default_rng(5)
    for (m, n), p, thr in itertools.product([(1, 1), (3, 7), (13, 13), (64, 50), (70, 129),
                                             (257, 90)], [7, 65521, 2147483647], [1, 8]):
        k = m if side == "left" else n
        t = rng.integers(1, p, (k, k), dtype=np.uint64).astype(np.uint32)
        if diag == "unit":
            t[np.arange(k), np.arange(k)] = 0  # Unit never reads the diagonal
        b = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        ref, ref_ops = O.ref_trsm(side, uplo, diag, t, b.copy(), p, thr, return_ops=True)
        mine = b.copy()
        ctr = G.OpCounter()
        G.trsm(int(side == "right"), int(uplo == "lower"), int(diag == "unit"), t, mine, p, ctr,
               threshold=thr)
        assert np.array_equal(mine, ref), (side, uplo, diag, m, n, p)
        assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == [int(x) for x in ref_ops]


def test_trsm_singular_diagonal_and_overlap():
    t = np.array([[1, 2, 3], [0, 0, 4], [0, 0, 5]], np.uint32)
    b = np.arange(6, dtype=np.uint32).reshape(2, 3)
    keep = b.copy()
    with pytest.raises(G.SingularMatrix):
        G.trsm(G.Side.Right, G.UpLo.Upper, G.Diag.NonUnit, t, b, 7)
    assert np.array_equal(b, keep)
    big = np.ones((4, 4), np.uint32)
    with pytest.raises(G.OverlapError):
        G.trsm(G.Side.Left, G.UpLo.Upper, G.Diag.Unit, big[:2, :2], big[1:3, :], 7)


def test_trsm_device_entry_large():
    import torch
    p, k, n = 65521, 1500, 700
    t = torch.empty((k, k), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(t, k, k, 31, p)
    b = torch.empty((k, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(b, k, n, 32, p)
    x = b.clone()
    G.trsm_dev(G.Side.Left, G.UpLo.Lower, G.Diag.Unit, t, x, k, n, p)
    # T_unit_lower * X == B
    tl = torch.tril(t, -1) + torch.eye(k, dtype=torch.int32, device="cuda")
    chk = torch.zeros_like(b)
    G.mm_dev(tl, x, chk, k, k, n, 1, 0, p)
    assert torch.equal(chk, b)
