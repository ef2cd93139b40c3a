"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/ranklab_gpu.h declares, validates arguments like the reference
(errors.hpp), computes the reference's exact op counts on the host, and fails
loudly (no CPU fallback) when asked to compute without a GPU."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1112_5717_b200 as G
from tests.helpers import load_npz_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_header_symbols_are_exported():
    hdr = open(os.path.join(ROOT, "include", "ranklab_gpu.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(rl_\w+)\s*\(", hdr, re.M))
    assert declared == set(G.EXPORTS)
    lib = G.lib()
    for name in declared:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    so = open(G.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


def test_field_validation_matches_reference():
    a = np.ones((2, 2), np.uint32)
    with pytest.raises(G.NotPrime):
        G.cup(a, 4)
    with pytest.raises(G.NotPrime):
        G.cup(a, 1)
    with pytest.raises(G.NotPrime):
        G.cup(a, 2**31 + 11)


def test_empty_shapes_need_no_device():
    # factor.cpp:32 / test_factor.cpp:245-256: rank 0, identity of order n
    a = np.zeros((0, 4), np.uint32)
    r = G.cup(a, 3)
    assert r.rank == 0 and list(r.col_perm) == [0, 1, 2, 3]
    b = np.zeros((4, 0), np.uint32)
    r = G.cup(b, 3)
    assert r.rank == 0 and len(r.col_perm) == 0
    # ple's degenerate return (factor.cpp:110): identity row_perm of order m
    pp = G.ple(b, 3)
    assert pp.rank == 0 and list(pp.row_perm) == [0, 1, 2, 3]
    pp = G.ple(a, 3)
    assert pp.rank == 0 and len(pp.row_perm) == 0


def test_mm_overlap_rejected():
    # kernels.cpp:38-39: C must not overlap A or B
    buf = np.zeros((4, 4), np.uint32)
    with pytest.raises(G.OverlapError):
        G.mm(buf[0:2, 0:2], buf[0:2, 1:3], buf[0:2, 1:3], 1, 0, 5)


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    a = np.ones((3, 3), np.uint32)
    with pytest.raises(G.CudaError):
        G.cup(a, 7)
    with pytest.raises(G.CudaError):
        G.mm(a, a, a.copy(), 1, 0, 7)
    with pytest.raises(G.CudaError):
        G.ple(a, 7)


def test_opcount_matches_reference_goldens():
    # OpCounter of cup is a function of (shape, rrp, ipiv)
    n = 0
    for c in load_npz_cases(os.path.join(ROOT, "tests", "golden", "cup_small.npz"),
                            ["p", "a", "rank", "rrp", "ops"]):
        a = c["a"].copy()
        m, nn = a.shape
        r = O.port_cup(a, int(c["p"]))
        ops = np.zeros(4, np.uint64)
        rrp = np.ascontiguousarray(r.rrp, np.uint32)
        ipiv = np.ascontiguousarray(r.ipiv, np.uint32)
        G._check(G.lib().rl_cup_opcount(m, nn, r.rank, G._ptr(rrp), G._ptr(ipiv), G._ptr(ops)))
        assert ops.tolist() == c["ops"].tolist(), (m, nn, int(c["p"]))
        n += 1
    assert n >= 300


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_trsm_opcount_matches_reference():
    # kernels.cpp:135-154 at several thresholds: charges are a function of shape
    import itertools
    rng = np.random.default_rng(1)
    for side, uplo, diag in itertools.product(["left", "right"], ["upper", "lower"],
                                              ["unit", "nonunit"]):
        for (m, n), thr in itertools.product([(1, 1), (3, 5), (7, 2), (16, 9), (33, 40)],
                                             [1, 2, 5, 64]):
            k = m if side == "left" else n
            t = rng.integers(1, 65521, (k, k), dtype=np.uint32)
            b = rng.integers(0, 65521, (m, n), dtype=np.uint32)
            _, ops = O.ref_trsm(side, uplo, diag, t, b, 65521, thr, return_ops=True)
            mine = G.trsm_opcount(int(side == "right"), int(uplo == "lower"),
                                  int(diag == "unit"), m, n, thr)
            assert list(ops) == list(mine), (side, uplo, diag, m, n, thr)


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_echelon_opcount_matches_reference():
    # echelon.cpp:5-47 charges = cup's (skeleton walk) + trsm/neg/trtri/trulm tallies
    for m, n in [(1, 1), (5, 5), (9, 7), (7, 9), (32, 32), (40, 25), (25, 40), (70, 70)]:
        for rk in sorted({0, 1, 3, min(m, n)}):
            p = 7 if rk < min(m, n) else 65521
            a = (O.ref_random_rank_matrix(m, n, rk, 5, p) if rk < min(m, n)
                 else O.port_random_matrix(m, n, 3, p))
            pc = O.port_cup(a.copy(), p)
            for reduced in (False, True):
                _, ops = O.ref_col_ech_trans(a.copy(), p, reduced, return_ops=True)
                cup_ops = np.zeros(4, np.uint64)
                rrp = np.ascontiguousarray(pc.rrp, np.uint32)
                ipiv = np.ascontiguousarray(pc.ipiv, np.uint32)
                G.lib().rl_cup_opcount(m, n, pc.rank, G._ptr(rrp), G._ptr(ipiv), G._ptr(cup_ops))
                mine = cup_ops + G.echelon_opcount(m, n, pc.rank, reduced)
                assert list(ops) == list(mine), (m, n, rk, reduced)


def test_trsm_errors_need_no_device():
    t = np.array([[1, 2, 3], [0, 0, 4], [0, 0, 5]], np.uint32)
    b = np.arange(6, dtype=np.uint32).reshape(2, 3)
    keep = b.copy()
    # the reference reports the index local to the base block its halving
    # recursion stops in (kernels.cpp:87-90; pinned against the reference in
    # oracle/shim_check.cpp): threshold 1 -> block [1] -> index 0, threshold 3 ->
    # one block [0, 3) -> index 1 (ascending traversal for Right/Upper)
    with pytest.raises(G.SingularMatrix, match="at 0"):
        G.trsm(G.Side.Right, G.UpLo.Upper, G.Diag.NonUnit, t, b, 7)
    with pytest.raises(G.SingularMatrix, match="at 1"):
        G.trsm(G.Side.Right, G.UpLo.Upper, G.Diag.NonUnit, t, b, 7, threshold=3)
    assert np.array_equal(b, keep)
    big = np.ones((4, 4), np.uint32)
    with pytest.raises(G.OverlapError):
        G.trsm(G.Side.Left, G.UpLo.Upper, G.Diag.Unit, big[:2, :2], big[1:3, :], 7)
    with pytest.raises(G.DimensionMismatch):
        G.trsm(G.Side.Left, G.UpLo.Upper, G.Diag.Unit, np.ones((3, 3), np.uint32),
               np.ones((2, 2), np.uint32), 7)
    # empty reductions return cup's degenerate answer without a device
    r = G.col_ech_trans(np.zeros((0, 3), np.uint32), 5)
    assert r.rank == 0 and list(r.col_perm) == [0, 1, 2]
    G.invert_in_place(np.zeros((0, 0), np.uint32), 5)


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU behaviour")
def test_reductions_fail_loudly_without_gpu():
    with pytest.raises(G.CudaError):
        G.col_ech_trans(np.eye(4, dtype=np.uint32), 7)
    with pytest.raises(G.CudaError):
        G.invert_in_place(np.eye(4, dtype=np.uint32), 7)
    with pytest.raises(G.CudaError):
        G.trsm(G.Side.Left, G.UpLo.Upper, G.Diag.Unit, np.eye(2, dtype=np.uint32),
               np.ones((2, 2), np.uint32), 7)
