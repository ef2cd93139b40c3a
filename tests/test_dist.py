"""Host logic of the multi-GPU single-matrix CUP (paper_1112_5717_b200/dist.py,
config 5's 1D block-cyclic column tiles), on CPU over gloo.

The per-rank compute here is the reference library (oracle/_ref) standing in
for the GPU (``OracleOps``: cup / trsm / mm on host copies); the tiling, the
per-owner broadcasts, the cross-rank column exchange for sigma, the U-row
shift and the early return are the product code under test.  Every result must
equal ``ranklab::cup`` of the whole matrix bit for bit (rank, row profile,
sigma, every body entry).  The same driver on the GPU is tests/test_gpu_dist.py.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from paper_1112_5717_b200 import dist as D

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


class OracleOps:
    """cup / trsm(Right, Upper, Unit) / mm through the unmodified reference on
    contiguous host copies of the torch CPU views (test infrastructure)."""

    def __init__(self, p):
        self.p = p

    @staticmethod
    def _np(t):
        return t.contiguous().numpy().view(np.uint32).copy()

    @staticmethod
    def _back(t, a):
        t.copy_(torch.from_numpy(a.view(np.int32)))

    def cup(self, t):
        a = self._np(t)
        res = O.ref_cup(a, self.p)
        self._back(t, a)
        return res.rank, res.rrp.astype(np.int64), res.sigma.astype(np.int64)

    def trsm_right_upper_unit(self, u, b):
        uu, bb = self._np(u), self._np(b)
        O.ref_trsm("right", "upper", "unit", uu, bb, self.p)
        self._back(b, bb)

    def trsm_left_lower_nonunit(self, t, b):
        tt, bb = self._np(t), self._np(b)
        O.ref_trsm("left", "lower", "nonunit", tt, bb, self.p)
        self._back(b, bb)

    def mm_sub(self, a, b, c, max_ctas=0):
        aa, bb, cc = self._np(a), self._np(b), self._np(c)
        O.ref_mm(aa, bb, cc, self.p - 1, 1, self.p)
        self._back(c, cc)


def _cases():
    """(name, matrix, p, tile, block) -- shapes/ranks/primes that exercise the
    early return, sigma exchanges across ranks and the U-row shift."""
    out = []
    rnd = np.random.default_rng(7)
    out.append(("full_square", O.ref_random_matrix(96, 96, 11, 65521), 65521, 8, 16))
    out.append(("full_wide", O.ref_random_matrix(40, 130, 12, 65521), 65521, 16, 16))
    out.append(("tall_early_return", O.ref_random_matrix(150, 37, 13, 65521), 65521, 8, 24))
    out.append(("rank_def_spread", O.ref_random_rank_matrix(90, 80, 30, 14, 65521), 65521, 8, 16))
    out.append(("rank_def_generic", O.ref_random_rank_matrix(64, 72, 40, 15, 65521, generic=True),
                65521, 4, 8))
    z = O.ref_random_matrix(70, 60, 16, 7)
    z[:, :17] = 0
    z[5::4, :] = 0
    out.append(("zero_cols_rows_gf7", z, 7, 8, 16))
    out.append(("gf2_small_tiles", rnd.integers(0, 2, (57, 63)).astype(np.uint32), 2, 3, 7))
    out.append(("gf3_block1", rnd.integers(0, 3, (20, 19)).astype(np.uint32), 3, 2, 1))
    out.append(("p31", O.ref_random_matrix(48, 50, 17, 2147483647), 2147483647, 8, 16))
    out.append(("one_col", O.ref_random_matrix(9, 1, 18, 11), 11, 4, 4))
    out.append(("zero", np.zeros((12, 10), np.uint32), 5, 4, 4))
    c2 = O.ref_random_matrix(60, 24, 19, 65521)
    c2 = np.ascontiguousarray(np.vstack([c2, c2])[np.random.default_rng(3).permutation(120)])
    out.append(("duplicated_rows", c2, 65521, 8, 16))
    return out


def _run_case(a, p, tile, block, world, rank, sb=None, window=None):
    tiles = D.ColumnTiles(a.shape[1], world, tile)
    full = torch.from_numpy(a.view(np.int32).copy())
    x = D.scatter_columns(full, tiles, rank)
    res = D.dist_cup(x, a.shape[0], a.shape[1], p, tiles, block=block,
                      superblock=sb or 3 * block, ops=OracleOps(p), window=window)
    body = D.gather_columns(x, a.shape[0], tiles).numpy().view(np.uint32)
    return res, body


def _check_case(name, a, p, res, body):
    ref_body = a.copy()
    ref = O.ref_cup(ref_body, p)
    assert res.rank == ref.rank, name
    assert np.array_equal(res.row_profile, ref.rrp), name
    assert np.array_equal(res.col_perm, ref.sigma), name
    assert np.array_equal(body, ref_body), name


def test_column_tiles_map():
    t = D.ColumnTiles(23, 3, 4)
    assert t.owner.tolist() == [0] * 4 + [1] * 4 + [2] * 4 + [0] * 4 + [1] * 4 + [2] * 3
    assert t.gpos[0].tolist() == [0, 1, 2, 3, 12, 13, 14, 15]
    assert sum(t.width(g) for g in range(3)) == 23
    for g in range(3):
        assert np.array_equal(t.gpos[g][t.local[t.gpos[g]]], t.gpos[g])
        for c in range(24):
            ls = t.lsuf(g, c)
            assert np.all(t.gpos[g][ls:] >= c) and np.all(t.gpos[g][:ls] < c)


@pytest.mark.parametrize("name,a,p,tile,block", _cases(), ids=[c[0] for c in _cases()])
def test_single_rank_equals_reference(name, a, p, tile, block):
    res, body = _run_case(a, p, tile, block, 1, 0)
    _check_case(name, a, p, res, body)


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    out = []
    try:
        for name, a, p, tile, block in _cases():
            res, body = _run_case(a, p, tile, block, world, rank)
            if rank == 0:
                _check_case(name, a, p, res, body)
                out.append(name)
        if rank == 0:
            q.put(out)
    except Exception as e:  # report to the parent instead of hanging it
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_gloo_multi_rank_equals_reference(world):
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
    assert got == [c[0] for c in _cases()], got
    for pr in procs:
        assert pr.exitcode == 0


@pytest.mark.parametrize("sb", [1, 2, 100])
def test_single_rank_superblock_sizes(sb):
    """Super-block = one row block (flat), two, and larger than the matrix."""
    for name, a, p, tile, block in _cases()[:6]:
        res, body = _run_case(a, p, tile, block, 1, 0, sb=sb * block)
        _check_case(name, a, p, res, body)


@pytest.mark.parametrize("window", [0, 1, 3, 8])
def test_single_rank_window_widths(window):
    """Window mode off (0), narrower than a block (pivots beyond it -> fallback)
    and wider: identical results."""
    for name, a, p, tile, block in _cases():
        res, body = _run_case(a, p, tile, block, 1, 0, window=window * block)
        _check_case(name, a, p, res, body)
