"""The drop-in boundary under the reference's threading and storage contract
(proj/README.md:164-168: no internal threads, disjoint views
may be processed concurrently; ranklab::Mat storage is a pageable std::vector,
matrix.hpp:176):

* concurrent host threads (cudaStreamPerThread contexts) and concurrent device
  streams give the same bytes as the oracle -- no shared workspace;
* pageable and pinned host buffers give the same bytes;
* the one-launch tiny-matrix path (<= 512 entries) is bit-exact, including the
  early return and dead rows;
* the batched host path with stride > m*n touches only the matrices' words.
"""
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _same(a, p, got_body, got):
    ob = a.copy()
    o = O.port_cup(ob, p)
    return (got.rank == o.rank and np.array_equal(got.row_profile, o.rrp)
            and np.array_equal(got.col_perm, o.sigma) and np.array_equal(got_body, ob))


def test_tiny_path_exhaustive_gf2_3x3_and_random_small():
    import paper_1112_5717_b200 as G
    for code in range(512):
        a = np.array([(code >> k) & 1 for k in range(9)], np.uint32).reshape(3, 3)
        b = a.copy()
        assert _same(a, 2, b, G.cup(b, 2)), code
    rng = np.random.default_rng(1)
    for t in range(300):
        m, n = int(rng.integers(1, 23)), int(rng.integers(1, 23))
        if m * n > 512:
            continue
        p = int(rng.choice([2, 3, 7, 65521, 8388593, 2**31 - 1]))
        a = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        if t % 3 == 0:
            a[:, : n // 2] = 0
        if t % 4 == 0:
            a[::2] = 0
        b = a.copy()
        assert _same(a, p, b, G.cup(b, p)), (m, n, p)


def test_tiny_path_strided_host_view():
    import paper_1112_5717_b200 as G
    rng = np.random.default_rng(2)
    big = rng.integers(0, 65521, (10, 40), dtype=np.uint64).astype(np.uint32)
    before = big.copy()
    view = big[:, 5:17]
    a = view.copy()
    g = G.cup(view, 65521)
    assert _same(a, 65521, np.ascontiguousarray(view), g)
    assert np.array_equal(big[:, :5], before[:, :5]) and np.array_equal(big[:, 17:], before[:, 17:])


def test_determinant_4x4_gf3_matches_cofactor():
    import paper_1112_5717_b200 as G
    rng = np.random.default_rng(3)
    for _ in range(2000):
        a = rng.integers(0, 3, (4, 4), dtype=np.uint64).astype(np.uint32)
        d = int(round(np.linalg.det(a.astype(np.float64)))) % 3
        assert G.determinant(a.copy(), 3) == d


@pytest.mark.parametrize("shape", [(700, 900), (2048, 2048)])
def test_pageable_and_pinned_host_buffers_agree(shape):
    import torch

    import paper_1112_5717_b200 as G
    m, n = shape
    rng = np.random.default_rng(m)
    a = rng.integers(0, 65521, (m, n), dtype=np.uint64).astype(np.uint32)
    a[::7] = 0
    pageable = a.copy()
    gp = G.cup(pageable, 65521)
    pinned_t = torch.empty((m, n), dtype=torch.int32).pin_memory()
    pinned = pinned_t.numpy().view(np.uint32)
    pinned[:] = a
    gq = G.cup(pinned, 65521)
    assert np.array_equal(pageable, pinned)
    assert gp.rank == gq.rank and np.array_equal(gp.col_perm, gq.col_perm)
    assert _same(a, 65521, pageable, gp)


def test_concurrent_host_threads():
    import paper_1112_5717_b200 as G
    rng = np.random.default_rng(4)
    jobs = []
    for t in range(8):
        m, n = [(300, 400), (3, 3), (1100, 700), (64, 256)][t % 4]
        p = [65521, 3, 2**31 - 1, 8388593][t % 4]
        a = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        if p == 3:
            a[:, 0] = 0
        jobs.append((a, p))
    out = [None] * len(jobs)
    errs = []

    def work(i):
        try:
            for _ in range(3):
                a, p = jobs[i]
                b = a.copy()
                g = G.cup(b, p)
                out[i] = (b, g)
                if not _same(a, p, b, g):
                    errs.append(i)
        except Exception as e:  # noqa: BLE001
            errs.append((i, repr(e)))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def test_concurrent_streams_same_shape_async():
    """Two same-shape factorizations enqueued fully asynchronously on two
    streams run on distinct engines (plans, scratch) and both stay exact."""
    import torch

    import paper_1112_5717_b200 as G
    n, p = 1536, 65521
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a1 = torch.empty((n, n), dtype=torch.int32, device="cuda")
    a2 = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(a1, n, n, 21, p)
    G.random_matrix_dev(a2, n, n, 22, p)
    h1 = a1.cpu().numpy().view(np.uint32).copy()
    h2 = a2.cpu().numpy().view(np.uint32).copy()
    torch.cuda.synchronize()
    for _ in range(2):
        w1, w2 = a1.clone(), a2.clone()
        torch.cuda.synchronize()
        G.cup_dev(w1, n, n, p, stream=s1, sync=False)
        G.cup_dev(w2, n, n, p, stream=s2, sync=False)
        torch.cuda.synchronize()
        for h, w in ((h1, w1), (h2, w2)):
            ob = h.copy()
            O.port_cup(ob, p)
            assert np.array_equal(w.cpu().numpy().view(np.uint32), ob)


def test_batched_host_stride_gap_untouched():
    import paper_1112_5717_b200 as G
    m = n = 40
    batch, stride, p = 5, 40 * 40 + 37, 8388593
    rng = np.random.default_rng(6)
    buf = rng.integers(0, p, (batch - 1) * stride + m * n, dtype=np.uint64).astype(np.uint32)
    orig = buf.copy()
    ranks = np.zeros(batch, np.int64)
    G._check(G.lib().rl_cup_batched_u32(G._ptr(buf), batch, m, n, stride, p, G._ptr(ranks), None, None))
    for t in range(batch):
        a = orig[t * stride:t * stride + m * n].reshape(m, n).copy()
        O.port_cup(a, p)
        assert np.array_equal(buf[t * stride:t * stride + m * n].reshape(m, n), a)
        if t < batch - 1:  # the gap between matrices is not the library's
            assert np.array_equal(buf[t * stride + m * n:(t + 1) * stride], orig[t * stride + m * n:(t + 1) * stride])
