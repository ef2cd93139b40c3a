"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors.  Bit-exact for every output: rank, row profile,
sigma, every entry of the packed [C\\U] body, and the reference's op counts."""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_1112_5717_b200 as G
from tests.helpers import c2_style, c4_batch, digest, load_npz_cases

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PRIMES = [2, 3, 7, 251, 257, 65521, 8388593, 2147483647]


def _digests():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


def _cup_recursive(a, p, ctr=None):
    """The device entry point always runs the recursive engine (the host entry
    routes small matrices to the single-CTA kernel)."""
    import torch
    m, n = a.shape
    if m * n == 0:
        return G.cup(a, p, ctr)
    d = torch.from_numpy(a.view(np.int32).copy()).cuda()
    r = G.cup_dev(d, m, n, p, ctr=ctr)
    a[...] = d.cpu().numpy().view(np.uint32)
    return r


def _check_cup(a, p, ctr_check=False):
    o_body = a.copy()
    o = O.port_cup(o_body, p)
    for fn in (G.cup, _cup_recursive):
        a_gpu = a.copy()
        ctr = G.OpCounter()
        g = fn(a_gpu, p, ctr)
        assert g.rank == o.rank, fn.__name__
        assert np.array_equal(g.row_profile, o.rrp), fn.__name__
        assert np.array_equal(g.col_perm, o.sigma), fn.__name__
        assert np.array_equal(a_gpu, o_body), f"{fn.__name__}: body mismatch at {np.argwhere(a_gpu != o_body)[:5]}"
    a_gpu, a_or = a_gpu, o_body
    if ctr_check and O.have_ref():
        r = O.ref_cup(a.copy(), p)
        assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == r.ops.tolist()
    return g


def test_golden_cup_cases():
    for c in load_npz_cases(os.path.join(GOLDEN, "cup_small.npz"),
                            ["p", "a", "body", "rank", "rrp", "sigma", "ops"]):
        for fn in (G.cup, _cup_recursive):
            a = c["a"].copy()
            ctr = G.OpCounter()
            r = fn(a, int(c["p"]), ctr)
            assert r.rank == int(c["rank"])
            assert np.array_equal(r.row_profile, c["rrp"])
            assert np.array_equal(r.col_perm, c["sigma"])
            assert np.array_equal(a, c["body"])
            assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == c["ops"].tolist()


def test_golden_mm_cases():
    for c in load_npz_cases(os.path.join(GOLDEN, "mm_small.npz"),
                            ["p", "a", "b", "c", "alpha", "beta", "out"]):
        out = c["c"].copy()
        G.mm(c["a"], c["b"], out, int(c["alpha"]), int(c["beta"]), int(c["p"]))
        assert np.array_equal(out, c["out"])


@pytest.mark.parametrize("p", PRIMES)
def test_mm_tensor_core_shapes(p):
    rng = np.random.default_rng(p % 1000)
    for (m, l, n) in [(128, 128, 128), (200, 300, 170), (129, 1000, 257), (64, 64, 64),
                      (33, 40, 35), (300, 16, 300)]:
        a = rng.integers(0, p, (m, l), dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, p, (l, n), dtype=np.uint64).astype(np.uint32)
        c = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        for alpha, beta in [(p - 1, 1), (1, 0), (3 % p, 2 % p)]:
            c1, c2 = c.copy(), c.copy()
            G.mm(a, b, c1, alpha, beta, p)
            O.port_mm(a, b, c2, alpha, beta, p)
            assert np.array_equal(c1, c2), (m, l, n, alpha, beta)


def test_mm_long_k_chunks():
    # K beyond the exact s32 accumulation bound is chunked (tc_kmax)
    p = 65521
    rng = np.random.default_rng(3)
    a = rng.integers(0, p, (130, 20000), dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, p, (20000, 70), dtype=np.uint64).astype(np.uint32)
    c = np.zeros((130, 70), np.uint32)
    G.mm(a, b, c, 1, 0, p)
    ref = np.zeros_like(c)
    O.port_mm(a, b, ref, 1, 0, p)
    assert np.array_equal(c, ref)


@pytest.mark.parametrize("p", PRIMES)
def test_cup_random_shapes(p):
    rng = np.random.default_rng(1000 + p % 97)
    for (m, n) in [(1, 1), (3, 5), (64, 64), (65, 129), (127, 300), (300, 127), (128, 128),
                   (257, 513), (513, 200)]:
        _check_cup(rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32), p,
                   ctr_check=(m * n < 40000))


@pytest.mark.parametrize("p", [2, 3, 65521, 8388593])
def test_cup_rank_deficient(p):
    rng = np.random.default_rng(5)
    for (m, n, r) in [(300, 200, 50), (200, 300, 120), (513, 257, 200), (100, 700, 60),
                      (640, 640, 333)]:
        seed = int(rng.integers(0, 2**62))
        if O.have_ref():
            a = O.ref_random_rank_matrix(m, n, r, seed, p, generic=bool(seed & 1))
        else:
            L = rng.integers(0, p, (m, r), dtype=np.uint64).astype(np.uint32)
            R = rng.integers(0, p, (r, n), dtype=np.uint64).astype(np.uint32)
            from tests.helpers import matmul_mod
            a = matmul_mod(L, R, p)
        g = _check_cup(a, p)
        assert g.rank <= r


def test_cup_structured_window_misses():
    """Pivots beyond the leading window (zero leading columns, zero rows,
    GF(2)/GF(3) dense rank deficiency) -> the exact fallback path."""
    rng = np.random.default_rng(11)
    p = 65521
    a = rng.integers(0, p, (300, 400), dtype=np.uint64).astype(np.uint32)
    a[:, :200] = 0
    _check_cup(a, p)
    a = rng.integers(0, p, (300, 400), dtype=np.uint64).astype(np.uint32)
    a[::3, :] = 0
    _check_cup(a, p)
    a = rng.integers(0, p, (256, 1024), dtype=np.uint64).astype(np.uint32)
    a[:, 100:900] = 0
    a[:, :100] = a[:, :100] * (np.arange(256)[:, None] % 2).astype(np.uint32)
    _check_cup(a, p)
    for q in (2, 3):
        L = rng.integers(0, q, (700, 90), dtype=np.uint64).astype(np.uint32)
        R = rng.integers(0, q, (90, 1100), dtype=np.uint64).astype(np.uint32)
        from tests.helpers import matmul_mod
        _check_cup(matmul_mod(L, R, q), q)


def test_cup_tall_early_return():
    # r1 == n early return (factor.cpp:47): rows below keep G (C data)
    rng = np.random.default_rng(12)
    for p in (65521, 7):
        _check_cup(rng.integers(0, p, (700, 90), dtype=np.uint64).astype(np.uint32), p)
        _check_cup(rng.integers(0, p, (1000, 300), dtype=np.uint64).astype(np.uint32), p)


def test_c1_matches_reference_digest():
    d = _digests()["c1"]
    a = O.port_random_matrix(1024, 1024, 1, 65521)
    ctr = G.OpCounter()
    r = G.cup(a, 65521, ctr)
    assert r.rank == d["rank"]
    assert np.array_equal(r.row_profile, np.arange(r.rank))
    assert digest(r.col_perm) == d["sigma"] and digest(a) == d["body"]
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == d["ops"]


def test_c2_style_matches_reference_digest():
    d = _digests()["c2s"]
    a = c2_style(1024, 2048, 512, 2, 65521)
    ctr = G.OpCounter()
    r = G.cup(a, 65521, ctr)
    assert r.rank == d["rank"] and r.row_profile.tolist() == d["rrp"]
    assert digest(r.col_perm) == d["sigma"] and digest(a) == d["body"]
    assert [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest] == d["ops"]


def test_c4_batched_matches_reference_digests():
    import torch
    d = _digests()["c4"]
    mats, ranks = c4_batch(16)
    dev = torch.from_numpy(mats.view(np.int32).copy()).cuda()
    rk, rrp, sig = G.cup_batched_dev(dev, 16, 256, 256, d["p"])
    body = dev.cpu().numpy().view(np.uint32)
    for t in range(16):
        e = d["mats"][t]
        assert rk[t] == e["rank"] == ranks[t]
        assert digest(rrp[t, :rk[t]]) == e["rrp"]
        assert digest(sig[t]) == e["sigma"]
        assert digest(body[t]) == e["body"]


def test_batched_small_primes_vs_oracle():
    import torch
    rng = np.random.default_rng(21)
    for p in (2, 3, 65521, 2147483647):
        mats = rng.integers(0, p, (6, 70, 90), dtype=np.uint64).astype(np.uint32)
        mats[1, :, :40] = 0
        mats[2, ::2, :] = 0
        dev = torch.from_numpy(mats.view(np.int32).copy()).cuda()
        rk, rrp, sig = G.cup_batched_dev(dev, 6, 70, 90, p)
        body = dev.cpu().numpy().view(np.uint32)
        for t in range(6):
            a = mats[t].copy()
            o = O.port_cup(a, p)
            assert rk[t] == o.rank and np.array_equal(rrp[t, :o.rank], o.rrp)
            assert np.array_equal(sig[t], o.sigma) and np.array_equal(body[t], a)


def test_batched_wide_first_panel_few_pivots():
    """256-column matrices whose leading 32-row panels hold few pivots (zero and
    repeated rows): the trailing update then spans more than 224 columns right of
    the panel's pivot block."""
    import torch
    rng = np.random.default_rng(77)
    for p, batch in ((8388593, 66), (65521, 5)):
        mats = rng.integers(0, p, (batch, 96, 256), dtype=np.uint64).astype(np.uint32)
        mats[0, :16, :] = 0                 # 16 pivots in panel 0: 240 columns right of them
        mats[1, 1:32, :] = 0                # a single pivot: 255 columns
        mats[2, 4:32, :] = mats[2, 0, :]    # copies of row 0 eliminate to zero rows
        mats[3, :40:2, :] = 0
        mats[4, 8:30, :] = 0
        dev = torch.from_numpy(mats.view(np.int32).copy()).cuda()
        rk, rrp, sig = G.cup_batched_dev(dev, batch, 96, 256, p)
        body = dev.cpu().numpy().view(np.uint32)
        for t in range(min(batch, 8)):
            a = mats[t].copy()
            o = O.port_cup(a, p)
            assert rk[t] == o.rank and np.array_equal(rrp[t, :o.rank], o.rrp), (p, t)
            assert np.array_equal(sig[t], o.sigma), (p, t)
            assert np.array_equal(body[t], a), (p, t, np.argwhere(body[t] != a)[:5])


def test_batched_shape_and_prime_sweep_vs_oracle():
    """The blocked batched kernel over ragged shapes (partial last panels, more
    rows than columns, m > 256), primes on both sides of 2^24 and inputs that
    force transpositions inside a row sub-block, zero rows and repeated rows."""
    import torch
    rng = np.random.default_rng(2027)
    shapes = [(33, 256), (64, 37), (130, 200), (256, 255), (300, 64), (100, 256), (31, 8), (257, 129)]
    for p in (2, 3, 251, 65521, 8388593, 16777259, 2147483647):
        for (m, n) in shapes:
            batch = 4
            mats = rng.integers(0, p, (batch, m, n), dtype=np.uint64).astype(np.uint32)
            mats[1, :, : n // 3] = 0                       # pivots start far right of column 0
            mats[2, ::3, :] = 0                            # zero rows inside every sub-block
            mats[2, 1::6, :] = mats[2, 4 % m, :]           # repeated rows
            if n > 8:                                      # low rank: product of thin factors
                k = max(1, min(m, n) // 4)
                lf = rng.integers(0, p, (m, k), dtype=np.uint64)
                rf = rng.integers(0, p, (k, n), dtype=np.uint64)
                acc = np.zeros((m, n), dtype=np.uint64)
                for j in range(k):                         # (products < 2^62: reduce per term)
                    acc = (acc + (lf[:, j:j + 1] * rf[j:j + 1, :]) % p) % p
                mats[3] = acc.astype(np.uint32)
            dev = torch.from_numpy(mats.view(np.int32).copy()).cuda()
            rk, rrp, sig = G.cup_batched_dev(dev, batch, m, n, p)
            body = dev.cpu().numpy().view(np.uint32)
            for t in range(batch):
                a = mats[t].copy()
                o = O.port_cup(a, p)
                assert rk[t] == o.rank and np.array_equal(rrp[t, :o.rank], o.rrp), (p, m, n, t)
                assert np.array_equal(sig[t], o.sigma), (p, m, n, t)
                assert np.array_equal(body[t], a), (p, m, n, t, np.argwhere(body[t] != a)[:5])


def test_large_properties_dev():
    """At full-size-class dimensions: structural outputs + Freivalds A = C*U*P."""
    import torch
    n, p = 4096, 65521
    src = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(src, n, n, 3, p)
    orig = src.cpu().numpy().view(np.uint32).copy()
    work = src.clone()
    r = G.cup_dev(work, n, n, p)
    body = work.cpu().numpy().view(np.uint32)
    assert r.rank == n and np.array_equal(r.row_profile, np.arange(n))
    assert O.freivalds_cup(orig, body, r.rank, r.col_perm, p, trials=2)
    # determinism: a second run is bit-identical
    work2 = src.clone()
    G.cup_dev(work2, n, n, p)
    assert torch.equal(work, work2)


def test_generator_matches_reference():
    import torch
    for (m, n, seed, p) in [(37, 53, 5, 65521), (64, 128, 2**64 - 3, 8388593)]:
        d = torch.empty((m, n), dtype=torch.int32, device="cuda")
        G.random_matrix_dev(d, m, n, seed, p)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), O.port_random_matrix(m, n, seed, p))


def test_rank_profile_and_determinant():
    rng = np.random.default_rng(31)
    for p in (7, 65521):
        a = rng.integers(0, p, (50, 50), dtype=np.uint64).astype(np.uint32)
        r, rrp = G.rank_and_profile(a.copy(), p)
        o = O.port_cup(a.copy(), p)
        assert r == o.rank and np.array_equal(rrp, o.rrp)
        if O.have_ref():
            assert G.determinant(a.copy(), p) == O.ref_determinant(a.copy(), p)
    # GF(7) worked example with a column swap: det = sign(P) * prod pivots
    a = np.array([[0, 1], [1, 0]], np.uint32)
    assert G.determinant(a.copy(), 7) == 6


def test_large_cup_freivalds_on_device():
    # a config-5-style instance at 32768^2 (4.3 GB): indexing beyond 2^31
    # elements, the full recursion depth; reconstruction checked on the device
    import torch
    from tests.helpers import freivalds_dev
    n, p = 32768, 65521
    orig = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(orig, n, n, 5, p)
    body = orig.clone()
    r = G.cup_dev(body, n, n, p)
    assert r.rank == n
    assert freivalds_dev(orig, body, r.rank, r.col_perm, p, trials=2)
    # a corrupted body must fail the same check
    body[n // 2, n // 2 + 7] = (int(body[n // 2, n // 2 + 7]) + 1) % p
    assert not freivalds_dev(orig, body, r.rank, r.col_perm, p, trials=1)
    del orig, body
    torch.cuda.empty_cache()


@pytest.mark.parametrize("p", [3, 8388593, 2147483647])
def test_cup_mid_sizes_all_paths(p):
    # >= 1024 rows: node inverses + their tensor-core GEMMs, split Schur updates,
    # side streams; non-16-bit primes take the 64-bit reduction paths
    rng = np.random.default_rng(77 + p % 1000)
    a = rng.integers(0, p, (1100, 1300), dtype=np.uint64).astype(np.uint32)
    _check_cup(a, p)
    # rank deficient with a shuffled profile at the same scale
    L = rng.integers(0, p, (1030, 700), dtype=np.uint64).astype(np.uint32)
    R = rng.integers(0, p, (700, 1200), dtype=np.uint64).astype(np.uint32)
    from tests.helpers import matmul_mod
    b = matmul_mod(L, R, p)
    b[1::4, :] = 0
    _check_cup(np.ascontiguousarray(b[rng.permutation(1030)]), p)


def test_cup_strided_view_large():
    # a window of a larger allocation (lda > n) through the device entry point
    import torch
    p, m, n, ld = 65521, 1200, 1100, 1536
    full = torch.empty((m, ld), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(full, m, ld, 9, p)
    orig = full[:, :n].cpu().numpy().view(np.uint32).copy()
    untouched = full[:, n:].clone()
    r = G.cup_dev(full, m, n, p, lda=ld)
    o_body = orig.copy()
    o = O.port_cup(o_body, p)
    assert r.rank == o.rank and np.array_equal(r.col_perm, o.sigma)
    assert np.array_equal(full[:, :n].cpu().numpy().view(np.uint32), o_body)
    assert torch.equal(full[:, n:], untouched)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,p,rank", [(2048, 3000, 65521, None), (3000, 2048, 65521, 1500), (520, 8100, 65521, None),
                                        (4096, 1100, 8388593, None)])
def test_host_path_split_copy_equals_device_path(m, n, p, rank):
    """rl_cup_u32 overlaps the H2D copy of the rows below the root split with the
    top half's factorization (external event wait inside the captured graph):
    same bytes as the device-resident path, twice (graph replay)."""
    import torch
    a = O.port_random_matrix(m, n, 41, p) if rank is None else O.ref_random_rank_matrix(m, n, rank, 42, p)
    d = torch.from_numpy(a.view(np.int32).copy()).cuda()
    g_dev = G.cup_dev(d, m, n, p)
    ref = d.cpu().numpy().view(np.uint32)
    for _ in range(2):
        h = a.copy()
        g = G.cup(h, p)
        assert g.rank == g_dev.rank
        assert np.array_equal(g.row_profile, g_dev.row_profile)
        assert np.array_equal(g.col_perm, g_dev.col_perm)
        assert np.array_equal(h, ref)


@pytest.mark.gpu
def test_batched_host_pipeline_equals_device_path():
    """rl_cup_batched_u32 (host matrices, chunked copy/factor/copy pipeline) gives
    the device path's bytes and metadata, for a batch that is not a multiple of
    the chunk count."""
    import torch
    mats, _ = c4_batch(19)
    a = np.ascontiguousarray(np.stack(mats)).astype(np.uint32)
    d = torch.from_numpy(a.view(np.int32).copy()).cuda()
    rk_d, rrp_d, sg_d = G.cup_batched_dev(d, a.shape[0], 256, 256, 8388593)
    h = a.copy()
    rk, rrp, sg = G.cup_batched(h, 8388593)
    assert np.array_equal(rk, rk_d) and np.array_equal(rrp, rrp_d) and np.array_equal(sg, sg_d)
    assert np.array_equal(h, d.cpu().numpy().view(np.uint32))


def test_cup_row_split_lanes_vs_oracle():
    # 8192 rows: the root's bottom half (4096 rows, k = 4096 > the column-split
    # bound) takes the row split -- its lower 2048 rows get their TRSM + Schur
    # update on a side lane, joined when node(4096, 4096) first touches them.
    # Rank-deficient with a thinned top half (r1 < w, so the root's Schur update
    # is non-empty) and a shuffled profile, so the lane's extents are dynamic.
    from tests.helpers import matmul_mod
    p = 65521
    rng = np.random.default_rng(5)
    L = rng.integers(0, p, (8192, 900), dtype=np.uint64).astype(np.uint32)
    R = rng.integers(0, p, (900, 1000), dtype=np.uint64).astype(np.uint32)
    b = matmul_mod(L, R, p)
    top = b[:4096]
    top[rng.random(4096) < 0.9] = 0
    b[4096:][2::3] = 0
    b[:4096] = top[rng.permutation(4096)]
    g = _check_cup(np.ascontiguousarray(b), p)
    assert 0 < int(np.searchsorted(g.row_profile, 4096)) < g.rank
