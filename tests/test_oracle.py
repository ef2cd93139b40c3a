"""CPU tests: the oracle (our C restatement) pinned against the reference's own
golden vectors and known-answer tests.  No GPU needed."""
import json
import os

import numpy as np
import pytest

import oracle as O
from tests.helpers import c2_style, c4_batch, digest, load_npz_cases

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix_pinned_stream():
    # test_reference.cpp:93-99
    s = O.splitmix64(0, 3)
    assert [int(x) for x in s] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_random_matrix_closed_form_matches_stream():
    # random_matrix draws row-major next() % p (reference.cpp:246-253)
    for p in (65521, 8388593, 7):
        a = O.port_random_matrix(7, 9, 2**64 - 5, p)
        s = O.splitmix64(2**64 - 5, 63)
        assert np.array_equal(a.ravel(), (s % np.uint64(p)).astype(np.uint32))


def test_cup_known_answers():
    # test_factor.cpp:27-61 / SPEC.md:317-320
    a = np.eye(3, dtype=np.uint32)
    r = O.port_cup(a, 7)
    assert r.rank == 3 and list(r.rrp) == [0, 1, 2] and list(r.sigma) == [0, 1, 2]
    assert np.array_equal(a, np.eye(3, dtype=np.uint32))
    z = np.zeros((3, 4), np.uint32)
    r = O.port_cup(z, 5)
    assert r.rank == 0 and list(r.sigma) == [0, 1, 2, 3] and not z.any()
    a = np.array([[2, 4], [1, 2]], np.uint32)
    r = O.port_cup(a, 5)
    assert r.rank == 1 and list(r.rrp) == [0] and list(r.sigma) == [0, 1]
    assert a.tolist() == [[2, 2], [1, 0]]
    # zero-branch shift (test_factor.cpp:155-167)
    a = np.array([[0, 1, 2, 3], [0, 2, 4, 6], [0, 1, 2, 3], [1, 1, 3, 4]], np.uint32)
    orig = a.copy()
    r = O.port_cup(a, 7)
    assert r.rank == 2 and list(r.rrp) == [0, 3]
    assert O.freivalds_cup(orig, a, r.rank, r.sigma, 7, trials=4)


def test_cup_prescribed_profile():
    # test_factor.cpp:63-97: GF(11) 7x5 with rrp [0, 3, 4]
    p = 11
    r0, r3, r4 = np.array([1, 2, 3, 4, 5]), np.array([0, 1, 7, 2, 6]), np.array([0, 0, 3, 1, 9])
    coeffs = [(1, 0, 0), (2, 0, 0), (6, 0, 0), (1, 1, 0), (3, 2, 1), (4, 5, 6), (7, 8, 9)]
    b = np.array([(k0 * r0 + k3 * r3 + k4 * r4) % p for k0, k3, k4 in coeffs], np.uint32)
    body = b.copy()
    r = O.port_cup(body, p)
    assert r.rank == 3 and list(r.rrp) == [0, 3, 4]
    assert O.freivalds_cup(b, body, r.rank, r.sigma, p, trials=4)


def test_port_matches_reference_goldens():
    n = 0
    for c in load_npz_cases(os.path.join(GOLDEN, "cup_small.npz"),
                            ["p", "a", "body", "rank", "rrp", "sigma"]):
        a = c["a"].copy()
        p = int(c["p"])
        r = O.port_cup(a, p)
        assert r.rank == int(c["rank"])
        assert np.array_equal(r.rrp, c["rrp"])
        assert np.array_equal(r.sigma, c["sigma"])
        assert np.array_equal(a, c["body"])
        n += 1
    assert n >= 300


def test_port_mm_matches_reference_goldens():
    for c in load_npz_cases(os.path.join(GOLDEN, "mm_small.npz"),
                            ["p", "a", "b", "c", "alpha", "beta", "out"]):
        out = c["c"].copy()
        O.port_mm(c["a"], c["b"], out, int(c["alpha"]), int(c["beta"]), int(c["p"]))
        assert np.array_equal(out, c["out"])


def test_exhaustive_gf2_3x3_reconstruction():
    # acceptance C1 / test_factor.cpp:99-117 (rank, profile and reconstruction)
    for bits in range(512):
        a = np.array([(bits >> k) & 1 for k in range(9)], np.uint32).reshape(3, 3)
        body = a.copy()
        r = O.port_cup(body, 2)
        # rank/profile by brute force: row i is in the profile iff it raises the rank
        rows = []
        basis = []
        for i in range(3):
            cand = basis + [a[i].tolist()]
            if _rank_gf2(cand) > len(basis):
                basis = cand
                rows.append(i)
        assert r.rank == len(rows) and list(r.rrp) == rows
        assert O.freivalds_cup(a, body, r.rank, r.sigma, 2, trials=3, seed=bits)


def _rank_gf2(rows):
    m = [int("".join(str(v) for v in row), 2) for row in rows]
    rank = 0
    for bit in reversed(range(3)):
        piv = next((x for x in m if x >> bit & 1), None)
        if piv is None:
            continue
        m = [x ^ piv if (x >> bit & 1) else x for x in m if x != piv]
        rank += 1
    return rank


def test_generators_reproduce_reference_inputs():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        d = json.load(f)
    assert digest(O.port_random_matrix(1024, 1024, 1, 65521)) == d["c1_input"]
    assert digest(c2_style(1024, 2048, 512, 2, 65521)) == d["c2s_input"]
    mats, ranks = c4_batch(4)
    for t in range(4):
        assert digest(mats[t]) == d["c4"]["mats"][t]["input"]
        assert ranks[t] == d["c4"]["mats"][t]["r_gen"]


@pytest.mark.slow
def test_port_c1_digest():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        d = json.load(f)["c1"]
    a = O.port_random_matrix(1024, 1024, 1, 65521)
    r = O.port_cup(a, 65521)
    assert r.rank == d["rank"] and digest(r.sigma) == d["sigma"] and digest(a) == d["body"]


@pytest.mark.skipif(not O.have_ref(), reason="reference library not built")
def test_port_matches_reference_random_sweep():
    rng = np.random.default_rng(7)
    for t in range(400):
        p = int(rng.choice([2, 3, 5, 7, 65521, 8388593]))
        m, n = (int(x) for x in rng.integers(0, 24, 2))
        a = rng.integers(0, p, (m, n), dtype=np.uint64).astype(np.uint32)
        if t % 3 == 0 and n > 2:
            a[:, : n // 2] = 0
        a1, a2 = a.copy(), a.copy()
        R, P = O.ref_cup(a1, p), O.port_cup(a2, p)
        assert R.rank == P.rank and np.array_equal(R.rrp, P.rrp)
        assert np.array_equal(R.sigma, P.sigma) and np.array_equal(a1, a2)
