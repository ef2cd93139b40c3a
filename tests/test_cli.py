"""The package CLI (python -m paper_1112_5717_b200, cli.py) against the
reference's command-line behaviour (proj/tools/main.cpp) rebuilt on the
reference library (oracle/_ref/ref_cli): byte-identical stdout, --out files and
exit codes.  CPU tests cover the text format's diagnostics and the seeded
generators; GPU tests run every subcommand end to end."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from paper_1112_5717_b200 import gen, textio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "ref_cli")
needs_cli = pytest.mark.skipif(not os.path.exists(REF_CLI), reason="oracle/_ref/ref_cli not built")


def _run(cmd, env=None):
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env=env)
    return r.returncode, r.stdout, r.stderr


def ours(*args):
    return _run([sys.executable, "-m", "paper_1112_5717_b200", *args])


def ref(*args):
    return _run([REF_CLI, *args])


def _write(path, a, p):
    with open(path, "w", newline="") as f:
        f.write(textio.format_matrix(a, p))


BAD = {
    "double_space": "2  2 7\n1 2\n3 4\n",
    "not_prime": "2 2 8\n1 2\n3 4\n",
    "big_modulus": "1 1 2147483648\n0\n",
    "entry_range": "2 2 7\n1 2\n3 7\n",
    "trailing": "2 2 7\n1 2 \n3 4\n",
    "short_row": "2 2 7\n1 2\n3\n",
    "missing_row": "2 2 7\n1 2\n",
    "crlf": "2 2 7\r\n1 2\n3 4\n",
    "letter": "2 2 7\n1 x\n3 4\n",
    "too_large": "1048577 1 7\n",
    "empty": "",
}


@needs_cli
@pytest.mark.parametrize("name", sorted(BAD))
def test_parse_errors_match_reference(tmp_path, name):
    # rejected before any device work: runs without a GPU
    f = tmp_path / "bad.mat"
    f.write_bytes(BAD[name].encode())
    assert ours("factor", "--in", str(f)) == ref("factor", "--in", str(f))


@needs_cli
def test_missing_file_and_usage(tmp_path):
    rc, out, err = ours("factor", "--in", str(tmp_path / "nope.mat"))
    assert (rc, out, err) == ref("factor", "--in", str(tmp_path / "nope.mat"))
    assert ours("factor")[0] == 1 and ours("frobnicate")[0] == 1
    assert ours("--help")[0] == 0


def test_text_roundtrip():
    import io
    a = O.port_random_matrix(7, 5, 3, 65521)
    b, p = textio.read_matrix(io.StringIO(textio.format_matrix(a, 65521)))
    assert p == 65521 and np.array_equal(a, b)
    z, p = textio.read_matrix(io.StringIO("3 0 5\n\n\n\n"))
    assert z.shape == (3, 0)


def _numpy_product(b, c, p):
    return ((b.astype(object) @ c.astype(object)) % p).astype(np.uint32)


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_generators_match_reference(monkeypatch):
    # reference.cpp:199-287 (products by an exact CPU product in this test)
    monkeypatch.setattr(gen, "_product", _numpy_product)
    for p in (7, 65521, 2147483647):
        for n, seed in ((1, 3), (6, 4), (17, 5)):
            assert np.array_equal(gen.random_nonsingular_matrix(n, seed, p),
                                  O.ref_random_nonsingular(n, seed, p))
            assert np.array_equal(gen.random_triangular_matrix(n, seed, p),
                                  O.ref_random_triangular(n, seed, p))
            assert np.array_equal(gen.random_matrix(n, n + 2, seed, p),
                                  O.ref_random_matrix(n, n + 2, seed, p))
        for (m, n, r) in ((9, 6, 3), (6, 9, 4), (12, 12, 0), (5, 8, 5)):
            for spread in (False, True):
                assert np.array_equal(gen.random_rank_matrix(m, n, r, 11, p, spread=spread),
                                      O.ref_random_rank_matrix(m, n, r, 11, p, generic=not spread))


# ------------------------------------------------------------------ GPU
def _cases(tmp_path):
    rng = np.random.default_rng(1)
    cases = []
    for k, (m, n, r, p) in enumerate([(5, 7, 5, 7), (40, 30, 30, 65521), (30, 40, 12, 65521),
                                      (70, 70, 70, 8388593), (64, 90, 20, 3)]):
        a = O.ref_random_rank_matrix(m, n, r, 100 + k, p, generic=False) if r < min(m, n) \
            else O.port_random_matrix(m, n, 100 + k, p)
        f = tmp_path / f"a{k}.mat"
        _write(f, a, p)
        cases.append((str(f), a, p))
    b = rng.integers(0, 5, (12, 12), dtype=np.uint64).astype(np.uint32)
    b[:, 3] = 0
    f = tmp_path / "z.mat"
    _write(f, b, 5)
    cases.append((str(f), b, 5))
    return cases


@pytest.mark.gpu
@needs_cli
def test_factor_and_echelon_byte_identical(tmp_path):
    for path, _, _ in _cases(tmp_path):
        for algo in ("cup", "ple"):
            for extra in ([], ["--expand"], ["--count-ops"], ["--expand", "--count-ops"]):
                args = ["factor", "--in", path, "--algo", algo, *extra]
                assert ours(*args) == ref(*args), args
        for extra in ([], ["--reduced"]):
            args = ["echelon", "--in", path, *extra]
            assert ours(*args) == ref(*args), args
    # --out files
    path = _cases(tmp_path)[1][0]
    o1, o2 = tmp_path / "o1.txt", tmp_path / "o2.txt"
    assert ours("factor", "--in", path, "--out", str(o1), "--count-ops") == \
        ref("factor", "--in", path, "--out", str(o2), "--count-ops")
    assert o1.read_bytes() == o2.read_bytes()


@pytest.mark.gpu
@needs_cli
def test_inverse_and_solve_byte_identical(tmp_path):
    p = 65521
    a = O.port_random_matrix(50, 50, 9, p)
    fa = tmp_path / "a.mat"
    _write(fa, a, p)
    assert ours("inverse", "--in", str(fa)) == ref("inverse", "--in", str(fa))
    s = O.ref_random_rank_matrix(40, 40, 25, 3, p, generic=False)
    fs = tmp_path / "s.mat"
    _write(fs, s, p)
    rc = ours("inverse", "--in", str(fs))
    assert rc == ref("inverse", "--in", str(fs)) and rc[0] == 1 and rc[2] == "SINGULAR\n"
    fr = tmp_path / "r.mat"
    _write(fr, np.ascontiguousarray(O.port_random_matrix(50, 1, 4, p)), p)
    assert ours("solve", "--in", str(fa), "--rhs", str(fr)) == \
        ref("solve", "--in", str(fa), "--rhs", str(fr))
    # rank-deficient: consistent (b = A x) and inconsistent right-hand sides
    x = O.port_random_matrix(40, 1, 5, p)
    bc = ((s.astype(object) @ x.astype(object)) % p).astype(np.uint32)
    fb = tmp_path / "bc.mat"
    _write(fb, bc, p)
    assert ours("solve", "--in", str(fs), "--rhs", str(fb)) == \
        ref("solve", "--in", str(fs), "--rhs", str(fb))
    bi = bc.copy()
    free = sorted(set(range(40)) - set(O.ref_cup(s.copy(), p).rrp.tolist()))
    bi[free[-1], 0] = (int(bi[free[-1], 0]) + 1) % p  # a non-pivot row breaks consistency
    fi = tmp_path / "bi.mat"
    _write(fi, bi, p)
    r1 = ours("solve", "--in", str(fs), "--rhs", str(fi))
    assert r1 == ref("solve", "--in", str(fs), "--rhs", str(fi)) and r1[0] == 3


@pytest.mark.gpu
@needs_cli
@pytest.mark.parametrize("args", [
    ["--algo", "cup", "--n", "96"],
    ["--algo", "cup", "--n", "80", "--m", "120", "--r", "50", "--placement", "spread", "--json"],
    ["--algo", "ple", "--n", "70", "--m", "50", "--r", "30", "--trials", "2"],
    ["--algo", "ple", "--n", "64", "--field", "7"],
    ["--algo", "mm", "--n", "65"],
    ["--algo", "trsm", "--n", "70", "--threshold", "8", "--json"],
    ["--algo", "colech", "--n", "60", "--seed", "9"],
    ["--algo", "redcolech", "--n", "60", "--field", "251"],
])
def test_bench_lines_byte_identical(args):
    r1, r2 = ours("bench", *args), ref("bench", *args)
    assert r1[0] == r2[0] == 0
    assert r1[1] == r2[1]
