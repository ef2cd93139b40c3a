"""Parity checkers for the CUP hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package.
The product (``paper_1112_5717_b200``) never imports it: the GPU path fails
loudly when its CUDA library is missing instead of falling back here.

Two checkers, both over numpy uint32 row-major matrices:

* ``port``  -- ``oracle/liboracle_port.so``: our plain-C restatement of the
  reference algorithm (``oracle/cup_oracle.c``, citing
  ``/root/reference/proj/src/factor.cpp:12-85`` etc.).
* ``ref``   -- ``oracle/_ref/libranklab_ref.so``: the UNMODIFIED reference
  library compiled from ``/root/reference/proj/src`` by ``oracle/Makefile``
  with a thin C wrapper (``oracle/ref_capi.cpp``).  Present wherever the
  build ran (it travels to the GPU box inside the repo snapshot).

The port is pinned against ``ref`` and the golden vectors in
``tests/golden`` by ``tests/test_oracle.py``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "liboracle_port.so")
REF_PATH = os.path.join(_HERE, "_ref", "libranklab_ref.so")

_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_u32 = C.c_uint32
_u64 = C.c_uint64

REF_STATUS = {0: "ok", 1: "DimensionMismatch", 2: "OverlapError", 3: "SingularMatrix",
              4: "NotPrime/ModulusOutOfRange", 9: "Error"}


class RefError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(REF_STATUS.get(code, f"status {code}"))
        self.code = code


@dataclass
class CupResult:
    rank: int
    rrp: np.ndarray          # uint32[rank]
    sigma: np.ndarray        # uint32[n]
    ops: np.ndarray | None = None   # (n_mul, n_addsub, n_divinv, n_ztest) for ref
    ipiv: np.ndarray | None = field(default=None)


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference (when its sources exist)."""
    import subprocess
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", _HERE, "-j8", *targets], check=True)


_port = None
_ref = None


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            build(ref=False)
        lib = C.CDLL(PORT_PATH)
        lib.oracle_cup_u32.argtypes = [_u32p, _i64, _i64, _i64, _u32, C.POINTER(_i64),
                                       _u32p, _u32p, _u32p]
        lib.oracle_cup_u32.restype = C.c_int
        lib.oracle_mm.argtypes = [_u32p, _i64, _u32p, _i64, _u32p, _i64, _i64, _i64, _i64,
                                  _u32, _u32, _u32]
        lib.oracle_random_matrix.argtypes = [_i64, _i64, _u64, _u32, _u32p]
        lib.oracle_splitmix64.argtypes = [_u64, _i64, _u64p]
        lib.oracle_cup_model_ops.argtypes = [_i64, _i64, _i64]
        lib.oracle_cup_model_ops.restype = C.c_double
        _port = lib
    return _port


def have_ref() -> bool:
    return os.path.exists(REF_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(REF_PATH + " (run make -C oracle ref)")
        lib = C.CDLL(REF_PATH)
        lib.ref_cup_u32.argtypes = [_u32p, _i64, _i64, _i64, _u32, C.POINTER(_i64), _u32p,
                                    _u32p, _u64p]
        lib.ref_ple_u32.argtypes = [_u32p, _i64, _i64, _i64, _u32, C.POINTER(_i64), _u32p,
                                    _u32p, _u64p]
        lib.ref_mm_u32.argtypes = [_u32p, _i64, _u32p, _i64, _u32p, _i64, _i64, _i64, _i64,
                                   _u32, _u32, _u32, _u64p]
        lib.ref_trsm_u32.argtypes = [C.c_int, C.c_int, C.c_int, _u32p, _i64, _i64, _u32p,
                                     _i64, _i64, _i64, _u32, _i64, _u64p]
        lib.ref_rank_and_profile_u32.argtypes = [_u32p, _i64, _i64, _i64, _u32,
                                                 C.POINTER(_i64), _u32p]
        lib.ref_determinant_u32.argtypes = [_u32p, _i64, _i64, _u32, C.POINTER(_u32)]
        lib.ref_col_ech_trans_u32.argtypes = [_u32p, _i64, _i64, _i64, _u32, C.c_int,
                                              C.POINTER(_i64), _u32p, _u32p, _u64p]
        lib.ref_invert_u32.argtypes = [_u32p, _i64, _i64, _u32, _u64p]
        lib.ref_random_matrix_u32.argtypes = [_i64, _i64, _u64, _u32, _u32p]
        lib.ref_random_rank_matrix_u32.argtypes = [_i64, _i64, _i64, _u64, _u32, C.c_int,
                                                   _u32p]
        lib.ref_random_nonsingular_u32.argtypes = [_i64, _u64, _u32, _u32p]
        lib.ref_random_triangular_u32.argtypes = [_i64, _u64, _u32, _u32p]
        lib.ref_naive_gauss_u32.argtypes = [_u32p, _i64, _i64, _u32, C.POINTER(_i64), _u32p]
        lib.ref_splitmix64.argtypes = [_u64, _i64, _u64p]
        _ref = lib
    return _ref


def _check(code: int) -> None:
    if code != 0:
        raise RefError(code)


# ----------------------------------------------------------------------------
# port (our restatement)
# ----------------------------------------------------------------------------

def port_cup(a: np.ndarray, p: int) -> CupResult:
    """In-place CUP of ``a`` (uint32, C-contiguous) with the reference pivot rule."""
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    m, n = a.shape
    rank = _i64(0)
    k = max(1, min(m, n))
    rrp = np.zeros(k, np.uint32)
    ipiv = np.zeros(k, np.uint32)
    sigma = np.zeros(max(n, 1), np.uint32)
    port_lib().oracle_cup_u32(a, m, n, n, p, C.byref(rank), rrp, sigma, ipiv)
    r = rank.value
    return CupResult(r, rrp[:r].copy(), sigma[:n].copy(), None, ipiv[:r].copy())


def port_mm(a, b, c, alpha, beta, p):
    m, l = a.shape
    n = b.shape[1]
    port_lib().oracle_mm(a, max(l, 1), b, max(n, 1), c, max(n, 1), m, l, n, alpha, beta, p)
    return c


def port_random_matrix(m: int, n: int, seed: int, p: int) -> np.ndarray:
    out = np.zeros((m, n), np.uint32)
    if m * n:
        port_lib().oracle_random_matrix(m, n, seed & (2**64 - 1), p, out)
    return out


def splitmix64(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.uint64)
    port_lib().oracle_splitmix64(seed & (2**64 - 1), count, out)
    return out


def cup_model_ops(m: int, n: int, r: int) -> float:
    """W(m,n,r) = 2mnr - (m+n)r^2 + (2/3)r^3 (bench.cpp:12-13)."""
    return 2.0 * m * n * r - (m + n) * r * r + (2.0 / 3.0) * r ** 3


# ----------------------------------------------------------------------------
# ref (the reference itself)
# ----------------------------------------------------------------------------

def ref_cup(a: np.ndarray, p: int) -> CupResult:
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    sigma = np.zeros(max(n, 1), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(ref_lib().ref_cup_u32(a, m, n, max(n, 1), p, C.byref(rank), rrp, sigma, ops))
    r = rank.value
    return CupResult(r, rrp[:r].copy(), sigma[:n].copy(), ops)


def ref_ple(a: np.ndarray, p: int):
    """ranklab::ple on ``a`` in place (factor.cpp:87-156): (rank, col_profile, row_perm, ops)."""
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    m, n = a.shape
    rank = _i64(0)
    prof = np.zeros(max(1, min(m, n)), np.uint32)
    perm = np.zeros(max(m, 1), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(ref_lib().ref_ple_u32(a, m, n, max(n, 1), p, C.byref(rank), prof, perm, ops))
    r = rank.value
    return r, prof[:r].copy(), perm[:m].copy(), ops


def ref_mm(a, b, c, alpha, beta, p):
    m, l = a.shape
    n = b.shape[1]
    ops = np.zeros(4, np.uint64)
    _check(ref_lib().ref_mm_u32(a, max(l, 1), b, max(n, 1), c, max(n, 1), m, l, n,
                                alpha, beta, p, ops))
    return c


def ref_trsm(side: str, uplo: str, diag: str, t, b, p, threshold=1, return_ops=False):
    k = t.shape[0]
    m, n = b.shape
    ops = np.zeros(4, np.uint64)
    _check(ref_lib().ref_trsm_u32(int(side == "right"), int(uplo == "lower"),
                                  int(diag == "unit"), t, max(k, 1), k, b, max(n, 1), m, n,
                                  p, threshold, ops))
    return (b, ops) if return_ops else b


def ref_rank_and_profile(a, p):
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    _check(ref_lib().ref_rank_and_profile_u32(a, m, n, max(n, 1), p, C.byref(rank), rrp))
    return rank.value, rrp[:rank.value].copy()


def ref_determinant(a, p):
    n = a.shape[0]
    d = _u32(0)
    _check(ref_lib().ref_determinant_u32(a, n, max(n, 1), p, C.byref(d)))
    return d.value


def ref_col_ech_trans(a, p, reduced=False, return_ops=False):
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    sigma = np.zeros(max(n, 1), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(ref_lib().ref_col_ech_trans_u32(a, m, n, max(n, 1), p, int(reduced),
                                           C.byref(rank), rrp, sigma, ops))
    r = rank.value
    res = CupResult(r, rrp[:r].copy(), sigma[:n].copy())
    return (res, ops) if return_ops else res


def ref_invert(a, p, return_ops=False):
    """invert_in_place; returns the status (0 ok, 3 singular) with the ops
    when return_ops, else raises on a nonzero status."""
    n = a.shape[0]
    ops = np.zeros(4, np.uint64)
    st = ref_lib().ref_invert_u32(a, n, max(n, 1), p, ops)
    if return_ops:
        return st, ops
    _check(st)
    return a


def ref_random_matrix(m, n, seed, p):
    out = np.zeros((m, n), np.uint32)
    _check(ref_lib().ref_random_matrix_u32(m, n, seed & (2**64 - 1), p, out))
    return out


def ref_random_rank_matrix(m, n, r, seed, p, generic=False):
    out = np.zeros((max(m, 1), max(n, 1)), np.uint32)[:m, :n].copy()
    _check(ref_lib().ref_random_rank_matrix_u32(m, n, r, seed & (2**64 - 1), p,
                                                int(generic), out))
    return out


def ref_random_nonsingular(n, seed, p):
    out = np.zeros((n, n), np.uint32)
    _check(ref_lib().ref_random_nonsingular_u32(n, seed & (2**64 - 1), p, out))
    return out


def ref_random_triangular(n, seed, p):
    out = np.zeros((n, n), np.uint32)
    _check(ref_lib().ref_random_triangular_u32(n, seed & (2**64 - 1), p, out))
    return out


def ref_naive_gauss(a, p):
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    _check(ref_lib().ref_naive_gauss_u32(a, m, n, p, C.byref(rank), rrp))
    return rank.value, rrp[:rank.value].copy()


def ref_splitmix64(seed, count):
    out = np.zeros(count, np.uint64)
    _check(ref_lib().ref_splitmix64(seed & (2**64 - 1), count, out))
    return out


# ----------------------------------------------------------------------------
# independent checks
# ----------------------------------------------------------------------------

def expand_cup(body: np.ndarray, rank: int):
    """Explicit C (m x r) and U (r x n, unit diagonal) from a packed body
    (factor.cpp:198-211)."""
    m, n = body.shape
    r = rank
    Cm = np.zeros((m, r), np.uint64)
    for j in range(r):
        Cm[j:, j] = body[j:, j]
    U = np.zeros((r, n), np.uint64)
    for i in range(r):
        U[i, i] = 1
        U[i, i + 1:] = body[i, i + 1:]
    return Cm, U


def freivalds_cup(orig: np.ndarray, body: np.ndarray, rank: int, sigma: np.ndarray,
                  p: int, trials: int = 2, seed: int = 1) -> bool:
    """Check A = C*U*P with random vectors: A*P^T*x == C*(U*x) mod p.

    Size-independent reconstruction check for large matrices.  Works blockwise
    in uint64 with periodic reduction (p < 2^31).
    """
    rng = np.random.default_rng(seed)
    m, n = orig.shape
    r = rank
    for _ in range(trials):
        x = rng.integers(0, p, size=n, dtype=np.uint64)
        # column j of A*P^T is column sigma[j] of A  ->  (A P^T x) = A @ y, y[sigma[j]] = x[j]
        y = np.zeros(n, np.uint64)
        y[sigma.astype(np.int64)] = x
        lhs = _matvec_mod(orig, y, p)
        # U*x (U unit upper r x n stored in body rows 0..r-1, cols > i)
        ux = np.zeros(r, np.uint64)
        for i0 in range(0, r, 512):
            i1 = min(r, i0 + 512)
            rows = body[i0:i1, :].astype(np.uint64)
            cols = np.arange(n)[None, :]
            rowsidx = np.arange(i0, i1)[:, None]
            rows = np.where(cols > rowsidx, rows, 0)
            ux[i0:i1] = (_matvec_mod(rows, x, p) + x[i0:i1]) % p
        # C*(Ux): C[i, j] = body[i, j] for j <= min(i, r-1)
        rhs = np.zeros(m, np.uint64)
        for i0 in range(0, m, 512):
            i1 = min(m, i0 + 512)
            rows = body[i0:i1, :r].astype(np.uint64)
            cols = np.arange(r)[None, :]
            rowsidx = np.arange(i0, i1)[:, None]
            rows = np.where(cols <= rowsidx, rows, 0)
            rhs[i0:i1] = _matvec_mod(rows, ux, p)
        if not np.array_equal(lhs % p, rhs % p):
            return False
    return True


def _matvec_mod(a: np.ndarray, x: np.ndarray, p: int) -> np.ndarray:
    """(a @ x) mod p for uint entries < p < 2^31, exact."""
    a = a.astype(np.uint64, copy=False)
    x = x.astype(np.uint64) % p
    out = np.zeros(a.shape[0], np.uint64)
    # each product < 2^62; accumulate 2 at a time is too slow -> reduce per column chunk
    step = 1 if p >= (1 << 31) else max(1, (1 << 63) // ((p - 1) * (p - 1) + 1) - 1)
    step = min(step, 4096)
    n = a.shape[1]
    for j0 in range(0, n, step):
        j1 = min(n, j0 + step)
        out = (out + (a[:, j0:j1] * x[None, j0:j1]).sum(axis=1, dtype=np.uint64) % p) % p
    return out
