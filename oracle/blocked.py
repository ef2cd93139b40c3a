"""Blocked, multithreaded CPU restatement of ``ranklab::cup`` -- TEST
INFRASTRUCTURE ONLY (see ``oracle/__init__.py``: only ``tests/``, ``smoke()``
and ``bench.py``'s CPU legs may use it; the product never does).

Why it exists: the reference (``/root/reference/proj/src/factor.cpp:30-85``) is
single-threaded at ~3e8 mod-p ops/s, so config 3 (16384^2, 2.9e12 ops) takes
hours and config 5 (65536^2, 1.9e14 ops) days.  This restatement runs the SAME
recursion -- row split k = m/2 (factor.cpp:35), top half, sigma_1 applied to
the bottom rows (factor.cpp:42), trsm(Right, Upper, Unit) (factor.cpp:45-46),
early return when r1 = n (factor.cpp:47), Schur update H <- A22 - G*V1
(factor.cpp:51-52), bottom half (factor.cpp:53), sigma_2 applied to V1
(factor.cpp:56), U-row shift (factor.cpp:62-70), composition
perm_compose(P2.embed_at(r1, n), P1) (factor.cpp:78-79, perm.cpp:41-79) --
but with the arithmetic done by multithreaded BLAS:

* ``mm`` (kernels.cpp:28-75): C <- C - A*B mod p as float64 GEMMs, exact while
  every partial sum stays below 2^53 (K-chunks of (2^53 - p) / (p-1)^2
  products: 2,098,176 for p = 65521, 127 for p = 8388593; for p >= 2^26 the
  A operand is split into 16-bit limbs first);
* ``trsm`` Right/Upper/Unit (kernels.cpp:135-154): the same halving recursion
  into that GEMM, base case column by column (kernels.cpp:92-101);
* leaves of <= ``leaf`` rows: ``oracle_cup_leaf_u32`` (oracle/cup_oracle.c),
  the iterative restatement of cup_base_row/cup_rec with delayed reduction.

Every intermediate is the reference's own intermediate (each sub-call's CUP
is unique given its input), so the bytes equal ``ranklab::cup``'s.  Pinned
bit-exactly against the compiled reference by ``tests/test_oracle_blocked.py``
(random shapes/primes/ranks, leaf sizes 1..64) and by
``tools/pin_scale_digests.py`` (config 1, the full config 2, all 4096 config-4
matrices), which then commits the config-3/config-5 digests in
``tests/golden/scale_digests.json``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import port_lib

_F53 = float(1 << 53)


def _lib():
    lib = port_lib()
    if not hasattr(lib, "_blocked_ready"):
        lib.oracle_cup_leaf_u32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_uint32,
                                            C.POINTER(C.c_int64), C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        lib.oracle_cup_leaf_u32.restype = C.c_int
        lib.oracle_digest_u32.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64]
        lib.oracle_digest_u32.restype = C.c_uint64
        lib._blocked_ready = True
    return lib


def digest(a: np.ndarray) -> int:
    """Order-independent 64-bit digest of a uint32 matrix (oracle_digest_u32;
    the device computes the same function in rl_digest_u32_dev)."""
    a = np.asarray(a)
    assert a.dtype == np.uint32 and a.ndim == 2 and (a.size == 0 or a.strides[1] == 4)
    m, n = a.shape
    if m * n == 0:
        return 0
    return int(_lib().oracle_digest_u32(a.ctypes.data, m, n, a.strides[0] // 4))


# ---------------------------------------------------------------------------
# exact mod-p GEMM on float64 BLAS
# ---------------------------------------------------------------------------

def _kchunk(p: int, amax: int) -> int:
    """Largest K with K * amax * (p-1) + p < 2^53."""
    return max(0, int((_F53 - p) // (float(amax) * float(p - 1)))) if p > 1 else 1 << 30


def _matmul_mod(A: np.ndarray, B: np.ndarray, p: int) -> np.ndarray:
    """(A @ B) mod p as float64 (entries of A, B canonical, uint32 views)."""
    M, K = A.shape
    N = B.shape[1]
    out = np.zeros((M, N), np.float64)
    if K == 0 or M == 0 or N == 0:
        return out
    kc = _kchunk(p, p - 1)
    if kc >= 1:
        for k0 in range(0, K, kc):
            k1 = min(K, k0 + kc)
            out += A[:, k0:k1].astype(np.float64) @ B[k0:k1, :].astype(np.float64)
            np.mod(out, p, out=out)
        return out
    # large p: A = A1 * 2^16 + A0 (limbs < 2^16), products < 2^47
    kc = max(1, _kchunk(p, 1 << 16))
    A64 = A.astype(np.int64)
    for limb in (1, 0):
        part = np.zeros((M, N), np.float64)
        Al = ((A64 >> (16 * limb)) & 0xFFFF).astype(np.float64)
        for k0 in range(0, K, kc):
            k1 = min(K, k0 + kc)
            part += Al[:, k0:k1] @ B[k0:k1, :].astype(np.float64)
            np.mod(part, p, out=part)
        if limb == 1:
            out = np.mod(part * 65536.0, p)
        else:
            out = np.mod(out + part, p)
    return out


def mm_sub(Cv: np.ndarray, A: np.ndarray, B: np.ndarray, p: int, block_bytes: int = 1 << 30) -> None:
    """Cv <- (Cv - A @ B) mod p in place (mm(a, b, c, neg_one, one),
    kernels.cpp:28-75); Cv, A, B uint32 views, Cv disjoint from A and B."""
    M, K = A.shape
    N = B.shape[1]
    if M == 0 or N == 0 or K == 0:
        return
    # column panels of B and C bound the float64 temporaries
    nc = max(256, min(N, block_bytes // (8 * max(K, M))))
    mc = max(256, min(M, block_bytes // (8 * max(nc, K))))
    for n0 in range(0, N, nc):
        n1 = min(N, n0 + nc)
        Bp = B[:, n0:n1]
        for m0 in range(0, M, mc):
            m1 = min(M, m0 + mc)
            prod = _matmul_mod(A[m0:m1], Bp, p)
            T = Cv[m0:m1, n0:n1].astype(np.float64)
            T -= prod
            np.mod(T, p, out=T)
            Cv[m0:m1, n0:n1] = T.astype(np.uint32)


def trsm_right_upper_unit(Bv: np.ndarray, U: np.ndarray, p: int, base: int = 48) -> None:
    """Bv <- Bv * U^{-1}, U unit upper (its stored diagonal is never read),
    in place (trsm(Right, Upper, Unit), kernels.cpp:135-154 and the base case
    kernels.cpp:92-101)."""
    K = U.shape[0]
    M = Bv.shape[0]
    if K == 0 or M == 0:
        return
    if K <= base:
        kc = _kchunk(p, p - 1)
        if kc >= base:
            X = Bv.astype(np.float64)
            Uf = np.triu(U.astype(np.float64), 1)
            for j in range(1, K):
                col = X[:, j] - X[:, :j] @ Uf[:j, j]
                X[:, j] = np.mod(col, p)
            Bv[:, :] = X.astype(np.uint32)
        else:
            for j in range(1, K):
                t = _matmul_mod(Bv[:, :j], U[:j, j:j + 1], p)[:, 0]
                Bv[:, j] = np.mod(Bv[:, j].astype(np.float64) - t, p).astype(np.uint32)
        return
    k = K // 2
    trsm_right_upper_unit(Bv[:, :k], U[:k, :k], p, base)
    mm_sub(Bv[:, k:], Bv[:, :k], U[:k, k:], p)
    trsm_right_upper_unit(Bv[:, k:], U[k:, k:], p, base)


def _apply_cols(V: np.ndarray, s: np.ndarray, row_block: int = 4096) -> None:
    """V <- V * P^T (new column j = old column s[j]; perm_apply_cols,
    perm.cpp:115-125), moving only the columns that change."""
    idx = np.nonzero(s != np.arange(s.shape[0], dtype=s.dtype))[0]
    if idx.size == 0 or V.shape[0] == 0:
        return
    src = s[idx].astype(np.int64)
    for r0 in range(0, V.shape[0], row_block):
        blk = V[r0:r0 + row_block]
        blk[:, idx] = blk[:, src]


class _Cup:
    def __init__(self, a: np.ndarray, p: int, leaf: int):
        self.a = a
        self.p = p
        self.leaf = max(1, leaf)
        self.N = a.shape[1]
        self.acc = np.zeros(max(1, self.N), np.uint64)
        self.lib = _lib()

    def leafcup(self, i0, m, c0):
        w = self.N - c0
        a = self.a
        kk = max(1, min(m, w))
        rrp = np.zeros(kk, np.uint32)
        ipiv = np.zeros(kk, np.uint32)
        sig = np.zeros(w, np.uint32)
        rank = C.c_int64(0)
        ptr = a.ctypes.data + 4 * (i0 * a.strides[0] // 4 + c0)
        self.lib.oracle_cup_leaf_u32(ptr, m, w, a.strides[0] // 4, self.p, C.byref(rank),
                                     rrp.ctypes.data, sig.ctypes.data, ipiv.ctypes.data,
                                     self.acc.ctypes.data)
        r = rank.value
        return r, rrp[:r].astype(np.int64), sig, ipiv[:r].astype(np.int64)

    def rec(self, i0, m, c0):
        """cup_rec on the view a[i0:i0+m, c0:N] (factor.cpp:30-81).
        Returns (rank, row profile local to i0, sigma (order w), pivot
        positions local to c0)."""
        w = self.N - c0
        if m == 0 or w == 0:
            return 0, np.zeros(0, np.int64), np.arange(w, dtype=np.uint32), np.zeros(0, np.int64)
        if m <= self.leaf:
            return self.leafcup(i0, m, c0)
        a, p = self.a, self.p
        k = m // 2
        r1, rrp1, s1, ip1 = self.rec(i0, k, c0)
        _apply_cols(a[i0 + k:i0 + m, c0:], s1)                                  # factor.cpp:42
        trsm_right_upper_unit(a[i0 + k:i0 + m, c0:c0 + r1], a[i0:i0 + r1, c0:c0 + r1], p)  # :45-46
        if r1 == w:                                                             # :47
            return r1, rrp1, s1, ip1
        mm_sub(a[i0 + k:i0 + m, c0 + r1:], a[i0 + k:i0 + m, c0:c0 + r1],
               a[i0:i0 + r1, c0 + r1:], p)                                      # :51-52
        r2, rrp2, s2, ip2 = self.rec(i0 + k, m - k, c0 + r1)                    # :53
        _apply_cols(a[i0:i0 + r1, c0 + r1:], s2)                                # :56
        for l in range(r2):                                                     # :62-70
            dst, src = r1 + l, k + l
            if src == dst:
                continue
            a[i0 + dst, c0 + dst + 1:] = a[i0 + src, c0 + dst + 1:]
            a[i0 + src, c0 + dst + 1:] = 0
        e = np.concatenate([np.arange(r1, dtype=np.int64), r1 + s2.astype(np.int64)])
        sig = s1[e]                                                             # :78-79
        return (r1 + r2, np.concatenate([rrp1, k + rrp2]), sig,
                np.concatenate([ip1, r1 + ip2]))


class BlockedCup:
    """Result of :func:`cup`: rank, row profile, sigma, pivot positions."""

    def __init__(self, rank, rrp, sigma, ipiv):
        self.rank = rank
        self.rrp = rrp
        self.sigma = sigma
        self.ipiv = ipiv


def cup(a: np.ndarray, p: int, leaf: int = 32) -> BlockedCup:
    """In-place CUP of the uint32 row-major matrix ``a`` over GF(p), p < 2^31
    prime; same outputs as ``ranklab::cup`` (rank, row profile, col_perm, packed
    [C\\U] body) plus the pivot positions ipiv."""
    assert a.dtype == np.uint32 and a.ndim == 2 and (a.size == 0 or a.strides[1] == 4)
    m, n = a.shape
    r, rrp, sig, ip = _Cup(a, int(p), leaf).rec(0, m, 0)
    return BlockedCup(r, rrp.astype(np.uint32), sig.astype(np.uint32), ip.astype(np.uint32))


def opcount(m: int, n: int, rrp: np.ndarray, ipiv: np.ndarray) -> tuple[int, int, int, int]:
    """The reference's exact OpCounter of cup (mul, addsub, divinv, ztest) from
    the shape, row profile and pivot positions: trsm Right/Upper/Unit charges
    R*r1(r1-1)/2 mul and add/sub (kernels.cpp:92-101, 149-154), the Schur mm
    R*(w-r1)*r1 of each (kernels.cpp:54-68), a pivot row (ipiv[j]-j+1) ztests,
    one inverse and w-1 mul, a dead row w ztests (factor.cpp:12-28)."""
    r = len(rrp)
    rpre = np.zeros(m + 1, np.int64)
    j = 0
    for i in range(m):
        rpre[i] = j
        if j < r and int(rrp[j]) == i:
            j += 1
    rpre[m] = j
    tot = [0, 0, 0, 0]
    stack = [(0, m, n)]
    while stack:
        i0, mm, w = stack.pop()
        if mm == 0 or w == 0:
            continue
        if mm == 1:
            jj = int(rpre[i0])
            if rpre[i0 + 1] > jj:
                tot[3] += int(ipiv[jj]) - jj + 1
                tot[2] += 1
                tot[0] += w - 1
            else:
                tot[3] += w
            continue
        k = mm // 2
        r1 = int(rpre[i0 + k] - rpre[i0])
        R = mm - k
        t = R * r1 * max(r1 - 1, 0) // 2
        tot[0] += t
        tot[1] += t
        if r1 < w:
            s = R * (w - r1) * r1
            tot[0] += s
            tot[1] += s
            stack.append((i0 + k, R, w - r1))
        stack.append((i0, k, w))
    return tuple(tot)
