"""CPU construction of the BASELINE.json configs -- TEST INFRASTRUCTURE ONLY.

Restates the reference's own generator recipes (paths relative
to /root/reference):

* ``random_matrix(m, n, seed, GF(p))``: entry (i, j) = the (i*n + j + 1)-th
  SplitMix64 output mod p (proj/src/reference.cpp:175-181, 246-253), via the
  port (``oracle_random_matrix``);
* ``SplitMix64::below(i) = next() % i`` (proj/include/ranklab/reference.hpp:48) and
  the Fisher-Yates shuffle ``for i = m..2: swap(s[i-1], s[below(i)])``
  (reference.cpp:269); ``perm_apply_rows``: new row i = old row s[i]
  (proj/src/perm.cpp:103-113);
* products L*R mod p through the blocked oracle's exact float64 GEMM (the
  product is unique, so any exact GEMM gives the reference's bytes).

The device builds the same matrices in ``paper_1112_5717_b200/workloads.py``;
``tests/test_gpu_workloads.py`` checks both agree.
"""
from __future__ import annotations

import numpy as np

from . import port_random_matrix, splitmix64
from .blocked import _matmul_mod

P16 = 65521
P23 = 8388593


def product_mod(L: np.ndarray, R: np.ndarray, p: int) -> np.ndarray:
    return _matmul_mod(L, R, p).astype(np.uint32)


def c1(seed: int = 1) -> tuple[np.ndarray, int]:
    return port_random_matrix(1024, 1024, seed, P16), P16


def c2_row_shuffle(m: int, seed: int) -> np.ndarray:
    s = np.arange(m, dtype=np.int64)
    rnd = splitmix64(seed, m)
    t = 0
    for i in range(m, 1, -1):
        j = int(rnd[t] % np.uint64(i))
        t += 1
        s[i - 1], s[j] = s[j], s[i - 1]
    return s


def c2(m: int = 4096, n: int = 8192, inner: int = 2048, seed: int = 2) -> tuple[np.ndarray, int]:
    """A = L*R mod p, rows i = 2 (mod 3) zeroed, rows shuffled."""
    p = P16
    L = port_random_matrix(m, inner, seed, p)
    R = port_random_matrix(inner, n, seed + 1, p)
    A = product_mod(L, R, p)
    A[2::3, :] = 0
    s = c2_row_shuffle(m, seed + 2)
    return np.ascontiguousarray(A[s]), p


def c3(seed: int = 3) -> tuple[np.ndarray, int]:
    return port_random_matrix(16384, 16384, seed, P16), P16


def c4_recipe(count: int = 4096, seed: int = 4):
    meta = splitmix64(seed, 3 * count)
    ranks = [128 + int(meta[3 * t] % np.uint64(129)) for t in range(count)]
    return ranks, [int(meta[3 * t + 1]) for t in range(count)], [int(meta[3 * t + 2]) for t in range(count)]


def c4_matrix(t: int, ranks, ls, rs) -> np.ndarray:
    r = ranks[t]
    L = port_random_matrix(256, r, ls[t], P23)
    R = port_random_matrix(r, 256, rs[t], P23)
    return product_mod(L, R, P23)


def c5(seed: int = 5) -> tuple[np.ndarray, int]:
    return port_random_matrix(65536, 65536, seed, P16), P16


def s1(n: int = 8192, inner: int = 6144, zero_cols: int = 40) -> tuple[np.ndarray, int]:
    """Swap-heavy rank-deficient case over GF(3): A = L*R (rank <= inner) with the
    first ``zero_cols`` columns zeroed, so almost every pivot needs a
    transposition (a random GF(3) entry is zero with probability 1/3)."""
    p = 3
    L = port_random_matrix(n, inner, 11, p)
    R = port_random_matrix(inner, n, 12, p)
    A = product_mod(L, R, p)
    A[:, :zero_cols] = 0
    return A, p
