"""The reference's seeded input generators (proj/src/reference.cpp:175-287),
restated with vectorised SplitMix64 (the generator is counter-based: draw k of
SplitMix64(seed) is mix(seed + (k+1)*gamma)), products on the device through
the exact mod-p GEMM (unique result, so bit-identical to naive_mm).  Used by
the CLI's ``bench`` subcommand, which mirrors the reference's cmd_bench."""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def draws(seed: int, k0: int, count: int) -> np.ndarray:
    """Draws k0 .. k0+count-1 of SplitMix64(seed) (reference.cpp:175-181)."""
    with np.errstate(over="ignore"):
        k = np.arange(k0 + 1, k0 + count + 1, dtype=np.uint64)
        z = np.uint64(seed & ((1 << 64) - 1)) + k * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


class _Stream:
    """Sequential view of the same stream (below(i) = next() % i, reference.hpp:48)."""

    def __init__(self, seed: int):
        self.seed, self.k = seed, 0

    def take(self, count: int) -> np.ndarray:
        out = draws(self.seed, self.k, count)
        self.k += count
        return out

    def below(self, i: int) -> int:
        return int(self.take(1)[0]) % i


def random_matrix(m: int, n: int, seed: int, p: int) -> np.ndarray:
    """reference.cpp:246-253: row-major draws reduced mod p."""
    return (draws(seed, 0, m * n) % np.uint64(p)).astype(np.uint32).reshape(m, n)


def _upper_unit_rows(rng: _Stream, n: int, p: int) -> np.ndarray:
    """Rows i = 0..n-1: diagonal 1 + below(p-1), then entries j > i (row-major)."""
    t = np.zeros((n, n), np.uint32)
    cnt = n * (n + 1) // 2
    d = rng.take(cnt)
    off = 0
    for i in range(n):
        t[i, i] = 1 + int(d[off]) % (p - 1)
        t[i, i + 1:] = (d[off + 1:off + n - i] % np.uint64(p)).astype(np.uint32)
        off += n - i
    return t


def _fisher_yates(rng: _Stream, n: int) -> np.ndarray:
    s = np.arange(n, dtype=np.uint32)
    if n > 1:
        d = rng.take(n - 1)
        for t, i in enumerate(range(n, 1, -1)):
            j = int(d[t]) % i
            s[i - 1], s[j] = s[j], s[i - 1]
    return s


def _product(b: np.ndarray, c: np.ndarray, p: int) -> np.ndarray:
    from . import mm
    out = np.zeros((b.shape[0], c.shape[1]), np.uint32)
    if b.shape[1] == 0 or out.size == 0:
        return out
    mm(b, c, out, 1, 0, p)
    return out


def random_nonsingular_matrix(n: int, seed: int, p: int) -> np.ndarray:
    """reference.cpp:255-272: (unit lower L) * (upper U, nonzero diagonal), columns shuffled."""
    rng = _Stream(seed)
    lo = np.eye(n, dtype=np.uint32)
    d = rng.take(n * (n - 1) // 2)
    off = 0
    for i in range(1, n):
        lo[i, :i] = (d[off:off + i] % np.uint64(p)).astype(np.uint32)
        off += i
    up = _upper_unit_rows(rng, n, p)
    a = _product(lo, up, p)
    s = _fisher_yates(rng, n)
    return np.ascontiguousarray(a[:, s])  # perm_apply_cols(a, s, false): new col j = old col s[j]


def _choose_sorted(rng: _Stream, k: int, r: int) -> np.ndarray:
    return np.sort(_fisher_yates(rng, k)[:r])


def random_rank_matrix(m: int, n: int, r: int, seed: int, p: int, spread: bool = False) -> np.ndarray:
    """reference.cpp:199-244: B (m x r, identity on the chosen rows, random below
    them) times C (r x n, identity on the chosen columns); Generic placement puts
    the profile on the leading rows/columns, Spread picks sorted random ones."""
    if r > min(m, n):
        raise ValueError(f"{r} > min({m},{n})")
    rng = _Stream(seed)
    if spread:
        rows = _choose_sorted(rng, m, r)
        cols = _choose_sorted(rng, n, r)
    else:
        rows = np.arange(r, dtype=np.uint32)
        cols = np.arange(r, dtype=np.uint32)
    b = np.zeros((m, r), np.uint32)
    chosen = np.zeros(m, bool)
    chosen[rows] = True
    b[rows, np.arange(r)] = 1 % p
    for i in range(m):
        if chosen[i]:
            continue
        c = int(np.searchsorted(rows, i))  # j with rows[j] < i (rows sorted)
        if c:
            b[i, :c] = (rng.take(c) % np.uint64(p)).astype(np.uint32)
    cm = np.zeros((r, n), np.uint32)
    chosen = np.zeros(n, bool)
    chosen[cols] = True
    cm[np.arange(r), cols] = 1 % p
    free = np.nonzero(~chosen)[0]
    if r and len(free):
        vals = (rng.take(r * len(free)) % np.uint64(p)).astype(np.uint32).reshape(len(free), r)
        cm[:, free] = vals.T
    return _product(b, cm, p)


def random_triangular_matrix(n: int, seed: int, p: int) -> np.ndarray:
    """reference.cpp:274-287, UpLo::Upper: nonzero diagonal, random strict upper part."""
    return _upper_unit_rows(_Stream(seed), n, p)
