"""Seeded BASELINE.json workloads built on the device, and batch sharding.

Every input is bit-identical to the reference's own recipe:

* ``random_matrix`` closed form (reference.cpp:246-253) -> ``random_matrix_dev``;
* config 2: A = L*R mod p (L = random_matrix(m, k, S), R = random_matrix(k, n, S+1)),
  rows i = 2 (mod 3) zeroed, rows shuffled by Fisher-Yates with SplitMix64(S+2)
  (reference.cpp:269, ``below(i) = next() % i``, reference.hpp:48), new row i =
  old row s[i] (perm_apply_rows, perm.cpp:103-113);
* config 4: meta = SplitMix64(S); matrix t has rank r_t = 128 + meta.below(129),
  L_t = random_matrix(256, r_t, meta.next()), R_t = random_matrix(r_t, 256, meta.next()),
  A_t = L_t * R_t mod p (p = 8388593).

The products run through this package's exact mod-p GEMM (``mm_dev``); the
result is unique, so any exact GEMM gives the reference's bytes.  The batch of
config 4 is sharded across ranks as contiguous slices (``shard_range``): the
matrices are independent, so no collective touches the data path.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(seed: int, count: int) -> list[int]:
    """SplitMix64 stream (reference.cpp:175-181)."""
    out, s = [], seed & MASK64
    for _ in range(count):
        s = (s + 0x9E3779B97F4A7C15) & MASK64
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        out.append(z ^ (z >> 31))
    return out


def c4_recipe(count: int, seed: int = 4):
    """(ranks r_t, L seeds, R seeds) of the first ``count`` config-4 matrices."""
    meta = splitmix64(seed, 3 * count)
    ranks = [128 + meta[3 * t] % 129 for t in range(count)]
    lseeds = [meta[3 * t + 1] for t in range(count)]
    rseeds = [meta[3 * t + 2] for t in range(count)]
    return ranks, lseeds, rseeds


def c2_row_shuffle(m: int, seed: int) -> np.ndarray:
    """Fisher-Yates permutation s of config 2 (new row i = old row s[i])."""
    s = np.arange(m, dtype=np.int64)
    rnd = splitmix64(seed, m)
    t = 0
    for i in range(m, 1, -1):
        j = rnd[t] % i
        t += 1
        s[i - 1], s[j] = s[j], s[i - 1]
    return s


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of n_items owned by ``rank`` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def c2_dev(m: int = 4096, n: int = 8192, inner: int = 2048, seed: int = 2, p: int = 65521,
           stream=None):
    """Config 2 matrix on the device (torch int32 tensor holding u32 values)."""
    import torch

    from . import mm_dev, random_matrix_dev
    L = torch.empty((m, inner), dtype=torch.int32, device="cuda")
    R = torch.empty((inner, n), dtype=torch.int32, device="cuda")
    A = torch.empty((m, n), dtype=torch.int32, device="cuda")
    random_matrix_dev(L, m, inner, seed, p, stream=stream)
    random_matrix_dev(R, inner, n, seed + 1, p, stream=stream)
    mm_dev(L, R, A, m, inner, n, 1, 0, p, stream=stream)
    A[2::3, :] = 0
    s = torch.from_numpy(c2_row_shuffle(m, seed + 2)).cuda()
    return A.index_select(0, s).contiguous()


def c4_dev(count: int = 4096, seed: int = 4, p: int = 8388593, lo: int = 0, hi: int | None = None,
           stream=None):
    """Matrices [lo, hi) of the config-4 batch on the device: (tensor [hi-lo, 256, 256], ranks)."""
    import torch

    from . import mm_dev, random_matrix_dev
    hi = count if hi is None else hi
    ranks, ls, rs = c4_recipe(hi, seed)
    out = torch.empty((hi - lo, 256, 256), dtype=torch.int32, device="cuda")
    Lb = torch.empty((256, 256), dtype=torch.int32, device="cuda")
    Rb = torch.empty((256, 256), dtype=torch.int32, device="cuda")
    for t in range(lo, hi):
        r = ranks[t]
        random_matrix_dev(Lb, 256, r, ls[t], p, lda=256, stream=stream)
        random_matrix_dev(Rb, r, 256, rs[t], p, lda=256, stream=stream)
        mm_dev(Lb, Rb, out[t - lo], 256, r, 256, 1, 0, p, lda=256, ldb=256, ldc=256, stream=stream)
    return out, ranks[lo:hi]
