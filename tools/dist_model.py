#!/usr/bin/env python3
"""Per-phase model of the distributed config-5 CUP (paper_1112_5717_b200/dist.py,
65536^2 over GF(65521), 1D block-cyclic 1024-column tiles, row blocks b = 1024,
super-blocks S = 4096, window mode) at N = 1, 2, 4, 8 ranks, from kernels timed
HERE on one B200 at the per-rank shapes (only one GPU is available, so N > 1 is
a model, not a measurement).

Per row block j (r = 1024 j pivots so far, generic input: full rank, sigma = id):
  chain_j  (serial, on the owner of column r / on every rank):
      window CUP of the 1024 x 2048 block (owner only)            t_cup
    + U rows beyond the window on own columns, trsm L/L/N          t_ub(n_loc)
    + in-super-block TRSM, rows below in the SB split by N          t_sbt(rows/N)
    + collectives: gather to owner 4 MB, broadcast 4 MB + meta,
      all-gather of the solved rows (rows x 1024 x 2 B)            at BW
  trail_j  (divisible, overlapped with chain_{j+1} by the lookahead):
      in-SB Schur update, rows below in the SB x n_loc x 1024       t_mm
    + every 4th block: the rows below the SB get one TRSM (split by
      N, all-gathered: rows x 4096 x 2 B) and one Schur update
      rows x n_loc x 4096                                           t_mm
  T(N) = sum_j max(chain_j, trail_{j-1}) + chain_0
BW = 350 GB/s per collective (assumed NCCL bus bandwidth on NVLink 5 for
4-500 MB messages; not measured here).
Usage: dist_model.py [--quick]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1112_5717_b200 as G  # noqa: E402

P = 65521
M = N_COLS = 65536
B, S, WIN = 1024, 4096, 2048
BW = 350e9
quick = "--quick" in sys.argv
cache = {}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def buf(rows, cols, seed):
    t = torch.empty((max(rows, 1), max(cols, 1)), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(t, t.shape[0], t.shape[1], seed, P)
    return t


def t_mm(m, n, k):
    """C (m x n) -= A (m x k) * B (k x n), the Schur update."""
    if m <= 0 or n <= 0 or k <= 0:
        return 0.0
    # quantise the shape (the model only needs the rate at this size)
    key = ("mm", -(-m // 1024) * 1024, -(-n // 2048) * 2048, k)
    if key not in cache:
        mm, nn = key[1], key[2]
        a, b, c = buf(mm, k, 1), buf(k, nn, 2), buf(mm, nn, 3)
        cache[key] = timed(lambda: G.mm_dev(a, b, c, mm, k, nn, P - 1, 1, P))
        del a, b, c
    return cache[key] * (m * n) / (key[1] * key[2])


def t_trsm(side, uplo, diag, m, n):
    if m <= 0 or n <= 0:
        return 0.0
    q = 1024
    key = ("trsm", side, uplo, diag, -(-m // q) * q, -(-n // q) * q)
    if key not in cache:
        mm, nn = key[4], key[5]
        k = mm if side == 0 else nn
        t = buf(k, k, 4)
        # a well-conditioned triangle: nonzero diagonal
        t.diagonal().clamp_(min=1)
        b = buf(mm, nn, 5)
        cache[key] = timed(lambda: G.trsm_dev(side, uplo, diag, t, b, mm, nn, P))
        del t, b
    return cache[key] * (m * n) / (key[4] * key[5])


def t_cup(rows, cols):
    key = ("cup", rows, cols)
    if key not in cache:
        src = buf(rows, cols, 6)
        w = torch.empty_like(src)

        def run():
            w.copy_(src)
            G.cup_dev(w, rows, cols, P, sync=False)
        cache[key] = timed(run)
    return cache[key]


def model(nr):
    total = 0.0
    chains, trails = [], []
    for j in range(M // B):
        r = j * B
        in_sb = (S - (j % (S // B) + 1) * B)            # rows below the block inside its SB
        n_loc = max(0, N_COLS - r - WIN) / nr            # own columns beyond the window
        chain = t_cup(B, WIN)
        chain += t_trsm(0, 1, 0, B, int(n_loc))          # U rows beyond the window (Left/Lower/NonUnit)
        chain += t_trsm(1, 0, 1, -(-in_sb // nr), B)     # in-SB TRSM, this rank's slice
        if nr > 1:
            chain += (2 * B * WIN * 2 + in_sb * B * 2) / BW
        trail = t_mm(in_sb, int(max(0, N_COLS - r - B) / nr), B)
        if (j + 1) % (S // B) == 0:                      # rows below the super-block
            below = M - (j + 1) * B
            trail += t_trsm(1, 0, 1, -(-below // nr), S)
            trail += t_mm(below, int(max(0, N_COLS - r - B) / nr), S)
            if nr > 1:
                trail += below * S * 2 / BW
        chains.append(chain)
        trails.append(trail)
    total = chains[0] + sum(max(chains[j], trails[j - 1]) for j in range(1, len(chains))) + trails[-1]
    return total, sum(chains), sum(trails)


def engine_c5():
    """The single-GPU engine on the whole matrix (bench.py's N = 1 line)."""
    a = buf(M, N_COLS, 5)
    w = torch.empty_like(a)

    def run():
        w.copy_(a)
        G.cup_dev(w, M, N_COLS, P, sync=False)
    t = timed(run, reps=2)
    del a, w
    torch.cuda.empty_cache()
    return t


def main():
    torch.cuda.set_device(0)
    print(__doc__.split("Usage")[0].strip())
    print()
    print(f"window CUP 1024 x {WIN}: {t_cup(B, WIN) * 1e3:.3f} ms (standalone)")
    eng = engine_c5()
    print(f"single-GPU engine, whole matrix (bench.py N = 1): {eng * 1e3:.1f} ms (measured)")
    for nr in (1, 2, 4, 8):
        T, C, W = model(nr)
        print(f"N={nr}: modelled {T * 1e3:8.1f} ms  (serial chain {C * 1e3:7.1f} ms, "
              f"divisible trailing work per rank {W * 1e3:7.1f} ms)  vs the engine: speed-up "
              f"{eng / T:5.2f}, efficiency {eng / T / nr:5.2f}")


if __name__ == "__main__":
    main()
