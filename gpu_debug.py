"""Quick GPU debug sweep: GEMM and CUP vs the oracle, prints every result."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, ".")
import oracle as O
import paper_1112_5717_b200 as G

def chk(name, ok):
    print(("PASS " if ok else "FAIL ") + name, flush=True)
    return ok

rng = np.random.default_rng(0)
# ---- GEMM
for (p, m, l, n) in [(65521, 128, 128, 128), (65521, 200, 300, 170), (65521, 256, 1000, 300),
                     (251, 130, 129, 300), (257, 64, 64, 64), (8388593, 150, 260, 70),
                     (2147483647, 140, 200, 90), (65521, 33, 40, 35), (3, 40, 50, 60), (65521, 1024, 4096, 512)]:
    try:
        a = rng.integers(0, p, (m, l)).astype(np.uint32); b = rng.integers(0, p, (l, n)).astype(np.uint32)
        c = rng.integers(0, p, (m, n)).astype(np.uint32)
        for alpha, beta in [(p - 1, 1), (1, 0), (5 % p, 3 % p)]:
            c1 = c.copy(); c2 = c.copy()
            G.mm(a, b, c1, alpha, beta, p)
            O.port_mm(a, b, c2, alpha, beta, p)
            ok = np.array_equal(c1, c2)
            if not ok:
                d = np.argwhere(c1 != c2)
                print("   mismatches", len(d), "first", d[:5], c1[tuple(d[0])], c2[tuple(d[0])])
            chk(f"mm p={p} {m}x{l}x{n} a={alpha} b={beta}", ok)
    except Exception:
        traceback.print_exc()
# ---- CUP
def cup_case(name, a, p):
    try:
        a1 = a.copy(); a2 = a.copy()
        t = time.time(); g = G.cup(a1, p); tg = time.time() - t
        o = O.port_cup(a2, p)
        ok = g.rank == o.rank and np.array_equal(g.row_profile, o.rrp) and np.array_equal(g.col_perm, o.sigma) and np.array_equal(a1, a2)
        if not ok:
            print("   rank", g.rank, o.rank, "rrp eq", np.array_equal(g.row_profile, o.rrp), "sigma eq", np.array_equal(g.col_perm, o.sigma))
            d = np.argwhere(a1 != a2); print("   body mismatches", len(d), d[:8])
        chk(f"cup {name} {a.shape} p={p} r={o.rank} ({tg*1e3:.1f} ms)", ok)
    except Exception:
        traceback.print_exc()

for p in [65521, 7, 2, 3, 8388593, 2147483647]:
    for (m, n) in [(1, 1), (3, 5), (64, 64), (65, 70), (100, 300), (200, 150), (128, 128), (257, 513)]:
        cup_case("rand", rng.integers(0, p, (m, n)).astype(np.uint32), p)
for p in [2, 3, 65521]:
    for (m, n, r) in [(300, 200, 50), (200, 300, 120), (513, 257, 200), (100, 700, 60)]:
        cup_case("rankdef", O.ref_random_rank_matrix(m, n, r, 11 + m + r, p) if O.have_ref() else rng.integers(0, p, (m, n)).astype(np.uint32), p)
a = rng.integers(0, 65521, (300, 400)).astype(np.uint32); a[:, :200] = 0; cup_case("zerolead", a, 65521)
a = rng.integers(0, 65521, (300, 400)).astype(np.uint32); a[::3, :] = 0; cup_case("zerorows", a, 65521)
a = O.port_random_matrix(1024, 1024, 1, 65521); cup_case("C1", a, 65521)
