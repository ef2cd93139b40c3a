"""Per-call overhead of the C ABI on tiny matrices (drop-in usage pattern)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1112_5717_b200 as G
rng = np.random.default_rng(0)
for shape, p, reps in [((3, 3), 3, 200), ((8, 8), 7, 200), ((40, 50), 65521, 100), ((256, 256), 65521, 20)]:
    a = rng.integers(0, p, shape).astype(np.uint32)
    G.cup(a.copy(), p)
    t = time.perf_counter()
    for _ in range(reps):
        G.cup(a.copy(), p)
    print(shape, "same shape: %.1f us/call" % ((time.perf_counter() - t) / reps * 1e6), flush=True)
t = time.perf_counter()
for i in range(100):
    m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    G.cup(rng.integers(0, 7, (m, n)).astype(np.uint32), 7)
print("random shapes: %.1f us/call" % ((time.perf_counter() - t) / 100 * 1e6), flush=True)
