"""Test-side input generators (numpy only) following the BASELINE.json recipes."""
import hashlib

import numpy as np

import oracle as O


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def matmul_mod(a, b, p):
    """Exact (a @ b) mod p for uint32 inputs < p < 2^31 (chunked uint64)."""
    a = a.astype(np.uint64)
    b = b.astype(np.uint64)
    k = a.shape[1]
    step = max(1, min(k, (1 << 63) // max(1, (p - 1) * (p - 1)) // 2))
    out = np.zeros((a.shape[0], b.shape[1]), np.uint64)
    for k0 in range(0, k, step):
        out = (out + (a[:, k0:k0 + step] @ b[k0:k0 + step, :]) % p) % p
    return out.astype(np.uint32)


def c2_style(m, n, inner, seed, p):
    """BASELINE config 2 recipe: A = L*R mod p with
    L = random_matrix(m, inner, seed), R = random_matrix(inner, n, seed+1),
    rows i = 2 (mod 3) zeroed, rows shuffled by Fisher-Yates with
    SplitMix64(seed+2) (reference.cpp:269), new row i = old row s[i]."""
    L = O.port_random_matrix(m, inner, seed, p)
    R = O.port_random_matrix(inner, n, seed + 1, p)
    A = matmul_mod(L, R, p)
    A[2::3, :] = 0
    s = np.arange(m, dtype=np.int64)
    rnd = O.splitmix64(seed + 2, m)
    t = 0
    for i in range(m, 1, -1):
        j = int(rnd[t] % np.uint64(i))
        t += 1
        s[i - 1], s[j] = s[j], s[i - 1]
    return np.ascontiguousarray(A[s, :])


def c4_batch(count, p=8388593, seed=4):
    """BASELINE config 4 recipe: meta = SplitMix64(seed); per matrix
    r = 128 + below(129), L = random_matrix(256, r, next), R = random_matrix(r, 256, next)."""
    meta = O.splitmix64(seed, 3 * count)
    mats, ranks = [], []
    for t in range(count):
        r = 128 + int(meta[3 * t] % np.uint64(129))
        L = O.port_random_matrix(256, r, int(meta[3 * t + 1]), p)
        R = O.port_random_matrix(r, 256, int(meta[3 * t + 2]), p)
        mats.append(matmul_mod(L, R, p))
        ranks.append(r)
    return np.stack(mats), ranks


def load_npz_cases(path, prefix_keys):
    z = np.load(path)
    n = int(z["count"])
    for i in range(n):
        yield {k: z[f"{k}_{i}"] for k in prefix_keys}


def freivalds_dev(orig, body, rank, sigma, p, trials=2, seed=1, block=2048):
    """Device-side A*P^T*x == C*(U*x) mod p for torch int32 matrices holding
    u32 values < p <= 2^16 (every partial sum < 2^53: exact in float64)."""
    import torch
    assert p <= 65536
    m, n = orig.shape
    r = int(rank)
    g = torch.Generator(device="cpu").manual_seed(seed)
    sig = torch.as_tensor(np.asarray(sigma, dtype=np.int64), device=orig.device)
    for _ in range(trials):
        x = torch.randint(0, p, (n,), generator=g, dtype=torch.int64).to(orig.device)
        y = torch.zeros(n, dtype=torch.int64, device=orig.device)
        y[sig] = x
        yd, xd = y.double(), x.double()
        lhs = torch.empty(m, dtype=torch.int64, device=orig.device)
        for i0 in range(0, m, block):
            i1 = min(m, i0 + block)
            lhs[i0:i1] = torch.remainder(orig[i0:i1].double() @ yd, p).long()
        ux = torch.empty(r, dtype=torch.int64, device=orig.device)
        for i0 in range(0, r, block):
            i1 = min(r, i0 + block)
            blk = torch.triu(body[i0:i1].double(), diagonal=i0 + 1)   # cols > row (unit diagonal implicit)
            ux[i0:i1] = torch.remainder(blk @ xd + xd[i0:i1], p).long()
        uxd = ux.double()
        rhs = torch.empty(m, dtype=torch.int64, device=orig.device)
        for i0 in range(0, m, block):
            i1 = min(m, i0 + block)
            blk = torch.tril(body[i0:i1, :r].double(), diagonal=i0)    # C: cols <= row, < r
            rhs[i0:i1] = torch.remainder(blk @ uxd, p).long()
        if not torch.equal(lhs, rhs):
            return False
    return True
