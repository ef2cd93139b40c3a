/*
 * oracle/cup_oracle.c -- CPU restatement of the reference CUP path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  The
 * product path (paper_1112_5717_b200/, libranklab_gpu.so) never links or
 * calls it.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * function here with oracle/_ref/libranklab_ref.so (built from
 * /root/reference/proj/src by oracle/Makefile) and with the golden vectors
 * committed under tests/golden/.
 *
 * What it restates (paths relative to /root/reference):
 *   - ranklab::cup            proj/src/factor.cpp:12-85.  Restated in the
 *     equivalent iterative form: rows are processed
 *     in order, the pivot of row i is the first nonzero at column positions
 *     [rank_before(i), n) (factor.cpp:15-21), it is brought to position r by
 *     a column TRANSPOSITION (factor.cpp:23-24, perm.cpp:21-26), the pivot
 *     stays raw and the rest of the row is scaled by its inverse
 *     (factor.cpp:25-26), every later row is eliminated right-looking
 *     (the Schur update of factor.cpp:51-52), and at the end the U rows are
 *     compacted to rows 0..r-1 with zero fill (the composed effect of the
 *     shift at factor.cpp:62-70).  sigma is the composition of the
 *     transpositions (perm_compose/embed_at, factor.cpp:78-79).
 *   - ranklab::mm             proj/src/kernels.cpp:28-75 (C <- aAB + bC mod p).
 *   - SplitMix64 / random_matrix  proj/src/reference.cpp:175-181, 246-253.
 *   - PrimeField::inv         proj/src/field.cpp:60-76 (any inverse is the
 *     same element; we use Fermat).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint32_t u32;
typedef uint64_t u64;

static u32 mulmod(u32 a, u32 b, u32 p) { return (u32)((u64)a * b % p); }

static u32 invmod(u32 a, u32 p) {
    /* Fermat a^(p-2); p prime (field.cpp:60-76 uses Euclid, same result). */
    u32 r = 1 % p, base = a % p, e = p - 2;
    while (e) {
        if (e & 1) r = mulmod(r, base, p);
        base = mulmod(base, base, p);
        e >>= 1;
    }
    return r;
}

/* SplitMix64 step (reference.cpp:175-181). */
static u64 splitmix_mix(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void oracle_splitmix64(u64 seed, int64_t count, u64* out) {
    u64 s = seed;
    for (int64_t t = 0; t < count; ++t) {
        s += 0x9E3779B97F4A7C15ull;
        out[t] = splitmix_mix(s);
    }
}

/* random_matrix(m, n, seed, GF(p)) (reference.cpp:246-253): entry (i,j) is
 * the (i*n+j+1)-th splitmix64 output reduced mod p. */
void oracle_random_matrix(int64_t m, int64_t n, u64 seed, u32 p, u32* out) {
    u64 s = seed;
    for (int64_t i = 0; i < m * n; ++i) {
        s += 0x9E3779B97F4A7C15ull;
        out[i] = (u32)(splitmix_mix(s) % p);
    }
}

/* C <- alpha*A*B + beta*C mod p; alpha, beta arbitrary canonical elements
 * (kernels.cpp:28-75; alpha == 0 or l == 0 short-circuits the product). */
void oracle_mm(const u32* a, int64_t lda, const u32* b, int64_t ldb, u32* c,
               int64_t ldc, int64_t m, int64_t l, int64_t n, u32 alpha, u32 beta,
               u32 p) {
    int no_product = (alpha == 0 || l == 0);
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            u64 cv = c[i * ldc + j];
            u64 t = beta == 0 ? 0 : (u64)mulmod((u32)cv, beta, p);
            if (!no_product) {
                u64 acc = 0;
                for (int64_t k = 0; k < l; ++k) {
                    acc += (u64)a[i * lda + k] * b[k * ldb + j] % p;
                    if (acc >= (1ull << 62)) acc %= p;
                }
                u32 s = (u32)(acc % p);
                s = mulmod(s, alpha, p);
                t = (t + s) % p;
            }
            c[i * ldc + j] = (u32)t;
        }
    }
}

/* In-place CUP.  a is m x n row-major with leading dimension lda, entries
 * canonical in [0,p).  Outputs: *rank, rrp[0..rank) (row rank profile),
 * sigma[0..n) (col_perm one-line), ipiv[0..rank) (absolute position of each
 * pivot when found; may be NULL).  Returns 0. */
int oracle_cup_u32(u32* a, int64_t m, int64_t n, int64_t lda, u32 p, int64_t* rank,
                   u32* rrp, u32* sigma, u32* ipiv) {
    int64_t r = 0;
    for (int64_t j = 0; j < n; ++j) sigma[j] = (u32)j;
    if (m == 0 || n == 0) { /* factor.cpp:32 */
        *rank = 0;
        return 0;
    }
    /* Delayed-reduction right-looking elimination; rows are eliminated
     * eagerly so row i is current when its pivot is searched. */
    for (int64_t i = 0; i < m; ++i) {
        u32* ri = a + i * lda;
        if (r == n) continue; /* early return of factor.cpp:47: rows keep G */
        int64_t c = -1;
        for (int64_t jj = r; jj < n; ++jj)
            if (ri[jj] != 0) { c = jj; break; }
        if (c < 0) continue; /* dead row: zero on [r, n) */
        if (c != r) { /* transposition T_{r,c} on every row (factor.cpp:23-24,42,56) */
            for (int64_t k = 0; k < m; ++k) {
                u32* rk = a + k * lda;
                u32 t = rk[r]; rk[r] = rk[c]; rk[c] = t;
            }
            u32 t = sigma[r]; sigma[r] = sigma[c]; sigma[c] = t;
        }
        if (ipiv) ipiv[r] = (u32)c;
        rrp[r] = (u32)i;
        u32 pinv = invmod(ri[r], p);
        for (int64_t jj = r + 1; jj < n; ++jj) ri[jj] = mulmod(ri[jj], pinv, p);
        /* Eliminate all later rows by pivot r: row_k[c'] -= row_k[r]*U[r][c']. */
        for (int64_t k = i + 1; k < m; ++k) {
            u32* rk = a + k * lda;
            u32 f = rk[r];
            if (f == 0) continue;
            u32 nf = p - f;
            for (int64_t jj = r + 1; jj < n; ++jj)
                rk[jj] = (u32)(((u64)nf * ri[jj] + rk[jj]) % p);
        }
        ++r;
    }
    /* Move U row j from row rrp[j] to row j, columns (j, n), zero-filling the
     * source: the composed effect of the shifts at factor.cpp:62-70. */
    for (int64_t j = 0; j < r; ++j) {
        int64_t src = rrp[j];
        if (src == j) continue;
        u32* d = a + j * lda;
        u32* s = a + src * lda;
        for (int64_t c = j + 1; c < n; ++c) {
            d[c] = s[c];
            s[c] = 0;
        }
    }
    *rank = r;
    return 0;
}

/* Leaf of the blocked oracle (oracle/blocked.py): the same CUP as
 * oracle_cup_u32 (same pivot rule, transpositions over all leaf rows, raw C
 * entries, normalised U rows moved to the top), computed LEFT-looking with
 * delayed reduction so a leaf of up to a few dozen rows costs one 64-bit
 * multiply-add per (pivot, column) instead of a modulo.  Row i first forms
 * its C entries C(i,j) = a_i[j] - sum_{j'<j} C(i,j') U_j'[j] (j < r, pivot
 * order), then its residual a_i[c] + sum_j (p - C(i,j)) U_j[c] for c >= r in
 * one u64 accumulator per column; the U rows U_j are the normalised pivot
 * rows (factor.cpp:25-26).  acc is caller scratch of n words.
 * Exact for p < 2^31: for p < 2^16 the lazy sum of <= 2^31 terms < 2^32 never
 * overflows; otherwise every product is reduced before it is added. */
int oracle_cup_leaf_u32(u32* a, int64_t m, int64_t n, int64_t lda, u32 p, int64_t* rank,
                        u32* rrp, u32* sigma, u32* ipiv, u64* acc) {
    int64_t r = 0;
    const int lazy = p <= 65536u;
    for (int64_t j = 0; j < n; ++j) sigma[j] = (u32)j;
    if (m == 0 || n == 0) { *rank = 0; return 0; }
    for (int64_t i = 0; i < m; ++i) {
        u32* ri = a + i * lda;
        /* C entries at the pivot positions found so far (once r == n these are
         * all the row holds: the TRSM output G of factor.cpp:45-47) */
        for (int64_t j = 0; j < r; ++j) {
            const u32* uj;
            u64 s = ri[j];
            for (int64_t j2 = 0; j2 < j; ++j2) {
                uj = a + (int64_t)rrp[j2] * lda;
                s += (u64)(p - ri[j2]) * uj[j] % p;
            }
            ri[j] = (u32)(s % p);
        }
        if (r == n) continue; /* factor.cpp:47 */
        /* residual on [r, n) */
        for (int64_t c = r; c < n; ++c) acc[c] = ri[c];
        for (int64_t j = 0; j < r; ++j) {
            const u32 nm = ri[j] ? p - ri[j] : 0u;
            if (!nm) continue;
            const u32* uj = a + (int64_t)rrp[j] * lda;
            if (lazy) {
                for (int64_t c = r; c < n; ++c) acc[c] += (u64)nm * uj[c];
            } else {
                for (int64_t c = r; c < n; ++c) acc[c] = (acc[c] + (u64)nm * uj[c] % p) % p;
            }
        }
        int64_t piv = -1;
        for (int64_t c = r; c < n; ++c) {
            ri[c] = (u32)(acc[c] % p);
            if (piv < 0 && ri[c]) piv = c;
        }
        if (piv < 0) continue;
        if (piv != r) { /* transposition on every leaf row (factor.cpp:23-24,42,56) */
            for (int64_t k = 0; k < m; ++k) {
                u32* rk = a + k * lda;
                u32 t = rk[r]; rk[r] = rk[piv]; rk[piv] = t;
            }
            u32 t = sigma[r]; sigma[r] = sigma[piv]; sigma[piv] = t;
        }
        if (ipiv) ipiv[r] = (u32)piv;
        rrp[r] = (u32)i;
        const u32 pinv = invmod(ri[r], p);
        for (int64_t c = r + 1; c < n; ++c) ri[c] = mulmod(ri[c], pinv, p);
        ++r;
    }
    for (int64_t j = 0; j < r; ++j) { /* U rows to rows 0..r-1 (factor.cpp:62-70) */
        int64_t src = rrp[j];
        if (src == j) continue;
        u32* d = a + j * lda;
        u32* s = a + src * lda;
        for (int64_t c = j + 1; c < n; ++c) { d[c] = s[c]; s[c] = 0; }
    }
    *rank = r;
    return 0;
}

/* Order-independent 64-bit digest of an m x n matrix: the sum mod 2^64 of
 * splitmix_mix(((i*n + j) << 32 | a[i][j]) + golden) over all entries (the
 * same function as the device's rl_digest_u32_dev, so the GPU tests compare
 * multi-GB bodies without copying them back). */
u64 oracle_digest_u32(const u32* a, int64_t m, int64_t n, int64_t lda) {
    u64 h = 0;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            const u64 e = (u64)(i * n + j);
            h += splitmix_mix((e << 32 | a[i * lda + j]) + 0x9E3779B97F4A7C15ull);
        }
    return h;
}

/* The reference's cost model (bench.cpp:12-13):
 * W(m,n,r) = 2mnr - (m+n)r^2 + (2/3)r^3 field operations. */
double oracle_cup_model_ops(int64_t m, int64_t n, int64_t r) {
    double dm = (double)m, dn = (double)n, dr = (double)r;
    return 2.0 * dm * dn * dr - (dm + dn) * dr * dr + (2.0 / 3.0) * dr * dr * dr;
}
