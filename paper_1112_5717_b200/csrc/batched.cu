// batched.cu -- CUP of many small independent matrices (config 4: 4096 x 256^2).
//
// One CTA per matrix, the matrix in global memory (its 256 KB working set stays
// L2-resident with up to 8 CTAs per SM), rows processed in order with the
// reference pivot rule (factor.cpp:12-28) and eager right-looking elimination;
// U rows are placed at the end (factor.cpp:62-70 composed).  Outputs per
// matrix: rank, row profile and pivot positions (sigma is composed on the host).
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {

__global__ void __launch_bounds__(256) cup_batched_kernel(u32* A, i64 stride, i32 m, i32 n, Fp f,
                                                          i32* ranks, i32* rrp_out, i32* ipiv_out,
                                                          i32 kcap) {
    __shared__ int s_wmin[8];
    __shared__ u32 s_pinv;
    __shared__ i32 s_rrp[1024];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u32* a = A + (i64)blockIdx.x * stride;
    i32* rrp = rrp_out + (i64)blockIdx.x * kcap;
    i32* ipiv = ipiv_out + (i64)blockIdx.x * kcap;
    int r = 0;
    for (int i = 0; i < m && r < n; ++i) {
        u32* ri = a + (i64)i * n;
        // first nonzero of row i at positions >= r
        int best = n;
        for (int c = r + tid; c < n; c += 256) {
            if (ri[c] != 0) {
                best = c;
                break;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) s_wmin[warp] = best;
        __syncthreads();
        int c = s_wmin[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) c = min(c, s_wmin[w]);
        __syncthreads();
        if (c >= n) continue;
        if (c != r) {
            for (int k = tid; k < m; k += 256) {
                u32* rk = a + (i64)k * n;
                const u32 t = rk[r];
                rk[r] = rk[c];
                rk[c] = t;
            }
            __syncthreads();
        }
        if (tid == 0) {
            s_pinv = inv_euclid(ri[r], f.p);
            if (r < 1024) s_rrp[r] = i;
            rrp[r] = i;
            ipiv[r] = c;
        }
        __syncthreads();
        const u32 pinv = s_pinv;
        for (int col = r + 1 + tid; col < n; col += 256) {
            const u32 u = mulmod(ri[col], pinv, f);
            ri[col] = u;
            const u32 nu = u ? f.p - u : 0u;
            for (int k = i + 1; k < m; ++k) {
                u32* rk = a + (i64)k * n;
                const u32 fk = rk[r];
                if (fk) rk[col] = red64((u64)fk * nu + rk[col], f);
            }
        }
        __syncthreads();
        ++r;
    }
    if (tid == 0) ranks[blockIdx.x] = r;
    __syncthreads();
    // place U rows: row j <- row rrp[j] on columns (j, n), zero-filling the source,
    // in increasing j for every column.
    for (int col = tid; col < n; col += 256) {
        for (int j = 0; j < r && j < col; ++j) {
            const i32 src = j < 1024 ? s_rrp[j] : rrp[j];
            if (src == j) continue;
            a[(i64)j * n + col] = a[(i64)src * n + col];
            a[(i64)src * n + col] = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// Blocked variant for n <= 256 (config 4): rows are taken in panels of PR = 32.
// A panel is factored in shared memory row by row with the same pivot rule
// (first nonzero at position >= r, transposition r <-> c applied to every row
// that is not final, raw pivot, normalised U row); its rows stay reduced u32
// words (32 KB), the lazy 64-bit sums live in registers only (see the panel
// loop).  Every trailing row is then updated once per panel: F = X_piv U_pp^{-1}
// and X_rest -= F U_rest on the FP64 tensor cores (trailing_dmma), or pivot by
// pivot by one warp per row when the panel held a transposition, p >= 2^24, or
// the panel is too wide.  46 KB of shared memory per CTA: four CTAs per SM.
#ifndef RL_BATCHED_PR
#define RL_BATCHED_PR 32
#endif
#ifndef RL_BATCHED_SB
#define RL_BATCHED_SB 4  // rows per sub-block of a panel (4 or 8): see the panel loop
#endif
#ifndef RL_BATCHED_NOTAB
#define RL_BATCHED_NOTAB 0  // 1: pivot inverses by the extended Euclid loop instead of the table (experiment)
#endif
#ifndef RL_BATCHED_FAST
#define RL_BATCHED_FAST 0  // 1: warp-level factorization of a panel's pivot window (generic position); measured slower, off
#endif
#ifndef RL_BATCHED_VEC
#define RL_BATCHED_VEC 1  // 16-byte panel loads and stores
#endif
#ifndef RL_BATCHED_CTAS
#define RL_BATCHED_CTAS 4  // CTAs per SM the register allocation is bounded for
#endif
#ifdef RL_BATCHED_TRACE  // per-phase cycle counts of a few CTAs (thread 0), printed at the end
#define BT_DECL long long bt_[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; long long bt_t = clock64()
#define BT_MARK(i) do { const long long bt_n = clock64(); bt_[i] += bt_n - bt_t; bt_t = bt_n; } while (0)
#else
#define BT_DECL
#define BT_MARK(i) do { } while (0)
#endif
constexpr int PR = RL_BATCHED_PR;  // panel rows
constexpr int BN = 256;
#ifndef RL_BATCHED_PS
#define RL_BATCHED_PS 260
#endif
constexpr int PS = RL_BATCHED_PS;  // row stride of the panel in shared memory (words): 16-byte rows; 260 puts
                                   // consecutive rows 4 banks apart (column reads down the rows: 4-way, not 32-way, conflicts)
static_assert(PS >= BN && PS % 4 == 0, "panel row stride");
constexpr int SB = RL_BATCHED_SB;
static_assert(PR == 32, "trailing_dmma's tiling assumes 32-row panels");
static_assert(SB == 4 || SB == 8, "row blocks of 4 or 8");

template <bool LAZY>
__device__ __forceinline__ u64 lazy_fma(u64 acc, u32 nf, u32 u, const Fp& f) {
    if (LAZY) return acc + (u64)nf * u;
    return addmod((u32)acc, mulmod(nf, u, f), f);
}

// x mod p for an integer-valued double 0 <= x < 2^52
__device__ __forceinline__ double dmod(double x, double pd, double ipd) {
    double r = fma(-floor(x * ipd), pd, x);
    r = r < 0.0 ? r + pd : r;
    return r >= pd ? r - pd : r;
}
__device__ __forceinline__ void dmma844(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
constexpr int XDS = 40;   // Xd row stride (doubles): rows 4 apart in banks -> 2 wavefronts per fragment load
constexpr int UDS = BN - PR + 8;  // Ud row stride (words), >= BN - PR, = 8 (mod 32): conflict-free fragments
static_assert(UDS % 32 == 8 && UDS % 8 == 0, "Ud stride");
// dynamic shared memory of cup_batched_blk_kernel (bytes)
constexpr int OFF_P = 0;                        // u32 [PR][BN] panel rows (reduced)
constexpr int OFF_UD = 0;                       // u32 [PR][UDS] U_rest, compacted in place from P
constexpr int OFF_XD = OFF_P + 4 * PR * PS;     // double [PR][XDS] U_pp^{-1}
constexpr int OFF_T = OFF_XD + 8 * PR * XDS;    // double [16][16] scratch of the doubling levels
constexpr int OFF_UPK = OFF_T + 8 * 256;        // u32 [PR (PR - 1) / 2] strict upper triangle of U_pp
constexpr int SMEM_BLK = OFF_UPK + 2048;
constexpr int OFF_FD = OFF_XD;                  // u32 [PR][SB] panel phase: multipliers of the row block's pivots
constexpr int LTS = 36;                         // row stride of Lt (words): 16-byte rows, 4-way store conflicts
constexpr int OFF_LT = OFF_XD;                  // u32 [PR][LTS] + [PR]: fast panel's multipliers and pivot inverses
constexpr int OFF_WBUF = OFF_XD;                // u32 [8][BN] row buffers of the pivot-by-pivot trailing path
static_assert(4 * PR * LTS + 4 * PR <= 8 * PR * XDS && 4 * PR * (PR - 1) / 2 <= 2048 && OFF_WBUF + 4 * 8 * BN <= SMEM_BLK && 4 * PR * SB <= 8 * PR * XDS,
              "shared-memory layout");

#ifdef RL_BATCHED_TRACE
__shared__ long long g_bt_mid;
#endif
__device__ __forceinline__ int upk_idx(int k, int i) { return k * (2 * PR - 1 - k) / 2 + (i - k - 1); }
// exact u32 -> double without the conversion pipe: 2^52 + w, minus 2^52
__device__ __forceinline__ double u2d(u32 w) {
    return __hiloint2double(0x43300000, (int)w) - 4503599627370496.0;
}

// The trailing rows of one panel (p < 2^24, no transposition in the panel), all
// products on the FP64 tensor cores (mma.sync m8n8k4): with U_pp the panel's
// unit upper pivot block (np x np) and U_rest its U rows right of it,
//   F = X_piv * U_pp^{-1}         (the C entries, the multipliers' negatives)
//   X_rest <- X_rest - F * U_rest
// -- the unique solution of the pivot-by-pivot elimination, so the bytes are
// the reference's.  Every term is an integer < 2^46 and a sum has at most
// 32 + 1 of them (< 2^52): exact in double, one reduction per output.  Warp =
// 8 trailing rows at a time: F (4 n8 tiles) by 32 DMMA against U_pp^{-1}, then
// its negation moves from the accumulator layout to the A-operand layout by
// shuffles and sweeps the row block's column tiles (C prefetched one tile ahead).
// U_rest stays u32 in shared memory (one wavefront per B fragment) and becomes
// a double in the register (u2d).
#ifndef RL_BATCHED_TRAIL_INLINE
#define RL_BATCHED_TRAIL_INLINE 0  // 1: inline trailing_dmma into the kernel (experiment)
#endif
#if RL_BATCHED_TRAIL_INLINE
#define RL_TRAIL_ATTR __forceinline__
#else
#define RL_TRAIL_ATTR __noinline__
#endif
__device__ RL_TRAIL_ATTR void trailing_dmma(u32* a, int m, int n, const Fp& f, int i0, int pr, int r0, int np,
                                           const i32* s_prow, unsigned char* sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q4 = lane & 3;
    const int cend = r0 + np, N = n - cend;
    const double pd = (double)f.p, ipd = 1.0 / pd;
    u32* Ud = reinterpret_cast<u32*>(sm + OFF_UD);        // [PR][UDS]
    double* Xd = reinterpret_cast<double*>(sm + OFF_XD);  // [PR][XDS]
    const u32* Pp = reinterpret_cast<const u32*>(sm + OFF_P);
    const u32* Upk = reinterpret_cast<const u32*>(sm + OFF_UPK);
    // (a) U_rest -> Ud, compacted in place from the panel rows (P under Ud): 16
    // rows per round, every thread loads its words, a barrier, then the stores
    // -- a round's destinations end below the next round's sources (pivot row j
    // sits in panel row s_prow[j] >= j and UDS <= BN), so one barrier per round
    // is enough.  U_pp (strict upper triangle, packed) was put aside at Upk.
    for (int q = 0; q < PR / 16; ++q) {
        u32 w[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + 256 * h;
            const int j = 16 * q + e / (UDS / 8), c0 = (e % (UDS / 8)) * 8;
            const bool on = e < 16 * (UDS / 8) && j < np;
            const u32* src = Pp + (on ? s_prow[j] : 0) * PS + cend + c0;
#pragma unroll
            for (int z = 0; z < 8; ++z) w[h][z] = (on && c0 + z < N) ? src[z] : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + 256 * h;
            const int j = 16 * q + e / (UDS / 8), c0 = (e % (UDS / 8)) * 8;
            if (e < 16 * (UDS / 8)) {
                *reinterpret_cast<uint4*>(Ud + j * UDS + c0) = make_uint4(w[h][0], w[h][1], w[h][2], w[h][3]);
                *reinterpret_cast<uint4*>(Ud + j * UDS + c0 + 4) = make_uint4(w[h][4], w[h][5], w[h][6], w[h][7]);
            }
        }
    }
    {   // diagonal 8 x 8 blocks of U_pp^{-1}: thread = (block, column), back substitution
        const int t = tid;
        if (t < PR) {
            const int b = t >> 3, c = t & 7, j = 8 * b + c;
            double x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = 0.0;
            x[c] = 1.0;
            // X[k][j] = -sum_{i=k+1..j} U[k][i] X[i][j]
#pragma unroll
            for (int kk = 7; kk >= 0; --kk) {
                if (kk < c) {
                    const int k = 8 * b + kk;
                    double acc = 0.0;
#pragma unroll
                    for (int ii = kk + 1; ii < 8; ++ii) {
                        if (ii <= c) {
                            const int i = 8 * b + ii;
                            const double u = (k < np && i < np) ? (double)Upk[upk_idx(k, i)] : 0.0;
                            acc = fma(u, x[ii], acc);
                        }
                    }
                    const double r = dmod(acc, pd, ipd);
                    x[kk] = r != 0.0 ? pd - r : 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < PR; ++k) Xd[k * XDS + j] = (k >> 3) == b ? x[k & 7] : 0.0;
        }
    }
    __syncthreads();
    // two doubling levels: X_AB = -X_AA * (U_AB * X_BB) for blocks of 8, then 16
    double* T = reinterpret_cast<double*>(sm + OFF_T);  // scratch [16][16]
#pragma unroll
    for (int h = 8; h <= PR / 2; h *= 2) {
        // pairs (A = [q*2h, q*2h+h), B = [q*2h+h, q*2h+2h)), entries of T = U_AB * X_BB
        const int npair = PR / (2 * h);
        for (int e = tid; e < npair * h * h; e += 256) {
            const int q = e / (h * h), rr = (e / h) % h, cc = e % h;
            const int ka = q * 2 * h + rr, jb = q * 2 * h + h + cc;
            double acc = 0.0;
            for (int i = 0; i < h; ++i) {
                const int ib = q * 2 * h + h + i;
                const double u = (ka < np && ib < np) ? (double)Upk[upk_idx(ka, ib)] : 0.0;
                acc = fma(u, Xd[ib * XDS + jb], acc);
            }
            T[(q * h + rr) * 16 + cc] = dmod(acc, pd, ipd);
        }
        __syncthreads();
        for (int e = tid; e < npair * h * h; e += 256) {
            const int q = e / (h * h), rr = (e / h) % h, cc = e % h;
            const int ka = q * 2 * h + rr, jb = q * 2 * h + h + cc;
            double acc = 0.0;
            for (int i = 0; i < h; ++i) acc = fma(Xd[ka * XDS + q * 2 * h + i], T[(q * h + i) * 16 + cc], acc);
            const double r = dmod(acc, pd, ipd);
            Xd[ka * XDS + jb] = r != 0.0 ? pd - r : 0.0;
        }
        __syncthreads();
    }
#ifdef RL_BATCHED_TRACE
    if (tid == 0) g_bt_mid = clock64();
#endif
    // (b) row blocks of 8 trailing rows per warp
    const int rbase = i0 + pr;
    const int R = m - rbase;
    const int ks_n = (np + 3) >> 2, tN = (N + 7) >> 3;
    for (int rb = warp; rb * 8 < R; rb += 8) {
        const int row = rbase + rb * 8 + g;
        const bool rok = row < m;
        u32* xr = a + (i64)row * n;
        // F = X_piv * U_pp^{-1}: four n8 tiles
        constexpr int KS = PR / 4, FT = PR / 8;
        double fa[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int k = 4 * ks + q4;
            fa[ks] = (rok && k < np) ? (double)__ldcg(xr + r0 + k) : 0.0;
        }
        double F[FT][2];
#pragma unroll
        for (int t = 0; t < FT; ++t) {
            F[t][0] = F[t][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
                if (ks < ks_n) dmma844(F[t][0], F[t][1], fa[ks], Xd[(4 * ks + q4) * XDS + 8 * t + g]);
        }
        // raw C entries to the pivot columns; negated multipliers in the A layout
        u32 nf[FT][2];
#pragma unroll
        for (int t = 0; t < FT; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int c = 8 * t + 2 * q4 + e;
                const u32 fv = (u32)dmod(F[t][e], pd, ipd);
                if (rok && c < np) xr[r0 + c] = fv;
                nf[t][e] = (c < np && fv) ? f.p - fv : 0u;
            }
        double na[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int src = g * 4 + (ks & 1) * 2 + (q4 >> 1);
            const u32 v0 = __shfl_sync(0xffffffffu, nf[ks >> 1][0], src);
            const u32 v1 = __shfl_sync(0xffffffffu, nf[ks >> 1][1], src);
            na[ks] = u2d((q4 & 1) ? v1 : v0);
        }
        // sweep the column tiles: C <- C + (p - F) * U_rest
        u32* cr = xr + cend + 2 * q4;
        u32 n0 = 0, n1 = 0;
        if (rok && tN > 0) {
            n0 = 2 * q4 < N ? __ldcg(cr) : 0u;
            n1 = 2 * q4 + 1 < N ? __ldcg(cr + 1) : 0u;
        }
        for (int tn = 0; tn < tN; ++tn) {
            const int cc = 8 * tn + 2 * q4;
            double c0 = u2d(n0), c1 = u2d(n1);
            if (tn + 1 < tN && rok) {  // next tile's C in flight during this one's products
                n0 = cc + 8 < N ? __ldcg(cr + 8 * (tn + 1)) : 0u;
                n1 = cc + 9 < N ? __ldcg(cr + 8 * (tn + 1) + 1) : 0u;
            }
            const u32* ub = Ud + q4 * UDS + 8 * tn + g;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
                if (ks < ks_n) dmma844(c0, c1, na[ks], u2d(ub[4 * ks * UDS]));
            if (rok) {
                if (cc < N) cr[8 * tn] = (u32)dmod(c0, pd, ipd);
                if (cc + 1 < N) cr[8 * tn + 1] = (u32)dmod(c1, pd, ipd);
            }
        }
    }
}

// Barrett reduction for the LAZY kernel (p < 2^24): with 2^(k-1) <= p < 2^k and
// x < 2^(2k+6) (up to 64 products of reduced elements), m = floor(2^(2k+6) / p):
//   q = floor(floor(x / 2^(k-1)) * m / 2^(k+7))  is within [x/p - 2, x/p]
// (Handbook of Applied Cryptography 14.42 with 6 spare bits), every operand a
// 32-bit word: two funnel shifts, one 32 x 32 -> 64 product, one 32-bit
// multiply-subtract -- about half the instructions of the 64-bit red64.
struct Bar24 {
    u32 m, s1, s2;
};
static Bar24 make_bar24(u32 p) {
    int k = 0;
    while ((p >> k) != 0) ++k;
    Bar24 b;
    b.m = (u32)((1ull << (2 * k + 6)) / p);
    b.s1 = (u32)(k - 1);
    b.s2 = (u32)(k + 7);
    return b;
}
__device__ __forceinline__ u32 red_b(u64 x, u32 p, const Bar24& b) {
    const u32 lo = (u32)x;
    const u32 t = __funnelshift_r(lo, (u32)(x >> 32), b.s1);
    const u64 pq = (u64)t * b.m;
    const u32 q = __funnelshift_r((u32)pq, (u32)(pq >> 32), b.s2);
    u32 r = lo - q * p;
    r = r >= 2 * p ? r - 2 * p : r;
    return r >= p ? r - p : r;
}

// x + nf * u mod p: through one product sum for p < 2^24 (LAZY), reduced at every
// product otherwise
template <bool LAZY>
__device__ __forceinline__ u32 fma_red(u32 x, u32 nf, u32 u, const Fp& f, const Bar24& b) {
    if (LAZY) return red_b((u64)nf * u + x, f.p, b);
    return addmod(x, mulmod(nf, u, f), f);
}

// Fast panel, step 1 (one warp): the panel's window columns [r0, r0 + 32) in
// place in shared memory, lane = column (see the kernel).  Compact loops on
// purpose: the fully unrolled register version was 15 K instructions that one
// warp runs once per panel -- instruction-fetch bound, 2.5x slower overall.
__device__ __noinline__ void fast_window(u32* P, u32* Lt, u32* pinvr, i32* s_prow, int* s_fast, int pr, int r0,
                                         int n, const Fp& f, const Bar24& bar, const u32* __restrict__ inv_tab) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int wc = r0 + lane;
    const bool in = wc < n;
    int jr = 0, k = 0;
    bool ok = true;
    for (; k < pr && ok; ++k) {
        const u32 xk = in ? P[k * PS + wc] : 0u;
        const unsigned msk = __ballot_sync(FULL, lane >= jr && xk != 0);
        u32 mine = 0, pinv = 0;
        if (msk != 0) {
            if (__ffs(msk) - 1 != jr) {  // its pivot is not at column r: a transposition
                ok = false;
            } else {
                const u32 pv = __shfl_sync(FULL, xk, jr);
                pinv = inv_tab ? __ldg(inv_tab + pv) : inv_euclid(pv, f.p);
                const bool act = in && lane > jr;
                const u32 u = act ? red_b((u64)xk * pinv, f.p, bar) : 0u;
                if (act) P[k * PS + wc] = u;
                // lane t holds row t's multiplier for this pivot (column jr of row t)
                const u32 fv = (lane > k && lane < pr) ? P[lane * PS + r0 + jr] : 0u;
                mine = fv ? f.p - fv : 0u;
                // eight rows at a time, loads before stores: eight independent
                // chains in flight (the compiler keeps a store ahead of the next load)
                int t = k + 1;
                if (t < pr) {  // the next row first: its entry at column jr + 1 is the likely next
                               // pivot, whose inverse is requested now and arrives under the loop
                    const u32 nf = __shfl_sync(FULL, mine, t);
                    u32 x1 = in ? P[t * PS + wc] : 0u;
                    if (act) {
                        x1 = red_b((u64)nf * u + x1, f.p, bar);
                        P[t * PS + wc] = x1;
                    }
                    const u32 pvn = __shfl_sync(FULL, x1, jr + 1);
                    if (inv_tab) {
                        [[maybe_unused]] u32 sink;
                        asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(sink) : "l"(inv_tab + pvn));
                    }
                    ++t;
                }
                for (; t + 7 < pr; t += 8) {
                    u32 nf[8], xv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) nf[q] = __shfl_sync(FULL, mine, t + q);
                    if (act) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) xv[q] = P[(t + q) * PS + wc];
#pragma unroll
                        for (int q = 0; q < 8; ++q) xv[q] = red_b((u64)nf[q] * u + xv[q], f.p, bar);
#pragma unroll
                        for (int q = 0; q < 8; ++q) P[(t + q) * PS + wc] = xv[q];
                    }
                }
                for (; t < pr; ++t) {
                    const u32 nf = __shfl_sync(FULL, mine, t);
                    if (act) P[t * PS + wc] = red_b((u64)nf * u + P[t * PS + wc], f.p, bar);
                }
                if (lane == 0) s_prow[jr] = k;
                ++jr;
            }
        }
        Lt[lane * LTS + k] = mine;
        if (lane == 0) pinvr[k] = pinv;
        __syncwarp();
    }
    for (; k < PR; ++k) {
        Lt[lane * LTS + k] = 0;
        if (lane == 0) pinvr[k] = 0;
    }
    if (lane == 0) {
        s_fast[0] = jr;
        s_fast[1] = ok ? 1 : 0;
    }
}

// Fast panel, step 2 (one thread per column c right of the window): forward
// substitution down the column against the multipliers of step 1, the finished
// entries read back from the column itself (a row without a pivot has zero
// multipliers against it); returns true if a row without a pivot is nonzero
// here (the panel is not generic).
__device__ __noinline__ bool fast_column(u32* P, const u32* Lt, const u32* pinvr, int pr, int c, const Fp& f,
                                         const Bar24& bar) {
    bool bad = false;
    for (int t = 0; t < pr; ++t) {
        u64 acc = P[t * PS + c];
        for (int j4 = 0; j4 < t; j4 += 4) {  // Lt[t][j] = 0 for j >= t
            const uint4 m4 = *reinterpret_cast<const uint4*>(Lt + t * LTS + j4);
            const u32* col = P + j4 * PS + c;
            acc += (u64)m4.x * col[0];
            acc += (u64)m4.y * col[PS];
            acc += (u64)m4.z * col[2 * PS];
            acc += (u64)m4.w * col[3 * PS];
        }
        const u32 v = red_b(acc, f.p, bar);
        const u32 pi = pinvr[t];
        bad |= (pi == 0 && v != 0);
        P[t * PS + c] = pi ? red_b((u64)v * pi, f.p, bar) : v;
    }
    return bad;
}

template <bool LAZY>
__global__ void __launch_bounds__(256, RL_BATCHED_CTAS) cup_batched_blk_kernel(
    u32* A, i64 stride, i32 m, i32 n, Fp f, Bar24 bar, i32* ranks, i32* rrp_out, i32* ipiv_out, i32 kcap,
    const u32* __restrict__ inv_tab) {
    extern __shared__ __align__(16) unsigned char smem_blk[];
    u32* P = reinterpret_cast<u32*>(smem_blk + OFF_P);        // [PR][BN] panel rows, reduced
    u32* s_fd = reinterpret_cast<u32*>(smem_blk + OFF_FD);    // [PR][SB] multipliers of the row block's pivots
    u32* wbuf = reinterpret_cast<u32*>(smem_blk + OFF_WBUF);  // [8][BN] per-warp row buffer
    __shared__ i32 s_rrp[BN], s_ipiv[BN], s_prow[PR];
    __shared__ u32 s_f[PR];
    __shared__ int s_wmin[8];
    __shared__ u32 s_pinv;
    __shared__ int s_fast[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u32* a = A + (i64)blockIdx.x * stride;
    const int nq = (n + 31) / 32;
    BT_DECL;
    const bool vec_ok = RL_BATCHED_VEC && (n & 3) == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0;
    int r = 0;
    for (int i0 = 0; i0 < m && r < n; i0 += PR) {
        const int pr = min(PR, m - i0);
        const int r0 = r;
        auto load_panel = [&]() {
            if (vec_ok) {  // 16-byte copies: a warp moves two rows per instruction
                const int n4 = n >> 2;
                for (int e = tid; e < pr * 64; e += 256) {
                    const int t = e >> 6, c4 = e & 63;
                    if (c4 < n4)
                        *reinterpret_cast<uint4*>(P + t * PS + 4 * c4) =
                            __ldcg(reinterpret_cast<const uint4*>(a + (i64)(i0 + t) * n) + c4);
                }
            } else {
                for (int t = warp; t < pr; t += 8)
                    for (int c = lane; c < n; c += 32) P[t * PS + c] = a[(i64)(i0 + t) * n + c];
            }
        };
        load_panel();
        __syncthreads();
        BT_MARK(0);
        // ---- fast panel (p < 2^24, pivots in generic position).  Warp 0 factors
        // the panel's 32-column window [r0, r0 + 32) alone, in registers (lane =
        // column, one register per row, no barrier on the pivot chain): row k's
        // pivot must be its first nonzero at window positions >= jr and sit at jr
        // exactly (no transposition); a row that is zero there is set aside as a
        // zero row.  Every other thread then finishes its own column right of the
        // window by one forward substitution against the multipliers warp 0 left
        // in shared memory (496 lazy products, one reduction per row) and checks
        // that the set-aside rows are zero there too.  Anything else (a pivot
        // outside the window, a transposition) reloads the panel and takes the
        // row-by-row loop below.  Same pivots, same values: each entry is the
        // same sum of products, grouped differently.
        bool fast_done = false;
        if (LAZY && RL_BATCHED_FAST) {
            u32* Lt = reinterpret_cast<u32*>(smem_blk + OFF_LT);  // [PR][LTS]: p - (C entry of row t for row k's pivot)
            u32* pinvr = Lt + PR * LTS;                           // [PR]: inverse of row k's pivot, 0 if it has none
            if (warp == 0) fast_window(P, Lt, pinvr, s_prow, s_fast, pr, r0, n, f, bar, inv_tab);
            BT_MARK(9);
            __syncthreads();
            BT_MARK(7);
            const int npf = s_fast[0];
            bool bad = s_fast[1] == 0;
            if (!bad && tid >= PR && r0 + tid < n) bad = fast_column(P, Lt, pinvr, pr, r0 + tid, f, bar);
            BT_MARK(8);
            if (__syncthreads_or(bad ? 1 : 0)) {  // not generic: start the panel over, row by row
                load_panel();
                __syncthreads();
            } else {
                fast_done = true;
                for (int j = tid; j < npf; j += 256) {
                    s_rrp[r0 + j] = i0 + s_prow[j];
                    s_ipiv[r0 + j] = r0 + j;
                }
                r = r0 + npf;
                __syncthreads();
            }
        }
        BT_MARK(6);
        if (!fast_done) {
        // ---- panel: rows in order, in row blocks of SB.  A pivot updates at once
        // only what the next steps read: its row block's remaining rows (every
        // thread its own column) and, for the rows below the row block, the SB
        // columns [bs_r, bs_r + SB) that hold this block's pivots -- the source of
        // the multipliers -- one entry per thread.  The other columns of the rows
        // below get the block's (at most SB) pivots in one pass when the block
        // ends (flush): one shared-memory round trip and one reduction per row
        // instead of one per pivot, the lazy 64-bit sum (< 2^49 for p < 2^24) in
        // a register, the normalised pivot entries of the own column in
        // registers, the multipliers in s_fd.  Same sums, grouped differently.
        int kb_end = min(SB, pr) - 1, bs_r = r, nb = 0;
        u32 ureg[SB];
#pragma unroll
        for (int j = 0; j < SB; ++j) ureg[j] = 0;
        auto flush = [&]() {
            const int c = tid;
            if (nb > 0 && c < n && c >= bs_r + SB) {
                for (int t = kb_end + 1; t < pr; ++t) {
                    u32 fm[SB];
#pragma unroll
                    for (int j4 = 0; j4 < SB; j4 += 4)
                        *reinterpret_cast<uint4*>(fm + j4) = *reinterpret_cast<const uint4*>(s_fd + t * SB + j4);
                    if (LAZY) {
                        u64 x = P[t * PS + c];
#pragma unroll
                        for (int j = 0; j < SB; ++j)
                            if (j < nb) x += (u64)fm[j] * ureg[j];
                        P[t * PS + c] = red_b(x, f.p, bar);
                    } else {
                        u32 x = P[t * PS + c];
#pragma unroll
                        for (int j = 0; j < SB; ++j)
                            if (j < nb) x = addmod(x, mulmod(fm[j], ureg[j], f), f);
                        P[t * PS + c] = x;
                    }
                }
            }
            nb = 0;
        };
        for (int k = 0; k < pr && r < n; ++k) {
            const int c = tid;
            if (k > kb_end) {  // next row block (barrier: row k's pivot columns were written by other threads)
                __syncthreads();
                flush();
                kb_end = min(kb_end + SB, pr - 1);
                bs_r = r;
                BT_MARK(10);
            }
            const u32 v = (c < n && c >= r) ? P[k * PS + c] : 0u;
            const unsigned msk = __ballot_sync(0xffffffffu, v != 0);
            if (lane == 0) s_wmin[warp] = msk ? warp * 32 + __ffs(msk) - 1 : BN;
            __syncthreads();
            int pc = r;
            if (P[k * PS + r] == 0) {  // (r < n) the usual case needs no scan
                pc = s_wmin[0];
#pragma unroll
                for (int w = 1; w < 8; ++w) pc = min(pc, s_wmin[w]);
            }
            BT_MARK(6);
            if (pc >= n) {  // no pivot: row k is zero at positions >= r
                __syncthreads();
                continue;
            }
            if (pc != r) {  // transposition r <-> pc on the panel rows and earlier U rows
                flush();    // column pc receives its pending pivots before it moves
                bs_r = r;
                __syncthreads();
                for (int t = tid; t < pr; t += 256) {
                    const u32 x = P[t * PS + r];
                    P[t * PS + r] = P[t * PS + pc];
                    P[t * PS + pc] = x;
                }
                for (int j = tid; j < r0; j += 256) {
                    u32* row = a + (i64)s_rrp[j] * n;
                    const u32 x = row[r];
                    row[r] = row[pc];
                    row[pc] = x;
                }
                __syncthreads();
            }
            u32 pinv;
            if (inv_tab) {  // p < 2^24: every thread loads the inverse (one cached word)
                pinv = __ldg(inv_tab + P[k * PS + r]);
            } else {        // one thread runs the extended Euclid
                if (tid == 0) s_pinv = inv_euclid(P[k * PS + r], f.p);
                __syncthreads();
                pinv = s_pinv;
            }
#ifdef RL_BATCHED_TRACE
            if (pinv == 0xffffffffu) bt_[11] = 1;  // (the load has returned)
#endif
            BT_MARK(7);
            // normalised U row
            u32 u = 0;
            if (c < n && c > r) {
                u = LAZY ? red_b((u64)P[k * PS + c] * pinv, f.p, bar) : mulmod(P[k * PS + c], pinv, f);
                P[k * PS + c] = u;
            }
            // multipliers of the panel rows below: column r holds the raw C entries
            if (tid > k && tid < pr) {
                const u32 fk = P[tid * PS + r];
                const u32 nfk = fk ? f.p - fk : 0u;
                s_f[tid] = nfk;
                if (tid > kb_end) s_fd[tid * SB + nb] = nfk;
            }
            if (tid == 0) {
                s_rrp[r] = i0 + k;
                s_ipiv[r] = pc;
                s_prow[r - r0] = k;
            }
            __syncthreads();
            BT_MARK(8);
            if (c < n && c > r) {
#pragma unroll
                for (int j = 0; j < SB; ++j)
                    if (j == nb) ureg[j] = u;
                for (int t = k + 1; t <= kb_end; ++t)
                    P[t * PS + c] = fma_red<LAZY>(P[t * PS + c], s_f[t], u, f, bar);
            }
            {   // the block's pivot columns on the rows below the row block
                const int t = kb_end + 1 + tid / SB, cc = bs_r + tid % SB;
                if (t < pr && cc > r && cc < n)
                    P[t * PS + cc] = fma_red<LAZY>(P[t * PS + cc], s_f[t], P[k * PS + cc], f, bar);
            }
            BT_MARK(9);
            ++nb;
            ++r;
            // no barrier: the next row's pivot search reads only this thread's
            // own column, and everything shared is written after the next barrier
        }
        BT_MARK(1);
        flush();
        __syncthreads();
        }  // !fast_done
        BT_MARK(1);
        // write the panel back (rows after the early return r == n keep their values)
        if (vec_ok) {
            const int n4 = n >> 2;
            for (int e = tid; e < pr * 64; e += 256) {
                const int t = e >> 6, c4 = e & 63;
                if (c4 < n4)
                    *(reinterpret_cast<uint4*>(a + (i64)(i0 + t) * n) + c4) =
                        *reinterpret_cast<const uint4*>(P + t * PS + 4 * c4);
            }
        } else {
            for (int t = warp; t < pr; t += 8)
                for (int c = lane; c < n; c += 32) a[(i64)(i0 + t) * n + c] = P[t * PS + c];
        }
        // the panel's unit upper pivot block U_pp (strict upper triangle, packed) is
        // put aside for trailing_dmma while the panel is still in shared memory
        const int np = r - r0;
        if (LAZY) {
            u32* Upk = reinterpret_cast<u32*>(smem_blk + OFF_UPK);
            for (int e = tid; e < PR * PR; e += 256) {
                const int k = e / PR, i = e % PR;
                if (k < i && i < np) Upk[upk_idx(k, i)] = P[s_prow[k] * PS + r0 + i];
            }
        }
        __syncthreads();
        BT_MARK(2);
        // ---- trailing rows
        bool any_swap = false;
        for (int j = r0; j < r; ++j) any_swap |= (s_ipiv[j] != j);
        // trailing_dmma stages at most UDS columns right of the pivot block (a
        // panel with fewer than PR - 8 pivots in a 256-column matrix has more)
        if (LAZY && np > 0 && !any_swap && n - r <= UDS) {
            trailing_dmma(a, m, n, f, i0, pr, r0, np, s_prow, smem_blk);
#ifdef RL_BATCHED_TRACE
            { const long long mid = g_bt_mid; bt_[3] += mid - bt_t; bt_t = mid; }
#endif
        } else if (np > 0) {  // one warp per row, pivot by pivot (transpositions, large p, wide panels)
            u32* wb = wbuf + warp * BN;
            for (int k = i0 + pr + warp; k < m; k += 8) {
                u32* row = a + (i64)k * n;
                for (int q = 0; q < nq; ++q) {
                    const int c = lane + 32 * q;
                    if (c < n) wb[c] = row[c];
                }
                __syncwarp();
                if (lane == 0)
                    for (int j = r0; j < r; ++j)
                        if (s_ipiv[j] != j) {
                            const u32 x = wb[j];
                            wb[j] = wb[s_ipiv[j]];
                            wb[s_ipiv[j]] = x;
                        }
                __syncwarp();
                u64 x[BN / 32];
#pragma unroll
                for (int q = 0; q < BN / 32; ++q) {
                    const int c = lane + 32 * q;
                    x[q] = (q < nq && c < n) ? wb[c] : 0u;
                }
                // pivots in column order; column cj = r0 + j lives in register block
                // Q = cj / 32 of lane cj % 32, so every index below is static
                int j = 0;
#pragma unroll
                for (int Q = 0; Q < BN / 32; ++Q) {
                    for (; j < np && ((r0 + j) >> 5) == Q; ++j) {
                        const int ll = (r0 + j) & 31;
                        const u32 fj = __shfl_sync(0xffffffffu, LAZY ? red64(x[Q], f) : (u32)x[Q], ll);
                        const u32 nf = fj ? f.p - fj : 0u;
                        const u32* U = P + s_prow[j] * PS;
                        if (lane == ll) x[Q] = fj;  // raw C entry
                        else if (lane > ll) x[Q] = lazy_fma<LAZY>(x[Q], nf, U[32 * Q + lane], f);
#pragma unroll
                        for (int q = Q + 1; q < BN / 32; ++q)
                            x[q] = lazy_fma<LAZY>(x[q], nf, U[32 * q + lane], f);
                    }
                }
#pragma unroll
                for (int q = 0; q < BN / 32; ++q) {
                    const int c = lane + 32 * q;
                    if (q < nq && c < n) row[c] = LAZY ? red64(x[q], f) : (u32)x[q];
                }
                __syncwarp();
            }
        }
        __syncthreads();
        BT_MARK(4);
    }
    if (tid == 0) ranks[blockIdx.x] = r;
    for (int j = tid; j < r; j += 256) {
        rrp_out[(i64)blockIdx.x * kcap + j] = s_rrp[j];
        ipiv_out[(i64)blockIdx.x * kcap + j] = s_ipiv[j];
    }
    __syncthreads();
    // place U rows: row j <- row rrp[j] on columns (j, n), zero-filling the source,
    // in increasing j for every column (factor.cpp:62-70 composed)
    for (int col = tid; col < n; col += 256) {
        for (int j = 0; j < r && j < col; ++j) {
            const i32 src = s_rrp[j];
            if (src == j) continue;
            a[(i64)j * n + col] = a[(i64)src * n + col];
            a[(i64)src * n + col] = 0;
        }
    }
#ifdef RL_BATCHED_TRACE
    __syncthreads();
    BT_MARK(5);
    if (tid == 0 && (blockIdx.x % 1024) == 700)
        printf("BT cta %d rank %d: load %lld panel %lld wb+upk %lld trail_setup %lld sweep %lld place %lld | "
               "pivot steps: search+bar1 %lld pinv %lld norm+mult+bar2 %lld update %lld blockflush %lld\n",
               blockIdx.x, r, bt_[0], bt_[1] + bt_[6] + bt_[7] + bt_[8] + bt_[9] + bt_[10], bt_[2], bt_[3], bt_[4],
               bt_[5], bt_[6], bt_[7], bt_[8], bt_[9], bt_[10]);
#endif
}

__global__ void inv_table_kernel(u32* tab, u32 p) {
    for (u32 x = blockIdx.x * blockDim.x + threadIdx.x; x < p; x += gridDim.x * blockDim.x)
        tab[x] = x ? inv_euclid(x, p) : 0u;
}

// x^{-1} mod p for every x < p (p < 2^24: at most 64 MB), built once per prime
// and device, so a pivot inverse on the batched kernel's serial chain is one
// cached load instead of an extended Euclid loop.  The build is synchronised
// once (a consumer on any other stream then sees a finished table), and at most
// kMaxTables tables live per process: a multi-modular caller cycling through
// primes evicts the least recently used one (after a device synchronisation,
// since an asynchronous batch may still read it).
const u32* inverse_table(u32 p, cudaStream_t s) {
    constexpr size_t kMaxTables = 4;
    struct Tab {
        u32* ptr;
        unsigned long long used;
    };
    static std::mutex mu;
    static std::map<std::pair<int, u32>, Tab> tabs;
    static unsigned long long tick = 0;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = tabs.find({dev, p});
    if (it != tabs.end()) {
        it->second.used = ++tick;
        return it->second.ptr;
    }
    if (tabs.size() >= kMaxTables) {
        auto victim = tabs.begin();
        for (auto j = tabs.begin(); j != tabs.end(); ++j)
            if (j->second.used < victim->second.used) victim = j;
        int cur = dev;
        RL_CUDA_CHECK(cudaSetDevice(victim->first.first));
        RL_CUDA_CHECK(cudaDeviceSynchronize());
        cudaFree(victim->second.ptr);
        RL_CUDA_CHECK(cudaSetDevice(cur));
        tabs.erase(victim);
    }
    u32* t = nullptr;
    if (cudaMalloc(&t, sizeof(u32) * p) != cudaSuccess) throw Error(8, "cudaMalloc failed");
    inv_table_kernel<<<4 * num_sms(), 256, 0, s>>>(t, p);
    RL_CUDA_CHECK(cudaGetLastError());
    RL_CUDA_CHECK(cudaStreamSynchronize(s));
    tabs.emplace(std::make_pair(dev, p), Tab{t, ++tick});
    return t;
}

}  // namespace

constexpr i64 kTableMinBatch = 64;

void cup_batched(u32* dA, i64 batch, i32 m, i32 n, i64 stride, u32 p, i32* d_ranks, i32* d_rrp,
                 i32* d_ipiv, i32 kcap, cudaStream_t s) {
    if (batch <= 0 || m <= 0 || n <= 0) return;
    // grid: one CTA per matrix (batch <= 2^31-1)
    const Fp f = make_fp(p);
    if (n <= BN) {
        const size_t smem = SMEM_BLK;
        static std::atomic<unsigned long long> attr_once{0};
        once_on_device(attr_once, [&] {
            RL_CUDA_CHECK(cudaFuncSetAttribute(cup_batched_blk_kernel<true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            RL_CUDA_CHECK(cudaFuncSetAttribute(cup_batched_blk_kernel<false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        });
        // the per-prime table pays off for real batches; a handful of matrices
        // take the in-kernel extended Euclid inverse (so does every p >= 2^24)
        if (p < (1u << 24))
            cup_batched_blk_kernel<true><<<(unsigned)batch, 256, smem, s>>>(
                dA, stride, m, n, f, make_bar24(p), d_ranks, d_rrp, d_ipiv, kcap,
                (batch >= kTableMinBatch && !RL_BATCHED_NOTAB) ? inverse_table(p, s) : nullptr);
        else
            cup_batched_blk_kernel<false><<<(unsigned)batch, 256, smem, s>>>(dA, stride, m, n, f, Bar24{0, 0, 0},
                                                                            d_ranks, d_rrp, d_ipiv, kcap, nullptr);
    } else {
        cup_batched_kernel<<<(unsigned)batch, 256, 0, s>>>(dA, stride, m, n, f, d_ranks, d_rrp, d_ipiv,
                                                           kcap);
    }
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
