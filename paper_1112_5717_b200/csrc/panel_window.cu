// panel_window.cu -- pivot discovery for one CUP leaf (the sequential critical
// path of the whole factorization).  See panel.cu for the leaf schedule.
//
// Reference semantics (proj/src/factor.cpp:12-28, 30-81): row i's pivot is the
// first nonzero at positions >= rank so far, swapped in by a transposition; the
// C entry C(k, j) is row k's value at pivot column j after eliminating pivots
// < j; U row j is the pivot row divided by its pivot beyond position j.
//
// Layout: the b x w window (w <= PW) plus a b x b identity block is held in
// registers as 64-bit LAZY accumulators; warp k%8 owns row k, lane l owns
// positions l + 32q (q < 4 window, q = 4, 5 identity).  Eliminating row k by
// pivot j (pivot row U_j unnormalised, inverse pinv_j) adds mult * U_j[x] with
// mult = -C(k,j) * pinv_j to every position (positions <= j become stale: C
// entries are kept exactly in s_C), so a step is one 64-bit multiply-add per
// element; only C(k,j) and the searched row are reduced mod p.  The C entries
// of a warp's 8 rows are gathered by shuffles and turned into multipliers by 8
// lanes in parallel.  Inverses: a shared-memory table for p < 2^16, Fermat
// otherwise.  Lockstep with lookahead: in step i the owner of row i+1 first
// applies pivot i to it, reduces and searches it (warp ballot) and publishes
// pivot i+1, then every warp updates its remaining rows; one CTA barrier per
// row.  The identity block yields the row transform Minv: V = Minv * P gives
// the U rows (pivot rows) and residuals (window-dead rows) of ANY column.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"
#include "uinv.cuh"

namespace rl {

LT_TABLE(window)

namespace {

// The lookahead warp runs alone on its SM sub-partition during the rank-8
// update (measured: window LU 21.7 -> 20.1 us, C3 21.66 -> 21.38 ms).
#ifndef RL_LA_ISOLATE
#define RL_LA_ISOLATE 1
#endif

// The leaf's U^{-1} computed at the end of the window kernel for a full
// speculative leaf (1) or only by the parallel U^{-1} kernel (0).  Measured: the
// leaf-pair transition drops 22.1 -> 17.4 us, but the window grows 27 -> 35 us
// (the doubling levels on CUDA cores): C3 21.45 vs 20.15 ms, so off.
#ifndef RL_WIN_UINV
#define RL_WIN_UINV 0
#endif

// row pitch (words) of the staged window: WT = 192 would put every row of a
// column in the same shared-memory bank
constexpr int RP = WT + 4;

constexpr unsigned FULL = 0xffffffffu;

template <class T>
__device__ __forceinline__ T sel4(const T (&v)[6], int q) {
    T t = v[0];
    t = (q == 1) ? v[1] : t;
    t = (q == 2) ? v[2] : t;
    t = (q == 3) ? v[3] : t;
    return t;
}
template <class T>
__device__ __forceinline__ void put4(T (&v)[6], int x, T val, int lane) {
    if (lane == (x & 31)) {
        const int q = x >> 5;
        v[0] = (q == 0) ? val : v[0];
        v[1] = (q == 1) ? val : v[1];
        v[2] = (q == 2) ? val : v[2];
        v[3] = (q == 3) ? val : v[3];
    }
}
__device__ __forceinline__ u64 shfl64(u64 v, int src) {
    const u32 lo = __shfl_sync(FULL, (u32)v, src);
    const u32 hi = __shfl_sync(FULL, (u32)(v >> 32), src);
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u64 get64(const u64 (&v)[6], int x) { return shfl64(sel4(v, x >> 5), x & 31); }
__device__ __forceinline__ u32 get32(const u32 (&v)[6], int x) {
    return __shfl_sync(FULL, sel4(v, x >> 5), x & 31);
}
__device__ __forceinline__ void swap64(u64 (&v)[6], int x, int y, int lane) {
    const u64 vx = get64(v, x), vy = get64(v, y);
    put4(v, x, vy, lane);
    put4(v, y, vx, lane);
}
__device__ __forceinline__ void swap32(u32 (&v)[6], int x, int y, int lane) {
    const u32 vx = get32(v, x), vy = get32(v, y);
    put4(v, x, vy, lane);
    put4(v, y, vx, lane);
}

template <bool SP>
__device__ __forceinline__ void axpy_row(u64 (&acc)[6], u32 mult, const u32 (&U)[6], const Fp& f) {
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        if (SP) acc[q] += (u64)mult * U[q];
        else acc[q] = red64(acc[q] + (u64)mult * U[q], f);
    }
}

struct WinShared {
    u32* s_R;            // [PB][WT] row values at search time (reduced)
    const uint16_t* s_inv;
    u32 (*s_C)[PB + 1];  // exact C entries C(k, j)
    int* s_c;            // [2] pivot column of the last searched row (-1: dead)
    u32* s_pinv;         // [2] its inverse
    u32* s_pv;           // [PB] pivot values
    u32* s_pinvA;        // [PB] their inverses
};

// Reduce row k, find its pivot (first nonzero window position >= rn), publish.
template <bool SP>
__device__ __forceinline__ void search_publish(const u64 (&acc)[6], int k, int rn, int w,
                                               const WinShared& S, int lane, const Fp& f) {
    u32 vals[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) vals[q] = SP ? red_sp(acc[q], f) : red64(acc[q], f);
    int c = -1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int x = lane + 32 * q;
        const unsigned msk = __ballot_sync(FULL, x >= rn && x < w && vals[q] != 0);
        if (c < 0 && msk) c = 32 * q + __ffs(msk) - 1;
    }
    u32 pinv = 0;
    if (c >= 0) {
        if (c != rn) swap32(vals, rn, c, lane);
        const u32 pv = get32(vals, rn);
        pinv = SP ? (u32)S.s_inv[pv] : invmod(pv, f);
        if (lane == 0) {
            S.s_pv[rn] = pv;
            S.s_pinvA[rn] = pinv;
        }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) S.s_R[k * RP + lane + 32 * q] = vals[q];
    if (lane == 0) {
        S.s_c[k & 1] = c;
        S.s_pinv[k & 1] = pinv;
    }
}

// Row inext: apply pivot (r, c, pinv, U) if any, then search and publish.
template <bool SP>
__device__ __forceinline__ void prio_step(u64 (&acc)[6], int k, bool piv, int r, int c, u32 pinv,
                                          const u32 (&U)[6], int rn, int w, const WinShared& S,
                                          int lane, const Fp& f) {
    if (piv) {
        if (c != r) swap64(acc, r, c, lane);
        const u64 ckr = get64(acc, r);
        const u32 ck = SP ? red_sp(ckr, f) : red64(ckr, f);
        if (lane == 0) S.s_C[k][r] = ck;
        const u32 mult = ck ? f.p - mulmod(ck, pinv, f) : 0u;
        axpy_row<SP>(acc, mult, U, f);
    }
    search_publish<SP>(acc, k, rn, w, S, lane, f);
}

constexpr int NW = 16;      // warps
constexpr int RW = PB / NW; // rows per warp (row k -> warp k % NW, slot k / NW)
constexpr int LB = 8;       // leaf block of the speculative LU

// (p - m) * u summed lazily: acc + (p - m) * u
template <bool SP>
__device__ __forceinline__ u64 fms(u64 acc, u32 m, u32 u, const Fp& f) {
    const u32 nm = m ? f.p - m : 0u;
    if (SP) return acc + (u64)nm * u;
    return acc + mulmod(nm, u, f);
}
// acc + nm * u (nm already negated)
template <bool SP>
__device__ __forceinline__ u64 fmsn(u64 acc, u32 nm, u32 u, const Fp& f) {
    if (SP) return acc + (u64)nm * u;
    return acc + mulmod(nm, u, f);
}
template <bool SP>
__device__ __forceinline__ u32 fred(u64 x, const Fp& f) {
    return SP ? red_sp(x, f) : red64(x, f);
}

// One warp factors the bt x bt diagonal block at rows/columns r0.. of s_R
// (element (k, c): lane (k&3)*8 + c holds v0 for k < 4 and v1 for k >= 4, the
// block's current values), writes back the block (U part reduced, C part raw),
// the negated multipliers s_M and the pivots; fail = 1 on a zero pivot.
template <bool SP>
__device__ __forceinline__ void diag_factor(u32* s_R, u32 (*s_C)[PB + 1], u32* s_pv, u32* s_pinvA,
                                            const uint16_t* s_inv, u32 (*s_M)[LB], int* s_fail,
                                            int r0, int bt, u32 v0, u32 v1, int lane, const Fp& f) {
    // fully unrolled (shuffle sources are constants); the whole warp takes the
    // same branch at every step, so a zero pivot stops it uniformly
    const int cc = lane & 7, k0 = lane >> 3, k1 = k0 + 4;
    int fail = 0;
#pragma unroll
    for (int j = 0; j < LB; ++j) {
        if (j < bt && !fail) {
            const u32 pv = __shfl_sync(FULL, j < 4 ? v0 : v1, (j & 3) * 8 + j);
            const u32 c0v = __shfl_sync(FULL, v0, k0 * 8 + j);          // C(k0, j)
            const u32 c1v = __shfl_sync(FULL, v1, (k1 - 4) * 8 + j);    // C(k1, j)
            const u32 uj = __shfl_sync(FULL, j < 4 ? v0 : v1, (j & 3) * 8 + cc);
            if (pv == 0) {
                fail = 1;
            } else {
                const u32 pinv = SP ? (u32)s_inv[pv] : invmod(pv, f);
                const u32 m0 = mulmod_t<SP>(c0v, pinv, f), m1 = mulmod_t<SP>(c1v, pinv, f);
                if (cc == j) {  // this lane holds C(k, j) for its rows
                    if (k0 > j && k0 < bt) s_M[r0 + k0][j] = m0 ? f.p - m0 : 0u;
                    if (k1 > j && k1 < bt) s_M[r0 + k1][j] = m1 ? f.p - m1 : 0u;
                }
                if (k0 > j && cc > j) v0 = submod(v0, mulmod_t<SP>(m0, uj, f), f);
                if (k1 > j && cc > j) v1 = submod(v1, mulmod_t<SP>(m1, uj, f), f);
                if (lane == 0) {
                    s_pv[r0 + j] = pv;
                    s_pinvA[r0 + j] = pinv;
                }
            }
        }
    }
    if (k0 < bt && cc < bt) {
        s_R[(r0 + k0) * RP + r0 + cc] = v0;
        if (cc < k0) s_C[r0 + k0][r0 + cc] = v0;
    }
    if (k1 < bt && cc < bt) {
        s_R[(r0 + k1) * RP + r0 + cc] = v1;
        if (cc < k1) s_C[r0 + k1][r0 + cc] = v1;
    }
    if (lane == 0) *s_fail = fail;
}

// Same contract as diag_factor, fraction-free: step j replaces row k by
// pv_j * row_k - R_k[j] * row_j (pv_j the current, scaled pivot), so no inverse
// sits on the serial chain (shuffle -> two independent products -> subtract).
// Row k then carries the scale S_k = pv_0 ... pv_{k-1} and its entry at column
// j < k the scale S_j; with T_j = S_j^{-1} the true values follow once per
// block, off the chain: U part R * T_k, C part R * T_j, negated multiplier
// -R_k[j] * pv_j^{-1} (the scales of rows j and k agree at step j), pivot
// pv_j * T_j and its inverse pv_j^{-1} * S_j.  A zero scaled pivot is a zero
// true pivot (the scales are products of nonzero pivots).
template <bool SP>
__device__ __forceinline__ void diag_factor_ff(u32* s_R, u32 (*s_C)[PB + 1], u32* s_pv, u32* s_pinvA,
                                               const uint16_t* s_inv, u32 (*s_M)[LB], int* s_fail,
                                               int r0, int bt, u32 v0, u32 v1, int lane, const Fp& f) {
    const int cc = lane & 7, k0 = lane >> 3, k1 = k0 + 4;
    int fail = 0;
    u32 pvs[LB];
    u32 S[LB + 1];
    S[0] = 1u % f.p;
    // branch-free: every lane runs every step, updates are selected
#pragma unroll
    for (int j = 0; j < LB; ++j) {
        const u32 pv = __shfl_sync(FULL, j < 4 ? v0 : v1, (j & 3) * 8 + j);
        const u32 c0v = __shfl_sync(FULL, v0, k0 * 8 + j);          // R(k0, j)
        const u32 c1v = __shfl_sync(FULL, v1, (k1 - 4) * 8 + j);    // R(k1, j)
        const u32 uj = __shfl_sync(FULL, j < 4 ? v0 : v1, (j & 3) * 8 + cc);
        const bool live = j < bt;
        fail |= (live && pv == 0) ? 1 : 0;
        const u32 n0 = submod(mulmod_t<SP>(pv, v0, f), mulmod_t<SP>(c0v, uj, f), f);
        const u32 n1 = submod(mulmod_t<SP>(pv, v1, f), mulmod_t<SP>(c1v, uj, f), f);
        const bool up = live && cc > j;
        v0 = (up && k0 > j) ? n0 : v0;
        v1 = (up && k1 > j) ? n1 : v1;
        pvs[j] = live ? pv : 1u % f.p;
        S[j + 1] = live ? mulmod_t<SP>(S[j], pv, f) : S[j];
    }
    if (lane == 0) *s_fail = fail;
    if (fail) return;  // uniform: the caller abandons the speculative path
    // one inverse per block row (table lookups / Fermat, in parallel), then
    // shuffles: lane j < bt holds pv_j^{-1} and T_j = S_j^{-1}
    u32 my_ipv = 0, my_T = 0;
    if (lane < bt) {
        u32 pvl = pvs[0], Sl = S[0];
#pragma unroll
        for (int j = 1; j < LB; ++j)
            if (lane == j) {
                pvl = pvs[j];
                Sl = S[j];
            }
        my_ipv = SP ? (u32)s_inv[pvl] : invmod(pvl, f);
        my_T = SP ? (u32)s_inv[Sl] : invmod(Sl, f);
        s_pv[r0 + lane] = mulmod_t<SP>(pvl, my_T, f);
        s_pinvA[r0 + lane] = mulmod_t<SP>(my_ipv, Sl, f);
    }
    const u32 T_k0 = __shfl_sync(FULL, my_T, k0), T_k1 = __shfl_sync(FULL, my_T, k1);
    const u32 T_c = __shfl_sync(FULL, my_T, cc), ipv_c = __shfl_sync(FULL, my_ipv, cc);
    if (k0 < bt && cc < bt) {
        if (cc < k0) {
            const u32 m = mulmod_t<SP>(v0, ipv_c, f);
            s_M[r0 + k0][cc] = m ? f.p - m : 0u;
            v0 = mulmod_t<SP>(v0, T_c, f);
            s_C[r0 + k0][r0 + cc] = v0;
        } else {
            v0 = mulmod_t<SP>(v0, T_k0, f);
        }
        s_R[(r0 + k0) * RP + r0 + cc] = v0;
    }
    if (k1 < bt && cc < bt) {
        if (cc < k1) {
            const u32 m = mulmod_t<SP>(v1, ipv_c, f);
            s_M[r0 + k1][cc] = m ? f.p - m : 0u;
            v1 = mulmod_t<SP>(v1, T_c, f);
            s_C[r0 + k1][r0 + cc] = v1;
        } else {
            v1 = mulmod_t<SP>(v1, T_k1, f);
        }
        s_R[(r0 + k1) * RP + r0 + cc] = v1;
    }
}

// Speculative pivot discovery for GENERIC leaves: blocked right-looking LU of
// the window without pivoting, in shared memory (s_R = [window | identity],
// reduced values).  If every diagonal value is nonzero, row i's first nonzero
// at positions >= i is position i itself, so this IS the CUP of the leaf
// (rrp = identity, no transpositions).  Per 8-row block: the block rows' right
// part is a column-parallel forward substitution, the rows below get their C
// entries by a row-parallel triangular solve, then a rank-8 lazy update -- during
// which the last warp already updates and factors the NEXT diagonal block (lookahead),
// so the serial 8 x 8 factorization is off the critical path.  Returns false
// (uniformly) on the first zero pivot; the caller then runs the exact path.
#ifdef RL_TRACE
__device__ unsigned long long g_wst[8][6];  // per 8-row block: start, (b)(c) done, lookahead done, end
#define WST(blk, k) do { if ((blk) < 8) g_wst[(blk)][(k)] = rl_now(); } while (0)
#define WCLK(var) const long long var = clock64()
#define WCYC(blk, k, v) do { if ((blk) < 8) g_wst[(blk)][(k)] = (unsigned long long)(v); } while (0)
#else
#define WST(blk, k)
#define WCLK(var)
#define WCYC(blk, k, v)
#endif
template <bool SP>
__device__ bool spec_lu(u32* s_R, u32 (*s_C)[PB + 1], u32* s_pv, u32* s_pinvA,
                        const uint16_t* s_inv, u32 (*s_M2)[PB][LB], int* s_fail, int b, int w,
                        const Fp& f) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (w < b) return false;
    // multipliers double-buffered by block parity: warp 0 writes the next block's
    // while the other warps still read the current block's
    {
        u32 (*s_M)[LB] = s_M2[0];
        const int cc = lane & 7, k0 = lane >> 3, k1 = k0 + 4, bt = min(LB, b);
        if (warp == NW - 1) {
            const u32 v0 = (k0 < bt && cc < bt) ? s_R[k0 * RP + cc] : 0u;
            const u32 v1 = (k1 < bt && cc < bt) ? s_R[k1 * RP + cc] : 0u;
            diag_factor_ff<SP>(s_R, s_C, s_pv, s_pinvA, s_inv, s_M, s_fail, 0, bt, v0, v1, lane, f);
        }
        __syncthreads();
    }
    for (int r0 = 0; r0 < b; r0 += LB) {
        if (*s_fail) return false;
        if (tid == 0) WST(r0 / LB, 0);
        u32 (*s_M)[LB] = s_M2[(r0 / LB) & 1];
        u32 (*s_Mn)[LB] = s_M2[((r0 / LB) + 1) & 1];
        const int bt = min(LB, b - r0);
        const int x0 = r0 + bt;  // first column right of the block
        // Columns still needed: the rest of the pivot block [x0, b) and the identity
        // block's first x0 columns [PW, PW + x0) -- its columns c >= x0 are still e_c
        // and the block rows are zero there, so no update touches them; window
        // columns >= b hold no pivot on this path (the tail kernel computes them as
        // V = Minv * P).
        const int Xw = max(0, b - x0);
        const int X = Xw + x0;
        const int R = b - x0;  // rows below the block
        if (tid < X) {
            // (b) block rows, column x: forward substitution down the block
            const int x = tid < Xw ? x0 + tid : PW + (tid - Xw);
            u32 col[LB];
#pragma unroll
            for (int k = 0; k < LB; ++k) {
                if (k < bt) {
                    u64 acc = s_R[(r0 + k) * RP + x];
#pragma unroll
                    for (int j = 0; j < k; ++j) acc = fmsn<SP>(acc, s_M[r0 + k][j], col[j], f);
                    col[k] = fred<SP>(acc, f);
                    s_R[(r0 + k) * RP + x] = col[k];
                }
            }
        } else if (tid >= 256 && tid - 256 < R) {
            // (c) rows below: C entries against the block and their multipliers
            const int k = x0 + tid - 256;
            u32 nm[LB];
#pragma unroll
            for (int j = 0; j < LB; ++j) {
                u64 acc = s_R[k * RP + r0 + j];
#pragma unroll
                for (int j2 = 0; j2 < j; ++j2) acc = fmsn<SP>(acc, nm[j2], s_R[(r0 + j2) * RP + r0 + j], f);
                const u32 cv = fred<SP>(acc, f);
                s_C[k][r0 + j] = cv;
                const u32 m = mulmod_t<SP>(cv, s_pinvA[r0 + j], f);
                nm[j] = m ? f.p - m : 0u;
            }
            uint4* dst = reinterpret_cast<uint4*>(&s_M[k][0]);
            dst[0] = make_uint4(nm[0], nm[1], nm[2], nm[3]);
            dst[1] = make_uint4(nm[4], nm[5], nm[6], nm[7]);
        }
        __syncthreads();
        if (tid == 0) WST(r0 / LB, 1);
        WCLK(cb0);
        if (R > 0) {
            const int nbt = min(LB, R);  // next diagonal block: rows/cols [x0, x0 + nbt)
            // The serial lookahead runs on the HIGHEST warp id: the SMSP arbiter
            // prefers high warp ids, so this latency-bound chain is not starved by
            // the rank-8 update sharing its scheduler.
            if (warp == NW - 1) {
                // lookahead: rank-8 update of the next diagonal block, then factor it
                const int cc = lane & 7, k0 = lane >> 3, k1 = k0 + 4;
                u32 v0 = 0, v1 = 0;
                if (k0 < nbt && cc < nbt) {
                    const uint4* mr = reinterpret_cast<const uint4*>(&s_M[x0 + k0][0]);
                    const uint4 m0 = mr[0], m1 = mr[1];
                    const u32 nmv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
                    u64 acc = s_R[(x0 + k0) * RP + x0 + cc];
#pragma unroll
                    for (int j = 0; j < LB; ++j) acc = fmsn<SP>(acc, nmv[j], s_R[(r0 + j) * RP + x0 + cc], f);
                    v0 = fred<SP>(acc, f);
                }
                if (k1 < nbt && cc < nbt) {
                    const uint4* mr = reinterpret_cast<const uint4*>(&s_M[x0 + k1][0]);
                    const uint4 m0 = mr[0], m1 = mr[1];
                    const u32 nmv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
                    u64 acc = s_R[(x0 + k1) * RP + x0 + cc];
#pragma unroll
                    for (int j = 0; j < LB; ++j) acc = fmsn<SP>(acc, nmv[j], s_R[(r0 + j) * RP + x0 + cc], f);
                    v1 = fred<SP>(acc, f);
                }
                WCLK(cl1);
                if (lane == 0) WCYC(r0 / LB, 4, cl1 - cb0);
                diag_factor_ff<SP>(s_R, s_C, s_pv, s_pinvA, s_inv, s_Mn, s_fail, x0, nbt, v0, v1, lane, f);
                WCLK(cl2);
                if (lane == 0) WCYC(r0 / LB, 2, cl2 - cb0);
            } else {
                // (d) rank-8 update of the rows below (a block with rows below is
                // full: bt == LB), except the next diagonal block (the last warp's)
                // Thread = a column PAIR (x, x + 1) (window part [x0, b), identity
                // part [PW, PW + x0)) and rows x0 + g (mod G): 8-byte shared loads and
                // stores, two independent multiply-add chains per row.
#if RL_LA_ISOLATE
                // the lookahead warp (NW - 1) alone on its SM sub-partition: the
                // warps sharing it (warp % 4 == 3) sit the update out
                const bool d_on = (warp & 3) != 3;
                const int n2 = (NW - NW / 4) * 32;
                const int t2 = d_on ? (warp - (warp >> 2)) * 32 + lane : 1 << 30;  // off: no iteration
#else
                const int t2 = tid, n2 = blockDim.x - 32;
#endif
                const int Xw2 = (Xw + 1) >> 1;
                const int X2 = Xw2 + x0 / 2;  // x0 is a multiple of LB here (R > 0)
                const int G = max(1, n2 / X2);
                const int xd = x0 + nbt;  // diagonal-block columns/rows end
                for (int e = t2; e < X2 * G; e += n2) {
                    const int ex = e % X2, g = e / X2;
                    const int x = ex < Xw2 ? x0 + 2 * ex : PW + 2 * (ex - Xw2);
                    const bool two = ex >= Xw2 || x + 1 < b;
                    const bool d0 = x < xd, d1 = x + 1 < xd;
                    u32 ua[LB], ub[LB];
#pragma unroll
                    for (int j = 0; j < LB; ++j) {
                        const uint2 uu = *reinterpret_cast<const uint2*>(&s_R[(r0 + j) * RP + x]);
                        ua[j] = uu.x;
                        ub[j] = uu.y;
                    }
                    for (int k = x0 + g; k < b; k += G) {
                        const bool s0 = d0 && k < xd, s1 = !two || (d1 && k < xd);
                        if (s0 && s1) continue;
                        const uint4* mrow = reinterpret_cast<const uint4*>(&s_M[k][0]);
                        const uint4 m0 = mrow[0], m1 = mrow[1];
                        const uint2 rv = *reinterpret_cast<const uint2*>(&s_R[k * RP + x]);
                        u64 a0 = rv.x, a1 = rv.y;
                        a0 = fmsn<SP>(a0, m0.x, ua[0], f);
                        a1 = fmsn<SP>(a1, m0.x, ub[0], f);
                        a0 = fmsn<SP>(a0, m0.y, ua[1], f);
                        a1 = fmsn<SP>(a1, m0.y, ub[1], f);
                        a0 = fmsn<SP>(a0, m0.z, ua[2], f);
                        a1 = fmsn<SP>(a1, m0.z, ub[2], f);
                        a0 = fmsn<SP>(a0, m0.w, ua[3], f);
                        a1 = fmsn<SP>(a1, m0.w, ub[3], f);
                        a0 = fmsn<SP>(a0, m1.x, ua[4], f);
                        a1 = fmsn<SP>(a1, m1.x, ub[4], f);
                        a0 = fmsn<SP>(a0, m1.y, ua[5], f);
                        a1 = fmsn<SP>(a1, m1.y, ub[5], f);
                        a0 = fmsn<SP>(a0, m1.z, ua[6], f);
                        a1 = fmsn<SP>(a1, m1.z, ub[6], f);
                        a0 = fmsn<SP>(a0, m1.w, ua[7], f);
                        a1 = fmsn<SP>(a1, m1.w, ub[7], f);
                        const u32 v0 = fred<SP>(a0, f), v1 = fred<SP>(a1, f);
                        if (!s0 && !s1) {
                            *reinterpret_cast<uint2*>(&s_R[k * RP + x]) = make_uint2(v0, v1);
                        } else if (!s0) {
                            s_R[k * RP + x] = v0;
                        } else {
                            s_R[k * RP + x + 1] = v1;
                        }
                    }
                }
                WCLK(cd);
                if (tid == 0) WCYC(r0 / LB, 5, cd - cb0);
            }
        }
        __syncthreads();
        if (tid == 0) WST(r0 / LB, 3);
    }
    return true;
}

template <bool SP>
__global__ void __launch_bounds__(NW * 32, 1) panel_window_kernel(PanelArgs a) {
    extern __shared__ __align__(16) uint8_t dsm[];
    __shared__ u32 s_C[PB][PB + 1];
    __shared__ i32 s_pos[PB], s_rrp[PB], s_rb[PB], s_por[PB];
    __shared__ i32 s_perm[PB], s_iperm[PB];  // speculative order: live rows first
    __shared__ unsigned long long s_deadw;
    __shared__ int s_live;
    __shared__ u32 s_pv[PB], s_pinvA[PB];
    __shared__ i32 s_sig[PW];
    __shared__ int s_c[2];
    __shared__ u32 s_pinv[2];
    __shared__ __align__(16) u32 s_M[2][PB][LB];
    __shared__ int s_fail;
    WinShared S;
    S.s_R = reinterpret_cast<u32*>(dsm);
    S.s_inv = reinterpret_cast<const uint16_t*>(dsm + PB * RP * 4);
    S.s_C = s_C;
    S.s_c = s_c;
    S.s_pinv = s_pinv;
    S.s_pv = s_pv;
    S.s_pinvA = s_pinvA;
    RL_STAMP(t_enter);
    u32* s_R = S.s_R;
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // the inverse table is static: start its copy before waiting for the
    // previous kernel (programmatic dependent launch)
    if (SP) {  // 128 KB inverse table
        const uint4* src = reinterpret_cast<const uint4*>(a.inv_table);
        uint4* dst = reinterpret_cast<uint4*>(dsm + PB * RP * 4);
#pragma unroll 4
        for (int e = tid; e < 65536 * 2 / 16; e += blockDim.x) cp_async16(dst + e, src + e);
    }
    pdl_wait();
    LT_BEGIN();
    const i32 c0 = __ldcg(a.rp + a.i0);
    const i32 W = a.N - c0;
    const int b = a.b;
    if (tid == 0) {
        ps->flag = 0;
        ps->counter = 0;
        ps->uinv_by_window = 0;
        ps->c0 = c0;
        ps->b = b;
        ps->W = W > 0 ? W : 0;
    }
    if (W <= 0) {  // rank already n: the rows keep their C data (factor.cpp:47)
        for (int i = tid; i < b; i += blockDim.x) a.rp[a.i0 + 1 + i] = c0;
        if (tid == 0) {
            *a.swapflag = 0;
            ps->w = 0;
            ps->r = 0;
            ps->spec = 0;
            ps->dead_mask = 0;
        }
        cp_async_wait_all();
        return;
    }
    const int w = W < PW ? W : PW;
    u64 acc[RW][6];
#pragma unroll
    for (int s = 0; s < RW; ++s) {
        const int k = warp + NW * s;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int x = lane + 32 * q;
            u32 val = 0;
            if (k < b && x < w) val = __ldcg(a.A + (i64)(a.i0 + k) * a.lda + c0 + x);
            acc[s][q] = val;
        }
        acc[s][4] = (lane == k) ? 1u : 0u;
        acc[s][5] = (lane + 32 == k) ? 1u : 0u;
    }
    // Rows that are zero across the whole window as loaded (e.g. zero rows of a
    // rank-deficient input: row operations keep them zero) have no pivot in it:
    // the speculative LU runs on the other rows only, in order ("live" rows
    // first), so such leaves stay on the fast path.  Whether those rows are also
    // zero beyond the window is checked by the tail (fallback otherwise).
    if (tid == 0) s_deadw = 0;
    __syncthreads();
#pragma unroll
    for (int s = 0; s < RW; ++s) {
        const int k = warp + NW * s;
        const bool nz = __any_sync(FULL, acc[s][0] | acc[s][1] | acc[s][2] | acc[s][3]);
        if (lane == 0 && k < b && !nz) atomicOr(&s_deadw, 1ull << k);
    }
    __syncthreads();
    const u64 deadw = s_deadw;
    if (tid < PB) {
        const int k = tid;
        const u64 below = deadw & ((1ull << k) - 1);
        const int live_before = k - __popcll(below);
        const int nlive = b - __popcll(deadw & (b >= 64 ? ~0ull : ((1ull << b) - 1)));
        if (k < b) {
            const bool dk = (deadw >> k) & 1;
            const int pos = dk ? nlive + (k - live_before) : live_before;
            s_perm[pos] = k;
            s_iperm[k] = pos;
        }
        if (k == 0) s_live = nlive;
    }
    __syncthreads();
    const int bl = s_live;
    // stage [window | identity] in that order for the speculative path
#pragma unroll
    for (int s = 0; s < RW; ++s) {
        const int k = warp + NW * s;
        if (k < b) {
            const int kp = s_iperm[k];
#pragma unroll
            for (int q = 0; q < 4; ++q) s_R[kp * RP + lane + 32 * q] = (u32)acc[s][q];
            s_R[kp * RP + PW + lane] = (lane == kp) ? 1u : 0u;
            s_R[kp * RP + PW + 32 + lane] = (lane + 32 == kp) ? 1u : 0u;
        }
    }
    cp_async_wait_all();
    __syncthreads();
#ifdef RL_TRACE
    // solo timing of the lookahead's diagonal factorization (all other warps at
    // the barrier): the same 8 x 8 block the first lookahead factors
    unsigned long long solo = 0;
    if (a.i0 == RL_TRACE_I0) {
        if (warp == NW - 1) {
            const int cc = lane & 7, k0 = lane >> 3, k1 = k0 + 4;
            const u32 v0 = s_R[k0 * RP + cc], v1 = s_R[k1 * RP + cc];
            __syncwarp();
            const long long c0 = clock64();
            diag_factor_ff<SP>(s_R, s_C, s_pv, s_pinvA, S.s_inv, s_M[1], &s_fail, 0, 8, v0, v1, lane, f);
            __syncwarp();
            solo = clock64() - c0;
            // restore the staged block and the flag
            s_R[k0 * RP + cc] = v0;
            s_R[k1 * RP + cc] = v1;
            if (lane == 0) { s_fail = 0; g_wst[7][4] = solo; }
        }
        __syncthreads();
    }
#endif
    RL_STAMP(t_loaded);
    LT_MARK(a.i0 / PB, 2);
    const bool spec = spec_lu<SP>(s_R, s_C, s_pv, s_pinvA, S.s_inv, s_M, &s_fail, bl, w, f);
    RL_STAMP(t_lu);
    int r = 0;
    if (spec) {
        r = bl;
        for (int e = tid; e < b; e += blockDim.x) {
            const int kp = s_iperm[e];
            const bool dk = kp >= bl;
            s_pos[e] = e;                       // no transposition
            if (e < bl) s_rrp[e] = s_perm[e];   // pivot e is the e-th live row
            s_rb[e] = 0;                        // set below
            s_por[e] = dk ? -1 : kp;
        }
        __syncthreads();
        for (int e = tid; e < b; e += blockDim.x)  // rank before row e = live rows before it
            s_rb[e] = e - __popcll(deadw & ((1ull << e) - 1));
        if (deadw) {  // a window-dead row may hold a pivot beyond the window: the
                      // tail's fallback then needs the original window
#pragma unroll
            for (int s2 = 0; s2 < RW; ++s2) {
                const int k = warp + NW * s2;
                if (k < b) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) ps->win_orig[k][lane + 32 * q] = (u32)acc[s2][q];
                }
            }
        }
        __syncthreads();
    } else {
    // exact lockstep path (any pivot structure): registers still hold the window.
    // Only here can a window-dead row appear, so only here is the original window
    // saved for the tail kernel's fallback restore.
#pragma unroll
    for (int s = 0; s < RW; ++s) {
        const int k = warp + NW * s;
        if (k < b) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ps->win_orig[k][lane + 32 * q] = (u32)acc[s][q];
        }
    }
    if (warp == 0) search_publish<SP>(acc[0], 0, 0, w, S, lane, f);
    __syncthreads();
    for (int i = 0; i < b; ++i) {
        const int c = s_c[i & 1];
        const u32 pinv = s_pinv[i & 1];
        const bool piv = c >= 0;
        if (tid == 0) {
            s_rb[i] = r;
            s_por[i] = piv ? r : -1;
            if (piv) {
                s_pos[r] = c;
                s_rrp[r] = i;
            }
        }
        u32 U[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) U[q] = piv ? s_R[i * RP + lane + 32 * q] : 0u;
        const int inext = i + 1;
        const int rn = r + (piv ? 1 : 0);
        if (inext < b && warp == (inext % NW)) {  // lookahead: row i+1 first
            switch (inext / NW) {
#define RL_PRIO(S_)                                                                 \
    case S_:                                                                       \
        prio_step<SP>(acc[S_], inext, piv, r, c, pinv, U, rn, w, S, lane, f);     \
        break;
                RL_PRIO(0) RL_PRIO(1) RL_PRIO(2) RL_PRIO(3)
#undef RL_PRIO
            }
        }
        if (piv && warp + NW * (RW - 1) > inext) {
            // the other rows of this warp (k = warp + NW*s > i+1), branch-free:
            // ineligible rows get a zero multiplier.
            if (c != r) {
#pragma unroll
                for (int s = 0; s < RW; ++s) {
                    const int k = warp + NW * s;
                    if (k > inext && k < b) swap64(acc[s], r, c, lane);
                }
            }
            // gather C(k, r) of the RW rows: lane s receives row s's value
            u64 mine = 0;
            const int qr = r >> 5, src = r & 31;
#pragma unroll
            for (int s = 0; s < RW; ++s) {
                const u64 v = shfl64(sel4(acc[s], qr), src);
                mine = (lane == s) ? v : mine;
            }
            u32 mult = 0;
            {
                const int k = warp + NW * lane;
                if (lane < RW && k > inext && k < b) {
                    const u32 ck = SP ? red_sp(mine, f) : red64(mine, f);
                    s_C[k][r] = ck;
                    mult = ck ? f.p - mulmod(ck, pinv, f) : 0u;
                }
            }
#pragma unroll
            for (int s = 0; s < RW; ++s) axpy_row<SP>(acc[s], __shfl_sync(FULL, mult, s), U, f);
        }
        r = rn;
        __syncthreads();
    }
    }  // exact path

    // ------------------------------------------------------------ finalize
    RL_STAMP(t_fact);
    LT_MARK(a.i0 / PB, 3);
    // the tail kernel (a programmatic dependent launch) may start now: it only
    // prefetches columns this kernel does not write on the speculative path,
    // and waits for this grid's completion before reading anything else
#ifndef RL_WIN_LATE_TRIGGER
    pdl_trigger();
#endif
    const int rt = r;
    // (the speculative path made no transposition: both loops are identities)
    if (!spec && warp == 1 && lane == 0) {  // window column permutation
        for (int x = 0; x < PW; ++x) s_sig[x] = x;
        for (int j = 0; j < rt; ++j) {
            const int cc = s_pos[j];
            const int t = s_sig[j];
            s_sig[j] = s_sig[cc];
            s_sig[cc] = t;
        }
    } else if (!spec && warp >= 2 && warp < 4) {  // later transpositions onto the pivot rows
        const int j = tid - 64;
        if (j < rt) {
            u32* Ur = s_R + s_rrp[j] * RP;
            for (int j2 = j + 1; j2 < rt; ++j2) {
                const int cc = s_pos[j2];
                if (cc != j2) {
                    const u32 t = Ur[j2];
                    Ur[j2] = Ur[cc];
                    Ur[cc] = t;
                }
            }
        }
    }
    __syncthreads();
    // (a) pivot-column region [c0, c0 + rt): C entries, raw pivots, normalised U
    // (b) exact path only: [c0 + rt, c0 + w) gets the original values in the final
    //     column order (the tail kernel replaces them with V = Minv * P).  The
    //     speculative path made no transposition, so those columns already hold that.
#ifdef RL_TRACE
    unsigned long long t_mid = 0;
#endif
    if (spec && bl == PB && b == PB) {
        // the common case (a full leaf, no window-dead row: row k is live row k):
        // four columns per thread, 16-byte shared loads and global stores, the
        // A entries and the Minv row in the same pass
        const bool av = ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0) && ((a.lda & 3) == 0) && ((c0 & 3) == 0);
#pragma unroll 2
        for (int e = tid; e < PB * PB / 4; e += blockDim.x) {
            const int k = e >> 4, x = (e & 15) << 2;
            const u32* R = s_R + k * RP;
            const u32 pi = s_pinvA[k];
            const uint4 rv = *reinterpret_cast<const uint4*>(R + x);
            const uint4 iv = *reinterpret_cast<const uint4*>(R + PW + x);
            u32 v[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int xq = x + q;
                v[q] = xq < k ? s_C[k][xq] : (xq == k ? v[q] : mulmod_t<SP>(v[q], pi, f));
            }
            u32* dst = a.A + (i64)(a.i0 + k) * a.lda + c0 + x;
            if (av) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) dst[q] = v[q];
            }
            *reinterpret_cast<uint4*>(&ps->Minv[k][x]) =
                make_uint4(mulmod_t<SP>(iv.x, pi, f), mulmod_t<SP>(iv.y, pi, f), mulmod_t<SP>(iv.z, pi, f),
                           mulmod_t<SP>(iv.w, pi, f));
        }
#ifdef RL_TRACE
        t_mid = rl_now();
#endif
        LT_MARK(a.i0 / PB, 4);
#if RL_WIN_UINV
        if (SP && a.uready) {
            // The leaf's U^{-1} here, from the normalised pivot block still in shared
            // memory (the inverse table's space is free after the LU): the readers
            // (bridge, node TRSM) then need not wait for the parallel U^{-1} kernel
            u32 (*Uw)[PB + 1] = reinterpret_cast<u32 (*)[PB + 1]>(dsm + PB * RP * 4);
            u32 (*Xw)[PB + 1] = Uw + PB;
            u32 (*Tw)[PB + 1] = Xw + PB;
            for (int e = tid; e < PB * PB; e += blockDim.x) {
                const int i = e / PB, kk = e % PB;
                Uw[i][kk] = kk > i ? mulmod_t<SP>(s_R[i * RP + kk], s_pinvA[i], f) : 0u;
                Xw[i][kk] = 0u;
            }
            __syncthreads();
            uinv_solve<SP>(Uw, Xw, Tw, PB, f);
            for (int e = tid; e < PB * PB / 4; e += blockDim.x) {
                const int i = e >> 4, kk = (e & 15) << 2;
                *reinterpret_cast<uint4*>(a.uinv + i * PB + kk) =
                    make_uint4(Xw[i][kk], Xw[i][kk + 1], Xw[i][kk + 2], Xw[i][kk + 3]);
            }
            __syncthreads();
            if (tid == 0) {
                ps->uinv_by_window = 1;
                uready_set(a.uready, a.epoch);
            }
        }
#endif
    } else if (spec) {
        // live row k' (original row s_perm[k']) has its pivot at column k': C
        // left of it, the raw pivot, U = reduced value * pivot^{-1} right of it;
        // Minv row k' scaled likewise.  Dead rows stay zero in the window, their
        // Minv row is e_k (residual = the row itself).
#pragma unroll 4
        for (int e = tid; e < PB * PB; e += blockDim.x) {
            const int kp = e / PB, x = e % PB;
            if (kp < bl && x < bl) {
                const u32 rv = s_R[kp * RP + x];
                const u32 val = x < kp ? s_C[kp][x] : (x == kp ? rv : mulmod_t<SP>(rv, s_pinvA[kp], f));
                a.A[(i64)(a.i0 + s_perm[kp]) * a.lda + c0 + x] = val;
            }
        }
#ifdef RL_TRACE
        t_mid = rl_now();
#endif
        LT_MARK(a.i0 / PB, 4);
#pragma unroll 4
        for (int e = tid; e < PB * PB; e += blockDim.x) {
            const int k = e / PB, i = e % PB;  // original rows
            u32 mi = 0, mr = 0;
            if (k < b && i < b) {
                const int kp = s_iperm[k], ip = s_iperm[i];
                if (kp < bl) {
                    mi = ip < bl ? mulmod_t<SP>(s_R[kp * RP + PW + ip], s_pinvA[kp], f) : 0u;
                    mr = ip == kp ? s_pv[kp] : ((ip < kp) ? s_C[kp][ip] : 0u);
                } else {
                    mi = (i == k) ? 1u % f.p : 0u;
                    mr = (i == k) ? 1u % f.p : 0u;
                }
            }
            ps->Minv[k][i] = mi;
            if (deadw) ps->Mr[k][i] = mr;  // fallback restore only
        }
    } else {
    const int xend = w;
    for (int e = tid; e < b * PW; e += blockDim.x) {
        const int k = e / PW, x = e % PW;
        if (x >= xend) continue;
        u32 val;
        if (x < rt) {
            const int rb = s_rb[k], j = s_por[k];
            if (x < rb) val = s_C[k][x];
            else if (j < 0) val = 0;
            else if (x == j) val = s_R[k * RP + x];
            else val = mulmod_t<SP>(s_R[k * RP + x], s_pinvA[j], f);
        } else {
            val = ps->win_orig[k][s_sig[x]];
        }
        a.A[(i64)(a.i0 + k) * a.lda + c0 + x] = val;
    }
    for (int e = tid; e < PB * PB; e += blockDim.x) {
        const int k = e / PB, i = e % PB;
        u32 mi = 0, mr = 0;
        if (k < b && i < b) {
            const int j = s_por[k];
            mi = s_R[k * RP + PW + i];
            if (j >= 0) mi = mulmod_t<SP>(mi, s_pinvA[j], f);
            if (i == k) {
                mr = j >= 0 ? s_pv[j] : 1u % f.p;
            } else if (i < k) {
                const int ji = s_por[i];
                if (ji >= 0) mr = s_C[k][ji];
            }
        }
        ps->Minv[k][i] = mi;
        ps->Mr[k][i] = mr;  // fallback restore only (exact path)
    }
    }
    RL_STAMP(t_f2);
    LT_MARK(a.i0 / PB, 5);
#ifdef RL_WIN_DELAY_NS
    if (threadIdx.x == 0) rl_spin_ns(RL_WIN_DELAY_NS);
#endif
    for (int e = tid; e < PB; e += blockDim.x) {
        const bool real = e < b;
        ps->piv_of_row[e] = real ? s_por[e] : -1;
        ps->rank_before[e] = real ? s_rb[e] : rt;
        if (e < rt) {
            a.rrp[c0 + e] = a.i0 + s_rrp[e];
            a.ipiv[c0 + e] = c0 + s_pos[e];
        }
        if (real) a.rp[a.i0 + 1 + e] = c0 + s_rb[e] + (s_por[e] >= 0 ? 1 : 0);
    }
    if (warp == 0) {
        u64 mask = 0;
        for (int k = lane; k < b; k += 32)
            if (s_por[k] < 0) mask |= 1ull << k;
        for (int off = 16; off > 0; off >>= 1) mask |= __shfl_xor_sync(FULL, mask, off);
        bool moved = false;
        if (!spec)
            for (int j = lane; j < rt; j += 32) moved |= s_pos[j] != j;
        moved = __any_sync(FULL, moved);
        if (lane == 0) {
            ps->dead_mask = mask;
            ps->w = w;
            ps->r = rt;
            ps->spec = spec ? 1 : 0;
            *a.swapflag = moved ? 1 : 0;
        }
    }
#ifdef RL_WIN_LATE_TRIGGER
    pdl_trigger();
#endif
    LT_END(a.i0 / PB);
#ifdef RL_TRACE
    if (a.i0 == RL_TRACE_I0 && tid == 0) {
        RL_STAMP(t_exit);
        printf("TRACE window enter %llu loaded %llu lu %llu fact %llu f1 %llu f2 %llu exit %llu spec %d\n",
               t_enter, t_loaded, t_lu, t_fact, t_mid, t_f2, t_exit, (int)spec);
        printf("TRACE solo diag_factor %llu cycles\n", g_wst[7][4]);
        for (int k = 0; k < 8; ++k)
            printf("TRACE wblk %d start %llu bc %llu end %llu | cycles: laupd %llu la %llu d(tid0) %llu\n", k,
                   g_wst[k][0], g_wst[k][1], g_wst[k][3], g_wst[k][4], g_wst[k][2], g_wst[k][5]);
    }
#endif
}

__global__ void inv_table_kernel(uint16_t* t, u32 p, Fp f) {
    const u32 x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < 65536) t[x] = (x == 0 || x >= p) ? 0 : (uint16_t)invmod(x, f);
}

}  // namespace

void build_inv_table(uint16_t* table, u32 p, cudaStream_t s) {
    inv_table_kernel<<<256, 256, 0, s>>>(table, p, make_fp(p));
    RL_CUDA_CHECK(cudaGetLastError());
}

void panel_window(const PanelArgs& a, cudaStream_t s) {
    const bool sp = a.f.p <= 65536u;
    const size_t smem = sizeof(u32) * PB * RP + (sp ? 65536 * 2 : 0);
    static std::atomic<unsigned long long> attr_once{0};
    once_on_device(attr_once, [&] {
        RL_CUDA_CHECK(cudaFuncSetAttribute(panel_window_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(sizeof(u32) * PB * RP + 65536 * 2)));
        RL_CUDA_CHECK(cudaFuncSetAttribute(panel_window_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(sizeof(u32) * PB * RP)));
    });
    RL_ONCE_MAX_SMEM(panel_window_kernel<true>);
    RL_ONCE_MAX_SMEM(panel_window_kernel<false>);
    if (sp) launch_pdl(panel_window_kernel<true>, dim3(1), dim3(NW * 32), smem, s, a);
    else launch_pdl(panel_window_kernel<false>, dim3(1), dim3(NW * 32), smem, s, a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
