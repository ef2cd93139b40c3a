// panel.cu -- the leaf's tail (everything right of its pivot columns), the leaf
// U^{-1}, the exact fallback, and the single-leaf triangular solve.
//
// Reference: cup_base_row and the row-halving recursion (proj/src/factor.cpp:12-85).
// A leaf is the CUP of a b x W block (W = n - rank_before(leaf)).  Given the
// pivot rule the result is unique, so this schedule is
// bit-exact:
//
//  panel_window_kernel (panel_window.cu, one CTA: the sequential critical path)
//    finds the leaf's pivots in its leading window and the row transform Minv:
//    V = Minv * P gives the U rows (pivot rows) and the residuals (window-dead
//    rows) of ANY column P of the leaf's rows.
//  panel_tail_kernel (grid)
//    V = Minv * P on 64 x 256 column tiles right of the pivot columns
//    (lower-triangular, 8 x 8 outputs per thread, lazy 64-bit accumulation).
//    Window-dead rows must come out zero; otherwise a pivot lies beyond the
//    window and the last CTA re-runs the leaf exactly (restore P = Mr * V,
//    row-by-row elimination over the full width).  One extra CTA inverts the
//    leaf's unit upper pivot block (blocked, 8 x 8 diagonal blocks) for the TRSMs
//    against it.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"
#include "uinv.cuh"

namespace rl {

namespace {

constexpr int TT = 64;   // tail tile width (columns per CTA tile)
constexpr int MIP = PB + 4;  // Minv pitch in the tail (16-byte rows for cp.async)

// Inverse of the leaf's unit upper pivot block U (r x r, rows rrp[c0+j],
// columns c0+j'), into uinv (PB x PB, zero padded).  Recursive doubling: the
// eight 8 x 8 diagonal blocks are inverted by eight warps at once, then pairs
// of s x s blocks merge (s = 8, 16, 32) through X_AB = -X_AA * (U_AB * X_BB),
// two fully parallel products per level (3 levels, 6 barriers).
template <bool SP>
__device__ void leaf_uinv(const PanelArgs& a, i32 c0, int rt, u32 (*U)[PB + 1], u32 (*X)[PB + 1],
                          u32 (*T)[PB + 1]) {
    const Fp f = a.f;
    const int tid = threadIdx.x, nt = blockDim.x;
    RL_STAMP(u0);
    __shared__ i32 s_row[PB];
    if (tid < PB) s_row[tid] = tid < rt ? __ldcg(a.rrp + c0 + tid) : 0;
    __syncthreads();
    RL_STAMP(u1);
#pragma unroll 4
    for (int e = tid; e < PB * PB; e += nt) {
        const int i = e / PB, k = e % PB;
        const bool ok = i < k && k < rt;
        cp_async4(&U[i][k], ok ? a.A + (i64)s_row[i] * a.lda + c0 + k : a.A, ok);
        X[i][k] = 0;
    }
    cp_async_wait_all();
    __syncthreads();
    RL_STAMP(u2);
#ifdef RL_TRACE
    const long long c2 = clock64();
#endif
    uinv_solve<SP>(U, X, T, rt, f);
#ifdef RL_TRACE
    const long long c3 = clock64();
#endif
    RL_STAMP(u3);
    RL_STAMP(u4);
    for (int e = tid; e < PB * PB; e += nt) a.uinv[e] = X[e / PB][e % PB];
    __syncthreads();
#ifdef RL_TRACE
    if (a.i0 == RL_TRACE_I0 && tid == 0) {
        RL_STAMP(u5);
        printf("TRACE uinv row %llu load %llu diag %llu levels %llu store %llu diag_cycles %lld\n", u1 - u0,
               u2 - u1, u3 - u2, u4 - u3, u5 - u4, c3 - c2);
    }
#endif
}

// Exact leaf CUP over the full width in global memory: used only when a pivot
// lies beyond the window (structured / small-p inputs).  One CTA.
__device__ void panel_fallback(const PanelArgs& a, u32* red_buf) {
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x, nt = blockDim.x;
    const i32 c0 = ps->c0, w = ps->w, b = ps->b;
    const i32 N = a.N;
    u32* A = a.A;
    const i64 lda = a.lda;
    // 1. restore: tail columns P = Mr * V, window from the saved original
    for (i32 colx = c0 + w + tid; colx < N; colx += nt) {
        u32 V[PB];
        for (int i = 0; i < b; ++i) V[i] = A[(i64)(a.i0 + i) * lda + colx];
        for (int i = 0; i < b; ++i) {
            u64 acc = 0;
            for (int i2 = 0; i2 <= i; ++i2) acc += mulmod(ps->Mr[i][i2], V[i2], f);
            A[(i64)(a.i0 + i) * lda + colx] = red64(acc, f);
        }
    }
    for (int e = tid; e < b * PW; e += nt) {
        const int i = e / PW, c = e % PW;
        if (c < w) A[(i64)(a.i0 + i) * lda + c0 + c] = ps->win_orig[i][c];
    }
    __threadfence_block();
    __syncthreads();
    // 2. row-by-row elimination over columns [c0, N)
    __shared__ u32 s_pinv;
    int r = 0;
    for (int i = 0; i < b; ++i) {
        u32* ri = A + (i64)(a.i0 + i) * lda;
        i32 best = N;
        for (i32 cc = c0 + r + tid; cc < N; cc += nt)
            if (ri[cc] != 0) {
                best = cc;
                break;
            }
        red_buf[tid] = (u32)best;
        __syncthreads();
        for (int s = nt / 2; s > 0; s >>= 1) {
            if (tid < s) red_buf[tid] = min(red_buf[tid], red_buf[tid + s]);
            __syncthreads();
        }
        const i32 c = (i32)red_buf[0];
        __syncthreads();
        if (c >= N) {
            if (tid == 0) a.rp[a.i0 + 1 + i] = c0 + r;
            continue;
        }
        const i32 pc = c0 + r;
        if (c != pc && tid < b) {
            u32* rk = A + (i64)(a.i0 + tid) * lda;
            const u32 t = rk[pc];
            rk[pc] = rk[c];
            rk[c] = t;
        }
        __threadfence_block();
        __syncthreads();
        if (tid == 0) {
            s_pinv = invmod(ri[pc], f);
            a.rrp[pc] = a.i0 + i;
            a.ipiv[pc] = c;
            if (c != pc) *a.swapflag = 1;
            a.rp[a.i0 + 1 + i] = pc + 1;
        }
        __syncthreads();
        const u32 pinv = s_pinv;
        for (i32 cc = pc + 1 + tid; cc < N; cc += nt) {
            const u32 u = mulmod(ri[cc], pinv, f);
            ri[cc] = u;
            const u32 nu = u ? f.p - u : 0u;
            for (int k = i + 1; k < b; ++k) {
                u32* rk = A + (i64)(a.i0 + k) * lda;
                const u32 fk = rk[pc];
                if (fk) rk[cc] = red64((u64)fk * nu + rk[cc], f);
            }
        }
        __threadfence_block();
        __syncthreads();
        ++r;
    }
    if (tid == 0) ps->r = r;
    __threadfence_block();
    __syncthreads();
}

constexpr int BPI = 80;  // byte-plane row pitch (bytes): conflict-free fragment loads

// acc[x][.] += Minv[ty + 16x][k] * P[k][4tx .. 4tx+3] for k in [k0, k1), rows x >= X0.
template <bool SP, int X0>
__device__ __forceinline__ void tail_mac(u64 (&acc)[4][4], const u32 (*Mi)[MIP],
                                         const u32 (*Ps)[TT + 4], int ty, int tx, int k0, int k1,
                                         const Fp& f) {
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
        const uint4 pv = *reinterpret_cast<const uint4*>(&Ps[k][4 * tx]);
#pragma unroll
        for (int x = X0; x < 4; ++x) {
            const u32 mv = Mi[ty + 16 * x][k];
            if (SP) {
                acc[x][0] += (u64)mv * pv.x;
                acc[x][1] += (u64)mv * pv.y;
                acc[x][2] += (u64)mv * pv.z;
                acc[x][3] += (u64)mv * pv.w;
            } else {
                acc[x][0] += mulmod(mv, pv.x, f);
                acc[x][1] += mulmod(mv, pv.y, f);
                acc[x][2] += mulmod(mv, pv.z, f);
                acc[x][3] += mulmod(mv, pv.w, f);
            }
        }
    }
}

// V = Minv * P on 64 x TT column tiles: thread (ty, tx) owns rows ty + 16x
// (x < 4, balancing the triangle) and columns 4tx..4tx+3 (one 16-byte shared
// load of P per 16 products).  Small tiles give many resident CTAs per SM.
template <bool SP>
__global__ void __launch_bounds__(256) panel_tail_kernel(PanelArgs a) {
    extern __shared__ __align__(16) u32 tsm[];
    u32 (*Mi)[MIP] = reinterpret_cast<u32 (*)[MIP]>(tsm);                     // [PB][MIP]
    u32 (*Ps)[TT + 4] = reinterpret_cast<u32 (*)[TT + 4]>(tsm + PB * MIP);    // [PB][TT+4]
    // p < 2^16: byte planes of Minv (row-major, k contiguous) and of the P tile
    // (transposed: column-major, k contiguous) for the tensor-core product
    uint8_t* planes = reinterpret_cast<uint8_t*>(tsm + PB * MIP + PB * (TT + 4));
    uint8_t (*Ml)[BPI] = reinterpret_cast<uint8_t (*)[BPI]>(planes);
    uint8_t (*Mh)[BPI] = reinterpret_cast<uint8_t (*)[BPI]>(planes + PB * BPI);
    uint8_t (*Pl)[BPI] = reinterpret_cast<uint8_t (*)[BPI]>(planes + 2 * PB * BPI);
    uint8_t (*Ph)[BPI] = reinterpret_cast<uint8_t (*)[BPI]>(planes + 2 * PB * BPI + TT * BPI);
    u32 (*Us)[PB + 1] = reinterpret_cast<u32 (*)[PB + 1]>(tsm);               // uinv scratch
    u32 (*Xs)[PB + 1] = reinterpret_cast<u32 (*)[PB + 1]>(tsm + PB * (PB + 1));
    u32 (*Ts)[PB + 1] = reinterpret_cast<u32 (*)[PB + 1]>(tsm + 2 * PB * (PB + 1));
    __shared__ u32 red_buf[256];
    __shared__ int s_last;
    RL_STAMP(t_enter);
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0) && (a.lda & 3) == 0;
    // Launched as a programmatic dependent of the window kernel: before its
    // grid completes, prefetch this CTA's first tile on the assumption of the
    // speculative path (rank b, no transposition -- the window then leaves
    // columns >= c0 + b untouched; c0 = rp[i0] is older than the window).
    const i32 c0_pre = __ldcg(a.rp + a.i0);
    const i32 cb_pre = vec ? ((c0_pre + a.b) & ~3) : c0_pre + a.b;
    const bool pre = a.prefetch && vec && blockIdx.x < gridDim.x - 1 && cb_pre + (i32)blockIdx.x * TT < a.N;
    if (pre) {
        const i32 cb = cb_pre + blockIdx.x * TT;
#pragma unroll
        for (int e = tid; e < PB * TT / 4; e += blockDim.x) {
            const int i = e / (TT / 4), cc = 4 * (e % (TT / 4));
            const int nb = i < a.b ? 4 * max(0, min(4, a.N - cb - cc)) : 0;
            cp_async16z(&Ps[i][cc], nb ? a.A + (i64)(a.i0 + i) * a.lda + cb + cc : a.A, nb);
        }
    }
    pdl_wait();
    pdl_trigger();
    const i32 c0 = ps->c0, W = ps->W, b = ps->b, rt = ps->r;
    const u64 dead = ps->dead_mask;
    const bool pre_ok = pre && ps->spec && rt == a.b && c0 == c0_pre && dead == 0;
    if (pre && !pre_ok) cp_async_wait_all();  // drain before the tile is reloaded
    u32 bad = 0;
#ifdef RL_TRACE
    unsigned long long t_loaded = 0, t_mac = 0;
#endif
    if (blockIdx.x == gridDim.x - 1) {
        // U^{-1} here for leaves with window-dead rows; with RL_UINV_IN_TAIL for
        // every leaf (otherwise the parallel panel_uinv kernel computes it)
        if (W > 0 && rt > 0 && (RL_UINV_IN_TAIL || dead != 0)) {
            leaf_uinv<SP>(a, c0, rt, Us, Xs, Ts);
        }
    } else if (W > 0) {
        if (SP) {
#pragma unroll
            for (int e = tid; e < PB * PB / 4; e += blockDim.x) {
                const int i = e / (PB / 4), k = 4 * (e % (PB / 4));
                const uint4 v = __ldcg(reinterpret_cast<const uint4*>(&ps->Minv[i][k]));
                *reinterpret_cast<u32*>(&Ml[i][k]) =
                    (v.x & 0xff) | (v.y & 0xff) << 8 | (v.z & 0xff) << 16 | (v.w & 0xff) << 24;
                *reinterpret_cast<u32*>(&Mh[i][k]) = (v.x >> 8 & 0xff) | (v.y >> 8 & 0xff) << 8 |
                                                     (v.z >> 8 & 0xff) << 16 | (v.w >> 8 & 0xff) << 24;
            }
        } else {
#pragma unroll
            for (int e = tid; e < PB * PB / 4; e += blockDim.x)
                cp_async16(&Mi[e / (PB / 4)][4 * (e % (PB / 4))], &ps->Minv[e / (PB / 4)][4 * (e % (PB / 4))]);
        }
        const int tx = tid & 15, ty = tid >> 4;
        const i32 col0 = c0 + rt;
        // 16-byte path: tiles start at col0 rounded down to 4 columns (the
        // extra leading columns are computed but neither stored nor checked)
        const i32 cbase = vec ? (col0 & ~3) : col0;
        const i32 ntile = (a.N - cbase + TT - 1) / TT;
        for (i32 t = blockIdx.x; t < ntile; t += gridDim.x - 1) {
            const i32 cb = cbase + t * TT;
            __syncthreads();
            if (t == (i32)blockIdx.x && pre_ok) {
                // the prefetched tile is this one (same rows, same columns)
            } else if (vec) {
#pragma unroll
                for (int e = tid; e < PB * TT / 4; e += blockDim.x) {
                    const int i = e / (TT / 4), cc = 4 * (e % (TT / 4));
                    const int nb = i < b ? 4 * max(0, min(4, a.N - cb - cc)) : 0;
                    cp_async16z(&Ps[i][cc], nb ? a.A + (i64)(a.i0 + i) * a.lda + cb + cc : a.A, nb);
                }
            } else {
#pragma unroll 4
                for (int e = tid; e < PB * TT; e += blockDim.x) {
                    const int i = e / TT, cc = e % TT;
                    const bool ok = i < b && cb + cc < a.N;
                    cp_async4(&Ps[i][cc], ok ? a.A + (i64)(a.i0 + i) * a.lda + cb + cc : a.A, ok);
                }
            }
            cp_async_wait_all();
            __syncthreads();
            RL_STAMP(t_ld);
#ifdef RL_TRACE
            t_loaded = t_ld;
#endif
            if constexpr (SP) {
                // P tile -> transposed byte planes (column c: 64 k bytes)
#pragma unroll
                for (int e = tid; e < TT * (PB / 4); e += blockDim.x) {
                    const int c = e % TT, k = 4 * (e / TT);
                    const u32 v0 = Ps[k][c], v1 = Ps[k + 1][c], v2 = Ps[k + 2][c], v3 = Ps[k + 3][c];
                    *reinterpret_cast<u32*>(&Pl[c][k]) =
                        (v0 & 0xff) | (v1 & 0xff) << 8 | (v2 & 0xff) << 16 | (v3 & 0xff) << 24;
                    *reinterpret_cast<u32*>(&Ph[c][k]) = (v0 >> 8 & 0xff) | (v1 >> 8 & 0xff) << 8 |
                                                         (v2 >> 8 & 0xff) << 16 | (v3 >> 8 & 0xff) << 24;
                }
                __syncthreads();
                // warp w: rows 16 (w & 3) .., columns 32 (w >> 2) .. (four n8 tiles);
                // V = S0 + 2^8 S1 + 2^16 S2 with S0 = lo*lo, S1 = lo*hi + hi*lo, S2 = hi*hi
                const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tg = lane & 3;
                const int rs = warp & 3, chn = warp >> 2;
                int S0[4][4] = {}, S1[4][4] = {}, S2[4][4] = {};
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    if (ks == 1 && rs < 2) break;  // Minv rows < 32 vanish for k >= 32
                    const int kk = 32 * ks + 4 * tg;
                    const int r0 = 16 * rs + g;
                    const u32 al[4] = {*reinterpret_cast<const u32*>(&Ml[r0][kk]),
                                       *reinterpret_cast<const u32*>(&Ml[r0 + 8][kk]),
                                       *reinterpret_cast<const u32*>(&Ml[r0][kk + 16]),
                                       *reinterpret_cast<const u32*>(&Ml[r0 + 8][kk + 16])};
                    const u32 ah[4] = {*reinterpret_cast<const u32*>(&Mh[r0][kk]),
                                       *reinterpret_cast<const u32*>(&Mh[r0 + 8][kk]),
                                       *reinterpret_cast<const u32*>(&Mh[r0][kk + 16]),
                                       *reinterpret_cast<const u32*>(&Mh[r0 + 8][kk + 16])};
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) {
                        const int n = 32 * chn + 8 * nt + g;
                        const u32 bl[2] = {*reinterpret_cast<const u32*>(&Pl[n][kk]),
                                           *reinterpret_cast<const u32*>(&Pl[n][kk + 16])};
                        const u32 bh[2] = {*reinterpret_cast<const u32*>(&Ph[n][kk]),
                                           *reinterpret_cast<const u32*>(&Ph[n][kk + 16])};
                        imma16832(S0[nt], al, bl);
                        imma16832(S1[nt], al, bh);
                        imma16832(S1[nt], ah, bl);
                        imma16832(S2[nt], ah, bh);
                    }
                }
                RL_STAMP(t_m);
#ifdef RL_TRACE
                t_mac = t_m;
#endif
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = 16 * rs + g + 8 * h;
                        if (i >= b) continue;
                        const i32 cx = cb + 32 * chn + 8 * nt + 2 * tg;
                        const u32 v0 = red_sp((u64)(u32)S0[nt][2 * h] + ((u64)(u32)S1[nt][2 * h] << 8) +
                                                  ((u64)(u32)S2[nt][2 * h] << 16), f);
                        const u32 v1 = red_sp((u64)(u32)S0[nt][2 * h + 1] + ((u64)(u32)S1[nt][2 * h + 1] << 8) +
                                                  ((u64)(u32)S2[nt][2 * h + 1] << 16), f);
                        const bool ok0 = cx >= col0 && cx < a.N, ok1 = cx + 1 >= col0 && cx + 1 < a.N;
                        u32* out = a.A + (i64)(a.i0 + i) * a.lda + cx;
                        const bool isdead = (dead >> i) & 1;
                        if (isdead) bad |= (ok0 ? v0 : 0u) | (ok1 ? v1 : 0u);
                        if (vec && ok0 && ok1) {
                            *reinterpret_cast<uint2*>(out) = make_uint2(v0, v1);
                        } else {
                            if (ok0) out[0] = v0;
                            if (ok1) out[1] = v1;
                        }
                    }
                }
            } else {
            // rows ty + 16x interleave short and long rows of the triangle
            u64 acc[4][4];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = 0;
            // Minv is lower triangular: row ty + 16x needs k <= ty + 16x only, so
            // the k range splits into four phases with a static set of rows each
            tail_mac<SP, 0>(acc, Mi, Ps, ty, tx, 0, min(b, ty + 1), f);
            tail_mac<SP, 1>(acc, Mi, Ps, ty, tx, ty + 1, min(b, ty + 17), f);
            tail_mac<SP, 2>(acc, Mi, Ps, ty, tx, ty + 17, min(b, ty + 33), f);
            tail_mac<SP, 3>(acc, Mi, Ps, ty, tx, ty + 33, min(b, ty + 49), f);
            RL_STAMP(t_m);
#ifdef RL_TRACE
            t_mac = t_m;
#endif
            const i32 cx = cb + 4 * tx;
            const bool full = vec && cx >= col0 && cx + 4 <= a.N;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int i = ty + 16 * x;
                if (i >= b) continue;
                u32* out = a.A + (i64)(a.i0 + i) * a.lda + cx;
                const bool isdead = (dead >> i) & 1;
                u32 v[4];
#pragma unroll
                for (int y = 0; y < 4; ++y) v[y] = SP ? red_sp(acc[x][y], f) : red64(acc[x][y], f);
                if (full) {
                    if (isdead) bad |= v[0] | v[1] | v[2] | v[3];
                    *reinterpret_cast<uint4*>(out) = make_uint4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        if (cx + y >= col0 && cx + y < a.N) {
                            if (isdead) bad |= v[y];
                            out[y] = v[y];
                        }
                    }
                }
            }
            }
        }
    }
    RL_STAMP(t_work);
    // Without window-dead rows no residual can be nonzero and no fallback is
    // possible: skip the grid-wide check (fence + last-CTA counter) entirely.
    // The decision is uniform: every CTA reads the same dead_mask.
#ifdef RL_TRACE
    if (a.i0 == RL_TRACE_I0 && tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 2))
        printf("TRACE tailw cta %d/%d enter %llu loaded %llu mac %llu work %llu\n", blockIdx.x,
               gridDim.x, t_enter, t_loaded, t_mac, t_work);
#endif
    if (W > 0 && dead == 0) return;
    if (__syncthreads_or(bad != 0) && tid == 0) atomicOr(&ps->flag, 1u);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&ps->counter, 1u) == gridDim.x - 1);
    __syncthreads();
#ifdef RL_TRACE
    if (a.i0 == RL_TRACE_I0 && tid == 0) {
        RL_STAMP(t_exit);
        printf("TRACE tail cta %d/%d enter %llu work %llu exit %llu\n", blockIdx.x, gridDim.x, t_enter,
               t_work, t_exit);
    }
#endif
    if (!s_last) return;
    __threadfence();
    if (atomicAdd(&ps->flag, 0u) != 0) {
        panel_fallback(a, red_buf);
        const int r2 = ps->r;
        if (r2 > 0) leaf_uinv<SP>(a, c0, r2, Us, Xs, Ts);
    }
    __syncthreads();
    if (tid == 0) {
        ps->counter = 0;
        ps->flag = 0;
        // U^{-1} of a leaf with window-dead rows (or no window) is final only now
        if (a.uready) uready_set(a.uready, a.epoch);
    }
}

// X <- X * Uinv for X = rows [row0, row0+M) x columns J (|J| = nJ <= PB):
// a 64 x nJ x nJ upper-triangular product per CTA tile, 4x4 outputs per thread.
template <bool SP>
__global__ void __launch_bounds__(256) trsm_leaf_kernel(TrsmLeafArgs a) {
    __shared__ u32 Ui[PB][PB + 1];
    __shared__ u32 Xs[64][PB + 1];
    const Fp f = a.f;
    const i32 j_lo = dyn_eval(a.j_lo, a.rp);
    const i32 nJ = dyn_eval(a.j_hi, a.rp) - j_lo;
    if (nJ <= 0 || a.M <= 0) return;
#pragma unroll 4
    for (int e = threadIdx.x; e < PB * PB; e += blockDim.x) cp_async4(&Ui[e / PB][e % PB], a.uinv + e, true);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    for (i32 r0 = blockIdx.x * 64; r0 < a.M; r0 += gridDim.x * 64) {
        __syncthreads();
#pragma unroll 4
        for (int e = threadIdx.x; e < 64 * PB; e += blockDim.x) {
            const int rr = e / PB, j = e % PB;
            const bool ok = r0 + rr < a.M && j < nJ;
            cp_async4(&Xs[rr][j], ok ? a.A + (i64)(a.row0 + r0 + rr) * a.lda + j_lo + j : a.A, ok);
        }
        cp_async_wait_all();
        __syncthreads();
        u64 acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = 0;
        const int kmax = min(nJ, tx * 4 + 4);
        for (int k = 0; k < kmax; ++k) {
            u32 xv[4], uv[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) xv[x] = Xs[ty * 4 + x][k];
#pragma unroll
            for (int y = 0; y < 4; ++y) uv[y] = Ui[k][tx * 4 + y];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    if (SP) acc[x][y] += (u64)xv[x] * uv[y];
                    else acc[x][y] += mulmod(xv[x], uv[y], f);
                }
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const i32 row = r0 + ty * 4 + x;
            if (row >= a.M) continue;
            u32* out = a.A + (i64)(a.row0 + row) * a.lda + j_lo;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int j = tx * 4 + y;
                if (j < nJ) out[j] = red64(acc[x][y], f);
            }
        }
    }
}

template <bool SP>
__global__ void __launch_bounds__(512) panel_uinv_kernel(PanelArgs a) {
    extern __shared__ __align__(16) u32 tsm[];
    const PanelScratch* ps = a.ps;
    const i32 c0 = ps->c0, W = ps->W, rt = ps->r;
    // (W <= 0 or window-dead rows: the tail kernel computes U^{-1} and sets the flag)
    if (W <= 0 || ps->dead_mask != 0 || ps->uinv_by_window) return;
    if (rt > 0)
        leaf_uinv<SP>(a, c0, rt, reinterpret_cast<u32 (*)[PB + 1]>(tsm),
                      reinterpret_cast<u32 (*)[PB + 1]>(tsm + PB * (PB + 1)),
                      reinterpret_cast<u32 (*)[PB + 1]>(tsm + 2 * PB * (PB + 1)));
    __syncthreads();
    if (threadIdx.x == 0 && a.uready) uready_set(a.uready, a.epoch);
}

}  // namespace

void panel_uinv(const PanelArgs& a, cudaStream_t s) {
    // The kernel needs 3 blocks of PB x (PB+1); it asks for 200 KB so that no
    // tail-kernel CTA (launched right after it) shares its SM: this latency-bound
    // chain ran ~3x slower beside the tail's multiply-add streams.
#ifndef RL_UINV_SMEM_KB
#define RL_UINV_SMEM_KB 200
#endif
    const size_t smem = std::max<size_t>(sizeof(u32) * 3 * PB * (PB + 1), RL_UINV_SMEM_KB * 1024);
    static std::atomic<unsigned long long> attr_once{0};
    once_on_device(attr_once, [&] {
        RL_CUDA_CHECK(cudaFuncSetAttribute(panel_uinv_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        RL_CUDA_CHECK(cudaFuncSetAttribute(panel_uinv_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    if (a.f.p <= 65536u) panel_uinv_kernel<true><<<1, 512, smem, s>>>(a);
    else panel_uinv_kernel<false><<<1, 512, smem, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

void panel_tail(const PanelArgs& a, cudaStream_t s) {
    // tiles: Minv + P tile; the U^{-1} CTA: U, X, T (3 blocks of PB x (PB+1))
    const size_t smem = std::max<size_t>(sizeof(u32) * (PB * MIP + PB * (TT + 4)) + 2 * (PB + TT) * BPI,
                                         sizeof(u32) * 3 * PB * (PB + 1));
    static std::atomic<unsigned long long> attr_once{0};
    once_on_device(attr_once, [&] {
        RL_CUDA_CHECK(cudaFuncSetAttribute(panel_tail_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        RL_CUDA_CHECK(cudaFuncSetAttribute(panel_tail_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    const int grid = std::max(1, std::min((a.N + TT - 1) / TT, 8 * num_sms())) + 1;
    RL_ONCE_MAX_SMEM(panel_tail_kernel<true>);
    RL_ONCE_MAX_SMEM(panel_tail_kernel<false>);
    // programmatic dependent launch: the CTAs start (and prefetch) while the
    // window kernel finishes; griddepcontrol.wait orders everything else
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (a.f.p <= 65536u) RL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, panel_tail_kernel<true>, a));
    else RL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, panel_tail_kernel<false>, a));
}

void trsm_leaf(const TrsmLeafArgs& a, cudaStream_t s) {
    if (a.M <= 0) return;
    const int grid = std::max(1, std::min((a.M + 63) / 64, 4 * num_sms()));
    if (a.f.p <= 65536u) trsm_leaf_kernel<true><<<grid, 256, 0, s>>>(a);
    else trsm_leaf_kernel<false><<<grid, 256, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
