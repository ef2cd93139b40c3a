// panel.cu -- base case of the CUP recursion on a leaf of b <= PB rows, and the
// leaf triangular solve.
//
// Reference: cup_base_row and the row-halving recursion (proj/src/factor.cpp:12-85).
// A leaf is the CUP of a b x W block (W = n - rank_before(leaf)): the pivot of
// row i is the first nonzero at positions >= rank so far (factor.cpp:15-21),
// brought to position r by a transposition (factor.cpp:23-24), kept raw while
// the rest of the row is scaled by its inverse (factor.cpp:25-26), and later
// rows are eliminated (factor.cpp:51-52).  Given the pivot rule the result is
// unique, so this schedule is bit-exact:
//
//  panel_window_kernel (one CTA: the sequential critical path)
//    The leading b x w window (w <= PW) plus a b x b identity block lives in
//    registers as 64-bit LAZY accumulators (warp k%8 owns row k, lane l owns
//    columns l + 32q): eliminating row k by pivot j adds mult * U_j[x] with
//    mult = -C(k,j) * pinv_j, and only the two values per row that decide
//    something are reduced (C(k,j) and, at search time, the row itself), so a
//    pivot step costs one 64-bit multiply-add per element.  Inverses come from
//    a shared-memory table for p < 2^16.  Lockstep with lookahead: during step
//    i the owner of row i+1 first applies pivot i to it, searches it (warp
//    ballot) and publishes the next pivot, then everyone updates the other
//    rows -- one CTA barrier per pivot.  The identity block yields the row
//    transform Minv with V = Minv * P (U rows for pivot rows, residuals for
//    window-dead rows) for ANY column.
//  panel_tail_kernel (grid)
//    V = Minv * P on 64 x 64 column tiles right of the leaf's pivot columns
//    (lower-triangular, lazy accumulation).  Window-dead rows must come out
//    zero; otherwise a pivot lies beyond the window and the last CTA re-runs
//    the leaf exactly (restore P = Mr * V, row-by-row elimination over the full
//    width).  One extra CTA inverts the leaf's unit upper pivot block for the
//    TRSMs against it.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {


// Inverse of the leaf's unit upper pivot block U (r x r, rows rrp[c0+j], columns
// c0+j'), into uinv (PB x PB, zero padded).  One CTA of 256 threads: 4 threads
// per column, back substitution X[i][c] = -sum_{k=i+1..c} U[i][k] X[k][c].
__device__ void leaf_uinv(const PanelArgs& a, i32 c0, int rt, u32 (*U)[PB + 1], u32 (*X)[PB + 1]) {
    const Fp f = a.f;
    const int tid = threadIdx.x;
    __shared__ i32 s_row[PB];
    if (tid < PB) s_row[tid] = tid < rt ? __ldcg(a.rrp + c0 + tid) : 0;
    __syncthreads();
#pragma unroll 4
    for (int e = tid; e < PB * PB; e += blockDim.x) {
        const int i = e / PB, k = e % PB;
        const bool ok = i < k && k < rt;
        cp_async4(&U[i][k], ok ? a.A + (i64)s_row[i] * a.lda + c0 + k : a.A, ok);
        X[i][k] = (i == k && i < rt) ? 1u % f.p : 0u;
    }
    cp_async_wait_all();
    __syncthreads();
    // rows of X from the bottom: X[i][:] = e_i - sum_{k>i} U[i][k] X[k][:];
    // thread = (column c, quarter part of the k range), products summed lazily
    // in 64 bits when p < 2^16 (<= 64 terms < 2^32 each).
    const int c = tid >> 2, part = tid & 3;
    const unsigned gm = 0xFu << ((tid & 31) & ~3);  // the 4 lanes of this column
    const bool sp = f.p <= 65536u;
    for (int i = rt - 2; i >= 0; --i) {
        u64 acc = 0;
        if (c > i && c < rt) {
            for (int k = i + 1 + part; k <= c; k += 4) {
                if (sp) acc += (u64)U[i][k] * X[k][c];
                else acc += mulmod(U[i][k], X[k][c], f);
            }
        }
        acc += __shfl_xor_sync(gm, acc, 1);
        acc += __shfl_xor_sync(gm, acc, 2);
        if (part == 0 && c > i && c < rt) {
            const u32 s = red64(acc, f);
            X[i][c] = s ? f.p - s : 0u;
        }
        __syncthreads();
    }
    for (int e = tid; e < PB * PB; e += blockDim.x) a.uinv[e] = X[e / PB][e % PB];
    __syncthreads();
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

// V = Minv * P on 64-column tiles (4 x 4 outputs per thread), the window-dead
// row check, and (last CTA) the exact fallback; the extra last-index CTA
// computes the leaf's U^{-1}.
template <bool SP>
__global__ void __launch_bounds__(256) panel_tail_kernel(PanelArgs a) {
    __shared__ u32 Mi[PB][PB + 1];
    __shared__ u32 Ps[PB][PB + 1];
    __shared__ u32 red_buf[256];
    __shared__ int s_last;
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x;
    const i32 c0 = ps->c0, W = ps->W, b = ps->b, rt = ps->r;
    u32 bad = 0;
    if (blockIdx.x == gridDim.x - 1) {
        if (W > 0 && rt > 0) leaf_uinv(a, c0, rt, Mi, Ps);
    } else if (W > 0) {
        const u64 dead = ps->dead_mask;
#pragma unroll 4
        for (int e = tid; e < PB * PB; e += blockDim.x)
            cp_async4(&Mi[e / PB][e % PB], &ps->Minv[e / PB][e % PB], true);
        const int tx = tid & 15, ty = tid >> 4;
        const i32 col0 = c0 + rt;
        const i32 ntile = (a.N - col0 + 63) / 64;
        for (i32 t = blockIdx.x; t < ntile; t += gridDim.x - 1) {
            const i32 cb = col0 + t * 64;
            __syncthreads();
#pragma unroll 4
            for (int e = tid; e < PB * 64; e += blockDim.x) {
                const int i = e >> 6, cc = e & 63;
                const bool ok = i < b && cb + cc < a.N;
                cp_async4(&Ps[i][cc], ok ? a.A + (i64)(a.i0 + i) * a.lda + cb + cc : a.A, ok);
            }
            cp_async_wait_all();
            __syncthreads();
            u64 acc[4][4];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = 0;
            const int kmax = min(b, ty * 4 + 4);
            for (int k = 0; k < kmax; ++k) {
                u32 mv[4], pv[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) mv[x] = Mi[ty * 4 + x][k];
#pragma unroll
                for (int y = 0; y < 4; ++y) pv[y] = Ps[k][tx * 4 + y];
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        if (SP) acc[x][y] += (u64)mv[x] * pv[y];
                        else acc[x][y] += mulmod(mv[x], pv[y], f);
                    }
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int i = ty * 4 + x;
                if (i >= b) continue;
                u32* out = a.A + (i64)(a.i0 + i) * a.lda + cb;
                const bool isdead = (dead >> i) & 1;
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const int cc = tx * 4 + y;
                    if (cb + cc < a.N) {
                        const u32 val = red64(acc[x][y], f);
                        if (isdead) bad |= val;
                        out[cc] = val;
                    }
                }
            }
        }
    }
    if (__syncthreads_or(bad != 0) && tid == 0) atomicOr(&ps->flag, 1u);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&ps->counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (atomicAdd(&ps->flag, 0u) != 0) {
        panel_fallback(a, red_buf);
        const int r2 = ps->r;
        if (r2 > 0) leaf_uinv(a, c0, r2, Mi, Ps);
    }
    if (tid == 0) {
        ps->counter = 0;
        ps->flag = 0;
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

}  // namespace

void panel_tail(const PanelArgs& a, cudaStream_t s) {
    const int grid = std::max(1, std::min((a.N + 63) / 64, 2 * num_sms())) + 1;
    if (a.f.p <= 65536u) panel_tail_kernel<true><<<grid, 256, 0, s>>>(a);
    else panel_tail_kernel<false><<<grid, 256, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

void trsm_leaf(const TrsmLeafArgs& a, cudaStream_t s) {
    if (a.M <= 0) return;
    const int grid = std::max(1, std::min((a.M + 63) / 64, 4 * num_sms()));
    if (a.f.p <= 65536u) trsm_leaf_kernel<true><<<grid, 256, 0, s>>>(a);
    else trsm_leaf_kernel<false><<<grid, 256, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
