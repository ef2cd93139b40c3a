// panel.cu -- base case of the CUP recursion on a leaf of <= PB rows, plus the
// small TRSM, permutation and placement kernels around it.
//
// Reference: cup_base_row and the row-halving recursion (proj/src/factor.cpp:12-85).
// A leaf of b rows is the CUP of a b x W block (W = n - rank_before(leaf)):
// pivot of row i = first nonzero at positions >= rank so far (factor.cpp:15-21),
// brought to position r by a transposition (factor.cpp:23-24), pivot kept raw
// and the rest of the row scaled by its inverse (factor.cpp:25-26), later rows
// eliminated (factor.cpp:51-52).  The result is unique given the pivot rule
// (PAPER.md:1648-1649), so any schedule that reproduces the pivot sequence is
// bit-exact.  Schedule used here:
//
//  1. panel_window_kernel (one CTA): factors the b x w leading window (w <= PW)
//     in shared memory.  Pivot discovery is FRACTION-FREE -- row_k <- pv*row_k
//     - row_k[r]*row_i -- which scales rows by nonzero factors and so preserves
//     every zero pattern, hence every pivot position, with no modular inverse
//     on the sequential critical path.  True values are recovered afterwards
//     in parallel: the stored entry at pivot column j of any row carries the
//     scale Q_j = prod_{j'<j} pv_j', U row j carries pv_j.
//  2. panel_tail_kernel (many CTAs, one column per thread): the columns right
//     of the window.  Pivot columns all lie in the window, so tail columns are
//     untouched by swaps and each one is an independent forward recurrence
//     over the b rows.  Window-dead rows must come out zero; if one does not,
//     its pivot lies beyond the window and the last CTA re-runs the leaf
//     exactly (restore + row-by-row elimination over the full width).
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {

__global__ void __launch_bounds__(256) panel_window_kernel(PanelArgs a) {
    __shared__ u32 win[PB][PW + 1];
    __shared__ i32 s_piv_of_row[PB], s_rank_before[PB], s_rrp[PB], s_ipiv[PB];
    __shared__ u32 s_pv[PB], s_Q[PB], s_pvinv[PB], s_Qinv[PB];
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const i32 c0 = __ldcg(a.rp + a.i0);
    const i32 W = a.N - c0;
    const int b = a.b;
    if (tid == 0) {
        ps->flag = 0;
        ps->counter = 0;
        ps->c0 = c0;
        ps->b = b;
        ps->W = W > 0 ? W : 0;
    }
    if (W <= 0) {  // rank already n: rows keep their C data (factor.cpp:47)
        for (int i = tid; i < b; i += blockDim.x) a.rp[a.i0 + 1 + i] = c0;
        if (tid == 0) {
            ps->w = 0;
            ps->r = 0;
        }
        for (int e = tid; e < PB; e += blockDim.x) {
            ps->piv_of_row[e] = -1;
            ps->rank_before[e] = 0;
        }
        return;
    }
    const int w = W < PW ? W : PW;
    for (int e = tid; e < PB * PW; e += blockDim.x) {
        const int i = e / PW, c = e % PW;
        u32 v = (i < b && c < w) ? __ldcg(a.A + (i64)(a.i0 + i) * a.lda + c0 + c) : 0u;
        win[i][c] = v;
        ps->win_orig[i][c] = v;
    }
    __syncthreads();

    int r = 0;
    const int col = tid & (PW - 1);
    const int half = tid >> 7;
    for (int i = 0; i < b; ++i) {
        // first nonzero of row i at positions >= r (each warp redundantly: no broadcast sync)
        int c = -1;
        for (int base = r; base < w; base += 32) {
            const int cc = base + lane;
            const bool nz = cc < w && win[i][cc] != 0;
            const unsigned msk = __ballot_sync(0xffffffffu, nz);
            if (msk) {
                c = base + __ffs(msk) - 1;
                break;
            }
        }
        if (tid == 0) s_rank_before[i] = r;
        if (c < 0) {
            if (tid == 0) s_piv_of_row[i] = -1;
            continue;
        }
        __syncthreads();  // every warp is done reading row i
        if (c != r) {
            if (tid < b) {
                const u32 t = win[tid][r];
                win[tid][r] = win[tid][c];
                win[tid][c] = t;
            }
            __syncthreads();
        }
        const u32 pv = win[i][r];
        if (tid == 0) {
            s_piv_of_row[i] = r;
            s_rrp[r] = i;
            s_ipiv[r] = c;
            s_pv[r] = pv;
        }
        if (col > r && col < w) {
            const u32 ui = win[i][col];
            for (int k = i + 1 + half; k < b; k += 2) {
                const u32 fk = win[k][r];
                const u64 x = (u64)pv * win[k][col] + (u64)(fk ? f.p - fk : 0u) * ui;
                win[k][col] = red64(x, f);
            }
        }
        __syncthreads();
        ++r;
    }
    __syncthreads();
    const int rt = r;
    // prefix products Q_j = prod_{j'<j} pv_j'
    if (warp == 0) {
        u32 v0 = lane < rt ? s_pv[lane] : 1u;
        u32 v1 = (lane + 32) < rt ? s_pv[lane + 32] : 1u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const u32 t0 = __shfl_up_sync(0xffffffffu, v0, off);
            const u32 t1 = __shfl_up_sync(0xffffffffu, v1, off);
            if (lane >= off) {
                v0 = mulmod(v0, t0, f);
                v1 = mulmod(v1, t1, f);
            }
        }
        const u32 tot0 = __shfl_sync(0xffffffffu, v0, 31);
        u32 e0 = __shfl_up_sync(0xffffffffu, v0, 1);
        u32 e1 = __shfl_up_sync(0xffffffffu, v1, 1);
        if (lane == 0) {
            e0 = 1u % f.p;
            e1 = 1u % f.p;
        }
        s_Q[lane] = e0;
        s_Q[lane + 32] = mulmod(e1, tot0, f);
    }
    __syncthreads();
    if (tid < PB) {
        s_pvinv[tid] = tid < rt ? invmod(s_pv[tid], f) : 0u;
    } else if (tid < 2 * PB) {
        const int j = tid - PB;
        s_Qinv[j] = j < rt ? invmod(s_Q[j], f) : 0u;
    }
    __syncthreads();
    // true values of the window, written back in place
    for (int e = tid; e < b * PW; e += blockDim.x) {
        const int k = e / PW, cc = e % PW;
        if (cc >= w) continue;
        const int rb = s_rank_before[k];
        const int j = s_piv_of_row[k];
        u32 v = win[k][cc];
        if (cc < rb) v = mulmod(v, s_Qinv[cc], f);
        else if (j >= 0) v = mulmod(v, cc == j ? s_Qinv[j] : s_pvinv[j], f);
        a.A[(i64)(a.i0 + k) * a.lda + c0 + cc] = v;
    }
    // metadata for the tail kernel and the recursion
    for (int e = tid; e < PB * PB; e += blockDim.x) {
        const int i = e / PB, i2 = e % PB;
        u32 v = 0;
        if (i < b && i2 < i) {
            const int j2 = s_piv_of_row[i2];
            if (j2 >= 0) v = mulmod(win[i][j2], s_Qinv[j2], f);
        }
        ps->Cr[i][i2] = v;
    }
    for (int e = tid; e < PB; e += blockDim.x) {
        const bool real = e < b;
        ps->piv_of_row[e] = real ? s_piv_of_row[e] : -1;
        ps->rank_before[e] = real ? s_rank_before[e] : rt;
        if (e < rt) {
            const u32 ptrue = mulmod(s_pv[e], s_Qinv[e], f);
            ps->pivval[e] = ptrue;
            ps->pinv[e] = mulmod(s_pvinv[e], s_Q[e], f);
            a.rrp[c0 + e] = a.i0 + s_rrp[e];
            a.ipiv[c0 + e] = c0 + s_ipiv[e];
        }
        if (real) a.rp[a.i0 + 1 + e] = c0 + s_rank_before[e] + (s_piv_of_row[e] >= 0 ? 1 : 0);
    }
    if (tid == 0) {
        ps->w = w;
        ps->r = rt;
    }
}

// Exact leaf CUP over the full width in global memory: used only when a pivot
// lies beyond the window (structured / small-p inputs).  One CTA.
__device__ void panel_fallback(const PanelArgs& a, u32 (*Cr)[PB], const i32* piv, u32* red_buf) {
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x, nt = blockDim.x;
    const i32 c0 = ps->c0, w = ps->w, b = ps->b;
    const i32 N = a.N;
    u32* A = a.A;
    const i64 lda = a.lda;
    // 1. restore the original tail: P_i = (pivot ? u_i * P_j : res_i) + sum_{i'<i} Cr[i][i'] u_i'
    for (i32 colx = c0 + w + tid; colx < N; colx += nt) {
        u32 u[PB];
        for (int i = 0; i < b; ++i) {
            const u32 o = A[(i64)(a.i0 + i) * lda + colx];
            u32 acc = piv[i] >= 0 ? mulmod(o, ps->pivval[piv[i]], f) : o;
            for (int i2 = 0; i2 < i; ++i2) acc = addmod(acc, mulmod(Cr[i][i2], u[i2], f), f);
            u[i] = piv[i] >= 0 ? o : 0u;
            A[(i64)(a.i0 + i) * lda + colx] = acc;
        }
    }
    // 2. restore the original window
    for (int e = tid; e < b * PW; e += nt) {
        const int i = e / PW, c = e % PW;
        if (c < w) A[(i64)(a.i0 + i) * lda + c0 + c] = ps->win_orig[i][c];
    }
    __threadfence_block();
    __syncthreads();
    // 3. row-by-row elimination over columns [c0, N)
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
}

template <bool SMALLP>
__global__ void __launch_bounds__(256) panel_tail_kernel(PanelArgs a) {
    __shared__ u32 Cr[PB][PB];
    __shared__ i32 piv[PB];
    __shared__ u32 pinv[PB];
    __shared__ u32 red_buf[256];
    __shared__ int s_last;
    PanelScratch* ps = a.ps;
    const Fp f = a.f;
    const int tid = threadIdx.x;
    const i32 c0 = ps->c0, W = ps->W, w = ps->w, b = ps->b;
    const i32 col_begin = c0 + w;
    for (int e = tid; e < PB * PB; e += blockDim.x) Cr[e / PB][e % PB] = ps->Cr[e / PB][e % PB];
    for (int e = tid; e < PB; e += blockDim.x) {
        piv[e] = ps->piv_of_row[e];
        pinv[e] = ps->pinv[e];
    }
    __syncthreads();
    u32 bad = 0;
    if (W > w) {
        for (i32 colx = col_begin + blockIdx.x * blockDim.x + tid; colx < a.N;
             colx += gridDim.x * blockDim.x) {
            u32 P[PB];
            u32 nu[PB];
#pragma unroll
            for (int i = 0; i < PB; ++i)
                P[i] = i < b ? __ldcg(a.A + (i64)(a.i0 + i) * a.lda + colx) : 0u;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
                u64 acc = P[i];
#pragma unroll
                for (int i2 = 0; i2 < i; ++i2) {
                    if (SMALLP) acc += (u64)Cr[i][i2] * nu[i2];
                    else acc += mulmod(Cr[i][i2], nu[i2], f);
                }
                const u32 val = red64(acc, f);
                const int pj = piv[i];
                if (pj >= 0) {
                    const u32 u = mulmod(val, pinv[pj], f);
                    P[i] = u;
                    nu[i] = u ? f.p - u : 0u;
                } else {
                    P[i] = val;
                    nu[i] = 0;
                    bad |= val;
                }
            }
#pragma unroll
            for (int i = 0; i < PB; ++i)
                if (i < b) a.A[(i64)(a.i0 + i) * a.lda + colx] = P[i];
        }
    }
    if (__syncthreads_or(bad != 0) && tid == 0) atomicOr(&ps->flag, 1u);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&ps->counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (atomicAdd(&ps->flag, 0u) != 0) panel_fallback(a, Cr, piv, red_buf);
    if (tid == 0) {
        ps->counter = 0;
        ps->flag = 0;
    }
}

// X <- X * U^{-1}, U = unit upper block of the leaf's pivots (kernels.cpp:92-101
// with Diag::Unit: the stored diagonal -- C's pivots -- is never read).
template <bool SMALLP>
__global__ void __launch_bounds__(128) trsm_leaf_kernel(TrsmLeafArgs a) {
    __shared__ u32 nU[PB][PB + 1];
    const Fp f = a.f;
    const i32 j_lo = dyn_eval(a.j_lo, a.rp);
    const i32 nJ = dyn_eval(a.j_hi, a.rp) - j_lo;
    if (nJ <= 0 || a.M <= 0) return;
    for (int e = threadIdx.x; e < PB * PB; e += blockDim.x) {
        const int jj = e / PB, j = e % PB;
        u32 v = 0;
        if (jj < j && j < nJ) {
            const u32 u = __ldcg(a.A + (i64)__ldcg(a.rrp + j_lo + jj) * a.lda + j_lo + j);
            v = u ? f.p - u : 0u;
        }
        nU[jj][j] = v;
    }
    __syncthreads();
    for (i32 row = blockIdx.x * blockDim.x + threadIdx.x; row < a.M;
         row += gridDim.x * blockDim.x) {
        u32* xr = a.A + (i64)(a.row0 + row) * a.lda + j_lo;
        u32 x[PB];
#pragma unroll
        for (int j = 0; j < PB; ++j) x[j] = j < nJ ? __ldcg(xr + j) : 0u;
#pragma unroll
        for (int j = 1; j < PB; ++j) {
            u64 acc = x[j];
#pragma unroll
            for (int j2 = 0; j2 < j; ++j2) {
                if (SMALLP) acc += (u64)x[j2] * nU[j2][j];
                else acc += mulmod(x[j2], nU[j2][j], f);
            }
            x[j] = red64(acc, f);
        }
#pragma unroll
        for (int j = 0; j < PB; ++j)
            if (j < nJ) xr[j] = x[j];
    }
}

// Ordered compaction of {j in [lo, hi) : pred(j)} into list[], 256 threads.
// Returns the count (uniform).  Entries keep increasing order.
template <class Pred>
__device__ int collect_ordered(i32 lo, i32 hi, Pred pred, i32* list, int* warp_cnt) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const i32 j = lo + tid;
    const bool take = j < hi && pred(j);
    const unsigned msk = __ballot_sync(0xffffffffu, take);
    if (lane == 0) warp_cnt[warp] = __popc(msk);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w2 = 0; w2 < 8; ++w2) {
        if (w2 < warp) off += warp_cnt[w2];
        tot += warp_cnt[w2];
    }
    if (take) list[off + __popc(msk & ((1u << lane) - 1))] = j;
    __syncthreads();
    return tot;
}

__global__ void __launch_bounds__(256) swaps_kernel(SwapArgs a) {
    __shared__ i32 list[256];
    __shared__ int warp_cnt[8];
    const i32 j_lo = dyn_eval(a.j_lo, a.rp), j_hi = dyn_eval(a.j_hi, a.rp);
    if (j_hi <= j_lo) return;
    i32 M, g_lo = 0;
    if (a.gather) {
        g_lo = dyn_eval(a.g_lo, a.rp);
        M = dyn_eval(a.g_hi, a.rp) - g_lo;
    } else {
        M = a.M;
    }
    if (M <= 0) return;
    const i32 row_t = blockIdx.x * blockDim.x + threadIdx.x;
    // rows handled by this thread: row_t, row_t + stride, ...
    for (i32 j0 = j_lo; j0 < j_hi; j0 += 256) {
        const i32* ip = a.ipiv;
        const int cnt = collect_ordered(
            j0, min(j_hi, j0 + 256), [ip](i32 j) { return __ldcg(ip + j) != j; }, list, warp_cnt);
        if (cnt) {
            for (i32 t = row_t; t < M; t += gridDim.x * blockDim.x) {
                const i32 row = a.gather ? __ldcg(a.gather + g_lo + t) : a.row0 + t;
                u32* rr = a.A + (i64)row * a.lda;
                for (int q = 0; q < cnt; ++q) {
                    const i32 j = list[q];
                    const i32 c = __ldcg(ip + j);
                    const u32 tmp = rr[j];
                    rr[j] = rr[c];
                    rr[c] = tmp;
                }
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) compact_kernel(u32* A, i64 lda, i32 m, i32 n, const i32* rp,
                                                      const i32* rrp) {
    __shared__ i32 list[256];
    __shared__ int warp_cnt[8];
    const i32 r = __ldcg(rp + m);
    const i32 c = blockIdx.x * blockDim.x + threadIdx.x;
    for (i32 j0 = 0; j0 < r; j0 += 256) {
        if (j0 >= (i32)((blockIdx.x + 1) * blockDim.x)) break;  // uniform: no column here > j0
        const int cnt = collect_ordered(
            j0, min(r, j0 + 256), [rrp](i32 j) { return __ldcg(rrp + j) != j; }, list, warp_cnt);
        if (c < n) {
            for (int q = 0; q < cnt; ++q) {
                const i32 j = list[q];
                if (c > j) {
                    const i32 src = __ldcg(rrp + j);
                    A[(i64)j * lda + c] = A[(i64)src * lda + c];
                    A[(i64)src * lda + c] = 0;
                }
            }
        }
        __syncthreads();
    }
}

__global__ void gen_kernel(u32* A, i64 lda, i64 m, i64 n, u64 seed, Fp f) {
    const i64 total = m * n;
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (i64)gridDim.x * blockDim.x) {
        u64 z = seed + (u64)(t + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        const i64 i = t / n, j = t % n;
        A[i * lda + j] = red64(z, f);
    }
}

}  // namespace

void panel_window(const PanelArgs& a, cudaStream_t s) {
    panel_window_kernel<<<1, 256, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

void panel_tail(const PanelArgs& a, cudaStream_t s) {
    const int grid = std::max(1, std::min((a.N + 255) / 256, 2 * num_sms()));
    if (a.f.p <= 65536u) panel_tail_kernel<true><<<grid, 256, 0, s>>>(a);
    else panel_tail_kernel<false><<<grid, 256, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

void trsm_leaf(const TrsmLeafArgs& a, cudaStream_t s) {
    if (a.M <= 0) return;
    const int grid = std::max(1, std::min((a.M + 127) / 128, 4 * num_sms()));
    if (a.f.p <= 65536u) trsm_leaf_kernel<true><<<grid, 128, 0, s>>>(a);
    else trsm_leaf_kernel<false><<<grid, 128, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

void apply_swaps(const SwapArgs& a, cudaStream_t s) {
    if (a.Mmax <= 0) return;
    const int grid = std::max(1, std::min((a.Mmax + 255) / 256, 2 * num_sms()));
    swaps_kernel<<<grid, 256, 0, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

void compact_u_rows(u32* A, i64 lda, i32 m, i32 n, const i32* rp, const i32* rrp,
                    cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    compact_kernel<<<(n + 255) / 256, 256, 0, s>>>(A, lda, m, n, rp, rrp);
    RL_CUDA_CHECK(cudaGetLastError());
}

void gen_random_matrix(u32* A, i64 lda, i64 m, i64 n, u64 seed, u32 p, cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    const i64 total = m * n;
    const int grid = (int)std::min<i64>((total + 255) / 256, (i64)num_sms() * 32);
    gen_kernel<<<grid, 256, 0, s>>>(A, lda, m, n, seed, make_fp(p));
    RL_CUDA_CHECK(cudaGetLastError());
}

void fill_rp0(i32* rp, cudaStream_t s) { RL_CUDA_CHECK(cudaMemsetAsync(rp, 0, sizeof(i32), s)); }

}  // namespace rl
