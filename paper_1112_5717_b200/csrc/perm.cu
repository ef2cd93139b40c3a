// perm.cu -- permutation application, final U-row placement and the seeded
// input generator.
//
// perm_apply_cols (proj/src/perm.cpp:115-125) is applied as the ordered list of
// transpositions T_{j, ipiv[j]} recorded by the pivot rule (perm.cpp:21-26,
// factor.cpp:23-24), in increasing j.  A job whose leaves made no
// transposition (per-leaf flags written by the panel kernels) returns at once;
// otherwise each chunk of 256 positions is composed into one gather map and
// applied by one warp per row (coalesced loads/stores of the moved positions).  The shift of factor.cpp:62-70, composed over the whole
// recursion, is one pass at the end (compact_kernel): per column, increasing j.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {

constexpr int SW = 1024;  // dense position window of one composed chunk

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

// Exclusive prefix of a per-thread flag over the CTA (256 threads); the caller
// adds the running total.  Contains barriers: every thread must call it.
__device__ __forceinline__ int collect_flag(bool take, int* warp_cnt) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned msk = __ballot_sync(0xffffffffu, take);
    __syncthreads();
    if (lane == 0) warp_cnt[warp] = __popc(msk);
    __syncthreads();
    int off = 0;
    for (int w2 = 0; w2 < warp; ++w2) off += warp_cnt[w2];
    return off + __popc(msk & ((1u << lane) - 1));
}

// One swap job: the ordered transpositions [j_lo, j_hi) on one set of rows.
__device__ __forceinline__ void swap_job(const SwapArgs& a, i32* list, int* warp_cnt) {
    if (a.leafflags) {  // no leaf of this job made a transposition: nothing to do
        int any = 0;
        for (i32 l = a.leaf_lo + (i32)threadIdx.x; l < a.leaf_hi; l += blockDim.x)
            any |= __ldcg(a.leafflags + l);
        if (!__syncthreads_or(any)) return;  // uniform
    }
    const i32 j_lo = dyn_eval(a.j_lo, a.rp), j_hi = dyn_eval(a.j_hi, a.rp);
    if (j_hi <= j_lo) return;  // uniform
    i32 M, g_lo = 0;
    if (a.gather) {
        g_lo = dyn_eval(a.g_lo, a.rp);
        M = dyn_eval(a.g_hi, a.rp) - g_lo;
    } else {
        M = a.M;
    }
    if (M <= 0) return;  // uniform
    // The transpositions of one chunk of (up to 256) consecutive positions are
    // composed ONCE per CTA into a gather map over a dense window of positions
    // [j0, j0 + SW): after the chunk, position j0 + u holds the value that was at
    // j0 + src[u] (laswp order: increasing j, each T_{j, ipiv[j]} with ipiv[j] >= j).
    // Then one WARP per row moves only the positions the chunk changes: loads
    // and stores of a row are issued together by 32 lanes (coalesced within the
    // window) instead of one thread walking the swaps of its row one dependent
    // pair at a time.  A chunk whose targets leave the window (a pivot found far
    // to the right) takes the per-row sequential walk.
    __shared__ i32 s_src[SW];
    __shared__ i32 s_mov[SW];
    __shared__ int s_far, s_nmov;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (i32 j0 = j_lo; j0 < j_hi; j0 += 256) {
        const i32* ip = a.ipiv;
        const int cnt = collect_ordered(
            j0, min(j_hi, j0 + 256), [ip](i32 j) { return __ldcg(ip + j) != j; }, list, warp_cnt);
        if (!cnt) continue;  // uniform (collect_ordered ends with a barrier)
        for (int u = threadIdx.x; u < SW; u += blockDim.x) s_src[u] = u;
        if (threadIdx.x == 0) s_far = 0;
        __syncthreads();
        if (threadIdx.x < cnt && __ldcg(ip + list[threadIdx.x]) >= j0 + SW) s_far = 1;
        __syncthreads();
        if (!s_far) {
            if (threadIdx.x == 0) {  // compose in order (positions are window-relative)
                for (int q = 0; q < cnt; ++q) {
                    const int x = list[q] - j0, y = __ldcg(ip + list[q]) - j0;
                    const i32 t = s_src[x];
                    s_src[x] = s_src[y];
                    s_src[y] = t;
                }
            }
            __syncthreads();
            // the positions that change, compacted
            int nm = 0;
            for (int u0 = 0; u0 < SW; u0 += blockDim.x) {
                const int u = u0 + threadIdx.x;
                const bool mv = u < SW && s_src[u] != u;
                const int k = collect_flag(mv, warp_cnt);
                if (mv) s_mov[nm + k] = u;
                nm += __syncthreads_count(mv);
            }
            if (threadIdx.x == 0) s_nmov = nm;
            __syncthreads();
            const int nmov = s_nmov;
            for (i32 t = blockIdx.x * nwarp + warp; t < M; t += gridDim.x * nwarp) {
                const i32 row = a.gather ? __ldcg(a.gather + g_lo + t) : a.row0 + t;
                u32* rr = a.A + (i64)row * a.lda + j0;
                // every value of the window is read before any is written
                u32 v[SW / 32];
#pragma unroll
                for (int q = 0; q < SW / 32; ++q) {
                    const int k = lane + 32 * q;
                    if (k < nmov) v[q] = rr[s_src[s_mov[k]]];
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < SW / 32; ++q) {
                    const int k = lane + 32 * q;
                    if (k < nmov) rr[s_mov[k]] = v[q];
                }
            }
        } else {
            const i32 row_t = blockIdx.x * blockDim.x + threadIdx.x;
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

// Consecutive swap jobs of the recursion touch disjoint row sets (the top
// halves of nested nodes, then a bottom half), so one launch runs them all;
// within a job every row is owned by one thread, which keeps the order.
__global__ void __launch_bounds__(256) swaps_kernel(SwapJobs jobs) {
    __shared__ i32 list[256];
    __shared__ int warp_cnt[8];
    pdl_wait();
    pdl_trigger();
    for (int q = 0; q < jobs.n; ++q) swap_job(jobs.job[q], list, warp_cnt);
}

// One CTA per 32-column block.  The moves "row j <- row rrp[j] on columns > j,
// source zeroed" of a chunk of (up to 256) non-trivial pivots are done in three
// parallel phases: read every source (they are original rows: rrp is strictly
// increasing and rrp[j] >= j, so no earlier move wrote them), zero the sources,
// write the destinations (a destination that is also a source of the same
// chunk is zeroed first, as in the sequential order).  Many independent
// coalesced loads are in flight instead of one dependent load per pivot.
__global__ void __launch_bounds__(256) compact_kernel(u32* A, i64 lda, i32 m, i32 n, const i32* rp,
                                                      const i32* rrp) {
    __shared__ i32 list[256];
    __shared__ int warp_cnt[8];
    __shared__ u32 S[256][32];
    pdl_wait();
    pdl_trigger();
    const i32 r = __ldcg(rp + m);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const i32 c = blockIdx.x * 32 + lane;
    for (i32 j0 = 0; j0 < r; j0 += 256) {
        if (j0 >= (i32)((blockIdx.x + 1) * 32)) break;  // uniform: no column here > j0
        const int cnt = collect_ordered(
            j0, min(r, j0 + 256), [rrp](i32 j) { return __ldcg(rrp + j) != j; }, list, warp_cnt);
        if (cnt == 0) continue;  // uniform
        for (int q = warp; q < cnt; q += 8) {
            const i32 j = list[q];
            if (c < n && c > j) S[q][lane] = A[(i64)__ldcg(rrp + j) * lda + c];
        }
        __syncthreads();
        for (int q = warp; q < cnt; q += 8) {
            const i32 j = list[q];
            if (c < n && c > j) A[(i64)__ldcg(rrp + j) * lda + c] = 0;
        }
        __syncthreads();
        for (int q = warp; q < cnt; q += 8) {
            const i32 j = list[q];
            if (c < n && c > j) A[(i64)j * lda + c] = S[q][lane];
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

void apply_swaps(const SwapJobs& jobs, cudaStream_t s) {
    int mmax = 0;
    for (int q = 0; q < jobs.n; ++q) mmax = std::max(mmax, jobs.job[q].Mmax);
    if (jobs.n <= 0 || mmax <= 0) return;
    // one warp per row in the composed path (8 rows per CTA per pass)
    const int grid = std::max(1, std::min((mmax + 7) / 8, 2 * num_sms()));
    RL_ONCE_MAX_SMEM(swaps_kernel);
    launch_pdl(swaps_kernel, dim3(grid), dim3(256), 0, s, jobs);
    RL_CUDA_CHECK(cudaGetLastError());
}

void compact_u_rows(u32* A, i64 lda, i32 m, i32 n, const i32* rp, const i32* rrp,
                    cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    RL_ONCE_MAX_SMEM(compact_kernel);
    launch_pdl(compact_kernel, dim3((n + 31) / 32), dim3(256), 0, s, A, lda, m, n, rp, rrp);
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
