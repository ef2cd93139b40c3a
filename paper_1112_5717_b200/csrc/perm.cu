// perm.cu -- permutation application, final U-row placement and the seeded
// input generator.
//
// perm_apply_cols (proj/src/perm.cpp:115-125) is applied as the ordered list of
// transpositions T_{j, ipiv[j]} recorded by the pivot rule (perm.cpp:21-26,
// factor.cpp:23-24), in increasing j.  A job whose leaves made no
// transposition (per-leaf flags written by the panel kernels) returns at once;
// otherwise each chunk of 256 positions is composed into one gather map (in
// parallel, far targets included) and applied by one warp per row (all loads of
// the moved positions in flight together, then all stores).  The shift of factor.cpp:62-70, composed over the whole
// recursion, is one pass at the end (compact_kernel): per column, increasing j.
#include <algorithm>
#include <climits>

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
//
// The transpositions of one chunk of (up to 256) consecutive positions j are
// composed ONCE per CTA into a gather map over SLOTS: slot u < SW is position
// j0 + u (the dense window the chunk's own positions and its near targets fall
// in), slots SW + i are the distinct far targets ipiv[j] >= j0 + SW (sorted).
// After the chunk, slot u holds the value that was at slot src[u] (laswp order:
// increasing j, each T_{j, ipiv[j]} with ipiv[j] >= j).  The map is built in
// parallel: every touched slot walks the chunk's transpositions backwards
// (cur <- the other end of each transposition that touches cur), so no thread
// runs a serial chain of dependent shared-memory swaps.  Then one WARP per row
// moves only the positions the chunk changes: every value is read before any
// is written, the loads and stores of a row are issued together by 32 lanes
// (independent, in flight at once) instead of one thread walking the swaps of
// its row one dependent pair at a time.
constexpr int NFAR = 256;          // far slots: at most one per transposition
constexpr int NSLOT = SW + NFAR;
constexpr int MV_PER_LANE = NSLOT / 32;

struct SwapSmem {
    i32 list[256];      // positions j of the chunk with ipiv[j] != j, increasing
    int2 tr[256];       // their transpositions as (slot of j, slot of ipiv[j])
    i32 farv[256];      // per transposition: its far target (INT_MAX if near)
    i32 ffv[256];       // the same at the first occurrence of each value only
    i32 farpos[NFAR];   // distinct far targets, increasing (slot SW + i)
    i32 src[NSLOT];     // composed gather map (slots)
    i32 mov[NSLOT];     // slots whose value changes, compacted
    int warp_cnt[8];
    int nfar, nmov;
};

__device__ __forceinline__ i32 slot_pos(const SwapSmem& S, i32 j0, i32 u) {
    return u < SW ? j0 + u : S.farpos[u - SW];
}

__device__ __forceinline__ void swap_job(const SwapArgs& a, SwapSmem& S) {
    const int tid = threadIdx.x;
    if (a.leafflags) {  // no leaf of this job made a transposition: nothing to do
        int any = 0;
        for (i32 l = a.leaf_lo + (i32)tid; l < a.leaf_hi; l += blockDim.x) any |= __ldcg(a.leafflags + l);
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
    const int warp = tid >> 5, lane = tid & 31, nwarp = blockDim.x >> 5;
    for (i32 j0 = j_lo; j0 < j_hi; j0 += 256) {
        const i32* ip = a.ipiv;
        const int cnt = collect_ordered(
            j0, min(j_hi, j0 + 256), [ip](i32 j) { return __ldcg(ip + j) != j; }, S.list, S.warp_cnt);
        if (!cnt) continue;  // uniform (collect_ordered ends with a barrier)
        // far targets: distinct values, ranked
        const i32 y = tid < cnt ? __ldcg(ip + S.list[tid]) : 0;
        const bool far = tid < cnt && y >= j0 + SW;
        S.farv[tid] = far ? y : INT_MAX;
        for (int u = tid; u < NSLOT; u += blockDim.x) S.src[u] = u;
        __syncthreads();
        bool first = far;  // first occurrence of its value
        if (far)
            for (int q = 0; q < tid; ++q) first &= S.farv[q] != y;
        S.ffv[tid] = first ? y : INT_MAX;
        const int nfar = __syncthreads_count(first);
        int rk = 0;  // distinct far targets below y
        if (far)
            for (int q = 0; q < cnt; ++q) rk += S.ffv[q] < y ? 1 : 0;
        if (first) S.farpos[rk] = y;
        if (tid < cnt) S.tr[tid] = make_int2(S.list[tid] - j0, far ? SW + rk : y - j0);
        __syncthreads();
        // composed map, in parallel: slot u's final value came from the slot
        // reached by walking the transpositions backwards from u
        for (int u = tid; u < SW + nfar; u += blockDim.x) {
            i32 cur = u;
            for (int q = cnt - 1; q >= 0; --q) {
                const int2 t = S.tr[q];
                cur = cur == t.x ? t.y : (cur == t.y ? t.x : cur);
            }
            S.src[u] = cur;
        }
        __syncthreads();
        // the slots that change, compacted
        int nm = 0;
        for (int u0 = 0; u0 < SW + nfar; u0 += blockDim.x) {
            const int u = u0 + tid;
            const bool mv = u < SW + nfar && S.src[u] != u;
            const int k = collect_flag(mv, S.warp_cnt);
            if (mv) S.mov[nm + k] = u;
            nm += __syncthreads_count(mv);
        }
        const int nmov = nm;
        for (i32 t = blockIdx.x * nwarp + warp; t < M; t += gridDim.x * nwarp) {
            const i32 row = a.gather ? __ldcg(a.gather + g_lo + t) : a.row0 + t;
            u32* rr = a.A + (i64)row * a.lda;
            // every value of the row's moved slots is read before any is written
            u32 v[MV_PER_LANE];
#pragma unroll
            for (int q = 0; q < MV_PER_LANE; ++q) {
                const int k = lane + 32 * q;
                if (k < nmov) v[q] = rr[slot_pos(S, j0, S.src[S.mov[k]])];
            }
            __syncwarp();
#pragma unroll
            for (int q = 0; q < MV_PER_LANE; ++q) {
                const int k = lane + 32 * q;
                if (k < nmov) rr[slot_pos(S, j0, S.mov[k])] = v[q];
            }
        }
        __syncthreads();
    }
}

// Consecutive swap jobs of the recursion touch disjoint row sets (the top
// halves of nested nodes, then a bottom half), so one launch runs them all;
// within a job every row is owned by one warp, which keeps the order.
__global__ void __launch_bounds__(256) swaps_kernel(SwapJobs jobs) {
    __shared__ SwapSmem S;
    pdl_wait();
    pdl_trigger();
    for (int q = 0; q < jobs.n; ++q) swap_job(jobs.job[q], S);
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

namespace {
__global__ void bump_epoch_kernel(i32* e) { *e += 1; }
}  // namespace
void bump_epoch(i32* epoch, cudaStream_t s) {
    bump_epoch_kernel<<<1, 1, 0, s>>>(epoch);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
