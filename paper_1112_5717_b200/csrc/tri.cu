// tri.cu -- dense mod-p GEMM driver, triangular inverses, and the operation
// tallies of the reference's triangular routines (see tri.h).
//
// Triangular inverse (trtri, proj/src/tri.cpp:13-40).  The reference recurses
// T = [[T1, V], [0, T2]] -> V <- -T1^{-1} V T2^{-1} with two triangular solves
// per level.  Here the 64 x 64 diagonal blocks are inverted first, all at once
// (one CTA per block, substitution in shared memory), and the levels above are
// two tensor-core GEMMs each on the dense triangle (zeros in the other half):
//     W <- V * T2^{-1};   V <- -(T1^{-1} * W)          (upper)
//     W <- V * T1^{-1};   V <- -(T2^{-1} * W)          (lower, V = T21)
// The inverse is unique, so this schedule is bit-exact with the reference.
#include <algorithm>
#include <vector>

#include "kernels.cuh"
#include "runtime.h"
#include "tri.h"

namespace rl {

namespace {

constexpr int TB = 64;  // diagonal block of the base inversion

__global__ void scale_kernel(u32* C, i64 ldc, i64 m, i64 n, u32 beta, Fp f) {
    const i64 total = m * n;
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (i64)gridDim.x * blockDim.x) {
        u32* c = C + (t / n) * ldc + (t % n);
        *c = beta == 0 ? 0u : mulmod(*c, beta, f);
    }
}

__global__ void tri_extract_kernel(u32* X, i64 ldx, const u32* S, i64 lds, i32 k, int upper,
                                   int unit, u32 one) {
    const i64 total = (i64)k * k;
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (i64)gridDim.x * blockDim.x) {
        const i32 i = (i32)(t / k), j = (i32)(t % k);
        u32 v = 0;
        if (i == j) v = unit ? one : S[(i64)i * lds + j];
        else if (upper ? j > i : j < i) v = S[(i64)i * lds + j];
        X[(i64)i * ldx + j] = v;
    }
}

__global__ void tri_store_kernel(u32* D, i64 ldd, const u32* X, i64 ldx, i32 k, int upper) {
    const i64 total = (i64)k * k;
    for (i64 t = (i64)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (i64)gridDim.x * blockDim.x) {
        const i32 i = (i32)(t / k), j = (i32)(t % k);
        if (upper ? j > i : j < i) D[(i64)i * ldd + j] = X[(i64)i * ldx + j];
    }
}

// One CTA per TB x TB diagonal block of X, thread j = column j of the block's
// inverse by substitution.  The sums run over the full block width (entries of
// R outside the triangle are zero), so every thread follows the same loop.
template <bool SP>
__global__ void __launch_bounds__(TB) tri_inv_base_kernel(u32* X, i64 ldx, i32 k, int upper, Fp f) {
    __shared__ u32 T[TB][TB + 1];
    __shared__ u32 R[TB][TB + 1];
    __shared__ u32 dinv[TB];
    const i32 o = blockIdx.x * TB;
    const int bs = min(TB, k - o);
    const int tid = threadIdx.x;
    for (int e = tid; e < TB * TB; e += TB) {
        const int i = e / TB, j = e % TB;
        T[i][j] = (i < bs && j < bs) ? X[(i64)(o + i) * ldx + o + j] : 0u;
        R[i][j] = 0;
    }
    __syncthreads();
    if (tid < bs) dinv[tid] = invmod(T[tid][tid], f);
    __syncthreads();
    const int j = tid;
    for (int step = 0; step < bs; ++step) {
        const int i = upper ? bs - 1 - step : step;
        u64 acc = 0;
        if (upper) {
            for (int u = i + 1; u < bs; ++u)
                acc += SP ? (u64)T[i][u] * R[u][j] : (u64)mulmod(T[i][u], R[u][j], f);
        } else {
            for (int u = 0; u < i; ++u)
                acc += SP ? (u64)T[i][u] * R[u][j] : (u64)mulmod(T[i][u], R[u][j], f);
        }
        u32 v = 0;
        if (i == j) {
            v = dinv[i];
        } else if (upper ? i < j : i > j) {
            const u32 sred = SP ? red_sp(acc, f) : red64(acc, f);
            v = mulmod(negmod(sred, f), dinv[i], f);
        }
        if (j < bs) R[i][j] = v;
        __syncthreads();
    }
    for (int e = tid; e < bs * bs; e += TB) {
        const int i = e / bs, jj = e % bs;
        X[(i64)(o + i) * ldx + o + jj] = R[i][jj];
    }
}

__global__ void compress_kernel(u32* A, i64 lda, i32 r, const i32* rrp) {
    const i32 c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= r) return;
    for (i32 j = c; j < r; ++j) {
        const i32 src = rrp[j];
        if (src == j) continue;
        u32* a = A + (i64)j * lda + c;
        u32* b = A + (i64)src * lda + c;
        const u32 t = *a;
        *a = *b;
        *b = t;
    }
}

__global__ void gather_rows_kernel(u32* T, const u32* A, i64 lda, i64 ncols, const i32* idx,
                                   i32 count) {
    for (i32 t = blockIdx.y; t < count; t += gridDim.y) {
        const u32* src = A + (i64)idx[2 * t + 1] * lda;
        for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < ncols;
             c += (i64)gridDim.x * blockDim.x)
            T[(i64)t * ncols + c] = src[c];
    }
}

__global__ void scatter_rows_kernel(u32* A, i64 lda, const u32* T, i64 ncols, const i32* idx,
                                    i32 count) {
    for (i32 t = blockIdx.y; t < count; t += gridDim.y) {
        u32* dst = A + (i64)idx[2 * t] * lda;
        for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < ncols;
             c += (i64)gridDim.x * blockDim.x)
            dst[c] = T[(i64)t * ncols + c];
    }
}

int grid_for(i64 work, int threads = 256) {
    return (int)std::max<i64>(1, std::min<i64>((work + threads - 1) / threads, (i64)num_sms() * 16));
}

void tri_inv_rec(u32* X, i64 ldx, i32 k, bool upper, const Fp& f, DevBuf& wbuf, cudaStream_t s) {
    if (k <= TB) return;
    const i32 h = TB * ((k + 2 * TB - 1) / (2 * TB));  // multiple of TB, TB <= h < k
    u32* X11 = X;
    u32* X22 = X + (i64)h * ldx + h;
    tri_inv_rec(X11, ldx, h, upper, f, wbuf, s);
    tri_inv_rec(X22, ldx, k - h, upper, f, wbuf, s);
    const u32 neg1 = f.p - 1;
    u32* W = (u32*)wbuf.get((size_t)h * (k - h) * 4);
    if (upper) {
        u32* V = X + h;  // h x (k - h)
        mm_dense(V, ldx, X22, ldx, W, k - h, h, k - h, k - h, 1 % f.p, 0, f, s);
        mm_dense(X11, ldx, W, k - h, V, ldx, h, h, k - h, neg1, 0, f, s);
    } else {
        u32* V = X + (i64)h * ldx;  // (k - h) x h
        mm_dense(V, ldx, X11, ldx, W, h, k - h, h, h, 1 % f.p, 0, f, s);
        mm_dense(X22, ldx, W, h, V, ldx, k - h, k - h, h, neg1, 0, f, s);
    }
}

}  // namespace

void mm_dense(const u32* A, i64 lda, const u32* B, i64 ldb, u32* C, i64 ldc, i64 m, i64 l, i64 n,
              u32 alpha, u32 beta, const Fp& f, cudaStream_t s, int max_ctas) {
    if (m == 0 || n == 0) return;
    const u32 p = f.p;
    if (alpha == 0 || l == 0) {  // kernels.cpp:43-52: product short-circuited
        if (beta == 1 % p) return;
        scale_kernel<<<grid_for(m * n), 256, 0, s>>>(C, ldc, m, n, beta, f);
        RL_CUDA_CHECK(cudaGetLastError());
        return;
    }
    const int L = limbs_for(p);
    const i64 kmax = tc_kmax(L);
    // Chunk K so every s32 accumulator stays exact; later chunks accumulate (beta = 1).
    for (i64 k0 = 0; k0 < l; k0 += kmax) {
        const i64 kc = std::min(kmax, l - k0);
        GemmArgs g{};
        g.A = A + k0;
        g.lda = lda;
        g.a_row0 = 0;
        g.B = B + k0 * ldb;
        g.ldb = ldb;
        g.gather = nullptr;
        g.C = C;
        g.ldc = ldc;
        g.c_row0 = 0;
        g.M = (i32)m;
        g.k_lo = dyn_c(0);
        g.k_hi = dyn_c((i32)kc);
        g.n_lo = dyn_c(0);
        g.n_hi = dyn_c((i32)n);
        g.rp = nullptr;
        g.alpha = alpha;
        g.beta = k0 == 0 ? beta : 1 % p;
        g.f = f;
        g.max_ctas = max_ctas;
        const bool tc = kc >= 32 && n >= 32 && m >= 32;
        if (tc) {
            // workspaces of the calling stream's context: concurrent mm_dense
            // calls on distinct streams never share them
            Scratch& sc = scratch_for(s);
            uint8_t* pa = (uint8_t*)sc.get(SS_MM_A2, tc_a2_bytes(L, m, kc));
            uint8_t* pb = (uint8_t*)sc.get(SS_MM_B2, tc_b2_bytes(L, n, kc));
            gemm_tc(g, L, kc, n, pa, pb, s);
        } else {
            gemm_simt(g, kc, n, s);
        }
    }
}

void tri_extract(u32* X, i64 ldx, const u32* S, i64 lds, i32 k, bool upper, bool unit, u32 p,
                 cudaStream_t s) {
    if (k <= 0) return;
    tri_extract_kernel<<<grid_for((i64)k * k), 256, 0, s>>>(X, ldx, S, lds, k, upper, unit, 1 % p);
    RL_CUDA_CHECK(cudaGetLastError());
}

void tri_store_strict(u32* D, i64 ldd, const u32* X, i64 ldx, i32 k, bool upper, cudaStream_t s) {
    if (k <= 1) return;
    tri_store_kernel<<<grid_for((i64)k * k), 256, 0, s>>>(D, ldd, X, ldx, k, upper);
    RL_CUDA_CHECK(cudaGetLastError());
}

void tri_inverse(u32* X, i64 ldx, i32 k, bool upper, const Fp& f, cudaStream_t s) {
    if (k <= 0) return;
    const int nb = (k + TB - 1) / TB;
    if (f.p <= 65536u) tri_inv_base_kernel<true><<<nb, TB, 0, s>>>(X, ldx, k, upper, f);
    else tri_inv_base_kernel<false><<<nb, TB, 0, s>>>(X, ldx, k, upper, f);
    RL_CUDA_CHECK(cudaGetLastError());
    tri_inv_rec(X, ldx, k, upper, f, scratch_for(s).buf[SS_TRI_W], s);
}

void compress_pivot_rows(u32* A, i64 lda, i32 r, const i32* d_rrp, cudaStream_t s) {
    if (r <= 0) return;
    compress_kernel<<<(r + 127) / 128, 128, 0, s>>>(A, lda, r, d_rrp);
    RL_CUDA_CHECK(cudaGetLastError());
}

void move_rows(u32* A, i64 lda, i64 ncols, const i32* d_idx, i32 count, cudaStream_t s) {
    if (count <= 0 || ncols <= 0) return;
    u32* T = (u32*)scratch_for(s).get(SS_MOVE, (size_t)count * ncols * 4);
    const dim3 grid((unsigned)std::min<i64>((ncols + 255) / 256, 64), (unsigned)std::min(count, 4096));
    gather_rows_kernel<<<grid, 256, 0, s>>>(T, A, lda, ncols, d_idx, count);
    RL_CUDA_CHECK(cudaGetLastError());
    scatter_rows_kernel<<<grid, 256, 0, s>>>(A, lda, T, ncols, d_idx, count);
    RL_CUDA_CHECK(cudaGetLastError());
}

// ------------------------------------------------------------- op tallies
// mm with alpha in {1, -1} and beta = 1 (every call inside trsm/trmm/trulm):
// l mul, l-1 add and the accumulate per output (kernels.cpp:53-73).
static void tally_mm_acc(OpTally& t, i64 m, i64 n, i64 l) {
    if (m == 0 || n == 0 || l == 0) return;
    const u64 e = (u64)m * (u64)n * (u64)l;
    t.mul += e;
    t.addsub += e;
}

// trsm_base (kernels.cpp:80-133): per index one inverse (NonUnit), per output
// row/column a dot product of the already-solved part and the NonUnit scaling.
static void tally_tri_base(OpTally& t, bool unit, i64 k, i64 width, bool solve) {
    const u64 tri = (u64)k * (u64)(k - 1) / 2;
    t.mul += (u64)width * tri + (unit ? 0 : (u64)width * (u64)k);
    t.addsub += (u64)width * tri;
    if (solve && !unit) t.divinv += (u64)k;
}

void tally_trsm(OpTally& t, int side, int uplo, bool unit, i64 k, i64 rows, i64 cols, i64 thr) {
    if (k == 0 || rows == 0 || cols == 0) return;
    if (thr < 1) thr = 1;
    if (k <= thr) {
        tally_tri_base(t, unit, k, side == SIDE_RIGHT ? rows : cols, true);
        return;
    }
    const i64 h = k / 2;
    // kernels.cpp:149-172: two half solves around one update
    if (side == SIDE_RIGHT) {
        tally_trsm(t, side, uplo, unit, h, rows, h, thr);
        tally_trsm(t, side, uplo, unit, k - h, rows, k - h, thr);
        if (uplo == UPLO_UPPER) tally_mm_acc(t, rows, k - h, h);
        else tally_mm_acc(t, rows, h, k - h);
    } else {
        tally_trsm(t, side, uplo, unit, h, h, cols, thr);
        tally_trsm(t, side, uplo, unit, k - h, k - h, cols, thr);
        if (uplo == UPLO_UPPER) tally_mm_acc(t, h, cols, k - h);
        else tally_mm_acc(t, k - h, cols, h);
    }
}

// trmm_rec (kernels.cpp:223-261) at threshold 1.
static void tally_trmm(OpTally& t, int side, int uplo, bool unit, i64 k, i64 rows, i64 cols) {
    if (k == 0 || rows == 0 || cols == 0) return;
    if (k <= 1) {
        tally_tri_base(t, unit, k, side == SIDE_RIGHT ? rows : cols, false);
        return;
    }
    const i64 h = k / 2;
    if (side == SIDE_RIGHT) {
        tally_trmm(t, side, uplo, unit, h, rows, h);
        tally_trmm(t, side, uplo, unit, k - h, rows, k - h);
        if (uplo == UPLO_UPPER) tally_mm_acc(t, rows, k - h, h);
        else tally_mm_acc(t, rows, h, k - h);
    } else {
        tally_trmm(t, side, uplo, unit, h, h, cols);
        tally_trmm(t, side, uplo, unit, k - h, k - h, cols);
        if (uplo == UPLO_UPPER) tally_mm_acc(t, h, cols, k - h);
        else tally_mm_acc(t, k - h, cols, h);
    }
}

// trtri (tri.cpp:13-40); the upper and lower recursions charge identically
// (their two solves have the same triangle sizes and right-hand sides).
void tally_trtri(OpTally& t, bool unit, i64 n) {
    if (n == 0) return;
    if (n == 1) {
        if (!unit) t.divinv += 1;
        return;
    }
    const i64 h = n / 2;
    tally_trsm(t, SIDE_RIGHT, UPLO_UPPER, unit, n - h, h, n - h, 1);
    tally_trsm(t, SIDE_LEFT, UPLO_UPPER, unit, h, h, n - h, 1);
    t.addsub += (u64)h * (u64)(n - h);  // V <- -V
    tally_trtri(t, unit, h);
    tally_trtri(t, unit, n - h);
}

// trulm with DiagOwner::LowerOwnsDiag (tri.cpp:42-63).
void tally_trulm_lower_owns(OpTally& t, i64 n) {
    if (n <= 1) return;
    const i64 h = n / 2;
    tally_trulm_lower_owns(t, h);
    tally_mm_acc(t, h, h, n - h);
    tally_trmm(t, SIDE_RIGHT, UPLO_LOWER, /*unit=*/false, n - h, h, n - h);
    tally_trmm(t, SIDE_LEFT, UPLO_UPPER, /*unit=*/true, n - h, n - h, h);
    tally_trulm_lower_owns(t, n - h);
}

// echelon.cpp:5-47 after the cup.
void tally_echelon(OpTally& t, i64 m, i64 n, i64 r, bool reduced) {
    tally_trsm(t, SIDE_LEFT, UPLO_UPPER, /*unit=*/true, r, r, n - r, 1);
    t.addsub += (u64)r * (u64)(n - r);
    tally_trtri(t, /*unit=*/true, r);
    if (!reduced) return;
    tally_trsm(t, SIDE_RIGHT, UPLO_LOWER, /*unit=*/false, r, m - r, r, 1);
    tally_trtri(t, /*unit=*/false, r);
    tally_trulm_lower_owns(t, r);
}

}  // namespace rl

namespace rl {
namespace {
__global__ void __launch_bounds__(256) transpose_kernel(u32* D, i64 ldd, const u32* S, i64 lds, i64 rows,
                                                        i64 cols) {
    __shared__ u32 t[32][33];
    const i64 r0 = (i64)blockIdx.y * 32, c0 = (i64)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows per pass
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const i64 r = r0 + ty + k, c = c0 + tx;
        if (r < rows && c < cols) t[ty + k][tx] = S[r * lds + c];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const i64 c = c0 + ty + k, r = r0 + tx;
        if (r < rows && c < cols) D[c * ldd + r] = t[tx][ty + k];
    }
}
}  // namespace

void transpose(u32* D, i64 ldd, const u32* S, i64 lds, i64 rows, i64 cols, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    const dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_kernel<<<grid, 256, 0, s>>>(D, ldd, S, lds, rows, cols);
    RL_CUDA_CHECK(cudaGetLastError());
}
}  // namespace rl
