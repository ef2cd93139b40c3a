// util.cu -- small device utilities of the C ABI:
//
//  * digest_u32: order-independent 64-bit digest of a device matrix (sum mod
//    2^64 of splitmix_mix((index << 32 | value) + golden)), the same function
//    as the oracle's oracle_digest_u32, so parity tests compare multi-GB
//    bodies (config 5: 17 GB) without copying them back;
//  * cup_tiny: CUP of a matrix of <= TINY_MAX entries in ONE launch -- the
//    input travels in the kernel's parameter block and every output (body,
//    rank, profile, pivot positions) is written straight into mapped pinned
//    host memory, so a call costs one launch and one stream synchronisation.
//    The reference's own callers make tens of millions of such calls
//    (acceptance.cpp:360-399: determinant of every 4x4 matrix over GF(3),
//    two threads); the algorithm is the iterative form of cup_rec
//    (factor.cpp:12-85): row i's pivot is the first
//    nonzero at positions >= rank, brought to position r by a transposition
//    of every row, the pivot stays raw, the rest of the row is scaled by its
//    inverse, later rows are eliminated, U rows move up at the end
//    (factor.cpp:62-70).
#include "kernels.cuh"
#include "runtime.h"
#include "util.h"

namespace rl {

namespace {

__device__ __forceinline__ u64 mix64(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void digest_kernel(const u32* __restrict__ A, i64 lda, i64 m, i64 n, unsigned long long* out) {
    u64 h = 0;
    for (i64 i = blockIdx.x; i < m; i += gridDim.x) {
        const u32* row = A + i * lda;
        const u64 base = (u64)(i * n);
        for (i64 j = threadIdx.x; j < n; j += blockDim.x)
            h += mix64((((base + (u64)j) << 32) | __ldg(row + j)) + 0x9E3779B97F4A7C15ull);
    }
    for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)h);
}

__device__ u32 inv_ext(u32 a, u32 p) {  // extended Euclid, a in [1, p)
    i64 t = 0, nt = 1;
    u32 r = p, nr = a;
    while (nr) {
        const u32 q = r / nr;
        const i64 tt = t - (i64)q * nt;
        t = nt;
        nt = tt;
        const u32 rr = r - q * nr;
        r = nr;
        nr = rr;
    }
    return (u32)(t < 0 ? t + p : t);
}

// One warp.  s[] holds the matrix row-major (m x n, m*n <= TINY_MAX).
__global__ void __launch_bounds__(32) cup_tiny_kernel(TinyIn in, TinyOut* out) {
    __shared__ u32 s[TINY_MAX];
    __shared__ i32 s_rrp[TINY_MAX], s_ipiv[TINY_MAX];
    const int lane = threadIdx.x;
    const int m = in.m, n = in.n;
    const Fp f = in.f;
    for (int e = lane; e < m * n; e += 32) s[e] = in.a[e];
    __syncwarp();
    int r = 0;
    for (int i = 0; i < m && r < n; ++i) {
        u32* ri = s + i * n;
        int c = -1;
        for (int j0 = r; j0 < n && c < 0; j0 += 32) {
            const int j = j0 + lane;
            const unsigned msk = __ballot_sync(0xffffffffu, j < n && ri[j] != 0);
            if (msk) c = j0 + __ffs(msk) - 1;
        }
        if (c < 0) continue;  // dead row: zero on [r, n)
        if (c != r) {         // transposition of positions r, c in every row (factor.cpp:23-24)
            for (int k = lane; k < m; k += 32) {
                const u32 t = s[k * n + r];
                s[k * n + r] = s[k * n + c];
                s[k * n + c] = t;
            }
            __syncwarp();
        }
        const u32 pinv = inv_ext(ri[r], f.p);
        for (int j = r + 1 + lane; j < n; j += 32) ri[j] = mulmod(ri[j], pinv, f);
        if (lane == 0) {
            s_rrp[r] = i;
            s_ipiv[r] = c;
        }
        __syncwarp();
        const int w = n - r - 1, rows = m - i - 1;
        for (int e = lane; e < rows * w; e += 32) {  // later rows: x_k -= x_k[r] * U_r
            const int k = i + 1 + e / w, j = r + 1 + e % w;
            const u32 fk = s[k * n + r];
            if (fk) s[k * n + j] = submod(s[k * n + j], mulmod(fk, ri[j], f), f);
        }
        __syncwarp();
        ++r;
    }
    for (int j = 0; j < r; ++j) {  // U row j from row rrp[j] (composed shift, factor.cpp:62-70)
        const int src = s_rrp[j];
        if (src != j) {
            for (int c2 = j + 1 + lane; c2 < n; c2 += 32) {
                s[j * n + c2] = s[src * n + c2];
                s[src * n + c2] = 0;
            }
        }
        __syncwarp();
    }
    for (int e = lane; e < m * n; e += 32) out->body[e] = s[e];
    for (int j = lane; j < r; j += 32) {
        out->rrp[j] = s_rrp[j];
        out->ipiv[j] = s_ipiv[j];
    }
    if (lane == 0) out->rank = r;
}

}  // namespace

void digest_u32(const u32* A, i64 lda, i64 m, i64 n, unsigned long long* d_out, cudaStream_t s) {
    RL_CUDA_CHECK(cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), s));
    if (m <= 0 || n <= 0) return;
    const int grid = (int)std::min<i64>(m, (i64)num_sms() * 8);
    digest_kernel<<<grid, 256, 0, s>>>(A, lda, m, n, d_out);
    RL_CUDA_CHECK(cudaGetLastError());
}

void cup_tiny(const TinyIn& in, TinyOut* out_mapped, cudaStream_t s) {
    cup_tiny_kernel<<<1, 32, 0, s>>>(in, out_mapped);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
