// batched.cu -- CUP of many small independent matrices (config 4: 4096 x 256^2).
//
// One CTA per matrix, the matrix in global memory (its 256 KB working set stays
// L2-resident with up to 8 CTAs per SM), rows processed in order with the
// reference pivot rule (factor.cpp:12-28) and eager right-looking elimination;
// U rows are placed at the end (factor.cpp:62-70 composed).  Outputs per
// matrix: rank, row profile and pivot positions (sigma is composed on the host).
#include <algorithm>

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
            s_pinv = invmod(ri[r], f);
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

}  // namespace

void cup_batched(u32* dA, i64 batch, i32 m, i32 n, i64 stride, u32 p, i32* d_ranks, i32* d_rrp,
                 i32* d_ipiv, i32 kcap, cudaStream_t s) {
    if (batch <= 0 || m <= 0 || n <= 0) return;
    // grid: one CTA per matrix (batch <= 2^31-1)
    cup_batched_kernel<<<(unsigned)batch, 256, 0, s>>>(dA, stride, m, n, make_fp(p), d_ranks, d_rrp,
                                                       d_ipiv, kcap);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
