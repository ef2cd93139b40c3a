// uinv.cuh -- inverse of a leaf's unit upper pivot block (shared by the U^{-1}
// kernel and the tail in panel.cu and by the window kernel, panel_window.cu).
// U, X, T: PB x (PB+1) words in shared memory; U holds the strict upper part
// (row i, column k > i, zero elsewhere), X receives U^{-1}.  Recursive doubling:
// the eight 8 x 8 diagonal blocks are inverted by eight warps at once, then pairs
// of s x s blocks merge (s = 8, 16, 32) through X_AB = -X_AA * (U_AB * X_BB), two
// fully parallel products per level (3 levels, 6 barriers).
#pragma once
#include "kernels.cuh"

namespace rl {
namespace uinv_detail {

// One doubling level: for every pair of SZ x SZ diagonal blocks (A, B):
// X_AB = -X_AA * (U_AB * X_BB).  The sums run over the full block width (X is
// zero below its diagonal), so the loops are fixed-length and unrolled.
template <bool SP, int SZ>
__device__ __forceinline__ void uinv_level(u32 (*U)[PB + 1], u32 (*X)[PB + 1], u32 (*T)[PB + 1], int tid,
                                           int nt, const Fp& f) {
    constexpr int NOUT = (PB / (2 * SZ)) * SZ * SZ;
    for (int e = tid; e < NOUT; e += nt) {
        const int pb = e / (SZ * SZ), rem = e % (SZ * SZ), i = rem / SZ, j = rem % SZ;
        const int A0 = pb * 2 * SZ, B0 = A0 + SZ;
        u64 acc = 0;
#pragma unroll
        for (int u = 0; u < SZ; ++u) {
            if (SP) acc += (u64)U[A0 + i][B0 + u] * X[B0 + u][B0 + j];
            else acc += mulmod(U[A0 + i][B0 + u], X[B0 + u][B0 + j], f);
        }
        T[A0 + i][B0 + j] = SP ? red_sp(acc, f) : red64(acc, f);
    }
    __syncthreads();
    for (int e = tid; e < NOUT; e += nt) {
        const int pb = e / (SZ * SZ), rem = e % (SZ * SZ), i = rem / SZ, j = rem % SZ;
        const int A0 = pb * 2 * SZ, B0 = A0 + SZ;
        u64 acc = 0;
#pragma unroll
        for (int u = 0; u < SZ; ++u) {
            if (SP) acc += (u64)X[A0 + i][A0 + u] * T[A0 + u][B0 + j];
            else acc += mulmod(X[A0 + i][A0 + u], T[A0 + u][B0 + j], f);
        }
        X[A0 + i][B0 + j] = negmod(SP ? red_sp(acc, f) : red64(acc, f), f);
    }
    __syncthreads();
}

}  // namespace uinv_detail

// X <- U^{-1} (rank rt <= PB: the diagonal is 1 below rt, 0 beyond; X must be
// zero below its diagonal on entry).  Every thread of the CTA calls it.
template <bool SP>
__device__ void uinv_solve(u32 (*U)[PB + 1], u32 (*X)[PB + 1], u32 (*T)[PB + 1], int rt, const Fp& f) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nt = blockDim.x;
    // diagonal blocks: warp w, lane c < 8 -> column c of block w
    if (warp < 8 && lane < 8) {
        const int base = 8 * warp, c = lane;
        u32 x[8];
#pragma unroll
        for (int i = 7; i >= 0; --i) {
            u64 acc = 0;
#pragma unroll
            for (int k = i + 1; k < 8; ++k)
                acc += SP ? (u64)U[base + i][base + k] * x[k] : (u64)mulmod(U[base + i][base + k], x[k], f);
            const u32 sum = SP ? red_sp(acc, f) : red64(acc, f);
            const u32 d = (i == c && base + i < rt) ? 1u % f.p : 0u;
            x[i] = i > c ? 0u : submod(d, sum, f);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) X[base + i][base + c] = x[i];
    }
    __syncthreads();
    uinv_detail::uinv_level<SP, 8>(U, X, T, tid, nt, f);
    uinv_detail::uinv_level<SP, 16>(U, X, T, tid, nt, f);
    uinv_detail::uinv_level<SP, 32>(U, X, T, tid, nt, f);
}

}  // namespace rl
