// trsm_tc.cu -- the fused node TRSM of trsm.cu on the legacy tensor cores.
//
// trsm(Right, Upper, Unit) against a skeleton node X of at most 4 leaves
// (proj/src/factor.cpp:45-46, the recursion of kernels.cpp:135-154): per row
// tile of G, leaf by leaf,
//     B_l <- B_l - sum_{l2 < l} G_l2 * U_{l2,l}      G_l = B_l * Uinv_l
// (block forward substitution; Uinv_l precomputed by the leaf's panel).  The
// CUDA-core kernel (trsm.cu) spends its time in 64-bit multiply-adds (C3:
// 25-35 us per 4-leaf node on the critical path); here every product is
// mma.sync m16n8k32 u8 x u8 -> s32 on two byte limbs (p <= 2^16: S0 = lo*lo,
// S1 = lo*hi + hi*lo, S2 = hi*hi; each sum of at most 64 products of bytes is
// below 2^31), combined in 64 bits and reduced once per output.  The U blocks
// are staged once per CTA as transposed byte planes [column][k], the solved
// G_l as byte planes [row][k] per leaf (64-byte k stride per leaf, so a leaf of
// any rank starts on an aligned fragment).  Rows beyond M are the identity over
// the node's pivots, so the same sweep yields U_X^{-1} (written to ninv).
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {

constexpr int TBP = 80;             // byte-plane pitch (bytes) of a 64-deep k row
constexpr int TTM = 32;             // rows of G per tile
constexpr int TGW = TN_MAXLEAF * PB + 4;  // pitch (words) of the u32 G tile
constexpr int TSTAGE = 5;           // U blocks staged per round (u32 scratch = 80 KB)

__device__ __forceinline__ u32 lob(u32 v, int s) { return (v >> s) & 0xff; }

// acc[t][e] = A(16 rows at r0, K = 64) * B(8 columns at n0 + 8t, K = 64),
// A planes [row][k] (pitch ap bytes), B planes [col][k] (pitch TBP)
template <int NT>
__device__ __forceinline__ void mma_k64(u64 (&acc)[NT][4], const uint8_t* Al, const uint8_t* Ah, int ap,
                                        const uint8_t* Bl, const uint8_t* Bh, int r0, int n0, int gq, int tg) {
    int S0[NT][4] = {}, S1[NT][4] = {}, S2[NT][4] = {};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
        const int kk = 32 * ks + 4 * tg;
        const u32 al[4] = {*reinterpret_cast<const u32*>(Al + (r0 + gq) * ap + kk),
                           *reinterpret_cast<const u32*>(Al + (r0 + gq + 8) * ap + kk),
                           *reinterpret_cast<const u32*>(Al + (r0 + gq) * ap + kk + 16),
                           *reinterpret_cast<const u32*>(Al + (r0 + gq + 8) * ap + kk + 16)};
        const u32 ah[4] = {*reinterpret_cast<const u32*>(Ah + (r0 + gq) * ap + kk),
                           *reinterpret_cast<const u32*>(Ah + (r0 + gq + 8) * ap + kk),
                           *reinterpret_cast<const u32*>(Ah + (r0 + gq) * ap + kk + 16),
                           *reinterpret_cast<const u32*>(Ah + (r0 + gq + 8) * ap + kk + 16)};
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int n = n0 + 8 * t + gq;
            const u32 bl[2] = {*reinterpret_cast<const u32*>(Bl + n * TBP + kk),
                               *reinterpret_cast<const u32*>(Bl + n * TBP + kk + 16)};
            const u32 bh[2] = {*reinterpret_cast<const u32*>(Bh + n * TBP + kk),
                               *reinterpret_cast<const u32*>(Bh + n * TBP + kk + 16)};
            imma16832(S0[t], al, bl);
            imma16832(S1[t], al, bh);
            imma16832(S1[t], ah, bl);
            imma16832(S2[t], ah, bh);
        }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e)
            acc[t][e] = (u64)(u32)S0[t][e] + ((u64)(u32)S1[t][e] << 8) + ((u64)(u32)S2[t][e] << 16);
}

// 256 threads = 8 warps: warp (wr, wc) computes rows 16 wr.. and columns 16 wc..
// (two n8 tiles) of the current leaf.
__global__ void __launch_bounds__(256, 1) trsm_node_tc_kernel(TrsmNodeArgs a) {
    extern __shared__ __align__(16) uint8_t tsm_[];
    const int nl_ = a.nleaf;
    const int nblk = nl_ + nl_ * (nl_ - 1) / 2;
    // [block][2 planes][64 cols][TBP]: blocks 0..nl_-1 the leaf inverses, then the
    // off-diagonal U_{l2,l} at nl_ + l(l-1)/2 + l2
    uint8_t* Up = tsm_;
    u32* Gs = reinterpret_cast<u32*>(Up + (size_t)nblk * 2 * PB * TBP);      // [TTM][TGW]
    uint8_t* Gp = reinterpret_cast<uint8_t*>(Gs + TTM * TGW);                 // [leaf][2][TTM][TBP]
    uint8_t* Bp = Gp + (size_t)TN_MAXLEAF * 2 * TTM * TBP;                    // [2][TTM][TBP]
    __shared__ i32 s_row[TN_MAXLEAF][PB];
    const Fp f = a.f;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tg = lane & 3;
    const int wr = warp & 1, wc = warp >> 1;
    pdl_wait();
    pdl_trigger();
    i32 lo[TN_MAXLEAF], hi[TN_MAXLEAF];
#pragma unroll
    for (int l = 0; l < TN_MAXLEAF; ++l) {
        lo[l] = l < nl_ ? dyn_eval(a.j_lo[l], a.rp) : 0;
        hi[l] = l < nl_ ? dyn_eval(a.j_hi[l], a.rp) : 0;
    }
    const i32 J0 = lo[0];
    const i32 nJ = hi[nl_ - 1] - J0;
    if (nJ <= 0 || (a.M <= 0 && !a.ninv)) return;
    for (int e = tid; e < (nl_ - 1) * PB; e += blockDim.x) {
        const int l = e / PB, t = e % PB;
        s_row[l][t] = t < hi[l] - lo[l] ? __ldcg(a.rrp + lo[l] + t) : 0;
    }
    __syncthreads();
    // ---- stage the U blocks: every block of a round copied asynchronously (u32,
    // row-major) into a scratch area that the G tile later reuses, one wait, then
    // transposed into byte planes [column][k] (thread = column, 4 consecutive k)
    auto block_of = [&](int q, int& l, int& l2) {
        if (q < nl_) {
            l = q;
            l2 = -1;
            return;
        }
        int r = q - nl_;
        l = 1;
        while (r >= l) {
            r -= l;
            ++l;
        }
        l2 = r;
    };
    u32* Tmp = Gs;  // TSTAGE blocks of PB x PB words
    if (tid < nl_ && a.uready[tid] && hi[tid] > lo[tid]) uready_wait(a.uready[tid], a.epoch);
    __syncthreads();
    const bool al = (a.lda & 3) == 0;
    for (int q0 = 0; q0 < nblk; q0 += TSTAGE) {
        const int nq = min(TSTAGE, nblk - q0);
        for (int qq = 0; qq < nq; ++qq) {
            int l, l2;
            block_of(q0 + qq, l, l2);
            const int nl = hi[l] - lo[l];
            const int n2 = l2 >= 0 ? hi[l2] - lo[l2] : nl;
            u32* dst = Tmp + qq * PB * PB;
            if (l2 < 0) {  // leaf inverse, row-major PB x PB, zero padded
                for (int e = tid; e < PB * PB / 4; e += blockDim.x) cp_async16(dst + e * 4, a.uinv[l] + e * 4);
            } else if (al && (lo[l] & 3) == 0) {
                for (int e = tid; e < PB * PB / 4; e += blockDim.x) {
                    const int k = e >> 4, c = (e & 15) * 4;
                    const int bytes = k < n2 ? 4 * max(0, min(4, nl - c)) : 0;
                    cp_async16z(dst + k * PB + c, bytes ? a.A + (i64)s_row[l2][k] * a.lda + lo[l] + c : a.A, bytes);
                }
            } else {
                for (int e = tid; e < PB * PB; e += blockDim.x) {
                    const int k = e / PB, c = e % PB;
                    const bool ok = k < n2 && c < nl;
                    cp_async4(dst + k * PB + c, ok ? a.A + (i64)s_row[l2][k] * a.lda + lo[l] + c : a.A, ok);
                }
            }
        }
        cp_async_wait_all();
        __syncthreads();
        for (int e = tid; e < nq * PB * (PB / 4); e += blockDim.x) {
            const int qq = e / (PB * (PB / 4)), w = e % (PB * (PB / 4));
            const int c = w & 63, k0 = (w >> 6) * 4;
            const u32* src = Tmp + qq * PB * PB + k0 * PB + c;
            const u32 x0 = src[0], x1 = src[PB], x2 = src[2 * PB], x3 = src[3 * PB];
            uint8_t* pl = Up + (size_t)(q0 + qq) * 2 * PB * TBP;
            *reinterpret_cast<u32*>(pl + c * TBP + k0) = lob(x0, 0) | lob(x1, 0) << 8 | lob(x2, 0) << 16 | lob(x3, 0) << 24;
            *reinterpret_cast<u32*>(pl + PB * TBP + c * TBP + k0) =
                lob(x0, 8) | lob(x1, 8) << 8 | lob(x2, 8) << 16 | lob(x3, 8) << 24;
        }
        __syncthreads();
    }
    const i32 Mtot = a.M + (a.ninv ? nJ : 0);
    for (i32 r0 = blockIdx.x * TTM; r0 < Mtot; r0 += gridDim.x * TTM) {
        __syncthreads();
        // ---- the G tile (u32): rows < M from A (async copies), virtual rows the identity
        for (int e = tid; e < TTM * (TN_MAXLEAF * PB); e += blockDim.x) {
            const int rr = e / (TN_MAXLEAF * PB), j = e % (TN_MAXLEAF * PB);
            const i32 r = r0 + rr;
            const bool ok = j < nJ && r < a.M;
            if (ok) cp_async4(&Gs[rr * TGW + j], a.A + (i64)(a.row0 + r) * a.lda + J0 + j, true);
            else Gs[rr * TGW + j] = (j < nJ && r >= a.M && r < Mtot && j == r - a.M) ? 1u % f.p : 0u;
        }
        cp_async_wait_all();
        __syncthreads();
        for (int l = 0; l < nl_; ++l) {
            const int nl = hi[l] - lo[l];
            const int ol = lo[l] - J0;
            // B_l <- B_l - sum_{l2 < l} G_l2 * U_{l2,l}, into the planes Bp
            u64 S[2][4];
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) S[t][e] = 0;
            for (int l2 = 0; l2 < l; ++l2) {
                u64 acc[2][4];
                const uint8_t* gl = Gp + (size_t)l2 * 2 * TTM * TBP;
                const uint8_t* ub = Up + (size_t)(nl_ + l * (l - 1) / 2 + l2) * 2 * PB * TBP;
                mma_k64<2>(acc, gl, gl + TTM * TBP, TBP, ub, ub + PB * TBP, 16 * wr, 16 * wc, gq, tg);
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) S[t][e] += acc[t][e];
            }
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = 16 * wr + gq + 8 * (e >> 1), c = 16 * wc + 8 * t + 2 * tg + (e & 1);
                    u32 v = 0;
                    if (c < nl) v = submod(Gs[r * TGW + ol + c], red_sp(S[t][e], f), f);
                    Bp[r * TBP + c] = (uint8_t)lob(v, 0);
                    Bp[TTM * TBP + r * TBP + c] = (uint8_t)lob(v, 8);
                }
            __syncthreads();
            // G_l = B_l * Uinv_l
            u64 acc[2][4];
            const uint8_t* ui = Up + (size_t)l * 2 * PB * TBP;
            mma_k64<2>(acc, Bp, Bp + TTM * TBP, TBP, ui, ui + PB * TBP, 16 * wr, 16 * wc, gq, tg);
            uint8_t* gl = Gp + (size_t)l * 2 * TTM * TBP;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = 16 * wr + gq + 8 * (e >> 1), c = 16 * wc + 8 * t + 2 * tg + (e & 1);
                    const u32 v = c < nl ? red_sp(acc[t][e], f) : 0u;
                    if (c < nl) Gs[r * TGW + ol + c] = v;
                    gl[r * TBP + c] = (uint8_t)lob(v, 0);
                    gl[TTM * TBP + r * TBP + c] = (uint8_t)lob(v, 8);
                }
            __syncthreads();
        }
        // ---- write back: rows < M into A, virtual rows into the node inverse
        for (int e = tid; e < TTM * (TN_MAXLEAF * PB); e += blockDim.x) {
            const int rr = e / (TN_MAXLEAF * PB), j = e % (TN_MAXLEAF * PB);
            const i32 r = r0 + rr;
            if (j >= nJ) continue;
            if (r < a.M) a.A[(i64)(a.row0 + r) * a.lda + J0 + j] = Gs[rr * TGW + j];
            else if (r < Mtot) a.ninv[(i64)(r - a.M) * NINV_LD + j] = Gs[rr * TGW + j];
        }
    }
}

}  // namespace

size_t trsm_node_tc_smem(int nleaf) {
    const int nblk = nleaf + nleaf * (nleaf - 1) / 2;
    const size_t tile = sizeof(u32) * TTM * TGW + (size_t)TN_MAXLEAF * 2 * TTM * TBP + 2 * TTM * TBP;
    const size_t stage = sizeof(u32) * TSTAGE * PB * PB;  // the staging scratch reuses the tile area
    return (size_t)nblk * 2 * PB * TBP + std::max(tile, stage);
}

void trsm_node_tc(const TrsmNodeArgs& a, cudaStream_t s) {
    const size_t smem = trsm_node_tc_smem(a.nleaf);
    static std::atomic<unsigned long long> attr_once{0};
    once_on_device(attr_once, [&] {
        RL_CUDA_CHECK(cudaFuncSetAttribute(trsm_node_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)trsm_node_tc_smem(TN_MAXLEAF)));
    });
    const int rows = a.M + (a.ninv ? NINV_LD : 0);  // host bound; the kernel uses the live nJ
    const int grid = std::max(1, std::min((rows + TTM - 1) / TTM, num_sms()));
    launch_pdl(trsm_node_tc_kernel, dim3(grid), dim3(256), smem, s, a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
