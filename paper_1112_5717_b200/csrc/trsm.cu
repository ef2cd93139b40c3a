// trsm.cu -- fused triangular solve against a small skeleton node.
//
// trsm(Right, Upper, Unit) of cup (proj/src/factor.cpp:45-46, kernels.cpp:135-154)
// recurses along the top node's skeleton.  For a node X of at most 4 leaves the
// whole recursion -- leaf solves G_l <- B_l U_l^{-1} and the updates
// B_l -= G_l' U_{l'l} between them (kernels.cpp:149-154) -- runs in ONE kernel:
// each CTA owns a 16-row tile of G held in shared memory and sweeps the leaves
// left to right (block forward substitution), with the leaf inverses U_l^{-1}
// precomputed by the leaves' panels and the off-diagonal blocks U_{l'l} gathered
// through the row profile.  Thread = (row, 4 consecutive columns): one broadcast
// load of G and one 16-byte load of U per 4 multiply-adds; products are summed
// lazily in 64 bits (p < 2^16) and reduced once per output.  Short tiles give
// many CTAs (4 per SM) so the sweep's latency hides behind parallelism.  The
// diagonal (C's pivots) is never read: Unit.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {

constexpr int TM = 16;                    // rows of G per CTA tile
constexpr int GW = TN_MAXLEAF * PB + 4;   // smem row pitch of the G tile (words)
constexpr int BW = PB + 4;                // pitch of a 64 x 64 block (16-byte aligned rows)

template <bool SP>
__device__ __forceinline__ void mac4(u64 (&acc)[4], u32 g, uint4 u, const Fp& f) {
    if (SP) {
        acc[0] += (u64)g * u.x;
        acc[1] += (u64)g * u.y;
        acc[2] += (u64)g * u.z;
        acc[3] += (u64)g * u.w;
    } else {
        acc[0] += mulmod(g, u.x, f);
        acc[1] += mulmod(g, u.y, f);
        acc[2] += mulmod(g, u.z, f);
        acc[3] += mulmod(g, u.w, f);
    }
}

template <bool SP>
__global__ void __launch_bounds__(256) trsm_node_kernel(TrsmNodeArgs a) {
    extern __shared__ __align__(16) u32 sm[];
    u32* Gs = sm;                 // [TM][GW]
    u32* Bk = sm + TM * GW;       // [PB][BW] block U_{l'l}
    u32* Ui = Bk + PB * BW;       // [PB][BW] leaf inverse
    __shared__ i32 s_row[PB];
    const Fp f = a.f;
    const int tid = threadIdx.x;
    const int row = tid >> 4, cg = tid & 15;  // thread -> (row, columns 4cg..4cg+3)
    i32 lo[TN_MAXLEAF], hi[TN_MAXLEAF];
#pragma unroll
    for (int l = 0; l < TN_MAXLEAF; ++l) {
        lo[l] = l < a.nleaf ? dyn_eval(a.j_lo[l], a.rp) : 0;
        hi[l] = l < a.nleaf ? dyn_eval(a.j_hi[l], a.rp) : 0;
    }
    const i32 J0 = lo[0];
    const i32 nJ = hi[a.nleaf - 1] - J0;
    if (nJ <= 0 || a.M <= 0) return;
    for (i32 r0 = blockIdx.x * TM; r0 < a.M; r0 += gridDim.x * TM) {
        __syncthreads();
        for (int e = tid; e < TM * nJ; e += blockDim.x) {
            const int rr = e / nJ, j = e % nJ;
            const bool ok = r0 + rr < a.M;
            cp_async4(&Gs[rr * GW + j], ok ? a.A + (i64)(a.row0 + r0 + rr) * a.lda + J0 + j : a.A, ok);
        }
        cp_async_wait_all();
        __syncthreads();
        for (int l = 0; l < a.nleaf; ++l) {
            const int nl = hi[l] - lo[l];
            if (nl <= 0) continue;
            const int ol = lo[l] - J0;
            u64 S[4] = {0, 0, 0, 0};
            // S = sum_{l' < l} G_l' * U[J_l', J_l]
            for (int l2 = 0; l2 < l; ++l2) {
                const int n2 = hi[l2] - lo[l2];
                if (n2 <= 0) continue;
                const int o2 = lo[l2] - J0;
                __syncthreads();
                if (tid < n2) s_row[tid] = __ldcg(a.rrp + lo[l2] + tid);
                __syncthreads();
#pragma unroll 4
                for (int e = tid; e < PB * PB; e += blockDim.x) {
                    const int k = e / PB, c = e % PB;
                    const bool ok = k < n2 && c < nl;
                    cp_async4(&Bk[k * BW + c], ok ? a.A + (i64)s_row[k] * a.lda + lo[l] + c : a.A, ok);
                }
                cp_async_wait_all();
                __syncthreads();
                const u32* grow = &Gs[row * GW + o2];
#pragma unroll 4
                for (int k = 0; k < n2; ++k)
                    mac4<SP>(S, grow[k], *reinterpret_cast<const uint4*>(&Bk[k * BW + 4 * cg]), f);
            }
            // B_l <- B_l - S (in the tile), then G_l = B_l * Uinv_l
            __syncthreads();
#pragma unroll 4
            for (int e = tid; e < PB * PB; e += blockDim.x)
                cp_async4(&Ui[(e / PB) * BW + e % PB], a.uinv[l] + e, true);
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int c = 4 * cg + y;
                if (c < nl) {
                    u32* g = &Gs[row * GW + ol + c];
                    *g = submod(*g, red64(S[y], f), f);
                }
            }
            cp_async_wait_all();
            __syncthreads();
            u64 O[4] = {0, 0, 0, 0};
            const int kmax = min(nl, 4 * cg + 4);  // Uinv is upper triangular
            const u32* grow = &Gs[row * GW + ol];
#pragma unroll 4
            for (int k = 0; k < kmax; ++k)
                mac4<SP>(O, grow[k], *reinterpret_cast<const uint4*>(&Ui[k * BW + 4 * cg]), f);
            __syncthreads();
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int c = 4 * cg + y;
                if (c < nl) Gs[row * GW + ol + c] = SP ? red_sp(O[y], f) : red64(O[y], f);
            }
        }
        __syncthreads();
        for (int e = tid; e < TM * nJ; e += blockDim.x) {
            const int rr = e / nJ, j = e % nJ;
            if (r0 + rr < a.M) a.A[(i64)(a.row0 + r0 + rr) * a.lda + J0 + j] = Gs[rr * GW + j];
        }
    }
}

}  // namespace

void trsm_node(const TrsmNodeArgs& a, cudaStream_t s) {
    if (a.M <= 0 || a.nleaf <= 0) return;
    const size_t smem = sizeof(u32) * (TM * GW + 2 * PB * BW);
    static bool attr = false;
    if (!attr) {
        RL_CUDA_CHECK(cudaFuncSetAttribute(trsm_node_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        RL_CUDA_CHECK(cudaFuncSetAttribute(trsm_node_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int grid = std::max(1, std::min((a.M + TM - 1) / TM, 16 * num_sms()));
    if (a.f.p <= 65536u) trsm_node_kernel<true><<<grid, 256, smem, s>>>(a);
    else trsm_node_kernel<false><<<grid, 256, smem, s>>>(a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
