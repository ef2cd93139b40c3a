// trsm.cu -- fused triangular solve against a small skeleton node.
//
// trsm(Right, Upper, Unit) of cup (proj/src/factor.cpp:45-46, kernels.cpp:135-154)
// recurses along the top node's skeleton.  For a node X of at most 4 leaves the
// whole recursion -- leaf solves G_l <- B_l U_l^{-1} and the updates
// B_l -= G_l' U_{l'l} between them (kernels.cpp:149-154) -- runs in ONE kernel:
// each CTA first stages every operand block of the node in shared memory (the
// leaf inverses U_l^{-1}, precomputed by the leaves' panels, and the
// off-diagonal blocks U_{l'l} gathered through the row profile: up to 10 blocks,
// 170 KB, loaded once with one wait), then sweeps its row tiles of G left to
// right (block forward substitution) without further global round trips.
// Thread = (rows rg + 16t, 4 consecutive columns): one 16-byte load of U feeds
// 4*TR multiply-adds; products are summed lazily in 64 bits (p < 2^16) and
// reduced once per output.  The diagonal (C's pivots) is never read: Unit.
#include <algorithm>

#include "kernels.cuh"
#include "runtime.h"

namespace rl {

namespace {

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

// Block index of U_{l2,l} (l2 < l) among the staged off-diagonal blocks.
__device__ __forceinline__ int pair_idx(int l2, int l) { return l * (l - 1) / 2 + l2; }

// Thread (rg, cg, kg) owns rows rg + 16 t (t < TR) and columns 4cg..4cg+3 of
// the current leaf, and the k-slice k = kg (mod KS) of every dot product: per k
// one 16-byte load of U feeds 4*TR multiply-adds; the KS partial sums meet in
// shared memory.  Splitting k shortens each thread's serial chain KS-fold (the
// sweep is latency-bound: few rows, long dot products).
template <bool SP, int TR, int KS>
__global__ void __launch_bounds__(256 * KS) trsm_node_kernel(TrsmNodeArgs a) {
    constexpr int TM = 16 * TR;
    constexpr int BLK = PB * BW;  // words per staged 64 x 64 block
    extern __shared__ __align__(16) u32 sm[];
    const int nl_ = a.nleaf;
    u32* Gs = sm;                                   // [TM][GW]
    u32* Ui = sm + TM * GW;                         // nleaf blocks: leaf inverses
    u32* Bk = Ui + nl_ * BLK;                       // nleaf(nleaf-1)/2 blocks U_{l2,l}
    u64* Pt = reinterpret_cast<u64*>(Bk + (nl_ * (nl_ - 1) / 2) * BLK);  // [KS-1][TM][PB] partials
    __shared__ i32 s_row[TN_MAXLEAF][PB];
    const Fp f = a.f;
    const int tid = threadIdx.x;
    const int kg = tid >> 8, t8 = tid & 255;
    const int rg = t8 >> 4, cg = t8 & 15;
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
    RL_STAMP(t_enter);
#ifdef RL_TRACE
    unsigned long long t_leaf[TN_MAXLEAF + 1] = {0, 0, 0, 0, 0};
#endif
    // ---- stage all operand blocks once (one wait)
    for (int e = tid; e < (nl_ - 1) * PB; e += blockDim.x) {
        const int l = e / PB, t = e % PB;
        s_row[l][t] = t < hi[l] - lo[l] ? __ldcg(a.rrp + lo[l] + t) : 0;
    }
    __syncthreads();
    // rows are 16-byte aligned iff lda is a multiple of 4; a block starting at a
    // column that is one too moves in 16-byte pieces (the common case: pivot
    // ranges start at multiples of the leaf size)
    const bool al = (a.lda & 3) == 0;
    for (int l = 0; l < nl_; ++l) {
        for (int e = tid; e < PB * PB / 4; e += blockDim.x)
            cp_async16(&Ui[l * BLK + (e >> 4) * BW + (e & 15) * 4], a.uinv[l] + e * 4);
        const int nl = hi[l] - lo[l];
        for (int l2 = 0; l2 < l; ++l2) {
            const int n2 = hi[l2] - lo[l2];
            u32* dst = Bk + pair_idx(l2, l) * BLK;
            if (al && (lo[l] & 3) == 0) {
                for (int e = tid; e < PB * PB / 4; e += blockDim.x) {
                    const int k = e >> 4, c = (e & 15) * 4;
                    const int bytes = k < n2 ? 4 * max(0, min(4, nl - c)) : 0;
                    cp_async16z(&dst[k * BW + c], bytes ? a.A + (i64)s_row[l2][k] * a.lda + lo[l] + c : a.A,
                                bytes);
                }
            } else {
#pragma unroll 4
                for (int e = tid; e < PB * PB; e += blockDim.x) {
                    const int k = e / PB, c = e % PB;
                    const bool ok = k < n2 && c < nl;
                    cp_async4(&dst[k * BW + c], ok ? a.A + (i64)s_row[l2][k] * a.lda + lo[l] + c : a.A, ok);
                }
            }
        }
    }
    const bool gal = al && (J0 & 3) == 0;
    // rows [M, M + nJ) are virtual: B = I over the node's pivots, so the sweep
    // also yields the node inverse U_X^{-1} (written to a.ninv)
    const i32 Mtot = a.M + (a.ninv ? nJ : 0);
    // partial sums of the other k-groups into group 0's accumulators
    auto gather = [&](u64 (&S)[TR][4]) {
        if (KS == 1) return;
        if (kg > 0) {
#pragma unroll
            for (int t = 0; t < TR; ++t)
#pragma unroll
                for (int y = 0; y < 4; ++y)
                    Pt[((kg - 1) * TM + rg + 16 * t) * PB + 4 * cg + y] = S[t][y];
        }
        __syncthreads();
        if (kg == 0) {
#pragma unroll
            for (int q = 1; q < KS; ++q)
#pragma unroll
                for (int t = 0; t < TR; ++t)
#pragma unroll
                    for (int y = 0; y < 4; ++y) S[t][y] += Pt[((q - 1) * TM + rg + 16 * t) * PB + 4 * cg + y];
        }
    };
    for (i32 r0 = blockIdx.x * TM; r0 < Mtot; r0 += gridDim.x * TM) {
        __syncthreads();
        if (r0 + TM > a.M && a.ninv) {  // tile touches the virtual identity rows
            for (int e = tid; e < TM * (TN_MAXLEAF * PB); e += blockDim.x) {
                const int rr = e / (TN_MAXLEAF * PB), j = e % (TN_MAXLEAF * PB);
                const i32 r = r0 + rr;
                if (r < a.M) {
                    if (j < nJ) Gs[rr * GW + j] = a.A[(i64)(a.row0 + r) * a.lda + J0 + j];
                } else {
                    Gs[rr * GW + j] = (j == r - a.M) ? 1u % f.p : 0u;
                }
            }
        } else if (gal) {
            for (int e = tid; e < TM * (TN_MAXLEAF * PB / 4); e += blockDim.x) {
                const int rr = e / (TN_MAXLEAF * PB / 4), j = (e % (TN_MAXLEAF * PB / 4)) * 4;
                const int bytes = r0 + rr < a.M ? 4 * max(0, min(4, nJ - j)) : 0;
                cp_async16z(&Gs[rr * GW + j], bytes ? a.A + (i64)(a.row0 + r0 + rr) * a.lda + J0 + j : a.A,
                            bytes);
            }
        } else {
            for (int e = tid; e < TM * nJ; e += blockDim.x) {
                const int rr = e / nJ, j = e % nJ;
                const bool ok = r0 + rr < a.M;
                cp_async4(&Gs[rr * GW + j], ok ? a.A + (i64)(a.row0 + r0 + rr) * a.lda + J0 + j : a.A, ok);
            }
        }
        cp_async_wait_all();
        __syncthreads();
#ifdef RL_TRACE
        t_leaf[0] = rl_now();
#endif
        for (int l = 0; l < nl_; ++l) {
            const int nl = hi[l] - lo[l];
            if (nl <= 0) continue;
            const int ol = lo[l] - J0;
            u64 S[TR][4];
#pragma unroll
            for (int t = 0; t < TR; ++t)
#pragma unroll
                for (int y = 0; y < 4; ++y) S[t][y] = 0;
            // S = sum_{l2 < l} G_l2 * U[J_l2, J_l]   (this group's k-slice)
            for (int l2 = 0; l2 < l; ++l2) {
                const int n2 = hi[l2] - lo[l2];
                const u32* B = Bk + pair_idx(l2, l) * BLK;
                const u32* g0 = &Gs[rg * GW + lo[l2] - J0];
#pragma unroll 4
                for (int k = kg; k < n2; k += KS) {
                    const uint4 u = *reinterpret_cast<const uint4*>(&B[k * BW + 4 * cg]);
#pragma unroll
                    for (int t = 0; t < TR; ++t) mac4<SP>(S[t], g0[16 * t * GW + k], u, f);
                }
            }
            if (l > 0) gather(S);
            // B_l <- B_l - S (in the tile), then G_l = B_l * Uinv_l
            if (kg == 0) {
#pragma unroll
                for (int t = 0; t < TR; ++t)
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        const int c = 4 * cg + y;
                        if (c < nl) {
                            u32* g = &Gs[(rg + 16 * t) * GW + ol + c];
                            *g = submod(*g, SP ? red_sp(S[t][y], f) : red64(S[t][y], f), f);
                        }
                    }
            }
            __syncthreads();
#pragma unroll
            for (int t = 0; t < TR; ++t)
#pragma unroll
                for (int y = 0; y < 4; ++y) S[t][y] = 0;
            const int kmax = min(nl, 4 * cg + 4);  // Uinv is upper triangular
            const u32* U = Ui + l * BLK;
            const u32* g1 = &Gs[rg * GW + ol];
#pragma unroll 4
            for (int k = kg; k < kmax; k += KS) {
                const uint4 u = *reinterpret_cast<const uint4*>(&U[k * BW + 4 * cg]);
#pragma unroll
                for (int t = 0; t < TR; ++t) mac4<SP>(S[t], g1[16 * t * GW + k], u, f);
            }
            gather(S);
            __syncthreads();
            if (kg == 0) {
#pragma unroll
                for (int t = 0; t < TR; ++t)
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        const int c = 4 * cg + y;
                        if (c < nl) Gs[(rg + 16 * t) * GW + ol + c] = SP ? red_sp(S[t][y], f) : red64(S[t][y], f);
                    }
            }
            __syncthreads();
#ifdef RL_TRACE
            t_leaf[l + 1] = rl_now();
#endif
        }
        if (r0 + TM > a.M && a.ninv) {
            for (int e = tid; e < TM * nJ; e += blockDim.x) {
                const int rr = e / nJ, j = e % nJ;
                const i32 r = r0 + rr;
                if (r < a.M) a.A[(i64)(a.row0 + r) * a.lda + J0 + j] = Gs[rr * GW + j];
                else if (r < Mtot) a.ninv[(i64)(r - a.M) * NINV_LD + j] = Gs[rr * GW + j];
            }
        } else if (gal) {
            for (int e = tid; e < TM * (TN_MAXLEAF * PB / 4); e += blockDim.x) {
                const int rr = e / (TN_MAXLEAF * PB / 4), j = (e % (TN_MAXLEAF * PB / 4)) * 4;
                if (r0 + rr >= a.M || j >= nJ) continue;
                u32* dst = a.A + (i64)(a.row0 + r0 + rr) * a.lda + J0 + j;
                const uint4 v = *reinterpret_cast<const uint4*>(&Gs[rr * GW + j]);
                if (j + 4 <= nJ) {
                    *reinterpret_cast<uint4*>(dst) = v;
                } else {
                    dst[0] = v.x;
                    if (j + 1 < nJ) dst[1] = v.y;
                    if (j + 2 < nJ) dst[2] = v.z;
                }
            }
        } else {
            for (int e = tid; e < TM * nJ; e += blockDim.x) {
                const int rr = e / nJ, j = e % nJ;
                if (r0 + rr < a.M) a.A[(i64)(a.row0 + r0 + rr) * a.lda + J0 + j] = Gs[rr * GW + j];
            }
        }
    }
#ifdef RL_TRACE
    if (a.M == 256 && nl_ == 4 && a.row0 == 8448 && threadIdx.x == 0 && blockIdx.x < 2) {
        RL_STAMP(t_exit);
        printf("TRACE trsm cta %d enter %llu staged %llu l0 %llu l1 %llu l2 %llu l3 %llu exit %llu\n", blockIdx.x,
               t_enter, t_leaf[0], t_leaf[1], t_leaf[2], t_leaf[3], t_leaf[4], t_exit);
    }
#endif
}

__global__ void ninv_assemble_kernel(u32* X, i32 ldx, const u32* Xa, i32 la, const u32* Xb, i32 lb,
                                     const u32* T2, i32 lt, Dyn a_lo, Dyn b_lo, Dyn b_hi, const i32* rp,
                                     i32 nmax) {
    const i32 a0 = dyn_eval(a_lo, rp), b0 = dyn_eval(b_lo, rp), b1 = dyn_eval(b_hi, rp);
    const i32 ra = b0 - a0, rx = b1 - a0;
    for (i64 e = (i64)blockIdx.x * blockDim.x + threadIdx.x; e < (i64)nmax * nmax;
         e += (i64)gridDim.x * blockDim.x) {
        const i32 i = (i32)(e / nmax), j = (i32)(e % nmax);
        if (i >= rx || j >= rx) continue;
        u32 v;
        if (i < ra) v = j < ra ? Xa[(i64)i * la + j] : T2[(i64)i * lt + (j - ra)];
        else v = j < ra ? 0u : Xb[(i64)(i - ra) * lb + (j - ra)];
        X[(i64)i * ldx + j] = v;
    }
}

template <bool SP, int TR, int KS>
void launch_node(const TrsmNodeArgs& a, cudaStream_t s) {
    constexpr int TM = 16 * TR;
    const int nblk = a.nleaf + a.nleaf * (a.nleaf - 1) / 2;
    const size_t part = KS > 1 ? sizeof(u64) * (KS - 1) * TM * PB : 0;
    const size_t smem = sizeof(u32) * (TM * GW + (size_t)nblk * PB * BW) + part;
    static std::atomic<unsigned long long> attr_once{0};
    once_on_device(attr_once, [&] {
        const size_t maxs = sizeof(u32) * (TM * GW + (size_t)10 * PB * BW) + part;
        RL_CUDA_CHECK(cudaFuncSetAttribute(trsm_node_kernel<SP, TR, KS>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)maxs));
    });
    // one staging of the U blocks per CTA: about one CTA per SM, each looping
    // over its row tiles
    const int per_sm = nblk >= 6 ? 1 : (nblk >= 3 ? 2 : 4);
    const int rows = a.M + (a.ninv ? NINV_LD : 0);  // host bound; the kernel uses the live nJ
    const int grid = std::max(1, std::min((rows + TM - 1) / TM, per_sm * num_sms()));
    launch_pdl(trsm_node_kernel<SP, TR, KS>, dim3(grid), dim3(256 * KS), smem, s, a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

void ninv_assemble(u32* X, i32 ldx, const u32* Xa, i32 la, const u32* Xb, i32 lb, const u32* T2, i32 lt,
                   Dyn a_lo, Dyn b_lo, Dyn b_hi, const i32* rp, i32 nmax, cudaStream_t s) {
    const int grid = std::max(1, std::min((nmax * nmax + 255) / 256, 2 * num_sms()));
    ninv_assemble_kernel<<<grid, 256, 0, s>>>(X, ldx, Xa, la, Xb, lb, T2, lt, a_lo, b_lo, b_hi, rp, nmax);
    RL_CUDA_CHECK(cudaGetLastError());
}

// Row tile per CTA: 32 rows for tall G (fewer staged-block loads per row, more
// products per shared load), 16 otherwise (more CTAs for short G).
// p <= 2^16 takes the tensor-core form (trsm_tc.cu) unless RL_TRSM_TC=0
#ifndef RL_TRSM_TC
#define RL_TRSM_TC 1
#endif
void trsm_node(const TrsmNodeArgs& a, cudaStream_t s) {
    if ((a.M <= 0 && !a.ninv) || a.nleaf <= 0) return;
    const bool sp = a.f.p <= 65536u;
    if (RL_TRSM_TC && sp) {
        trsm_node_tc(a, s);
        return;
    }
    if (a.M >= 32 * num_sms()) {
        if (sp) launch_node<true, 2, 1>(a, s);
        else launch_node<false, 2, 1>(a, s);
    } else {
        if (sp) launch_node<true, 1, 4>(a, s);
        else launch_node<false, 1, 4>(a, s);
    }
}

}  // namespace rl
