// bridge.cu -- the step between the two leaves of a leaf-pair node, fused.
//
// In the recursion (proj/src/factor.cpp:39-53) a node of two leaves, after its
// top leaf is factored, applies the top leaf's transpositions to the bottom
// rows (factor.cpp:42, perm_apply_cols), solves G <- X * U_top^{-1} for the
// bottom rows' columns at the top pivots (trsm Right/Upper/Unit,
// factor.cpp:45-46) and updates the bottom rows' remaining columns
// C <- C - G * U_top (mm, factor.cpp:51-52).  Only the columns the bottom leaf's
// window reads ([rp[b0], rp[b0] + PW)) are on the critical path; this kernel
// does the swaps, the solve and that slice's update in ONE launch (one CTA,
// p <= 2^16), both products on the legacy tensor cores (mma.sync m16n8k32
// u8 x u8 -> s32, two byte limbs: S0 = lo*lo, S1 = lo*hi + hi*lo, S2 = hi*hi,
// every sum at most 2*64*255^2 < 2^31), replacing a swap job, a trsm kernel and
// a GEMM launch.  The rest of the bottom rows' columns is updated by the wide
// GEMM on the side stream, which reads the G written here.
#include "kernels.cuh"
#include "runtime.h"

namespace rl {

LT_TABLE(bridge)

namespace {

constexpr int BP = 80;  // byte-plane row pitch: conflict-free mma fragment loads

__device__ __forceinline__ u32 lo4(u32 a, u32 b, u32 c, u32 d) {
    return (a & 0xff) | (b & 0xff) << 8 | (c & 0xff) << 16 | (d & 0xff) << 24;
}
__device__ __forceinline__ u32 hi4(u32 a, u32 b, u32 c, u32 d) {
    return (a >> 8 & 0xff) | (b >> 8 & 0xff) << 8 | (c >> 8 & 0xff) << 16 | (d >> 8 & 0xff) << 24;
}

// acc[t][e] += A(16 rows at r0, K = 64) * B(8 columns at n0 + 8t, K = 64)
template <int NT>
__device__ __forceinline__ void mma64(u64 (&acc)[NT][4], const uint8_t (*Al)[BP], const uint8_t (*Ah)[BP],
                                      const uint8_t (*Bl)[BP], const uint8_t (*Bh)[BP], int r0, int n0,
                                      int gq, int tg) {
    int S0[NT][4] = {}, S1[NT][4] = {}, S2[NT][4] = {};
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
        const int kk = 32 * ks + 4 * tg;
        const u32 al[4] = {*reinterpret_cast<const u32*>(&Al[r0 + gq][kk]),
                           *reinterpret_cast<const u32*>(&Al[r0 + gq + 8][kk]),
                           *reinterpret_cast<const u32*>(&Al[r0 + gq][kk + 16]),
                           *reinterpret_cast<const u32*>(&Al[r0 + gq + 8][kk + 16])};
        const u32 ah[4] = {*reinterpret_cast<const u32*>(&Ah[r0 + gq][kk]),
                           *reinterpret_cast<const u32*>(&Ah[r0 + gq + 8][kk]),
                           *reinterpret_cast<const u32*>(&Ah[r0 + gq][kk + 16]),
                           *reinterpret_cast<const u32*>(&Ah[r0 + gq + 8][kk + 16])};
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int n = n0 + 8 * t + gq;
            const u32 bl[2] = {*reinterpret_cast<const u32*>(&Bl[n][kk]),
                               *reinterpret_cast<const u32*>(&Bl[n][kk + 16])};
            const u32 bh[2] = {*reinterpret_cast<const u32*>(&Bh[n][kk]),
                               *reinterpret_cast<const u32*>(&Bh[n][kk + 16])};
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

// raw operand staging (u32, row pitch +4 words: 16-byte aligned rows)
constexpr int XP = PB + 4, UP = PW + 4;
constexpr size_t RAW_BYTES = sizeof(u32) * (2 * PB * XP + 2 * PB * UP);  // X, U^{-1}, U slice, C slice
#ifndef RL_BRIDGE_SMEM
#define RL_BRIDGE_SMEM 0  // (a larger request keeps other CTAs off its SM)
#endif
constexpr size_t BRIDGE_SMEM = RAW_BYTES > RL_BRIDGE_SMEM ? RAW_BYTES : RL_BRIDGE_SMEM;

// rows [0, rows) x words [0, cols) of a row-major global block (row r at
// base + rowoff(r), cols valid of width) into smem dst[r][.] with pitch dp;
// 16-byte copies where aligned, zero fill outside (rows >= nrows, cols >= ncols)
template <class RowOff>
__device__ __forceinline__ void stage(u32* dst, int dp, int rows, int cols, int nrows, int ncols, bool aligned,
                                      RowOff rowoff) {
    const int q4 = cols / 4;
    for (int e = threadIdx.x; e < rows * q4; e += blockDim.x) {
        const int r = e / q4, c = (e % q4) * 4;
        u32* d = dst + r * dp + c;
        const int nv = r < nrows ? max(0, min(4, ncols - c)) : 0;
        if (nv == 0) {
            *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
            continue;
        }
        const u32* src = rowoff(r) + c;
        if (aligned) {
            cp_async16z(d, src, 4 * nv);
        } else {
#pragma unroll
            for (int z = 0; z < 4; ++z) cp_async4(d + z, z < nv ? src + z : src, z < nv);
        }
    }
}

__global__ void __launch_bounds__(256, 1) bridge_kernel(BridgeArgs a) {
    extern __shared__ __align__(16) u32 raw[];
    u32* Xr = raw;              // [PB][XP]  X at the top pivots
    u32* Ir = Xr + PB * XP;     // [PB][XP]  U_top^{-1}
    u32* Ur = Ir + PB * XP;     // [PB][UP]  U_top at the slice
    u32* Cr = Ur + PB * UP;     // [PB][UP]  the bottom rows at the slice
    __shared__ __align__(16) uint8_t Xl[PB][BP], Xh[PB][BP];   // X, then G  [row][k]
    __shared__ __align__(16) uint8_t Il[PB][BP], Ih[PB][BP];   // U^{-1}     [col][k]
    __shared__ __align__(16) uint8_t Ul[PW][BP], Uh[PW][BP];   // U slice    [col][k]
    __shared__ i32 s_urow[PB];
    LT_BEGIN();
    // Launched as a programmatic dependent of the top leaf's tail, which starts
    // only once the top leaf's window completed: rank prefix, pivots, flags and
    // U^{-1} are final unless the tail can fall back (window-dead rows), and the
    // bottom rows are not the tail's.  So everything but the U slice (the
    // tail's output) is fetched before waiting for the tail.
    const bool early = __ldcg(&a.ps->dead_mask) == 0;
    if (!early) pdl_wait();
    const Fp f = a.f;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tg = lane & 3;
    const i32 j_lo = dyn_eval(a.j_lo, a.rp);
    const i32 nl = dyn_eval(a.j_hi, a.rp) - j_lo;  // top rank r1 <= PB
    const int M = a.M;
#ifdef RL_BRIDGE_DELAY_NS
    if (threadIdx.x == 0) rl_spin_ns(RL_BRIDGE_DELAY_NS);
    __syncthreads();
#endif
    if (nl <= 0 || M <= 0) {  // uniform: no pivot above, nothing to solve or update
        if (early) pdl_wait();  // (the successor's reads must not overtake the tail)
        LT_END(a.row0 / PB);
        return;
    }
    const i32 n_lo = dyn_eval(a.n_lo, a.rp);
    const int ns = max(0, min(PW, a.N - n_lo));  // live slice width
    const bool swapped = __ldcg(a.swapflag) != 0;
    if (tid < PB) s_urow[tid] = tid < nl ? __ldcg(a.rrp + j_lo + tid) : -1;
    // (1) the top leaf's transpositions on the bottom rows, in increasing j (all
    //     columns: a target may lie beyond the slice)
    if (swapped) {
        if (tid < M) {
            u32* row = a.A + (i64)(a.row0 + tid) * a.lda;
            for (i32 j = j_lo; j < j_lo + nl; ++j) {
                const i32 t = __ldcg(a.ipiv + j);
                if (t != j) {
                    const u32 x = row[j];
                    row[j] = row[t];
                    row[t] = x;
                }
            }
        }
    }
    __syncthreads();  // s_urow, swaps
    LT_MARK(a.row0 / PB, 2);
    // (2) every operand in flight at once (cp.async), one wait
    const bool lda4 = (a.lda & 3) == 0 && (reinterpret_cast<uintptr_t>(a.A) & 15) == 0;
    const u32* A = a.A;
    const i64 lda = a.lda, row0 = a.row0;
    stage(Xr, XP, PB, PB, M, nl, lda4 && (j_lo & 3) == 0, [&](int r) { return A + (row0 + r) * lda + j_lo; });
    if (a.uready) {  // the leaf's U^{-1} comes from a kernel on another stream
        if (tid == 0) uready_wait(a.uready, a.epoch);
        __syncthreads();
    }
    stage(Ir, XP, PB, PB, nl, nl, (reinterpret_cast<uintptr_t>(a.uinv) & 15) == 0,
          [&](int r) { return a.uinv + r * PB; });
    stage(Cr, UP, PB, PW, M, ns, lda4 && (n_lo & 3) == 0, [&](int r) { return A + (row0 + r) * lda + n_lo; });
    if (early) pdl_wait();
    pdl_trigger();
    stage(Ur, UP, PB, PW, nl, ns, lda4 && (n_lo & 3) == 0,
          [&](int r) { return A + (i64)s_urow[r] * lda + n_lo; });
    cp_async_wait_all();
    __syncthreads();
    // byte planes: X [row][k]; U^{-1} and U slice transposed [col][k]
    for (int e = tid; e < PB * (PB / 4); e += 256) {
        const int r = e >> 4, k = (e & 15) * 4;
        const uint4 v = *reinterpret_cast<const uint4*>(Xr + r * XP + k);
        *reinterpret_cast<u32*>(&Xl[r][k]) = lo4(v.x, v.y, v.z, v.w);
        *reinterpret_cast<u32*>(&Xh[r][k]) = hi4(v.x, v.y, v.z, v.w);
    }
    for (int e = tid; e < (PB / 4) * (PB + PW); e += 256) {
        const int k = (e / (PB + PW)) * 4, n = e % (PB + PW);
        const bool inv = n < PB;
        const u32* src = inv ? Ir + n : Ur + (n - PB);
        const int sp = inv ? XP : UP;
        const u32 v0 = src[k * sp], v1 = src[(k + 1) * sp], v2 = src[(k + 2) * sp], v3 = src[(k + 3) * sp];
        uint8_t* lo = inv ? &Il[n][k] : &Ul[n - PB][k];
        uint8_t* hi = inv ? &Ih[n][k] : &Uh[n - PB][k];
        *reinterpret_cast<u32*>(lo) = lo4(v0, v1, v2, v3);
        *reinterpret_cast<u32*>(hi) = hi4(v0, v1, v2, v3);
    }
    __syncthreads();
    LT_MARK(a.row0 / PB, 3);
    const int rs = warp & 3, cw = warp >> 2;  // warp: rows 16 rs.., columns 32 cw.. (G) / 64 cw.. (slice)
    // (3) G = X * U^{-1}
    u64 g[4][4];
    mma64<4>(g, Xl, Xh, Il, Ih, 16 * rs, 32 * cw, gq, tg);
    __syncthreads();  // every warp is done reading X
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int r = 16 * rs + gq + 8 * (e >> 1), c = 32 * cw + 8 * t + 2 * tg + (e & 1);
            const u32 v = (r < M && c < nl) ? red_sp(g[t][e], f) : 0u;
            Xl[r][c] = (uint8_t)v;
            Xh[r][c] = (uint8_t)(v >> 8);
            Xr[r * XP + c] = v;
        }
    __syncthreads();
    // G back to its place (coalesced rows)
    for (int e = tid; e < M * PB; e += 256) {
        const int r = e / PB, c = e % PB;
        if (c < nl) a.A[(row0 + r) * lda + j_lo + c] = Xr[r * XP + c];
    }
    LT_MARK(a.row0 / PB, 4);
    // (4) slice -= G * U_top[:, slice]
    if (ns > 64 * cw) {
        u64 acc[8][4];
        mma64<8>(acc, Xl, Xh, Ul, Uh, 16 * rs, 64 * cw, gq, tg);
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = 16 * rs + gq + 8 * (e >> 1), c = 64 * cw + 8 * t + 2 * tg + (e & 1);
                Cr[r * UP + c] = submod(Cr[r * UP + c], red_sp(acc[t][e], f), f);
            }
    }
    __syncthreads();
    for (int e = tid; e < M * PW; e += 256) {
        const int r = e / PW, c = e % PW;
        if (c < ns) a.A[(row0 + r) * lda + n_lo + c] = Cr[r * UP + c];
    }
    LT_END(a.row0 / PB);
}

}  // namespace

void bridge(const BridgeArgs& a, cudaStream_t s) {
    RL_ONCE_SMEM_LIMIT(bridge_kernel, BRIDGE_SMEM);
    launch_pdl(bridge_kernel, dim3(1), dim3(256), BRIDGE_SMEM, s, a);
    RL_CUDA_CHECK(cudaGetLastError());
}

}  // namespace rl
