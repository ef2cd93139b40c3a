// kernels.cuh -- argument blocks and launchers of every device kernel of the
// CUP path.  All rank-dependent extents are Dyn expressions over the
// device-resident rank prefix rp[], so launches never need a host sync.
#pragma once
#include "common.cuh"

// The leaf's U^{-1} computed by the tail kernel's last CTA (1) instead of a
// separate kernel on a side stream (0).
#ifndef RL_UINV_IN_TAIL
#define RL_UINV_IN_TAIL 0
#endif

namespace rl {

// ----------------------------------------------------------------------- GEMM
// C(r, n) <- beta*C(r, n) + alpha * sum_k A(r, k) * B(k, n)   (mod p)
//   A(r, k) = A[(a_row0 + r) * lda + k_lo + k]
//   B(k, n) = B[g(k) * ldb + n_lo + n],  g(k) = gather ? gather[k_lo + k] : k_lo + k
//   C(r, n) = C[(c_row0 + r) * ldc + n_lo + n]
//   r < M (static), k < K = k_hi - k_lo, n < N = n_hi - n_lo.
// This single form covers the reference mm seam (kernels.hpp:26-27) and every
// multiply inside cup: the Schur update H <- H - G*V1 (factor.cpp:51-52) and the
// TRSM-internal updates (kernels.cpp:149-154), where B rows are U rows gathered
// through the row profile.
struct GemmArgs {
    const u32* A;
    i64 lda;
    i32 a_row0;
    const u32* B;
    i64 ldb;
    const i32* gather;
    u32* C;
    i64 ldc;
    i32 c_row0;
    i32 M;
    Dyn k_lo, k_hi, n_lo, n_hi;
    const i32* rp;
    u32 alpha, beta;
    Fp f;
    int b_from0;   // B(k, n) = B[k * ldb + n]: a dense K x N operand (no k_lo/n_lo offsets)
    int a_from0;   // A(r, k) = A[(a_row0 + r) * lda + k]: a dense operand (no k_lo offset)
    int c_from0;   // C(r, n) = C[(c_row0 + r) * ldc + n]: a dense result (no n_lo offset)
    i32 n_cap;     // > 0: the column range ends at min(n_hi, n_cap)
    i32 max_ctas;  // > 0: grid bound (leave SMs free for a concurrent kernel)
};

// Number of 8-bit limbs for canonical elements of GF(p).
static inline int limbs_for(u32 p) {
    u32 v = p - 1;
    int bits = 0;
    while (v) {
        ++bits;
        v >>= 1;
    }
    int L = (bits + 7) / 8;
    return L < 1 ? 1 : L;
}
// Exactness bound: every s32 accumulator sums L*K products of two u8 limbs
// (each <= 255^2), so L*K*65025 < 2^31.
static inline i64 tc_kmax(int L) { return L <= 2 ? 16384 : 8192; }
static inline int tc_nt(int L) { return L == 1 ? 256 : (L == 2 ? 128 : 64); }

size_t tc_a2_bytes(int L, i64 M, i64 Kmax);
size_t tc_b2_bytes(int L, i64 Nmax, i64 Kmax);

// Packs A and B into limb tiles then runs the tcgen05 kernel.  `a2`/`b2` are
// workspaces of tc_a2_bytes/tc_b2_bytes for the static bounds (Kmax, Nmax).
void gemm_tc(const GemmArgs& g, int L, i64 Kmax, i64 Nmax, uint8_t* a2, uint8_t* b2,
             cudaStream_t s);
// phase 0: only the two pack kernels; phase 1: only the tcgen05 kernel (profiling);
// 2: both.
void gemm_tc_split(const GemmArgs& g, int L, i64 Kmax, i64 Nmax, uint8_t* a2, uint8_t* b2,
                   cudaStream_t s, int phase);
// CUDA-core fallback for skinny shapes (K or N tiny).
void gemm_simt(const GemmArgs& g, i64 Kmax, i64 Nmax, cudaStream_t s);

// ---------------------------------------------------------------------- panel
constexpr int PB = 64;        // rows per leaf panel
constexpr int PW = 128;       // leading window width (pivot search)
constexpr int WT = PW + PB;   // window + identity block (row transform)

struct PanelScratch {
    i32 c0, W, w, r, b;
    i32 spec;      // the window took the speculative (no-transposition) path
    i32 uinv_by_window;  // the window kernel already wrote U^{-1} (and set its flag)
    u32 flag;      // a window-dead row has a nonzero tail residual -> fallback
    u32 counter;   // last-CTA detection in the tail kernel
    u64 dead_mask;          // bit i: row i of the leaf has no pivot in the window
    i32 piv_of_row[PB];     // pivot index (local) of row i, -1 if dead
    i32 rank_before[PB];
    alignas(16) u32 Minv[PB][PB];  // row transform: V = Minv * P (U rows / residuals)
    u32 Mr[PB][PB];         // its inverse: P = Mr * V (fallback restore)
    u32 win_orig[PB][PW];   // original window (fallback restore)
};

struct PanelArgs {
    u32* A;
    i64 lda;
    i32 i0, b, N;
    i32* rp;
    i32* rrp;
    i32* ipiv;
    PanelScratch* ps;
    u32* uinv;     // PB x PB: inverse of this leaf's unit upper pivot block
    const uint16_t* inv_table;  // p < 2^16: inv_table[x] = x^{-1} mod p (else unused)
    i32* swapflag;  // this leaf's "made a transposition" flag (read by the swap jobs)
    i32* uready;    // this leaf's U^{-1}-ready flag (set to *epoch once uinv is written)
    const i32* epoch;
    Fp f;
    // tail only: the launch has no cross-stream join, so its programmatic
    // predecessor (the window) is the only kernel that may still run when its
    // CTAs start -- the tile prefetch before pdl_wait() is then safe
    int prefetch;
};
// inv_table[x] = x^{-1} mod p for x in [1, p) (p <= 65536), inv_table[0] = 0.
void build_inv_table(uint16_t* table, u32 p, cudaStream_t s);
void panel_window(const PanelArgs& a, cudaStream_t s);
void panel_tail(const PanelArgs& a, cudaStream_t s);
// The leaf's U^{-1} on its own (one CTA), for a stream parallel to the tail;
// does nothing when the leaf has window-dead rows (the tail then computes it,
// after a possible fallback).
void panel_uinv(const PanelArgs& a, cudaStream_t s);

// X <- X * U^{-1} for the unit upper block of one leaf's pivots J = [j_lo, j_hi)
// (|J| <= PB): rows [row0, row0 + M) of A, columns J; U^{-1} precomputed by
// the leaf's panel (uinv, PB x PB row-major).
struct TrsmLeafArgs {
    u32* A;
    i64 lda;
    i32 row0, M;
    Dyn j_lo, j_hi;
    const i32* rp;
    const u32* uinv;
    Fp f;
};
void trsm_leaf(const TrsmLeafArgs& a, cudaStream_t s);

// G <- G * U_X^{-1} for a skeleton node X of <= 4 leaves (<= 256 rows, pivots
// J = [j_lo[0], j_hi[nleaf-1]) contiguous): block forward substitution fused in
// one kernel (per 64-row tile of G: G_l = (B_l - sum_{l'<l} G_l' U_{l'l}) Uinv_l),
// replacing nleaf leaf solves and nleaf-1 GEMMs.
constexpr int TN_MAXLEAF = 4;
struct TrsmNodeArgs {
    u32* A;
    i64 lda;
    i32 row0, M;
    int nleaf;
    Dyn j_lo[TN_MAXLEAF], j_hi[TN_MAXLEAF];
    const u32* uinv[TN_MAXLEAF];
    const i32* uready[TN_MAXLEAF];  // when set: wait for each leaf's U^{-1} (== *epoch)
    const i32* epoch;
    const i32* rp;
    const i32* rrp;
    Fp f;
    u32* ninv;     // optional: also solve I * U_X^{-1} into ninv (NINV_LD x NINV_LD)
};
constexpr int NINV_LD = TN_MAXLEAF * PB;   // 256: pitch of a node inverse
// (M = 0 with ninv set: only the node inverse)
void trsm_node(const TrsmNodeArgs& a, cudaStream_t s);
// The same on the legacy tensor cores (trsm_tc.cu, p <= 2^16).
void trsm_node_tc(const TrsmNodeArgs& a, cudaStream_t s);

// Inverse of a unit upper block from its two diagonal halves (pivots
// [a_lo, b_lo) and [b_lo, b_hi), Dyn over rp):  X = [[Xa, T2], [0, Xb]] with
// T2 = -Xa * U_ab * Xb precomputed; every pitch static, nmax >= the live size.
void ninv_assemble(u32* X, i32 ldx, const u32* Xa, i32 la, const u32* Xb, i32 lb, const u32* T2, i32 lt,
                   Dyn a_lo, Dyn b_lo, Dyn b_hi, const i32* rp, i32 nmax, cudaStream_t s);

// The step between the two leaves of a leaf-pair node in ONE launch (bridge.cu,
// p <= 2^16): the top leaf's transpositions on the bottom rows (if its flag is
// set), G <- X * U_top^{-1} at the top pivots (written in place) and the window
// slice [n_lo, n_lo + PW) of the bottom rows updated by -G * U_top.
struct BridgeArgs {
    u32* A;
    i64 lda;
    i32 row0, M;     // bottom rows [row0, row0 + M), M <= PB
    Dyn j_lo, j_hi;  // the top leaf's pivots
    Dyn n_lo;        // slice start
    i32 N;           // matrix columns
    const i32* rp;
    const i32* rrp;
    const i32* ipiv;
    const u32* uinv;      // the top leaf's U^{-1} (PB x PB)
    const i32* uready;    // when set: wait for it (== *epoch) before reading uinv
    const i32* epoch;
    const i32* swapflag;  // the top leaf's "made a transposition" flag
    const PanelScratch* ps;  // the top leaf's panel scratch (dead_mask)
    Fp f;
};
void bridge(const BridgeArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- permutation
// Apply the transpositions T_{j, ipiv[j]} for j in [j_lo, j_hi) in increasing j
// to rows of A (perm_apply_cols of factor.cpp:42 / :56).  Rows are either the
// range [row0, row0 + M) or, when `gather` is set, rows gather[g_lo .. g_hi).
struct SwapArgs {
    u32* A;
    i64 lda;
    i32 row0, M;
    const i32* gather;
    Dyn g_lo, g_hi;
    Dyn j_lo, j_hi;
    const i32* rp;
    const i32* ipiv;
    i32 Mmax;
    // the job's transpositions are the pivots of leaves [leaf_lo, leaf_hi): when
    // none of their flags is set (generic inputs) the job is skipped without
    // scanning ipiv
    const i32* leafflags;
    i32 leaf_lo, leaf_hi;
};
constexpr int MAX_SWAP_JOBS = 8;
struct SwapJobs {
    SwapArgs job[MAX_SWAP_JOBS];
    int n;
};
// Row-disjoint swap jobs in one launch (applied in job order per row).
void apply_swaps(const SwapJobs& jobs, cudaStream_t s);

// Final placement of U rows (composed shifts of factor.cpp:62-70): for every
// pivot j with rrp[j] != j, row j, columns (j, n) <- row rrp[j], and the source
// is zero-filled; applied in increasing j per column.
void compact_u_rows(u32* A, i64 lda, i32 m, i32 n, const i32* rp, const i32* rrp,
                    cudaStream_t s);

// Closed-form random_matrix (reference.cpp:246-253) generated on device.
void gen_random_matrix(u32* A, i64 lda, i64 m, i64 n, u64 seed, u32 p, cudaStream_t s);

void fill_rp0(i32* rp, cudaStream_t s);
void bump_epoch(i32* epoch, cudaStream_t s);

// Data plane of the distributed CUP (dist.cu, paper_1112_5717_b200/dist.py).
void dist_pack(const u32* src, i64 lds, i64 rows, i64 cols, int wire16, void* dst, cudaStream_t s);
void dist_unpack(const void* src, i64 rows, i64 cols, int wire16, u32* dst, i64 ldd, const i64* colmap, i64 off,
                 cudaStream_t s);
void dist_select(const u32* src, i64 lds, i64 rows, const i64* colmap, i64 off, i64 cols, u32* dst, i64 ldd,
                 cudaStream_t s);
void dist_shift_u_rows(u32* x, i64 ldx, i64 cols, i64 r, i64 i0, i64 rt, const i64* gpos, cudaStream_t s);

}  // namespace rl
