// tri.h -- dense mod-p GEMM driver, triangular inverses and the reductions that
// follow cup: col_ech_trans / red_col_ech_trans (proj/src/echelon.cpp:5-47),
// invert_in_place (proj/src/solvers.cpp:24-31) and the trsm seam
// (proj/src/kernels.cpp:135-154, 264-271).  Every result of these routines is a
// unique field value (an inverse, a solve, a product), so the GPU schedule --
// triangular inverse by recursive doubling on the tensor-core GEMM -- is
// bit-exact with the reference's recursive substitution.
#pragma once
#include "common.cuh"

namespace rl {

// C <- beta*C + alpha*A*B (m x l x n, row-major, arbitrary leading dims), the
// reference mm contract (kernels.hpp:26-27); K is chunked by the exact-
// accumulation bound, tensor cores above 32 in every dimension.  max_ctas > 0
// bounds the persistent grid (leaves SMs to a kernel running beside it).
void mm_dense(const u32* A, i64 lda, const u32* B, i64 ldb, u32* C, i64 ldc, i64 m, i64 l, i64 n,
              u32 alpha, u32 beta, const Fp& f, cudaStream_t s, int max_ctas = 0);

// X (k x k dense) <- the triangle of S: upper -> entries j > i, lower -> j < i,
// the diagonal from S (unit = false) or 1 (unit = true), zeros elsewhere.  A
// Unit extraction never reads S's diagonal (kernels.hpp:35-36).
void tri_extract(u32* X, i64 ldx, const u32* S, i64 lds, i32 k, bool upper, bool unit, u32 p,
                 cudaStream_t s);
// D's strict triangle (upper: j > i, lower: j < i) <- X's; D's diagonal and the
// other triangle are not touched.
void tri_store_strict(u32* D, i64 ldd, const u32* X, i64 ldx, i32 k, bool upper, cudaStream_t s);
// In place X <- X^{-1} for a dense k x k triangular X with nonzero diagonal
// (zeros in the other triangle).
void tri_inverse(u32* X, i64 ldx, i32 k, bool upper, const Fp& f, cudaStream_t s);

// red_col_ech_trans's pivot-row compression (echelon.cpp:32-36): for j = 0..r-1
// in order, swap rows j and rrp[j] over columns [0, j].
void compress_pivot_rows(u32* A, i64 lda, i32 r, const i32* d_rrp, cudaStream_t s);
// Row permutation "new row i <- old row tau[i]" for the listed rows only
// (perm_apply_rows, perm.cpp:103-113); d_idx holds pairs (i, tau[i]).
void move_rows(u32* A, i64 lda, i64 ncols, const i32* d_idx, i32 count, cudaStream_t s);

// D (cols x rows) <- S^T (S rows x cols); 32 x 32 shared-memory tiles, both
// sides coalesced (HBM-bound: 8 bytes per element).
void transpose(u32* D, i64 ldd, const u32* S, i64 lds, i64 rows, i64 cols, cudaStream_t s);

// Operation charges of the reference's routines (field.hpp:63-98 buckets
// {mul, addsub, divinv, ztest}), a pure function of the shapes and the
// threshold: the reference never skips zeros.
struct OpTally {
    u64 mul = 0, addsub = 0, divinv = 0, ztest = 0;
};
enum { SIDE_LEFT = 0, SIDE_RIGHT = 1 };
enum { UPLO_UPPER = 0, UPLO_LOWER = 1 };
void tally_trsm(OpTally& t, int side, int uplo, bool unit, i64 k, i64 rows, i64 cols, i64 threshold);
void tally_trtri(OpTally& t, bool unit, i64 n);
void tally_trulm_lower_owns(OpTally& t, i64 n);
// Everything col_ech_trans (reduced: red_col_ech_trans) charges after its cup.
void tally_echelon(OpTally& t, i64 m, i64 n, i64 r, bool reduced);

}  // namespace rl
