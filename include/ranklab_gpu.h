/*
 * ranklab_gpu.h -- C ABI of the B200-native CUP library (libranklab_gpu.so).
 *
 * Drop-in boundary for the reference's hot path (paths relative to
 * /root/reference).  Plain pointers and sizes only; matrices are row-major
 * uint32 with leading dimension `ld` (>= cols), entries canonical in [0, p),
 * p prime, 2 <= p < 2^31 (proj/include/ranklab/field.hpp:38-49).  Every entry
 * point returns an RL_* status; the C++ shim rethrows the
 * matching ranklab::Error subclass (proj/include/ranklab/errors.hpp:9-66).
 *
 * Functions taking host pointers copy to the device, compute there and copy
 * back; the *_dev variants take device pointers and a cudaStream_t (as void*,
 * NULL = legacy default stream) and keep all compute on the GPU.  There is no
 * CPU fallback: without a usable CUDA device every call returns RL_ECUDA.
 *
 * Threading (proj/README.md:164-168): every entry point is re-entrant.  Plans,
 * workspaces and copy streams are cached per (device, stream); host-pointer
 * calls run on cudaStreamPerThread, so distinct host threads never share them
 * and never wait for each other.  Calls on the same stream serialise.
 * Host buffers may be pinned (cudaHostAlloc/cudaHostRegister: the copies run
 * on copy streams overlapped with the factorization) or pageable (staged
 * through a pinned ring by host threads); matrices of <= 512 entries take a
 * one-launch path (input in the kernel parameters, outputs through mapped
 * pinned memory).
 */
#ifndef RANKLAB_GPU_H
#define RANKLAB_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RL_OK = 0,
    RL_EDIM = 1,       /* ranklab::DimensionMismatch */
    RL_EOVERLAP = 2,   /* ranklab::OverlapError */
    RL_ESINGULAR = 3,  /* ranklab::SingularMatrix / SingularDiagonal */
    RL_EFIELD = 4,     /* ranklab::NotPrime / ModulusOutOfRange */
    RL_ECUDA = 5,      /* CUDA runtime failure (ranklab::Error) */
    RL_ENCCL = 6,      /* NCCL failure (ranklab::Error) */
    RL_EINVAL = 7,     /* invalid argument (null pointer, ld < cols, ...) */
    RL_ENOMEM = 8      /* device allocation failed */
};

/* Field-op tallies in the order of ranklab::OpCounter (field.hpp:16-34):
 * ops[0] = n_mul, ops[1] = n_addsub, ops[2] = n_divinv, ops[3] = n_ztest.
 * Filled exactly from the recursion skeleton, the row profile and the pivot
 * positions (no counting on the device). */

/* In-place CUP: A <- packed [C\U], returns rank, row rank profile rrp[0..rank)
 * (capacity min(m,n)) and the column permutation sigma[0..n) with
 * A = C * U * P, column j of A*P^T = column sigma[j] of A.
 * Replaces: PackedCup ranklab::cup(MatView a, OpCounter& ctr)
 *           proj/include/ranklab/factor.hpp:34, proj/src/factor.cpp:85.
 * Any of rank/rrp/sigma/ops may be NULL. */
int rl_cup_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* rank,
               uint32_t* rrp, uint32_t* sigma, uint64_t* ops);

/* Same on a device-resident matrix; outputs are HOST pointers (may be NULL).
 * No host synchronisation happens before the outputs are requested. */
int rl_cup_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint32_t p,
                   int64_t* rank, uint32_t* rrp, uint32_t* sigma, uint64_t* ops,
                   void* stream);

/* PLE, cup's column-split mirror, in place: A = P*L*E, body [L\E] (L unit lower,
 * normalised; E row echelon with raw pivots).  col_profile (cap min(m,n)) =
 * pivot columns, increasing; row_perm (order m) = P; ops (NULL ok) = the
 * reference's exact charges.  Computed as cup(A^T)^T on the device (identical
 * by construction, factor.cpp:87-156 mirrors factor.cpp:30-81).
 * Replaces: PackedPle ranklab::ple(MatView a, OpCounter& ctr)
 *           proj/include/ranklab/factor.hpp:37, proj/src/factor.cpp:156. */
int rl_ple_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* rank,
               uint32_t* col_profile, uint32_t* row_perm, uint64_t* ops);
int rl_ple_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint32_t p,
                   int64_t* rank, uint32_t* col_profile, uint32_t* row_perm, uint64_t* ops,
                   void* stream);

/* Batched CUP of `batch` independent m x n matrices stored contiguously
 * (matrix t at dA + t*stride), device pointers; ranks[t] on the host.
 * rrp (batch x min(m,n)) and sigma (batch x n) are host arrays or NULL. */
int rl_cup_batched_u32_dev(uint32_t* dA, int64_t batch, int64_t m, int64_t n, int64_t stride,
                           uint32_t p, int64_t* ranks, uint32_t* rrp, uint32_t* sigma,
                           void* stream);
/* Same on HOST matrices (in place): the batch is copied in, factored and copied
 * back in chunks on three streams (PCIe both ways overlapped with the factoring;
 * pinned host memory gets the full link rate). */
int rl_cup_batched_u32(uint32_t* A, int64_t batch, int64_t m, int64_t n, int64_t stride,
                       uint32_t p, int64_t* ranks, uint32_t* rrp, uint32_t* sigma);

/* C <- alpha*A*B + beta*C (mod p); A m x l, B l x n, C m x n.
 * Replaces: void ranklab::mm(ConstMatView a, ConstMatView b, MatView c,
 *           Elem alpha, Elem beta, OpCounter&)  proj/include/ranklab/kernels.hpp:26-27
 *           (the library's declared substitution seam, kernels.hpp:13-19).
 * RL_EOVERLAP when C overlaps A or B (kernels.cpp:38-39).  ops may be NULL. */
int rl_mm_u32(const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t* C,
              int64_t ldc, int64_t m, int64_t l, int64_t n, uint32_t alpha, uint32_t beta,
              uint32_t p, uint64_t* ops);
int rl_mm_u32_dev(const uint32_t* dA, int64_t lda, const uint32_t* dB, int64_t ldb,
                  uint32_t* dC, int64_t ldc, int64_t m, int64_t l, int64_t n, uint32_t alpha,
                  uint32_t beta, uint32_t p, void* stream);
/* rl_mm_u32_dev with the persistent GEMM grid bounded to max_ctas CTAs (0 = all
 * SMs), so a latency-bound kernel on another stream (the distributed driver's
 * lookahead row-block factorization) finds SMs free. */
int rl_mm_u32_dev_grid(const uint32_t* dA, int64_t lda, const uint32_t* dB, int64_t ldb,
                       uint32_t* dC, int64_t ldc, int64_t m, int64_t l, int64_t n, uint32_t alpha,
                       uint32_t beta, uint32_t p, int max_ctas, void* stream);

/* Replaces: std::pair<size_t, std::vector<uint32_t>> ranklab::rank_and_profile(MatView,
 *           OpCounter&)  proj/include/ranklab/solvers.hpp:13-14 (input consumed). */
int rl_rank_and_profile_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p,
                            int64_t* rank, uint32_t* rrp);

/* Replaces: Elem ranklab::determinant(MatView, OpCounter&)  solvers.hpp:16
 * (sign(P) * product of pivots; input consumed). */
int rl_determinant_u32(uint32_t* A, int64_t n, int64_t lda, uint32_t p, uint32_t* det);

/* Column echelon transforms: cup, then (echelon.cpp:5-21) the body becomes
 * [C\X] with X the strict upper part of U^{-1}; with reduced != 0
 * (echelon.cpp:23-47) it becomes [[X1, X2], [R2, 0]] after the pivot-row
 * compression.  rank/rrp/sigma as rl_cup_u32; ops (NULL ok) = the exact
 * charges of cup plus the reduction.
 * Replaces: EchelonTransform ranklab::col_ech_trans(MatView, OpCounter&) and
 *           ReducedEchelonTransform ranklab::red_col_ech_trans(MatView, OpCounter&)
 *           proj/include/ranklab/echelon.hpp:28-29. */
int rl_col_ech_trans_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p,
                         int reduced, int64_t* rank, uint32_t* rrp, uint32_t* sigma,
                         uint64_t* ops);
int rl_col_ech_trans_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint32_t p,
                             int reduced, int64_t* rank, uint32_t* rrp, uint32_t* sigma,
                             uint64_t* ops, void* stream);

/* A <- A^{-1} in place (n x n).  RL_ESINGULAR when rank < n; the body then
 * holds red_col_ech_trans's output, as in the reference.
 * Replaces: void ranklab::invert_in_place(MatView, OpCounter&)
 *           proj/include/ranklab/solvers.hpp:19-22, proj/src/solvers.cpp:24-31. */
int rl_invert_u32(uint32_t* A, int64_t n, int64_t lda, uint32_t p, uint64_t* ops);
int rl_invert_u32_dev(uint32_t* dA, int64_t n, int64_t lda, uint32_t p, uint64_t* ops,
                      void* stream);

/* Triangular solve B <- T^{-1} B (side 0 = Left, T m x m) or B T^{-1}
 * (side 1 = Right, T n x n); uplo 0 = Upper, 1 = Lower; diag 1 = Unit (the
 * stored diagonal is never read), 0 = NonUnit.  B is m x n.  RL_EOVERLAP when
 * T overlaps B; RL_ESINGULAR for a zero NonUnit diagonal (B untouched; the
 * message names the index the reference would report).  ops (NULL ok) are
 * the reference's charges at `threshold`.
 * Replaces: void ranklab::trsm(Side, UpLo, Diag, ConstMatView t, MatView b,
 *           OpCounter&, size_t threshold)  proj/include/ranklab/kernels.hpp:37-38. */
int rl_trsm_u32(int side, int uplo, int diag, const uint32_t* T, int64_t ldt, uint32_t* B,
                int64_t ldb, int64_t m, int64_t n, uint32_t p, int64_t threshold,
                uint64_t* ops);
int rl_trsm_u32_dev(int side, int uplo, int diag, const uint32_t* dT, int64_t ldt,
                    uint32_t* dB, int64_t ldb, int64_t m, int64_t n, uint32_t p,
                    int64_t threshold, uint64_t* ops, void* stream);

/* Host-only op tallies (no device needed): the reference's trsm charges, and
 * what col_ech_trans (reduced: red_col_ech_trans) charges after its cup for
 * an m x n input of rank r. */
int rl_trsm_opcount(int side, int uplo, int diag, int64_t m, int64_t n, int64_t threshold,
                    uint64_t* ops);
int rl_echelon_opcount(int64_t m, int64_t n, int64_t r, int reduced, uint64_t* ops);

/* Seeded inputs generated on the device, bit-identical to
 * ranklab::random_matrix(m, n, seed, GF(p))  proj/src/reference.cpp:246-253. */
int rl_random_matrix_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint64_t seed,
                             uint32_t p, void* stream);

/* Order-independent 64-bit digest of a device matrix: the sum mod 2^64 of
 * splitmix_mix(((i*n + j) << 32 | A[i][j]) + 0x9E3779B97F4A7C15) over all
 * entries (splitmix_mix = the reference's SplitMix64 finaliser,
 * reference.cpp:177-180).  Test helper: the parity tests compare the packed
 * bodies of the benchmark configs (up to 17 GB) against CPU digests without
 * copying them back. */
int rl_digest_u32_dev(const uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint64_t* digest,
                      void* stream);

/* Data plane of the distributed CUP (config 5, paper_1112_5717_b200/dist.py),
 * enqueued on `stream`, no synchronisation.  Not a reference interface: the
 * reference has no multi-GPU path; these replace the eager tensor ops around
 * the NCCL collectives.
 *   pack:   dst (rows x cols, contiguous) <- src (ld lds); wire16 != 0: int16
 *           words x - 2^15 (p <= 2^16), else uint32.
 *   unpack: dst[r * ldd + colmap[c] - off] <- src[r * cols + c] (colmap NULL:
 *           c), undoing the 16-bit offset when wire16.
 *   select: dst[r * ldd + c] <- src[r * lds + colmap[c] - off], c < cols.
 *   shift:  for each column l < cols and j < min(rt, gpos[l] - r):
 *           x[r + j][l] <- x[i0 + j][l], x[i0 + j][l] <- 0, j increasing (the
 *           U-row move of factor.cpp:62-70 on one rank's columns; gpos[l] is
 *           column l's global position). */
int rl_dist_pack_u32_dev(const uint32_t* src, int64_t lds, int64_t rows, int64_t cols, int wire16, void* dst,
                         void* stream);
int rl_dist_unpack_u32_dev(const void* src, int64_t rows, int64_t cols, int wire16, uint32_t* dst, int64_t ldd,
                           const int64_t* colmap, int64_t off, void* stream);
int rl_dist_select_cols_u32_dev(const uint32_t* src, int64_t lds, int64_t rows, const int64_t* colmap,
                                int64_t off, int64_t cols, uint32_t* dst, int64_t ldd, void* stream);
int rl_dist_shift_u_rows_dev(uint32_t* x, int64_t ldx, int64_t cols, int64_t r, int64_t i0, int64_t rt,
                             const int64_t* gpos, void* stream);

/* Message of the last failing call on this thread ("" if none). */
const char* rl_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int rl_version(void);

/* Introspection for benchmarks: number of GEMM / tensor-core GEMM / panel /
 * leaf-TRSM launches of the last CUP plan built for (m, n, lda, p), and its
 * GEMM workspace in bytes, kernel launches per factorization.  stats[0..5]. */
int rl_cup_plan_stats(int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* stats);

/* Host-only (no device needed): the exact OpCounter charges of ranklab::cup
 * for an m x n input with the given rank, row profile and pivot positions
 * (ipiv[j] = column position where pivot j was found).  ops[4] as above. */
int rl_cup_opcount(int64_t m, int64_t n, int64_t rank, const uint32_t* rrp, const uint32_t* ipiv,
                   uint64_t* ops);

/* Benchmark helper: times the pack kernels and the tcgen05 GEMM kernel of
 * C <- C - A*B (m x l x n, dense device buffers) separately, averaged over
 * `iters` launches (CUDA events on `stream`).  l must respect the exact
 * accumulation bound (16384 for p < 2^16). */
int rl_profile_gemm_dev(const uint32_t* dA, const uint32_t* dB, uint32_t* dC, int64_t m,
                        int64_t l, int64_t n, uint32_t p, int iters, float* ms_pack,
                        float* ms_gemm, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RANKLAB_GPU_H */
