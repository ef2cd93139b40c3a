// util.h -- small device utilities (util.cu).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace rl {

// Matrices of at most TINY_MAX entries take the one-launch path: the input is
// the kernel's parameter block, the outputs land in mapped pinned host memory.
constexpr int TINY_MAX = 512;

struct TinyIn {
    u32 a[TINY_MAX];
    i32 m, n;
    Fp f;
};
struct TinyOut {
    i32 rank;
    i32 rrp[TINY_MAX];
    i32 ipiv[TINY_MAX];
    u32 body[TINY_MAX];
};

// *d_out <- digest of the m x n matrix at A (row stride lda), asynchronously on s.
void digest_u32(const u32* A, i64 lda, i64 m, i64 n, unsigned long long* d_out, cudaStream_t s);
// CUP of in.m x in.n (m*n <= TINY_MAX) into *out_mapped (host-mapped memory).
void cup_tiny(const TinyIn& in, TinyOut* out_mapped, cudaStream_t s);

}  // namespace rl
