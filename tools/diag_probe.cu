// Cycle count of the 8 x 8 unit-upper back substitution used by leaf_uinv
// (panel.cu), in isolation, and of its building blocks (red_sp / red32 chains).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1112_5717_b200/csrc -o tools/diag_probe tools/diag_probe.cu
#include <cstdio>
#include "common.cuh"

constexpr int PB = 64;

template <int VAR>
__global__ void diag(const u32* in, long long* out, u32* sink, Fp f, int rt) {
    __shared__ u32 U[PB][PB + 1], X[PB][PB + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < PB * PB; e += blockDim.x) U[e / PB][e % PB] = in[e] % f.p;
    __syncthreads();
    const u32 one = 1u % f.p;
    long long t0 = clock64();
    if (warp < 8 && lane < 8) {
        const int base = 8 * warp, c = lane;
        u32 x[8];
#pragma unroll
        for (int i = 7; i >= 0; --i) {
            u64 acc = 0;
#pragma unroll
            for (int k = i + 1; k < 8; ++k) acc += (u64)U[base + i][base + k] * x[k];
            const u32 sum = red_sp(acc, f);
            u32 d;
            if (VAR == 0) d = (i == c && base + i < rt) ? 1u % f.p : 0u;
            else d = (i == c) ? one : 0u;
            x[i] = i > c ? 0u : submod(d, sum, f);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) X[base + i][base + c] = x[i];
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) out[VAR] = t1 - t0;
    // red_sp dependent chain
    u32 v = in[tid] % f.p;
    long long t2 = clock64();
#pragma unroll 16
    for (int i = 0; i < 1024; ++i) v = red_sp((u64)v * 40000u + 12345u, f);
    long long t3 = clock64();
    if (tid == 0) out[2 + VAR] = t3 - t2;
    sink[tid] = v + X[tid & 63][tid >> 3];
}

int main() {
    u32* in;
    long long* out;
    u32* sink;
    cudaMalloc(&in, PB * PB * 4);
    cudaMemset(in, 7, PB * PB * 4);
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 4096);
    Fp f = make_fp(65521);
    for (int rep = 0; rep < 2; ++rep) {
        diag<0><<<1, 512>>>(in, out, sink, f, 64);
        diag<1><<<1, 512>>>(in, out, sink, f, 64);
    }
    long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("diag 8x8 backsub: orig %lld cycles, hoisted one %lld cycles; red_sp chain %.1f / %.1f cycles per op\n",
           h[0], h[1], h[2] / 1024.0, h[3] / 1024.0);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
