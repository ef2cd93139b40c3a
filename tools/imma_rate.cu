// Legacy warp-level integer MMA (mma.sync m16n8k32 u8 x u8 -> s32) throughput
// and latency on this GPU, versus the CUDA-core IMAD.WIDE path.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/imma_rate tools/imma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CH>
__global__ void k(int* out, long long* cyc, int iters) {
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 7 + i;
    b[0] = threadIdx.x;
    b[1] = threadIdx.x * 3;
    int d[CH][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) imma(d[c], a, b);
    }
    long long t1 = clock64();
    int s = 0;
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    int* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4 * 8);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    long long h;
    // latency: one warp, one chain
    k<1><<<1, 32>>>(out, cyc, iters);
    k<1><<<1, 32>>>(out, cyc, iters);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mma.sync m16n8k32 u8: dependent latency %.1f cycles\n", (double)h / iters);
    // throughput: 148 SMs x 16 warps x 4 chains
    for (int warps : {4, 8, 16}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        k<4><<<148, 32 * warps>>>(out, cyc, iters);
        cudaEventRecord(e0);
        k<4><<<148, 32 * warps>>>(out, cyc, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double macs = 148.0 * warps * 4 * iters * (16.0 * 8 * 32);
        printf("warps/SM %2d: %.1f int8 TOPS (%.0f MAC/clk/SM by clock64)\n", warps, 2 * macs / (ms * 1e-3) / 1e12,
               (double)warps * 4 * iters * 16 * 8 * 32 / h);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
