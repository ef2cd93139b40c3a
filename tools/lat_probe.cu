// Dependent-chain latency of the accumulate forms (one warp, clock64 deltas).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k(const uint32_t* in, unsigned long long* out, uint64_t* sink) {
    uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1];
    // u64 += u32*u32 chain
    uint64_t acc = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) acc += (uint64_t)(uint32_t)acc * b;
    long long t1 = clock64();
    // u32 chain
    uint32_t x = a;
    long long t2 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x * b + a;
    long long t3 = clock64();
    // shared-memory load chain
    __shared__ uint32_t sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
    __syncwarp();
    uint32_t idx = threadIdx.x;
    long long t4 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) idx = sm[idx];
    long long t5 = clock64();
    // double fma chain
    double d = a;
    long long t6 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) d = fma(d, 1.0000001, (double)b);
    long long t7 = clock64();
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t3 - t2;
        out[2] = t5 - t4;
        out[3] = t7 - t6;
    }
    sink[threadIdx.x] = acc + x + idx + (uint64_t)d;
}

int main() {
    uint32_t* in;
    unsigned long long* out;
    uint64_t* sink;
    cudaMalloc(&in, 4096);
    cudaMemset(in, 3, 4096);
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 4096);
    k<<<1, 32>>>(in, out, sink);
    k<<<1, 32>>>(in, out, sink);
    unsigned long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: u64+=u32*u32 %.2f  u32 mad %.2f  LDS %.2f  DFMA %.2f\n",
           h[0] / (double)N, h[1] / (double)N, h[2] / (double)N, h[3] / (double)N);
    return 0;
}
