// Microbenchmark: throughput of the multiply-accumulate forms usable for exact
// mod-p sums on CUDA cores: u64 += u32*u32 (IMAD.WIDE), double fma (DFMA),
// u32 IMAD (mad.lo), float FFMA.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mac_rate tools/mac_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ACC = 16, ITERS = 4096;

__global__ void k_wide(const uint32_t* in, uint64_t* out) {
    uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1];
    uint64_t acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) acc[i] += (uint64_t)(a + i) * b;
        a ^= it;
    }
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(const uint32_t* in, double* out) {
    double a = in[threadIdx.x], b = in[threadIdx.x + 1];
    double acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) acc[i] = fma(a + i, b, acc[i]);
        a += 1.0;
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad(const uint32_t* in, uint32_t* out) {
    uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1];
    uint32_t acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) acc[i] += (a + i) * b;
        a ^= it;
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(const uint32_t* in, float* out) {
    float a = in[threadIdx.x], b = in[threadIdx.x + 1];
    float acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) acc[i] = fmaf(a + i, b, acc[i]);
        a += 1.0f;
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K, class T>
void run(const char* name, K k, uint32_t* in, T* out, int sms) {
    const int blocks = sms * 8, threads = 256;
    k<<<blocks, threads>>>(in, out);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(in, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = (double)blocks * threads * ITERS * ACC;
    printf("%-34s %8.3f ms  %7.2f T MAC/s  %6.1f MAC/clk/SM (at 1.9 GHz)\n", name, ms, macs / ms / 1e9,
           macs / (ms * 1e-3) / sms / 1.9e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* in;
    cudaMalloc(&in, 4096 * 4);
    cudaMemset(in, 1, 4096 * 4);
    void* out;
    cudaMalloc(&out, (size_t)sms * 8 * 256 * 8);
    run("u64 += u32*u32 (IMAD.WIDE)", k_wide, in, (uint64_t*)out, sms);
    run("double fma (DFMA)", k_dfma, in, (double*)out, sms);
    run("u32 += u32*u32 (IMAD)", k_imad, in, (uint32_t*)out, sms);
    run("float fma (FFMA)", k_ffma, in, (float*)out, sms);
    return 0;
}
