// Microbenchmark: per-launch cost of a chain of dependent kernels in a CUDA
// graph, with and without programmatic dependent launch (PDL).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launch_lat tools/launch_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
#if __CUDA_ARCH__ >= 900
    cudaGridDependencySynchronize();
#endif
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) p[0] += 1;
}

int main() {
    int* d;
    cudaMalloc(&d, 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int pdl = 0; pdl < 2; ++pdl) {
        for (int grid : {1, 148}) {
            const int N = 4000;
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < N; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                cudaLaunchKernelEx(&cfg, k_empty, d);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t ge;
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("pdl=%d grid=%d: %.3f us per dependent launch\n", pdl, grid, ms * 1e3 / N);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
