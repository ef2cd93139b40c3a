// runtime.h -- host-side runtime helpers: errors, device properties.
#pragma once
#include <utility>
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace rl {

// Mirrors the reference error hierarchy (proj/include/ranklab/errors.hpp:9-66)
// at the C-ABI boundary: every exception is mapped to an RL_E* status code.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct CudaError : Error {
    CudaError(cudaError_t e, const char* what, const char* file, int line)
        : Error(5 /*RL_ECUDA*/, std::string("CUDA error ") + cudaGetErrorString(e) + " at " +
                                    file + ":" + std::to_string(line) + " (" + what + ")") {}
};

int num_sms();

// Every kernel of the CUP path prefers the maximum shared-memory carveout, so
// consecutive launches (1 KB ... 200 KB of shared memory) never make an SM
// reconfigure its L1/shared split between kernels.  Once per kernel.
template <class F>
inline void prefer_max_smem(F* kernel) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel),
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
#define RL_ONCE_MAX_SMEM(kernel)          \
    do {                                  \
        static bool once_ = false;        \
        if (!once_) {                     \
            prefer_max_smem(kernel);      \
            once_ = true;                 \
        }                                 \
    } while (0)

// Launch as a programmatic dependent of the previous kernel on the stream (the
// kernel must follow the pdl_wait/pdl_trigger protocol, common.cuh): its CTAs
// may start while the predecessor finishes, hiding launch latency inside the
// captured graph's dependent chains.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Growable device scratch buffer (workspaces of the host-pointer entry points
// and of the dense/triangular helpers; callers hold the C-ABI mutex).
struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (ptr) cudaFree(ptr);
            ptr = nullptr;
            cap = 0;
            if (cudaMalloc(&ptr, bytes) != cudaSuccess) throw Error(8 /*RL_ENOMEM*/, "cudaMalloc failed");
            cap = bytes;
        }
        return ptr;
    }
};

}  // namespace rl
