// runtime.h -- host-side runtime helpers: errors, device properties.
#pragma once
#include <utility>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
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

// The calling thread's current device (every per-device cache is keyed by it).
int current_device();
// SM count of the current device (cached per device).
int num_sms();

// Runs fn exactly once per (call site, device); a concurrent caller on another
// host thread WAITS until that first run completed (a kernel must not be
// launched before its shared-memory attribute is set).
template <class F>
inline void once_on_device(std::atomic<unsigned long long>& done, F&& fn) {
    const unsigned long long bit = 1ull << (current_device() & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    static std::mutex mu;  // one per F (call site), shared by the devices
    std::lock_guard<std::mutex> lk(mu);
    if (done.load(std::memory_order_relaxed) & bit) return;
    fn();
    done.fetch_or(bit, std::memory_order_release);
}
#define RL_ONCE_PER_DEVICE()                                 \
    ([]() -> std::atomic<unsigned long long>& {              \
        static std::atomic<unsigned long long> m_{0};        \
        return m_;                                           \
    }())

// Every kernel of the CUP path prefers the maximum shared-memory carveout, so
// consecutive launches (1 KB ... 200 KB of shared memory) never make an SM
// reconfigure its L1/shared split between kernels.  Once per kernel and device.
template <class F>
inline void prefer_max_smem(F* kernel) {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel),
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
#define RL_ONCE_MAX_SMEM(kernel)                                     \
    do {                                                             \
        static std::atomic<unsigned long long> once_{0};             \
        once_on_device(once_, [&] { prefer_max_smem(kernel); });     \
    } while (0)
// cudaFuncSetAttribute(kernel, MaxDynamicSharedMemorySize, bytes) once per device.
#define RL_ONCE_SMEM_LIMIT(kernel, bytes)                                                   \
    do {                                                                                    \
        static std::atomic<unsigned long long> once_{0};                                    \
        once_on_device(once_, [&] {                                                         \
            RL_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                               (int)(bytes)));                              \
        });                                                                                 \
    } while (0)

// RL_NO_PDL=1 launches every kernel as a plain dependent (debugging aid).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RL_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

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
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    RL_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Growable device scratch buffer (workspaces of the host-pointer entry points
// and of the dense/triangular helpers; one set per call context, see Scratch).
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

// Per-(device, stream) call context.  The C-ABI entry points hold `mu` for the
// duration of a call, so calls on DISTINCT streams never share a workspace and
// never wait for each other, while calls on the same stream (which the GPU
// serialises anyway) cannot reallocate a buffer under an in-flight call.
// cudaStreamPerThread is one handle for all threads: its contexts are keyed by
// the calling thread as well (each thread has its own per-thread stream).
enum ScratchSlot {
    SS_A, SS_B, SS_C, SS_META, SS_TRANS,          // host-pointer entry points
    SS_X, SS_Y, SS_T, SS_IDX, SS_PERM,            // echelon / inverse / trsm seam
    SS_MM_A2, SS_MM_B2, SS_TRI_W, SS_MOVE,        // dense helpers (tri.cu)
    SS_PROF_A2, SS_PROF_B2, SS_DIGEST,            // benchmark / test helpers
    SS_COUNT
};
struct Scratch {
    std::mutex mu;
    int device = 0;
    DevBuf buf[SS_COUNT];
    cudaStream_t aux[4] = {};     // copy streams of the host-buffer paths (lazy)
    cudaEvent_t ev[96] = {};      // their events (lazy)
    void* pinned = nullptr;       // pinned staging ring of the pageable-host path (lazy)
    size_t pinned_cap = 0;
    void* pinned_out = nullptr;   // its device -> host ring (pipelined pageable path, lazy)
    size_t pinned_out_cap = 0;
    unsigned* host_flags = nullptr;  // mapped pinned words the copy streams wait on (lazy)
    void* host_mapped = nullptr;  // mapped pinned result block of the tiny-matrix path (lazy)
    void* get(int slot, size_t bytes) { return buf[slot].get(bytes); }
    cudaStream_t aux_stream(int i);
    cudaEvent_t event(int i);
    void* pinned_ring(size_t bytes);
    void* pinned_ring_out(size_t bytes);
    unsigned* flags();  // 16 words of mapped pinned memory, zeroed
};
Scratch& scratch_for(cudaStream_t s);
// The host-buffer entry points' stream: one NON-blocking stream per (host
// thread, device), so those calls never synchronise implicitly with the legacy
// stream (or with work another thread is capturing into a graph).
cudaStream_t host_stream();

}  // namespace rl
