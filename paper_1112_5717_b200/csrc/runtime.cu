// runtime.cu -- per-device and per-stream host state of the library.
//
// The reference's threading contract (proj/README.md:164-168): no internal
// threads, disjoint views may be processed concurrently.  Here that means no
// process-global mutable state on the compute path: caches are keyed by the
// device, workspaces by (device, stream), so concurrent calls on distinct
// streams -- or distinct host threads using cudaStreamPerThread -- proceed in
// parallel (SURVEY.md 8(b) "Threading").
#include <cstdlib>
#include <map>
#include <memory>
#include <thread>
#include <tuple>

#include "common.cuh"
#include "runtime.h"

// The launch sequence of one factorization spans ~20 streams (critical path,
// side streams, row-split and tile lanes, copy streams); with the default 8
// hardware work queues, a stream blocked on an event (a tile lane waiting for
// its rows to arrive from the host) stalls the other streams sharing its
// queue.  Ask for the maximum (32) when the library is loaded -- before the
// host program creates its CUDA context -- unless the user chose a value.
__attribute__((constructor)) static void rl_max_connections() {
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
}

namespace rl {

int current_device() {
    int d = 0;
    RL_CUDA_CHECK(cudaGetDevice(&d));
    return d;
}

int num_sms() {
    static std::atomic<int> cache[64] = {};
    const int d = current_device() & 63;
    int n = cache[d].load(std::memory_order_relaxed);
    if (!n) {
        RL_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device()));
        cache[d].store(n, std::memory_order_relaxed);
    }
    return n;
}

namespace {
struct ScratchKey {
    int dev;
    cudaStream_t s;
    std::thread::id tid;  // only for cudaStreamPerThread
    bool operator<(const ScratchKey& o) const {
        return std::tie(dev, s, tid) < std::tie(o.dev, o.s, o.tid);
    }
};
std::mutex g_scratch_mu;
std::map<ScratchKey, std::unique_ptr<Scratch>>& scratch_map() {
    static auto* m = new std::map<ScratchKey, std::unique_ptr<Scratch>>();  // never destroyed:
    return *m;  // CUDA objects must not be released after the driver shut down
}
}  // namespace

Scratch& scratch_for(cudaStream_t s) {
    ScratchKey k{current_device(), s, s == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id()};
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    auto& m = scratch_map();
    auto it = m.find(k);
    if (it != m.end()) return *it->second;
    auto sc = std::make_unique<Scratch>();
    sc->device = k.dev;
    Scratch& ref = *sc;
    m.emplace(k, std::move(sc));
    return ref;
}

cudaStream_t host_stream() {
    thread_local cudaStream_t per_dev[64] = {};
    const int d = current_device() & 63;
    if (!per_dev[d]) RL_CUDA_CHECK(cudaStreamCreateWithFlags(&per_dev[d], cudaStreamNonBlocking));
    return per_dev[d];
}

cudaStream_t Scratch::aux_stream(int i) {
    if (!aux[i]) RL_CUDA_CHECK(cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking));
    return aux[i];
}

cudaEvent_t Scratch::event(int i) {
    if (i < 0 || i >= (int)(sizeof(ev) / sizeof(ev[0]))) throw Error(7 /*RL_EINVAL*/, "copy event pool exhausted");
    if (!ev[i]) RL_CUDA_CHECK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    return ev[i];
}

void* Scratch::pinned_ring(size_t bytes) {
    if (bytes > pinned_cap) {
        if (pinned) cudaFreeHost(pinned);
        pinned = nullptr;
        pinned_cap = 0;
        if (cudaMallocHost(&pinned, bytes) != cudaSuccess) throw Error(8 /*RL_ENOMEM*/, "cudaMallocHost failed");
        pinned_cap = bytes;
    }
    return pinned;
}

void* Scratch::pinned_ring_out(size_t bytes) {
    if (bytes > pinned_out_cap) {
        if (pinned_out) cudaFreeHost(pinned_out);
        pinned_out = nullptr;
        pinned_out_cap = 0;
        if (cudaMallocHost(&pinned_out, bytes) != cudaSuccess) throw Error(8 /*RL_ENOMEM*/, "cudaMallocHost failed");
        pinned_out_cap = bytes;
    }
    return pinned_out;
}

unsigned* Scratch::flags() {
    if (!host_flags) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, 64, cudaHostAllocMapped) != cudaSuccess)
            throw Error(8 /*RL_ENOMEM*/, "cudaHostAlloc (mapped) failed");
        host_flags = static_cast<unsigned*>(p);
    }
    for (int i = 0; i < 16; ++i) host_flags[i] = 0;
    return host_flags;
}

}  // namespace rl
