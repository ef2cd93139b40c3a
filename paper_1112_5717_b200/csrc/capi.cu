// capi.cu -- the extern "C" boundary (include/ranklab_gpu.h).
//
// Maps the reference's C++ contracts onto plain pointers: validation and error
// codes follow proj/include/ranklab/errors.hpp (DimensionMismatch, OverlapError,
// SingularMatrix, NotPrime/ModulusOutOfRange), field validation follows
// PrimeField (proj/src/field.cpp:24-58).  Engines (plans + workspaces + graphs)
// are cached per (m, n, lda, p) behind a mutex; calls are re-entrant per stream.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/ranklab_gpu.h"
#include "cup.h"
#include "kernels.cuh"
#include "runtime.h"
#include "tri.h"
#include "util.h"

namespace rl {
void cup_batched(u32* dA, i64 batch, i32 m, i32 n, i64 stride, u32 p, i32* d_ranks, i32* d_rrp,
                 i32* d_ipiv, i32 kcap, cudaStream_t s);
}

using namespace rl;

namespace {

thread_local std::string g_last_error;

u64 mulmod_host(u64 a, u64 b, u64 m) { return (u64)((unsigned __int128)a * b % m); }
u64 powmod_host(u64 a, u64 e, u64 m) {
    u64 r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = mulmod_host(r, a, m);
        a = mulmod_host(a, a, m);
        e >>= 1;
    }
    return r;
}
// Deterministic Miller-Rabin (the witness set decides all 64-bit inputs).
bool is_prime(u64 n) {
    if (n < 2) return false;
    for (u64 q : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull})
        if (n % q == 0) return n == q;
    u64 d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    for (u64 a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
        u64 x = powmod_host(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < s; ++i) {
            x = mulmod_host(x, x, n);
            if (x == n - 1) {
                comp = false;
                break;
            }
        }
        if (comp) return false;
    }
    return true;
}

void check_field(u32 p) {
    if (p < 2 || p >= (1u << 31)) throw Error(RL_EFIELD, "modulus outside [2, 2^31)");
    if (!is_prime(p)) throw Error(RL_EFIELD, "modulus is not prime");
}

template <class F>
int guard(F&& f) {
    try {
        f();
        g_last_error.clear();
        return RL_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = "host allocation failed";
        return RL_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return RL_EINVAL;
    }
}

// Engines (plan + workspaces + captured graph) are cached per (device, stream,
// m, n, lda, p): a call on one stream never touches another stream's engine,
// so concurrent factorizations on distinct streams run in parallel.  The cache
// is bounded; an evicted engine waits for its last (possibly asynchronous) run.
struct Key {
    int dev;
    cudaStream_t s;
    std::thread::id tid;  // cudaStreamPerThread: one engine set per host thread
    i64 m, n, lda;
    u32 p;
    bool split = false;  // host-buffer engine with the split H2D wait
    bool operator<(const Key& o) const {
        return std::tie(dev, s, tid, m, n, lda, p, split) <
               std::tie(o.dev, o.s, o.tid, o.m, o.n, o.lda, o.p, o.split);
    }
};
struct Cached {
    std::shared_ptr<CupEngine> e;
    unsigned long long used = 0;
};
std::mutex g_engines_mu;
std::map<Key, Cached> g_engines;
unsigned long long g_tick = 0;
constexpr size_t kMaxEngines = 16;

std::shared_ptr<CupEngine> engine_for(i64 m, i64 n, i64 lda, u32 p, cudaStream_t s, bool split = false) {
    Key k{current_device(), s, s == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id(),
          m, n, lda, p, split};
    std::shared_ptr<CupEngine> victim;  // destroyed outside the lock
    {
        std::lock_guard<std::mutex> lk(g_engines_mu);
        auto it = g_engines.find(k);
        if (it != g_engines.end()) {
            it->second.used = ++g_tick;
            return it->second.e;
        }
        if (g_engines.size() >= kMaxEngines) {
            auto lru = g_engines.end();
            for (auto j = g_engines.begin(); j != g_engines.end(); ++j)
                if (j->second.e.use_count() == 1 && (lru == g_engines.end() || j->second.used < lru->second.used))
                    lru = j;
            if (lru != g_engines.end()) {
                victim = std::move(lru->second.e);
                g_engines.erase(lru);
            }
        }
    }
    victim.reset();
    auto e = std::make_shared<CupEngine>((i32)m, (i32)n, lda, p);
    std::lock_guard<std::mutex> lk(g_engines_mu);
    auto res = g_engines.emplace(k, Cached{e, ++g_tick});
    return res.first->second.e;
}

// One C-ABI call's hold on its stream's context (workspaces, copy streams):
// calls on the same stream serialise here, calls on distinct streams do not.
struct Call {
    Scratch& sc;
    std::unique_lock<std::mutex> lk;
    explicit Call(cudaStream_t s) : sc(scratch_for(s)), lk(sc.mu) {}
};

void require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw Error(RL_ECUDA, "no CUDA device (the GPU path has no CPU fallback)");
}

void check_dims(i64 m, i64 n, i64 ld) {
    if (m < 0 || n < 0) throw Error(RL_EDIM, "negative dimension");
    if (m > (1ll << 30) || n > (1ll << 30)) throw Error(RL_EDIM, "dimension too large");
    if (n > 0 && ld < n) throw Error(RL_EINVAL, "leading dimension smaller than column count");
}

// Byte-range rectangle overlap of two row-major windows (ConstMatView::overlaps,
// matrix.hpp:54-59, generalised to raw pointers).
bool windows_overlap(const u32* a, i64 ar, i64 ac, i64 lda, const u32* c, i64 cr, i64 cc, i64 ldc) {
    if (ar == 0 || ac == 0 || cr == 0 || cc == 0) return false;
    const char* a0 = (const char*)a;
    const char* a1 = (const char*)(a + (ar - 1) * lda + ac);
    const char* c0 = (const char*)c;
    const char* c1 = (const char*)(c + (cr - 1) * ldc + cc);
    if (a1 <= c0 || c1 <= a0) return false;
    if (lda != ldc) return true;  // conservative
    const i64 off = (i64)(c - a);  // element offset of C's origin in A's frame
    const i64 orow = off >= 0 ? off / lda : -((-off + lda - 1) / lda);
    const i64 ocol = off - orow * lda;
    // C occupies rows [orow, orow+cr), cols [ocol, ocol+cc) of A's frame
    // (cols may spill past lda only if ocol + cc > lda: treat conservatively)
    if (ocol + cc > lda) return true;
    const bool row_hit = orow < ar && 0 < orow + cr;
    const bool col_hit = ocol < ac && 0 < ocol + cc;
    return row_hit && col_hit;
}

void cup_dev_impl(u32* dA, i64 m, i64 n, i64 lda, u32 p, i64* rank, u32* rrp, u32* sigma,
                  u64* ops, cudaStream_t s) {
    check_field(p);
    check_dims(m, n, lda);
    if (m == 0 || n == 0) {  // factor.cpp:32: rank 0, identity, storage untouched
        if (rank) *rank = 0;
        if (sigma) for (i64 j = 0; j < n; ++j) sigma[j] = (u32)j;
        if (ops) std::fill(ops, ops + 4, 0ull);
        return;
    }
    require_device();
    i64 r = 0;
    std::vector<u32> rrp_h((size_t)std::min(m, n)), ipiv_h((size_t)std::min(m, n));
    {
        Call call(s);
        auto e = engine_for(m, n, lda, p, s);
        e->run(dA, s, /*use_graph=*/m * n >= (1 << 18));  // capture pays off for large plans
        if (!rank && !rrp && !sigma && !ops) return;  // fully asynchronous
        e->results(&r, rrp_h.data(), ipiv_h.data(), s);
    }
    if (rank) *rank = r;
    if (rrp) std::copy(rrp_h.begin(), rrp_h.begin() + r, rrp);
    if (sigma) sigma_from_ipiv(n, r, ipiv_h.data(), sigma);
    if (ops) cup_opcount(m, n, r, rrp_h.data(), ipiv_h.data(), ops);
}

void copy_h2d_2d(u32* d, i64 dld, const u32* h, i64 hld, i64 rows, i64 cols, cudaStream_t s) {
    if (rows == 0 || cols == 0) return;
    RL_CUDA_CHECK(cudaMemcpy2DAsync(d, dld * 4, h, hld * 4, cols * 4, rows, cudaMemcpyHostToDevice, s));
}
void copy_d2h_2d(u32* h, i64 hld, const u32* d, i64 dld, i64 rows, i64 cols, cudaStream_t s) {
    if (rows == 0 || cols == 0) return;
    RL_CUDA_CHECK(cudaMemcpy2DAsync(h, hld * 4, d, dld * 4, cols * 4, rows, cudaMemcpyDeviceToHost, s));
}

void mm_dev_impl(const u32* dA, i64 lda, const u32* dB, i64 ldb, u32* dC, i64 ldc, i64 m, i64 l,
                 i64 n, u32 alpha, u32 beta, u32 p, cudaStream_t s, int max_ctas = 0) {
    mm_dense(dA, lda, dB, ldb, dC, ldc, m, l, n, alpha, beta, make_fp(p), s, max_ctas);
}

// cup of a device matrix, results on the host (synchronises s).  Small shapes
// run as one CTA (one launch), larger ones through the cached engine.
void factor_on_device(u32* dA, i64 m, i64 n, i64 lda, u32 p, cudaStream_t s, i64* r,
                      std::vector<u32>& rrp_h, std::vector<u32>& ipiv_h) {
    const i64 kcap = std::min(m, n);
    rrp_h.assign((size_t)kcap, 0);
    ipiv_h.assign((size_t)kcap, 0);
    if (m <= 64 && n <= 256 && lda == n) {
        i32* dmeta = (i32*)scratch_for(s).get(SS_META, (size_t)(1 + 2 * kcap) * 4);
        cup_batched(dA, 1, (i32)m, (i32)n, m * n, p, dmeta, dmeta + 1, dmeta + 1 + kcap, (i32)kcap, s);
        std::vector<i32> meta((size_t)(1 + 2 * kcap));
        RL_CUDA_CHECK(cudaMemcpyAsync(meta.data(), dmeta, meta.size() * 4, cudaMemcpyDeviceToHost, s));
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
        *r = meta[0];
        std::copy((const u32*)&meta[1], (const u32*)&meta[1] + *r, rrp_h.begin());
        std::copy((const u32*)&meta[1 + kcap], (const u32*)&meta[1 + kcap] + *r, ipiv_h.begin());
        return;
    }
    auto e = engine_for(m, n, lda, p, s);
    e->run(dA, s, m * n >= (1 << 18));
    e->results(r, rrp_h.data(), ipiv_h.data(), s);  // synchronises s
}

// Is host memory at h page-locked (cudaHostAlloc / cudaHostRegister)?
bool host_pinned(const void* h) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// RL_PAGEABLE_DIRECT=1: pageable buffers go straight to cudaMemcpy2DAsync (the
// driver's own synchronous staging) -- kept for the benchmark comparison.
bool pageable_direct() {
    static const bool v = [] {
        const char* e = getenv("RL_PAGEABLE_DIRECT");
        return e && e[0] == '1';
    }();
    return v;
}

// rows x cols words between row-strided host buffers, split over host threads
// (a single core copies pageable memory at ~10 GB/s, well below PCIe).
void par_copy_rows(u32* dst, i64 dld, const u32* src, i64 sld, i64 rows, i64 cols) {
    const size_t bytes = (size_t)rows * cols * 4;
    const int T = bytes >= (8u << 20) ? 8 : 1;
    auto part = [&](int t) {
        const i64 r0 = rows * t / T, r1 = rows * (t + 1) / T;
        if (dld == cols && sld == cols) {
            std::memcpy(dst + r0 * dld, src + r0 * sld, (size_t)(r1 - r0) * cols * 4);
        } else {
            for (i64 i = r0; i < r1; ++i) std::memcpy(dst + i * dld, src + i * sld, (size_t)cols * 4);
        }
    };
    if (T == 1) return part(0);
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(part, t);
    part(0);
    for (auto& x : th) x.join();
}

// Pageable host -> device through a ring of R pinned slots: host threads fill
// slot k % R while the DMA of the previous chunks runs; a slot is refilled
// only after the DMA that read it completed (its event).
constexpr int kRing = 4;
constexpr size_t kChunkBytes = 32u << 20;
void staged_h2d(u32* d, i64 dld, const u32* h, i64 hld, i64 rows, i64 cols, Scratch& sc, cudaStream_t s) {
    const i64 crow = std::max<i64>(1, (i64)(kChunkBytes / ((size_t)cols * 4)));
    u32* ring = (u32*)sc.pinned_ring((size_t)kRing * crow * cols * 4);
    i64 k = 0;
    for (i64 r0 = 0; r0 < rows; r0 += crow, ++k) {
        const i64 nr = std::min(crow, rows - r0);
        const int slot = (int)(k % kRing);
        u32* buf = ring + (size_t)slot * crow * cols;
        if (k >= kRing) RL_CUDA_CHECK(cudaEventSynchronize(sc.event(slot)));
        par_copy_rows(buf, cols, h + r0 * hld, hld, nr, cols);
        RL_CUDA_CHECK(cudaMemcpy2DAsync(d + r0 * dld, dld * 4, buf, cols * 4, cols * 4, nr,
                                        cudaMemcpyHostToDevice, s));
        RL_CUDA_CHECK(cudaEventRecord(sc.event(slot), s));
    }
}

// Device -> pageable host: the DMA of up to R chunks runs ahead of the host
// threads draining the ring.
void staged_d2h(u32* h, i64 hld, const u32* d, i64 dld, i64 rows, i64 cols, Scratch& sc, cudaStream_t s) {
    const i64 crow = std::max<i64>(1, (i64)(kChunkBytes / ((size_t)cols * 4)));
    u32* ring = (u32*)sc.pinned_ring((size_t)kRing * crow * cols * 4);
    const i64 nchunks = (rows + crow - 1) / crow;
    auto issue = [&](i64 k) {
        const i64 r0 = k * crow, nr = std::min(crow, rows - r0);
        const int slot = (int)(k % kRing);
        RL_CUDA_CHECK(cudaMemcpy2DAsync(ring + (size_t)slot * crow * cols, cols * 4, d + r0 * dld, dld * 4,
                                        cols * 4, nr, cudaMemcpyDeviceToHost, s));
        RL_CUDA_CHECK(cudaEventRecord(sc.event(kRing + slot), s));
    };
    for (i64 k = 0; k < std::min<i64>(kRing, nchunks); ++k) issue(k);
    for (i64 k = 0; k < nchunks; ++k) {
        const i64 r0 = k * crow, nr = std::min(crow, rows - r0);
        const int slot = (int)(k % kRing);
        RL_CUDA_CHECK(cudaEventSynchronize(sc.event(kRing + slot)));
        par_copy_rows(h + r0 * hld, hld, ring + (size_t)slot * crow * cols, cols, nr, cols);
        if (k + kRing < nchunks) issue(k + kRing);
    }
}

// One-launch CUP of a matrix of <= TINY_MAX entries (util.cu): the input rides
// in the kernel parameters, the outputs come back through mapped pinned memory.
void tiny_cup(const u32* A, i64 m, i64 n, i64 lda, u32 p, Scratch& sc, cudaStream_t s, i64* r,
              std::vector<u32>& rrp_h, std::vector<u32>& ipiv_h) {
    TinyIn in;
    for (i64 i = 0; i < m; ++i)
        for (i64 j = 0; j < n; ++j) in.a[i * n + j] = A[i * lda + j];
    in.m = (i32)m;
    in.n = (i32)n;
    in.f = make_fp(p);
    if (!sc.host_mapped)
        RL_CUDA_CHECK(cudaHostAlloc(&sc.host_mapped, sizeof(TinyOut), cudaHostAllocMapped));
    TinyOut* ho = (TinyOut*)sc.host_mapped;
    TinyOut* dout = nullptr;
    RL_CUDA_CHECK(cudaHostGetDevicePointer((void**)&dout, ho, 0));
    cup_tiny(in, dout, s);
    RL_CUDA_CHECK(cudaStreamSynchronize(s));
    *r = ho->rank;
    const i64 kcap = std::min(m, n);
    rrp_h.assign((size_t)kcap, 0);
    ipiv_h.assign((size_t)kcap, 0);
    for (i64 j = 0; j < *r; ++j) {
        rrp_h[j] = (u32)ho->rrp[j];
        ipiv_h[j] = (u32)ho->ipiv[j];
    }
    u32* Aw = const_cast<u32*>(A);
    for (i64 i = 0; i < m; ++i)
        for (i64 j = 0; j < n; ++j) Aw[i * lda + j] = ho->body[i * n + j];
}

// Host-pinned CUP with PCIe overlapped along the recursion's spines (the
// splits of factor.cpp:35).  In: rows [0, m/2^D) are copied first and factored
// while the rest crosses the link in order on a second stream; each left-spine
// node (0, mm) waits for its bottom rows right before it first touches them.
// Out: each right-spine node's top half goes back as soon as it is factored
// (final unless a later transposition or U-row move reaches it: then it is
// copied again).  Copy streams and events belong to the calling stream's context.
void cup_host_overlapped_tiles(u32* A, i64 m, i64 n, i64 lda, u32 p, u32* dA, Scratch& sc, cudaStream_t s,
                               i64* r, std::vector<u32>& rrp_h, std::vector<u32>& ipiv_h,
                               const std::shared_ptr<CupEngine>& e);

void cup_host_overlapped(u32* A, i64 m, i64 n, i64 lda, u32 p, u32* dA, Scratch& sc, cudaStream_t s, i64* r,
                         std::vector<u32>& rrp_h, std::vector<u32>& ipiv_h) {
    {
        auto e = engine_for(m, n, n, p, s, true);
        if (e->tile_rows() > 0 && (m + e->tile_rows() - 1) / e->tile_rows() <= 40)
            return cup_host_overlapped_tiles(A, m, n, lda, p, dA, sc, s, r, rrp_h, ipiv_h, e);
    }
    constexpr int D = 3;
    cudaStream_t cs = sc.aux_stream(0), cs2 = sc.aux_stream(1);
    cudaEvent_t top = sc.event(2 * kRing);
    cudaEvent_t evw[D], evd[D];
    for (int d = 0; d < D; ++d) {
        evw[d] = sc.event(2 * kRing + 1 + d);
        evd[d] = sc.event(2 * kRing + 1 + D + d);
    }
    CupEngine::NodeEvents waits, dones;
    // left spine: node (0, sz[d]), sz[0] = m, sz[d+1] = sz[d] / 2
    i64 sz[D + 1];
    sz[0] = m;
    for (int d = 0; d < D; ++d) sz[d + 1] = sz[d] / 2;
    copy_h2d_2d(dA, n, A, lda, sz[D], n, s);
    RL_CUDA_CHECK(cudaEventRecord(top, s));
    RL_CUDA_CHECK(cudaStreamWaitEvent(cs, top, 0));
    for (int d = D - 1; d >= 0; --d) {
        copy_h2d_2d(dA + sz[d + 1] * n, n, A + sz[d + 1] * lda, lda, sz[d] - sz[d + 1], n, cs);
        RL_CUDA_CHECK(cudaEventRecord(evw[d], cs));
        waits[{0, (i32)sz[d]}] = evw[d];
    }
    // right spine: node (lo[d], len[d]); its top half [lo, lo + len/2) goes back
    i64 lo[D], len[D], cut = 0;
    for (int d = 0; d < D; ++d) {
        lo[d] = d == 0 ? 0 : lo[d - 1] + len[d - 1] / 2;
        len[d] = d == 0 ? m : len[d - 1] - len[d - 1] / 2;
        dones[{(i32)lo[d], (i32)len[d]}] = evd[d];
    }
    const i64 kcap = std::min(m, n);
    rrp_h.assign((size_t)kcap, 0);
    ipiv_h.assign((size_t)kcap, 0);
    auto e = engine_for(m, n, n, p, s, true);
    e->set_host_overlap(waits, dones);
    e->run(dA, s, true);
    for (int d = 0; d < D; ++d) {
        RL_CUDA_CHECK(cudaStreamWaitEvent(cs2, evd[d], 0));
        copy_d2h_2d(A + lo[d] * lda, lda, dA + lo[d] * n, n, len[d] / 2, n, cs2);
        cut = lo[d] + len[d] / 2;
    }
    e->results(r, rrp_h.data(), ipiv_h.data(), s);  // synchronises s
    copy_d2h_2d(A + cut * lda, lda, dA + cut * n, n, m - cut, n, s);
    RL_CUDA_CHECK(cudaStreamSynchronize(cs2));
    bool ident = true;
    for (i64 j = 0; j < *r && ident; ++j) ident = ipiv_h[(size_t)j] == (u32)j && rrp_h[(size_t)j] == (u32)j;
    if (!ident) copy_d2h_2d(A, lda, dA, n, cut, n, s);
}

// The same for an engine with the tiled top level (cup.cu, CupEngine::tiled):
// tile 0 is copied first; every later tile crosses the link in order on a copy
// stream with its own event, which the launch sequence waits on right before it
// first touches those rows (the side lane of the tile's piece, or the critical
// path); each tile goes back as soon as it is factored (final unless a later
// transposition or U-row move reaches it: then everything is copied again).
bool host_graph() {
    static const bool v = [] {
        const char* e = getenv("RL_HOST_GRAPH");
        return !e || atoi(e) != 0;
    }();
    return v;
}

void cup_host_overlapped_tiles(u32* A, i64 m, i64 n, i64 lda, u32 p, u32* dA, Scratch& sc, cudaStream_t s,
                               i64* r, std::vector<u32>& rrp_h, std::vector<u32>& ipiv_h,
                               const std::shared_ptr<CupEngine>& e) {
    const i64 g = e->tile_rows();
    const i64 T = (m + g - 1) / g;
    cudaStream_t cs = sc.aux_stream(0), cs2 = sc.aux_stream(1);
    cudaEvent_t top = sc.event(2 * kRing);
    CupEngine::RowEvents in, out;
    copy_h2d_2d(dA, n, A, lda, std::min(g, m), n, s);
    RL_CUDA_CHECK(cudaEventRecord(top, s));
    RL_CUDA_CHECK(cudaStreamWaitEvent(cs, top, 0));
    for (i64 t = 1; t < T; ++t) {
        const i64 lo = t * g, hi = std::min(m, lo + g);
        copy_h2d_2d(dA + lo * n, n, A + lo * lda, lda, hi - lo, n, cs);
        cudaEvent_t ev = sc.event(2 * kRing + 1 + (int)t);
        RL_CUDA_CHECK(cudaEventRecord(ev, cs));
        in.push_back({{(i32)lo, (i32)hi}, ev});
    }
    for (i64 t = 0; t + 1 < T; ++t)
        out.push_back({{(i32)(t * g), (i32)std::min(m, t * g + g)}, sc.event(2 * kRing + 1 + (int)T + (int)t)});
    const i64 kcap = std::min(m, n);
    rrp_h.assign((size_t)kcap, 0);
    ipiv_h.assign((size_t)kcap, 0);
    e->set_host_rows(in, out);
    // (The tile lanes wait on late copy events: with the default 8 hardware
    // work queues a blocked lane stalls the streams sharing its queue, the
    // critical path among them -- runtime.cu raises CUDA_DEVICE_MAX_CONNECTIONS
    // to 32 before the context exists: C3 e2e 40.6 -> 27.4 ms.)
    e->run(dA, s, host_graph());
    for (const auto& o : out) {
        RL_CUDA_CHECK(cudaStreamWaitEvent(cs2, o.second, 0));
        copy_d2h_2d(A + (i64)o.first.first * lda, lda, dA + (i64)o.first.first * n, n,
                    o.first.second - o.first.first, n, cs2);
    }
    const i64 cut = (T - 1) * g;
    e->results(r, rrp_h.data(), ipiv_h.data(), s);  // synchronises s
    copy_d2h_2d(A + cut * lda, lda, dA + cut * n, n, m - cut, n, s);
    RL_CUDA_CHECK(cudaStreamSynchronize(cs2));
    bool ident = true;
    for (i64 j = 0; j < *r && ident; ++j) ident = ipiv_h[(size_t)j] == (u32)j && rrp_h[(size_t)j] == (u32)j;
    if (!ident) copy_d2h_2d(A, lda, dA, n, cut, n, s);
}

// Pageable host buffers (a std::vector-backed ranklab::Mat, matrix.hpp:176) with a
// tiled engine: the tile pipeline of cup_host_overlapped_tiles, staged through two
// pinned rings of kPgSlots tiles.  Every copy is enqueued BEFORE the launch
// sequence (so its events are recorded before the graph waits on them); a copy
// stream holds each DMA back with a stream-memory wait on a mapped host word
// until the host threads have filled (in) or drained (out) the slot.  The host
// then fills tile t + 1 while tile t crosses the link and the factorization runs.
constexpr int kPgSlots = 3;

// cuStreamWaitValue32 through the runtime's driver entry-point lookup: no link
// dependency on libcuda, so the library still loads on a machine without a
// driver (where every compute entry fails with RL_ECUDA instead).
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn() {
    static WaitValueFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<WaitValueFn>(p);
    }();
    if (!fn) throw Error(RL_ECUDA, "cuStreamWaitValue32 unavailable");
    return fn;
}

void cup_host_pageable_tiles(u32* A, i64 m, i64 n, i64 lda, u32 p, u32* dA, Scratch& sc, cudaStream_t s,
                             i64* r, std::vector<u32>& rrp_h, std::vector<u32>& ipiv_h,
                             const std::shared_ptr<CupEngine>& e) {
    const i64 g = e->tile_rows();
    const i64 T = (m + g - 1) / g;
    const size_t slot = (size_t)g * n;  // words
    u32* ring_in = (u32*)sc.pinned_ring(kPgSlots * slot * 4);
    u32* ring_out = (u32*)sc.pinned_ring_out(kPgSlots * slot * 4);
    volatile unsigned* flags = sc.flags();  // [0]: tiles staged, [1]: tiles drained
    CUdeviceptr f_in = 0, f_out = 0;
    {
        void* dp = nullptr;
        RL_CUDA_CHECK(cudaHostGetDevicePointer(&dp, (void*)flags, 0));
        f_in = (CUdeviceptr)dp;
        f_out = f_in + sizeof(unsigned);
    }
    cudaStream_t cs = sc.aux_stream(0), cs2 = sc.aux_stream(1);
    auto rows_of = [&](i64 t) { return std::min(g, m - t * g); };
    // tile 0 first, synchronously staged
    par_copy_rows(ring_in, n, A, lda, rows_of(0), n);
    copy_h2d_2d(dA, n, ring_in, n, rows_of(0), n, s);
    cudaEvent_t top = sc.event(2 * kRing);
    RL_CUDA_CHECK(cudaEventRecord(top, s));
    RL_CUDA_CHECK(cudaStreamWaitEvent(cs, top, 0));
    CupEngine::RowEvents in, out;
    std::vector<cudaEvent_t> ev_in(T, nullptr), ev_d2h(T, nullptr);
    for (i64 t = 1; t < T; ++t) {
        auto st = wait_value_fn()((CUstream)cs, f_in, (cuuint32_t)t, CU_STREAM_WAIT_VALUE_GEQ);
        if (st != CUDA_SUCCESS) throw Error(RL_ECUDA, "cuStreamWaitValue32 failed");
        copy_h2d_2d(dA + t * g * n, n, ring_in + (size_t)(t % kPgSlots) * slot, n, rows_of(t), n, cs);
        ev_in[t] = sc.event(2 * kRing + 1 + (int)t);
        RL_CUDA_CHECK(cudaEventRecord(ev_in[t], cs));
        in.push_back({{(i32)(t * g), (i32)(t * g + rows_of(t))}, ev_in[t]});
    }
    for (i64 t = 0; t + 1 < T; ++t)
        out.push_back({{(i32)(t * g), (i32)(t * g + rows_of(t))}, sc.event(2 * kRing + 1 + (int)T + (int)t)});
    const i64 kcap = std::min(m, n);
    rrp_h.assign((size_t)kcap, 0);
    ipiv_h.assign((size_t)kcap, 0);
    e->set_host_rows(in, out);
    e->run(dA, s, host_graph());
    // device -> host, enqueued after the launch sequence that records the events
    for (i64 t = 0; t + 1 < T; ++t) {
        RL_CUDA_CHECK(cudaStreamWaitEvent(cs2, out[(size_t)t].second, 0));
        if (t >= kPgSlots) {  // the slot's previous tile drained by the host
            auto st = wait_value_fn()((CUstream)cs2, f_out, (cuuint32_t)(t - kPgSlots + 1),
                                      CU_STREAM_WAIT_VALUE_GEQ);
            if (st != CUDA_SUCCESS) throw Error(RL_ECUDA, "cuStreamWaitValue32 failed");
        }
        copy_d2h_2d(ring_out + (size_t)(t % kPgSlots) * slot, n, dA + t * g * n, n, rows_of(t), n, cs2);
        ev_d2h[t] = sc.event(2 * kRing + 1 + 2 * (int)T + (int)t);
        RL_CUDA_CHECK(cudaEventRecord(ev_d2h[t], cs2));
    }
    // host side: fill the in-ring ahead of the DMA, drain the out-ring behind it
    i64 t_in = 1, t_out = 0;
    while (t_in < T || t_out + 1 < T) {
        bool progressed = false;
        // slot t % kPgSlots last held tile t - kPgSlots: its DMA must be done
        auto slot_free = [&](i64 t) {
            if (t < kPgSlots) return true;
            const i64 prev = t - kPgSlots;
            return cudaEventQuery(prev == 0 ? top : ev_in[prev]) == cudaSuccess;
        };
        if (t_in < T && slot_free(t_in)) {
            par_copy_rows(ring_in + (size_t)(t_in % kPgSlots) * slot, n, A + t_in * g * lda, lda, rows_of(t_in), n);
            std::atomic_thread_fence(std::memory_order_seq_cst);
            flags[0] = (unsigned)t_in;
            ++t_in;
            progressed = true;
        }
        if (t_out + 1 < T && cudaEventQuery(ev_d2h[t_out]) == cudaSuccess) {
            par_copy_rows(A + t_out * g * lda, lda, ring_out + (size_t)(t_out % kPgSlots) * slot, n, rows_of(t_out),
                          n);
            std::atomic_thread_fence(std::memory_order_seq_cst);
            flags[1] = (unsigned)(t_out + 1);
            ++t_out;
            progressed = true;
        }
        if (!progressed) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    e->results(r, rrp_h.data(), ipiv_h.data(), s);  // synchronises s
    const i64 cut = (T - 1) * g;
    staged_d2h(A + cut * lda, lda, dA + cut * n, n, m - cut, n, sc, s);
    bool ident = true;
    for (i64 j = 0; j < *r && ident; ++j) ident = ipiv_h[(size_t)j] == (u32)j && rrp_h[(size_t)j] == (u32)j;
    if (!ident) staged_d2h(A, lda, dA, n, cut, n, sc, s);
}

// ple (factor.cpp:87-156) is cup's column-split mirror: the recursion splits
// columns at k = n/2 where cup splits rows at m/2, the base case searches a
// column where cup searches a row, L is normalised where U is, E keeps raw
// pivots where C does, and the L-column move mirrors the U-row shift.  So
// ple(A) = cup(A^T)^T exactly -- body, col_profile = cup's row profile, row_perm =
// the inverse of cup's column permutation, and the same charges (trsm(Left,Lower,Unit) and
// trsm(Right,Upper,Unit) charge alike, mm is symmetric).  The device path
// transposes into a workspace, factors, and transposes back (lock held).
void ple_on_device(u32* dA, i64 m, i64 n, i64 lda, u32 p, cudaStream_t s, i64* rank, u32* col_profile,
                   u32* row_perm, u64* ops) {
    u32* dT = (u32*)scratch_for(s).get(SS_TRANS, (size_t)m * n * 4);
    transpose(dT, m, dA, lda, m, n, s);
    i64 r = 0;
    std::vector<u32> rrp_h, ipiv_h;
    factor_on_device(dT, n, m, m, p, s, &r, rrp_h, ipiv_h);
    transpose(dA, lda, dT, m, n, m, s);
    RL_CUDA_CHECK(cudaStreamSynchronize(s));
    if (rank) *rank = r;
    if (col_profile) std::copy(rrp_h.begin(), rrp_h.begin() + r, col_profile);
    if (row_perm) {  // A^T = E^T L^T P^T: cup's column permutation is P^T
        std::vector<u32> sig((size_t)m);
        sigma_from_ipiv(m, r, ipiv_h.data(), sig.data());
        for (i64 i = 0; i < m; ++i) row_perm[sig[i]] = (u32)i;
    }
    if (ops) cup_opcount(n, m, r, rrp_h.data(), ipiv_h.data(), ops);
}

// ple's degenerate return (factor.cpp:110): rank 0, identity of order m.
void ple_empty(i64 m, i64* rank, u32* row_perm, u64* ops) {
    if (rank) *rank = 0;
    if (row_perm) for (i64 i = 0; i < m; ++i) row_perm[i] = (u32)i;
    if (ops) std::fill(ops, ops + 4, 0ull);
}

// The reductions after cup on a device matrix (echelon.cpp:5-47): body
// [C\U] -> [C\X] (col_ech_trans) or [[X1, X2], [R2, 0]] (reduced).
void echelon_after_cup(u32* dA, i64 m, i64 n, i64 lda, u32 p, i64 r, const u32* rrp_h,
                       bool reduced, cudaStream_t s) {
    if (r == 0) return;
    const Fp f = make_fp(p);
    Scratch& sc = scratch_for(s);
    DevBuf &xbuf = sc.buf[SS_X], &ybuf = sc.buf[SS_Y], &tbuf = sc.buf[SS_T], &ibuf = sc.buf[SS_IDX];
    // X <- U1^{-1} (unit upper); X2 <- -U1^{-1} U2; strict triangle of U1 <- X's
    u32* X = (u32*)xbuf.get((size_t)r * r * 4);
    tri_extract(X, r, dA, lda, (i32)r, /*upper=*/true, /*unit=*/true, p, s);
    tri_inverse(X, r, (i32)r, /*upper=*/true, f, s);
    if (n > r) {
        u32* T = (u32*)tbuf.get((size_t)r * (n - r) * 4);
        mm_dense(X, r, dA + r, lda, T, n - r, r, r, n - r, p - 1, 0, f, s);
        RL_CUDA_CHECK(cudaMemcpy2DAsync(dA + r, lda * 4, T, (n - r) * 4, (n - r) * 4, r,
                                        cudaMemcpyDeviceToDevice, s));
    }
    tri_store_strict(dA, lda, X, r, (i32)r, /*upper=*/true, s);
    if (!reduced) return;
    // pivot rows of C onto the diagonal, then R2 <- L2 L1^{-1}, X1 <- U1^{-1} L1^{-1}
    i32* d_rrp = (i32*)ibuf.get((size_t)r * 4);
    RL_CUDA_CHECK(cudaMemcpyAsync(d_rrp, rrp_h, (size_t)r * 4, cudaMemcpyHostToDevice, s));
    compress_pivot_rows(dA, lda, (i32)r, d_rrp, s);
    u32* Y = (u32*)ybuf.get((size_t)r * r * 4);
    tri_extract(Y, r, dA, lda, (i32)r, /*upper=*/false, /*unit=*/false, p, s);
    tri_inverse(Y, r, (i32)r, /*upper=*/false, f, s);
    if (m > r) {
        u32* T = (u32*)tbuf.get((size_t)(m - r) * r * 4);
        mm_dense(dA + r * lda, lda, Y, r, T, r, m - r, r, r, 1 % p, 0, f, s);
        RL_CUDA_CHECK(cudaMemcpy2DAsync(dA + r * lda, lda * 4, T, r * 4, r * 4, m - r,
                                        cudaMemcpyDeviceToDevice, s));
    }
    mm_dense(X, r, Y, r, dA, lda, r, r, r, 1 % p, 0, f, s);
}

// new row i <- old row sigma^{-1}(i): A^{-1} = P^T X (solvers.cpp:29-30).
void rows_by_inverse_perm(u32* dA, i64 n, i64 lda, const u32* sigma, cudaStream_t s) {
    std::vector<i32> idx;
    for (i64 j = 0; j < n; ++j)
        if ((i64)sigma[j] != j) {  // new row sigma[j] <- old row j
            idx.push_back((i32)sigma[j]);
            idx.push_back((i32)j);
        }
    if (idx.empty()) return;
    i32* d = (i32*)scratch_for(s).get(SS_PERM, idx.size() * 4);
    RL_CUDA_CHECK(cudaMemcpyAsync(d, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, s));
    move_rows(dA, lda, n, d, (i32)(idx.size() / 2), s);
    RL_CUDA_CHECK(cudaStreamSynchronize(s));  // idx must outlive the copy
}

void col_ech_dev_impl(u32* dA, i64 m, i64 n, i64 lda, u32 p, bool reduced, i64* rank, u32* rrp,
                      u32* sigma, u64* ops, cudaStream_t s) {
    i64 r = 0;
    std::vector<u32> rrp_h, ipiv_h;
    factor_on_device(dA, m, n, lda, p, s, &r, rrp_h, ipiv_h);
    echelon_after_cup(dA, m, n, lda, p, r, rrp_h.data(), reduced, s);
    if (rank) *rank = r;
    if (rrp) std::copy(rrp_h.begin(), rrp_h.begin() + r, rrp);
    if (sigma) sigma_from_ipiv(n, r, ipiv_h.data(), sigma);
    if (ops) {
        cup_opcount(m, n, r, rrp_h.data(), ipiv_h.data(), ops);
        OpTally t;
        tally_echelon(t, m, n, r, reduced);
        ops[0] += t.mul;
        ops[1] += t.addsub;
        ops[2] += t.divinv;
        ops[3] += t.ztest;
    }
}

// trsm seam (kernels.hpp:37-38): B <- T^{-1} B (left) or B T^{-1} (right), via
// the dense inverse of the triangle and one GEMM.
void trsm_dev_impl(int side, int uplo, int diag, const u32* dT, i64 ldt, u32* dB, i64 ldb, i64 m,
                   i64 n, u32 p, cudaStream_t s) {
    const i64 k = side == SIDE_LEFT ? m : n;
    if (k == 0 || m == 0 || n == 0) return;
    const Fp f = make_fp(p);
    Scratch& sc = scratch_for(s);
    u32* X = (u32*)sc.get(SS_X, (size_t)k * k * 4);
    const bool upper = uplo == UPLO_UPPER;
    tri_extract(X, k, dT, ldt, (i32)k, upper, diag != 0, p, s);
    tri_inverse(X, k, (i32)k, upper, f, s);
    u32* T = (u32*)sc.get(SS_T, (size_t)m * n * 4);
    if (side == SIDE_LEFT) mm_dense(X, k, dB, ldb, T, n, m, k, n, 1 % p, 0, f, s);
    else mm_dense(dB, ldb, X, k, T, n, m, k, n, 1 % p, 0, f, s);
    RL_CUDA_CHECK(cudaMemcpy2DAsync(dB, ldb * 4, T, n * 4, n * 4, m, cudaMemcpyDeviceToDevice, s));
}

// The reference raises SingularDiagonal(d) at the first zero pivot its
// traversal meets (kernels.cpp:87-90): trsm_rec halves the triangle (k = n/2)
// down to blocks of <= threshold and visits them in ascending order for
// Right/Upper and Left/Lower, descending for the other two, each block's
// diagonal in the same direction -- and d is the index LOCAL to the base block
// (trsm_base sees only its sub-view).  Returns -1 when the diagonal has no zero.
i64 first_zero_diagonal(int side, int uplo, const std::vector<u32>& diag, i64 threshold) {
    const bool ascending = (side == SIDE_RIGHT) == (uplo == UPLO_UPPER);
    const i64 th = threshold < 1 ? 1 : threshold;
    std::function<i64(i64, i64)> rec = [&](i64 off, i64 n) -> i64 {
        if (n == 0) return -1;
        if (n <= th) {
            for (i64 t = 0; t < n; ++t) {
                const i64 d = ascending ? t : n - 1 - t;
                if (diag[(size_t)(off + d)] == 0) return d;
            }
            return -1;
        }
        const i64 k = n / 2;
        const i64 first = ascending ? rec(off, k) : rec(off + k, n - k);
        if (first >= 0) return first;
        return ascending ? rec(off + k, n - k) : rec(off, k);
    };
    return rec(0, (i64)diag.size());
}

void check_trsm_args(int side, int uplo, int diag, i64 m, i64 n, i64 ldt, i64 ldb) {
    if (side < 0 || side > 1 || uplo < 0 || uplo > 1 || diag < 0 || diag > 1)
        throw Error(RL_EINVAL, "trsm: side/uplo/diag out of range");
    if (m < 0 || n < 0) throw Error(RL_EDIM, "negative dimension");
    const i64 k = side == SIDE_LEFT ? m : n;
    if (k > 0 && ldt < k) throw Error(RL_EINVAL, "trsm: ldt smaller than the triangle");
    if (n > 0 && ldb < n) throw Error(RL_EINVAL, "trsm: ldb smaller than the column count");
}

void trsm_ops(int side, int uplo, int diag, i64 m, i64 n, i64 threshold, u64* ops) {
    if (!ops) return;
    OpTally t;
    tally_trsm(t, side, uplo, diag != 0, side == SIDE_LEFT ? m : n, m, n, threshold);
    ops[0] = t.mul;
    ops[1] = t.addsub;
    ops[2] = t.divinv;
    ops[3] = t.ztest;
}

// invert_in_place (solvers.cpp:24-31) on a device matrix.
void invert_dev_impl(u32* dA, i64 n, i64 lda, u32 p, u64* ops, cudaStream_t s) {
    i64 r = 0;
    std::vector<u32> sigma((size_t)n);
    col_ech_dev_impl(dA, n, n, lda, p, /*reduced=*/true, &r, nullptr, sigma.data(), ops, s);
    if (r < n) throw Error(RL_ESINGULAR, "singular matrix");  // body = red_col_ech_trans's
    rows_by_inverse_perm(dA, n, lda, sigma.data(), s);
}
}  // namespace

extern "C" {

int rl_version(void) { return 100; }

const char* rl_last_error(void) { return g_last_error.c_str(); }

int rl_cup_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* rank,
                   uint32_t* rrp, uint32_t* sigma, uint64_t* ops, void* stream) {
    return guard([&] {
        if (!dA && m * n > 0) throw Error(RL_EINVAL, "null matrix");
        cup_dev_impl(dA, m, n, lda, p, rank, rrp, sigma, ops, (cudaStream_t)stream);
    });
}

int rl_cup_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* rank,
               uint32_t* rrp, uint32_t* sigma, uint64_t* ops) {
    return guard([&] {
        if (!A && m * n > 0) throw Error(RL_EINVAL, "null matrix");
        check_field(p);
        check_dims(m, n, lda);
        if (m == 0 || n == 0) {
            cup_dev_impl(nullptr, m, n, lda, p, rank, rrp, sigma, ops, nullptr);
            return;
        }
        require_device();
        cudaStream_t s = host_stream();
        Call call(s);
        Scratch& sc = call.sc;
        i64 r = 0;
        std::vector<u32> rrp_h, ipiv_h;
        if (m * n <= TINY_MAX) {
            tiny_cup(A, m, n, lda, p, sc, s, &r, rrp_h, ipiv_h);
        } else {
            u32* dA = (u32*)sc.get(SS_A, (size_t)m * n * 4);
            std::shared_ptr<CupEngine> te;
            const bool pageable = !host_pinned(A) && !pageable_direct();
            if (pageable && m * n >= (1 << 22) && (te = engine_for(m, n, n, p, s, true))->tile_rows() > 0 &&
                (m + te->tile_rows() - 1) / te->tile_rows() <= 24) {
                cup_host_pageable_tiles(A, m, n, lda, p, dA, sc, s, &r, rrp_h, ipiv_h, te);
            } else if (pageable) {
                // pageable storage (ranklab::Mat is a std::vector, matrix.hpp:176): staged
                // through the context's pinned ring by host threads, chunk by chunk
                staged_h2d(dA, n, A, lda, m, n, sc, s);
                factor_on_device(dA, m, n, n, p, s, &r, rrp_h, ipiv_h);
                staged_d2h(A, lda, dA, n, m, n, sc, s);
            } else if (m * n >= (1 << 22) && m >= 8 * PB) {
                cup_host_overlapped(A, m, n, lda, p, dA, sc, s, &r, rrp_h, ipiv_h);
            } else {
                copy_h2d_2d(dA, n, A, lda, m, n, s);
                factor_on_device(dA, m, n, n, p, s, &r, rrp_h, ipiv_h);
                copy_d2h_2d(A, lda, dA, n, m, n, s);
            }
            RL_CUDA_CHECK(cudaStreamSynchronize(s));
        }
        if (rank) *rank = r;
        if (rrp) std::copy(rrp_h.begin(), rrp_h.begin() + r, rrp);
        if (sigma) sigma_from_ipiv(n, r, ipiv_h.data(), sigma);
        if (ops) cup_opcount(m, n, r, rrp_h.data(), ipiv_h.data(), ops);
    });
}

int rl_ple_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* rank,
                   uint32_t* col_profile, uint32_t* row_perm, uint64_t* ops, void* stream) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, lda);
        if (m == 0 || n == 0) return ple_empty(m, rank, row_perm, ops);
        if (!dA) throw Error(RL_EINVAL, "null matrix");
        require_device();
        Call call((cudaStream_t)stream);
        ple_on_device(dA, m, n, lda, p, (cudaStream_t)stream, rank, col_profile, row_perm, ops);
    });
}

int rl_ple_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* rank,
               uint32_t* col_profile, uint32_t* row_perm, uint64_t* ops) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, lda);
        if (m == 0 || n == 0) return ple_empty(m, rank, row_perm, ops);
        if (!A) throw Error(RL_EINVAL, "null matrix");
        require_device();
        cudaStream_t s = host_stream();
        Call call(s);
        u32* dA = (u32*)call.sc.get(SS_A, (size_t)m * n * 4);
        copy_h2d_2d(dA, n, A, lda, m, n, s);
        ple_on_device(dA, m, n, n, p, s, rank, col_profile, row_perm, ops);
        copy_d2h_2d(A, lda, dA, n, m, n, s);
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int rl_col_ech_trans_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint32_t p,
                             int reduced, int64_t* rank, uint32_t* rrp, uint32_t* sigma,
                             uint64_t* ops, void* stream) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, lda);
        if (m == 0 || n == 0) {  // cup's degenerate return; nothing to reduce
            cup_dev_impl(nullptr, m, n, lda, p, rank, rrp, sigma, ops, nullptr);
            return;
        }
        if (!dA) throw Error(RL_EINVAL, "null matrix");
        require_device();
        Call call((cudaStream_t)stream);
        col_ech_dev_impl(dA, m, n, lda, p, reduced != 0, rank, rrp, sigma, ops, (cudaStream_t)stream);
    });
}

int rl_col_ech_trans_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p, int reduced,
                         int64_t* rank, uint32_t* rrp, uint32_t* sigma, uint64_t* ops) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, lda);
        if (m == 0 || n == 0) {
            cup_dev_impl(nullptr, m, n, lda, p, rank, rrp, sigma, ops, nullptr);
            return;
        }
        if (!A) throw Error(RL_EINVAL, "null matrix");
        require_device();
        cudaStream_t s = host_stream();
        Call call(s);
        u32* dA = (u32*)call.sc.get(SS_A, (size_t)m * n * 4);
        copy_h2d_2d(dA, n, A, lda, m, n, s);
        col_ech_dev_impl(dA, m, n, n, p, reduced != 0, rank, rrp, sigma, ops, s);
        copy_d2h_2d(A, lda, dA, n, m, n, s);
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int rl_invert_u32_dev(uint32_t* dA, int64_t n, int64_t lda, uint32_t p, uint64_t* ops,
                      void* stream) {
    return guard([&] {
        check_field(p);
        check_dims(n, n, lda);
        if (ops) std::fill(ops, ops + 4, 0ull);
        if (n == 0) return;
        if (!dA) throw Error(RL_EINVAL, "null matrix");
        require_device();
        Call call((cudaStream_t)stream);
        invert_dev_impl(dA, n, lda, p, ops, (cudaStream_t)stream);
    });
}

int rl_invert_u32(uint32_t* A, int64_t n, int64_t lda, uint32_t p, uint64_t* ops) {
    return guard([&] {
        check_field(p);
        check_dims(n, n, lda);
        if (ops) std::fill(ops, ops + 4, 0ull);
        if (n == 0) return;
        if (!A) throw Error(RL_EINVAL, "null matrix");
        require_device();
        cudaStream_t s = host_stream();
        Call call(s);
        u32* dA = (u32*)call.sc.get(SS_A, (size_t)n * n * 4);
        copy_h2d_2d(dA, n, A, lda, n, n, s);
        int st = RL_OK;
        try {
            invert_dev_impl(dA, n, n, p, ops, s);
        } catch (const Error& e) {
            if (e.code != RL_ESINGULAR) throw;
            st = RL_ESINGULAR;  // the body still holds the reduced transform (as the reference)
        }
        copy_d2h_2d(A, lda, dA, n, n, n, s);
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
        if (st != RL_OK) throw Error(st, "singular matrix");
    });
}

int rl_trsm_u32_dev(int side, int uplo, int diag, const uint32_t* dT, int64_t ldt, uint32_t* dB,
                    int64_t ldb, int64_t m, int64_t n, uint32_t p, int64_t threshold, uint64_t* ops,
                    void* stream) {
    return guard([&] {
        check_field(p);
        check_trsm_args(side, uplo, diag, m, n, ldt, ldb);
        const i64 k = side == SIDE_LEFT ? m : n;
        if (m == 0 || n == 0) {
            if (ops) std::fill(ops, ops + 4, 0ull);
            return;
        }
        require_device();
        cudaStream_t s = (cudaStream_t)stream;
        Call call(s);
        if (!diag) {
            std::vector<u32> dg((size_t)k);
            RL_CUDA_CHECK(cudaMemcpy2DAsync(dg.data(), 4, dT, (ldt + 1) * 4, 4, k,
                                            cudaMemcpyDeviceToHost, s));
            RL_CUDA_CHECK(cudaStreamSynchronize(s));
            const i64 d = first_zero_diagonal(side, uplo, dg, threshold);
            if (d >= 0) throw Error(RL_ESINGULAR, "singular diagonal at " + std::to_string(d));
        }
        trsm_ops(side, uplo, diag, m, n, threshold, ops);
        trsm_dev_impl(side, uplo, diag, dT, ldt, dB, ldb, m, n, p, s);
    });
}

int rl_trsm_u32(int side, int uplo, int diag, const uint32_t* T, int64_t ldt, uint32_t* B,
                int64_t ldb, int64_t m, int64_t n, uint32_t p, int64_t threshold, uint64_t* ops) {
    return guard([&] {
        check_field(p);
        check_trsm_args(side, uplo, diag, m, n, ldt, ldb);
        const i64 k = side == SIDE_LEFT ? m : n;
        if (windows_overlap(T, k, k, ldt, B, m, n, ldb)) throw Error(RL_EOVERLAP, "trsm: T overlaps B");
        if (m == 0 || n == 0) {
            if (ops) std::fill(ops, ops + 4, 0ull);
            return;
        }
        if (!diag) {
            std::vector<u32> dg((size_t)k);
            for (i64 d = 0; d < k; ++d) dg[d] = T[d * ldt + d];
            const i64 d = first_zero_diagonal(side, uplo, dg, threshold);
            if (d >= 0) throw Error(RL_ESINGULAR, "singular diagonal at " + std::to_string(d));
        }
        trsm_ops(side, uplo, diag, m, n, threshold, ops);
        require_device();
        cudaStream_t s = host_stream();
        Call call(s);
        u32* dT = (u32*)call.sc.get(SS_A, (size_t)k * k * 4);
        u32* dB = (u32*)call.sc.get(SS_B, (size_t)m * n * 4);
        copy_h2d_2d(dT, k, T, ldt, k, k, s);
        copy_h2d_2d(dB, n, B, ldb, m, n, s);
        trsm_dev_impl(side, uplo, diag, dT, k, dB, n, m, n, p, s);
        copy_d2h_2d(B, ldb, dB, n, m, n, s);
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int rl_trsm_opcount(int side, int uplo, int diag, int64_t m, int64_t n, int64_t threshold,
                    uint64_t* ops) {
    return guard([&] {
        check_trsm_args(side, uplo, diag, m, n, side == SIDE_LEFT ? m : n, n);
        if (!ops) throw Error(RL_EINVAL, "null ops");
        trsm_ops(side, uplo, diag, m, n, threshold, ops);
    });
}

int rl_echelon_opcount(int64_t m, int64_t n, int64_t r, int reduced, uint64_t* ops) {
    return guard([&] {
        if (!ops) throw Error(RL_EINVAL, "null ops");
        if (m < 0 || n < 0 || r < 0 || r > std::min(m, n)) throw Error(RL_EDIM, "bad shape/rank");
        OpTally t;
        tally_echelon(t, m, n, r, reduced != 0);
        ops[0] = t.mul;
        ops[1] = t.addsub;
        ops[2] = t.divinv;
        ops[3] = t.ztest;
    });
}

int rl_rank_and_profile_u32(uint32_t* A, int64_t m, int64_t n, int64_t lda, uint32_t p,
                            int64_t* rank, uint32_t* rrp) {
    return rl_cup_u32(A, m, n, lda, p, rank, rrp, nullptr, nullptr);
}

int rl_determinant_u32(uint32_t* A, int64_t n, int64_t lda, uint32_t p, uint32_t* det) {
    return guard([&] {
        check_field(p);
        check_dims(n, n, lda);
        if (!det) throw Error(RL_EINVAL, "null det");
        std::vector<u32> sigma((size_t)n);
        i64 r = 0;
        int st = rl_cup_u32(A, n, n, lda, p, &r, nullptr, sigma.data(), nullptr);
        if (st != RL_OK) throw Error(st, g_last_error);
        if (r < n) {
            *det = 0;
            return;
        }
        if (n == 0) {
            *det = 1 % p;
            return;
        }
        u64 d = A[0];
        for (i64 j = 1; j < n; ++j) d = d * A[j * lda + j] % p;  // solvers.cpp:18-19
        // sign of sigma by cycle decomposition (perm.cpp:50-63)
        std::vector<uint8_t> seen((size_t)n, 0);
        i64 transp = 0;
        for (i64 s0 = 0; s0 < n; ++s0) {
            if (seen[s0]) continue;
            i64 len = 0;
            for (i64 j = s0; !seen[j]; j = sigma[j]) {
                seen[j] = 1;
                ++len;
            }
            transp += len - 1;
        }
        if (transp % 2) d = d == 0 ? 0 : p - d;
        *det = (u32)d;
    });
}

int rl_mm_u32_dev(const uint32_t* dA, int64_t lda, const uint32_t* dB, int64_t ldb, uint32_t* dC,
                  int64_t ldc, int64_t m, int64_t l, int64_t n, uint32_t alpha, uint32_t beta,
                  uint32_t p, void* stream) {
    return guard([&] {
        check_field(p);
        if (m < 0 || l < 0 || n < 0) throw Error(RL_EDIM, "negative dimension");
        if (alpha >= p || beta >= p) throw Error(RL_EINVAL, "alpha/beta not canonical");
        require_device();
        Call call((cudaStream_t)stream);
        mm_dev_impl(dA, lda, dB, ldb, dC, ldc, m, l, n, alpha, beta, p, (cudaStream_t)stream);
    });
}

int rl_mm_u32_dev_grid(const uint32_t* dA, int64_t lda, const uint32_t* dB, int64_t ldb,
                       uint32_t* dC, int64_t ldc, int64_t m, int64_t l, int64_t n, uint32_t alpha,
                       uint32_t beta, uint32_t p, int max_ctas, void* stream) {
    return guard([&] {
        check_field(p);
        if (m < 0 || l < 0 || n < 0) throw Error(RL_EDIM, "negative dimension");
        if (alpha >= p || beta >= p) throw Error(RL_EINVAL, "alpha/beta not canonical");
        if (max_ctas < 0) throw Error(RL_EINVAL, "negative grid bound");
        require_device();
        Call call((cudaStream_t)stream);
        mm_dev_impl(dA, lda, dB, ldb, dC, ldc, m, l, n, alpha, beta, p, (cudaStream_t)stream,
                    max_ctas);
    });
}

int rl_mm_u32(const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t* C,
              int64_t ldc, int64_t m, int64_t l, int64_t n, uint32_t alpha, uint32_t beta,
              uint32_t p, uint64_t* ops) {
    return guard([&] {
        check_field(p);
        if (m < 0 || l < 0 || n < 0) throw Error(RL_EDIM, "negative dimension");
        if (alpha >= p || beta >= p) throw Error(RL_EINVAL, "alpha/beta not canonical");
        if (windows_overlap(A, m, l, lda, C, m, n, ldc)) throw Error(RL_EOVERLAP, "mm: C overlaps A");
        if (windows_overlap(B, l, n, ldb, C, m, n, ldc)) throw Error(RL_EOVERLAP, "mm: C overlaps B");
        if (ops) {  // exact charges of kernels.cpp:41-74
            std::fill(ops, ops + 4, 0ull);
            const u64 e = (u64)m * (u64)n;
            const u32 one = 1 % p, neg = p - 1;
            if (alpha == 0 || l == 0) {
                if (beta != 0 && beta != one) ops[0] += e;
            } else {
                ops[0] += e * (u64)l;
                ops[1] += e * (u64)(l - 1);
                if (alpha != one && alpha != neg) ops[0] += e;
                if (beta == 0) {
                    if (alpha == neg && alpha != one) ops[1] += e;
                } else if (beta == one) {
                    ops[1] += e;
                } else {
                    ops[0] += e;
                    ops[1] += e;
                }
            }
        }
        if (m == 0 || n == 0) return;
        require_device();
        cudaStream_t s = host_stream();
        Call call(s);
        u32* dA = (u32*)call.sc.get(SS_A, (size_t)std::max<i64>(m * l, 1) * 4);
        u32* dB = (u32*)call.sc.get(SS_B, (size_t)std::max<i64>(l * n, 1) * 4);
        u32* dC = (u32*)call.sc.get(SS_C, (size_t)m * n * 4);
        copy_h2d_2d(dA, l, A, lda, m, l, s);
        copy_h2d_2d(dB, n, B, ldb, l, n, s);
        copy_h2d_2d(dC, n, C, ldc, m, n, s);
        mm_dev_impl(dA, l, dB, n, dC, n, m, l, n, alpha, beta, p, s);
        copy_d2h_2d(C, ldc, dC, n, m, n, s);
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
    });
}

int rl_random_matrix_u32_dev(uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint64_t seed,
                             uint32_t p, void* stream) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, lda);
        require_device();
        gen_random_matrix(dA, lda, m, n, seed, p, (cudaStream_t)stream);
    });
}

int rl_digest_u32_dev(const uint32_t* dA, int64_t m, int64_t n, int64_t lda, uint64_t* digest,
                      void* stream) {
    return guard([&] {
        check_dims(m, n, lda);
        if (!digest) throw Error(RL_EINVAL, "null digest");
        *digest = 0;
        if (m == 0 || n == 0) return;
        if (!dA) throw Error(RL_EINVAL, "null matrix");
        require_device();
        cudaStream_t s = (cudaStream_t)stream;
        Call call(s);
        auto* d = (unsigned long long*)call.sc.get(SS_DIGEST, sizeof(unsigned long long));
        digest_u32(dA, lda, m, n, d, s);
        unsigned long long h = 0;
        RL_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s));
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
        *digest = h;
    });
}

int rl_dist_pack_u32_dev(const uint32_t* src, int64_t lds, int64_t rows, int64_t cols, int wire16, void* dst,
                         void* stream) {
    return guard([&] {
        if (rows < 0 || cols < 0 || lds < cols) throw Error(RL_EDIM, "bad piece shape");
        if (rows > 0 && cols > 0 && (!src || !dst)) throw Error(RL_EINVAL, "null buffer");
        require_device();
        dist_pack(src, lds, rows, cols, wire16, dst, (cudaStream_t)stream);
    });
}
int rl_dist_unpack_u32_dev(const void* src, int64_t rows, int64_t cols, int wire16, uint32_t* dst, int64_t ldd,
                           const int64_t* colmap, int64_t off, void* stream) {
    return guard([&] {
        if (rows < 0 || cols < 0 || (!colmap && ldd < cols)) throw Error(RL_EDIM, "bad piece shape");
        if (rows > 0 && cols > 0 && (!src || !dst)) throw Error(RL_EINVAL, "null buffer");
        require_device();
        dist_unpack(src, rows, cols, wire16, dst, ldd, colmap, off, (cudaStream_t)stream);
    });
}
int rl_dist_select_cols_u32_dev(const uint32_t* src, int64_t lds, int64_t rows, const int64_t* colmap,
                                int64_t off, int64_t cols, uint32_t* dst, int64_t ldd, void* stream) {
    return guard([&] {
        if (rows < 0 || cols < 0 || ldd < cols) throw Error(RL_EDIM, "bad piece shape");
        if (rows > 0 && cols > 0 && (!src || !dst || !colmap)) throw Error(RL_EINVAL, "null buffer");
        require_device();
        dist_select(src, lds, rows, colmap, off, cols, dst, ldd, (cudaStream_t)stream);
    });
}
int rl_dist_shift_u_rows_dev(uint32_t* x, int64_t ldx, int64_t cols, int64_t r, int64_t i0, int64_t rt,
                             const int64_t* gpos, void* stream) {
    return guard([&] {
        if (cols < 0 || rt < 0 || r < 0 || i0 < r || ldx < cols) throw Error(RL_EDIM, "bad shift");
        if (cols && rt && (!x || !gpos)) throw Error(RL_EINVAL, "null buffer");
        require_device();
        dist_shift_u_rows(x, ldx, cols, r, i0, rt, gpos, (cudaStream_t)stream);
    });
}

int rl_cup_batched_u32_dev(uint32_t* dA, int64_t batch, int64_t m, int64_t n, int64_t stride,
                           uint32_t p, int64_t* ranks, uint32_t* rrp, uint32_t* sigma,
                           void* stream) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, n);
        if (batch < 0) throw Error(RL_EDIM, "negative batch");
        if (stride < m * n) throw Error(RL_EINVAL, "stride smaller than m*n");
        const i64 kcap = std::max<i64>(1, std::min(m, n));
        if (batch == 0) return;
        if (m == 0 || n == 0) {
            for (i64 t = 0; t < batch; ++t) {
                if (ranks) ranks[t] = 0;
                if (sigma) for (i64 j = 0; j < n; ++j) sigma[t * n + j] = (u32)j;
            }
            return;
        }
        require_device();
        cudaStream_t s = (cudaStream_t)stream;
        Call call(s);
        i32* dmeta = (i32*)call.sc.get(SS_META, (size_t)batch * (1 + 2 * kcap) * 4);
        i32* d_ranks = dmeta;
        i32* d_rrp = dmeta + batch;
        i32* d_ipiv = d_rrp + batch * kcap;
        cup_batched(dA, batch, (i32)m, (i32)n, stride, p, d_ranks, d_rrp, d_ipiv, (i32)kcap, s);
        if (!ranks && !rrp && !sigma) return;  // stays asynchronous
        std::vector<i32> h((size_t)batch * (1 + 2 * kcap));
        RL_CUDA_CHECK(cudaMemcpyAsync(h.data(), dmeta, h.size() * 4, cudaMemcpyDeviceToHost, s));
        RL_CUDA_CHECK(cudaStreamSynchronize(s));
        for (i64 t = 0; t < batch; ++t) {
            const i64 r = h[t];
            if (ranks) ranks[t] = r;
            const u32* rp_t = (const u32*)&h[batch + t * kcap];
            const u32* ip_t = (const u32*)&h[batch + batch * kcap + t * kcap];
            if (rrp) for (i64 j = 0; j < r; ++j) rrp[t * kcap + j] = rp_t[j];
            if (sigma) sigma_from_ipiv(n, r, ip_t, sigma + t * n);
        }
    });
}

// Batched CUP of host-resident matrices: the batch crosses PCIe in chunks on a
// copy stream, each chunk is factored as soon as it has landed and goes back on
// a second copy stream while the next one is factored (three-stage pipeline;
// both link directions and the SMs busy at once).
int rl_cup_batched_u32(uint32_t* A, int64_t batch, int64_t m, int64_t n, int64_t stride, uint32_t p,
                       int64_t* ranks, uint32_t* rrp, uint32_t* sigma) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, n);
        if (batch < 0) throw Error(RL_EDIM, "negative batch");
        if (stride < m * n) throw Error(RL_EINVAL, "stride smaller than m*n");
        const i64 kcap = std::max<i64>(1, std::min(m, n));
        if (batch == 0) return;
        if (m == 0 || n == 0) {
            for (i64 t = 0; t < batch; ++t) {
                if (ranks) ranks[t] = 0;
                if (sigma) for (i64 j = 0; j < n; ++j) sigma[t * n + j] = (u32)j;
            }
            return;
        }
        if (!A) throw Error(RL_EINVAL, "null matrix");
        require_device();
        Call call(host_stream());
        cudaStream_t sh = call.sc.aux_stream(0), sc = call.sc.aux_stream(1), sd = call.sc.aux_stream(2);
        u32* dA = (u32*)call.sc.get(SS_A, (size_t)batch * stride * 4);
        i32* dmeta = (i32*)call.sc.get(SS_META, (size_t)batch * (1 + 2 * kcap) * 4);
        i32* d_ranks = dmeta;
        i32* d_rrp = dmeta + batch;
        i32* d_ipiv = d_rrp + batch * kcap;
        // 16 chunks: H2D of chunk c+1, the factorization of chunk c and D2H of
        // chunk c-1 overlap on three streams; each chunk's metadata (ranks, row
        // profiles, transpositions) comes back into pinned memory ahead of its
        // bodies and is expanded on the host while the later chunks are in flight
        const i64 chunks = std::min<i64>(batch, 16);
        i32* h = (i32*)call.sc.pinned_ring_out((size_t)batch * (1 + 2 * kcap) * 4);
        i32* h_ranks = h;
        i32* h_rrp = h + batch;
        i32* h_ipiv = h_rrp + batch * kcap;
        std::vector<cudaEvent_t> ev_in((size_t)chunks), ev_out((size_t)chunks), ev_meta((size_t)chunks);
        for (i64 c = 0; c < chunks; ++c) {
            RL_CUDA_CHECK(cudaEventCreateWithFlags(&ev_in[c], cudaEventDisableTiming));
            RL_CUDA_CHECK(cudaEventCreateWithFlags(&ev_out[c], cudaEventDisableTiming));
            RL_CUDA_CHECK(cudaEventCreateWithFlags(&ev_meta[c], cudaEventDisableTiming));
        }
        for (i64 c = 0; c < chunks; ++c) {
            const i64 t0 = batch * c / chunks, t1 = batch * (c + 1) / chunks;
            // matrix t is the m*n words at A + t*stride: copy exactly those (the
            // caller's buffer may end right after the last matrix's m*n words)
            const size_t pitch = (size_t)stride * 4, width = (size_t)m * n * 4;
            RL_CUDA_CHECK(cudaMemcpy2DAsync(dA + t0 * stride, pitch, A + t0 * stride, pitch, width, t1 - t0,
                                            cudaMemcpyHostToDevice, sh));
            RL_CUDA_CHECK(cudaEventRecord(ev_in[c], sh));
            RL_CUDA_CHECK(cudaStreamWaitEvent(sc, ev_in[c], 0));
            cup_batched(dA + t0 * stride, t1 - t0, (i32)m, (i32)n, stride, p, d_ranks + t0,
                        d_rrp + t0 * kcap, d_ipiv + t0 * kcap, (i32)kcap, sc);
            RL_CUDA_CHECK(cudaEventRecord(ev_out[c], sc));
            RL_CUDA_CHECK(cudaStreamWaitEvent(sd, ev_out[c], 0));
            RL_CUDA_CHECK(cudaMemcpyAsync(h_ranks + t0, d_ranks + t0, (size_t)(t1 - t0) * 4,
                                          cudaMemcpyDeviceToHost, sd));
            RL_CUDA_CHECK(cudaMemcpyAsync(h_rrp + t0 * kcap, d_rrp + t0 * kcap, (size_t)(t1 - t0) * kcap * 4,
                                          cudaMemcpyDeviceToHost, sd));
            RL_CUDA_CHECK(cudaMemcpyAsync(h_ipiv + t0 * kcap, d_ipiv + t0 * kcap, (size_t)(t1 - t0) * kcap * 4,
                                          cudaMemcpyDeviceToHost, sd));
            RL_CUDA_CHECK(cudaEventRecord(ev_meta[c], sd));
            RL_CUDA_CHECK(cudaMemcpy2DAsync(A + t0 * stride, pitch, dA + t0 * stride, pitch, width, t1 - t0,
                                            cudaMemcpyDeviceToHost, sd));
        }
        cudaError_t first_err = cudaSuccess;
        for (i64 c = 0; c < chunks; ++c) {
            const i64 t0 = batch * c / chunks, t1 = batch * (c + 1) / chunks;
            const cudaError_t e = cudaEventSynchronize(ev_meta[c]);
            if (e != cudaSuccess) {
                first_err = e;
                break;
            }
            for (i64 t = t0; t < t1; ++t) {
                const i64 r = h_ranks[t];
                if (ranks) ranks[t] = r;
                const u32* rp_t = (const u32*)(h_rrp + t * kcap);
                const u32* ip_t = (const u32*)(h_ipiv + t * kcap);
                if (rrp) for (i64 j = 0; j < r; ++j) rrp[t * kcap + j] = rp_t[j];
                if (sigma) sigma_from_ipiv(n, r, ip_t, sigma + t * n);
            }
        }
        const cudaError_t e_sc = cudaStreamSynchronize(sc), e_sd = cudaStreamSynchronize(sd);
        for (i64 c = 0; c < chunks; ++c) {
            cudaEventDestroy(ev_in[c]);
            cudaEventDestroy(ev_out[c]);
            cudaEventDestroy(ev_meta[c]);
        }
        RL_CUDA_CHECK(first_err);
        RL_CUDA_CHECK(e_sc);
        RL_CUDA_CHECK(e_sd);
    });
}

// Times one mod-p GEMM C <- C - A*B (m x l x n) on device buffers: pack kernels
// and the tcgen05 kernel separately, each averaged over `iters` launches with
// CUDA events on `stream`.  For benchmarks / roofline only.
int rl_profile_gemm_dev(const uint32_t* dA, const uint32_t* dB, uint32_t* dC, int64_t m,
                        int64_t l, int64_t n, uint32_t p, int iters, float* ms_pack,
                        float* ms_gemm, void* stream) {
    return guard([&] {
        check_field(p);
        require_device();
        cudaStream_t s = (cudaStream_t)stream;
        Call call(s);
        const int L = limbs_for(p);
        if (l > tc_kmax(L)) throw Error(RL_EINVAL, "profile: l exceeds the exact-accumulation bound");
        GemmArgs g{};
        g.A = dA; g.lda = l; g.B = dB; g.ldb = n; g.C = dC; g.ldc = n; g.M = (i32)m;
        g.k_lo = dyn_c(0); g.k_hi = dyn_c((i32)l); g.n_lo = dyn_c(0); g.n_hi = dyn_c((i32)n);
        g.alpha = p - 1; g.beta = 1 % p; g.f = make_fp(p);
        uint8_t* pa = (uint8_t*)call.sc.get(SS_PROF_A2, tc_a2_bytes(L, m, l));
        uint8_t* pb = (uint8_t*)call.sc.get(SS_PROF_B2, tc_b2_bytes(L, n, l));
        cudaEvent_t e0, e1, e2;
        RL_CUDA_CHECK(cudaEventCreate(&e0));
        RL_CUDA_CHECK(cudaEventCreate(&e1));
        RL_CUDA_CHECK(cudaEventCreate(&e2));
        gemm_tc_split(g, L, l, n, pa, pb, s, 0);  // warm-up
        gemm_tc_split(g, L, l, n, pa, pb, s, 1);
        float tp = 0, tg = 0;
        for (int it = 0; it < iters; ++it) {
            RL_CUDA_CHECK(cudaEventRecord(e0, s));
            gemm_tc_split(g, L, l, n, pa, pb, s, 0);
            RL_CUDA_CHECK(cudaEventRecord(e1, s));
            gemm_tc_split(g, L, l, n, pa, pb, s, 1);
            RL_CUDA_CHECK(cudaEventRecord(e2, s));
            RL_CUDA_CHECK(cudaEventSynchronize(e2));
            float a = 0, b = 0;
            RL_CUDA_CHECK(cudaEventElapsedTime(&a, e0, e1));
            RL_CUDA_CHECK(cudaEventElapsedTime(&b, e1, e2));
            tp += a;
            tg += b;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
        *ms_pack = tp / iters;
        *ms_gemm = tg / iters;
    });
}

int rl_cup_plan_stats(int64_t m, int64_t n, int64_t lda, uint32_t p, int64_t* stats) {
    return guard([&] {
        check_field(p);
        check_dims(m, n, lda);
        // the most recently used engine of this shape on this device
        std::shared_ptr<CupEngine> e;
        {
            std::lock_guard<std::mutex> lk(g_engines_mu);
            unsigned long long best = 0;
            const int dev = current_device();
            for (auto& kv : g_engines)
                if (kv.first.dev == dev && kv.first.m == m && kv.first.n == n && kv.first.lda == lda &&
                    kv.first.p == p && !kv.first.split && kv.second.used >= best) {
                    best = kv.second.used;
                    e = kv.second.e;
                }
        }
        if (!e) e = engine_for(m, n, lda, p, nullptr);
        const auto& st = e->stats();
        stats[0] = st.gemms;
        stats[1] = st.tc_gemms;
        stats[2] = st.panels;
        stats[3] = st.trsm_leaves;
        stats[4] = (int64_t)e->workspace_bytes();
        stats[5] = st.launches;
    });
}

}  // extern "C"

extern "C" {
// Host-only: the reference's exact OpCounter charges of cup() from the shape,
// the row profile and the pivot positions (see cup_opcount in cup.cu).
int rl_cup_opcount(int64_t m, int64_t n, int64_t rank, const uint32_t* rrp, const uint32_t* ipiv,
                   uint64_t* ops) {
    return guard([&] {
        if (!ops) throw Error(RL_EINVAL, "null ops");
        if (m < 0 || n < 0 || rank < 0 || rank > std::min(m, n)) throw Error(RL_EDIM, "bad shape");
        cup_opcount(m, n, rank, rrp, ipiv, ops);
    });
}
}
