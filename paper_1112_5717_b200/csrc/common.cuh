// common.cuh -- shared device helpers for the B200 CUP library.
//
// Field arithmetic follows ranklab::PrimeField (proj/include/ranklab/field.hpp:45-107):
// elements are canonical uint32 in [0,p), 2 <= p < 2^31.  Reduction of 64-bit
// intermediates uses a Barrett constant m64 = floor((2^64-1)/p): q = hi64(x*m64)
// underestimates floor(x/p) by at most 1, so one conditional subtract yields the
// canonical remainder for every x < 2^64.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Timeline tracing (tools/trace_cup.py, `make trace`): kernels print per-CTA
// %globaltimer stamps for the leaf at row RL_TRACE_I0.  Compiled out otherwise.
#ifdef RL_TRACE
#ifndef RL_TRACE_I0
#define RL_TRACE_I0 8192
#endif
__device__ __forceinline__ unsigned long long rl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}
#define RL_STAMP(var) const unsigned long long var = rl_now()
#else
#define RL_STAMP(var)
#endif

typedef uint32_t u32;
typedef uint64_t u64;
typedef int32_t i32;
typedef int64_t i64;

struct Fp {
    u32 p;
    u32 m32;  // floor((2^32-1)/p): 32-bit Barrett for x < 2^32
    u64 m64;  // floor((2^64-1)/p)
    u32 r32;  // 2^32 mod p
};

static inline Fp make_fp(u32 p) {
    Fp f;
    f.p = p;
    f.m32 = (u32)(0xFFFFFFFFu / p);
    f.m64 = ~0ull / (u64)p;
    f.r32 = (u32)((1ull << 32) % p);
    return f;
}

__device__ __forceinline__ u32 red64(u64 x, const Fp& f) {
    u64 q = __umul64hi(x, f.m64);
    u64 r = x - q * (u64)f.p;
    return (u32)(r >= f.p ? r - f.p : r);
}

// x < 2^32
__device__ __forceinline__ u32 red32(u32 x, const Fp& f) {
    u32 q = __umulhi(x, f.m32);
    u32 r = x - q * f.p;
    return r >= f.p ? r - f.p : r;
}

// Short-latency reduction for p <= 2^16 and x < 2^40 (lazy accumulators of at
// most 2^8 products of canonical elements): x = hi*2^32 + lo with hi < 2^8.
__device__ __forceinline__ u32 red_sp(u64 x, const Fp& f) {
    const u32 t = red32((u32)x, f) + (u32)(x >> 32) * f.r32;  // < 2^25
    return red32(t, f);
}

__device__ __forceinline__ u32 mulmod(u32 a, u32 b, const Fp& f) {
    return red64((u64)a * b, f);
}

// a, b < p <= 2^16: the product fits 32 bits.
__device__ __forceinline__ u32 mulmod_sp(u32 a, u32 b, const Fp& f) { return red32(a * b, f); }
template <bool SP>
__device__ __forceinline__ u32 mulmod_t(u32 a, u32 b, const Fp& f) {
    return SP ? mulmod_sp(a, b, f) : mulmod(a, b, f);
}

__device__ __forceinline__ u32 addmod(u32 a, u32 b, const Fp& f) {
    u32 s = a + b;  // a,b < 2^31 so no wrap
    return s >= f.p ? s - f.p : s;
}

__device__ __forceinline__ u32 submod(u32 a, u32 b, const Fp& f) {
    return a >= b ? a - b : a + (f.p - b);
}

__device__ __forceinline__ u32 negmod(u32 a, const Fp& f) { return a == 0 ? 0 : f.p - a; }

// Modular inverse of a != 0 by Fermat (p prime).  Any inverse algorithm yields
// the same element (field.cpp:60-76 uses extended Euclid).
__device__ __forceinline__ u32 invmod(u32 a, const Fp& f) {
    u32 r = 1 % f.p, b = a, e = f.p - 2;
    while (e) {
        if (e & 1) r = mulmod(r, b, f);
        b = mulmod(b, b, f);
        e >>= 1;
    }
    return r;
}

// Inverse by the extended Euclidean algorithm (a in [1, p)): ~0.84 ln p division
// steps on average, far shorter than Fermat's exponentiation chain.
__device__ __forceinline__ u32 inv_euclid(u32 a, u32 p) {
    // 32-bit throughout: remainders < p < 2^31 and |coefficients| <= p
    u32 r0 = p, r1 = a;
    int t0 = 0, t1 = 1;
    while (r1 != 0) {
        const u32 q = r0 / r1;
        const u32 r2 = r0 - q * r1;
        const int t2 = t0 - (int)q * t1;
        r0 = r1;
        r1 = r2;
        t0 = t1;
        t1 = t2;
    }
    return (u32)(t0 < 0 ? t0 + (int)p : t0);
}

// Asynchronous global -> shared copies (LDGSTS): a copy loop issues every load
// before anything waits, instead of one memory round trip per iteration.
// src_bytes = 0 zero-fills the destination (out-of-range elements).
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}
// 16-byte copy of which the first src_bytes (0..16) come from gmem, the rest
// zero-filled (gmem must be 16-byte aligned; it is not read when src_bytes = 0).
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, int src_bytes) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// A device-evaluated index: value = (idx >= 0 ? rp[idx] : 0) + cst.  All
// rank-dependent shapes of the CUP recursion are expressed this way, so the
// whole launch sequence is static (graph-capturable) while the sizes come from
// the device-resident rank prefix rp[i] = rank of rows [0, i).
struct Dyn {
    i32 idx;
    i32 cst;
};
__host__ __device__ inline Dyn dyn_c(i32 c) { return Dyn{-1, c}; }
__host__ __device__ inline Dyn dyn_rp(i32 i, i32 c = 0) { return Dyn{i, c}; }

// Programmatic dependent launch (launch_pdl in runtime.h).  Protocol of every
// kernel launched that way: touch no global memory produced by the previous
// kernel before pdl_wait() (which waits for that grid's completion and memory
// flush), and call pdl_trigger() only after it -- so when a kernel's CTAs
// start early, every kernel before its predecessor has completed.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Legacy warp-level tensor-core MMA: D(16x8, s32) += A(16x32, u8, row) *
// B(32x8, u8, col).  Fragments (PTX ISA, mma.m16n8k32 .u8): lane = 4*g + t;
// a0/a2: row g, a1/a3: row g+8, bytes k = 4t..4t+3 (+16 for a2/a3);
// b0/b1: column g, bytes k = 4t..4t+3 (+16 for b1); d0/d1: row g, columns
// 2t, 2t+1; d2/d3: row g+8.  About 2 K u8 MAC/clk/SM here (tools/imma_rate.cu),
// against 23.6 IMAD.WIDE: the p < 2^16 tail runs on it with 2 byte limbs.
__device__ __forceinline__ void imma16832(int (&d)[4], const u32 (&a)[4], const u32 (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// U^{-1}-ready flags (cup.cu): a leaf's flag holds the factorization's epoch once
// its U^{-1} is in global memory; consumers wait on it instead of on a stream event.
__device__ __forceinline__ void uready_set(i32* flag, const i32* epoch) {
    __threadfence();
    const i32 v = __ldcg(epoch);
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
__device__ __forceinline__ void uready_wait(const i32* flag, const i32* epoch) {
    const i32 want = __ldcg(epoch);
    for (;;) {
        i32 v;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v == want) break;
        __nanosleep(64);
    }
}
__device__ __forceinline__ i32 dyn_eval(const Dyn& d, const i32* rp) {
    return (d.idx >= 0 ? __ldcg(rp + d.idx) : 0) + d.cst;
}



// Leaf-chain probe (tuning builds, -DRL_LEAFTRACE): per kernel and leaf, the
// globaltimer after pdl_wait and at exit, in a per-file device table read back
// by rl_lt_dump_<file>() (tools/leaftrace.py).
#ifdef RL_LEAFTRACE
__device__ __forceinline__ unsigned long long rl_gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define LT_TABLE(name)                                                        \
    static __device__ unsigned long long g_lt[1024][8];                       \
    extern "C" int rl_lt_dump_##name(unsigned long long* h) {                 \
        return (int)cudaMemcpyFromSymbol(h, g_lt, sizeof(g_lt));             \
    }
#define LT_BEGIN() const unsigned long long lt_t0 = rl_gt()
#define LT_MARK(key, i)                                                       \
    do {                                                                      \
        if (threadIdx.x == 0 && (key) >= 0 && (key) < 1024) g_lt[(key)][(i)] = rl_gt(); \
    } while (0)
#define LT_END(key)                                                           \
    do {                                                                      \
        if (threadIdx.x == 0 && (key) >= 0 && (key) < 1024) {                 \
            g_lt[(key)][0] = lt_t0;                                           \
            g_lt[(key)][1] = rl_gt();                                         \
        }                                                                     \
    } while (0)
#else
#define LT_TABLE(name)
#define LT_BEGIN()
#define LT_MARK(key, i)
#define LT_END(key)
#endif

// Critical-path probes (tuning builds only): busy-wait ns nanoseconds.
__device__ __forceinline__ void rl_spin_ns(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

#define RL_CUDA_CHECK(x)                                                  \
    do {                                                                  \
        cudaError_t _e = (x);                                             \
        if (_e != cudaSuccess) throw rl::CudaError(_e, #x, __FILE__, __LINE__); \
    } while (0)
