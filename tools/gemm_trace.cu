// Per-CTA phase timeline of one gemm_tc_kernel launch (globaltimer stamps):
// 0 entry, 1 after setup (TMEM alloc + barrier init), 2 first stage landed
// (MMA thread), 3 last MMA committed, 4 accumulator ready (epilogue warp 2),
// 5 epilogue done, 6 exit.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRL_GEMM_TRACE \
//        --expt-relaxed-constexpr -o tools/gemm_trace tools/gemm_trace.cu -lcuda
// Usage: gemm_trace M K N p
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1112_5717_b200/csrc/gemm_tc.cu"

namespace rl {
int num_sms() {
    int d = 0, n = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
}
}  // namespace rl

int main(int argc, char** argv) {
    using namespace rl;
    const int M = argc > 1 ? atoi(argv[1]) : 64, K = argc > 2 ? atoi(argv[2]) : 64,
              N = argc > 3 ? atoi(argv[3]) : 8192;
    const u32 p = argc > 4 ? (u32)atoi(argv[4]) : 65521u;

    u32 *A, *B, *C;
    cudaMalloc(&A, (size_t)M * K * 4);
    cudaMalloc(&B, (size_t)K * N * 4);
    cudaMalloc(&C, (size_t)M * N * 4);
    cudaMemset(A, 0, (size_t)M * K * 4);
    cudaMemset(B, 0, (size_t)K * N * 4);
    cudaMemset(C, 0, (size_t)M * N * 4);
    const int L = limbs_for(p);
    uint8_t *a2, *b2;
    cudaMalloc(&a2, tc_a2_bytes(L, M, K));
    cudaMalloc(&b2, tc_b2_bytes(L, N, K));
    GemmArgs g{};
    g.A = A; g.lda = K; g.B = B; g.ldb = N; g.C = C; g.ldc = N; g.M = M;
    g.k_lo = dyn_c(0); g.k_hi = dyn_c(K); g.n_lo = dyn_c(0); g.n_hi = dyn_c(N);
    g.alpha = p - 1; g.beta = 1; g.f = make_fp(p);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int rep = 0; rep < 3; ++rep) {
        gemm_tc_split(g, L, K, N, a2, b2, s, 0);
        cudaStreamSynchronize(s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        gemm_tc_split(g, L, K, N, a2, b2, s, 1);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> tr(1024 * 8);
        cudaMemcpyFromSymbol(tr.data(), g_gemm_trace, tr.size() * 8);
        const int NT = tc_nt(L);
        const int ctas = std::min(((M + 127) / 128) * ((N + NT - 1) / NT), num_sms());
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < ctas; ++c) t0 = std::min(t0, tr[c * 8]);
        double avg[7] = {0};
        for (int c = 0; c < ctas; ++c)
            for (int i = 0; i < 7; ++i) avg[i] += (double)(tr[c * 8 + i] - t0) / ctas / 1e3;
        printf("rep %d: event %.1f us, %d CTAs; avg stamps (us from first entry):", rep, ms * 1e3, ctas);
        for (int i = 0; i < 7; ++i) printf(" %.2f", avg[i]);
        printf("  | CTA0:");
        for (int i = 0; i < 7; ++i) printf(" %.2f", (tr[i] - t0) / 1e3);
        printf("\n");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
