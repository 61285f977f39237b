// Kernel microbenchmarks behind the C ABI (instrumentation, include/espec_c.h):
// one decode GEMV shape timed in isolation with CUDA events, weights rotated
// over enough copies that every launch streams from HBM (> 2x L2).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../../include/espec_c.h"
#include "common.cuh"
#include "kernels.h"

using namespace espec_dev;

extern "C" espec_status espec_bench_gemv(int K, int N, int T, int nprob, int epi, int iters, int device,
                                         double* us_per_launch, double* bytes_per_launch) {
    if (K <= 0 || N <= 0 || T <= 0 || T > 16 || nprob < 1 || nprob > kMaxProblems || iters < 1) return ESPEC_CONFIG;
    if (epi != EPI_STORE && epi != EPI_RESID && epi != EPI_SILU) return ESPEC_CONFIG;
    if (K % 16 || N % 32) return ESPEC_SHAPE;
    if (cudaSetDevice(device) != cudaSuccess) return ESPEC_CUDA;
    const size_t wbytes = (size_t)K * N * 2 * nprob;
    const int nrot = (int)std::max<size_t>(2, (size_t)(512ull << 20) / wbytes + 1);
    std::vector<void*> W(nrot * nprob, nullptr);
    float *x = nullptr, *out = nullptr, *resid = nullptr, *stats = nullptr, *part = nullptr;
    unsigned* tickets = nullptr;
    cudaStream_t s;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto& w : W) {
        cudaMalloc(&w, (size_t)K * N * 2);
        launch_fill_normal(DT_BF16, w, (long long)K * N, 0.02f, 1234, s);
    }
    const size_t pf = std::max<size_t>(sgemv_partial_floats(K, N), 16);
    cudaMalloc(&x, sizeof(float) * 16 * K * nprob);
    cudaMalloc(&out, sizeof(float) * 16 * N * nprob);
    cudaMalloc(&resid, sizeof(float) * 16 * N * nprob);
    cudaMalloc(&stats, sizeof(float) * 16 * (N / 32 + 1) * nprob);
    cudaMalloc(&part, sizeof(float) * pf * nprob);
    cudaMalloc(&tickets, sizeof(unsigned) * (N / 32 + 1) * nprob);
    cudaMemsetAsync(tickets, 0, sizeof(unsigned) * (N / 32 + 1) * nprob, s);
    cudaMemsetAsync(resid, 0, sizeof(float) * 16 * N * nprob, s);
    launch_fill_normal(DT_F32, x, 16LL * K * nprob, 1.0f, 99, s);
    auto batch = [&](int r) {
        GemvBatch b;
        for (int p = 0; p < nprob; ++p) {
            GemvProblem& P = b.p[p];
            P.W = W[r * nprob + p];
            P.K = K;
            P.N = N;
            P.ldw = N;
            P.x = x + (size_t)p * 16 * K;
            P.ldx = K;
            P.partial = part + pf * p;
            P.tickets = tickets + (size_t)(N / 32 + 1) * p;
            P.out = out + (size_t)p * 16 * N;
            P.ldo = epi == EPI_SILU ? N / 2 : N;
            P.resid = resid + (size_t)p * 16 * N;
            P.ldr = N;
            P.stats_out = stats + (size_t)p * 16 * (N / 32 + 1);
            P.stat_tiles_out = N / 32;
        }
        return b;
    };
    PassView pv;
    KvView kv;
    for (int i = 0; i < 3; ++i) launch_gemv(epi, DT_BF16, batch(i % nrot), nprob, T, pv, kv, s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) launch_gemv(epi, DT_BF16, batch(i % nrot), nprob, T, pv, kv, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    *us_per_launch = 1000.0 * ms / iters;
    *bytes_per_launch = (double)wbytes;
    for (auto& w : W) cudaFree(w);
    cudaFree(x);
    cudaFree(out);
    cudaFree(resid);
    cudaFree(stats);
    cudaFree(part);
    cudaFree(tickets);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    return err == cudaSuccess ? ESPEC_OK : ESPEC_CUDA;
}
