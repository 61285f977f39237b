// Kernel microbenchmarks behind the C ABI (instrumentation, include/espec_c.h):
// one decode GEMV shape timed in isolation with CUDA events, weights rotated
// over enough copies that every launch streams from HBM (> 2x L2).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../../include/espec_c.h"
#include "common.cuh"
#include "kernels.h"

using namespace espec_dev;

static espec_status espec_bench_gemv_impl(int K, int N, int T, int nprob, int epi, int iters, int device,
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

// Decode/verify attention over a paged bf16 cache in isolation: T query rows
// (the last T rows of a ctx-row context, causal), n_heads = G * n_kv.
static espec_status espec_bench_attn_impl(int T, int n_heads, int n_kv, int dh, int ctx, int nprob, int iters,
                                         int device, double* us_per_launch, double* bytes_per_launch) {
    if (T < 1 || T > 16 || n_kv < 1 || n_heads % n_kv || (dh != 64 && dh != 128) || ctx < T || nprob < 1 ||
        nprob > kMaxProblems || iters < 1)
        return ESPEC_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return ESPEC_CUDA;
    const int page_rows = 64, n_layers = nprob;
    const int n_pages = (ctx + page_rows - 1) / page_rows;
    const long long page_elems = (long long)n_layers * 2 * n_kv * page_rows * dh;
    void* pool = nullptr;
    int *table = nullptr, *rows = nullptr, *pos = nullptr, *vis = nullptr;
    unsigned long long* anc = nullptr;
    float *q = nullptr, *out = nullptr, *ws = nullptr;
    unsigned* tk = nullptr;
    cudaStream_t s;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMalloc(&pool, (size_t)n_pages * page_elems * 2);
    launch_fill_normal(DT_BF16, pool, (long long)n_pages * page_elems, 1.0f, 7, s);
    std::vector<int> h_table(n_pages), h_rows(T), h_pos(T), h_vis(T);
    for (int p = 0; p < n_pages; ++p) h_table[p] = p;
    for (int t = 0; t < T; ++t) {
        h_rows[t] = ctx - T + t;
        h_pos[t] = h_rows[t];
        h_vis[t] = h_rows[t] + 1;
    }
    cudaMalloc(&table, sizeof(int) * n_pages);
    cudaMalloc(&rows, sizeof(int) * T);
    cudaMalloc(&pos, sizeof(int) * T);
    cudaMalloc(&vis, sizeof(int) * T);
    cudaMalloc(&anc, sizeof(unsigned long long) * T);
    cudaMemcpy(table, h_table.data(), sizeof(int) * n_pages, cudaMemcpyHostToDevice);
    cudaMemcpy(rows, h_rows.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
    cudaMemcpy(pos, h_pos.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
    cudaMemcpy(vis, h_vis.data(), sizeof(int) * T, cudaMemcpyHostToDevice);
    cudaMemset(anc, 0, sizeof(unsigned long long) * T);
    const size_t wsf = attn_ws_floats(16, n_heads, dh, ctx + 64);
    const size_t tkn = attn_tickets(16, n_heads, n_kv);
    cudaMalloc(&q, sizeof(float) * (size_t)nprob * 16 * n_heads * dh);
    cudaMalloc(&out, sizeof(float) * (size_t)nprob * 16 * n_heads * dh);
    cudaMalloc(&ws, sizeof(float) * wsf * nprob);
    cudaMalloc(&tk, sizeof(unsigned) * tkn * nprob);
    cudaMemset(tk, 0, sizeof(unsigned) * tkn * nprob);
    launch_fill_normal(DT_F32, q, (long long)nprob * 16 * n_heads * dh, 1.0f, 3, s);
    KvView kv;
    kv.pool = pool;
    kv.page_table = table;
    kv.page_rows = page_rows;
    kv.n_layers = n_layers;
    kv.n_kv = n_kv;
    kv.dh = dh;
    kv.dtype = DT_BF16;
    kv.page_elems = page_elems;
    kv.pool_pages = n_pages;
    {
        const int cap = (ctx + 64 + page_rows - 1) / page_rows * page_rows;  // as Cache::view()
        kv.attn_ppi = attn_pages_per_item(cap);
    }
    PassView pv;
    pv.T = T;
    pv.rows = rows;
    pv.pos = pos;
    pv.vis_end = vis;
    pv.anc = anc;
    pv.tree_base = ctx;
    pv.total = ctx;
    pv.new_lo = ctx - T;  // as in the engine: the pass's own rows are the last T
    AttnBatch b;
    for (int p = 0; p < nprob; ++p) {
        b.p[p].q = q + (size_t)p * 16 * n_heads * dh;
        b.p[p].out = out + (size_t)p * 16 * n_heads * dh;
        b.p[p].layer = p;
        b.p[p].ws = ws + wsf * p;
        b.p[p].tickets = tk + tkn * p;
    }
    for (int i = 0; i < 3; ++i) launch_attention(b, nprob, n_heads, pv, kv, s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) launch_attention(b, nprob, n_heads, pv, kv, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    *us_per_launch = 1000.0 * ms / iters;
    *bytes_per_launch = (double)nprob * 2.0 * ctx * n_kv * dh * 2;
    cudaFree(pool);
    cudaFree(table);
    cudaFree(rows);
    cudaFree(pos);
    cudaFree(vis);
    cudaFree(anc);
    cudaFree(q);
    cudaFree(out);
    cudaFree(ws);
    cudaFree(tk);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    return err == cudaSuccess ? ESPEC_OK : ESPEC_CUDA;
}

// Prefill GEMM (tcgen05) in isolation: M rows x K -> N (store epilogue).
static espec_status espec_bench_tc_impl(int M, int K, int N, int iters, int device, double* us_per_launch,
                                       double* flops_per_launch) {
    if (M < 1 || M > 256 || K % 16 || N % 32 || iters < 1) return ESPEC_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return ESPEC_CUDA;
    void* W = nullptr;
    float *x = nullptr, *out = nullptr, *rms = nullptr;
    __nv_bfloat16* xa = nullptr;
    cudaStream_t s;
    cudaEvent_t e0, e1;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMalloc(&W, (size_t)K * N * 2);
    launch_fill_normal(DT_BF16, W, (long long)K * N, 0.02f, 1234, s);
    cudaMalloc(&x, sizeof(float) * (size_t)M * K);
    cudaMalloc(&out, sizeof(float) * (size_t)M * N);
    cudaMalloc(&rms, sizeof(float) * 256);
    cudaMalloc(&xa, sizeof(__nv_bfloat16) * tc_xa_elems(M, K));
    launch_fill_normal(DT_F32, x, (long long)M * K, 1.0f, 99, s);
    GemvProblem P;
    P.W = W;
    P.K = K;
    P.N = N;
    P.ldw = N;
    P.x = x;
    P.ldx = K;
    P.out = out;
    P.ldo = N;
    float* part = nullptr;
    unsigned* tks = nullptr;
    const size_t pf = tc_part_floats(K, N);
    if (pf) {
        cudaMalloc(&part, sizeof(float) * pf);
        cudaMalloc(&tks, sizeof(unsigned) * 1024);
        cudaMemset(tks, 0, sizeof(unsigned) * 1024);
        P.tc_part = part;
        P.tc_tickets = tks;
    }
    PassView pv;
    KvView kv;
    for (int i = 0; i < 2; ++i) launch_tc_gemm(EPI_STORE, P, M, pv, kv, xa, rms, s);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) launch_tc_gemm(EPI_STORE, P, M, pv, kv, xa, rms, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    *us_per_launch = 1000.0 * ms / iters;
    *flops_per_launch = 2.0 * M * (double)K * N;
    cudaFree(W);
    cudaFree(x);
    cudaFree(out);
    cudaFree(rms);
    if (part) cudaFree(part);
    if (tks) cudaFree(tks);
    cudaFree(xa);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    return err == cudaSuccess ? ESPEC_OK : ESPEC_CUDA;
}

// Correctness probe of the prefill GEMM: out = bf16(x) . W for M rows with
// host fp32 inputs (W logical K x N, row-major), packed on device.
static espec_status espec_probe_tc_impl(int M, int K, int N, const float* x_host, const float* w_host, float* out_host,
                                       int device) {
    if (M < 1 || M > 256 || K % 16 || N % 32) return ESPEC_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return ESPEC_CUDA;
    std::vector<__nv_bfloat16> wb((size_t)K * N);
    for (size_t i = 0; i < wb.size(); ++i) wb[i] = __float2bfloat16_rn(w_host[i]);
    void *Wl = nullptr, *W = nullptr;
    float *x = nullptr, *out = nullptr, *rms = nullptr;
    __nv_bfloat16* xa = nullptr;
    cudaMalloc(&Wl, (size_t)K * N * 2);
    cudaMalloc(&W, packed_elems(K, N) * 2);
    cudaMemcpy(Wl, wb.data(), (size_t)K * N * 2, cudaMemcpyHostToDevice);
    launch_pack(Wl, K, N, W, false, 0);
    cudaMalloc(&x, sizeof(float) * (size_t)M * K);
    cudaMalloc(&out, sizeof(float) * (size_t)M * N);
    cudaMalloc(&rms, sizeof(float) * 256);
    cudaMalloc(&xa, sizeof(__nv_bfloat16) * tc_xa_elems(M, K));
    cudaMemcpy(x, x_host, sizeof(float) * (size_t)M * K, cudaMemcpyHostToDevice);
    cudaMemset(out, 0, sizeof(float) * (size_t)M * N);
    GemvProblem P;
    P.W = W;
    P.K = K;
    P.N = N;
    P.ldw = N;
    P.x = x;
    P.ldx = K;
    P.out = out;
    P.ldo = N;
    float* part = nullptr;
    unsigned* tks = nullptr;
    const size_t pf = tc_part_floats(K, N);
    if (pf) {
        cudaMalloc(&part, sizeof(float) * pf);
        cudaMalloc(&tks, sizeof(unsigned) * 1024);
        cudaMemset(tks, 0, sizeof(unsigned) * 1024);
        P.tc_part = part;
        P.tc_tickets = tks;
    }
    PassView pv;
    KvView kv;
    launch_tc_gemm(EPI_STORE, P, M, pv, kv, xa, rms, 0);
    cudaMemcpy(out_host, out, sizeof(float) * (size_t)M * N, cudaMemcpyDeviceToHost);
    const cudaError_t err = cudaGetLastError();
    cudaFree(Wl);
    cudaFree(W);
    cudaFree(x);
    cudaFree(out);
    cudaFree(rms);
    if (part) cudaFree(part);
    if (tks) cudaFree(tks);
    cudaFree(xa);
    return err == cudaSuccess ? ESPEC_OK : ESPEC_CUDA;
}

// One decode GEMV (EPI_STORE or EPI_RESID with zero residual) on host data:
// x [T][K] fp32, w [K][N] fp32 (rounded to bf16, packed), out [T][N]. Used by
// the batch-invariance tests (a row's result must not depend on T).
static espec_status espec_probe_gemv_impl(int T, int K, int N, int epi, const float* x_host, const float* w_host,
                                         float* out_host, int device) {
    if (T < 1 || T > 16 || K % 16 || N % 32 || (epi != EPI_STORE && epi != EPI_RESID)) return ESPEC_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return ESPEC_CUDA;
    std::vector<__nv_bfloat16> wb((size_t)K * N);
    for (size_t i = 0; i < wb.size(); ++i) wb[i] = __float2bfloat16_rn(w_host[i]);
    void *Wl = nullptr, *W = nullptr;
    float *x = nullptr, *out = nullptr, *resid = nullptr, *stats = nullptr, *part = nullptr;
    unsigned* tickets = nullptr;
    cudaMalloc(&Wl, (size_t)K * N * 2);
    cudaMalloc(&W, packed_elems(K, N) * 2);
    cudaMemcpy(Wl, wb.data(), (size_t)K * N * 2, cudaMemcpyHostToDevice);
    launch_pack(Wl, K, N, W, false, 0);
    cudaMalloc(&x, sizeof(float) * 16 * K);
    cudaMalloc(&out, sizeof(float) * 16 * N);
    cudaMalloc(&resid, sizeof(float) * 16 * N);
    cudaMalloc(&stats, sizeof(float) * 16 * (N / 32 + 1));
    const size_t pf = std::max<size_t>(sgemv_partial_floats(K, N), 16);
    cudaMalloc(&part, sizeof(float) * pf);
    cudaMalloc(&tickets, sizeof(unsigned) * (N / 32 + 1));
    cudaMemset(tickets, 0, sizeof(unsigned) * (N / 32 + 1));
    cudaMemset(resid, 0, sizeof(float) * 16 * N);
    cudaMemcpy(x, x_host, sizeof(float) * (size_t)T * K, cudaMemcpyHostToDevice);
    GemvBatch b;
    GemvProblem& P = b.p[0];
    P.W = W; P.K = K; P.N = N; P.ldw = N; P.x = x; P.ldx = K; P.out = out; P.ldo = N;
    P.partial = part; P.tickets = tickets;
    P.resid = resid; P.ldr = N; P.stats_out = stats; P.stat_tiles_out = N / 32;
    PassView pv;
    KvView kv;
    launch_sgemv(epi, b, 1, T, pv, kv, 0);
    cudaMemcpy(out_host, out, sizeof(float) * (size_t)T * N, cudaMemcpyDeviceToHost);
    const cudaError_t err = cudaGetLastError();
    cudaFree(Wl); cudaFree(W); cudaFree(x); cudaFree(out); cudaFree(resid); cudaFree(stats); cudaFree(part);
    cudaFree(tickets);
    return err == cudaSuccess ? ESPEC_OK : ESPEC_CUDA;
}

// The launch wrappers throw DevError on a rejected launch; nothing crosses
// the C ABI as an exception.
template <typename F>
static espec_status mb_guard(F&& f) {
    try {
        return f();
    } catch (const DevError& x) {
        fprintf(stderr, "%s\n", x.what());
        return (espec_status)x.code;
    } catch (const std::exception& x) {
        fprintf(stderr, "%s\n", x.what());
        return ESPEC_CHECK;
    }
}

extern "C" espec_status espec_bench_gemv(int K, int N, int T, int nprob, int epi, int iters, int device,
                                         double* us_per_launch, double* bytes_per_launch) {
    return mb_guard([&] { return espec_bench_gemv_impl(K, N, T, nprob, epi, iters, device, us_per_launch, bytes_per_launch); });
}
extern "C" espec_status espec_bench_attn(int T, int n_heads, int n_kv, int d_head, int ctx, int nprob, int iters,
                                         int device, double* us_per_launch, double* bytes_per_launch) {
    return mb_guard([&] {
        return espec_bench_attn_impl(T, n_heads, n_kv, d_head, ctx, nprob, iters, device, us_per_launch, bytes_per_launch);
    });
}
extern "C" espec_status espec_bench_tc(int M, int K, int N, int iters, int device, double* us_per_launch,
                                       double* flops_per_launch) {
    return mb_guard([&] { return espec_bench_tc_impl(M, K, N, iters, device, us_per_launch, flops_per_launch); });
}
extern "C" espec_status espec_probe_tc(int M, int K, int N, const float* x, const float* w, float* out, int device) {
    return mb_guard([&] { return espec_probe_tc_impl(M, K, N, x, w, out, device); });
}
extern "C" espec_status espec_probe_gemv(int T, int K, int N, int epi, const float* x, const float* w, float* out,
                                         int device) {
    return mb_guard([&] { return espec_probe_gemv_impl(T, K, N, epi, x, w, out, device); });
}
