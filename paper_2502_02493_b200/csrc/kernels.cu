// sm_100a kernels for the EasySpec decode loop (the bf16 GEMV lives in
// gemv_stream.cu).
//
// This file holds the fp32 parity-mode GEMV (the reference model in fp32:
// CUDA-core FMA over the row-major layout, 8 warps splitting K, a CTA per
// (256-column tile, K split)), the embedding / residual kernels, paged-KV
// attention, KV commit compaction, greedy acceptance and weight init.
// Fused prologue/epilogue semantics are shared with the bf16 path: RMSNorm
// from row sum-of-squares partials (one per 32 columns), residual add + row
// stats, SiLU over [gate16 | up16] packed groups, RoPE + paged-KV write,
// argmax. Reduction order never depends on T (batch invariance).
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "attn_common.cuh"

namespace espec_dev {

#define CK(x) DEV_CK(x)

void dev_fail(int code, const std::string& msg) { throw DevError(code, msg); }

void dev_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    (void)cudaGetLastError();  // clear a non-sticky launch error so the engine stays usable
    dev_fail(DEV_ERR_CUDA, std::string(what) + " failed: " + cudaGetErrorString(e) + " (" + file + ":" +
                               std::to_string(line) + ")");
}

void ensure_smem(const void* kernel, int bytes, unsigned long long& mask) {
    int dev = 0;
    DEV_CK(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask & bit) return;
    DEV_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    mask |= bit;
}

// ---------------------------------------------------------------------------
// GEMV planning
// ---------------------------------------------------------------------------

GemvPlan gemv_plan(int K, int N) {
    GemvPlan p;
    p.tiles = (N + kTileN - 1) / kTileN;
    // ~4 waves of CTAs over 148 SMs, K chunks of at most 1024 rows, a
    // multiple of 64 (8 warps x 8-row unroll).
    const int target = 4 * 148;
    int splits = (target + p.tiles - 1) / p.tiles;
    const int max_splits = (K + 63) / 64;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    int kc = (K + splits - 1) / splits;
    kc = (kc + 63) / 64 * 64;
    if (kc > 1024) kc = 1024;
    p.kc = kc;
    p.splits = (K + kc - 1) / kc;
    return p;
}

size_t gemv_partial_floats(int K, int N) {
    const GemvPlan p = gemv_plan(K, N);
    return (size_t)p.splits * 16 * (size_t)p.tiles * kTileN;
}

struct GemvLaunch {
    GemvBatch b;
    PassView pass;
    KvView kv;
    int t0, T;  // rows [t0, t0+T) of the pass, T <= TM
    int tiles, splits, kc;
};

// ---------------------------------------------------------------------------
// fp32 GEMV kernel (parity mode)
// ---------------------------------------------------------------------------

__device__ __forceinline__ bool am_better(float v, int i, float bv, int bi) {
    return v > bv || (v == bv && i < bi);
}

template <int TM, int EPI>
__global__ void __launch_bounds__(kThreads) gemv_f32_kernel(const __grid_constant__ GemvLaunch L) {
    extern __shared__ __align__(16) float smem[];
    __shared__ float inv_rms[TM];
    __shared__ float red_small[8 * TM];
    __shared__ int red_idx[8 * TM];
    __shared__ unsigned s_last;

    pdl_wait();
    pdl_trigger();
    const GemvProblem& P = L.b.p[blockIdx.z];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile = blockIdx.x, split = blockIdx.y;
    const int T = L.T, t0 = L.t0;
    const int n0 = tile * kTileN;
    const int k0 = split * L.kc;
    const int kn = min(P.K - k0, L.kc);

    // ---- prologue: fused RMSNorm of the input rows (proj/src/matrix.cpp:118-137)
    if (tid < TM) {
        float r = 1.f;
        if (P.gain != nullptr && tid < T) {
            float ss = 0.f;
            for (int i = 0; i < P.stat_tiles_in; ++i) ss += P.stats_in[(t0 + tid) * P.stat_tiles_in + i];
            const float ms = ss / (float)P.K;
            r = 1.0f / sqrtf(ms + P.eps);
        }
        inv_rms[tid] = r;
    }
    __syncthreads();

    float s[TM];
    {
        float* xs = smem;  // [kc][TM]
        for (int i = tid; i < kn * TM; i += kThreads) {
            const int kk = i / TM, t = i - kk * TM;
            float v = 0.f;
            if (t < T) {
                v = P.x[(size_t)(t0 + t) * P.ldx + k0 + kk];
                if (P.gain != nullptr) v = __fmul_rn(__fmul_rn(v, inv_rms[t]), P.gain[k0 + kk]);
            }
            xs[kk * TM + t] = v;
        }
        __syncthreads();

        // ---- main loop: stream W[k0:k0+kn, n0:n0+256]
        constexpr int U = 8;
        float acc[TM][8];
#pragma unroll
        for (int t = 0; t < TM; ++t)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[t][c] = 0.f;

        const int col = n0 + lane * 8;
        const bool col_ok = col < P.ldw;
        const float* Wb = reinterpret_cast<const float*>(P.W) + (size_t)k0 * P.ldw + col;
        for (int kk = warp; kk < kn; kk += 8 * U) {
            W8<float> w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = kk + 8 * u;
                if (k < kn && col_ok) w[u].load(Wb + (size_t)k * P.ldw);
                else w[u].zero();
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = kk + 8 * u;
                if (k < kn) {
                    float wf[8];
                    w[u].to_f32(wf);
                    const float* xr = xs + k * TM;
                    float xv[TM];
#pragma unroll
                    for (int t = 0; t < TM; ++t) xv[t] = xr[t];
#pragma unroll
                    for (int t = 0; t < TM; ++t)
#pragma unroll
                        for (int c = 0; c < 8; ++c) acc[t][c] = __fmaf_rn(xv[t], wf[c], acc[t][c]);
                }
            }
        }
        __syncthreads();  // xs no longer needed

        // ---- cross-warp reduction (fixed warp order)
        float* red = smem;  // [8][TM][256]
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            float4* dst = reinterpret_cast<float4*>(red + ((size_t)warp * TM + t) * kTileN + lane * 8);
            dst[0] = make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
            dst[1] = make_float4(acc[t][4], acc[t][5], acc[t][6], acc[t][7]);
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            float v = 0.f;
#pragma unroll
            for (int w = 0; w < 8; ++w) v += red[((size_t)w * TM + t) * kTileN + tid];
            s[t] = v;
        }
    }

    const int c = n0 + tid;  // this thread's output column
    if (L.splits > 1) {
        const size_t plane = (size_t)L.tiles * kTileN;
#pragma unroll
        for (int t = 0; t < TM; ++t)
            if (t < T) P.partial[((size_t)split * 16 + t) * plane + c] = s[t];
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const unsigned tk = atomicAdd(&P.tickets[tile], 1u);
            s_last = (tk == (unsigned)L.splits - 1) ? 1u : 0u;
            if (s_last) P.tickets[tile] = 0u;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            float v = 0.f;
            if (t < T)
                for (int sp = 0; sp < L.splits; ++sp) v += __ldcg(&P.partial[((size_t)sp * 16 + t) * plane + c]);
            s[t] = v;
        }
    }

    // ---- epilogues
    if constexpr (EPI == EPI_STORE) {
        if (c < P.N)
#pragma unroll
            for (int t = 0; t < TM; ++t)
                if (t < T) P.out[(size_t)(t0 + t) * P.ldo + c] = s[t];
    } else if constexpr (EPI == EPI_RESID) {
        // h_mid = h + attn  /  h_next = h_mid + mlp  (proj/src/draft_engine.cpp:15-19, 50-54)
        // row sum-of-squares partial per 32 columns (one warp)
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            float sq = 0.f;
            if (t < T && c < P.N) {
                const float y = __fadd_rn(P.resid[(size_t)(t0 + t) * P.ldr + c], s[t]);
                P.out[(size_t)(t0 + t) * P.ldo + c] = y;
                sq = y * y;
            }
            sq = warp_sum(sq);
            if (lane == 0 && t < T && c < P.N) P.stats_out[(t0 + t) * P.stat_tiles_out + c / 32] = sq;
        }
    } else if constexpr (EPI == EPI_SILU) {
        // packed group of 32 columns = [gate 16 | up 16]; gate = silu(x.Wg) * (x.Wu)
        // (proj/src/model.cpp:197-210)
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            const float up = __shfl_down_sync(0xffffffffu, s[t], 16);
            const int j = (c / 32) * 16 + lane;
            if (t < T && lane < 16 && j < P.N / 2) {
                const float g = s[t];
                const float si = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
                P.out[(size_t)(t0 + t) * P.ldo + j] = __fmul_rn(si, up);
            }
        }
    } else if constexpr (EPI == EPI_QKV) {
        // q = rope(h·Wq), k = rope(h·Wk), v = h·Wv; K/V written to the cache rows
        // of the pass (proj/src/model.cpp:130-138, rotary proj/src/matrix.cpp:159-194).
        const int qd = P.n_heads * P.dh, kd = P.n_kv * P.dh;
        const int region = c < qd ? 0 : (c < qd + kd ? 1 : 2);
        const int base = region == 0 ? 0 : (region == 1 ? qd : qd + kd);
        const int within = c - base;
        const int head = within / P.dh, i = within - head * P.dh;
        const int pair = i >> 1;
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            const float other = __shfl_xor_sync(0xffffffffu, s[t], 1);
            if (t >= T || c >= P.N) continue;
            float y = s[t];
            if (region < 2) {
                const float2 cs_sn = P.rope[(size_t)L.pass.pos[t0 + t] * (P.dh >> 1) + pair];
                const float cs = cs_sn.x, sn = cs_sn.y;
                const float x0 = (i & 1) ? other : s[t];
                const float x1 = (i & 1) ? s[t] : other;
                y = (i & 1) ? __fadd_rn(__fmul_rn(x0, sn), __fmul_rn(x1, cs))
                            : __fsub_rn(__fmul_rn(x0, cs), __fmul_rn(x1, sn));
            }
            if (region == 0) {
                P.out[(size_t)(t0 + t) * P.ldo + c] = y;
            } else {
                const long long off = kv_off(L.kv, P.layer, region - 1, head, L.pass.rows[t0 + t]) + i;
                if (L.kv.dtype == DT_BF16) st_f(reinterpret_cast<__nv_bfloat16*>(L.kv.pool) + off, y);
                else st_f(reinterpret_cast<float*>(L.kv.pool) + off, y);
            }
        }
    } else if constexpr (EPI == EPI_ARGMAX) {
        // logits = norm(h)·E^T ; greedy pick = first maximum (proj/src/matrix.cpp:196-202)
        float bv[TM];
        int bi[TM];
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            bv[t] = -INFINITY;
            bi[t] = 0x7fffffff;
            if (t < T && c < P.vocab) {
                if (P.logits) P.logits[(size_t)(t0 + t) * P.ld_logits + c] = s[t];
                bv[t] = s[t];
                bi[t] = c;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv[t], o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi[t], o);
                if (am_better(ov, oi, bv[t], bi[t])) { bv[t] = ov; bi[t] = oi; }
            }
            if (lane == 0) { red_small[warp * TM + t] = bv[t]; red_idx[warp * TM + t] = bi[t]; }
        }
        __syncthreads();
        if (tid < TM && tid < T) {
            float v = -INFINITY;
            int ix = 0x7fffffff;
            for (int w = 0; w < 8; ++w)
                if (am_better(red_small[w * TM + tid], red_idx[w * TM + tid], v, ix)) {
                    v = red_small[w * TM + tid];
                    ix = red_idx[w * TM + tid];
                }
            P.am_val[(t0 + tid) * L.tiles + tile] = v;
            P.am_idx[(t0 + tid) * L.tiles + tile] = ix;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const unsigned tk = atomicAdd(&P.tickets[L.tiles], 1u);
            s_last = (tk == (unsigned)L.tiles - 1) ? 1u : 0u;
            if (s_last) P.tickets[L.tiles] = 0u;
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (tid < TM && tid < T) {
            float v = -INFINITY;
            int ix = 0x7fffffff;
            for (int tl = 0; tl < L.tiles; ++tl) {
                const float ov = __ldcg(&P.am_val[(t0 + tid) * L.tiles + tl]);
                const int oi = __ldcg(&P.am_idx[(t0 + tid) * L.tiles + tl]);
                if (am_better(ov, oi, v, ix)) { v = ov; ix = oi; }
            }
            P.tok_out[t0 + tid] = ix + P.col_base;
            if (P.tok_val) P.tok_val[t0 + tid] = v;
        }
    }
}

template <int TM, int EPI>
static void gemv_launch_t(const GemvLaunch& L, int nprob, cudaStream_t s) {
    const size_t smem = sizeof(float) * (size_t)max(L.kc * TM, 8 * TM * kTileN);
    static unsigned long long configured = 0;
    ensure_smem((const void*)gemv_f32_kernel<TM, EPI>, 8 * 8 * kTileN * (int)sizeof(float), configured);
    dim3 grid(L.tiles, L.splits, nprob);
    CK(launch_pdl(gemv_f32_kernel<TM, EPI>, grid, dim3(kThreads), smem, s, L));
}

template <int EPI>
static void gemv_dispatch_tm(const GemvLaunch& L, int nprob, cudaStream_t s) {
    if (L.T <= 1) gemv_launch_t<1, EPI>(L, nprob, s);
    else if (L.T <= 2) gemv_launch_t<2, EPI>(L, nprob, s);
    else if (L.T <= 4) gemv_launch_t<4, EPI>(L, nprob, s);
    else gemv_launch_t<8, EPI>(L, nprob, s);
}

int gemv_rows_per_launch(int wdtype) { return wdtype == DT_BF16 ? 16 : 8; }

static thread_local bool g_prefill = false;
void set_prefill_mode(bool on) {
    static const bool enabled = [] {
        const char* e = getenv("ESPEC_TC_PREFILL");
        return e == nullptr || atoi(e) != 0;
    }();
    g_prefill = on && enabled;
}

size_t gemv_partial_floats(int K, int N, int wdtype) {
    if (wdtype == DT_BF16) return sgemv_partial_floats(K, (N + 31) / 32 * 32);
    const GemvPlan p = gemv_plan(K, N);
    return (size_t)p.splits * 16 * (size_t)p.tiles * kTileN;
}

int gemv_col_tiles(int K, int N, int wdtype) {
    if (wdtype == DT_BF16) return (N + 31) / 32;
    return gemv_plan(K, N).tiles;
}

bool gemv_fused_push_ok(int wdtype, int T) { return wdtype == DT_BF16 && !(g_prefill && T > 16); }

void launch_gemv(int epi, int wdtype, const GemvBatch& b, int nprob, int T, const PassView& pass,
                 const KvView& kv, cudaStream_t s, SgPool* pool) {
    if (T <= 0 || nprob <= 0) return;
    if (wdtype == DT_BF16) {
        if (g_prefill && T > 16 && epi != EPI_ARGMAX && b.p[0].tc_xa != nullptr) {
            for (int i = 0; i < nprob; ++i) launch_tc_gemm(epi, b.p[i], T, pass, kv, b.p[i].tc_xa, b.p[i].tc_rms, s);
            return;
        }
        launch_sgemv(epi, b, nprob, T, pass, kv, s, pool);
        return;
    }
    GemvLaunch L;
    L.b = b;
    L.pass = pass;
    L.kv = kv;
    const GemvPlan plan = gemv_plan(b.p[0].K, b.p[0].N);
    L.tiles = plan.tiles;
    L.splits = plan.splits;
    L.kc = plan.kc;
    const int rows = gemv_rows_per_launch(wdtype);
    for (int t0 = 0; t0 < T; t0 += rows) {
        L.t0 = t0;
        L.T = min(rows, T - t0);
        switch (epi) {
            case EPI_STORE: gemv_dispatch_tm<EPI_STORE>(L, nprob, s); break;
            case EPI_RESID: gemv_dispatch_tm<EPI_RESID>(L, nprob, s); break;
            case EPI_SILU: gemv_dispatch_tm<EPI_SILU>(L, nprob, s); break;
            case EPI_QKV: gemv_dispatch_tm<EPI_QKV>(L, nprob, s); break;
            case EPI_ARGMAX: gemv_dispatch_tm<EPI_ARGMAX>(L, nprob, s); break;
        }
    }
}

// Pre-packed bf16 layout = the tcgen05 / UMMA canonical K-major
// "interleave" (no-swizzle) layout, tiled per 32-column group:
//   element (k, n) lives at (g*KT + kt)*512 + (n8*2 + kh)*64 + r*8 + c
// with g = n/32, kt = k/16, n8 = (n%32)/8, kh = (k%16)/8, r = n%8, c = k%8.
// A 1 KB block (g, kt) is eight 8x8 core matrices (8 n-rows x 16 bytes of
// consecutive k): its two k-halves of one n8 tile are adjacent (LBO 128 B)
// and n8 tiles are 256 B apart (SBO), so consecutive groups' blocks laid
// side by side in shared memory form one uniform K-major UMMA operand tile
// (prefill tcgen05 GEMM), while a decode warp gets its mma.sync B fragments
// for two n8 tiles with one ldmatrix.x4 at block + lane*16.
__host__ __device__ __forceinline__ size_t pack_index(int k, int n, int KT) {
    const int g = n >> 5, n8 = (n & 31) >> 3, r = n & 7;
    const int kt = k >> 4, kh = (k & 15) >> 3, c = k & 7;
    return ((size_t)g * KT + kt) * 512 + (n8 * 2 + kh) * 64 + r * 8 + c;
}

__global__ void pack_kernel(const __nv_bfloat16* src, int K, int ldw, __nv_bfloat16* dst, int unpack) {
    const int KT = (K + 15) / 16;
    const long long total = (long long)KT * 16 * ldw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(i / ldw), n = (int)(i - (long long)k * ldw);
        const size_t p = pack_index(k, n, KT);
        if (unpack) {
            if (k < K) dst[i] = src[p];
        } else {
            dst[p] = k < K ? src[i] : __float2bfloat16_rn(0.f);
        }
    }
}

size_t packed_elems(int K, int ldw) { return (size_t)((K + 15) / 16) * 16 * (size_t)ldw; }

void launch_pack(const void* logical, int K, int ldw, void* packed, bool unpack, cudaStream_t s) {
    pack_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(unpack ? packed : logical), K, ldw,
                                        reinterpret_cast<__nv_bfloat16*>(unpack ? const_cast<void*>(logical) : packed),
                                        unpack ? 1 : 0);
}

// ---------------------------------------------------------------------------
// embedding gather / residual add (+ row sum-of-squares partials)
// ---------------------------------------------------------------------------

// Row sum-of-squares partials are one per 32 columns (one warp): the same
// granularity the GEMV epilogues write, so the consumer's RMSNorm prologue
// sums them in the same fixed order whatever produced the row.
template <typename WT>
__global__ void __launch_bounds__(kThreads) embed_kernel(const WT* emb, int d, const int* arena, const int* idx,
                                                        float* h, float* stats, int stat_tiles) {
    pdl_wait();
    pdl_trigger();
    const int t = blockIdx.y, c = blockIdx.x * kThreads + threadIdx.x;
    const int tok = arena[idx[t]];
    float v = 0.f;
    if (c < d) {
        v = ld_f(emb + (size_t)tok * d + c);
        h[(size_t)t * d + c] = v;
    }
    const float sq = warp_sum(v * v);
    if ((threadIdx.x & 31) == 0 && c < d) stats[t * stat_tiles + c / kStatTile] = sq;
}

void launch_embed(int wdtype, const void* emb, int d, const int* arena, const int* idx, int T, float* h,
                  float* stats, cudaStream_t s) {
    if (T <= 0) return;
    dim3 grid((d + kThreads - 1) / kThreads, T);
    const int st = (d + kStatTile - 1) / kStatTile;
    if (wdtype == DT_BF16)
        CK(launch_pdl(embed_kernel<__nv_bfloat16>, grid, dim3(kThreads), 0, s,
                      reinterpret_cast<const __nv_bfloat16*>(emb), d, arena, idx, h, stats, st));
    else
        CK(launch_pdl(embed_kernel<float>, grid, dim3(kThreads), 0, s, reinterpret_cast<const float*>(emb), d, arena,
                      idx, h, stats, st));
}

__global__ void __launch_bounds__(kThreads) add_stats_kernel(float* h, const float* a, int d, float* stats,
                                                            int stat_tiles) {
    pdl_wait();
    pdl_trigger();
    const int t = blockIdx.y, c = blockIdx.x * kThreads + threadIdx.x;
    float y = 0.f;
    if (c < d) {
        y = __fadd_rn(h[(size_t)t * d + c], a[(size_t)t * d + c]);
        h[(size_t)t * d + c] = y;
    }
    const float sq = warp_sum(y * y);
    if ((threadIdx.x & 31) == 0 && c < d) stats[t * stat_tiles + c / kStatTile] = sq;
}

void launch_add_stats(float* h, const float* a, int d, int T, float* stats, cudaStream_t s) {
    if (T <= 0) return;
    dim3 grid((d + kThreads - 1) / kThreads, T);
    CK(launch_pdl(add_stats_kernel, grid, dim3(kThreads), 0, s, h, a, d, stats, (d + kStatTile - 1) / kStatTile));
}

// ---------------------------------------------------------------------------
// attention over the paged cache with a tree-aware mask
// (proj/src/model.cpp:140-192; mask semantics proj/src/kv_cache.cpp:43-60)
// ---------------------------------------------------------------------------

constexpr int kAttnRows = 64;    // key rows per split (fixed: independent of T)
constexpr int kAttnPairs = 64;   // (query, head) pairs per CTA
constexpr int kAttnThreads = 128;

size_t attn_ws_floats(int T, int n_heads, int dh, int max_rows) {
    const size_t splits = (size_t)(max_rows + kAttnRows - 1) / kAttnRows;
    // covers both layouts: fp32 [split][n_kv][T*G][dh+2] and bf16 mma
    // [chunk][n_kv * mtiles][16][dh+4]
    // tcgen05 kernel: [chunk][n_kv * pair groups][128][dh + 4], at most
    // T * H + 128 * H rows per chunk (chunks <= splits)
    return splits * (size_t)(T * n_heads + 128 * n_heads) * (dh + 4);
}
int attn_pages_per_item(int cap) {
    static const int forced = [] {
        const char* e = std::getenv("ESPEC_ATTN_PPI");
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return forced;
    // tcgen05 attention (attn_tc.cu), measured (profiles/r2_attn_tc.txt): 2 pages
    // per CTA at short context, 4-8 as the context grows (fewer chunk partials
    // for the combine kernel, pages processed two per softmax step)
    return cap <= 2048 ? 2 : cap <= 4096 ? 4 : cap <= 32768 ? 8 : 16;
}

size_t attn_tickets(int T, int n_heads, int n_kv) {
    const int G = n_heads / n_kv;
    const int pb = (T * G + 15) / 16;  // >= the fp32 kernel's 64-pair blocks
    return (size_t)n_kv * pb;
}

struct AttnLaunch {
    AttnBatch b;
    PassView pass;
    KvView kv;
    int n_heads, G, splits, pblocks;
};

template <typename KT>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(const __grid_constant__ AttnLaunch L) {
    extern __shared__ __align__(16) float sm[];
    __shared__ unsigned s_last;
    pdl_wait();
    pdl_trigger();
    const AttnProblem& A = L.b.p[blockIdx.z];
    const int dh = L.kv.dh, G = L.G, H = L.n_heads;
    const int split = blockIdx.x;
    const int hk = blockIdx.y % L.kv.n_kv, pb = blockIdx.y / L.kv.n_kv;
    const int T = L.pass.T;
    const int P0 = pb * kAttnPairs;
    const int NP = min(kAttnPairs, T * G - P0);
    const int j0 = split * kAttnRows;
    const int nr = max(0, min(kAttnRows, L.pass.total - j0));
    const int ld = dh + 1;
    float* qs = sm;                          // [64][dh+1]
    float* ks = qs + kAttnPairs * ld;        // [64][dh+1] (K, then V)
    float* sc = ks + kAttnRows * ld;         // [64 pairs][64 rows]
    const int tid = threadIdx.x;
    const KT* pool = reinterpret_cast<const KT*>(L.kv.pool);

    for (int i = tid; i < NP * dh; i += kAttnThreads) {
        const int p = i / dh, d = i - p * dh;
        const int pp = P0 + p, t = pp / G, g = pp - t * G;
        qs[p * ld + d] = A.q[(size_t)t * H * dh + (hk * G + g) * dh + d];
    }
    for (int i = tid; i < nr * dh; i += kAttnThreads) {
        const int r = i / dh, d = i - r * dh;
        ks[r * ld + d] = ld_f(pool + kv_off(L.kv, A.layer, 0, hk, j0 + r) + d);
    }
    __syncthreads();
    // scores: thread block = 4 pairs x 8 rows
    const float inv_sqrt = 1.0f / sqrtf((float)dh);
    {
        const int pi = tid >> 3, ji = tid & 7;
        float a[4][8];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) a[x][y] = 0.f;
        if (pi * 4 < NP) {
            for (int d = 0; d < dh; ++d) {
                float qv[4], kv8[8];
#pragma unroll
                for (int x = 0; x < 4; ++x) qv[x] = qs[(pi * 4 + x) * ld + d];
#pragma unroll
                for (int y = 0; y < 8; ++y) kv8[y] = ks[(ji + 8 * y) * ld + d];
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 8; ++y) a[x][y] = __fmaf_rn(qv[x], kv8[y], a[x][y]);
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const int p = pi * 4 + x;
                if (p >= NP) continue;
                const int t = (P0 + p) / G;
#pragma unroll
                for (int y = 0; y < 8; ++y) {
                    const int r = ji + 8 * y;
                    const bool ok = r < nr && visible(L.pass, t, j0 + r);
                    sc[p * kAttnRows + r] = ok ? __fmul_rn(a[x][y], inv_sqrt) : -INFINITY;
                }
            }
        }
    }
    __syncthreads();
    // load V over K
    for (int i = tid; i < nr * dh; i += kAttnThreads) {
        const int r = i / dh, d = i - r * dh;
        ks[r * ld + d] = ld_f(pool + kv_off(L.kv, A.layer, 1, hk, j0 + r) + d);
    }
    // per pair: max, exp, sum (one warp per pair, lanes over rows)
    __shared__ float pm[kAttnPairs], pl[kAttnPairs];
    const int warp = tid >> 5, lane = tid & 31;
    for (int p = warp; p < NP; p += kAttnThreads / 32) {
        float v0 = lane < nr ? sc[p * kAttnRows + lane] : -INFINITY;
        float v1 = lane + 32 < nr ? sc[p * kAttnRows + lane + 32] : -INFINITY;
        const float m = warp_max(fmaxf(v0, v1));
        float e0 = 0.f, e1 = 0.f;
        if (m != -INFINITY) {
            e0 = v0 == -INFINITY ? 0.f : expf(v0 - m);
            e1 = v1 == -INFINITY ? 0.f : expf(v1 - m);
        }
        sc[p * kAttnRows + lane] = e0;
        sc[p * kAttnRows + lane + 32] = e1;
        const float l = warp_sum(e0 + e1);
        if (lane == 0) { pm[p] = m; pl[p] = l; }
    }
    __syncthreads();
    // O[p][d] = sum_r e[p][r] v[r][d]
    const size_t pair_stride = (size_t)dh + 2;
    float* wsb = A.ws + (((size_t)split * L.kv.n_kv + hk) * (size_t)(T * G)) * pair_stride;
    for (int i = tid; i < NP * dh; i += kAttnThreads) {
        const int p = i / dh, d = i - p * dh;
        float o = 0.f;
        for (int r = 0; r < nr; ++r) o = __fmaf_rn(sc[p * kAttnRows + r], ks[r * ld + d], o);
        wsb[(size_t)(P0 + p) * pair_stride + d] = o;
    }
    for (int p = tid; p < NP; p += kAttnThreads) {
        wsb[(size_t)(P0 + p) * pair_stride + dh] = pm[p];
        wsb[(size_t)(P0 + p) * pair_stride + dh + 1] = pl[p];
    }
    // last split combines (fixed split order)
    __threadfence();
    __syncthreads();
    unsigned* ticket = A.tickets + blockIdx.y;
    if (tid == 0) {
        const unsigned tk = atomicAdd(ticket, 1u);
        s_last = (tk == (unsigned)L.splits - 1) ? 1u : 0u;
        if (s_last) *ticket = 0u;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const size_t split_stride = (size_t)L.kv.n_kv * (size_t)(T * G) * pair_stride;
    const float* wsh = A.ws + (size_t)hk * (size_t)(T * G) * pair_stride;
    for (int i = tid; i < NP * dh; i += kAttnThreads) {
        const int p = i / dh, d = i - p * dh;
        const size_t po = (size_t)(P0 + p) * pair_stride;
        float M = -INFINITY;
        for (int sp = 0; sp < L.splits; ++sp) M = fmaxf(M, __ldcg(wsh + sp * split_stride + po + dh));
        float num = 0.f, den = 0.f;
        if (M != -INFINITY)
            for (int sp = 0; sp < L.splits; ++sp) {
                const float m = __ldcg(wsh + sp * split_stride + po + dh);
                if (m == -INFINITY) continue;
                const float f = expf(m - M);
                num = __fmaf_rn(f, __ldcg(wsh + sp * split_stride + po + d), num);
                den = __fmaf_rn(f, __ldcg(wsh + sp * split_stride + po + dh + 1), den);
            }
        const int pp = P0 + p, t = pp / G, g = pp - t * G;
        A.out[(size_t)t * H * dh + (hk * G + g) * dh + d] = den > 0.f ? num / den : 0.f;
    }
}

// ---------------------------------------------------------------------------
// bf16 KV: tensor-core split-KV attention (mma.sync m16n8k16).
// CTA = 4 warps = 4 consecutive 64-row key splits (one KV page each) of one
// kv head and one 16-pair m-tile ((query, q-head) pairs of the GQA group).
// Per warp: S = Q K^T (ldmatrix K from smem), masked online softmax in
// registers, O = P V (P re-used from the S accumulators as the A operand,
// ldmatrix.trans V). Warps combine in shared memory; CTAs along the context
// combine through a split workspace, last CTA in fixed order.
// ---------------------------------------------------------------------------

static bool attn_tc_path(const KvView& kv) {
    return kv.dtype == DT_BF16 && kv.page_rows == 64 && (kv.dh == 64 || kv.dh == 128);
}
int attention_launches(const PassView& pass, const KvView& kv, int n_heads, int nprob) {
    if (!attn_tc_path(kv)) return 1;
    const int pages = (pass.total + 63) / 64;
    const int ppi = attn_tc_ppi(pass, kv, n_heads, nprob);
    const int chunks = (pages + ppi - 1) / ppi;
    return chunks > 1 && !attn_tc_cluster(chunks, pass.T) ? 2 : 1;
}

void launch_attention(const AttnBatch& b, int nprob, int n_heads, const PassView& pass, const KvView& kv,
                      cudaStream_t s) {
    if (pass.T <= 0 || nprob <= 0) return;
    AttnLaunch L;
    L.b = b;
    L.pass = pass;
    L.kv = kv;
    L.n_heads = n_heads;
    L.G = n_heads / kv.n_kv;
    L.splits = (pass.total + kAttnRows - 1) / kAttnRows;
    L.pblocks = (pass.T * L.G + kAttnPairs - 1) / kAttnPairs;
    const size_t smem = sizeof(float) * ((size_t)(kAttnPairs + kAttnRows) * (kv.dh + 1) + kAttnPairs * kAttnRows);
    static unsigned long long configured[2] = {0, 0};
    dim3 grid(L.splits, kv.n_kv * L.pblocks, nprob);
    if (attn_tc_path(kv)) {
        launch_attention_tc(b, nprob, n_heads, pass, kv, s);
    } else if (kv.dtype == DT_BF16) {
        ensure_smem((const void*)attn_kernel<__nv_bfloat16>, 200 * 1024, configured[1]);
        CK(launch_pdl(attn_kernel<__nv_bfloat16>, grid, dim3(kAttnThreads), smem, s, L));
    } else {
        ensure_smem((const void*)attn_kernel<float>, 200 * 1024, configured[0]);
        CK(launch_pdl(attn_kernel<float>, grid, dim3(kAttnThreads), smem, s, L));
    }
}

// ---------------------------------------------------------------------------
// KV commit compaction (proj/src/kv_cache.cpp:62-94)
// ---------------------------------------------------------------------------

template <typename KT>
__global__ void kv_move_kernel(KvView kv, const int* src, const int* dst, int n) {
    // grid: (layer*2+kind, kv head); sequential over the path keeps the
    // reference's in-order memcpy semantics (dst <= src, ascending).
    pdl_wait();
    pdl_trigger();
    const int lk = blockIdx.x, head = blockIdx.y;
    const int layer = lk >> 1, kind = lk & 1;
    KT* pool = reinterpret_cast<KT*>(kv.pool);
    for (int i = 0; i < n; ++i) {
        if (src[i] == dst[i]) continue;
        const long long so = kv_off(kv, layer, kind, head, src[i]);
        const long long dof = kv_off(kv, layer, kind, head, dst[i]);
        for (int d = threadIdx.x; d < kv.dh; d += blockDim.x) pool[dof + d] = pool[so + d];
        __syncthreads();
    }
}

void launch_kv_move(const KvView& kv, const int* src, const int* dst, int n, cudaStream_t s) {
    if (n <= 0) return;
    dim3 grid(kv.n_layers * 2, kv.n_kv);
    if (kv.dtype == DT_BF16) CK(launch_pdl(kv_move_kernel<__nv_bfloat16>, grid, dim3(128), 0, s, kv, src, dst, n));
    else CK(launch_pdl(kv_move_kernel<float>, grid, dim3(128), 0, s, kv, src, dst, n));
}

// ---------------------------------------------------------------------------
// greedy acceptance (proj/src/verifier.cpp:86-177 at temperature 0)
// ---------------------------------------------------------------------------

__global__ void accept_greedy_kernel(AcceptArgs a) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x != 0) return;
    int target = a.base_argmax[0];
    int parent = -1, m = 0;
    for (int depth = 1; depth <= a.n_levels; ++depth) {
        const int first = parent < 0 ? 0 : a.node_first_child[parent];
        const int count = parent < 0 ? a.root_children : a.node_n_children[parent];
        if (count == 0) break;
        int acc = -1;
        // Greedy siblings: accept the sibling equal to the base argmax. (The
        // reference throws when a rejected first sibling exhausts the one-hot
        // draft distribution, proj/src/verifier.cpp:156-157; with one sibling
        // per level both rules coincide.)
        for (int i = 0; i < count; ++i) {
            const int ni = first + i;
            if (a.tok_arena[a.node_tok_idx[ni]] == target) {
                acc = ni;
                break;
            }
            if (a.strict_siblings && i + 1 < count) {
                if (a.err) *a.err = 4;  // "sibling candidates exhaust the draft distribution"
                break;
            }
        }
        if (acc < 0) break;
        a.outcome[2 + m] = acc;
        a.outcome[2 + a.n_levels + m] = a.tok_arena[a.node_tok_idx[acc]];
        a.tok_arena_w[a.commit_at + m] = a.tok_arena[a.node_tok_idx[acc]];
        ++m;
        target = a.base_argmax[1 + acc];
        parent = acc;
    }
    a.outcome[0] = m;
    a.outcome[1] = target;
    a.tok_arena_w[a.commit_at + m] = target;
}

void launch_accept_greedy(const AcceptArgs& a, cudaStream_t s) { CK(launch_pdl(accept_greedy_kernel, dim3(1), dim3(32), 0, s, a)); }

// ---------------------------------------------------------------------------
// perf-mode weight init: N(0, sd) from a counter-based hash (Box-Muller)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_normal_kernel(T* dst, long long n, float sd, uint64_t seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint64_t h1 = mix64(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)i * 2 + 1);
        const uint64_t h2 = mix64(h1 + 0x632BE59BD9B4E019ULL);
        const float u1 = ((h1 >> 40) + 0.5f) * (1.0f / 16777216.0f);
        const float u2 = (h2 >> 40) * (1.0f / 16777216.0f);
        const float r = sqrtf(-2.0f * __logf(u1));
        st_f(dst + i, r * __cosf(6.283185307f * u2) * sd);
    }
}

template <typename T>
__global__ void fill_const_kernel(T* dst, long long n, float v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        st_f(dst + i, v);
}

void launch_fill_normal(int dtype, void* dst, long long n, float sd, uint64_t seed, cudaStream_t s) {
    const int blocks = 148 * 8;
    if (dtype == DT_BF16) fill_normal_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<__nv_bfloat16*>(dst), n, sd, seed);
    else fill_normal_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<float*>(dst), n, sd, seed);
}

// Sharded N(0, sd) fill: element (k, c) of this rank's K x ld block takes
// the value of global element (k + row_off, gcol(c)) of the full logical
// matrix (K_full x N_full), so every TP degree holds slices of one model.
template <typename T>
__global__ void fill_normal_map_kernel(T* dst, int K, int ld, ColMap m, int row_off, long long n_full, float sd) {
    const long long total = (long long)K * ld;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(i / ld), c = (int)(i - (long long)k * ld);
        long long g = -1;
        uint64_t seed = m.seed;
        if (m.gateup) {
            // packed [gate16 | up16] per 32 local columns
            const int j = (c >> 5) * 16 + (c & 15);
            if (j < m.f_loc) {
                g = (long long)m.f_base + j;
                if (c & 16) seed = m.seed2;
            }
        } else {
            for (int q = 0; q < m.nseg; ++q)
                if (c >= m.lc0[q] && c < m.lc0[q] + m.len[q]) g = m.gc0[q] + (c - m.lc0[q]);
        }
        float v = 0.f;
        if (g >= 0) {
            const uint64_t idx = (uint64_t)(k + row_off) * (uint64_t)n_full + (uint64_t)g;
            const uint64_t h1 = mix64(seed * 0x9E3779B97F4A7C15ULL + idx * 2 + 1);
            const uint64_t h2 = mix64(h1 + 0x632BE59BD9B4E019ULL);
            const float u1 = ((h1 >> 40) + 0.5f) * (1.0f / 16777216.0f);
            const float u2 = (h2 >> 40) * (1.0f / 16777216.0f);
            v = sqrtf(-2.0f * __logf(u1)) * __cosf(6.283185307f * u2) * sd;
        }
        st_f(dst + i, v);
    }
}

void launch_fill_normal_map(int dtype, void* dst, int K, int ld, const ColMap& m, int row_off, long long n_full,
                            float sd, cudaStream_t s) {
    const int blocks = 148 * 8;
    if (dtype == DT_BF16)
        fill_normal_map_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<__nv_bfloat16*>(dst), K, ld, m, row_off, n_full, sd);
    else
        fill_normal_map_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<float*>(dst), K, ld, m, row_off, n_full, sd);
}

void launch_fill_const(int dtype, void* dst, long long n, float v, cudaStream_t s) {
    const int blocks = 148 * 4;
    if (dtype == DT_BF16) fill_const_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<__nv_bfloat16*>(dst), n, v);
    else fill_const_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<float*>(dst), n, v);
}

template <typename T>
__global__ void transpose_kernel(const T* src, int rows, int cols, T* dst, int ldd) {
    __shared__ T tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = src[(size_t)r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[(size_t)c * ldd + r] = tile[threadIdx.x][i];
    }
}

void launch_transpose(int dtype, const void* src, int rows, int cols, void* dst, int ldd, cudaStream_t s) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
    if (dtype == DT_BF16)
        transpose_kernel<<<grid, block, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(src), rows, cols,
                                                 reinterpret_cast<__nv_bfloat16*>(dst), ldd);
    else
        transpose_kernel<<<grid, block, 0, s>>>(reinterpret_cast<const float*>(src), rows, cols,
                                                 reinterpret_cast<float*>(dst), ldd);
}

}  // namespace espec_dev
