// Prompt-prefill GEMM on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Prefill is the one place on the EasySpec path where M (prompt rows) is a
// real contraction dimension: 256-row chunks of
// the prompt through every projection of both models. Decode passes (M <= 16)
// stay on the HBM-streaming GEMV (gemv_stream.cu).
//
// One CTA computes a 128 x 256 output tile over all of K:
//   warp 0  TMA producer: 1-D bulk copies of the A tile (16 KB: 128 rows x 64 k,
//           pre-packed by pack_a_kernel) and of eight 1 KB weight blocks per
//           k-step (32 KB) into a 4-stage shared-memory ring (mbarrier
//           complete_tx);
//   warp 1  allocates 256 TMEM columns; lane 0 issues tcgen05.mma
//           (kind::f16, M=128, N=256, K=16, fp32 accumulate in TMEM) — four per
//           stage — and releases each stage with tcgen05.commit;
//   warps 2-5 epilogue: tcgen05.ld 32 columns at a time (each thread one row),
//           then the same fused epilogues as the decode GEMV (residual + row
//           statistics, SiLU(gate)*up, RoPE + paged-KV write, store).
// Operands are UMMA canonical K-major "interleave" tiles: the weights are
// stored that way in HBM (kernels.cu pack_index) and a k-step's eight 1 KB
// group blocks placed side by side form one N=256 operand (LBO 128 B between
// the two k-halves of a core matrix column, SBO 256 B between 8-row core
// matrices); A uses the same layout for its 128 rows.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace espec_dev {

constexpr int kTcM = 128;
constexpr int kTcN = 256;             // 8 x 32-column weight groups
constexpr int kTcKStep = 16;          // one tcgen05.mma (bf16)
constexpr int kTcStepsPerStage = 4;   // 64 k per stage
constexpr int kTcStages = 4;
constexpr int kTcAStage = kTcM * kTcKStep * kTcStepsPerStage * 2;  // 16 KB
constexpr int kTcBStage = kTcN * kTcKStep * kTcStepsPerStage * 2;  // 32 KB
constexpr int kTcStageBytes = kTcAStage + kTcBStage;
constexpr int kTcThreads = 6 * 32;

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tc_mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(b)), "r"(n));
}
__device__ __forceinline__ void tc_mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            tc_smem(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tc_smem(dst)),
                 "l"(src), "r"(bytes), "r"(tc_smem(bar))
                 : "memory");
}
// UMMA shared-memory descriptor, K-major SWIZZLE_NONE (CuTe UMMA::SmemDescriptor):
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), layout 0.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor: D f32, A/B bf16, both K-major, N=256, M=128
constexpr uint32_t kTcIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

struct TcLaunch {
    GemvProblem P;
    PassView pass;
    KvView kv;
    int t0, T;       // rows [t0, t0+T) of the pass
    int KS;          // k-steps (K/16, K padded to 16)
    int mtiles;
    const __nv_bfloat16* xa;  // packed A: [mtile][KS][16 m8][2 kh][8 rows][8] bf16
};

// epilogue for one (row, 32-column group): v = 32 fp32 sums of that row
template <int EPI>
__device__ __forceinline__ void tc_epilogue(const TcLaunch& L, int t, int g, const float (&v)[32]) {
    const GemvProblem& P = L.P;
    const int c0 = g * 32;
    if constexpr (EPI == EPI_STORE) {
        float* o = P.out + (size_t)t * P.ldo + c0;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (c0 + j < P.N) o[j] = v[j];
    } else if constexpr (EPI == EPI_RESID) {
        float* o = P.out + (size_t)t * P.ldo + c0;
        const float* r = P.resid + (size_t)t * P.ldr + c0;
        float sq = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (c0 + j < P.N) {
                const float y = __fadd_rn(r[j], v[j]);
                o[j] = y;
                sq = __fmaf_rn(y, y, sq);
            }
        P.stats_out[t * P.stat_tiles_out + g] = sq;
    } else if constexpr (EPI == EPI_SILU) {
        float* o = P.out + (size_t)t * P.ldo + g * 16;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (g * 16 + j < P.N / 2) o[j] = __fmul_rn(__fdiv_rn(v[j], __fadd_rn(1.0f, expf(-v[j]))), v[16 + j]);
    } else if constexpr (EPI == EPI_QKV) {
        const int qd = P.n_heads * P.dh, kd = P.n_kv * P.dh;
        const int pos = L.pass.pos[t];
        const int row = L.pass.rows[t];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const int c = c0 + j;
            if (c >= P.N) break;
            const int region = c < qd ? 0 : (c < qd + kd ? 1 : 2);
            const int base = region == 0 ? 0 : (region == 1 ? qd : qd + kd);
            const int within = c - base;
            const int head = within / P.dh, i = within - head * P.dh;
            float y0 = v[j], y1 = v[j + 1];
            if (region < 2) {
                const double inv_freq = pow((double)P.rope_theta, -2.0 * (i >> 1) / (double)P.dh);
                const double th = (double)pos * inv_freq;
                const float cs = (float)cos(th), sn = (float)sin(th);
                y0 = __fsub_rn(__fmul_rn(v[j], cs), __fmul_rn(v[j + 1], sn));
                y1 = __fadd_rn(__fmul_rn(v[j], sn), __fmul_rn(v[j + 1], cs));
            }
            if (region == 0) {
                P.out[(size_t)t * P.ldo + c] = y0;
                P.out[(size_t)t * P.ldo + c + 1] = y1;
            } else {
                const KvView& kv = L.kv;
                const int page = kv.page_table[row / kv.page_rows];
                const long long off = (long long)page * kv.page_elems +
                                      ((((long long)P.layer * 2 + (region - 1)) * kv.n_kv + head) * kv.page_rows +
                                       row % kv.page_rows) * kv.dh + i;
                if (kv.dtype == DT_BF16) {
                    *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(kv.pool) + off) =
                        __floats2bfloat162_rn(y0, y1);
                } else {
                    float* kp = reinterpret_cast<float*>(kv.pool) + off;
                    kp[0] = y0;
                    kp[1] = y1;
                }
            }
        }
    }
}

template <int EPI>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gemm_kernel(const __grid_constant__ TcLaunch L) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages], acc_bar;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntile = blockIdx.x, mt = blockIdx.y;
    const int g0 = ntile * (kTcN / 32);
    const int KS = L.KS;
    const int n_stages_total = (KS + kTcStepsPerStage - 1) / kTcStepsPerStage;
    const int ngroups = L.P.ldw / 32;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            tc_mbar_init(&full_bar[s], 1);
            tc_mbar_init(&empty_bar[s], 1);
        }
        tc_mbar_init(&acc_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&tmem_base)),
                     "r"(kTcN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ---------------- producer (weights need no dependency; A does)
        if (lane == 0) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            const char* A = reinterpret_cast<const char*>(L.xa) + (size_t)mt * KS * (kTcM * kTcKStep * 2);
            const char* B = reinterpret_cast<const char*>(L.P.W);
            const size_t KT = (size_t)KS;  // weight k-blocks per group (K padded to 16)
            for (int st = 0; st < n_stages_total; ++st) {
                const int s = st % kTcStages;
                const uint32_t ph = (uint32_t)(st / kTcStages) & 1u;
                tc_mbar_wait(&empty_bar[s], ph ^ 1u);
                const int ks0 = st * kTcStepsPerStage;
                const int nks = min(kTcStepsPerStage, KS - ks0);
                int ng = min(kTcN / 32, ngroups - g0);
                tc_mbar_expect(&full_bar[s], (uint32_t)(nks * (kTcM * kTcKStep * 2) + nks * ng * 1024));
                unsigned char* sa = sm + (size_t)s * kTcStageBytes;
                unsigned char* sb = sa + kTcAStage;
                tc_bulk(sa, A + (size_t)ks0 * (kTcM * kTcKStep * 2), (uint32_t)(nks * kTcM * kTcKStep * 2), &full_bar[s]);
                for (int k = 0; k < nks; ++k)
                    for (int gl = 0; gl < ng; ++gl)
                        tc_bulk(sb + (size_t)k * (kTcN / 32) * 1024 + gl * 1024,
                                B + (((size_t)(g0 + gl)) * KT + ks0 + k) * 1024, 1024u, &full_bar[s]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread)
        if (lane == 0) {
            const uint32_t d = tmem_base;
            for (int st = 0; st < n_stages_total; ++st) {
                const int s = st % kTcStages;
                tc_mbar_wait(&full_bar[s], (uint32_t)(st / kTcStages) & 1u);
                tc_fence_after();
                const int ks0 = st * kTcStepsPerStage;
                const int nks = min(kTcStepsPerStage, KS - ks0);
                const uint32_t sa = tc_smem(sm + (size_t)s * kTcStageBytes);
                const uint32_t sb = sa + kTcAStage;
                for (int k = 0; k < nks; ++k) {
                    const uint64_t da = umma_desc(sa + k * (kTcM * kTcKStep * 2), 128, 256);
                    const uint64_t db = umma_desc(sb + k * (kTcN / 32) * 1024, 128, 256);
                    const uint32_t acc = (st > 0 || k > 0) ? 1u : 0u;
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                        "l"(da), "l"(db), "r"(kTcIdesc), "r"(acc));
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    tc_smem(&empty_bar[s])));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                tc_smem(&acc_bar)));
        }
    } else {
        // ---------------- epilogue warps 2..5: TMEM lanes 32*(warp%4) ..
        asm volatile("griddepcontrol.wait;" ::: "memory");
        tc_mbar_wait(&acc_bar, 0);
        tc_fence_after();
        const int lane_base = 32 * (warp & 3);
        const int r = lane_base + lane;            // row within the tile
        const int t = L.t0 + mt * kTcM + r;        // pass row
        const bool ok = mt * kTcM + r < L.T;
        const int ng = min(kTcN / 32, ngroups - g0);
        for (int gl = 0; gl < ng; ++gl) {
            uint32_t u[32];
            const uint32_t taddr = tmem_base + ((uint32_t)lane_base << 16) + (uint32_t)(gl * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
                  "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]),
                  "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]),
                  "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]),
                  "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(u[j]);
            if (ok) tc_epilogue<EPI>(L, t, g0 + gl, v);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcN));
    }
}

// ---------------------------------------------------------------------------
// A packing: rows [t0, t0+T) of x (fp32), RMSNorm'd with `gain` from the
// per-32-column statistics when gain != nullptr, to bf16 canonical tiles
// [mtile][KS][m8][kh][8 rows][8 k]; rows >= T are zero.
// ---------------------------------------------------------------------------

__global__ void tc_rms_kernel(GemvProblem P, int t0, int T, float* inv_rms) {
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (t >= T) return;
    float r = 1.f;
    if (P.gain != nullptr) {
        float ss = 0.f;
        const float* st = P.stats_in + (size_t)(t0 + t) * P.stat_tiles_in;
        for (int i = lane; i < P.stat_tiles_in; i += 32) ss += st[i];
        ss = warp_sum(ss);
        r = 1.0f / sqrtf(ss / (float)P.K + P.eps);
    }
    if (lane == 0) inv_rms[t] = r;
}

__global__ void tc_pack_a_kernel(GemvProblem P, int t0, int T, int KS, int mtiles, const float* inv_rms,
                                 __nv_bfloat16* xa) {
    pdl_wait();
    pdl_trigger();
    // one thread = one 16-byte core-matrix row: (mtile, ks, m8, kh, r)
    const long long total = (long long)mtiles * KS * 16 * 2 * 8;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i & 7), kh = (int)((i >> 3) & 1), m8 = (int)((i >> 4) & 15);
        const long long rest = i >> 8;
        const int ks = (int)(rest % KS), mt = (int)(rest / KS);
        const int m = mt * kTcM + m8 * 8 + r;
        const int k0 = ks * 16 + kh * 8;
        float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (m < T) {
            const float* xr = P.x + (size_t)(t0 + m) * P.ldx;
            const float s = inv_rms[m];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = k0 + j;
                if (k < P.K) {
                    float x = xr[k];
                    if (P.gain != nullptr) x = __fmul_rn(__fmul_rn(x, s), P.gain[k]);
                    v[j] = x;
                }
            }
        }
        uint4 o;
        __nv_bfloat162 b0 = __floats2bfloat162_rn(v[0], v[1]), b1 = __floats2bfloat162_rn(v[2], v[3]);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[4], v[5]), b3 = __floats2bfloat162_rn(v[6], v[7]);
        o.x = *reinterpret_cast<uint32_t*>(&b0);
        o.y = *reinterpret_cast<uint32_t*>(&b1);
        o.z = *reinterpret_cast<uint32_t*>(&b2);
        o.w = *reinterpret_cast<uint32_t*>(&b3);
        reinterpret_cast<uint4*>(xa)[i] = o;
    }
}

template <int EPI>
static void tc_launch_t(const TcLaunch& L, int ntiles, cudaStream_t s) {
    static bool configured = false;
    const int smem = kTcStages * kTcStageBytes;
    if (!configured) {
        cudaFuncSetAttribute(tc_gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        configured = true;
    }
    launch_pdl(tc_gemm_kernel<EPI>, dim3(ntiles, L.mtiles), dim3(kTcThreads), (size_t)smem, s, L);
}

size_t tc_xa_elems(int rows, int K) {
    const int mtiles = (rows + kTcM - 1) / kTcM;
    return (size_t)mtiles * ((K + 15) / 16) * kTcM * 16;
}

// Prefill GEMM for rows [0, T) of the problem; workspace xa (tc_xa_elems
// bf16) and inv_rms (T floats).
void launch_tc_gemm(int epi, const GemvProblem& P, int T, const PassView& pass, const KvView& kv,
                    __nv_bfloat16* xa, float* inv_rms, cudaStream_t s) {
    if (T <= 0) return;
    TcLaunch L;
    L.P = P;
    L.pass = pass;
    L.kv = kv;
    L.t0 = 0;
    L.T = T;
    L.KS = (P.K + 15) / 16;
    L.mtiles = (T + kTcM - 1) / kTcM;
    L.xa = xa;
    tc_rms_kernel<<<(T + 7) / 8, 256, 0, s>>>(P, 0, T, inv_rms);
    const long long total = (long long)L.mtiles * L.KS * 256;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_pdl(tc_pack_a_kernel, dim3(blocks), dim3(256), 0, s, P, 0, T, L.KS, L.mtiles, (const float*)inv_rms, xa);
    const int ntiles = (P.ldw / 32 + kTcN / 32 - 1) / (kTcN / 32);
    switch (epi) {
        case EPI_STORE: tc_launch_t<EPI_STORE>(L, ntiles, s); break;
        case EPI_RESID: tc_launch_t<EPI_RESID>(L, ntiles, s); break;
        case EPI_SILU: tc_launch_t<EPI_SILU>(L, ntiles, s); break;
        case EPI_QKV: tc_launch_t<EPI_QKV>(L, ntiles, s); break;
        default: fprintf(stderr, "tc_gemm: epilogue %d not supported for prefill\n", epi);
    }
}

}  // namespace espec_dev
