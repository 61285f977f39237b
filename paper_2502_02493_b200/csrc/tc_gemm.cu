// Prompt-prefill GEMM on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Prefill is the one place on the EasySpec path where M (prompt rows) is a
// real contraction dimension: 256-row chunks of
// the prompt through every projection of both models. Decode passes (M <= 16)
// stay on the HBM-streaming GEMV (gemv_stream.cu).
//
// One CTA computes a 256 x 256 output tile (two 128-row UMMA accumulators
// sharing every weight tile) over its K split (split-K when the N tiles
// alone cannot fill 148 SMs; the last split reduces partials in order):
//   warp 0  TMA producer: 1-D bulk copies of the A tiles (2 x 16 KB: 256 rows x
//           64 k, pre-packed by pack_a_kernel) and of eight 1 KB weight blocks
//           per k-step (32 KB) into a 3-stage shared-memory ring (mbarrier
//           complete_tx);
//   warp 1  allocates all 512 TMEM columns; lane 0 issues tcgen05.mma
//           (kind::f16, M=128, N=256, K=16, fp32 accumulate in TMEM) — eight
//           per stage — and releases each stage with tcgen05.commit;
//   warps 2-9 epilogue: tcgen05.ld 32 columns at a time (each thread one row;
//           two warps per TMEM lane quarter take alternate 32-column groups),
//           then the same fused epilogues as the decode GEMV (residual + row
//           statistics, SiLU(gate)*up, RoPE + paged-KV write, store).
// Operands are UMMA canonical K-major "interleave" tiles: the weights are
// stored that way in HBM (kernels.cu pack_index) and a k-step's eight 1 KB
// group blocks placed side by side form one N=256 operand (LBO 128 B between
// the two k-halves of a core matrix column, SBO 256 B between 8-row core
// matrices); A uses the same layout for its 128 rows.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace espec_dev {

constexpr int kTcM = 128;             // rows per UMMA (one TMEM accumulator)
constexpr int kTcMSub = 2;            // UMMA row blocks per CTA: 256 rows share each weight tile
constexpr int kTcN = 256;             // 8 x 32-column weight groups
constexpr int kTcKStep = 16;          // one tcgen05.mma (bf16)
constexpr int kTcStepsPerStage = 4;   // 64 k per stage
constexpr int kTcStages = 3;
constexpr int kTcABlock = kTcM * kTcKStep * 2;                      // 4 KB: 128 rows x 16 k
constexpr int kTcAStage = kTcMSub * kTcABlock * kTcStepsPerStage;   // 32 KB
constexpr int kTcBStage = kTcN * kTcKStep * kTcStepsPerStage * 2;   // 32 KB
constexpr int kTcStageBytes = kTcAStage + kTcBStage;
constexpr int kTcEpiWarps = 8;  // two per TMEM lane quarter
constexpr int kTcThreads = (2 + kTcEpiWarps) * 32;
constexpr int kTcMinStagesPerSplit = 8;  // >= 512 k per K-split

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

struct alignas(64) TcLaunch {
    // the packed weights as a 3-D TMA tensor [k-step][group][1 KB block]
    // (uint32 elements; dims = {256, ngroups, KT}, strides {KT KB, 1 KB}) so one
    // cp.async.bulk.tensor box (256 x 8 groups x 4 k-steps = 32 KB) lands a
    // whole stage in the k-step-major order the N=256 UMMA operand needs
    CUtensorMap tmB;
    int use_tma;
    GemvProblem P;
    PassView pass;
    KvView kv;
    int t0, T;       // rows [t0, t0+T) of the pass
    int KS;          // k-steps (K/16, K padded to 16)
    int mtiles;      // 128-row blocks of A (1 or 2)
    int ksplits;     // K split across grid.z; partials reduced by the last CTA
    const __nv_bfloat16* xa;  // packed A: [mtile][KS][16 m8][2 kh][8 rows][8] bf16
    float* part;              // [ksplits][256][ldw] fp32 partial tiles (ksplits > 1)
    unsigned* tickets;        // [ntiles]
};

// epilogue for one (row, 32-column group): v = 32 fp32 sums of that row
template <int EPI>
__device__ __forceinline__ void tc_epilogue(const TcLaunch& L, int t, int g, const float (&v)[32]) {
    const GemvProblem& P = L.P;
    const int c0 = g * 32;
    // (each thread owns one row: 16-byte vector stores when the group is
    // whole and the row pointer aligned, which every engine shape satisfies)
    if constexpr (EPI == EPI_STORE) {
        float* o = P.out + (size_t)t * P.ldo + c0;
        if (c0 + 32 <= P.N && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c0 + j < P.N) o[j] = v[j];
        }
    } else if constexpr (EPI == EPI_RESID) {
        float* o = P.out + (size_t)t * P.ldo + c0;
        const float* r = P.resid + (size_t)t * P.ldr + c0;
        float sq = 0.f;
        if (c0 + 32 <= P.N && ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(r)) & 15) == 0) {
            float4 rr[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) rr[q] = *reinterpret_cast<const float4*>(r + 4 * q);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float y0 = __fadd_rn(rr[q].x, v[4 * q]), y1 = __fadd_rn(rr[q].y, v[4 * q + 1]);
                const float y2 = __fadd_rn(rr[q].z, v[4 * q + 2]), y3 = __fadd_rn(rr[q].w, v[4 * q + 3]);
                *reinterpret_cast<float4*>(o + 4 * q) = make_float4(y0, y1, y2, y3);
                sq = __fmaf_rn(y0, y0, sq);
                sq = __fmaf_rn(y1, y1, sq);
                sq = __fmaf_rn(y2, y2, sq);
                sq = __fmaf_rn(y3, y3, sq);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c0 + j < P.N) {
                    const float y = __fadd_rn(r[j], v[j]);
                    o[j] = y;
                    sq = __fmaf_rn(y, y, sq);
                }
        }
        P.stats_out[t * P.stat_tiles_out + g] = sq;
    } else if constexpr (EPI == EPI_SILU) {
        float* o = P.out + (size_t)t * P.ldo + g * 16;
        float y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = __fmul_rn(__fdiv_rn(v[j], __fadd_rn(1.0f, expf(-v[j]))), v[16 + j]);
        if (g * 16 + 16 <= P.N / 2 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (g * 16 + j < P.N / 2) o[j] = y[j];
        }
    } else if constexpr (EPI == EPI_QKV) {
        // every load of the group first (row metadata, page id, the rotary
        // factors of its 16 column pairs), then the arithmetic and the
        // stores: loads issued after a store cannot be hoisted above it (the
        // pointers may alias), which made each pair a serial L2 round trip
        const int qd = P.n_heads * P.dh, kd = P.n_kv * P.dh;
        const int pos = L.pass.pos[t];
        const int row = L.pass.rows[t];
        const KvView& kv = L.kv;
        const int page = c0 + 32 > qd && c0 < P.N ? kv.page_table[row / kv.page_rows] : 0;
        float2 cs_sn[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const int c = c0 + j;
            cs_sn[j >> 1] = make_float2(1.f, 0.f);
            if (c < P.N && c < qd + kd) {
                const int base = c < qd ? 0 : qd;
                const int i = (c - base) % P.dh;
                cs_sn[j >> 1] = __ldg(&P.rope[(size_t)pos * (P.dh >> 1) + (i >> 1)]);
            }
        }
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
                const float cs = cs_sn[j >> 1].x, sn = cs_sn[j >> 1].y;
                y0 = __fsub_rn(__fmul_rn(v[j], cs), __fmul_rn(v[j + 1], sn));
                y1 = __fadd_rn(__fmul_rn(v[j], sn), __fmul_rn(v[j + 1], cs));
            }
            if (region == 0) {
                *reinterpret_cast<float2*>(P.out + (size_t)t * P.ldo + c) = make_float2(y0, y1);
            } else {
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
    __shared__ unsigned s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntile = blockIdx.x, z = blockIdx.z;
    const int g0 = ntile * (kTcN / 32);
    const int KS = L.KS;
    const int nm = L.mtiles;  // active 128-row blocks
    const int stages_all = (KS + kTcStepsPerStage - 1) / kTcStepsPerStage;
    const int st0 = (int)((long long)z * stages_all / L.ksplits);
    const int st1 = (int)((long long)(z + 1) * stages_all / L.ksplits);
    const int ngroups = L.P.ldw / 32;
    const int ng = min(kTcN / 32, ngroups - g0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            tc_mbar_init(&full_bar[s], 1);
            tc_mbar_init(&empty_bar[s], 1);
        }
        tc_mbar_init(&acc_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // two 128 x 256 fp32 accumulators = all 512 TMEM columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&tmem_base)),
                     "r"(kTcMSub * kTcN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        // ---------------- producer (weights need no dependency; A does: the
        // first ring's weight boxes are issued before griddepcontrol.wait,
        // overlapping the predecessor's tail)
        if (lane == 0) {
            const char* A = reinterpret_cast<const char*>(L.xa);
            const char* B = reinterpret_cast<const char*>(L.P.W);
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            const size_t KT = (size_t)KS;
            auto issue_b = [&](int st, int s) {
                const int ks0 = st * kTcStepsPerStage;
                const int nks = min(kTcStepsPerStage, KS - ks0);
                // a tensor box always transfers its full 32 KB (out-of-range
                // groups / k-steps arrive as zeros)
                tc_mbar_expect(&full_bar[s], (uint32_t)(nm * nks * kTcABlock + (L.use_tma ? kTcBStage : nks * ng * 1024)));
                unsigned char* sb = sm + (size_t)s * kTcStageBytes + kTcAStage;
                if (L.use_tma) {
                    // weights are read once per launch: L2 evict-first
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
                        "[%1, {%2, %3, %4}], [%5], %6;" ::"r"(tc_smem(sb)),
                        "l"(reinterpret_cast<uint64_t>(&L.tmB)), "r"(0), "r"(g0), "r"(ks0), "r"(tc_smem(&full_bar[s])),
                        "l"(pol)
                        : "memory");
                } else {
                    for (int k = 0; k < nks; ++k)
                        for (int gl = 0; gl < ng; ++gl)
                            tc_bulk(sb + (size_t)k * (kTcN / 32) * 1024 + gl * 1024,
                                    B + (((size_t)(g0 + gl)) * KT + ks0 + k) * 1024, 1024u, &full_bar[s]);
                }
            };
            const int npre = min(kTcStages, st1 - st0);
            for (int i = 0; i < npre; ++i) issue_b(st0 + i, i);
            asm volatile("griddepcontrol.wait;" ::: "memory");
            for (int st = st0; st < st1; ++st) {
                const int i = st - st0, s = i % kTcStages;
                if (i >= npre) {
                    tc_mbar_wait(&empty_bar[s], ((uint32_t)(i / kTcStages) & 1u) ^ 1u);
                    issue_b(st, s);
                }
                const int ks0 = st * kTcStepsPerStage;
                const int nks = min(kTcStepsPerStage, KS - ks0);
                unsigned char* sa = sm + (size_t)s * kTcStageBytes;
                for (int m = 0; m < nm; ++m)
                    tc_bulk(sa + (size_t)m * kTcStepsPerStage * kTcABlock,
                            A + ((size_t)m * KS + ks0) * kTcABlock, (uint32_t)(nks * kTcABlock), &full_bar[s]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread)
        if (lane == 0) {
            for (int st = st0; st < st1; ++st) {
                const int i = st - st0, s = i % kTcStages;
                tc_mbar_wait(&full_bar[s], (uint32_t)(i / kTcStages) & 1u);
                tc_fence_after();
                const int ks0 = st * kTcStepsPerStage;
                const int nks = min(kTcStepsPerStage, KS - ks0);
                const uint32_t sa = tc_smem(sm + (size_t)s * kTcStageBytes);
                const uint32_t sb = sa + kTcAStage;
                for (int k = 0; k < nks; ++k) {
                    const uint64_t db = umma_desc(sb + k * (kTcN / 32) * 1024, 128, 256);
                    const uint32_t acc = (i > 0 || k > 0) ? 1u : 0u;
                    for (int m = 0; m < nm; ++m) {
                        const uint64_t da = umma_desc(sa + (m * kTcStepsPerStage + k) * kTcABlock, 128, 256);
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_base + m * kTcN),
                            "l"(da), "l"(db), "r"(kTcIdesc), "r"(acc));
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    tc_smem(&empty_bar[s])));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                tc_smem(&acc_bar)));
        }
    } else {
        // ---------------- epilogue warps 2..9: TMEM lanes 32*(warp%4) .., column
        // groups half, half + 2, ... (half = which of the quarter's two warps)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        tc_mbar_wait(&acc_bar, 0);
        tc_fence_after();
        const int lane_base = 32 * (warp & 3);
        const int half = (warp - 2) >> 2;
        const int ldw = L.P.ldw;
        for (int m = 0; m < nm; ++m) {
            const int r = m * kTcM + lane_base + lane;  // row within the CTA's 256
            const bool ok = r < L.T;
            for (int gl = half; gl < ng; gl += 2) {
                uint32_t u[32];
                const uint32_t taddr = tmem_base + ((uint32_t)lane_base << 16) + (uint32_t)(m * kTcN + gl * 32);
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
                if (L.ksplits == 1) {
                    if (ok) tc_epilogue<EPI>(L, L.t0 + r, g0 + gl, v);
                } else if (ok) {
                    float4* pp = reinterpret_cast<float4*>(L.part + ((size_t)z * 256 + r) * ldw + (g0 + gl) * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j) pp[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                }
            }
        }
        if (L.ksplits > 1) {
            // last K-split CTA of this tile sums the partials in split order
            asm volatile("bar.sync 1, %0;" ::"n"(kTcEpiWarps * 32) : "memory");
            if (threadIdx.x == 64) {
                unsigned tk;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(tk) : "l"(L.tickets + ntile) : "memory");
                s_last = tk == (unsigned)L.ksplits - 1 ? 1u : 0u;
                if (s_last) L.tickets[ntile] = 0u;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kTcEpiWarps * 32) : "memory");
            if (s_last) {
                for (int m = 0; m < nm; ++m) {
                    const int r = m * kTcM + lane_base + lane;
                    if (r >= L.T) continue;
                    for (int gl = half; gl < ng; gl += 2) {
                        float v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = 0.f;
                        // split order kept; the loads of up to 4 splits in
                        // flight per round trip (one split per round trip
                        // serialised the tail on L2 latency)
                        for (int z0 = 0; z0 < L.ksplits; z0 += 4) {
                            float4 q[4][8];
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                const float4* pp = reinterpret_cast<const float4*>(
                                    L.part + ((size_t)(z0 + b) * 256 + r) * ldw + (g0 + gl) * 32);
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    q[b][j] = z0 + b < L.ksplits ? __ldcg(pp + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                            }
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                if (z0 + b >= L.ksplits) break;
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    v[4 * j] += q[b][j].x;
                                    v[4 * j + 1] += q[b][j].y;
                                    v[4 * j + 2] += q[b][j].z;
                                    v[4 * j + 3] += q[b][j].w;
                                }
                            }
                        }
                        tc_epilogue<EPI>(L, L.t0 + r, g0 + gl, v);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcMSub * kTcN));
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
    static unsigned long long configured = 0;
    const int smem = kTcStages * kTcStageBytes;
    ensure_smem((const void*)tc_gemm_kernel<EPI>, smem, configured);
    DEV_CK(launch_pdl(tc_gemm_kernel<EPI>, dim3(ntiles, 1, L.ksplits), dim3(kTcThreads), (size_t)smem, s, L));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
static bool tc_encode_b(CUtensorMap& m, const void* W, int KT, int ngroups) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    static const bool off = std::getenv("ESPEC_TC_NO_TMA") != nullptr;
    if (!encode || off) return false;
    const cuuint64_t dims[3] = {256, (cuuint64_t)ngroups, (cuuint64_t)KT};
    const cuuint64_t strides[2] = {(cuuint64_t)KT * 1024, 1024};
    const cuuint32_t box[3] = {256, (cuuint32_t)(kTcN / 32), (cuuint32_t)kTcStepsPerStage};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(W), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

size_t tc_xa_elems(int rows, int K) {
    const int mtiles = (rows + kTcM - 1) / kTcM;
    return (size_t)mtiles * ((K + 15) / 16) * kTcM * 16;
}

// K splits for an output of ldw columns: fill ~148 SMs when the N tiles
// alone do not, keeping >= 512 k per split.
static int tc_ksplits(int K, int ldw) {
    const int ntiles = (ldw / 32 + kTcN / 32 - 1) / (kTcN / 32);
    const int stages = ((K + 15) / 16 + kTcStepsPerStage - 1) / kTcStepsPerStage;
    int ks = 148 / ntiles;
    if (ks > stages / kTcMinStagesPerSplit) ks = stages / kTcMinStagesPerSplit;
    return ks < 1 ? 1 : ks;
}

size_t tc_part_floats(int K, int ldw) {
    const int ks = tc_ksplits(K, ldw);
    return ks > 1 ? (size_t)ks * 256 * ldw : 0;
}

// Prefill GEMM for rows [0, T) (T <= 256) of the problem; workspace xa
// (tc_xa_elems bf16), inv_rms (T floats), part (tc_part_floats) + tickets.
void launch_tc_gemm(int epi, const GemvProblem& P, int T, const PassView& pass, const KvView& kv,
                    __nv_bfloat16* xa, float* inv_rms, cudaStream_t s) {
    if (T <= 0) return;
    if (T > kTcMSub * kTcM)
        dev_fail(DEV_ERR_CUDA, "tc_gemm: " + std::to_string(T) + " rows exceed the 256-row prefill chunk");
    TcLaunch L;
    L.use_tma = tc_encode_b(L.tmB, P.W, (P.K + 15) / 16, P.ldw / 32) ? 1 : 0;
    L.P = P;
    L.pass = pass;
    L.kv = kv;
    L.t0 = 0;
    L.T = T;
    L.KS = (P.K + 15) / 16;
    L.mtiles = (T + kTcM - 1) / kTcM;
    L.xa = xa;
    L.ksplits = P.tc_part ? tc_ksplits(P.K, P.ldw) : 1;
    L.part = P.tc_part;
    L.tickets = P.tc_tickets;
    tc_rms_kernel<<<(T + 7) / 8, 256, 0, s>>>(P, 0, T, inv_rms);
    DEV_CK(cudaGetLastError());
    const long long total = (long long)L.mtiles * L.KS * 256;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    DEV_CK(launch_pdl(tc_pack_a_kernel, dim3(blocks), dim3(256), 0, s, P, 0, T, L.KS, L.mtiles, (const float*)inv_rms, xa));
    const int ntiles = (P.ldw / 32 + kTcN / 32 - 1) / (kTcN / 32);
    switch (epi) {
        case EPI_STORE: tc_launch_t<EPI_STORE>(L, ntiles, s); break;
        case EPI_RESID: tc_launch_t<EPI_RESID>(L, ntiles, s); break;
        case EPI_SILU: tc_launch_t<EPI_SILU>(L, ntiles, s); break;
        case EPI_QKV: tc_launch_t<EPI_QKV>(L, ntiles, s); break;
        default: dev_fail(DEV_ERR_CUDA, "tc_gemm: epilogue " + std::to_string(epi) + " not supported for prefill");
    }
}

}  // namespace espec_dev
