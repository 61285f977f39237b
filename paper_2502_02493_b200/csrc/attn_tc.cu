// Decode / verify attention on the 5th-generation tensor cores (tcgen05,
// sm_100a) over the paged bf16 KV cache.
//
// Semantics: attention_forward (proj/src/model.cpp:140-192) with the tree mask
// of proj/src/kv_cache.cpp:43-60: softmax(q k^T / sqrt(dh)) v over the visible
// cache rows, GQA query pairs p = t * G + g of one kv head as the M rows.
//
// One CTA = (chunk of kv.attn_ppi 64-row pages, kv head, 128 query pairs):
//   warp 16, lane 0  streams the chunk's K/V pages through a kTcaStages-deep
//                    ring (two 4-D tensor-map boxes per K or V page, 128-byte
//                    swizzle: exactly the UMMA K-major layout for K and the
//                    MN-major layout for V) and issues the MMAs
//                      S = Q K^T   (M 128, N 64 keys, K dh; both K-major)
//                      PV = P V    (M 128, N dh, K 64 keys; V MN-major)
//                    into double-buffered TMEM tiles;
//   warps 0-15       softmax: warp w serves TMEM lane quarter w % 4 (query
//                    pairs 32 (w % 4) + lane) and column group j = w / 4:
//                    keys [16 j, 16 j + 16) of each page and output dims
//                    [DH/4 j, DH/4 (j + 1)). Per page: its 16 scores from
//                    TMEM, scale + mask, the row max over the four groups
//                    (shared memory, fixed order), exp, P (bf16) into the
//                    shared tile the PV MMA reads, and O = O * alpha + PV for
//                    its dims in registers (fp32).
// S(i+1) runs on the tensor core while the softmax of page i runs; PV(i)
// while the softmax of page i+1 runs. Four threads per row keep each
// thread's serial work per page short (16 keys, DH/4 dims) and give every
// scheduler four warps. Chunks along the context combine in fixed chunk
// order through a split workspace (last CTA of the kv head).
// A row's arithmetic depends only on its query, the visible keys and the
// chunking (a function of the cache capacity), never on the pass (batch
// invariance: a row is bit-identical in a 1-row and a 16-row pass).
// Pages wholly below the pass's first written row are loaded before
// griddepcontrol.wait (written by kernels that completed before this kernel's
// predecessor started), overlapping the QKV GEMV's tail.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "attn_common.cuh"
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace espec_dev {

constexpr int kTcaStages = 6;  // three steps of two pages
constexpr int kTcaRows = 128;             // query pairs per CTA (UMMA M)
constexpr int kTcaSoftmaxWarps = 16;
constexpr int kTcaSoftmax = 32 * kTcaSoftmaxWarps;
constexpr int kTcaThreads = kTcaSoftmax + 32;
constexpr int kTcaMaxChunks = 64;
constexpr int kTcaMaxPpi = 64;
constexpr int kTcaMaxTickets = 1 << 14;  // (problem, kv head, pair group) counters per stream

template <int DH>
struct TcaLayout {
    static constexpr int kQ = 0;                                  // [DH/64][128 rows][64] bf16, SW128
    static constexpr int kRing = kQ + kTcaRows * DH * 2;          // stages x (K [DH/64][64][64], V same)
    static constexpr int kStage = 2 * 64 * DH * 2;
    // a page's P tile ([128 rows][64 keys] bf16, 16 KB): at DH = 128 it reuses
    // the page's K buffer (K is dead once the page's QK MMA completed, and the
    // stage is refilled only after the page's PV MMA, the P reader, completed);
    // at DH = 64 the K buffer is 8 KB and P gets [2 steps][2 pages] of its own
    static constexpr bool kPInK = DH >= 128;
    static constexpr int kP = kRing + kTcaStages * kStage;
    static constexpr int kPBuf = kTcaRows * 64 * 2;
    static constexpr int kRed = kP + (kPInK ? 0 : 4 * kPBuf);      // [workers][rows] partial row maxima / sums (512)
    static constexpr int kBars = kRed + 4 * kTcaRows * 4;          // mbarriers, tmem base, page table
    static constexpr int kFlag = kBars + 256 + 4 * kTcaMaxPpi;   // ticket path: "this CTA combines"
    static constexpr int kBytes = kFlag + 16;
};

// UMMA shared-memory descriptor, 128-byte swizzle (layout type 2), version 1:
// start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46).
__device__ __forceinline__ uint64_t tca_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D f32, A/B bf16, A K-major, B K- or MN-major, M = 128
__host__ __device__ constexpr uint32_t tca_idesc(int n, int b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(kTcaRows >> 4) << 24);
}
__device__ __forceinline__ void tca_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tca_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tca_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tca_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 2^x (MUFU.EX2; ex2(-inf) = 0)
__device__ __forceinline__ float tca_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t u[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(u[j]);
}

// the scores of one worker in both pages of a step: KW columns at each of two
// TMEM addresses, one wait
template <int KW>
__device__ __forceinline__ void tmem_ld_pair(uint32_t a0, uint32_t a1, float (&v0)[KW], float (&v1)[KW]) {
    if constexpr (KW == 16) {
        tmem_ld16(a0, v0);
        tmem_ld16(a1, v1);
    } else if constexpr (KW == 8) {
        uint32_t u[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%16];\n"
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%17];\n"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
              "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
            : "r"(a0), "r"(a1)
            : "memory");
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v0[j] = __uint_as_float(u[j]);
            v1[j] = __uint_as_float(u[8 + j]);
        }
    } else {
        static_assert(KW == 4, "4, 8 or 16 keys per worker");
        uint32_t u[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%8];\n"
            "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [%9];\n"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
            : "r"(a0), "r"(a1)
            : "memory");
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v0[j] = __uint_as_float(u[j]);
            v1[j] = __uint_as_float(u[4 + j]);
        }
    }
}

__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Fixed-order combine of one row's 16 output dims over the chunk partials
// (values, max in the log2 domain, denominator): chunk weights 2^(m_ch - M),
// denominator and weighted sum in chunk order, CB chunks' loads in flight per
// round trip (CB changes only the load schedule, not the arithmetic). ml(ch) -> (m, l), x(ch, v) -> dims [4 v, 4 v + 4) of the slice.
// One arithmetic for the combine kernel (global partials) and the cluster
// path (partials in the cluster's shared memory), so a row is bit-identical
// whichever path its pass takes.
template <int CB, int NV, class ML, class X>
__device__ __forceinline__ void tca_combine(int nchunks, ML ml, X x, float4 (&acc)[NV], float& den) {
    float M = -INFINITY;  // (exact in any order; 8 loads in flight per round trip)
    for (int ch0 = 0; ch0 < nchunks; ch0 += 8) {
        float mm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mm[q] = ch0 + q < nchunks ? ml(ch0 + q).x : -INFINITY;
#pragma unroll
        for (int q = 0; q < 8; ++q) M = fmaxf(M, mm[q]);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    den = 0.f;
    for (int ch0 = 0; ch0 < nchunks; ch0 += CB) {
        float4 xv[CB][NV];
        float2 mv[CB];
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            const bool in = ch0 + q < nchunks;
            mv[q] = in ? ml(ch0 + q) : make_float2(-INFINITY, 0.f);
#pragma unroll
            for (int v = 0; v < NV; ++v) xv[q][v] = in ? x(ch0 + q, v) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < CB; ++q) {
            if (ch0 + q >= nchunks) break;
            float f = 0.f;
            if (M != -INFINITY && mv[q].x != -INFINITY) {
                f = tca_ex2(mv[q].x - M);
                den = __fmaf_rn(f, mv[q].y, den);
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                acc[v].x = __fmaf_rn(f, xv[q][v].x, acc[v].x);
                acc[v].y = __fmaf_rn(f, xv[q][v].y, acc[v].y);
                acc[v].z = __fmaf_rn(f, xv[q][v].z, acc[v].z);
                acc[v].w = __fmaf_rn(f, xv[q][v].w, acc[v].w);
            }
        }
    }
}

// ESPEC_ATTN_TRACE slots per CTA (%globaltimer): 0 start, 1 past
// griddepcontrol.wait, 2 first K page, 3 pages done, 4 end, 5 cluster
// synced, 6 prologue page loads issued, 7 first K page landed, 53 Q tile
// written; per step s < 8: 8+s QK(s) issued, 16+s PV(s) issued (MMA thread),
// 24+s S(s) seen, 32+s PV(s) seen, 40+s P(s) written (softmax thread 0);
// step 2 phases (softmax thread 0): 48 scores loaded, 49 row max exchanged,
// 50 exponentials summed, 51 fold done, 52 P stored
constexpr int kTcaTraceSlots = 64;

struct TcaLaunch {
    CUtensorMap kvmap;  // 4-D swizzled view of the KV pool (tca_tensor_map)
    AttnBatch b;
    PassView pass;
    KvView kv;
    int n_heads, G;
    unsigned long long* trace = nullptr;
    // how the chunks of a (kv head, pair group) combine (nchunks > 1):
    // 0: the PDL-launched combine kernel; 1: inside one cluster through DSMEM;
    // 2: the last chunk CTA to finish (ticket) combines from the workspace
    int cluster = 0;
    int* ticket = nullptr;  // mode 2: one arrival counter per (problem, kv head, pair group), zero between launches
};

// Pages are processed in steps of two (pages 2s, 2s + 1 of the chunk): one
// softmax round trip (scores, row max, probabilities, output fold) per step.
template <int DH, int REP>
__global__ void __launch_bounds__(kTcaThreads, 1) attn_tc_kernel(const __grid_constant__ TcaLaunch L) {
    static_assert(REP == 1 || REP == 2 || REP == 4, "row copies per tile");
    using LY = TcaLayout<DH>;
    constexpr int S = kTcaStages;   // = two steps of two pages
    constexpr int PS = DH + 4;      // workspace row: DH values, max, denominator
    constexpr int DQ = DH / 4;      // output dims per softmax thread
    static_assert(kTcaStages == 6, "the ring holds three steps of two pages");
    extern __shared__ __align__(1024) unsigned char smraw[];
    // the swizzled tiles need 1024-byte alignment: no static shared memory, so
    // the dynamic window starts aligned (checked)
    unsigned char* sm = smraw;
    if (smem_u32(smraw) & 1023u) __trap();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const AttnProblem& A = L.b.p[blockIdx.z];
    const PassView& pass = L.pass;
    const KvView& kv = L.kv;
    const int G = L.G, H = L.n_heads, P = pass.T * G, n_kv = kv.n_kv;
    const int hk = blockIdx.y % n_kv, mg = blockIdx.y / n_kv;
    const int ngroups = (P + kTcaRows - 1) / kTcaRows;
    const int bx = blockIdx.x, nchunks = gridDim.x;
    const int pg0 = bx * kv.attn_ppi, pg1 = min((pass.total + 63) / 64, pg0 + kv.attn_ppi);
    const int n = pg1 - pg0, nsteps = (n + 1) >> 1;

    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + LY::kBars);
    uint64_t* k_full = bars;            // [S] per page stage
    uint64_t* v_full = bars + S;        // [S]
    uint64_t* kv_empty = bars + 2 * S;  // [S]  PV of the stage's page done (tcgen05.commit)
    uint64_t* q_full = bars + 3 * S;    // softmax-thread arrivals
    uint64_t* s_full = q_full + 1;      // [2]  a step's S tile ready (commit)
    uint64_t* p_full = s_full + 2;      // [2]  a step's P written (softmax arrivals)
    uint64_t* pv_full = p_full + 2;     // [2]  a step's PV tile ready (commit)
    uint64_t* pv_free = pv_full + 2;    // [2]  PV tile read (softmax arrivals)
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(pv_free + 2);
    int* s_page = reinterpret_cast<int*>(sm + LY::kBars + 256);
    float* red = reinterpret_cast<float*>(sm + LY::kRed);  // [4 REP workers][128 / REP rows]
    unsigned long long* tr =
        L.trace ? L.trace + (((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * kTcaTraceSlots : nullptr;
    auto kbuf = [&](int st) { return sm + LY::kRing + st * LY::kStage; };
    auto vbuf = [&](int st) { return sm + LY::kRing + st * LY::kStage + LY::kStage / 2; };
    auto pbuf = [&](int s, int pp) {  // P tile of page 2 s + pp
        return LY::kPInK ? kbuf((2 * s + pp) % S) : sm + LY::kP + ((s & 1) * 2 + pp) * LY::kPBuf;
    };
    auto issue = [&](int i, int page) {  // K and V of page pg0 + i into stage i % S
        const int st = i % S;
        for (int kind = 0; kind < 2; ++kind) {
            uint64_t* bar = kind ? &v_full[st] : &k_full[st];
            unsigned char* dst = kind ? vbuf(st) : kbuf(st);
            const int lkh = (A.layer * 2 + kind) * n_kv + hk;
            mbar_arrive_expect_tx(bar, 64 * DH * 2);
#pragma unroll
            for (int h = 0; h < DH / 64; ++h)
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4, %5}], [%6];" ::"r"(smem_u32(dst + h * 8192)),
                    "l"(reinterpret_cast<uint64_t>(&L.kvmap)), "r"(h * 64), "r"(0), "r"(lkh), "r"(page),
                    "r"(smem_u32(bar))
                    : "memory");
        }
    };
    auto stable = [&](int pg) { return (pg + 1) * 64 <= pass.new_lo; };

    // ---- prologue (before the dependency wait): barriers, TMEM, stable pages
    if (tr && tid == 0) atomicMax(tr, gtimer());
    if (tid == kTcaSoftmax) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        mbar_init(q_full, kTcaSoftmax);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&p_full[b], kTcaSoftmax);
            mbar_init(&pv_full[b], 1);
            mbar_init(&pv_free[b], kTcaSoftmax);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the ring's page ids in one round trip (a load per issue would
        // serialise behind each TMA issue's memory clobber)
        int pt[S];
#pragma unroll
        for (int i = 0; i < S; ++i) pt[i] = i < n ? kv.page_table[pg0 + i] : 0;
#pragma unroll
        for (int i = 0; i < S; ++i)
            if (i < n && stable(pg0 + i)) issue(i, pt[i]);
        if (tr) tr[6] = gtimer();
    }
    // S tiles (two pages each) at columns [0, 256), PV tiles at [256, 256 + 2 DH):
    // 512 columns, allocated before the dependent grid may launch (no TMEM wait cycles)
    if (warp == kTcaSoftmaxWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tca_fence_before();
    __syncthreads();
    tca_fence_after();
    const uint32_t tmem = *s_tmem;
    pdl_wait();
    if (tr && tid == 0) atomicMax(tr + 1, gtimer());
    pdl_trigger();

    if (warp == kTcaSoftmaxWarps) {
        // ---------------- producer + MMA issuer
        if (lane == 0) {
            for (int i0 = 0; i0 < n; i0 += 8) {  // 8 loads in flight per round trip
                int v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = i0 + k < n ? kv.page_table[pg0 + i0 + k] : 0;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (i0 + k < n) s_page[i0 + k] = v[k];
            }
            for (int i = 0; i < n && i < S; ++i)
                if (!stable(pg0 + i)) issue(i, s_page[i]);
            if (tr) tr[55] = gtimer();
            const uint32_t qaddr = smem_u32(sm + LY::kQ);
            const uint32_t id_s = tca_idesc(64, 0), id_pv = tca_idesc(DH, 1);
            // one thread issues three independent streams as their inputs
            // land (polling, so none waits behind another): QK(s) when the
            // step's K pages are in and S buffer s & 1 is free, PV(s) when
            // P(s), the V pages and PV buffer s & 1 are ready, and the refill
            // of a page's stage with the page S later once PV released it
            auto qk = [&](int s) {  // S[s & 1] = Q [K(2s) | K(2s + 1)]^T
                for (int pp = 0; pp < 2 && 2 * s + pp < n; ++pp) {
                    const int i = 2 * s + pp, st = i % S;
                    if (tr && i == 0) atomicMax(tr + 2, gtimer());
                    const uint32_t kaddr = smem_u32(kbuf(st));
#pragma unroll
                    for (int kk = 0; kk < DH / 16; ++kk)
                        tca_mma(tmem + (s & 1) * 128 + pp * 64,
                                tca_desc(qaddr + (kk >> 2) * (kTcaRows * 128) + (kk & 3) * 32, 16, 1024),
                                tca_desc(kaddr + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_s, kk > 0);
                }
                if (tr && s < 8) tr[8 + s] = gtimer();
                tca_commit(&s_full[s & 1]);
            };
            auto pv = [&](int s) {  // PV[s & 1] = P(2s) V(2s) + P(2s + 1) V(2s + 1)
                const int b = s & 1;
                if (tr && s < 8) tr[16 + s] = gtimer();
                for (int pp = 0; pp < 2 && 2 * s + pp < n; ++pp) {
                    const int i = 2 * s + pp, st = i % S;
                    const uint32_t paddr = smem_u32(pbuf(s, pp)), vaddr = smem_u32(vbuf(st));
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)  // 16 keys per MMA
                        tca_mma(tmem + 256 + b * DH, tca_desc(paddr + kk * 32, 16, 1024),
                                tca_desc(vaddr + kk * 2048, 8192, 1024), id_pv, pp > 0 || kk > 0);
                }
                tca_commit(&pv_full[b]);
                for (int pp = 0; pp < 2 && 2 * s + pp < n; ++pp) tca_commit(&kv_empty[(2 * s + pp) % S]);
            };
            auto pages_in = [&](uint64_t* full, int s) {
                for (int pp = 0; pp < 2 && 2 * s + pp < n; ++pp) {
                    const int i = 2 * s + pp;
                    if (!mbar_test(&full[i % S], (uint32_t)(i / S) & 1u)) return false;
                }
                return true;
            };
            if (tr) {
                mbar_wait(&k_full[0], 0);
                tr[7] = gtimer();
            }
            mbar_wait(q_full, 0);
            if (tr) tr[53] = gtimer();
            tca_fence_after();
            int qn = 0, pn = 0, rn = 0;  // next QK step, next PV step, next page to refill
            while (pn < nsteps) {
                // S buffer qn & 1 is free once PV(qn - 2) was issued (after P(qn - 2))
                if (qn < nsteps && qn <= pn + 1 && pages_in(k_full, qn)) {
                    tca_fence_after();
                    qk(qn++);
                }
                if (pn < qn && mbar_test(&p_full[pn & 1], (uint32_t)(pn >> 1) & 1u) &&
                    (pn < 2 || mbar_test(&pv_free[pn & 1], (uint32_t)((pn - 2) >> 1) & 1u)) && pages_in(v_full, pn)) {
                    tca_fence_after();
                    pv(pn++);
                }
                while (rn + S < n && rn / 2 < pn && mbar_test(&kv_empty[rn % S], (uint32_t)(rn / S) & 1u)) {
                    issue(rn + S, s_page[rn + S]);
                    ++rn;
                }
            }
        }
    } else {
        // ---------------- softmax warps
        // REP copies of the group's rows fill the 128-row tile (REP 4: <= 32
        // rows, 2: <= 64, else 1): tile row t holds pair row t % R, so every
        // TMEM lane quarter (a warp reads only its own quarter's lanes) has
        // live rows, and the 4 REP warps of a row split its keys: KW = 16 /
        // REP keys of each page per worker (the exponentials per warp fall by
        // REP and spread over all four SM sub-partitions). A row's arithmetic
        // does not depend on REP (batch invariance): 16 key units of 4 keys
        // per page, each with its own running denominator, summed by one
        // pairwise tree at the end.
        constexpr int R = kTcaRows / REP;  // canonical rows
        constexpr int KW = 16 / REP;       // keys of each page per worker
        constexpr int U = KW / 4;          // key units per worker
        constexpr int NW = 4 * REP;        // workers per row
        const int qtr = warp & 3, grp = warp >> 2;
        const int t = qtr * 32 + lane;  // tile row = TMEM lane
        const int r = t % R;            // the pair row it holds
        const int w = (t / R) * 4 + grp;  // worker: keys [w KW, w KW + KW) of each page
        const bool owner = t < R;       // copy 0: folds PV and holds output dims [grp DQ, grp DQ + DQ)
        const int p = mg * kTcaRows + r;
        const bool valid = p < P;
        const int bar_row = 2 + qtr % (4 / REP);  // named barrier of the 4 REP warps sharing these rows
        constexpr int bar_n = 128 * REP;
        int ve = 0;
        unsigned long long an = 0ull;
        {
            // Q row (this thread's DH/4 dims) -> bf16 shared tile (K-major, 128-byte swizzle)
            const float* q = valid ? A.q + (size_t)(p / G) * H * DH + (hk * G + p % G) * DH : nullptr;
            if (valid) {
                ve = pass.vis_end[p / G];
                an = pass.anc[p / G];
            }
            unsigned char* qrow = sm + LY::kQ + t * 128;
#pragma unroll
            for (int cc = 0; cc < DQ / 8; ++cc) {  // 16-byte chunks of 8 dims
                const int c = grp * (DQ / 8) + cc;
                float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
                if (valid) {
                    a = *reinterpret_cast<const float4*>(q + c * 8);
                    b = *reinterpret_cast<const float4*>(q + c * 8 + 4);
                }
                const uint4 u = make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                                           pack_bf16x2(b.z, b.w));
                *reinterpret_cast<uint4*>(qrow + (c >> 3) * (kTcaRows * 128) + (((c & 7) ^ (t & 7)) * 16)) = u;
            }
            if (tr && tid == 0) tr[54] = gtimer();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(q_full);
        }
        const int vmin = valid ? min(ve, pass.total) : 0x7fffffff;
        // scores in the log2 domain: s * log2(e) / sqrt(dh), probabilities by ex2
        const float qscale = 1.4426950408889634f / sqrtf((float)DH);
        // a lane quarter with no valid pair (e.g. rows 64-127 of a 96-pair
        // pass) only keeps the barrier counts: its P / PV rows are never read
        const bool idle = mg * kTcaRows + (qtr * 32) % R >= P;
        const uint32_t trow = tmem + ((uint32_t)(qtr * 32) << 16);
        float o[DQ];
#pragma unroll
        for (int d = 0; d < DQ; ++d) o[d] = 0.f;
        float m = -INFINITY, alpha_prev = 0.f;
        float lu[U];
#pragma unroll
        for (int u = 0; u < U; ++u) lu[u] = 0.f;
        auto fold = [&](int s) {  // o = o * alpha(s) + PV(s) over this thread's dims
            const int b = s & 1;
            mbar_wait(&pv_full[b], (uint32_t)(s >> 1) & 1u);
            if (tr && tid == 0 && s < 8) tr[32 + s] = gtimer();
            if (idle || !owner) {
                mbar_arrive(&pv_free[b]);
                return;
            }
            tca_fence_after();
#pragma unroll
            for (int c = 0; c < DQ / 16; ++c) {
                float v[16];
                tmem_ld16(trow + 256 + b * DH + grp * DQ + c * 16, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) o[c * 16 + j] = __fmaf_rn(o[c * 16 + j], alpha_prev, v[j]);
            }
            tca_fence_before();
            mbar_arrive(&pv_free[b]);
        };
        for (int s = 0; s < nsteps; ++s) {
            const int b = s & 1;
            mbar_wait(&s_full[b], (uint32_t)(s >> 1) & 1u);
            if (tr && tid == 0 && s < 8) tr[24 + s] = gtimer();
            if (idle) {
                if (s > 0) fold(s - 1);
                mbar_arrive(&p_full[b]);
                continue;
            }
            tca_fence_after();
            // this worker's keys of each page of the step
            float sc[2][KW];
            tmem_ld_pair<KW>(trow + b * 128 + w * KW, trow + b * 128 + 64 + w * KW, sc[0], sc[1]);
            const bool ph = tr && tid == 0 && s == 2;
            if (ph) tr[48] = gtimer();
            float mx = -INFINITY;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
                const int j0 = (pg0 + 2 * s + pp) * 64 + w * KW;
                if (j0 + KW <= vmin) {  // below every causal prefix: no per-key test
#pragma unroll
                    for (int j = 0; j < KW; ++j) {
                        sc[pp][j] = __fmul_rn(sc[pp][j], qscale);
                        mx = fmaxf(mx, sc[pp][j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < KW; ++j) {
                        const bool ok = valid && visible_rows(pass, ve, an, j0 + j);
                        sc[pp][j] = ok ? __fmul_rn(sc[pp][j], qscale) : -INFINITY;
                        mx = fmaxf(mx, sc[pp][j]);
                    }
                }
            }
            // row max over the workers (exact in any order; the second
            // barrier: every worker has read before the next step writes)
            red[w * R + r] = mx;
            named_bar(bar_row, bar_n);
#pragma unroll
            for (int k = 0; k < NW; ++k) mx = fmaxf(mx, red[k * R + r]);
            named_bar(bar_row, bar_n);
            if (ph) tr[49] = gtimer();
            const float mn = fmaxf(m, mx);
            // rescale of the running sums (exactly 1 while the max holds, 0
            // while nothing was visible yet)
            const float alpha = m == -INFINITY ? 0.f : (mn == m ? 1.f : tca_ex2(m - mn));
            m = mn;
            const float mo = m == -INFINITY ? 0.f : m;  // ex2(-inf - 0) = 0 for masked keys
#pragma unroll
            for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                for (int j = 0; j < KW; ++j) sc[pp][j] = tca_ex2(sc[pp][j] - mo);
#pragma unroll
            for (int u = 0; u < U; ++u) {  // a unit's 8 keys of the step in order
                float su = 0.f;
#pragma unroll
                for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                    for (int j = 0; j < 4; ++j) su += sc[pp][4 * u + j];
                lu[u] = __fmaf_rn(lu[u], alpha, su);
            }
            if (ph) tr[50] = gtimer();
            // P (bf16) -> the K-major 128-byte-swizzled tile of each page of the
            // step, row r (its K buffer, dead since QK(s) completed, or a P
            // buffer whose previous reader PV(s - 2) completed before fold(s - 2))
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
                if (pp == 1 && 2 * s + 1 >= n) break;
                unsigned char* prow = pbuf(s, pp) + r * 128;
                const float* v = sc[pp];
                if constexpr (KW >= 8) {
#pragma unroll
                    for (int h = 0; h < KW / 8; ++h) {
                        const int c = w * (KW / 8) + h;
                        const uint4 u = make_uint4(pack_bf16x2(v[8 * h], v[8 * h + 1]), pack_bf16x2(v[8 * h + 2], v[8 * h + 3]),
                                                   pack_bf16x2(v[8 * h + 4], v[8 * h + 5]), pack_bf16x2(v[8 * h + 6], v[8 * h + 7]));
                        *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) * 16)) = u;
                    }
                } else {
                    const int c = w >> 1;
                    *reinterpret_cast<uint2*>(prow + ((c ^ (r & 7)) * 16) + (w & 1) * 8) =
                        make_uint2(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]));
                }
            }
            if (ph) tr[52] = gtimer();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tca_fence_before();
            mbar_arrive(&p_full[b]);
            if (tr && tid == 0 && s < 8) tr[40 + s] = gtimer();
            // the previous step's PV (issued one step ago) into the output
            if (s > 0) fold(s - 1);
            if (ph) tr[51] = gtimer();
            alpha_prev = alpha;
        }
        if (nsteps > 0) fold(nsteps - 1);
        if (!idle) {  // (an idle quarter's warps skip this together)
            // the row's denominator: the pairwise tree over the 16 key units
            // (each worker's own units first, then the workers')
            float lw = lu[0];
            if constexpr (U == 2) lw = lu[0] + lu[1];
            if constexpr (U == 4) lw = (lu[0] + lu[1]) + (lu[2] + lu[3]);
            red[w * R + r] = lw;
            named_bar(bar_row, bar_n);
            float v[NW];
#pragma unroll
            for (int k = 0; k < NW; ++k) v[k] = red[k * R + r];
#pragma unroll
            for (int k = NW; k > 1; k >>= 1)
#pragma unroll
                for (int i = 0; i < k / 2; ++i) v[i] = v[2 * i] + v[2 * i + 1];
            const float l = v[0];
            if (tr && tid == 0) atomicMax(tr + 3, gtimer());
            if (valid && owner) {
                if (nchunks == 1) {
                    const size_t off = (size_t)(p / G) * H * DH + (hk * G + p % G) * DH + grp * DQ;
#pragma unroll
                    for (int c = 0; c < DQ / 16; ++c) {
                        float4 acc[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            acc[v] = make_float4(o[c * 16 + 4 * v], o[c * 16 + 4 * v + 1], o[c * 16 + 4 * v + 2],
                                                 o[c * 16 + 4 * v + 3]);
                        attn_store_row<DH>(A, off + c * 16, acc, l);
                    }
                } else {
                    // chunk partial: to this CTA's shared memory (cluster path;
                    // the ring is dead: every page's MMAs completed) or to the
                    // split workspace for the combine kernel
                    float* prow = L.cluster == 1 ? reinterpret_cast<float*>(sm + LY::kRing) + (size_t)r * PS
                                            : A.ws + (((size_t)bx * (n_kv * ngroups) + blockIdx.y) * kTcaRows + r) * PS;
#pragma unroll
                    for (int c = 0; c < DQ / 4; ++c)
                        *reinterpret_cast<float4*>(prow + grp * DQ + 4 * c) =
                            make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
                    if (grp == 0) *reinterpret_cast<float2*>(prow + DH) = make_float2(m, l);
                }
            }
        }
    }
    if (L.cluster == 2 && nchunks > 1) {
        // ticket combine: every chunk CTA has written its partial rows to the
        // workspace; the last to arrive combines them (the combine kernel's
        // arithmetic and thread mapping: bit-identical rows) — no cluster
        // co-scheduling, no combine launch and no extra dependency hop
        int* last = reinterpret_cast<int*>(sm + LY::kFlag);
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            int* ctr = L.ticket + (size_t)blockIdx.z * gridDim.y + blockIdx.y;
            const int arrived = atomicAdd(ctr, 1);
            const int is_last = arrived == nchunks - 1;
            if (is_last) *ctr = 0;  // every chunk has arrived: ready for the next launch
            *last = is_last;
            __threadfence();
        }
        __syncthreads();
        if (*last) {
            // 4 output dims per thread item (the same per-element arithmetic
            // as the 16-dim items of the combine kernel): 8 chunks' loads in
            // flight without spilling the softmax path's registers
            constexpr int CPR = DH / 4;
            const int R = min(kTcaRows, P - mg * kTcaRows);
            const size_t cstride = (size_t)(n_kv * ngroups) * kTcaRows * PS;
            for (int it = tid; it < R * CPR; it += kTcaThreads) {
                const int rr = it / CPR, c0 = (it % CPR) * 4;
                const float* base = A.ws + ((size_t)blockIdx.y * kTcaRows + rr) * PS;
                float4 acc[1];
                float den;
                tca_combine<8>(
                    nchunks, [&](int ch) { return __ldcg(reinterpret_cast<const float2*>(base + ch * cstride + DH)); },
                    [&](int ch, int v) {
                        return __ldcg(reinterpret_cast<const float4*>(base + ch * cstride + c0 + 4 * v));
                    },
                    acc, den);
                const int pp = mg * kTcaRows + rr;
                attn_store_row<DH>(A, (size_t)(pp / G) * H * DH + (hk * G + pp % G) * DH + c0, acc, den);
            }
        }
        if (tr && tid == 0) atomicMax(tr + 56, gtimer());
    }
    if (L.cluster == 1) {
        __syncwarp();
        // the cluster's CTAs hold the chunks of this (kv head, pair group);
        // CTA c combines rows [c R / chunks, (c + 1) R / chunks). Every CTA
        // pushes each partial row to its combiner's shared memory (remote
        // stores: no round trips), then each combines from local memory.
        const int R = min(kTcaRows, P - mg * kTcaRows);
        const int RPO = (R + nchunks - 1) / nchunks + 1;  // rows per combiner, bound
        auto r_lo = [&](int c) { return c * R / nchunks; };
        float* part = reinterpret_cast<float*>(sm + LY::kRing);  // [128][PS] own partial rows
        float* recv = part + kTcaRows * PS;                          // [chunk][RPO][PS] rows to combine
        cluster_sync_all();  // every CTA's ring is dead: receive areas may be written
        if (tr && tid == 0) tr[5] = gtimer();
        for (int it = tid; it < R * (PS / 4); it += kTcaThreads) {
            const int rr = it / (PS / 4), q4 = it % (PS / 4);
            int c = rr * nchunks / R;
            while (c + 1 < nchunks && rr >= r_lo(c + 1)) ++c;
            while (rr < r_lo(c)) --c;
            const float4 v = *reinterpret_cast<const float4*>(part + rr * PS + 4 * q4);
            const uint32_t dst = dsmem_addr(smem_u32(recv + ((bx * RPO) + (rr - r_lo(c))) * PS + 4 * q4), (uint32_t)c);
            asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                         "f"(v.w)
                         : "memory");
        }
        cluster_sync_all();  // the pushed rows are visible; no remote access after this
        const int r0 = r_lo(bx), r1 = r_lo(bx + 1);
        for (int it = tid; it < (r1 - r0) * (DH / 16); it += kTcaThreads) {
            const int lr = it / (DH / 16), c0 = (it % (DH / 16)) * 16;
            const float* row = recv + lr * PS;
            float4 acc[4];
            float den;
            tca_combine<2>(
                nchunks, [&](int ch) { return *reinterpret_cast<const float2*>(row + (size_t)ch * RPO * PS + DH); },
                [&](int ch, int v) { return *reinterpret_cast<const float4*>(row + (size_t)ch * RPO * PS + c0 + 4 * v); },
                acc, den);
            const int pp = mg * kTcaRows + r0 + lr;
            attn_store_row<DH>(A, (size_t)(pp / G) * H * DH + (hk * G + pp % G) * DH + c0, acc, den);
        }
        if (tr) atomicMax(tr + 56, gtimer());
    }
    // TMEM is no longer read: release it
    tca_fence_before();
    __syncthreads();
    if (warp == kTcaSoftmaxWarps) {
        tca_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
    if (tr && tid == 0) atomicMax(tr + 4, gtimer());
}

// Cross-chunk combine (chunks > 1), its own PDL-launched kernel so the
// partials are combined by many CTAs at once: CTA = 32 query pairs of one
// (kv head, pair group, problem); thread = (pair, 16 output dims). Chunk
// weights 2^(m_ch - M) and the denominator in fixed chunk order, then the
// weighted sum of the chunk partials in fixed chunk order (8 chunks' loads in
// flight per round trip).
template <int DH>
__global__ void __launch_bounds__(32 * (DH / 16)) attn_tc_combine_kernel(const __grid_constant__ TcaLaunch L,
                                                                          int nchunks) {
    constexpr int PS = DH + 4;
    constexpr int CPR = DH / 16;
    pdl_wait();
    pdl_trigger();
    const AttnProblem& A = L.b.p[blockIdx.z];
    const int G = L.G, H = L.n_heads, P = L.pass.T * G, n_kv = L.kv.n_kv;
    const int ngroups = (P + kTcaRows - 1) / kTcaRows;
    const int by = blockIdx.y;  // (pair group, kv head) as in attn_tc_kernel
    const int hk = by % n_kv, mg = by / n_kv;
    const int r = blockIdx.x * 32 + threadIdx.x / CPR, c0 = (threadIdx.x % CPR) * 16;
    const int p = mg * kTcaRows + r;
    if (r >= kTcaRows || p >= P) return;
    const size_t cstride = (size_t)(n_kv * ngroups) * kTcaRows * PS;
    const float* base = A.ws + ((size_t)by * kTcaRows + r) * PS;
    float4 acc[4];
    float den;
    tca_combine<8>(
        nchunks, [&](int ch) { return __ldcg(reinterpret_cast<const float2*>(base + ch * cstride + DH)); },
        [&](int ch, int v) { return __ldcg(reinterpret_cast<const float4*>(base + ch * cstride + c0 + 4 * v)); }, acc,
        den);
    attn_store_row<DH>(A, (size_t)(p / G) * H * DH + (hk * G + p % G) * DH + c0, acc, den);
}

// 4-D tensor map of a bf16 KV pool: {dh, 64 rows, (layer, k|v, kv head),
// page}, box {64, 64, 1, 1}, 128-byte swizzle; encoded once per pool.
static void tca_tensor_map(CUtensorMap& m, const KvView& kv) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) dev_fail(DEV_ERR_CUDA, "attention: cuTensorMapEncodeTiled is unavailable");
    if (kv.pool_pages <= 0) dev_fail(DEV_ERR_CUDA, "attention: KvView.pool_pages is not set");
    struct Entry {
        const void* pool;
        long long page_elems;
        int n_layers, n_kv, dh, pages;
        CUtensorMap map;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : cache)
        if (e.pool == kv.pool && e.page_elems == kv.page_elems && e.n_layers == kv.n_layers && e.n_kv == kv.n_kv &&
            e.dh == kv.dh && e.pages == kv.pool_pages) {
            m = e.map;
            return;
        }
    const cuuint64_t dims[4] = {(cuuint64_t)kv.dh, 64, (cuuint64_t)kv.n_layers * 2 * kv.n_kv,
                                (cuuint64_t)kv.pool_pages};
    const cuuint64_t strides[3] = {(cuuint64_t)kv.dh * 2, (cuuint64_t)64 * kv.dh * 2, (cuuint64_t)kv.page_elems * 2};
    const cuuint32_t box[4] = {64, 64, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, kv.pool, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        dev_fail(DEV_ERR_CUDA, "attention: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    cache.push_back({kv.pool, kv.page_elems, kv.n_layers, kv.n_kv, kv.dh, kv.pool_pages, m});
}

// Chunks of one (kv head, pair group) combine inside their cluster when
// they fit one (2..ESPEC_ATTN_CLUSTER CTAs, default the portable 8; up to 16
// opts in to non-portable clusters, which measured 1.8x slower at 16 chunks
// as a 16-SM cluster rarely finds a free GPC): no workspace round trip, no
// combine launch (~1 us per attention isolated, profiles/r2_cluster.txt).
// ESPEC_ATTN_CLUSTER=0 keeps the combine kernel.
// Single-row passes (T = 1: at most G <= 8 pair rows) with more chunks than
// a cluster holds let the last chunk CTA to finish combine (mode 2): 8 rows x
// 16 chunks are two L2 round trips on one SM, cheaper than a combine launch
// (isolated drafter T = 1 ctx 8K 16.4 -> 15.7 us). Wider passes keep the
// combine kernel: one SM combining 48 rows x 8 chunks measured 4-8 us slower
// (profiles/r2_attn_ticket.txt). ESPEC_ATTN_COMBINE=ticket forces mode 2
// whenever chunks > 1, =kernel never uses it.
int attn_tc_cluster(int chunks, int T) {
    static const int cap = [] {
        const char* e = std::getenv("ESPEC_ATTN_CLUSTER");
        return e ? std::min(16, std::atoi(e)) : 8;
    }();
    static const int ticket = [] {  // 1 force, 0 auto, -1 never
        const char* e = std::getenv("ESPEC_ATTN_COMBINE");
        if (!e) return 0;
        const std::string v(e);
        return v == "ticket" ? 1 : v == "kernel" ? -1 : 0;
    }();
    if (chunks < 2) return 0;
    if (ticket > 0) return 2;
    if (chunks <= cap) return 1;
    return ticket == 0 && T == 1 ? 2 : 0;
}

// per-(device, stream) ticket counters (zeroed once; every launch leaves them
// zero); launches on one stream never overlap in their ticket phase (each
// follows griddepcontrol.wait, i.e. the completion of every earlier kernel)
static int* tca_tickets(cudaStream_t s) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, int*>> all;
    int dev = 0;
    DEV_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    for (auto& e : all)
        if (e.first.first == dev && e.first.second == s) return e.second;
    int* p = nullptr;
    DEV_CK(cudaMalloc(&p, sizeof(int) * kTcaMaxTickets));
    DEV_CK(cudaMemset(p, 0, sizeof(int) * kTcaMaxTickets));
    DEV_CK(cudaDeviceSynchronize());
    all.push_back({{dev, s}, p});
    return p;
}

// Pages per chunk CTA of a launch: the cache's capacity rule (kv.attn_ppi),
// doubled while a batched launch (nprob > 1: a fuzzy group's layers) would
// need more than one wave of CTAs — at ctx 512 a 4-layer group of the C2
// drafter is 5 chunks x 8 kv heads x 4 = 160 CTAs, a second wave for 12 of
// them — up to 8 pages per CTA (4 softmax steps): longer chunks lose more
// to their serial step chain than the extra waves cost (C5 sweep, ctx 8K:
// doubling 8 -> 32 pages per CTA made the lp 4 / 8 draft stage 0.4-0.7 ms
// slower; ctx 512: draft stage -0.15 ms, ctx 2K -0.1 ms;
// profiles/r2_attn_wave.txt). Single-problem launches (every base pass, so
// verify and vanilla rows stay bitwise equal) keep the capacity rule.
// ESPEC_ATTN_WAVE=0 disables.
int attn_tc_ppi(const PassView& pass, const KvView& kv, int n_heads, int nprob) {
    static const bool on = [] {
        const char* e = std::getenv("ESPEC_ATTN_WAVE");
        return !(e && std::atoi(e) == 0);
    }();
    int ppi = kv.attn_ppi;
    if (!on || nprob <= 1) return ppi;
    const int pages = (pass.total + 63) / 64;
    const int groups = (pass.T * (n_heads / kv.n_kv) + kTcaRows - 1) / kTcaRows;
    auto ctas = [&](int q) { return (long long)((pages + q - 1) / q) * kv.n_kv * groups * nprob; };
    while (ctas(ppi) > 148 && ppi * 2 <= 8 && (pages + ppi - 1) / ppi > 1) ppi *= 2;
    return ppi;
}

template <int DH>
static void attn_tc_launch(const AttnBatch& b, int nprob, int n_heads, const PassView& pass, const KvView& kv_in,
                           cudaStream_t s) {
    KvView kv = kv_in;
    kv.attn_ppi = attn_tc_ppi(pass, kv_in, n_heads, nprob);
    TcaLaunch L;
    tca_tensor_map(L.kvmap, kv);
    L.b = b;
    L.pass = pass;
    L.kv = kv;
    L.n_heads = n_heads;
    L.G = n_heads / kv.n_kv;
    const int splits = (pass.total + 63) / 64;
    const int chunks = (splits + kv.attn_ppi - 1) / kv.attn_ppi;
    if (chunks > kTcaMaxChunks || kv.attn_ppi > kTcaMaxPpi)
        dev_fail(DEV_ERR_CUDA, "attention: context of " + std::to_string(pass.total) + " rows exceeds the " +
                                   std::to_string(kTcaMaxChunks * kv.attn_ppi * 64) +
                                   "-row split-combine limit of this cache capacity");
    const int groups = (pass.T * L.G + kTcaRows - 1) / kTcaRows;
    dim3 grid(chunks, kv.n_kv * groups, nprob);
    const size_t smem = TcaLayout<DH>::kBytes;
    static_assert(TcaLayout<128>::kBytes <= 227 * 1024, "attention tiles exceed the shared-memory opt-in");
    // row copies per tile: all four TMEM lane quarters busy for small passes
    // (ESPEC_ATTN_REP=1 forces one copy; the results do not depend on it)
    static const int rep_cap = [] {
        const char* e = std::getenv("ESPEC_ATTN_REP");
        return e ? std::atoi(e) : 4;
    }();
    const int P = pass.T * L.G;
    const int rep = groups > 1 ? 1 : (P <= 32 && rep_cap >= 4) ? 4 : (P <= 64 && rep_cap >= 2) ? 2 : 1;
    auto kernel = rep == 4 ? attn_tc_kernel<DH, 4> : rep == 2 ? attn_tc_kernel<DH, 2> : attn_tc_kernel<DH, 1>;
    static unsigned long long configured[3] = {0, 0, 0};
    ensure_smem((const void*)kernel, (int)smem, configured[rep >> 1]);
    // diagnostic: ESPEC_ATTN_TRACE=T,n traces the n-th launch with T pass rows
    // (kTcaTraceSlots %globaltimer stamps per CTA) into gpurun_out/attn_trace.txt
    static int tT = -1, tn = -1;
    static bool parsed = false;
    if (!parsed) {
        parsed = true;
        if (const char* e = std::getenv("ESPEC_ATTN_TRACE")) std::sscanf(e, "%d,%d", &tT, &tn);
    }
    static unsigned long long* tbuf = nullptr;
    static int seen = 0;
    const size_t nblk = (size_t)grid.x * grid.y * grid.z;
    bool traced = false;
    if (tn >= 0 && pass.T == tT && seen++ == tn && nblk <= 4096) {
        if (!tbuf) DEV_CK(cudaMalloc(&tbuf, sizeof(unsigned long long) * kTcaTraceSlots * 4096));
        DEV_CK(cudaMemset(tbuf, 0, sizeof(unsigned long long) * kTcaTraceSlots * 4096));
        DEV_CK(cudaDeviceSynchronize());
        L.trace = tbuf;
        traced = true;
    }
    L.cluster = attn_tc_cluster(chunks, pass.T);
    if (L.cluster == 2) {
        if ((size_t)grid.y * grid.z > (size_t)kTcaMaxTickets)
            dev_fail(DEV_ERR_CUDA, "attention: too many (problem, kv head) groups for the ticket combine");
        L.ticket = tca_tickets(s);
    }
    if (L.cluster == 1 && chunks > 8) {
        static bool nonportable[3] = {false, false, false};
        if (!nonportable[rep >> 1]) {
            DEV_CK(cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            nonportable[rep >> 1] = true;
        }
    }
    if (L.cluster == 1)
        DEV_CK(launch_pdl_cluster(kernel, grid, dim3(kTcaThreads), smem, s, chunks, L));
    else
        DEV_CK(launch_pdl(kernel, grid, dim3(kTcaThreads), smem, s, L));
    if (chunks > 1 && L.cluster == 0) {
        const int rows = std::min(kTcaRows, pass.T * L.G);
        DEV_CK(launch_pdl(attn_tc_combine_kernel<DH>, dim3((rows + 31) / 32, kv.n_kv * groups, nprob),
                          dim3(32 * (DH / 16)), 0, s, L, chunks));
    }
    if (traced) {
        std::vector<unsigned long long> h(kTcaTraceSlots * nblk);
        DEV_CK(cudaStreamSynchronize(s));
        DEV_CK(cudaMemcpy(h.data(), tbuf, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen("gpurun_out/attn_trace.txt", "w")) {
            std::fprintf(f, "grid %d %d %d T %d total %d ppi %d\n", grid.x, grid.y, grid.z, pass.T, pass.total,
                         kv.attn_ppi);
            for (size_t i = 0; i < nblk; ++i) {
                for (int e = 0; e < kTcaTraceSlots; ++e) std::fprintf(f, " %llu", h[i * kTcaTraceSlots + e]);
                std::fprintf(f, "\n");
            }
            std::fclose(f);
        }
    }
}

void launch_attention_tc(const AttnBatch& b, int nprob, int n_heads, const PassView& pass, const KvView& kv,
                         cudaStream_t s) {
    if (kv.dh == 128) attn_tc_launch<128>(b, nprob, n_heads, pass, kv, s);
    else attn_tc_launch<64>(b, nprob, n_heads, pass, kv, s);
}

}  // namespace espec_dev
