// Stream-K tensor-core GEMV for bf16 decode projections (sm_100a).
//
// y[T x N] = epilogue(norm?(x)[T x K] · W[K x N]) with T <= 16 rows and W
// streamed once from HBM. W is stored pre-packed in 1 KB core-matrix blocks
// (kernels.cu pack_index, the UMMA canonical K-major core-matrix layout): a
// 32-column group g is one contiguous run of K/16 1 KB blocks. The work is cut into *units* (problem, k-chunk j, group g) of
// up to kUnitBlocks blocks, ordered (problem, j, g) with g fastest, and every
// CTA of a persistent 1-CTA-per-SM grid takes one contiguous, balanced range
// of units (the split depends only on K, N and the problem count).
//
// Per CTA: one producer warp streams the CTA's weight bytes with 1-D TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx) through a 16-stage x 8 KB
// shared-memory ring — 128 KB in flight per SM without register pressure —
// while 8 consumer warps each take one 1 KB block per stage: ldmatrix the
// activation fragment from a staged bf16 copy of x, two ldmatrix.x4 for the
// weight fragments, four mma.m16n8k16 (fp32 accumulate). At the end of a unit
// the 8 warp accumulators are summed in fixed warp order through shared
// memory; units whose group is split over several k-chunks write a partial
// and the last-arriving CTA (per-group ticket) sums the partials in fixed
// k-chunk order. Every row's reduction order is therefore independent of T
// and of which CTA ran which unit (batch invariance).
//
// Programmatic dependent launch: the producer starts streaming weights
// before `griddepcontrol.wait`, so a GEMV's HBM pipeline fills while the
// previous kernel (which produces x) drains; consumers wait before reading x.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "sgemv_epi.cuh"

namespace espec_dev {

constexpr int kSgConsumers = 8;                    // warps 0-7: tensor-core consumers
constexpr int kSgProducer = kSgConsumers;          // warp 8: TMA producer
constexpr int kSgEpi = kSgConsumers + 1;           // warps 9..: unit epilogues, round-robin over units
// epilogue warps (= reduction buffers): 4 for <= 8 rows, 2 for 16 rows
// epilogue warps launched (the reduction buffers actually used, L.ne <= this,
// are chosen per launch: 2 for 13-16 rows so the weight ring keeps 4 stages)
template <int TM> constexpr int sg_ne() { return 4; }
template <int TM> constexpr int sg_threads() { return (kSgConsumers + 1 + sg_ne<TM>()) * 32; }
// Stage = 32 (TM=8; TM=16 by default) or 16 (TM=16, ESPEC_SG_SBLK16=16) 1 KB
// blocks, so one mbarrier wait (~90 cycles even when already complete) is
// amortised over several mma blocks (see sg_sblk).
constexpr int kSgMaxStages = 16;
constexpr int kSgSlots = 2;      // (problem, k-chunk) activation slots per CTA
constexpr int kSgMaxUnitBlocks = 128;              // 2048 k-rows per unit
constexpr int kSgSms = 148;
constexpr int kSgSmemLimit = 227 * 1024 - 2048;    // dynamic smem budget (static smem aside)

struct SgLaunch {
    GemvBatch b;
    PassView pass;
    KvView kv;
    int t0, T;
    int KT, kcb, nK, ngroups, units, xld, stages, rotate;
    int xrows;  // activation rows held per slot (rows >= xrows read zeros)
    int ef;     // weights loaded with an L2 evict-first policy (ESPEC_SG_EVICT_FIRST, default 1)
    int ne;     // epilogue warps / reduction buffers in use (<= sg_ne<TM>())
    int nslots; // activation slots (kSgSlots, or 1 with pair-aligned CTA ranges)
    int aligned;  // pair-aligned ranges: every CTA's static range lies in ONE (problem, k-chunk) pair
    int sblk;   // 1 KB blocks per ring stage (TM=8: 32; TM=16: 16 or 32, see sg_sblk)
    int rrows;  // rows per warp in a reduction buffer (TM=8: 8; TM=16: the pass rows)
    unsigned long long* trace;  // diagnostic timeline (ESPEC_SG_TRACE) or nullptr
    // Tail pool (ESPEC_SG_POOL): the last pool_f groups of every (problem,
    // k-chunk) pair are not in any CTA's static range; CTAs that hold the
    // pair's activations claim them one by one (pool_ctr[pair]) after their
    // static range, absorbing the spread in per-SM finish times. A unit's sums
    // do not depend on which CTA computes it (bitwise-identical results).
    int pool_f, nstatic;
    unsigned* pool_ctr;
};

constexpr int kSgPoolBanks = 16, kSgPoolPairs = 512;
__device__ unsigned g_sg_pool[kSgPoolBanks * kSgPoolPairs];

SgPlan sgemv_plan(int K, int ldw, int nprob) {
    SgPlan p;
    p.KT = (K + 15) / 16;
    p.ngroups = ldw / 32;
    // Largest unit (<= 128 blocks = 2048 k-rows) that still leaves >= 2 units
    // per SM, so the contiguous per-CTA ranges balance to within a few %.
    // Depends on (K, N) only: the reduction tree never depends on T.
    static const int min_units = [] {
        const char* e = std::getenv("ESPEC_SG_UNITS_PER_SM");
        return e ? std::atoi(e) : 2;
    }();
    int kcb = kSgMaxUnitBlocks;
    while (kcb > 8 && (long long)p.ngroups * ((p.KT + kcb - 1) / kcb) < (long long)min_units * kSgSms) kcb /= 2;
    if (kcb > p.KT) kcb = p.KT;
    p.kcb = kcb;
    p.nK = (p.KT + kcb - 1) / kcb;
    p.units = nprob * p.nK * p.ngroups;
    p.grid = p.units < kSgSms ? p.units : kSgSms;
    // every CTA range must touch at most kSgSlots (problem, k-chunk) pairs
    for (int c = 0; c < p.grid; ++c) {
        const long long s = (long long)c * p.units / p.grid, e = (long long)(c + 1) * p.units / p.grid;
        if (e > s && (e - 1) / p.ngroups - s / p.ngroups + 1 > kSgSlots)
            throw std::runtime_error("sgemv_plan: K x problems too large for the activation slots");
    }
    return p;
}

// Wide plan (drafter only, see set_sgemv_wide): T-dependent units as long as
// the activation slots hold just the pass's T rows — usually the whole K in
// ONE unit, so no split-K partials, tickets or end-of-launch reductions. The
// smallest k-chunk count whose per-CTA load is within 20% of the mean is
// taken, never more chunks than the (K, N) plan (workspace bound).
static constexpr int kWideSlotBytes = 64 * 1024;
static bool sgemv_plan_wide(int K, int ldw, int nprob, int T, SgPlan& out) {
    const SgPlan base = sgemv_plan(K, ldw, nprob);
    SgPlan p = base;
    for (int nK = 1; nK <= base.nK; ++nK) {
        const int kcb = (p.KT + nK - 1) / nK;
        if ((long long)kSgSlots * T * (kcb * 16 + 8) * 2 > kWideSlotBytes) continue;
        const long long units = (long long)nprob * nK * p.ngroups;
        const long long waves = (units + kSgSms - 1) / kSgSms;
        if (waves * kSgSms * 5 > units * 6) continue;  // > 20% imbalance
        p.kcb = kcb;
        p.nK = (p.KT + kcb - 1) / kcb;
        p.units = nprob * p.nK * p.ngroups;
        p.grid = p.units < kSgSms ? p.units : kSgSms;
        bool ok = true;
        for (int c = 0; c < p.grid && ok; ++c) {
            const long long s0 = (long long)c * p.units / p.grid, e0 = (long long)(c + 1) * p.units / p.grid;
            if (e0 > s0 && (e0 - 1) / p.ngroups - s0 / p.ngroups + 1 > kSgSlots) ok = false;
        }
        if (!ok) continue;
        out = p;
        return true;
    }
    return false;
}

static thread_local bool g_wide = false;
void set_sgemv_wide(bool on) { g_wide = on; }

size_t sgemv_partial_floats(int K, int ldw) {
    const SgPlan p = sgemv_plan(K, ldw, 1);
    return p.nK > 1 ? (size_t)p.nK * 16 * ldw : 0;
}

// smem = ring (stages x 8 KB) + activation slots (xrows rows) + reduction buffers
static int sg_ne_used(int TM, int xrows, int ns) {
    static const int big = [] {  // epilogue warps for 13-16 rows (ESPEC_SG_NE16; default 4 with one slot, else 3)
        const char* e = std::getenv("ESPEC_SG_NE16");
        return e ? std::max(1, std::min(4, std::atoi(e))) : 0;
    }();
    static const int mid = [] {  // epilogue warps for 9-12 rows (ESPEC_SG_NE9)
        const char* e = std::getenv("ESPEC_SG_NE9");
        return e ? std::max(1, std::min(4, std::atoi(e))) : 4;
    }();
    if (TM == 8) return 4;
    return xrows > 12 ? (big ? big : ns == 1 ? 4 : 3) : mid;
}
// Reduction buffers hold only the rows a pass has (rows >= T are never read
// back): at T = 9-12 that is up to 28 KB more weight ring per SM.
static int sg_red_rows(int TM, int xrows) { return TM == 8 ? 8 : xrows; }
static size_t sg_fixed_bytes(int TM, int kcb, int xrows, int ns) {
    return (size_t)ns * xrows * (kcb * 16 + 8) * 2 +
           (size_t)sg_ne_used(TM, xrows, ns) * kSgConsumers * sg_red_rows(TM, xrows) * 32 * 4;
}
// 16-row stages: 32 blocks (one 32-block group: every consumer warp takes its
// 4-block run each stage) whenever two such stages fit, else 16 blocks (half a
// group; half of the warps sit a stage out). Measured at T = 9 (C2 base
// gate/up): 16-block stages 178 us, 32-block 157 us. ESPEC_SG_SBLK16=16 forces
// the 16-block stages.
static int sg_sblk(int TM, int kcb, int xrows, int ns) {
    static const int force16 = [] {
        const char* e = std::getenv("ESPEC_SG_SBLK16");
        return e && std::atoi(e) == 16;
    }();
    if (TM == 8) return 32;
    const long long room = (long long)kSgSmemLimit - (long long)sg_fixed_bytes(TM, kcb, xrows, ns);
    return !force16 && room >= 2 * 32 * 1024 ? 32 : 16;
}
static int sg_stage_bytes(int TM, int kcb, int xrows, int ns) { return sg_sblk(TM, kcb, xrows, ns) * 1024; }
static int sg_stages(int TM, int kcb, int xrows, int ns) {
    const long long room = (long long)kSgSmemLimit - (long long)sg_fixed_bytes(TM, kcb, xrows, ns);
    int st = (int)(room / sg_stage_bytes(TM, kcb, xrows, ns));
    if (st > kSgMaxStages) st = kSgMaxStages;
    if (st < 2) throw std::runtime_error("sgemv: shared memory too small for the weight ring");
    return st;
}
static size_t sg_smem_bytes(int TM, int kcb, int xrows, int ns) {
    return (size_t)sg_stages(TM, kcb, xrows, ns) * sg_stage_bytes(TM, kcb, xrows, ns) + sg_fixed_bytes(TM, kcb, xrows, ns);
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------

// Diagnostic timeline (ESPEC_SG_TRACE, tools/sg_trace.py): per CTA,
// %globaltimer (max over the recording threads) at 0 CTA start, 1 consumers
// past griddepcontrol.wait, 2 activations staged, 3 consumers done,
// 4 epilogue warps done.
constexpr int kSgTraceEv = 16;
__device__ __forceinline__ void sg_tr(unsigned long long* tr, int ev) {
    if (tr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        atomicMax(tr + (size_t)blockIdx.x * kSgTraceEv + ev, t);
    }
}

template <int TM, int EPI, int SB>
__global__ void __launch_bounds__(sg_threads<TM>(), 1) sgemv_kernel(const __grid_constant__ SgLaunch L) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full_bar[kSgMaxStages];
    __shared__ __align__(8) uint64_t empty_bar[kSgMaxStages];
    constexpr int NE = sg_ne<TM>();
    __shared__ __align__(8) uint64_t red_full[NE];
    __shared__ __align__(8) uint64_t red_empty[NE];
    __shared__ __align__(16) uint4 s_xzero[2];  // 32 zero bytes: A rows a slot does not hold

    constexpr int kStageBlocks = SB;  // == L.sblk (compile-time: a runtime stage size costs 13 % at T = 16)
    constexpr int kStageBytes = kStageBlocks * 1024;
    const int stages = L.stages;
    unsigned char* ring = sm;
    __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm + (size_t)stages * kStageBytes);
    const int xslot = L.xrows * L.xld;  // elements per activation slot
    // 8-row passes always use two slots and balanced ranges (compile-time, so
    // their code is unchanged by the 16-row options)
    const bool aligned = TM == 16 && L.aligned;
    const int nslots = TM == 8 ? kSgSlots : L.nslots;
    float* red = reinterpret_cast<float*>(sm + (size_t)stages * kStageBytes + (size_t)nslots * xslot * 2);
    const int RR = TM == 8 ? 8 : L.rrows;           // rows per warp slice of a reduction buffer
    const int kRedBuf = kSgConsumers * RR * 32;     // floats per reduction buffer

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nlin = L.pool_f ? L.nstatic : L.units;  // static (range-assigned) units
    const int Gs = L.ngroups - L.pool_f;              // static groups per pair
    // static index -> unit (pair-major, groups [0, Gs) of every pair)
    auto sunit = [&](int x) { return (x / Gs) * L.ngroups + x % Gs; };
    // Pair-aligned ranges (L.aligned): pair p owns CTAs [p*G/np, (p+1)*G/np)
    // and splits its Gs static groups evenly over them.
    auto pcta0 = [&](int pr) { return (int)((long long)pr * gridDim.x / (nlin / Gs)); };
    int start, end;
    if (aligned) {
        const int npairs = nlin / Gs;
        const int pr = (int)(((long long)(blockIdx.x + 1) * npairs - 1) / gridDim.x);
        const int c0 = pcta0(pr), np = pcta0(pr + 1) - c0, c = (int)blockIdx.x - c0;
        start = pr * Gs + (int)((long long)c * Gs / np);
        end = pr * Gs + (int)((long long)(c + 1) * Gs / np);
    } else {
        start = (int)((long long)blockIdx.x * nlin / gridDim.x);
        end = (int)((long long)(blockIdx.x + 1) * nlin / gridDim.x);
    }
    const int pair0 = sunit(start) / L.ngroups;
    __shared__ int s_stage_unit[kSgMaxStages];  // pool units: unit id of the stage that starts it (-1: done)
    __shared__ int s_red_unit[sg_ne<TM>()];     // pool units: unit id handed to epilogue warp e (-1: done)
    // Processing order: the range rotated so that units with g = 0 (mod R),
    // R the nominal range length, come first. Every CTA then handles group g
    // near step (g mod R) whatever its k-chunk, so the k-chunks of one group
    // finish at about the same time and the final (last-chunk) reductions are
    // spread over the kernel instead of piling up at its end.
    const int len = end - start;
    const int R = (nlin + gridDim.x - 1) / gridDim.x;
    int off = L.rotate && !L.pool_f && !aligned ? (R - (start % L.ngroups) % R) % R : 0;
    if (off >= len) off = 0;

    if (tid < 2) s_xzero[tid] = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kSgConsumers);
        }
        for (int e = 0; e < L.ne; ++e) {
            mbar_init(&red_full[e], kSgConsumers);
            mbar_init(&red_empty[e], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) sg_tr(L.trace, 0);
    // let the next kernel in the stream start its weight prefetch early
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == kSgProducer) {
        // ---------------- producer: stream this CTA's weight range (no dependency on earlier kernels)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t pol = l2_policy_evict_first();
            auto stream_unit = [&](int u) {
                const int g = u % L.ngroups, pair = u / L.ngroups;
                const int prob = pair / L.nK, j = pair - prob * L.nK;
                const int kb0 = j * L.kcb, nb = min(L.kcb, L.KT - kb0);
                const char* src = reinterpret_cast<const char*>(L.b.p[prob].W) + ((size_t)g * L.KT + kb0) * 1024;
                for (int b = 0; b < nb; b += kStageBlocks) {
                    const uint32_t bytes = (uint32_t)min(kStageBlocks, nb - b) * 1024u;
                    mbar_wait(&empty_bar[stage], phase ^ 1u);
                    if (b == 0) s_stage_unit[stage] = u;  // released by the arrive below
                    mbar_arrive_expect_tx(&full_bar[stage], bytes);
                    if (L.ef)
                        tma_bulk_g2s_hint(ring + (size_t)stage * kStageBytes, src + (size_t)b * 1024, bytes,
                                          &full_bar[stage], pol);
                    else
                        tma_bulk_g2s(ring + (size_t)stage * kStageBytes, src + (size_t)b * 1024, bytes, &full_bar[stage]);
                    if (++stage == stages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            };
            for (int i = 0; i < len; ++i) stream_unit(sunit(start + (i + off) % len));
            if (L.pool_f) {
                // claim the pool units of the pairs this CTA holds; the last of
                // the F + (CTAs holding the pair) claims resets the counter
                auto cta_of = [&](long long x) { return (int)(((x + 1) * gridDim.x - 1) / nlin); };
                const int p_hi = len > 0 ? sunit(end - 1) / L.ngroups : pair0 - 1;
                for (int pr = p_hi; pr >= pair0 && len > 0; --pr) {
                    const unsigned holders =
                        aligned ? (unsigned)(pcta0(pr + 1) - pcta0(pr))
                                  : (unsigned)(cta_of((long long)(pr + 1) * Gs - 1) - cta_of((long long)pr * Gs) + 1);
                    for (;;) {
                        const unsigned k = atomicAdd(&L.pool_ctr[pr], 1u);
                        if (k == (unsigned)L.pool_f + holders - 1u) atomicExch(&L.pool_ctr[pr], 0u);
                        if (k >= (unsigned)L.pool_f) break;
                        stream_unit(pr * L.ngroups + Gs + (int)k);
                    }
                }
                // sentinel stage: no data, unit -1
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                s_stage_unit[stage] = -1;
                mbar_arrive(&full_bar[stage]);
            }
        }
        return;
    }

    // x, stats, workspaces and outputs are shared with earlier kernels
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) sg_tr(L.trace, 1);

    if (warp >= kSgEpi) {
        // ---------------- epilogue warps: warp 9 finishes even units, warp 10 odd units
        const int e = warp - kSgEpi;
        uint32_t phase = 0;
        if (e >= L.ne) return;
        __shared__ int s_pos[16];
        __shared__ long long s_kvrow[16];
        __shared__ float s_rms[kMaxProblems][TM];
        // RMSNorm prologue, second half: the consumers staged x * gain (no
        // statistics on their critical path); each row's 1/rms scales its sums
        // here. Computed once per CTA while the consumers run their first unit.
        const int nprob = L.units / (L.ngroups * L.nK);
        for (int q = e; q < nprob * TM; q += L.ne) {
            const int pb = q / TM, t = q - pb * TM;
            const GemvProblem& P = L.b.p[pb];
            float r = 1.f;
            if (P.gain != nullptr && t < L.T) {
                float ss = 0.f;
                const float* st = P.stats_in + (size_t)(L.t0 + t) * P.stat_tiles_in;
#pragma unroll 8
                for (int i = lane; i < P.stat_tiles_in; i += 32) ss += __ldcg(st + i);
                ss = warp_sum(ss);
                r = 1.0f / sqrtf(ss / (float)P.K + P.eps);
            }
            if (lane == 0) s_rms[pb][t] = r;
        }
        if constexpr (EPI == EPI_QKV) {
            // the pass's row metadata (rotary position, paged-KV row base),
            // once per CTA while the consumers run their first unit — not two
            // dependent loads on every unit's epilogue
            if (e == 0 && lane < L.T) {
                s_pos[lane] = L.pass.pos[L.t0 + lane];
                const int row = L.pass.rows[L.t0 + lane];
                s_kvrow[lane] = (long long)L.kv.page_table[row / L.kv.page_rows] * L.kv.page_elems +
                                (long long)(row % L.kv.page_rows) * L.kv.dh;
            }
        }
        named_bar(3, L.ne * 32);
        constexpr bool kResid = TM == 8 && (EPI == EPI_RESID || EPI == EPI_STORE);
        int i = e;
        for (;; i += L.ne) {
            const bool pooled = i >= len;
            if (pooled && !L.pool_f) break;
            int u;
            if (pooled) {
                // pool unit: its id arrives with its sums
                mbar_wait(&red_full[e], phase);
                u = s_red_unit[e];
                if (u < 0) break;
            } else {
                u = sunit(start + (i + off) % len);
            }
            const int g = u % L.ngroups, pair = u / L.ngroups;
            const int prob = pair / L.nK, j = pair - prob * L.nK;
            const GemvProblem& P = L.b.p[prob];
            // residual rows of this unit's columns, loaded before its sums
            // arrive (only the unit's finisher writes them, so they are final)
            float pre[TM];
            if constexpr (kResid) {
                const int c = g * 32 + lane;
#pragma unroll
                for (int t = 0; t < TM; ++t)
                    pre[t] = t < L.T && c < P.N && P.resid != nullptr ? __ldcg(P.resid + (size_t)(L.t0 + t) * P.ldr + c) : 0.f;
            }
            // QKV: the rotary factors of this unit's column (q / k regions)
            float2 rope[TM];
            if constexpr (EPI == EPI_QKV && TM == 8) {
                const int c = g * 32 + lane;
                const int i = (c % P.dh) >> 1;  // q and k regions start at multiples of dh
                const bool rot = c < (P.n_heads + P.n_kv) * P.dh;
#pragma unroll
                for (int t = 0; t < TM; ++t)
                    rope[t] = rot && t < L.T ? P.rope[(size_t)s_pos[t] * (P.dh >> 1) + i] : make_float2(1.f, 0.f);
            }
            if (!pooled) mbar_wait(&red_full[e], phase);
            phase ^= 1u;
            const float* rb = red + e * kRedBuf;
            float v[TM];
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                float acc = 0.f;
#pragma unroll
                if (t < RR)
                    for (int w = 0; w < kSgConsumers; ++w) acc += rb[(w * RR + t) * 32 + lane];
                v[t] = acc;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&red_empty[e]);
            if (L.nK > 1) {
                // partial for (j, g); the last of the nK chunks of group g finishes it
                const int ldw = L.ngroups * 32;
                float* pp = P.partial + (size_t)j * 16 * ldw + g * 32 + lane;
#pragma unroll
                for (int t = 0; t < TM; ++t)
                    if (t < L.T) pp[(size_t)t * ldw] = v[t];
                __syncwarp();
                unsigned last = 0;
                if (lane == 0) {
                    last = ticket_acq_rel(&P.tickets[g]) == (unsigned)L.nK - 1 ? 1u : 0u;
                    if (last) P.tickets[g] = 0u;
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (!last) continue;
                // sum the nK partials in fixed k-chunk order; loads batched so
                // they are all in flight together
                const float* q = P.partial + g * 32 + lane;
#pragma unroll
                for (int t = 0; t < TM; ++t) v[t] = 0.f;
                constexpr int JB = TM == 8 ? 4 : 4;  // chunks per batch of loads
                for (int jj = 0; jj < L.nK; jj += JB) {
                    float ld[JB][TM];
#pragma unroll
                    for (int c = 0; c < JB; ++c)
#pragma unroll
                        for (int t = 0; t < TM; ++t)
                            ld[c][t] = (jj + c < L.nK && t < L.T) ? __ldcg(q + ((size_t)(jj + c) * 16 + t) * ldw) : 0.f;
#pragma unroll
                    for (int c = 0; c < JB; ++c)
#pragma unroll
                        for (int t = 0; t < TM; ++t)
                            if (jj + c < L.nK) v[t] += ld[c][t];
                }
            }
            if (P.gain != nullptr)
#pragma unroll
                for (int t = 0; t < TM; ++t) v[t] = __fmul_rn(v[t], s_rms[prob][t]);
            SgEpiCtx ctx{L.pass, L.kv, L.T, L.t0, L.ngroups};
            if constexpr (EPI == EPI_QKV) {
                ctx.pos = s_pos;
                ctx.kv_row = s_kvrow;
                if (TM == 8) ctx.rope = rope;
            }
            if constexpr (kResid) ctx.pre = pre;
            sg_epilogue<TM, EPI>(ctx, P, g, v, lane);
        }
        if (lane == 0) sg_tr(L.trace, 4);
        return;
    }

    // ---------------- consumers (warps 0-7)
    const int T = L.T, t0 = L.t0;
    const int pair1 = end > start ? sunit(end - 1) / L.ngroups : pair0;
    const int kc = L.kcb * 16;
    for (int s = 0; s <= pair1 - pair0; ++s) {
        const int pair = pair0 + s, prob = pair / L.nK, j = pair - prob * L.nK;
        const GemvProblem& P = L.b.p[prob];
        __nv_bfloat16* xd = xs + (size_t)s * xslot;
        const int k0 = j * kc;
        const int kq = kc >> 2;
        // rows >= T are zero
        for (int i = T * kq + tid; i < L.xrows * kq; i += kSgConsumers * 32) {
            const int t = i / kq, kk = (i - t * kq) * 4;
            *reinterpret_cast<uint2*>(xd + t * L.xld + kk) = make_uint2(0u, 0u);
        }
        constexpr int NT = kSgConsumers * 32;
        if (P.x_bf16) {
            // activations already bf16 (producer-rounded): straight copy
            constexpr int U = TM == 8 ? 16 : 8;
            const __nv_bfloat16* xb16 = reinterpret_cast<const __nv_bfloat16*>(P.x);
            for (int i0 = tid; i0 < T * kq; i0 += NT * U) {
                uint2 v[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int i = i0 + q * NT;
                    const int t = i / kq, k = k0 + (i - t * kq) * 4;
                    v[q] = make_uint2(0u, 0u);
                    if (i < T * kq && k < P.K) v[q] = __ldcg(reinterpret_cast<const uint2*>(xb16 + (size_t)(t0 + t) * P.ldx + k));
                }
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int i = i0 + q * NT;
                    if (i >= T * kq) break;
                    const int t = i / kq, kk = (i - t * kq) * 4;
                    *reinterpret_cast<uint2*>(xd + t * L.xld + kk) = v[q];
                }
            }
            continue;
        }
        // fp32 rows with the RMSNorm prologue's first half: x * gain rounded to
        // bf16 (the epilogue applies each row's 1/rms to its sums, so the row
        // statistics are off the consumers' critical path), batches of U
        // independent row and gain loads per thread in flight per round trip
        constexpr int U = TM == 8 ? 8 : 4;  // (the 16-row variant's registers are tighter)
        for (int i0 = tid; i0 < T * kq; i0 += NT * U) {
            float4 v[U], gn[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int i = i0 + q * NT;
                const int t = i / kq, k = k0 + (i - t * kq) * 4;
                v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                gn[q] = make_float4(1.f, 1.f, 1.f, 1.f);
                if (i < T * kq && k < P.K) {  // K is a multiple of 16
                    v[q] = __ldcg(reinterpret_cast<const float4*>(P.x + (size_t)(t0 + t) * P.ldx + k));
                    if (P.gain != nullptr) gn[q] = __ldg(reinterpret_cast<const float4*>(P.gain + k));
                }
            }
            if (tid == 0 && s == 0 && i0 == tid && L.trace) {  // diagnostic: the first rows landed
                if (v[0].x + gn[U - 1].w == 12345.f) asm volatile("trap;");
                sg_tr(L.trace, 5);
            }
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int i = i0 + q * NT;
                if (i >= T * kq) break;
                const int t = i / kq, kk = (i - t * kq) * 4;
                float4 w = v[q];
                if (P.gain != nullptr) {
                    w.x = __fmul_rn(w.x, gn[q].x);
                    w.y = __fmul_rn(w.y, gn[q].y);
                    w.z = __fmul_rn(w.z, gn[q].z);
                    w.w = __fmul_rn(w.w, gn[q].w);
                }
                const __nv_bfloat162 lo = __floats2bfloat162_rn(w.x, w.y), hi = __floats2bfloat162_rn(w.z, w.w);
                uint2 pk;
                pk.x = *reinterpret_cast<const uint32_t*>(&lo);
                pk.y = *reinterpret_cast<const uint32_t*>(&hi);
                *reinterpret_cast<uint2*>(xd + t * L.xld + kk) = pk;
            }
            if (tid == 0 && s == 0 && i0 == tid && L.trace) sg_tr(L.trace, 6);  // diagnostic: the first batch stored
        }
    }
    named_bar(1, kSgConsumers * 32);
    if (tid == 0) sg_tr(L.trace, 2);

    int stage = 0;
    uint32_t phase = 0;
    uint32_t rphase[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) rphase[e] = 0u;
    const int gid = lane >> 2, tig = lane & 3;
    int i = 0;
    for (;; ++i) {
        const bool pooled = i >= len;
        if (pooled && !L.pool_f) break;
        int u;
        if (pooled) {
            // pool unit (or the producer's end sentinel) announced with its first stage
            mbar_wait(&full_bar[stage], phase);
            u = s_stage_unit[stage];
            if (u < 0) break;
        } else {
            u = sunit(start + (i + off) % len);
        }
        const int pair = u / L.ngroups;
        const int j = pair % L.nK;
        const int nb = min(L.kcb, L.KT - j * L.kcb);
        const __nv_bfloat16* xb = xs + (size_t)(pair - pair0) * xslot;
        const int xr = TM == 16 ? (lane & 7) + ((lane >> 3) & 1) * 8 : (lane & 7);  // ldmatrix row of this lane
        const bool xz = xr >= L.xrows;  // row not held: read the zero block
        const __nv_bfloat16* xrow = TM == 16 ? xb + xr * L.xld + (lane >> 4) * 8 : xb + xr * L.xld + ((lane >> 3) & 1) * 8;
        const uint32_t xzero = smem_u32(&s_xzero[0]);
        float acc[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
        for (int b = 0; b < nb; b += kStageBlocks) {
            if (!(pooled && b == 0)) mbar_wait(&full_bar[stage], phase);
            // This warp's run of 4 blocks. Both row variants use the SAME
            // block -> warp map (warp w owns blocks 4w..4w+3 of every 32-block
            // group of the unit; the 16-row variant's 16-block stages hold half
            // a group, so half of the warps sit a stage out), hence the same
            // per-row sum order whatever the pass size (batch invariance).
            constexpr int kRun = 4;
            const int bbase = TM == 8 || kStageBlocks == 32
                                  ? warp * kRun
                                  : (((b / kStageBlocks) & 1) == (warp >> 2) ? (warp & 3) * kRun : kStageBlocks);
            uint32_t w[kRun][8];
            uint32_t a[kRun][4];
#pragma unroll
            for (int i = 0; i < kRun; ++i) {
                const int bi = bbase + i;
                if (bi < kStageBlocks && b + bi < nb) {
                    // canonical K-major block: core matrices (n8, khalf) at
                    // (2*n8 + khalf)*128 B -> b0/b1 of n8 tiles 0,1 then 2,3
                    const uint32_t wb = smem_u32(ring + (size_t)stage * kStageBytes + bi * 1024 + lane * 16);
                    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                                 : "r"(wb));
                    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(w[i][4]), "=r"(w[i][5]), "=r"(w[i][6]), "=r"(w[i][7])
                                 : "r"(wb + 512));
                    const uint32_t xa = xz ? xzero : smem_u32(xrow + (b + bi) * 16);
                    if constexpr (TM == 16) {
                        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(a[i][0]), "=r"(a[i][1]), "=r"(a[i][2]), "=r"(a[i][3])
                                     : "r"(xa));
                    } else {
                        asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                                     : "=r"(a[i][0]), "=r"(a[i][2])
                                     : "r"(xa));
                        a[i][1] = a[i][3] = 0u;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < kRun; ++i) {
                if (bbase + i < kStageBlocks && b + bbase + i < nb) {
                    mma16816(acc[0], a[i], w[i][0], w[i][1]);
                    mma16816(acc[1], a[i], w[i][2], w[i][3]);
                    mma16816(acc[2], a[i], w[i][4], w[i][5]);
                    mma16816(acc[3], a[i], w[i][6], w[i][7]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[stage]);
            if (++stage == stages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        // hand the warp's partial sums to this unit's epilogue warp
        const int e = i % L.ne;
        mbar_wait(&red_empty[e], rphase[e] ^ 1u);
        rphase[e] ^= 1u;
        float* rw = red + e * kRedBuf + warp * RR * 32;
        if (warp == 0 && lane == 0) s_red_unit[e] = u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int col = q * 8 + 2 * tig;
            rw[gid * 32 + col] = acc[q][0];
            rw[gid * 32 + col + 1] = acc[q][1];
            if (TM == 16 && gid + 8 < RR) {
                rw[(gid + 8) * 32 + col] = acc[q][2];
                rw[(gid + 8) * 32 + col + 1] = acc[q][3];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&red_full[e]);
    }
    if (L.pool_f) {
        // end sentinel to every epilogue warp (each waits on its next index)
        for (int q = 0; q < L.ne; ++q) {
            const int e = (i + q) % L.ne;
            mbar_wait(&red_empty[e], rphase[e] ^ 1u);
            rphase[e] ^= 1u;
            if (warp == 0 && lane == 0) s_red_unit[e] = -1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&red_full[e]);
        }
    }
    if (lane == 0) sg_tr(L.trace, 3);
}

// ---------------------------------------------------------------------------
// host launch
// ---------------------------------------------------------------------------

static bool g_pdl = true;
void set_pdl(bool on) { g_pdl = on; }
bool pdl_enabled() { return g_pdl; }

template <int TM, int EPI, int SB>
static void sg_launch_t(const SgLaunch& L, int grid, size_t smem, cudaStream_t s) {
    static unsigned long long configured = 0;
    ensure_smem((const void*)sgemv_kernel<TM, EPI, SB>, kSgSmemLimit, configured);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(sg_threads<TM>());
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DEV_CK(cudaLaunchKernelEx(&cfg, sgemv_kernel<TM, EPI, SB>, L));
}

template <int TM, int SB>
static void sg_dispatch(int epi, const SgLaunch& L, int grid, size_t smem, cudaStream_t s) {
    switch (epi) {
        case EPI_STORE: sg_launch_t<TM, EPI_STORE, SB>(L, grid, smem, s); break;
        case EPI_RESID: sg_launch_t<TM, EPI_RESID, SB>(L, grid, smem, s); break;
        case EPI_SILU: sg_launch_t<TM, EPI_SILU, SB>(L, grid, smem, s); break;
        case EPI_QKV: sg_launch_t<TM, EPI_QKV, SB>(L, grid, smem, s); break;
        case EPI_ARGMAX: sg_launch_t<TM, EPI_ARGMAX, SB>(L, grid, smem, s); break;
    }
}

// ESPEC_SG_TRACE="K,N,T,n[,cnt]": trace cnt consecutive launches (any shape)
// starting at the n-th launch of that shape; the buffer is allocated and
// zeroed up front so the traced launches sit in an undisturbed stream.
static struct {
    int K = -1, N = -1, T = -1, n = -1, cnt = 1, next = -1, seen = 0;
    unsigned long long* buf = nullptr;
    std::string head;
} g_trace;

static int sg_trace_slot(const GemvBatch& b, int nprob, int T, int epi, const SgPlan& p) {
    static bool parsed = false;
    if (!parsed) {
        parsed = true;
        if (const char* e = std::getenv("ESPEC_SG_TRACE")) {
            std::sscanf(e, "%d,%d,%d,%d,%d", &g_trace.K, &g_trace.N, &g_trace.T, &g_trace.n, &g_trace.cnt);
            const size_t bytes = sizeof(unsigned long long) * kSgTraceEv * kSgSms * g_trace.cnt;
            cudaMalloc(&g_trace.buf, bytes);
            cudaMemset(g_trace.buf, 0, bytes);
            cudaDeviceSynchronize();
        }
    }
    if (!g_trace.buf) return -1;
    if (g_trace.next < 0 && b.p[0].K == g_trace.K && b.p[0].N == g_trace.N && T == g_trace.T &&
        g_trace.seen++ == g_trace.n)
        g_trace.next = 0;
    if (g_trace.next < 0 || g_trace.next >= g_trace.cnt) return -1;
    char hd[160];
    std::snprintf(hd, sizeof hd, "epi %d K %d N %d T %d nprob %d units %d nK %d grid %d\n", epi, b.p[0].K, b.p[0].N, T,
                  nprob, p.units, p.nK, p.grid);
    g_trace.head += hd;
    return g_trace.next++;
}

static void sg_trace_dump(cudaStream_t s) {
    std::vector<unsigned long long> h((size_t)kSgTraceEv * kSgSms * g_trace.cnt);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), g_trace.buf, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen("gpurun_out/sg_trace.txt", "w")) {
        std::fputs(g_trace.head.c_str(), f);
        for (size_t r = 0; r < h.size() / kSgTraceEv; ++r) {
            for (int e = 0; e < kSgTraceEv; ++e) std::fprintf(f, " %llu", h[r * kSgTraceEv + e]);
            std::fprintf(f, "\n");
        }
        std::fclose(f);
    }
}

size_t sgemv_pool_words() { return (size_t)kSgPoolBanks * kSgPoolPairs; }

void sgemv_pool_reset(SgPool& p, cudaStream_t s) {
    if (p.dev) DEV_CK(cudaMemsetAsync(p.dev, 0, sizeof(unsigned) * sgemv_pool_words(), s));
    p.next = 0;
}

void launch_sgemv(int epi, const GemvBatch& b, int nprob, int T, const PassView& pass, const KvView& kv,
                  cudaStream_t s, SgPool* pool) {
    if (T <= 0 || nprob <= 0) return;
    SgPlan p = sgemv_plan(b.p[0].K, b.p[0].ldw, nprob);
    bool wide = false;
    if (g_wide && T <= 8) wide = sgemv_plan_wide(b.p[0].K, b.p[0].ldw, nprob, T, p);
    SgLaunch L;
    L.b = b;
    L.pass = pass;
    L.kv = kv;
    L.KT = p.KT;
    L.kcb = p.kcb;
    L.nK = p.nK;
    L.ngroups = p.ngroups;
    L.units = p.units;
    L.xld = p.kcb * 16 + 8;
    static const int rotate = [] {
        const char* e = std::getenv("ESPEC_SG_ROTATE");
        return e ? std::atoi(e) : 0;  // measured slower on B200 (DRAM locality); off by default
    }();
    L.rotate = rotate;
    // tail pool (see SgLaunch): ESPEC_SG_POOL = percent of each pair's groups
    // (12 % measured best of 8 / 12 / 16: -1.5 % per EasySpec step, -4 % vanilla)
    static const int pool_pct = [] {
        const char* e = std::getenv("ESPEC_SG_POOL");
        return e ? std::atoi(e) : 12;
    }();
    L.pool_f = 0;
    L.nstatic = p.units;
    L.pool_ctr = nullptr;
    {
        const int npairs = p.units / p.ngroups;
        const int F = p.ngroups * pool_pct / 100;
        const int Gs = p.ngroups - F;
        const long long ns = (long long)npairs * Gs;
        bool ok = pool_pct > 0 && F >= 1 && Gs >= 1 && p.units >= 4 * p.grid && npairs <= kSgPoolPairs && ns >= p.grid;
        for (int c = 0; c < p.grid && ok; ++c) {
            const long long s0 = (long long)c * ns / p.grid, e0 = (long long)(c + 1) * ns / p.grid;
            if (e0 > s0 && (e0 - 1) / Gs - s0 / Gs + 1 > kSgSlots) ok = false;
        }
        if (ok) {
            L.pool_f = F;
            L.nstatic = (int)ns;
        }
    }
    static SgPool g_pool[64];  // pool == nullptr: per-device process-wide banks
    if (L.pool_f && !pool) {
        int dev = 0;
        DEV_CK(cudaGetDevice(&dev));
        pool = &g_pool[dev & 63];
        if (!pool->dev) {
            void* a = nullptr;
            DEV_CK(cudaGetSymbolAddress(&a, g_sg_pool));
            pool->dev = static_cast<unsigned*>(a);
        }
    }
    static const int align16 = [] {
        const char* e = std::getenv("ESPEC_SG_ALIGN16");
        return e ? std::atoi(e) : 1;
    }();
    for (int t0 = 0; t0 < T; t0 += 16) {
        L.t0 = t0;
        // a fresh counter bank per pass: a pass's producers claim pool units
        // before griddepcontrol.wait, i.e. possibly while the previous pass
        // (same call or previous launch) is still claiming from its bank
        if (L.pool_f) L.pool_ctr = pool->dev + (size_t)(pool->next++ % kSgPoolBanks) * kSgPoolPairs;
        L.T = T - t0 < 16 ? T - t0 : 16;
        const int TM = L.T <= 8 ? 8 : 16;
        L.xrows = L.T;  // slots hold only the pass rows (layout only: the plan, hence every sum, is unchanged)
        // 16-row passes: pair-aligned CTA ranges need ONE activation slot, so
        // T x 4 KB more weight ring per SM (the ring depth bounds these
        // launches). A unit's sums do not depend on which CTA runs it, so this
        // is layout only. Taken when the largest per-CTA load is no larger than
        // with balanced ranges (pairs get floor/ceil(G / npairs) CTAs) and the two-slot
        // ring is under 96 KB. Measured (isolated, C2 base): gate/up T = 16
        // 214 -> 167 us, head 463 -> 376 us; the 14-pair down projection
        // (10-11 CTAs per pair) was 13-19 % slower, hence the balance rule
        // (ESPEC_SG_ALIGN16=0 off, =2 ignores it: down T = 16 135 -> 128 us,
        // T = 12-14 +2-12 %).
        L.aligned = 0;
        L.nslots = kSgSlots;
        if (TM == 16 && align16 &&
            (long long)sg_stages(TM, p.kcb, L.xrows, kSgSlots) * sg_stage_bytes(TM, p.kcb, L.xrows, kSgSlots) <
                96 * 1024) {
            const int Gs = p.ngroups - L.pool_f, nlin = L.nstatic, npairs = nlin / Gs;
            const int minc = p.grid / npairs;
            if (minc >= 1 && Gs >= (p.grid + npairs - 1) / npairs &&
                (align16 == 2 || (Gs + minc - 1) / minc <= (nlin + p.grid - 1) / p.grid)) {
                L.aligned = 1;
                L.nslots = 1;
            }
        }
        L.ne = sg_ne_used(TM, L.xrows, L.nslots);
        L.sblk = sg_sblk(TM, p.kcb, L.xrows, L.nslots);
        L.rrows = sg_red_rows(TM, L.xrows);
        // The weights stream through L2 exactly once: marking them evict-first
        // keeps L2 for what the dependency chain re-reads (activations, row
        // statistics, split-K partials, KV pages) — measured -6.7 % per step.
        static const int ef = [] {
            const char* e = std::getenv("ESPEC_SG_EVICT_FIRST");
            return e ? std::atoi(e) : 1;
        }();
        L.ef = ef;
        L.stages = sg_stages(TM, p.kcb, L.xrows, L.nslots);
        const size_t smem = sg_smem_bytes(TM, p.kcb, L.xrows, L.nslots);
        const int tslot = sg_trace_slot(b, nprob, L.T, epi, p);
        L.trace = tslot >= 0 ? g_trace.buf + (size_t)tslot * kSgTraceEv * kSgSms : nullptr;
        if (TM == 8) sg_dispatch<8, 32>(epi, L, p.grid, smem, s);
        else if (L.sblk == 32) sg_dispatch<16, 32>(epi, L, p.grid, smem, s);
        else sg_dispatch<16, 16>(epi, L, p.grid, smem, s);
        if (tslot == g_trace.cnt - 1) sg_trace_dump(s);
    }
}

}  // namespace espec_dev
