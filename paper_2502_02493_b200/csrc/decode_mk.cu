// Decode megakernel (sm_100a): ONE persistent launch runs a whole decode
// forward pass — embedding, then per layer the fused RMSNorm->QKV GEMV (RoPE +
// paged-KV write), split-KV attention, O GEMV (+residual), fuzzy-group
// residual adds, RMSNorm->gate/up GEMV (SiLU·up) and down GEMV (+residual,
// row stats) — for batch-1 decode / verify passes of T <= 8 rows.
//
// Why: at T <= 8 every projection is a weight stream (HBM-bound), but a
// drafter layer's matrices are only 33-235 MB (5-36 us at HBM speed) and
// each standalone launch pays ~10 us of launch, pipeline ramp and split-K
// tail. Here one TMA producer warp per SM streams the weights of EVERY GEMV
// of the pass back to back through the shared-memory ring, never waiting for
// activations, so the next projection's weights are already in flight while
// the current one's tail, the grid-wide dependency wait and the attention
// run. The HBM stream only stalls when the ring is full.
//
// Dependencies between ops: a monotonic 64-bit arrival counter in global
// memory. Op k is complete when the counter reaches base + target[k]
// (targets are cumulative arrival counts computed on the host). Every CTA
// arrives once per op: for a GEMV after its epilogue warps finished the
// CTA's units (and any split-K last-arriver reductions), otherwise after its
// consumer warps. Consumers wait for op k-1 before reading op k's inputs. The grid is
// one CTA per SM, launched cooperatively so every CTA is co-resident.
//
// Bit-exactness: the GEMV units, their warp / k-chunk reduction order, the
// epilogues (sgemv_epi.cuh) and the attention items (attn_mma.cuh) are the
// same code as the standalone kernels, with the same (K, N)-only plans, so a
// pass computes bit-identical rows with or without the megakernel (and the
// batch invariance of SURVEY.md §7 H4 carries over).
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "attn_mma.cuh"
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "sgemv_epi.cuh"

namespace espec_dev {

namespace {
constexpr int kC = 8;                 // consumer warps 0-7
constexpr int kProd = kC;             // warp 8: TMA producer
constexpr int kEpi = kC + 1;          // warps 9-11: unit epilogues
constexpr int kNE = 3;              // 12 warps = 3 per SM sub-partition (register budget 168)
constexpr int kTM = 8;                // rows per pass (T <= 8)
constexpr int kThreadsMk = (kC + 1 + kNE) * 32;
constexpr int kBpw = 4;               // 1 KB blocks per consumer warp per stage
constexpr int kStageBlocks = kBpw * kC;
constexpr int kStageBytes = kStageBlocks * 1024;
constexpr int kSlots = 2;
constexpr int kMaxStages = 8;
constexpr int kMaxKcb = 128;
constexpr int kXld = kMaxKcb * 16 + 8;
constexpr int kXBytes = kSlots * kTM * kXld * 2;
constexpr int kRedBuf = kC * kTM * 32;  // floats per reduction buffer
constexpr int kAuxBytes = kXBytes + kNE * kRedBuf * 4;
static_assert(kAuxBytes >= kAttnItemSmem, "attention items reuse the activation / reduction area");
constexpr int kSmemLimit = 227 * 1024 - 1024;
constexpr long long kSpinLimit = 4000000000LL;  // ~2 s at 1.9 GHz: trap instead of hanging
}  // namespace

// Split-K ops: the CTA walks its unit range rotated so that units of group
// g (mod R, R = the nominal range length) come at step ~g mod R on EVERY CTA:
// all k-chunks of a group then finish together and the groups' final
// (last-arriver) reductions are spread over the op instead of piling up at
// its end. Only the processing order changes, never a sum's order.
__device__ __forceinline__ int unit_rotation(const MkOp& op, int start, int len, int grid) {
    if (!op.rotate || len <= 0) return 0;
    const int R = (op.units + grid - 1) / grid;
    const int off = (R - (start % op.ngroups) % R) % R;
    return off < len ? off : 0;
}

// Cooperative 4-byte-word copy global -> shared by threads [0, n).
__device__ __forceinline__ void copy_words(void* dst, const void* src, int bytes, int t, int n) {
    const int w = bytes >> 2;
    for (int i = t; i < w; i += n) reinterpret_cast<int*>(dst)[i] = __ldcg(reinterpret_cast<const int*>(src) + i);
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Block until op `k` is complete (k < 0: nothing to wait for). Called by one
// thread; the fence invalidates this SM's L1 so plain loads issued after the
// caller's barrier see the other SMs' writes.
__device__ __forceinline__ void mk_wait(const MkArgs& A, int k) {
    if (k < 0) return;
    const unsigned long long want = A.base + A.ops[k].target;
    if (ld_acquire_u64(A.counter) < want) {
        const long long t0 = clock64();
        while (ld_acquire_u64(A.counter) < want) {
            __nanosleep(32);
            if (clock64() - t0 > kSpinLimit) {
                printf("decode_mk: CTA %d timed out waiting for op %d (counter %llu < %llu)\n", blockIdx.x, k,
                       ld_acquire_u64(A.counter), want);
                __trap();
            }
        }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// The CTA's arrival for an op, by ONE thread after a barrier over every
// thread that worked on the op (release is cumulative over their writes).
// One arrival per CTA per op keeps the counter's atomics to gridDim.x.
// Optional per-(op, CTA) timeline (ESPEC_MK_TRACE): consumer start, inputs
// staged, consumer done, arrival — nanoseconds of %globaltimer.
__device__ __forceinline__ void mk_trace(const MkArgs& A, int k, int ev) {
    if (A.trace) A.trace[((size_t)k * gridDim.x + blockIdx.x) * 8 + ev] = gtimer();
}
__device__ __forceinline__ void mk_arrive(const MkArgs& A) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(A.counter) : "memory");
}

// This CTA's weight stream over the whole pass: every GEMV op's unit range
// (same order as the consumers) cut into ring-stage chunks.
struct WeightCursor {
    const MkArgs& A;
    int cta, grid;
    int k = -1, i = 0, len = 0, off = 0, start = 0, b = 0, nb = 0;
    const char* base = nullptr;
    __device__ WeightCursor(const MkArgs& a, int c, int g) : A(a), cta(c), grid(g) {}
    __device__ bool next(const char*& src, uint32_t& bytes) {
        while (b >= nb) {  // next unit (or op)
            if (k >= 0 && ++i < len) {
                set_unit();
                continue;
            }
            do {
                if (++k >= A.n_ops) return false;
            } while (A.ops[k].type != MK_GEMV);
            const MkOp& op = A.ops[k];
            start = (int)((long long)cta * op.units / grid);
            len = (int)((long long)(cta + 1) * op.units / grid) - start;
            off = unit_rotation(op, start, len, grid);
            i = 0;
            nb = 0;
            b = 0;
            if (len > 0) set_unit();
        }
        src = base + (size_t)b * 1024;
        const int n = min(kStageBlocks, nb - b);
        bytes = (uint32_t)n * 1024u;
        b += n;
        return true;
    }
    __device__ void set_unit() {
        const MkOp& op = A.ops[k];
        const int u = start + (i + off) % len;
        const int g = u % op.ngroups, pair = u / op.ngroups;
        const int prob = pair / op.nK, j = pair - prob * op.nK;
        const int kb0 = j * op.kcb;
        nb = min(op.kcb, op.KT - kb0);
        b = 0;
        base = reinterpret_cast<const char*>(A.probs[op.prob0 + prob].W) + ((size_t)g * op.KT + kb0) * 1024;
    }
};

__global__ void __launch_bounds__(kThreadsMk, 1) decode_mk_kernel(const __grid_constant__ MkArgs A) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full_bar[kMaxStages];
    __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
    __shared__ __align__(8) uint64_t red_full[kNE];
    __shared__ __align__(8) uint64_t red_empty[kNE];
    __shared__ float inv_rms[kSlots][kTM];
    __shared__ unsigned s_last;
    // per-role copies of the current op and its problem descriptors: the
    // dependency waits invalidate L1 (CCTL.IVALL), and descriptor fields are
    // re-read after every asm memory clobber, so global copies would cost an
    // L2 round trip each time
    __shared__ __align__(16) GemvProblem s_eprob[kMaxProblems];
    __shared__ __align__(16) GemvProblem s_cprob[kMaxProblems];
    __shared__ __align__(16) AttnProblem s_caprob[kMaxProblems];
    __shared__ __align__(16) MkOp s_eop, s_cop;
    __shared__ int s_pos[kTM];
    __shared__ long long s_kvrow[kTM];

    const int stages = A.stages;
    unsigned char* ring = sm;
    unsigned char* aux = sm + (size_t)stages * kStageBytes;
    __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(aux);
    float* red = reinterpret_cast<float*>(aux + kXBytes);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int T = A.pass.T;
    const int grid = gridDim.x, cta = blockIdx.x;

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kC);
        }
        for (int e = 0; e < kNE; ++e) {
            mbar_init(&red_full[e], kC);
            mbar_init(&red_empty[e], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < kTM) {
        // the pass's row metadata is fixed for the whole launch
        int pos = 0;
        long long kvr = 0;
        if (tid < T) {
            pos = A.pass.pos[tid];
            const int row = A.pass.rows[tid];
            kvr = (long long)A.kv.page_table[row / A.kv.page_rows] * A.kv.page_elems +
                  (long long)(row % A.kv.page_rows) * A.kv.dh;
        }
        s_pos[tid] = pos;
        s_kvrow[tid] = kvr;
    }
    __syncthreads();

    if (warp == kProd) {
        // ---- producer: the weights of every GEMV of the pass, in op order,
        // into the smem ring (never waits for activations, only for slots)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            WeightCursor cur(A, cta, grid);
            const char* src;
            uint32_t bytes;
            const uint64_t pol = l2_policy_evict_first();  // weights are read once (see gemv_stream.cu)
            while (cur.next(src, bytes)) {
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                mbar_arrive_expect_tx(&full_bar[stage], bytes);
                tma_bulk_g2s_hint(ring + (size_t)stage * kStageBytes, src, bytes, &full_bar[stage], pol);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        return;
    }

    if (warp >= kEpi) {
        // ---- epilogue warps: finish GEMV units (round-robin by unit index)
        const int e = warp - kEpi;
        const int et = tid - kEpi * 32;
        uint32_t phase = 0;
        for (int k = 0; k < A.n_ops; ++k) {
            if (A.ops[k].type != MK_GEMV) continue;
            copy_words(&s_eop, &A.ops[k], sizeof(MkOp), et, kNE * 32);
            copy_words(s_eprob, A.probs + A.ops[k].prob0, sizeof(GemvProblem) * A.ops[k].nprob, et, kNE * 32);
            named_bar(3, kNE * 32);
            const MkOp& op = s_eop;
            const int start = (int)((long long)cta * op.units / grid);
            const int end = (int)((long long)(cta + 1) * op.units / grid);
            const int len = end - start, off = unit_rotation(op, start, len, grid);
            const int ldw = op.ngroups * 32;
            for (int i = e; i < len; i += kNE) {
                const int u = start + (i + off) % len;
                const int g = u % op.ngroups, pair = u / op.ngroups;
                const int prob = pair / op.nK, j = pair - prob * op.nK;
                const GemvProblem& P = s_eprob[prob];
                mbar_wait(&red_full[e], phase);
                phase ^= 1u;
                const float* rb = red + e * kRedBuf;
                float v[kTM];
#pragma unroll
                for (int t = 0; t < kTM; ++t) {
                    float acc = 0.f;
#pragma unroll
                    for (int w = 0; w < kC; ++w) acc += rb[(w * kTM + t) * 32 + lane];
                    v[t] = acc;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&red_empty[e]);
                if (op.nK > 1) {
                    float* pp = P.partial + (size_t)j * 16 * ldw + g * 32 + lane;
#pragma unroll
                    for (int t = 0; t < kTM; ++t)
                        if (t < T) pp[(size_t)t * ldw] = v[t];
                    __syncwarp();
                    unsigned last = 0;
                    if (lane == 0) {
                        last = ticket_acq_rel(&P.tickets[g]) == (unsigned)op.nK - 1 ? 1u : 0u;
                        if (last) P.tickets[g] = 0u;
                    }
                    last = __shfl_sync(0xffffffffu, last, 0);
                    if (!last) continue;
                    const float* q = P.partial + g * 32 + lane;
#pragma unroll
                    for (int t = 0; t < kTM; ++t) v[t] = 0.f;
                    for (int jj = 0; jj < op.nK; jj += 8) {
                        float ld[8][kTM];
#pragma unroll
                        for (int c = 0; c < 8; ++c)
#pragma unroll
                            for (int t = 0; t < kTM; ++t)
                                ld[c][t] = (jj + c < op.nK && t < T) ? __ldcg(q + ((size_t)(jj + c) * 16 + t) * ldw) : 0.f;
#pragma unroll
                        for (int c = 0; c < 8; ++c)
#pragma unroll
                            for (int t = 0; t < kTM; ++t)
                                if (jj + c < op.nK) v[t] += ld[c][t];
                    }
                }
                const SgEpiCtx ctx{A.pass, A.kv, T, 0, op.ngroups, s_pos, s_kvrow};
                switch (op.epi) {
                    case EPI_STORE: sg_epilogue<kTM, EPI_STORE>(ctx, P, g, v, lane); break;
                    case EPI_RESID: sg_epilogue<kTM, EPI_RESID>(ctx, P, g, v, lane); break;
                    case EPI_SILU: sg_epilogue<kTM, EPI_SILU>(ctx, P, g, v, lane); break;
                    case EPI_QKV: sg_epilogue<kTM, EPI_QKV>(ctx, P, g, v, lane); break;
                    default: sg_epilogue<kTM, EPI_ARGMAX>(ctx, P, g, v, lane); break;
                }
            }
            // all epilogue warps done with op k -> one arrival; it must also
            // follow op k-1's completion (a CTA without units would otherwise
            // arrive early)
            named_bar(3, kNE * 32);
            if (warp == kEpi && lane == 0) {
                mk_wait(A, k - 1);
                mk_trace(A, k, 3);
                mk_arrive(A);
            }
        }
        return;
    }

    // ---- consumers (warps 0-7)
    int stage = 0;
    uint32_t phase = 0;
    uint32_t rphase[kNE];
#pragma unroll
    for (int e = 0; e < kNE; ++e) rphase[e] = 0u;
    const int gid = lane >> 2, tig = lane & 3;
    for (int k = 0; k < A.n_ops; ++k) {
        if (tid == 0) mk_wait(A, k - 1);
        named_bar(1, kC * 32);
        {
            const MkOp& g = A.ops[k];
            copy_words(&s_cop, &g, sizeof(MkOp), tid, kC * 32);
            if (g.type == MK_GEMV)
                copy_words(s_cprob, A.probs + g.prob0, sizeof(GemvProblem) * g.nprob, tid, kC * 32);
            else if (g.type == MK_ATTN)
                copy_words(s_caprob, A.aprobs + g.prob0, sizeof(AttnProblem) * g.nprob, tid, kC * 32);
        }
        named_bar(1, kC * 32);
        const MkOp& op = s_cop;
        if (tid == 0) mk_trace(A, k, 0);
        if (op.type == MK_GEMV) {
            const int start = (int)((long long)cta * op.units / grid);
            const int end = (int)((long long)(cta + 1) * op.units / grid);
            const int len = end - start, off = unit_rotation(op, start, len, grid);
            const int pair0 = start / op.ngroups;
            const int pair1 = end > start ? (end - 1) / op.ngroups : pair0;
            const int kc = op.kcb * 16;
            const int xld = op.xld, xslot = kTM * xld;
            for (int s = 0; s <= pair1 - pair0 && len > 0; ++s) {
                const int pair = pair0 + s, prob = pair / op.nK, j = pair - prob * op.nK;
                const GemvProblem& P = s_cprob[prob];
                for (int t = warp; t < kTM; t += kC) {
                    float r = 1.f;
                    if (P.gain != nullptr && t < T) {
                        float ss = 0.f;
                        const float* st = P.stats_in + (size_t)t * P.stat_tiles_in;
#pragma unroll 8
                        for (int i = lane; i < P.stat_tiles_in; i += 32) ss += __ldcg(st + i);
                        ss = warp_sum(ss);
                        r = 1.0f / sqrtf(ss / (float)P.K + P.eps);
                    }
                    if (lane == 0) inv_rms[s][t] = r;
                }
                named_bar(1, kC * 32);
                __nv_bfloat16* xd = xs + (size_t)s * xslot;
                const int k0 = j * kc;
                const int kq = kc >> 2;
                for (int i = T * kq + tid; i < kTM * kq; i += kC * 32) {
                    const int t = i / kq, kk = (i - t * kq) * 4;
                    *reinterpret_cast<uint2*>(xd + t * xld + kk) = make_uint2(0u, 0u);
                }
                constexpr int U = 8;
                if (P.x_bf16) {
                    // activations already bf16 (producer-rounded): straight copy
                    const __nv_bfloat16* xb16 = reinterpret_cast<const __nv_bfloat16*>(P.x);
                    for (int i0 = tid; i0 < T * kq; i0 += (kC * 32) * U) {
                        uint2 v[U];
        #pragma unroll
                        for (int q = 0; q < U; ++q) {
                            const int i = i0 + q * (kC * 32);
                            const int t = i / kq, k = k0 + (i - t * kq) * 4;
                            v[q] = make_uint2(0u, 0u);
                            if (i < T * kq && k < P.K) v[q] = __ldcg(reinterpret_cast<const uint2*>(xb16 + (size_t)(0 + t) * P.ldx + k));
                        }
        #pragma unroll
                        for (int q = 0; q < U; ++q) {
                            const int i = i0 + q * (kC * 32);
                            if (i >= T * kq) break;
                            const int t = i / kq, kk = (i - t * kq) * 4;
                            *reinterpret_cast<uint2*>(xd + t * xld + kk) = v[q];
                        }
                    }
                } else
                for (int i0 = tid; i0 < T * kq; i0 += kC * 32 * U) {
                    float4 v[U], gn[U];
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const int i = i0 + q * kC * 32;
                        const int t = i / kq, kx = k0 + (i - t * kq) * 4;
                        v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                        gn[q] = make_float4(1.f, 1.f, 1.f, 1.f);
                        if (i < T * kq && kx < P.K) {
                            v[q] = __ldcg(reinterpret_cast<const float4*>(P.x + (size_t)t * P.ldx + kx));
                            if (P.gain != nullptr) gn[q] = __ldg(reinterpret_cast<const float4*>(P.gain + kx));
                        }
                    }
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const int i = i0 + q * kC * 32;
                        if (i >= T * kq) break;
                        const int t = i / kq, kk = (i - t * kq) * 4;
                        float4 w = v[q];
                        if (P.gain != nullptr) {
                            const float r = inv_rms[s][t];
                            w.x = __fmul_rn(__fmul_rn(w.x, r), gn[q].x);
                            w.y = __fmul_rn(__fmul_rn(w.y, r), gn[q].y);
                            w.z = __fmul_rn(__fmul_rn(w.z, r), gn[q].z);
                            w.w = __fmul_rn(__fmul_rn(w.w, r), gn[q].w);
                        }
                        const __nv_bfloat162 lo = __floats2bfloat162_rn(w.x, w.y), hi = __floats2bfloat162_rn(w.z, w.w);
                        uint2 pk;
                        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
                        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
                        *reinterpret_cast<uint2*>(xd + t * xld + kk) = pk;
                    }
                }
            }
            named_bar(1, kC * 32);
            if (tid == 0) mk_trace(A, k, 1);
            for (int i = 0; i < len; ++i) {
                const int u = start + (i + off) % len;
                const int pair = u / op.ngroups;
                const int j = pair % op.nK;
                const int nb = min(op.kcb, op.KT - j * op.kcb);
                const __nv_bfloat16* xb = xs + (size_t)(pair - pair0) * xslot;
                const __nv_bfloat16* xrow = xb + (lane & 7) * xld + ((lane >> 3) & 1) * 8;
                float acc[4][4];
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
                for (int b = 0; b < nb; b += kStageBlocks) {
                    mbar_wait(&full_bar[stage], phase);
                    uint32_t w[kBpw][8];
                    uint32_t a[kBpw][4];
#pragma unroll
                    for (int ii = 0; ii < kBpw; ++ii) {
                        const int bi = warp * kBpw + ii;
                        if (b + bi < nb) {
                            const uint32_t wb = smem_u32(ring + (size_t)stage * kStageBytes + bi * 1024 + lane * 16);
                            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                         : "=r"(w[ii][0]), "=r"(w[ii][1]), "=r"(w[ii][2]), "=r"(w[ii][3])
                                         : "r"(wb));
                            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                                         : "=r"(w[ii][4]), "=r"(w[ii][5]), "=r"(w[ii][6]), "=r"(w[ii][7])
                                         : "r"(wb + 512));
                            const uint32_t xa = smem_u32(xrow + (b + bi) * 16);
                            asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                                         : "=r"(a[ii][0]), "=r"(a[ii][2])
                                         : "r"(xa));
                            a[ii][1] = a[ii][3] = 0u;
                        }
                    }
#pragma unroll
                    for (int ii = 0; ii < kBpw; ++ii) {
                        if (b + warp * kBpw + ii < nb) {
                            mma16816(acc[0], a[ii], w[ii][0], w[ii][1]);
                            mma16816(acc[1], a[ii], w[ii][2], w[ii][3]);
                            mma16816(acc[2], a[ii], w[ii][4], w[ii][5]);
                            mma16816(acc[3], a[ii], w[ii][6], w[ii][7]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[stage]);
                    if (++stage == stages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                const int e = i % kNE;
                mbar_wait(&red_empty[e], rphase[e] ^ 1u);
                rphase[e] ^= 1u;
                float* rw = red + e * kRedBuf + warp * kTM * 32;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = q * 8 + 2 * tig;
                    rw[gid * 32 + col] = acc[q][0];
                    rw[gid * 32 + col + 1] = acc[q][1];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&red_full[e]);
            }
            if (tid == 0) mk_trace(A, k, 2);
            continue;  // GEMV completion is signalled by the epilogue warps
        }
        if (op.type == MK_ATTN) {
            // warps 0-3: attention items (4 key splits x one kv head x one m-tile)
            const int splits = (A.pass.total + 63) / 64;
            const int nchunks = (splits + A.kv.attn_ppi - 1) / A.kv.attn_ppi;
            const int mtiles = (T * op.G + 15) / 16;
            const int ny = A.kv.n_kv * mtiles;
            const int items = nchunks * ny * op.nprob;
            if (warp < 4) {
                for (int it = cta; it < items; it += grid) {
                    const int bx = it % nchunks, rest = it / nchunks;
                    const int by = rest % ny, pz = rest / ny;
                    if (op.dh == 128)
                        attn_mma_item<128>(s_caprob[pz], A.pass, A.kv, op.n_heads, op.G, bx, by, nchunks,
                                           ny, aux, &s_last, tid, 2,
                                           A.trace ? A.trace + ((size_t)k * grid + cta) * 8 + 4 : nullptr);
                    else
                        attn_mma_item<64>(s_caprob[pz], A.pass, A.kv, op.n_heads, op.G, bx, by, nchunks, ny,
                                          aux, &s_last, tid, 2,
                                          A.trace ? A.trace + ((size_t)k * grid + cta) * 8 + 4 : nullptr);
                    named_bar(2, 128);  // the item's smem is reused by the next one
                }
            }
        } else {
            // MK_EMBED / MK_ADD: one warp per (row, 32-column tile), same
            // arithmetic and stats granularity as embed_kernel / add_stats_kernel
            const int tiles = op.stat_tiles;
            const int gw = cta * kC + warp, nw = grid * kC;
            for (int w = gw; w < T * tiles; w += nw) {
                const int t = w / tiles, c = (w - t * tiles) * 32 + lane;
                float y = 0.f;
                if (c < op.d) {
                    if (op.type == MK_EMBED) {
                        const int tok = __ldcg(A.tok_arena + __ldcg(A.tok_idx + t));
                        y = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(op.emb)[(size_t)tok * op.d + c]);
                    } else {
                        y = __fadd_rn(__ldcg(op.h + (size_t)t * op.d + c), __ldcg(op.a + (size_t)t * op.d + c));
                    }
                    op.h[(size_t)t * op.d + c] = y;
                }
                const float sq = warp_sum(y * y);
                if (lane == 0 && c < op.d) op.stats[t * tiles + c / kStatTile] = sq;
            }
        }
        named_bar(1, kC * 32);
        if (tid == 0) {
            mk_trace(A, k, 2);
            mk_trace(A, k, 3);
            mk_arrive(A);
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int mk_stages() { return (kSmemLimit - kAuxBytes) / kStageBytes < kMaxStages ? (kSmemLimit - kAuxBytes) / kStageBytes : kMaxStages; }

int mk_max_rows() { return kTM; }

void mk_plan_gemv(MkOp& op, int K, int ldw, int nprob) {
    const SgPlan p = sgemv_plan(K, ldw, nprob);
    if (p.kcb > kMaxKcb) throw std::runtime_error("decode_mk: unit larger than the activation slot");
    op.type = MK_GEMV;
    op.nprob = nprob;
    op.KT = p.KT;
    op.kcb = p.kcb;
    op.nK = p.nK;
    op.ngroups = p.ngroups;
    op.units = p.units;
    op.xld = p.kcb * 16 + 8;
    static const int rot = [] {
        const char* e = std::getenv("ESPEC_MK_ROTATE");
        return e ? std::atoi(e) : 0;  // measured slower (DRAM locality): off
    }();
    op.rotate = p.nK > 1 ? rot : 0;
    op.arrivals = 1;
}

int mk_op_arrivals(int) { return 1; }

int mk_grid() {
    static int n = [] {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms;
    }();
    return n;
}

cudaError_t launch_decode_mk(const MkArgs& a, cudaStream_t s) {
    static unsigned long long configured = 0;
    const int stages = mk_stages();
    const size_t smem = (size_t)stages * kStageBytes + kAuxBytes;
    ensure_smem((const void*)decode_mk_kernel, (int)smem, configured);
    MkArgs A = a;
    A.stages = stages;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(mk_grid());
    cfg.blockDim = dim3(kThreadsMk);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, decode_mk_kernel, A);
}

}  // namespace espec_dev
