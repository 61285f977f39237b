// Shared attention pieces: paged-KV addressing, tree-aware visibility and the
// tensor-core split-KV attention item (mma.sync m16n8k16 over bf16 KV pages),
// used by the standalone attention kernel (kernels.cu) and the decode
// megakernel (decode_mk.cu) so both produce bit-identical outputs.
// Attention semantics: proj/src/model.cpp:140-192; mask proj/src/kv_cache.cpp:43-60.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace espec_dev {

__device__ __forceinline__ long long kv_off(const KvView& kv, int layer, int kind, int head, int row) {
    const int page = kv.page_table[row / kv.page_rows];
    const int r = row % kv.page_rows;
    return (long long)page * kv.page_elems +
           ((((long long)layer * 2 + kind) * kv.n_kv + head) * kv.page_rows + r) * kv.dh;
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}

// visible() with the row's vis_end / ancestor mask already in registers
__device__ __forceinline__ bool visible_rows(const PassView& P, int vis_end, unsigned long long anc, int j) {
    if (j >= P.total) return false;
    if (j < vis_end) return true;
    const int o = j - P.tree_base;
    return o >= 0 && o < 64 && ((anc >> o) & 1ull);
}
__device__ __forceinline__ bool visible(const PassView& P, int t, int j) {
    if (j >= P.total) return false;
    if (j < P.vis_end[t]) return true;
    const int o = j - P.tree_base;
    return o >= 0 && o < 64 && ((P.anc[t] >> o) & 1ull);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}

// Element offset of (key row, head dim col) inside one staged K or V page:
// SWZ = false: the page as one contiguous [64][DH] run (1-D bulk copy);
// SWZ = true: DH/64 blocks of [64 rows][64 dims] in the TMA 128-byte swizzle
// (16-byte chunk c of row r at c ^ (r & 7)), so the 8 rows an ldmatrix reads
// at one column fall in 8 different bank groups.
template <int DH, bool SWZ>
__device__ __forceinline__ int attn_page_off(int row, int col) {
    if (!SWZ) return row * DH + col;
    return (col >> 6) * 64 * 64 + row * 64 + ((((col & 63) >> 3) ^ (row & 7)) << 3) + (col & 7);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// 16 output values (one pair row, 16 consecutive dims) = acc / den: fp32, or
// bf16 rounded to nearest (exactly what the O GEMV's staging would do) when
// the consumer takes bf16 activations
template <int DH>
__device__ __forceinline__ void attn_store_row(const AttnProblem& A, size_t off, const float4 (&acc)[4], float den) {
    float y[16];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        y[4 * v] = den > 0.f ? acc[v].x / den : 0.f;
        y[4 * v + 1] = den > 0.f ? acc[v].y / den : 0.f;
        y[4 * v + 2] = den > 0.f ? acc[v].z / den : 0.f;
        y[4 * v + 3] = den > 0.f ? acc[v].w / den : 0.f;
    }
    if (A.out_bf16) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const __nv_bfloat162 b = __floats2bfloat162_rn(y[2 * j], y[2 * j + 1]);
            pk[j] = *reinterpret_cast<const uint32_t*>(&b);
        }
        uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(A.out) + off);
        o[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        o[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    } else {
        float* o = A.out + off;
#pragma unroll
        for (int v = 0; v < 4; ++v)
            *reinterpret_cast<float4*>(o + 4 * v) = make_float4(y[4 * v], y[4 * v + 1], y[4 * v + 2], y[4 * v + 3]);
    }
}

// ---------------------------------------------------------------------------
// Per-warp pieces of the tensor-core split-KV attention. A warp owns 16 query
// pairs (one m-tile: GQA pairs p = t * G + g as M rows) and keys
// [16 kq, 16 kq + 16) of every 64-row page; it keeps an online softmax across
// the pages of its chunk. Four key-quarter warps combine in fixed order, then
// chunks along the context combine in fixed chunk order. Every row's
// arithmetic depends only on the context and the chunking (kv.attn_ppi, a
// function of the cache capacity), never on the pass or the CTA layout, so the
// per-CTA item (decode megakernel) and the whole-head kernel (attn_mma_kernel)
// produce bit-identical rows (batch invariance).
// ---------------------------------------------------------------------------

template <int DH>
struct AttnWarp {
    uint32_t qa[DH / 16][4];  // Q A-fragments (pairs 16 mt + gid / + 8), bf16
    float o[DH / 8][4];       // running P V
    float m_r[2], l_r[2];     // running max / denominator of the two rows
    int vmin;                 // min causal prefix end over the warp's valid rows
    int ve[2];                // visibility: causal prefix end ...
    unsigned long long an[2]; // ... and tree ancestor mask of the two rows
    int pr[2];                // pair index of the two rows
};

// Q fragments and visibility of m-tile mt for this lane (after the dependency wait).
template <int DH>
__device__ __forceinline__ void attn_warp_init(AttnWarp<DH>& W, const AttnProblem& A, const PassView& pass, int H,
                                               int G, int hk, int mt, int lane) {
    const int gid = lane >> 2, tig = lane & 3, P = pass.T * G;
    W.pr[0] = mt * 16 + gid;
    W.pr[1] = mt * 16 + gid + 8;
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
        W.ve[ri] = 0;
        W.an[ri] = 0ull;
        const int p = W.pr[ri];
        if (p < P) {
            W.ve[ri] = pass.vis_end[p / G];
            W.an[ri] = pass.anc[p / G];
        }
    }
    {
        int v = 0x7fffffff;
        if (W.pr[0] < P) v = min(v, W.ve[0]);
        if (W.pr[1] < P) v = min(v, W.ve[1]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
        W.vmin = min(v, pass.total);
    }
    const int p0 = W.pr[0], p1 = W.pr[1];
    const float* q0 = nullptr;
    const float* q1 = nullptr;
    if (p0 < P) q0 = A.q + (size_t)(p0 / G) * H * DH + (hk * G + p0 % G) * DH;
    if (p1 < P) q1 = A.q + (size_t)(p1 / G) * H * DH + (hk * G + p1 % G) * DH;
#pragma unroll
    for (int s = 0; s < DH / 16; ++s) {
        const int c = s * 16 + 2 * tig;
        float2 a = q0 ? *reinterpret_cast<const float2*>(q0 + c) : make_float2(0.f, 0.f);
        float2 b = q1 ? *reinterpret_cast<const float2*>(q1 + c) : make_float2(0.f, 0.f);
        float2 cc = q0 ? *reinterpret_cast<const float2*>(q0 + c + 8) : make_float2(0.f, 0.f);
        float2 d = q1 ? *reinterpret_cast<const float2*>(q1 + c + 8) : make_float2(0.f, 0.f);
        W.qa[s][0] = pack_bf16x2(a.x, a.y);
        W.qa[s][1] = pack_bf16x2(b.x, b.y);
        W.qa[s][2] = pack_bf16x2(cc.x, cc.y);
        W.qa[s][3] = pack_bf16x2(d.x, d.y);
    }
    W.m_r[0] = W.m_r[1] = -INFINITY;
    W.l_r[0] = W.l_r[1] = 0.f;
#pragma unroll
    for (int d = 0; d < DH / 8; ++d) W.o[d][0] = W.o[d][1] = W.o[d][2] = W.o[d][3] = 0.f;
}

// One step over up to two pages (np = 1 or 2): QK^T of this warp's 16 keys
// of each page (j0[i] = first key row), scale + mask, one online-softmax
// update over the step's keys, O += P V. Pairing two pages per step gives four
// independent HMMA chains and halves the serial softmax / rescale work per key.
// A page whose keys are all beyond the context is skipped: it would only add
// exact zeros, so a row's result does not depend on whether its step held one
// or two pages (batch invariance across context lengths).
template <int DH, bool SWZ = false>
__device__ __forceinline__ void attn_warp_step(AttnWarp<DH>& W, const __nv_bfloat16* const (&Ks)[2],
                                               const __nv_bfloat16* const (&Vs)[2], uint64_t* const (&mbk)[2],
                                               uint64_t* const (&mbv)[2], const uint32_t (&ph)[2], int np,
                                               const PassView& pass, int P, const int (&j0)[2], int kq, int lane) {
    constexpr int NT = DH / 8;
    const int tig = lane & 3;
    int nr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) nr[i] = i < np ? max(0, min(16, pass.total - j0[i])) : 0;
    if (nr[0] <= 0) return;  // pages are in key order: nothing visible in this step
    const bool two = nr[1] > 0;
    const float inv_sqrt = 1.0f / sqrtf((float)DH);
    float sc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
    mbar_wait(mbk[0], ph[0]);
    if (two) mbar_wait(mbk[1], ph[1]);
#pragma unroll
    for (int s = 0; s < DH / 16; s += 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= 2 && !two) continue;
            uint32_t b[4];
            ldsm_x4(b, Ks[j >> 1] + attn_page_off<DH, SWZ>(kq * 16 + (j & 1) * 8 + (lane & 7), s * 16 + (lane >> 3) * 8));
            mma_bf16_16816(sc[j], W.qa[s], b[0], b[1]);
            mma_bf16_16816(sc[j], W.qa[s + 1], b[2], b[3]);
        }
    }
    // scale + mask; one online-softmax update over the step's keys. Keys
    // below every row's causal prefix (W.vmin, the committed context) need no
    // per-element test: one warp-uniform branch for the whole step.
    float mx[2] = {-INFINITY, -INFINITY};
    const int jend = two ? j0[1] + 16 : j0[0] + 16;
    if (jend <= W.vmin && (!two || j0[1] == j0[0] + 64)) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j >= 2 && !two) {
#pragma unroll
                for (int e = 0; e < 4; ++e) sc[j][e] = -INFINITY;
                continue;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ri = e >> 1;
                sc[j][e] = W.pr[ri] < P ? __fmul_rn(sc[j][e], inv_sqrt) : -INFINITY;
                mx[ri] = fmaxf(mx[ri], sc[j][e]);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int pi = j >> 1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ri = e >> 1;
                const int key = (j & 1) * 8 + 2 * tig + (e & 1);
                const bool ok = (pi == 0 || two) && W.pr[ri] < P && key < nr[pi] &&
                                visible_rows(pass, W.ve[ri], W.an[ri], j0[pi] + key);
                sc[j][e] = ok ? __fmul_rn(sc[j][e], inv_sqrt) : -INFINITY;
                mx[ri] = fmaxf(mx[ri], sc[j][e]);
            }
        }
    }
    float alpha[2];
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
        mx[ri] = fmaxf(mx[ri], __shfl_xor_sync(0xffffffffu, mx[ri], 1));
        mx[ri] = fmaxf(mx[ri], __shfl_xor_sync(0xffffffffu, mx[ri], 2));
        const float mn = fmaxf(W.m_r[ri], mx[ri]);
        // rescale of the running sums (exactly 1 while the max holds, 0 while
        // nothing was visible yet)
        alpha[ri] = W.m_r[ri] == -INFINITY ? 0.f : (mn == W.m_r[ri] ? 1.f : expf(W.m_r[ri] - mn));
        W.m_r[ri] = mn;
    }
    float sum[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int ri = e >> 1;
            const float v = sc[j][e] == -INFINITY ? 0.f : expf(sc[j][e] - W.m_r[ri]);
            sc[j][e] = v;
            sum[ri] += v;
        }
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
        sum[ri] += __shfl_xor_sync(0xffffffffu, sum[ri], 1);
        sum[ri] += __shfl_xor_sync(0xffffffffu, sum[ri], 2);
        W.l_r[ri] = __fmaf_rn(W.l_r[ri], alpha[ri], sum[ri]);
    }
    // x 1 is exact: skip the rescale while every row's max holds (warp-uniform)
    if (!__all_sync(0xffffffffu, alpha[0] == 1.f && alpha[1] == 1.f)) {
#pragma unroll
        for (int d = 0; d < NT; ++d) {
            W.o[d][0] *= alpha[0];
            W.o[d][1] *= alpha[0];
            W.o[d][2] *= alpha[1];
            W.o[d][3] *= alpha[1];
        }
    }
    // O += P V, one k-step of 16 keys per page
    mbar_wait(mbv[0], ph[0]);
    if (two) mbar_wait(mbv[1], ph[1]);
#pragma unroll
    for (int pi = 0; pi < 2; ++pi) {
        if (pi == 1 && !two) break;
        uint32_t pa[4];
        pa[0] = pack_bf16x2(sc[2 * pi][0], sc[2 * pi][1]);
        pa[1] = pack_bf16x2(sc[2 * pi][2], sc[2 * pi][3]);
        pa[2] = pack_bf16x2(sc[2 * pi + 1][0], sc[2 * pi + 1][1]);
        pa[3] = pack_bf16x2(sc[2 * pi + 1][2], sc[2 * pi + 1][3]);
#pragma unroll
        for (int d = 0; d < NT; d += 2) {
            uint32_t b[4];
            // matrices: (keys 0..7, dims 8d), (keys 8..15, dims 8d), (keys 0..7, dims 8d+8), (keys 8..15, dims 8d+8)
            const int mi = lane >> 3;
            ldsm_x4_t(b, Vs[pi] + attn_page_off<DH, SWZ>(kq * 16 + (mi & 1) * 8 + (lane & 7), d * 8 + (mi >> 1) * 8));
            mma_bf16_16816(W.o[d], pa, b[0], b[1]);
            mma_bf16_16816(W.o[d + 1], pa, b[2], b[3]);
        }
    }
}

// Scratch of one m-tile's 4-warp combine: [4][16][DH] partial O, then
// (m, l, warp weight) per (warp, row), then row max / denominator.
template <int DH>
constexpr int attn_tile_scratch_floats() {
    return 4 * 16 * DH + 3 * 64 + 32;
}

// Fixed-order 4-warp combine of one m-tile (128 threads t = 32 kq + lane,
// named barrier bar_id), then either the final output (one chunk) or the
// chunk's partial rows [16][DH + 4] (values, max, denominator) at wsb.
template <int DH>
__device__ __forceinline__ void attn_tile_finish(const AttnWarp<DH>& W, float* Os, int t, int bar_id,
                                                 const AttnProblem& A, int H, int G, int hk, int mt, int P,
                                                 int nchunks, float* wsb) {
    constexpr int NT = DH / 8;
    const int kq = t >> 5, lane = t & 31, gid = lane >> 2, tig = lane & 3;
    float* Ms = Os + 4 * 16 * DH;  // [4][16]
    float* Ls = Ms + 64;           // [4][16]
    float* Fw = Ls + 64;           // [4][16] warp weights exp(m_w - M)
    float* Rm = Fw + 64;           // [16] row max
    float* Rd = Rm + 16;           // [16] row denominator
#pragma unroll
    for (int d = 0; d < NT; ++d) {
        const int c = d * 8 + 2 * tig;
        *reinterpret_cast<float2*>(&Os[(kq * 16 + gid) * DH + c]) = make_float2(W.o[d][0], W.o[d][1]);
        *reinterpret_cast<float2*>(&Os[(kq * 16 + gid + 8) * DH + c]) = make_float2(W.o[d][2], W.o[d][3]);
    }
    if (tig == 0) {
        Ms[kq * 16 + gid] = W.m_r[0];
        Ms[kq * 16 + gid + 8] = W.m_r[1];
        Ls[kq * 16 + gid] = W.l_r[0];
        Ls[kq * 16 + gid + 8] = W.l_r[1];
    }
    named_bar(bar_id, 128);
    if (t < 16) {  // per-row weights, fixed warp order
        const int r = t;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, Ms[w * 16 + r]);
        float den = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float m = Ms[w * 16 + r];
            float f = 0.f;
            if (M != -INFINITY && m != -INFINITY) {
                f = expf(m - M);
                den = __fmaf_rn(f, Ls[w * 16 + r], den);
            }
            Fw[w * 16 + r] = f;
        }
        Rm[r] = M;
        Rd[r] = den;
    }
    named_bar(bar_id, 128);
    constexpr int PS = DH + 4;     // workspace row: DH values, M, den (float4-aligned)
    constexpr int CPR = DH / 16;   // threads per row
    for (int it = t; it < 16 * CPR; it += 128) {
        const int r = it / CPR, c0 = (it % CPR) * 16;
        float4 acc[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float f = Fw[w * 16 + r];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float4 x = *reinterpret_cast<const float4*>(&Os[(w * 16 + r) * DH + c0 + 4 * v]);
                acc[v].x = __fmaf_rn(f, x.x, acc[v].x);
                acc[v].y = __fmaf_rn(f, x.y, acc[v].y);
                acc[v].z = __fmaf_rn(f, x.z, acc[v].z);
                acc[v].w = __fmaf_rn(f, x.w, acc[v].w);
            }
        }
        const int p = mt * 16 + r;
        if (nchunks == 1) {
            if (p < P) attn_store_row<DH>(A, (size_t)(p / G) * H * DH + (hk * G + p % G) * DH + c0, acc, Rd[r]);
        } else {
#pragma unroll
            for (int v = 0; v < 4; ++v) *reinterpret_cast<float4*>(wsb + r * PS + c0 + 4 * v) = acc[v];
            if (c0 == 0) {
                wsb[r * PS + DH] = Rm[r];
                wsb[r * PS + DH + 1] = Rd[r];
            }
        }
    }
}

// Scratch of one m-tile's cross-chunk combine (fac, sden, (m, l) pairs).
constexpr int attn_combine_scratch_floats(int nchunks) { return nchunks * 16 + 16 + 2 * nchunks * 16; }

// Cross-chunk combine of one m-tile (run by the last CTA of its kv head):
// chunk partials at base + ch * cstride, fixed chunk order.
template <int DH>
__device__ __forceinline__ void attn_tile_combine(float* scr, int t, int bar_id, const AttnProblem& A, int H, int G,
                                                  int hk, int mt, int P, int nchunks, const float* base,
                                                  size_t cstride) {
    constexpr int PS = DH + 4;
    float* fac = scr;                   // [nchunks][16]
    float* sden = scr + nchunks * 16;   // [16]
    float2* ml = reinterpret_cast<float2*>(sden + 16);  // [nchunks][16] (m, l)
    // (m, l) of every chunk: one float2 load each, all issued together
    for (int i = t; i < nchunks * 16; i += 128) {
        const int ch = i >> 4, r = i & 15;
        ml[i] = __ldcg(reinterpret_cast<const float2*>(base + ch * cstride + r * PS + DH));
    }
    named_bar(bar_id, 128);
    if (t < 16) {
        const int r = t;
        float M = -INFINITY;
        for (int ch = 0; ch < nchunks; ++ch) M = fmaxf(M, ml[ch * 16 + r].x);
        float den = 0.f;
        for (int ch = 0; ch < nchunks; ++ch) {
            const float m = ml[ch * 16 + r].x;
            float f = 0.f;
            if (M != -INFINITY && m != -INFINITY) {
                f = expf(m - M);
                den = __fmaf_rn(f, ml[ch * 16 + r].y, den);
            }
            fac[ch * 16 + r] = f;
        }
        sden[r] = den;
    }
    named_bar(bar_id, 128);
    constexpr int CPR = DH / 16;
    for (int it = t; it < 16 * CPR; it += 128) {
        const int r = it / CPR, c0 = (it % CPR) * 16;
        const int p = mt * 16 + r;
        if (p >= P) continue;
        float4 acc[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        // CB chunks' loads in flight per round trip (the sum order is the
        // chunk order whatever CB is)
        constexpr int CB = 8;
        for (int ch0 = 0; ch0 < nchunks; ch0 += CB) {
            float4 x[CB][4];
#pragma unroll
            for (int q = 0; q < CB; ++q)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    x[q][v] = ch0 + q < nchunks
                                  ? __ldcg(reinterpret_cast<const float4*>(base + (ch0 + q) * cstride + r * PS + c0 + 4 * v))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                if (ch0 + q >= nchunks) break;
                const float f = fac[(ch0 + q) * 16 + r];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    acc[v].x = __fmaf_rn(f, x[q][v].x, acc[v].x);
                    acc[v].y = __fmaf_rn(f, x[q][v].y, acc[v].y);
                    acc[v].z = __fmaf_rn(f, x[q][v].z, acc[v].z);
                    acc[v].w = __fmaf_rn(f, x[q][v].w, acc[v].w);
                }
            }
        }
        attn_store_row<DH>(A, (size_t)(p / G) * H * DH + (hk * G + p % G) * DH + c0, acc, sden[r]);
    }
}

// Issue the K and V page copies of page pg into stage buffers (one 1-D TMA
// bulk copy each: a 64-row page of one kv head is one contiguous run).
template <int DH>
__device__ __forceinline__ void attn_issue_page(const KvView& kv, int layer, int hk, int pg, __nv_bfloat16* kdst,
                                                __nv_bfloat16* vdst, uint64_t* mbk, uint64_t* mbv) {
    const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(kv.pool);
    uint64_t pol = 0;
    if (kv.l2_hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (kv.l2_hint == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    __nv_bfloat16* dst[2] = {kdst, vdst};
    uint64_t* mb[2] = {mbk, mbv};
    for (int kind = 0; kind < 2; ++kind) {
        const void* src = pool + kv_off(kv, layer, kind, hk, pg * 64);
        mbar_arrive_expect_tx(mb[kind], 64 * DH * 2);
        if (kv.l2_hint) tma_bulk_g2s_hint(dst[kind], src, 64 * DH * 2, mb[kind], pol);
        else tma_bulk_g2s(dst[kind], src, 64 * DH * 2, mb[kind]);
    }
}

// The same page (physical page index) through a 4-D tensor map of the pool ({dh, row, (layer, k|v,
// kv head), page}, box {64, 64, 1, 1}, 128-byte swizzle): DH / 64 boxes per K
// or V page into attn_page_off<DH, true> order. dst must be 1024-byte aligned.
template <int DH>
__device__ __forceinline__ void attn_issue_page_tmap(const KvView& kv, const void* tmap, int layer, int hk, int page,
                                                     __nv_bfloat16* kdst, __nv_bfloat16* vdst, uint64_t* mbk,
                                                     uint64_t* mbv) {
    uint64_t pol = 0;
    if (kv.l2_hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (kv.l2_hint == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if (kv.l2_hint == 0) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    __nv_bfloat16* dst[2] = {kdst, vdst};
    uint64_t* mb[2] = {mbk, mbv};
    for (int kind = 0; kind < 2; ++kind) {
        const int lkh = (layer * 2 + kind) * kv.n_kv + hk;
        mbar_arrive_expect_tx(mb[kind], 64 * DH * 2);
#pragma unroll
        for (int h = 0; h < DH / 64; ++h)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
                "[%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst[kind] + h * 64 * 64)),
                "l"(reinterpret_cast<uint64_t>(tmap)), "r"(h * 64), "r"(0), "r"(lkh), "r"(page),
                "r"(smem_u32(mb[kind])), "l"(pol)
                : "memory");
    }
}

// Item shared memory: two stages of K and V pages (4 x 64 x DH bf16), then
// the 4-warp combine and the cross-item combine reuse it; the four
// mbarriers sit above.
constexpr int kAttnMaxChunks = 256;  // 64-row page chunks per (kv head, m-tile): contexts up to 16K rows
constexpr int kAttnBarOffset = 72 * 1024;
constexpr int kAttnItemSmem = kAttnBarOffset + 64;
static_assert(4 * 64 * 128 * 2 <= kAttnBarOffset, "double-buffered K/V pages must fit below the barriers");
static_assert(attn_tile_scratch_floats<128>() * 4 <= kAttnBarOffset, "4-warp combine scratch");
static_assert(attn_combine_scratch_floats(kAttnMaxChunks) * 4 <= kAttnBarOffset, "cross-chunk combine scratch");
// One item of the split-KV attention on 4 warps (threads tid 0..127, named
// barrier bar_id): kv.attn_ppi 64-row key pages (chunk bx) of one kv head
// and one 16-pair m-tile (by = m-tile * n_kv + kv head), double-buffered.
// Used by the decode megakernel (items spread over its SMs).
template <int DH>
__device__ __forceinline__ void attn_mma_item(const AttnProblem& A, const PassView& pass, const KvView& kv,
                                              int n_heads, int G_, int bx, int by, int nchunks_, int ny,
                                              unsigned char* smraw, unsigned* s_last_p, int tid, int bar_id,
                                              unsigned long long* dbg = nullptr) {
    unsigned& s_last = *s_last_p;
    const int G = G_, H = n_heads, T = pass.T, P = T * G;
    const int n_kv = kv.n_kv;
    const int hk = by % n_kv, mt = by / n_kv;
    const int warp = tid >> 5, lane = tid & 31;
    const int ppi = kv.attn_ppi;
    const int splits = (pass.total + 63) / 64;
    const int pg0 = bx * ppi, pg1 = min(splits, pg0 + ppi);
    // stage st: K at st*2*64*DH, V at (st*2+1)*64*DH (bf16 elements)
    __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(smraw);
    uint64_t* mb = reinterpret_cast<uint64_t*>(smraw + kAttnBarOffset);  // [stage][K|V]
    // the buffers were last written through the generic proxy (megakernel:
    // activation slots / earlier items); order that before the TMA writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    auto issue = [&](int pg) {  // tid 0 only
        const int st = (pg - pg0) & 1;
        attn_issue_page<DH>(kv, A.layer, hk, pg, buf + (size_t)(st * 2) * 64 * DH, buf + (size_t)(st * 2 + 1) * 64 * DH,
                            &mb[st * 2], &mb[st * 2 + 1]);
    };
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&mb[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int pg = pg0; pg < pg1 && pg < pg0 + 2; ++pg) issue(pg);
    }
    AttnWarp<DH> W;
    attn_warp_init<DH>(W, A, pass, H, G, hk, mt, lane);
    named_bar(bar_id, 128);  // barriers initialised before anyone waits on them
    // steps of two pages (stages 0 and 1), refilled together
    for (int pg = pg0; pg < pg1; pg += 2) {
        const uint32_t ph = (uint32_t)((pg - pg0) >> 1) & 1u;
        if (dbg && pg == pg0 && lane == 0 && pass.total > pg * 64 + warp * 16) {
            mbar_wait(&mb[0], ph);
            atomicMax(dbg + 2, gtimer());
        }
        const __nv_bfloat16* const Ks[2] = {buf, buf + (size_t)2 * 64 * DH};
        const __nv_bfloat16* const Vs[2] = {buf + (size_t)64 * DH, buf + (size_t)3 * 64 * DH};
        uint64_t* const mk[2] = {&mb[0], &mb[2]};
        uint64_t* const mv[2] = {&mb[1], &mb[3]};
        const uint32_t phs[2] = {ph, ph};
        const int j0[2] = {pg * 64 + warp * 16, (pg + 1) * 64 + warp * 16};
        attn_warp_step<DH>(W, Ks, Vs, mk, mv, phs, min(2, pg1 - pg), pass, P, j0, warp, lane);
        named_bar(bar_id, 128);  // both stages consumed by every warp
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int q = pg + 2; q < pg1 && q < pg + 4; ++q) issue(q);
        }
    }
    if (dbg && lane == 0) atomicMax(dbg + 3, gtimer());
    if (tid == 0) {  // the barriers' memory is plain data from here on
        for (int i = 0; i < 4; ++i)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&mb[i])) : "memory");
    }
    const int nchunks = nchunks_;
    constexpr int PS = DH + 4;
    float* wsb = A.ws + (((size_t)bx * ny + by) * 16) * PS;
    attn_tile_finish<DH>(W, reinterpret_cast<float*>(smraw), tid, bar_id, A, H, G, hk, mt, P, nchunks, wsb);
    if (nchunks == 1) return;
    // Cross-CTA combine (last CTA of this (kv head, m-tile)), fixed chunk order.
    named_bar(bar_id, 128);
    if (dbg && tid == 0) atomicMax(dbg + 4, gtimer());
    unsigned* ticket = A.tickets + by;
    if (tid == 0) {
        unsigned tk;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(tk) : "l"(ticket) : "memory");
        s_last = (tk == (unsigned)nchunks - 1) ? 1u : 0u;
        if (s_last) *ticket = 0u;
    }
    named_bar(bar_id, 128);
    if (!s_last) return;
    attn_tile_combine<DH>(reinterpret_cast<float*>(smraw), tid, bar_id, A, H, G, hk, mt, P, nchunks,
                          A.ws + ((size_t)by * 16) * PS, (size_t)ny * 16 * PS);
    if (dbg && tid == 0) atomicMax(dbg + 5, gtimer());
}

}  // namespace espec_dev
