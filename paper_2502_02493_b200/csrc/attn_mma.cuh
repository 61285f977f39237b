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

// Item shared memory: two stages of K and V pages (4 x 64 x DH bf16), then
// the 4-warp combine and the cross-item combine reuse it; the four
// mbarriers sit above.
constexpr int kAttnMaxChunks = 256;  // 64-row pages per (kv head, m-tile): contexts up to 16K rows
constexpr int kAttnBarOffset = 72 * 1024;
constexpr int kAttnItemSmem = kAttnBarOffset + 64;
static_assert(4 * 64 * 128 * 2 <= kAttnBarOffset, "double-buffered K/V pages must fit below the barriers");
// One CTA item of the split-KV attention: 4 warps (threads tid 0..127, named
// barrier bar_id) over kv.attn_ppi 64-row key pages (chunk bx) of one kv
// head and one 16-pair m-tile (by = m-tile * n_kv + kv head), 16 keys per
// warp per page; chunks along the context combine through a split
// workspace, last item in fixed chunk order. Used by attn_mma_kernel
// (one item per CTA) and by the decode megakernel (items spread over SMs).
template <int DH>
__device__ __forceinline__ void attn_mma_item(const AttnProblem& A, const PassView& pass, const KvView& kv,
                                              int n_heads, int G_, int bx, int by, int nchunks_, int ny,
                                              unsigned char* smraw, unsigned* s_last_p, int tid, int bar_id,
                                              unsigned long long* dbg = nullptr) {
    unsigned& s_last = *s_last_p;
    constexpr int LDK = DH;               // bf16 elements per smem row (unpadded: one bulk copy per page)
    constexpr int NT = DH / 8;            // n8 tiles over head dims
    const int G = G_, H = n_heads, T = pass.T, P = T * G;
    const int n_kv = kv.n_kv;
    const int hk = by % n_kv, mt = by / n_kv;
    const int warp = tid >> 5, lane = tid & 31, gid = lane >> 2, tig = lane & 3;
    // item = kv.attn_ppi consecutive 64-row pages (chunk bx) of one kv head
    // and one 16-pair m-tile; warp w takes keys [16w, 16w + 16) of every page
    // (online softmax across the pages), so each warp's serial chain per page
    // is 16 + 16 mma and a 16-key softmax. K/V pages are double-buffered.
    const int ppi = kv.attn_ppi;
    const int splits = (pass.total + 63) / 64;
    const int pg0 = bx * ppi, pg1 = min(splits, pg0 + ppi);
    const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(kv.pool);
    // stage st: K at st*2*64*DH, V at (st*2+1)*64*DH (bf16 elements)
    __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(smraw);
    // one 1-D TMA bulk copy per K or V page (a 64-row page of one kv head is a
    // contiguous run); mbarriers [stage][K|V] above the buffers
    uint64_t* mb = reinterpret_cast<uint64_t*>(smraw + kAttnBarOffset);
    // the buffers were last written through the generic proxy (megakernel:
    // activation slots / earlier items); order that before the TMA writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    auto issue = [&](int pg) {  // tid 0 only
        const int st = (pg - pg0) & 1;
        uint64_t pol = 0;
        if (kv.l2_hint == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        if (kv.l2_hint == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        for (int kind = 0; kind < 2; ++kind) {
            void* dst = buf + (size_t)(st * 2 + kind) * 64 * DH;
            const void* src = pool + kv_off(kv, A.layer, kind, hk, pg * 64);
            mbar_arrive_expect_tx(&mb[st * 2 + kind], 64 * DH * 2);
            if (kv.l2_hint) tma_bulk_g2s_hint(dst, src, 64 * DH * 2, &mb[st * 2 + kind], pol);
            else tma_bulk_g2s(dst, src, 64 * DH * 2, &mb[st * 2 + kind]);
        }
    };
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&mb[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int pg = pg0; pg < pg1 && pg < pg0 + 2; ++pg) issue(pg);
    }
    // visibility of this lane's two query rows, loaded once up front (the
    // loads overlap the K/V copies instead of sitting in the softmax's path)
    int ve[2] = {0, 0};
    unsigned long long an[2] = {0ull, 0ull};
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
        const int p = mt * 16 + gid + 8 * ri;
        if (p < P) {
            ve[ri] = pass.vis_end[p / G];
            an[ri] = pass.anc[p / G];
        }
    }
    // Q A-fragments (pairs 16mt + gid / +8), scaled later on the scores
    uint32_t qa[DH / 16][4];
    {
        const int p0 = mt * 16 + gid, p1 = p0 + 8;
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
            qa[s][0] = pack_bf16x2(a.x, a.y);
            qa[s][1] = pack_bf16x2(b.x, b.y);
            qa[s][2] = pack_bf16x2(cc.x, cc.y);
            qa[s][3] = pack_bf16x2(d.x, d.y);
        }
    }
    named_bar(bar_id, 128);  // barriers initialised before anyone waits on them
    float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
    float o[NT][4];
#pragma unroll
    for (int d = 0; d < NT; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
    const float inv_sqrt = 1.0f / sqrtf((float)DH);
    const int pr[2] = {mt * 16 + gid, mt * 16 + gid + 8};
    for (int pg = pg0; pg < pg1; ++pg) {
        const int st = (pg - pg0) & 1;
        const uint32_t ph = (uint32_t)((pg - pg0) >> 1) & 1u;
        const __nv_bfloat16* Ks = buf + (size_t)(st * 2) * 64 * DH;
        const __nv_bfloat16* Vs = buf + (size_t)(st * 2 + 1) * 64 * DH;
        const int j0 = pg * 64 + warp * 16;
        const int nr = max(0, min(16, pass.total - j0));  // this warp's keys in the page
        if (nr > 0) {
            mbar_wait(&mb[st * 2], ph);
            if (dbg && pg == pg0 && lane == 0) atomicMax(dbg + 2, gtimer());
            float sc[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
#pragma unroll
                for (int s = 0; s < DH / 16; s += 2) {
                    uint32_t b[4];
                    ldsm_x4(b, Ks + (warp * 16 + j * 8 + (lane & 7)) * DH + s * 16 + (lane >> 3) * 8);
                    mma_bf16_16816(sc[j], qa[s], b[0], b[1]);
                    mma_bf16_16816(sc[j], qa[s + 1], b[2], b[3]);
                }
            }
            // scale + mask, online softmax over this page's 16 keys of the warp
            float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int ri = e >> 1;
                    const int key = j * 8 + 2 * tig + (e & 1);
                    const bool ok = pr[ri] < P && key < nr && visible_rows(pass, ve[ri], an[ri], j0 + key);
                    sc[j][e] = ok ? __fmul_rn(sc[j][e], inv_sqrt) : -INFINITY;
                    mx[ri] = fmaxf(mx[ri], sc[j][e]);
                }
            float alpha[2];
#pragma unroll
            for (int ri = 0; ri < 2; ++ri) {
                mx[ri] = fmaxf(mx[ri], __shfl_xor_sync(0xffffffffu, mx[ri], 1));
                mx[ri] = fmaxf(mx[ri], __shfl_xor_sync(0xffffffffu, mx[ri], 2));
                const float mn = fmaxf(m_r[ri], mx[ri]);
                // rescale of the running sums (exactly 1 while the max holds,
                // 0 while nothing was visible yet)
                alpha[ri] = m_r[ri] == -INFINITY ? 0.f : (mn == m_r[ri] ? 1.f : expf(m_r[ri] - mn));
                m_r[ri] = mn;
            }
            float sum[2] = {0.f, 0.f};
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int ri = e >> 1;
                    const float v = sc[j][e] == -INFINITY ? 0.f : expf(sc[j][e] - m_r[ri]);
                    sc[j][e] = v;
                    sum[ri] += v;
                }
#pragma unroll
            for (int ri = 0; ri < 2; ++ri) {
                sum[ri] += __shfl_xor_sync(0xffffffffu, sum[ri], 1);
                sum[ri] += __shfl_xor_sync(0xffffffffu, sum[ri], 2);
                l_r[ri] = __fmaf_rn(l_r[ri], alpha[ri], sum[ri]);
            }
#pragma unroll
            for (int d = 0; d < NT; ++d) {
                o[d][0] *= alpha[0];
                o[d][1] *= alpha[0];
                o[d][2] *= alpha[1];
                o[d][3] *= alpha[1];
            }
            mbar_wait(&mb[st * 2 + 1], ph);
            // O += P V over the 16 keys (one k-step)
            uint32_t pa[4];
            pa[0] = pack_bf16x2(sc[0][0], sc[0][1]);
            pa[1] = pack_bf16x2(sc[0][2], sc[0][3]);
            pa[2] = pack_bf16x2(sc[1][0], sc[1][1]);
            pa[3] = pack_bf16x2(sc[1][2], sc[1][3]);
#pragma unroll
            for (int d = 0; d < NT; d += 2) {
                uint32_t b[4];
                // matrices: (keys 0..7, dims 8d), (keys 8..15, dims 8d), (keys 0..7, dims 8d+8), (keys 8..15, dims 8d+8)
                const int mi = lane >> 3;
                ldsm_x4_t(b, Vs + (warp * 16 + (mi & 1) * 8 + (lane & 7)) * DH + d * 8 + (mi >> 1) * 8);
                mma_bf16_16816(o[d], pa, b[0], b[1]);
                mma_bf16_16816(o[d + 1], pa, b[2], b[3]);
            }
        }
        named_bar(bar_id, 128);  // stage st consumed by every warp
        if (tid == 0 && pg + 2 < pg1) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(pg + 2);
        }
    }
    if (dbg && lane == 0) atomicMax(dbg + 3, gtimer());
    if (tid == 0) {  // the barriers' memory is plain data from here on
        for (int i = 0; i < 4; ++i)
            asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&mb[i])) : "memory");
    }
    float* Os = reinterpret_cast<float*>(smraw);           // [4][16][DH]
    float* Ms = Os + 4 * 16 * DH;                          // [4][16]
    float* Ls = Ms + 64;                                   // [4][16]
    float* Fw = Ls + 64;                                   // [4][16] warp weights exp(m_w - M)
    float* Rm = Fw + 64;                                   // [16] row max
    float* Rd = Rm + 16;                                   // [16] row denominator
#pragma unroll
    for (int d = 0; d < NT; ++d) {
        const int c = d * 8 + 2 * tig;
        *reinterpret_cast<float2*>(&Os[(warp * 16 + gid) * DH + c]) = make_float2(o[d][0], o[d][1]);
        *reinterpret_cast<float2*>(&Os[(warp * 16 + gid + 8) * DH + c]) = make_float2(o[d][2], o[d][3]);
    }
    if (tig == 0) {
        Ms[warp * 16 + gid] = m_r[0];
        Ms[warp * 16 + gid + 8] = m_r[1];
        Ls[warp * 16 + gid] = l_r[0];
        Ls[warp * 16 + gid + 8] = l_r[1];
    }
    named_bar(bar_id, 128);
    if (tid < 16) {  // per-row weights, fixed warp order
        const int r = tid;
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
    const int nchunks = nchunks_;
    constexpr int PS = DH + 4;  // workspace row: DH values, M, den (float4-aligned)
    float* wsb = A.ws + (((size_t)bx * ny + by) * 16) * PS;
    {
        // thread -> (row r, 16 consecutive dims)
        constexpr int CPR = DH / 16;  // threads per row
        for (int it = tid; it < 16 * CPR; it += 128) {
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
                if (p < P) {
                    attn_store_row<DH>(A, (size_t)(p / G) * H * DH + (hk * G + p % G) * DH + c0, acc, Rd[r]);
                }
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
    const size_t cstride = (size_t)ny * 16 * PS;
    const float* base = A.ws + ((size_t)by * 16) * PS;
    // per-row chunk weights f = exp(m_ch - M) and denominator, once per row
    float* fac = Os;                          // [nchunks <= kAttnMaxChunks][16]
    float* sden = Os + kAttnMaxChunks * 16;   // [16]
    // (m, l) of every chunk: one float2 load each, all issued together
    float2* ml = reinterpret_cast<float2*>(Os + kAttnMaxChunks * 16 + 16);  // [nchunks][16]
    for (int i = tid; i < nchunks * 16; i += 128) {
        const int ch = i >> 4, r = i & 15;
        ml[i] = __ldcg(reinterpret_cast<const float2*>(base + ch * cstride + r * PS + DH));
    }
    named_bar(bar_id, 128);
    if (tid < 16) {
        const int r = tid;
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
    for (int it = tid; it < 16 * CPR; it += 128) {
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
    if (dbg && tid == 0) atomicMax(dbg + 5, gtimer());
}

}  // namespace espec_dev
