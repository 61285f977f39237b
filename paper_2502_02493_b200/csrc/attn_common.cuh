// Attention pieces shared by the attention kernels: paged-KV addressing,
// tree-aware visibility and the output-row store.
// Attention semantics: proj/src/model.cpp:140-192; mask proj/src/kv_cache.cpp:43-60.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace espec_dev {

__device__ __forceinline__ long long kv_off(const KvView& kv, int layer, int kind, int head, int row) {
    const int page = kv.page_table[row / kv.page_rows];
    const int r = row % kv.page_rows;
    return (long long)page * kv.page_elems +
           ((((long long)layer * 2 + kind) * kv.n_kv + head) * kv.page_rows + r) * kv.dh;
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

// 16 output values (one pair row, 16 consecutive dims) = acc / den: fp32, or
// bf16 rounded to nearest (exactly what the O GEMV's staging would do) when
// the consumer takes bf16 activations
template <int DH, int NV>
__device__ __forceinline__ void attn_store_row(const AttnProblem& A, size_t off, const float4 (&acc)[NV], float den) {
    float y[4 * NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        y[4 * v] = den > 0.f ? acc[v].x / den : 0.f;
        y[4 * v + 1] = den > 0.f ? acc[v].y / den : 0.f;
        y[4 * v + 2] = den > 0.f ? acc[v].z / den : 0.f;
        y[4 * v + 3] = den > 0.f ? acc[v].w / den : 0.f;
    }
    if (A.out_bf16) {
        uint32_t pk[2 * NV];
#pragma unroll
        for (int j = 0; j < 2 * NV; ++j) {
            const __nv_bfloat162 b = __floats2bfloat162_rn(y[2 * j], y[2 * j + 1]);
            pk[j] = *reinterpret_cast<const uint32_t*>(&b);
        }
        __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(A.out) + off;
        if constexpr (NV == 1) {
            *reinterpret_cast<uint2*>(ob) = make_uint2(pk[0], pk[1]);
        } else {
#pragma unroll
            for (int v = 0; v < NV / 2; ++v)
                reinterpret_cast<uint4*>(ob)[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
        }
    } else {
        float* o = A.out + off;
#pragma unroll
        for (int v = 0; v < NV; ++v)
            *reinterpret_cast<float4*>(o + 4 * v) = make_float4(y[4 * v], y[4 * v + 1], y[4 * v + 2], y[4 * v + 3]);
    }
}

}  // namespace espec_dev
