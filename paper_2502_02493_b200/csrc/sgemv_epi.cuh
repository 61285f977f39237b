// Fused GEMV unit epilogue (RESID + row stats / SiLU·up / RoPE + paged-KV
// write / store / argmax), shared by the stream-K GEMV and the decode
// megakernel so both compute bit-identical rows.
#pragma once
#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace espec_dev {

struct SgEpiCtx {
    const PassView& pass;
    const KvView& kv;
    int T, t0, ngroups;
    // optional per-row metadata of rows [t0, t0+T) (decode megakernel: shared
    // memory): rotary position and the row's paged-KV base offset
    // page_table[row / page_rows] * page_elems + (row % page_rows) * dh
    const int* pos = nullptr;
    const long long* kv_row = nullptr;
    // optional residual rows already loaded by the caller (resid of the
    // unit's column for rows t < T)
    const float* pre = nullptr;
    // optional rotary factors (cos, sin) of the unit's column for rows t < T
    const float2* rope = nullptr;
};

// Unit epilogue, run by one epilogue warp: lane = column within the 32-column
// group, v[t] = the unit's full sum for row t (after the k-chunk reduction).
template <int TM, int EPI>
__device__ __forceinline__ void sg_epilogue(const SgEpiCtx& L, const GemvProblem& P, int g, const float (&v)[TM],
                                            int lane) {
    const int T = L.T, t0 = L.t0;
    const int c = g * 32 + lane;
    if (EPI == EPI_RESID || (EPI == EPI_STORE && P.resid != nullptr)) {
        // h_mid = h + attn / h_next = h_mid + mlp (proj/src/draft_engine.cpp:15-19) + row stats.
        // Fuzzy groups fuse their residual adds here (same fp32 operations, same
        // order as separate add kernels): a STORE problem with `resid` is the
        // group's first h += attn_0; `resid2` adds the next layer's attn_{i+1}
        // right after h += mlp_i.
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            if (t >= T) break;
            float sq = 0.f;
            if (c < P.N) {
                float y = __fadd_rn(L.pre ? L.pre[t] : __ldcg(P.resid + (size_t)(t0 + t) * P.ldr + c), v[t]);
                if (EPI == EPI_RESID && P.resid2 != nullptr)
                    y = __fadd_rn(y, __ldcg(P.resid2 + (size_t)(t0 + t) * P.ldr2 + c));
                P.out[(size_t)(t0 + t) * P.ldo + c] = y;
                sq = y * y;
            }
            sq = warp_sum(sq);
            if (lane == 0) P.stats_out[(t0 + t) * P.stat_tiles_out + g] = sq;
        }
    } else if constexpr (EPI == EPI_STORE) {
        if (P.push_n > 0) {
            // tensor-parallel partial: straight into every rank's receive slot
            // (NVLink stores, tile by tile as the GEMV finishes its columns)
#pragma unroll
            for (int t = 0; t < TM; ++t)
                if (t < T && c < P.N)
                    for (int p = 0; p < P.push_n; ++p) P.push[p][(size_t)(t0 + t) * P.N + c] = v[t];
        } else {
#pragma unroll
            for (int t = 0; t < TM; ++t)
                if (t < T && c < P.N) P.out[(size_t)(t0 + t) * P.ldo + c] = v[t];
        }
    }
    if constexpr (EPI == EPI_SILU) {
        // packed group = [gate 16 | up 16]: silu(gate) * up (proj/src/model.cpp:197-210)
        const int a = g * 16 + lane;
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            const float up = __shfl_down_sync(0xffffffffu, v[t], 16);
            if (t < T && lane < 16 && a < P.N / 2) {
                const float y = __fmul_rn(__fdiv_rn(v[t], __fadd_rn(1.0f, expf(-v[t]))), up);
                if (P.out_bf16)
                    reinterpret_cast<__nv_bfloat16*>(P.out)[(size_t)(t0 + t) * P.ldo + a] = __float2bfloat16_rn(y);
                else
                    P.out[(size_t)(t0 + t) * P.ldo + a] = y;
            }
        }
    } else if constexpr (EPI == EPI_QKV) {
        // q = rope(h.Wq), k = rope(h.Wk), v = h.Wv ; K/V into the paged cache
        // (proj/src/model.cpp:130-138, rotary proj/src/matrix.cpp:159-194)
        const int qd = P.n_heads * P.dh, kd = P.n_kv * P.dh;
        const int region = c < qd ? 0 : (c < qd + kd ? 1 : 2);
        const int base = region == 0 ? 0 : (region == 1 ? qd : qd + kd);
        const int within = c - base;
        const int head = within / P.dh, i = within - head * P.dh;
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            const float other = __shfl_xor_sync(0xffffffffu, v[t], 1);
            if (t >= T || c >= P.N) continue;
            float y = v[t];
            if (region < 2) {
                const int pos = L.pos ? L.pos[t] : L.pass.pos[t0 + t];
                const float2 cs_sn = L.rope ? L.rope[t] : P.rope[(size_t)pos * (P.dh >> 1) + (i >> 1)];
                const float cs = cs_sn.x, sn = cs_sn.y;
                y = (i & 1) ? __fadd_rn(__fmul_rn(other, sn), __fmul_rn(v[t], cs))
                            : __fsub_rn(__fmul_rn(v[t], cs), __fmul_rn(other, sn));
            }
            if (region == 0) {
                P.out[(size_t)(t0 + t) * P.ldo + c] = y;
            } else {
                const long long off =
                    (L.kv_row ? L.kv_row[t] + ((((long long)P.layer * 2 + (region - 1)) * L.kv.n_kv + head) * L.kv.page_rows) * L.kv.dh
                              : sg_kv_off(L.kv, P.layer, region - 1, head, L.pass.rows[t0 + t])) + i;
                if (L.kv.dtype == DT_BF16) reinterpret_cast<__nv_bfloat16*>(L.kv.pool)[off] = __float2bfloat16_rn(y);
                else reinterpret_cast<float*>(L.kv.pool)[off] = y;
            }
        }
    } else if constexpr (EPI == EPI_ARGMAX) {
        // logits = norm(h).E^T ; greedy pick = first maximum (proj/src/matrix.cpp:196-202)
#pragma unroll
        for (int t = 0; t < TM; ++t) {
            if (t >= T) break;
            float bv = -INFINITY;
            int bi = 0x7fffffff;
            if (c < P.vocab) {
                if (P.logits) P.logits[(size_t)(t0 + t) * P.ld_logits + c] = v[t];
                bv = v[t];
                bi = c;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (sg_better(ov, oi, bv, bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) {
                P.am_val[(t0 + t) * L.ngroups + g] = bv;
                P.am_idx[(t0 + t) * L.ngroups + g] = bi;
            }
        }
        // last group to finish reduces the per-group maxima (fixed-order-free:
        // max with lowest-index tie-break is order independent)
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) {
            last = ticket_acq_rel(&P.tickets[L.ngroups]) == (unsigned)L.ngroups - 1 ? 1u : 0u;
            if (last) P.tickets[L.ngroups] = 0u;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            for (int t = 0; t < T; ++t) {
                float fv = -INFINITY;
                int fi = 0x7fffffff;
                for (int q = lane; q < L.ngroups; q += 32) {
                    const float ov = __ldcg(&P.am_val[(t0 + t) * L.ngroups + q]);
                    const int oi = __ldcg(&P.am_idx[(t0 + t) * L.ngroups + q]);
                    if (sg_better(ov, oi, fv, fi)) {
                        fv = ov;
                        fi = oi;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, fv, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, fi, o);
                    if (sg_better(ov, oi, fv, fi)) {
                        fv = ov;
                        fi = oi;
                    }
                }
                if (lane == 0) {
                    P.tok_out[t0 + t] = fi + P.col_base;
                    if (P.tok_val) P.tok_val[t0 + t] = fv;
                }
            }
        }
    }
}

}  // namespace espec_dev
