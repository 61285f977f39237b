// Sampling, tree-child selection and rejection-sampling verification on
// device (sm_100a). These restate the reference's T > 0 path and its
// multi-sibling tree levels:
//   softmax_temp          proj/src/matrix.cpp:88-116
//   select_children       proj/src/draft_engine.cpp:141-186
//   residual_distribution proj/src/verifier.cpp:25-43
//   sample_from           proj/src/verifier.cpp:70-84
//   verify_tree           proj/src/verifier.cpp:86-177
// The random stream is the reference's: the host draws xoshiro256** uniforms
// in stream order and the kernels consume them through a device cursor, so
// the order of draws (draft selections level by level, then one uniform per
// tested sibling, then the bonus) is exactly the reference's; the host
// advances its generator by the number consumed.
//
// Vocabulary-wide passes are single-CTA (1024 threads, each thread owning a
// contiguous slice of the vocabulary); every reduction and prefix scan has a
// fixed order, so results are deterministic.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace espec_dev {

constexpr int kSThreads = 1024;
constexpr int kSWarps = kSThreads / 32;

#define SCK(x) DEV_CK(x)

__device__ __forceinline__ bool s_better(float v, int i, float bv, int bi) { return v > bv || (v == bv && i < bi); }

// ---- fixed-order block reductions / scans (1024 threads) ----

__device__ double block_sum_d(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = red[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0) red[32] = w;
    }
    __syncthreads();
    const double r = red[32];
    __syncthreads();
    return r;
}

__device__ float block_sum_f(float v, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        float w = warp_sum(red[lane]);
        if (lane == 0) red[32] = w;
    }
    __syncthreads();
    const float r = red[32];
    __syncthreads();
    return r;
}

__device__ float block_max_f(float v, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_max(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        float w = warp_max(red[lane]);
        if (lane == 0) red[32] = w;
    }
    __syncthreads();
    const float r = red[32];
    __syncthreads();
    return r;
}

// argmax with the reference's tie-break (first maximum, matrix.cpp:196-202)
__device__ int block_argmax(float v, int i, float* redv, int* redi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (s_better(ov, oi, v, i)) {
            v = ov;
            i = oi;
        }
    }
    if (lane == 0) {
        redv[warp] = v;
        redi[warp] = i;
    }
    __syncthreads();
    if (warp == 0) {
        float w = redv[lane];
        int wi = redi[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, w, o);
            const int oi = __shfl_xor_sync(0xffffffffu, wi, o);
            if (s_better(ov, oi, w, wi)) {
                w = ov;
                wi = oi;
            }
        }
        if (lane == 0) redi[32] = wi;
    }
    __syncthreads();
    const int r = redi[32];
    __syncthreads();
    return r;
}

// First index t (scanning up from 0, skipping weights <= 0) whose inclusive
// prefix exceeds u, or the last positive index if none does (the inverse-CDF
// walks of select_children / sample_from). w(t) is the weight of token t.
// Thread i owns the slice [i*C, (i+1)*C); slice sums are scanned in a fixed
// order and thread i's interval is [incl[i-1], incl[i]) — the same stored
// numbers for both neighbours, so the intervals partition the line exactly.
template <typename W>
__device__ int block_inverse_cdf(int V, double u, W w, double* incl, int* sidx) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int C = (V + kSThreads - 1) / kSThreads;
    const int lo = threadIdx.x * C, hi = min(V, lo + C);
    double local = 0.0;
    int last_pos = -1;
    for (int t = lo; t < hi; ++t) {
        const double x = w(t);
        if (x > 0.0) {
            local += x;
            last_pos = t;
        }
    }
    double inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    incl[threadIdx.x] = inc;  // warp-local inclusive
    if (threadIdx.x == 0) {
        sidx[0] = 0x7fffffff;
        sidx[1] = -1;
    }
    __syncthreads();
    if (warp == 0) {  // warp offsets, sequential in warp order
        double off = 0.0;
        for (int q = 0; q < lane; ++q) off += incl[q * 32 + 31];
        incl[kSThreads + lane] = off;
    }
    __syncthreads();
    const double hi_b = incl[kSThreads + warp] + inc;
    __syncthreads();
    incl[threadIdx.x] = hi_b;  // global inclusive prefix of slice sums
    __syncthreads();
    const double lo_b = threadIdx.x == 0 ? 0.0 : incl[threadIdx.x - 1];
    if (u >= lo_b && u < hi_b) {
        double cum = lo_b;
        int pick = -1;
        for (int t = lo; t < hi; ++t) {
            const double x = w(t);
            if (x <= 0.0) continue;
            cum += x;
            pick = t;
            if (u < cum) break;
        }
        if (pick >= 0) atomicMin(&sidx[0], pick);
    }
    if (last_pos >= 0) atomicMax(&sidx[1], last_pos);
    __syncthreads();
    const int r = sidx[0] != 0x7fffffff ? sidx[0] : sidx[1];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// softmax_temp over rows of logits
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kSThreads) softmax_rows_kernel(SoftmaxArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ float redf[33];
    __shared__ int redi[33];
    const int row = blockIdx.x;
    const float* l = a.logits + (size_t)a.src_row[row] * a.ld_logits;
    float* p = a.dists + (size_t)a.dst_row[row] * a.ld_dists;
    const int V = a.vocab;
    bool bad = false;
    for (int t = threadIdx.x; t < V; t += kSThreads) bad |= !isfinite(l[t]);
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) atomicExch(a.err, 1);  // DomainError: non-finite logit
        return;
    }
    if (a.temperature == 0.0f) {
        float bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int t = threadIdx.x; t < V; t += kSThreads)
            if (s_better(l[t], t, bv, bi)) {
                bv = l[t];
                bi = t;
            }
        const int am = block_argmax(bv, bi, redf, redi);
        for (int t = threadIdx.x; t < V; t += kSThreads) p[t] = t == am ? 1.0f : 0.0f;
        return;
    }
    float mx = -INFINITY;
    for (int t = threadIdx.x; t < V; t += kSThreads) mx = fmaxf(mx, l[t]);
    mx = block_max_f(mx, redf);
    float sum = 0.f;
    for (int t = threadIdx.x; t < V; t += kSThreads) {
        const float ex = expf(__fdiv_rn(__fsub_rn(l[t], mx), a.temperature));
        p[t] = ex;
        sum += ex;
    }
    sum = block_sum_f(sum, redf);
    for (int t = threadIdx.x; t < V; t += kSThreads) p[t] = __fdiv_rn(p[t], sum);
}

void launch_softmax_rows(const SoftmaxArgs& a, int rows, cudaStream_t s) {
    if (rows <= 0) return;
    SCK(launch_pdl(softmax_rows_kernel, dim3(rows), dim3(kSThreads), 0, s, a));
}

// ---------------------------------------------------------------------------
// select_children for the frontier rows of one draft level, in row order
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kSThreads) select_children_kernel(SelectArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ double redd[33];
    __shared__ double incl[kSThreads + 32];
    __shared__ float redf[33];
    __shared__ int redi[33];
    __shared__ int sidx[2];
    __shared__ int chosen[kMaxWidth];
    const int V = a.vocab;
    for (int row = 0; row < a.rows; ++row) {
        const int k = a.width[row];
        int* out = a.tok_arena + a.child_at[row];
        if (a.temperature == 0.0f) {
            // top-k by (logit desc, id asc)
            const float* l = a.logits + (size_t)a.logit_row[row] * a.ld_logits;
            for (int r0 = 0; r0 < k; ++r0) {
                float bv = -INFINITY;
                int bi = 0x7fffffff;
                for (int t = threadIdx.x; t < V; t += kSThreads) {
                    bool taken = false;
                    for (int q = 0; q < r0; ++q) taken |= chosen[q] == t;
                    if (!taken && s_better(l[t], t, bv, bi)) {
                        bv = l[t];
                        bi = t;
                    }
                }
                const int best = block_argmax(bv, bi, redf, redi);
                if (threadIdx.x == 0) {
                    chosen[r0] = best;
                    out[r0] = best;
                }
                __syncthreads();
            }
            continue;
        }
        // k sequential draws without replacement over double weights
        const float* p = a.dists + (size_t)a.dist_row[row] * a.ld_dists;
        double local = 0.0;
        const int C = (V + kSThreads - 1) / kSThreads;
        for (int t = threadIdx.x * C; t < min(V, (int)(threadIdx.x + 1) * C); ++t) local += (double)p[t];
        double mass = block_sum_d(local, redd);
        int cnt = 0;
        for (int round = 0; round < k && mass > 1e-12; ++round) {
            const double u = a.uniforms[*a.cursor + round] * mass;
            const int n_ch = cnt;
            auto w = [&](int t) -> double {
                for (int q = 0; q < n_ch; ++q)
                    if (chosen[q] == t) return 0.0;
                return (double)p[t];
            };
            const int pick = block_inverse_cdf(V, u, w, incl, sidx);
            if (pick < 0) break;
            if (threadIdx.x == 0) {
                chosen[cnt] = pick;
                out[cnt] = pick;
            }
            mass -= (double)p[pick];
            ++cnt;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            *a.cursor += cnt;
            if (cnt < k) atomicExch(a.err, 2);  // draft distribution exhausted before the tree width
        }
        __syncthreads();
    }
}

void launch_select_children(const SelectArgs& a, cudaStream_t s) {
    if (a.rows <= 0) return;
    SCK(launch_pdl(select_children_kernel, dim3(1), dim3(kSThreads), 0, s, a));
}

// ---------------------------------------------------------------------------
// verify_tree at T > 0 (and vanilla sampling: an empty tree)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kSThreads) verify_sample_kernel(VerifyArgs a) {
    pdl_wait();
    pdl_trigger();
    __shared__ double redd[33];
    __shared__ double incl[kSThreads + 32];
    __shared__ int sidx[2];
    __shared__ int zeroed[kMaxWidth];
    const int V = a.vocab;
    const int C = (V + kSThreads - 1) / kSThreads;
    const int lo = threadIdx.x * C, hi = min(V, lo + C);
    float* target = a.target;
    for (int t = lo; t < hi; ++t) target[t] = a.base_dists[t];  // row 0: the frontier
    __syncthreads();
    int cursor = *a.cursor;
    int parent = -1, m = 0;
    bool failed = false;
    for (int depth = 1; depth <= a.n_levels && !failed; ++depth) {
        const int first = parent < 0 ? 0 : a.node_first_child[parent];
        const int count = parent < 0 ? a.root_children : a.node_n_children[parent];
        if (count == 0) break;
        const float* dist = a.draft_dists + (size_t)a.node_prob_index[first] * a.ld_dists;
        double local = 0.0;
        for (int t = lo; t < hi; ++t) local += (double)dist[t];
        double dm = block_sum_d(local, redd);
        int nz = 0;
        int acc = -1;
        for (int i = 0; i < count; ++i) {
            const int ni = first + i;
            const int tok = a.tok_arena[a.node_tok_idx[ni]];
            const double p_tok = target[tok];
            const int nzi = nz;
            auto ld = [&](int t) -> double {
                for (int q = 0; q < nzi; ++q)
                    if (zeroed[q] == t) return 0.0;
                return (double)dist[t];
            };
            const double pp_tok = ld(tok) / dm;
            const double u = a.uniforms[cursor++];
            if (!(pp_tok > 0.0)) {
                failed = true;  // CheckError: drafted token carries zero draft probability
                if (threadIdx.x == 0) atomicExch(a.err, 3);
                break;
            }
            const double ratio = p_tok / pp_tok;
            if (u < (ratio < 1.0 ? ratio : 1.0)) {
                acc = ni;
                break;
            }
            // target = norm(max(0, target - p'))  (residual_distribution)
            double mloc = 0.0;
            for (int t = lo; t < hi; ++t) {
                const float clamped = (float)(ld(t) / dm);
                const double diff = (double)target[t] - clamped;
                if (diff > 0.0) mloc += diff;
            }
            const double mass = block_sum_d(mloc, redd);
            if (!(mass < 1e-9)) {
                for (int t = lo; t < hi; ++t) {
                    const float clamped = (float)(ld(t) / dm);
                    const double diff = (double)target[t] - clamped;
                    const float tmp = diff > 0.0 ? (float)diff : 0.0f;
                    target[t] = (float)((double)tmp / mass);
                }
            }
            __syncthreads();
            dm -= ld(tok);
            if (threadIdx.x == 0) zeroed[nz] = tok;
            ++nz;
            __syncthreads();
            if (dm <= 1e-9 && i + 1 < count) {
                failed = true;  // CheckError: sibling candidates exhaust the draft distribution
                if (threadIdx.x == 0) atomicExch(a.err, 4);
                break;
            }
        }
        if (acc < 0 || failed) break;
        if (threadIdx.x == 0) {
            a.outcome[2 + m] = acc;
            a.outcome[2 + a.n_levels + m] = a.tok_arena[a.node_tok_idx[acc]];
            a.tok_arena_w[a.commit_at + m] = a.tok_arena[a.node_tok_idx[acc]];
        }
        ++m;
        const float* nb = a.base_dists + (size_t)(acc + 1) * a.ld_dists;
        for (int t = lo; t < hi; ++t) target[t] = nb[t];
        __syncthreads();
        parent = acc;
    }
    if (failed) return;
    // bonus = sample_from(target)
    const double u = a.uniforms[cursor++];
    auto wt = [&](int t) -> double { return (double)target[t]; };
    const int bonus = block_inverse_cdf(V, u, wt, incl, sidx);
    if (threadIdx.x == 0) {
        if (bonus < 0) atomicExch(a.err, 5);  // CheckError: sampling from an all-zero distribution
        a.outcome[0] = m;
        a.outcome[1] = bonus < 0 ? 0 : bonus;
        a.tok_arena_w[a.commit_at + m] = bonus < 0 ? 0 : bonus;
        *a.cursor = cursor;
    }
}

void launch_verify_sample(const VerifyArgs& a, cudaStream_t s) {
    SCK(launch_pdl(verify_sample_kernel, dim3(1), dim3(kSThreads), 0, s, a));
}

}  // namespace espec_dev
