// Tensor-parallel collectives over NVLink peer memory (sm_100a).
//
// One process (or one engine shard) per GPU. Every rank owns a symmetric
// receive region — recv[2 parities][world senders][slot floats] plus
// flags[2][world] — that its peers map (CUDA IPC across processes, plain
// device pointers between shards of one process). A collective is one
// kernel per rank:
//   1. push: the CTAs copy this rank's contribution into every rank's
//      recv[parity][rank] slot with ordinary stores over NVLink, then
//      fence at system scope;
//   2. signal: the last CTA (ticket) writes the call's sequence number into
//      flags[parity][rank] of every rank (st.release.sys);
//   3. wait: every CTA spins on its local flags[parity][s] for all senders
//      (ld.acquire.sys);
//   4. combine: each CTA reads its slice of all senders' slots (L2, never
//      L1: peers write behind it) and reduces them in rank order 0..N-1 —
//      a fixed order, so the sum of a row never depends on the message size
//      (T) and greedy speculative decoding stays equal to greedy vanilla.
// Two parities let call k+1 push while a slow peer still reads call k.
// Between GPUs the kernel lets its successor launch early (PDL) so the next
// GEMV streams weights while this one waits on peers. Shards sharing ONE GPU
// (the single-device test harness) must not: a pre-launched successor
// parked on every SM could starve the peer shard that this kernel waits on.
// Sequence numbers only grow, so flags never need resetting.
// Shard proxy (CommView::loopback): one engine impersonates every rank of a
// TP-N group on one GPU, so a single-GPU run exposes the per-GPU step of a
// TP-N deployment (shard-sized GEMVs, N-slot collectives) without peers.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace espec_dev {

#define CCK(x) DEV_CK(x)

constexpr int kCommThreads = 256;
constexpr int kCommMaxCtas = 32;

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float* slot(const CommView& c, float* base, int par, int sender) {
    return base + ((size_t)par * c.world + sender) * c.slot_floats;
}

// steps 2 + 3: after every CTA pushed, the last one signals; all wait.
__device__ void comm_signal_wait(const CommView& c, uint64_t seq, int par) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tk;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(tk) : "l"(c.ticket) : "memory");
        if (c.debug) printf("[dev] rank %d seq %llu block %d ticket %u of %d\n", c.rank, (unsigned long long)seq, blockIdx.x, tk, gridDim.x);
        if (tk == gridDim.x - 1) {
            *c.ticket = 0u;
            __threadfence_system();
            for (int p = 0; p < c.world; ++p)
                st_release_sys(c.peer_flags[p] + (size_t)par * c.world + (c.loopback ? p : c.rank), seq);
        }
        const long long t0 = clock64();
        for (int s = 0; s < c.world; ++s) {
            const uint64_t* f = c.flags_local + (size_t)par * c.world + s;
            while (ld_acquire_sys(f) < seq) {
                // a peer that never arrives is a broken group: fail the
                // kernel (~20 s at 2 GHz) instead of hanging the GPU
                if (clock64() - t0 > 40000000000LL) {
                    printf("espec collective: rank %d timed out waiting for rank %d (seq %llu, flag %llu, block %d/%d)\n",
                           c.rank, s, (unsigned long long)seq, (unsigned long long)ld_acquire_sys(f), blockIdx.x,
                           gridDim.x);
                    // reported as ESPEC_NCCL at the iteration's outcome read
                    // (the context stays usable; the engine must be rebuilt)
                    if (c.err) atomicExch(c.err, kCommErrTimeout);
                    break;
                }
            }
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// all-reduce of a rows x d fp32 block (row-parallel GEMV partials)
// ---------------------------------------------------------------------------

__device__ __forceinline__ size_t ar_row(const AllreduceArgs& a, int r, int ld) {
    if (a.rows_per_block <= 0) return (size_t)r * ld;
    return (size_t)(r / a.rows_per_block) * a.block_stride + (size_t)(r % a.rows_per_block) * ld;
}

enum : int { PH_PUSH = 1, PH_SYNC = 2, PH_COMBINE = 4, PH_ALL = 7 };

__global__ void __launch_bounds__(kCommThreads, 6) allreduce_rows_kernel(CommView c, uint64_t seq, AllreduceArgs a,
                                                                        int phases) {
    pdl_wait();
    if (c.early_trigger) pdl_trigger();  // the next GEMV may stream its weights while this one waits on peers
    const int par = (int)(seq & 1);
    const int d = a.d;
    const int groups = a.rows * ((d + 31) / 32);  // (row, 32-column group) units
    const int g0 = (int)((long long)blockIdx.x * groups / gridDim.x);
    const int g1 = (int)((long long)(blockIdx.x + 1) * groups / gridDim.x);
    const int gpr = (d + 31) / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // 1. push this rank's partial to every rank (packed rows x d)
    if (phases & PH_PUSH)
    for (int g = g0 + warp; g < g1; g += kCommThreads / 32) {
        const int r = g / gpr, col = (g - r * gpr) * 32 + lane;
        if (col < d) {
            const bool zero = a.rows_per_block > 0 && ((a.zero_blocks >> (r / a.rows_per_block)) & 1u);
            const float v = zero ? 0.f : a.src[ar_row(a, r, a.ld_src) + col];
            for (int p = 0; p < c.world; ++p) slot(c, c.peer_recv[p], par, c.loopback ? p : c.rank)[(size_t)r * d + col] = v;
        }
    }
    if (phases & PH_SYNC) comm_signal_wait(c, seq, par);
    if (!(phases & PH_COMBINE)) return;
    // 4. combine in rank order + epilogue
    for (int g = g0 + warp; g < g1; g += kCommThreads / 32) {
        const int r = g / gpr, gc = g - r * gpr, col = gc * 32 + lane;
        float v = 0.f;
        if (col < d)
            for (int s = 0; s < c.world; ++s) v += __ldcg(slot(c, c.recv_local, par, s) + (size_t)r * d + col);
        if (a.mode == AR_STORE) {
            if (col < d) a.out[ar_row(a, r, a.ldo) + col] = v;
        } else {
            // residual add + row statistics (the RESID epilogue of the 1-GPU path)
            float sq = 0.f;
            if (col < d) {
                const float y = __fadd_rn(a.resid[ar_row(a, r, a.ldr) + col], v);
                a.out[ar_row(a, r, a.ldo) + col] = y;
                sq = y * y;
            }
            sq = warp_sum(sq);
            if (lane == 0) a.stats[r * a.stat_tiles + gc] = sq;
        }
    }
}

void launch_allreduce_rows(CommView& c, const AllreduceArgs& a, cudaStream_t s) {
    if (a.rows <= 0) return;
    if ((size_t)a.rows * a.d > c.slot_floats)
        dev_fail(DEV_ERR_COMM, "allreduce: " + std::to_string(a.rows) + " x " + std::to_string(a.d) + " exceeds the " +
                                   std::to_string(c.slot_floats) + "-float comm slot");
    const uint64_t seq = ++c.seq;
    if (getenv("ESPEC_TRACE_COMM")) fprintf(stderr, "[comm] rank %d allreduce seq %llu rows %d\n", c.rank, (unsigned long long)seq, a.rows);
    const int groups = a.rows * ((a.d + 31) / 32);
    int ctas = (groups + 7) / 8;
    if (ctas > kCommMaxCtas) ctas = kCommMaxCtas;
    if (c.local_sync) {
        if (!a.prepushed)
            CCK(launch_pdl(allreduce_rows_kernel, dim3(ctas), dim3(kCommThreads), 0, s, c, seq, a, (int)PH_PUSH));
        c.local_sync(c.local_ctx, c.rank, s);
        CCK(launch_pdl(allreduce_rows_kernel, dim3(ctas), dim3(kCommThreads), 0, s, c, seq, a, (int)PH_COMBINE));
    } else {
        CCK(launch_pdl(allreduce_rows_kernel, dim3(ctas), dim3(kCommThreads), 0, s, c, seq, a,
                       a.prepushed ? (int)(PH_SYNC | PH_COMBINE) : (int)PH_ALL));
    }
}

// The receive slot that rank `c.rank` fills in every rank's region for the
// NEXT collective call (its parity), as a GEMV epilogue push target.
float* comm_push_slot(const CommView& c, int p) {
    const uint64_t par = (c.seq + 1) & 1;
    const int sender = c.loopback ? p : c.rank;
    return c.peer_recv[p] + ((size_t)par * c.world + sender) * c.slot_floats;
}

// ---------------------------------------------------------------------------
// all-gather of column slices: dst[r][s*cols + j] = src_s[r][j]
// (vocab-parallel logits for sampling)
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kCommThreads, 6) allgather_cols_kernel(CommView c, uint64_t seq, GatherColsArgs a,
                                                                        int phases) {
    pdl_wait();
    if (c.early_trigger) pdl_trigger();
    const int par = (int)(seq & 1);
    const long long n = (long long)a.rows * a.cols;
    const long long i0 = (long long)blockIdx.x * kCommThreads + threadIdx.x;
    const long long stride = (long long)gridDim.x * kCommThreads;
    if (phases & PH_PUSH)
        for (long long i = i0; i < n; i += stride) {
            const int r = (int)(i / a.cols), j = (int)(i - (long long)r * a.cols);
            const float v = a.src[(size_t)r * a.ld_src + j];
            for (int p = 0; p < c.world; ++p) slot(c, c.peer_recv[p], par, c.loopback ? p : c.rank)[i] = v;
        }
    if (phases & PH_SYNC) comm_signal_wait(c, seq, par);
    if (!(phases & PH_COMBINE)) return;
    for (int s = 0; s < c.world; ++s)
        for (long long i = i0; i < n; i += stride) {
            const int r = (int)(i / a.cols), j = (int)(i - (long long)r * a.cols);
            a.dst[(size_t)r * a.ld_dst + (size_t)s * a.cols + j] = __ldcg(slot(c, c.recv_local, par, s) + i);
        }
}

void launch_allgather_cols(CommView& c, const GatherColsArgs& a, cudaStream_t s) {
    if (a.rows <= 0) return;
    if ((size_t)a.rows * a.cols > c.slot_floats)
        dev_fail(DEV_ERR_COMM, "allgather: " + std::to_string(a.rows) + " x " + std::to_string(a.cols) +
                                   " exceeds the comm slot");
    const uint64_t seq = ++c.seq;
    long long n = (long long)a.rows * a.cols;
    int ctas = (int)((n + kCommThreads * 4 - 1) / (kCommThreads * 4));
    if (ctas > kCommMaxCtas) ctas = kCommMaxCtas;
    if (ctas < 1) ctas = 1;
    if (c.local_sync) {
        CCK(launch_pdl(allgather_cols_kernel, dim3(ctas), dim3(kCommThreads), 0, s, c, seq, a, (int)PH_PUSH));
        c.local_sync(c.local_ctx, c.rank, s);
        CCK(launch_pdl(allgather_cols_kernel, dim3(ctas), dim3(kCommThreads), 0, s, c, seq, a, (int)PH_COMBINE));
    } else {
        CCK(launch_pdl(allgather_cols_kernel, dim3(ctas), dim3(kCommThreads), 0, s, c, seq, a, (int)PH_ALL));
    }
}

// ---------------------------------------------------------------------------
// vocab-parallel greedy pick: every rank has (max, argmax) of its vocabulary
// slice per row; gather them and keep the first maximum (matrix.cpp:196-202)
// ---------------------------------------------------------------------------

__global__ void allgather_argmax_kernel(CommView c, uint64_t seq, int T, const float* val, const int* idx,
                                        int* tok_out, int phases) {
    pdl_wait();
    if (c.early_trigger) pdl_trigger();
    const int par = (int)(seq & 1);
    if (phases & PH_PUSH)
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const float v = val[t];
        const float ib = __int_as_float(idx[t]);
        for (int p = 0; p < c.world; ++p) {
            float* d = slot(c, c.peer_recv[p], par, c.loopback ? p : c.rank);
            d[2 * t] = v;
            d[2 * t + 1] = ib;
        }
    }
    if (phases & PH_SYNC) comm_signal_wait(c, seq, par);
    if (!(phases & PH_COMBINE)) return;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        float bv = -INFINITY;
        int bi = 0x7fffffff;
        for (int s = 0; s < c.world; ++s) {
            const float* d = slot(c, c.recv_local, par, s);
            const float v = __ldcg(d + 2 * t);
            const int i = __float_as_int(__ldcg(d + 2 * t + 1));
            if (v > bv || (v == bv && i < bi)) {
                bv = v;
                bi = i;
            }
        }
        tok_out[t] = bi;
    }
}

void launch_allgather_argmax(CommView& c, int T, const float* val, const int* idx, int* tok_out, cudaStream_t s) {
    if (T <= 0) return;
    if ((size_t)2 * T > c.slot_floats)
        dev_fail(DEV_ERR_COMM, "argmax all-gather: " + std::to_string(T) + " rows exceed the comm slot");
    const uint64_t seq = ++c.seq;
    if (getenv("ESPEC_TRACE_COMM")) fprintf(stderr, "[comm] rank %d argmax seq %llu\n", c.rank, (unsigned long long)seq);
    if (c.local_sync) {
        CCK(launch_pdl(allgather_argmax_kernel, dim3(1), dim3(128), 0, s, c, seq, T, val, idx, tok_out, (int)PH_PUSH));
        c.local_sync(c.local_ctx, c.rank, s);
        CCK(launch_pdl(allgather_argmax_kernel, dim3(1), dim3(128), 0, s, c, seq, T, val, idx, tok_out, (int)PH_COMBINE));
    } else {
        CCK(launch_pdl(allgather_argmax_kernel, dim3(1), dim3(128), 0, s, c, seq, T, val, idx, tok_out, (int)PH_ALL));
    }
}

}  // namespace espec_dev
