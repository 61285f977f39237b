// Host-side interface of the sm_100a kernels (launchers live in kernels.cu).
//
// Data layout in HBM:
//   * weights: every projection is stored K-major, W[K][ldw] row-major with
//     y = x · W (the reference's own matmul layout, proj/src/matrix.cpp:38-57);
//     ldw is padded to a multiple of 8 (fp32) / 32 (bf16, stored pre-packed
//     in the UMMA canonical K-major core-matrix layout, see pack_index). QKV of one layer is fused
//     column-wise [q | k | v]; gate/up are fused and interleaved per 32
//     columns [gate16 | up16] so one packed column group owns both halves of
//     its SiLU·up epilogue.
//   * hidden rows are fp32 [T][d]; their RMSNorm statistics travel as
//     per-32-column sum-of-squares partials stats[T][ceil(d/32)].
//   * KV cache: paged pool; page p holds kPage rows for every layer:
//     pool[p][layer][k|v][kv_head][row][d_head], located through a page table.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace espec_dev {

// Host-side failure of a launch wrapper: a rejected launch, a capacity guard
// or a collective that cannot run. Thrown (never printed and swallowed); the
// engine's C ABI maps `code` onto espec_status (7 CUDA, 8 collective).
enum : int { DEV_ERR_CUDA = 7, DEV_ERR_COMM = 8 };
struct DevError : std::runtime_error {
    int code;
    DevError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void dev_fail(int code, const std::string& msg);
// cudaError_t -> DevError(DEV_ERR_CUDA) with the call site.
void dev_check(cudaError_t e, const char* what, const char* file, int line);
#define DEV_CK(x) ::espec_dev::dev_check((x), #x, __FILE__, __LINE__)
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device context: set it
// once per (kernel, device). `mask` is the kernel's own bit set of devices.
// Thread-safe enough for the engine's use (one host thread per engine; a
// racing duplicate set is harmless).
void ensure_smem(const void* kernel, int bytes, unsigned long long& mask);

enum DType : int { DT_F32 = 0, DT_BF16 = 1 };

enum Epilogue : int {
    EPI_STORE = 0,   // out = x·W
    EPI_RESID = 1,   // out = resid + x·W ; writes row sum-of-squares partials
    EPI_SILU = 2,    // out = silu(gate) * up over interleaved gate/up tiles
    EPI_QKV = 3,     // RoPE(q), RoPE(k) ; q -> q buffer, k/v -> paged KV cache
    EPI_ARGMAX = 4,  // logits (optional store) + per-row argmax -> token ids
};

// Paged KV cache view.
struct KvView {
    void* pool = nullptr;
    const int* page_table = nullptr;  // logical block -> physical page
    int page_rows = 64;
    int n_layers = 0, n_kv = 0, dh = 0;
    int dtype = 0;                    // DType
    long long page_elems = 0;         // elements per page (all layers)
    int pool_pages = 0;               // pages in the pool (tensor-map extent)
    // 64-row pages per attention item (bf16 path). A function of the cache
    // capacity only — never of the pass — so every row's reduction tree is
    // the same in any pass (batch invariance).
    int attn_ppi = 1;
    int l2_hint = 0;  // attention page loads: 0 default, 1 evict-first, 2 evict-last L2 policy
};

// Per-pass row metadata (device pointers), indexed by pass row t.
struct PassView {
    int T = 0;                 // rows in the pass
    const int* rows = nullptr; // cache row of each input row
    const int* pos = nullptr;  // rotary position of each row
    const int* vis_end = nullptr;                 // rows [0, vis_end) visible
    const unsigned long long* anc = nullptr;      // tree rows visible: bit i -> row tree_base+i
    int tree_base = 0;
    int total = 0;             // rows stored in the cache during this pass
    // lowest cache row this pass writes (0 = unknown): K/V pages wholly below
    // it are final before the pass starts (attention may load them before
    // its dependency wait)
    int new_lo = 0;
};

constexpr int kMaxTp = 8;  // tensor-parallel group size limit

struct GemvProblem {
    const void* W = nullptr;
    int K = 0, N = 0, ldw = 0;
    const float* x = nullptr;
    int ldx = 0;
    // bf16 decode GEMV only: x holds bf16 activations (no RMSNorm prologue;
    // the producer already rounded them exactly as the staging would)
    int x_bf16 = 0;
    // fused RMSNorm prologue (gain == nullptr: none)
    const float* gain = nullptr;
    const float* stats_in = nullptr;
    int stat_tiles_in = 0;
    float eps = 1e-5f;
    // workspace
    float* partial = nullptr;     // [splits][16][tiles*256]
    unsigned* tickets = nullptr;  // [tiles] (+1 for argmax)
    // epilogue
    float* out = nullptr;
    int ldo = 0;
    int out_bf16 = 0;               // EPI_SILU, bf16 decode GEMV only: out holds bf16
    const float* resid = nullptr;   // RESID (and a fused STORE, bf16 decode GEMV only): out = resid + x.W
    int ldr = 0;
    const float* resid2 = nullptr;  // RESID, bf16 decode GEMV only: out = (resid + x.W) + resid2
    int ldr2 = 0;
    float* stats_out = nullptr;
    int stat_tiles_out = 0;
    // EPI_QKV
    int n_heads = 0, n_kv = 0, dh = 0, layer = 0;
    const float2* rope = nullptr;  // [position][dh/2] (cos, sin), see ModelDev::build_rope
    // EPI_ARGMAX
    int vocab = 0;
    float* logits = nullptr;  // [T][ld_logits] or nullptr
    int ld_logits = 0;
    float* am_val = nullptr;  // [T][tiles]
    int* am_idx = nullptr;
    int* tok_out = nullptr;   // [T]
    float* tok_val = nullptr; // [T] optional: the max itself (vocab-parallel gather)
    int col_base = 0;         // added to argmax indices (vocab-parallel slice offset)
    // prefill (tcgen05) workspace: packed bf16 A tiles and per-row 1/rms
    __nv_bfloat16* tc_xa = nullptr;
    float* tc_rms = nullptr;
    float* tc_part = nullptr;        // split-K partial tiles (nullptr: no split)
    unsigned* tc_tickets = nullptr;
    // EPI_STORE, bf16 decode GEMV: the tensor-parallel partial goes straight
    // into every rank's NVLink receive slot (push[p] = rank p's slot for this
    // rank and call, rows packed [t][N]) as each output tile finishes, instead
    // of to `out` — the all-reduce's push phase fused into the GEMV epilogue
    float* push[kMaxTp] = {};
    int push_n = 0;
};

constexpr int kMaxProblems = 8;
struct GemvBatch {
    GemvProblem p[kMaxProblems];
};

// Split planning depends only on (K, N): never on T or the group size, so a
// row's result is bit-identical whichever batch it is computed in (batch
// invariance).
struct GemvPlan {
    int tiles, splits, kc;
};
GemvPlan gemv_plan(int K, int N);                     // fp32 parity path
size_t gemv_partial_floats(int K, int N, int wdtype);  // workspace floats one problem needs
int gemv_col_tiles(int K, int N, int wdtype);          // argmax partials per row

// bf16 stream-K GEMV (gemv_stream.cu): units (problem, k-chunk, 32-column
// group) of kcb 1 KB blocks, contiguous balanced ranges over <= 148 CTAs.
struct SgPlan {
    int KT, kcb, nK, ngroups, units, grid;
};
SgPlan sgemv_plan(int K, int ldw, int nprob);
size_t sgemv_partial_floats(int K, int ldw);
// Tail-pool claim counters of one stream (engine): banks rotate per launch
// PASS (16-row slice), so two in-flight passes never share counters even when
// PDL lets a pass's producer claim before its predecessor finished.
struct SgPool {
    unsigned* dev = nullptr;  // [sgemv_pool_words()], zeroed by sgemv_pool_reset
    unsigned next = 0;        // next bank (host)
};
size_t sgemv_pool_words();
void sgemv_pool_reset(SgPool& p, cudaStream_t s);
// pool == nullptr: a process-wide bank set (single-stream microbenchmarks only)
void launch_sgemv(int epi, const GemvBatch& b, int nprob, int T, const PassView& pass, const KvView& kv,
                  cudaStream_t s, SgPool* pool = nullptr);
// Thread-local: while on, launch_sgemv may pick a T-dependent "wide" plan
// (whole-K units, activation slots of T rows). Rows then depend on the pass
// size, so the engine enables it for the DRAFTER only: drafter numerics only
// steer which tokens are proposed, while the base keeps the (K, N)-only plan
// that makes greedy verification lossless (batch invariance).
void set_sgemv_wide(bool on);
// Prompt prefill (tc_gemm.cu): while prefill mode is on (thread-local, set by
// the engine around prompt chunks), bf16 launch_gemv calls with more than 16
// rows run on tcgen05 (M=128 x N=256 tiles, TMEM accumulators) instead of the
// decode GEMV. Decode passes never use it, so their batch invariance holds.
void set_prefill_mode(bool on);
size_t tc_xa_elems(int rows, int K);
size_t tc_part_floats(int K, int ldw);
void launch_tc_gemm(int epi, const GemvProblem& P, int T, const PassView& pass, const KvView& kv,
                    __nv_bfloat16* xa, float* inv_rms, cudaStream_t s);
// Programmatic dependent launch on/off (default on; ESPEC_PDL=0 disables).
void set_pdl(bool on);
bool pdl_enabled();

// Rows handled per GEMV launch (bf16 mma path: 16; fp32 FMA path: 8).
int gemv_rows_per_launch(int wdtype);
// bf16 GEMV weights are stored pre-packed in the UMMA canonical K-major layout (kernels.cu
// pack_index); K x ldw logical <-> packed, ldw a multiple of 32.
size_t packed_elems(int K, int ldw);
void launch_pack(const void* logical, int K, int ldw, void* packed, bool unpack, cudaStream_t s);

// y = epilogue(norm?(x) · W) for T rows, over nprob same-shape problems.
// true when launch_gemv(wdtype, T) runs the bf16 decode GEMV (the kernel with
// the fused TP push epilogue), i.e. not the fp32 GEMV or the tcgen05 prefill
bool gemv_fused_push_ok(int wdtype, int T);
void launch_gemv(int epi, int wdtype, const GemvBatch& b, int nprob, int T, const PassView& pass,
                 const KvView& kv, cudaStream_t s, SgPool* pool = nullptr);

// h[t] = embedding[tok[t]] (fp32), + stats.
void launch_embed(int wdtype, const void* emb, int d, const int* tok_arena, const int* tok_idx, int T,
                  float* h, float* stats, cudaStream_t s);
// h += a (T x d), + stats.
void launch_add_stats(float* h, const float* a, int d, int T, float* stats, cudaStream_t s);

struct AttnProblem {
    const float* q = nullptr;   // [T][H*dh]
    float* out = nullptr;       // [T][H*dh] (fp32, or bf16 when out_bf16)
    int out_bf16 = 0;           // bf16 item path only
    int layer = 0;
    float* ws = nullptr;        // split partials
    unsigned* tickets = nullptr;
};
struct AttnBatch {
    AttnProblem p[kMaxProblems];
};
size_t attn_ws_floats(int T, int n_heads, int dh, int max_rows);
// 64-row pages per bf16 attention item for a cache of `capacity_rows`
// (ESPEC_ATTN_PPI overrides); see KvView::attn_ppi
int attn_pages_per_item(int capacity_rows);
size_t attn_tickets(int T, int n_heads, int n_kv);
void launch_attention(const AttnBatch& b, int nprob, int n_heads, const PassView& pass, const KvView& kv,
                      cudaStream_t s);
// bf16 paged KV, 64-row pages, d_head 64 / 128: the tcgen05 kernel (attn_tc.cu)
void launch_attention_tc(const AttnBatch& b, int nprob, int n_heads, const PassView& pass, const KvView& kv,
                         cudaStream_t s);
// kernels one launch_attention call issues (the tcgen05 path adds a combine
// kernel when the context spans more than one chunk)
int attn_tc_cluster(int chunks, int T);  // 1: chunks combine inside a cluster, 2: last chunk CTA combines (attn_tc.cu)
int attention_launches(const PassView& pass, const KvView& kv, int n_heads, int nprob);
int attn_tc_ppi(const PassView& pass, const KvView& kv, int n_heads, int nprob);  // pages per chunk CTA of one launch

// Copy cache rows src[i] -> dst[i] for every layer (commit_path compaction).
void launch_kv_move(const KvView& kv, const int* src, const int* dst, int n, cudaStream_t s);

// Greedy acceptance over a drafted tree (see kernels.cu for the walk).
struct AcceptArgs {
    int n_nodes = 0, n_levels = 0, root_children = 0;
    const int* node_parent = nullptr;    // [n_nodes]
    const int* node_first_child = nullptr;
    const int* node_n_children = nullptr;
    const int* node_tok_idx = nullptr;   // index into tok arena
    const int* tok_arena = nullptr;
    const int* base_argmax = nullptr;    // [1 + n_nodes] base argmax for frontier + each node
    int* outcome = nullptr;              // [2 + 2*n_levels]: m, bonus, path[n_levels], tokens[n_levels]
    int* tok_arena_w = nullptr;          // accepted tokens + bonus are appended at commit_at
    int commit_at = 0;
    // 1: the reference's rule (proj/src/verifier.cpp:146-158) — at T = 0 the
    // draft distribution is one-hot at the first sibling, so rejecting it
    // with more siblings left raises CheckError (err = 4); 0: accept the
    // sibling equal to the base argmax (identical whenever the reference
    // does not throw)
    int strict_siblings = 0;
    int* err = nullptr;
};
void launch_accept_greedy(const AcceptArgs& a, cudaStream_t s);

// ---- T > 0 sampling and multi-sibling tree levels (sample.cu) ----
constexpr int kMaxWidth = 16;  // children per drafted node

// dists[dst_row[r]] = softmax_temp(logits[src_row[r]], temperature)
// (one-hot at the first argmax when temperature == 0).
struct SoftmaxArgs {
    const float* logits = nullptr;
    int ld_logits = 0;
    const int* src_row = nullptr;
    float* dists = nullptr;
    int ld_dists = 0;
    const int* dst_row = nullptr;
    int vocab = 0;
    float temperature = 0.f;
    int* err = nullptr;  // set to 1 on a non-finite logit (DomainError)
};
void launch_softmax_rows(const SoftmaxArgs& a, int rows, cudaStream_t s);

// select_children for `rows` frontier rows in order: T = 0 top-k of the
// logits row; T > 0 `width` draws without replacement from the dists row,
// consuming uniforms at *cursor. Children go to tok_arena[child_at[r] + i].
struct SelectArgs {
    int rows = 0, vocab = 0;
    float temperature = 0.f;
    const float* logits = nullptr;
    int ld_logits = 0;
    const int* logit_row = nullptr;
    const float* dists = nullptr;
    int ld_dists = 0;
    const int* dist_row = nullptr;
    const int* width = nullptr;
    const int* child_at = nullptr;
    int* tok_arena = nullptr;
    const double* uniforms = nullptr;
    int* cursor = nullptr;
    int* err = nullptr;  // 2: draft distribution exhausted before the width
};
void launch_select_children(const SelectArgs& a, cudaStream_t s);

// verify_tree at T > 0 over the drafted tree (n_levels = 0: vanilla
// sampling). base_dists rows: frontier, then one per node; draft_dists
// indexed by node_prob_index. Writes outcome = {m, bonus, path[n_levels],
// tokens[n_levels]} and appends accepted tokens + bonus to tok_arena_w.
struct VerifyArgs {
    int vocab = 0, n_levels = 0, root_children = 0;
    const int* node_first_child = nullptr;
    const int* node_n_children = nullptr;
    const int* node_tok_idx = nullptr;
    const int* node_prob_index = nullptr;
    const int* tok_arena = nullptr;
    const float* base_dists = nullptr;
    const float* draft_dists = nullptr;
    int ld_dists = 0;
    float* target = nullptr;  // [vocab] scratch
    const double* uniforms = nullptr;
    int* cursor = nullptr;
    int* outcome = nullptr;
    int* tok_arena_w = nullptr;
    int commit_at = 0;
    int* err = nullptr;  // 3..5: CheckError conditions of verify_tree / sample_from
};
void launch_verify_sample(const VerifyArgs& a, cudaStream_t s);

// ---- tensor-parallel collectives over NVLink peer memory (comm.cu) ----
constexpr int kCommErrTimeout = 6;  // engine error-slot code (see EngineImpl::sync_outcome)
struct CommView {
    int rank = 0, world = 1;
    size_t slot_floats = 0;          // floats per (parity, sender) slot
    float* recv_local = nullptr;     // this rank's [2][world][slot_floats]
    uint64_t* flags_local = nullptr; // this rank's [2][world]
    float* peer_recv[kMaxTp] = {};   // every rank's recv region (self included)
    uint64_t* peer_flags[kMaxTp] = {};
    unsigned* ticket = nullptr;      // local: last-CTA election
    int* err = nullptr;              // engine error slot: kCommErrTimeout when a peer never arrives
    uint64_t seq = 0;                // collectives issued so far (host side)
    int early_trigger = 1;           // PDL-trigger the successor before waiting (GPUs not shared)
    int debug = 0;                   // ESPEC_TRACE_COMM: device-side trace
    // shard proxy (one engine standing in for all `world` ranks on one GPU):
    // every push lands in all sender slots of this rank's own region and every
    // flag is set locally, so each collective moves and waits like a TP-N one
    // (its sums are world x this rank's partial: timing, not numerics)
    int loopback = 0;
    // Shards sharing ONE GPU (single-device harness): device-side spinning
    // could wait on a peer whose copies queue behind this rank's work, so the
    // push and combine run as two kernels and local_sync orders them with
    // CUDA events across the shards' streams instead (host barrier + event
    // waits). nullptr between GPUs.
    void (*local_sync)(void* ctx, int rank, cudaStream_t s) = nullptr;
    void* local_ctx = nullptr;
};
enum AllreduceMode : int { AR_STORE = 0, AR_RESID = 1 };
struct AllreduceArgs {
    int rows = 0, d = 0;
    const float* src = nullptr;  // this rank's partial [rows][ld_src]
    int ld_src = 0;
    int mode = AR_STORE;
    float* out = nullptr;
    int ldo = 0;
    const float* resid = nullptr;  // AR_RESID: out = resid + sum, + row stats
    int ldr = 0;
    float* stats = nullptr;
    int stat_tiles = 0;
    // src / out rows come in blocks: row r at (r / rows_per_block) * block_stride
    // + (r % rows_per_block) * ld (0 = one block)
    int rows_per_block = 0;
    size_t block_stride = 0;
    // blocks (bit b = rows [b * rows_per_block, (b + 1) * rows_per_block)) this
    // rank contributes as exact zeros without reading src: the layer-parallel
    // placement's exchange, where only a slot's owner computed it
    unsigned zero_blocks = 0;
    // every rank's slot was already filled by the producing GEMV's epilogue
    // (GemvProblem::push): only signal, wait and combine
    int prepushed = 0;
};
void launch_allreduce_rows(CommView& c, const AllreduceArgs& a, cudaStream_t s);
struct GatherColsArgs {
    int rows = 0, cols = 0;  // each rank's slice: rows x cols
    const float* src = nullptr;
    int ld_src = 0;
    float* dst = nullptr;    // rows x (world*cols)
    int ld_dst = 0;
};
void launch_allgather_cols(CommView& c, const GatherColsArgs& a, cudaStream_t s);
// rank p's receive slot that this rank fills for the next collective call
float* comm_push_slot(const CommView& c, int p);
// vocab-parallel argmax: (val, idx) per row from every rank -> first maximum
void launch_allgather_argmax(CommView& c, int T, const float* val, const int* idx, int* tok_out, cudaStream_t s);

// Deterministic N(0, sd) init from a counter hash (perf-mode weights).
void launch_fill_normal(int dtype, void* dst, long long n, float sd, uint64_t seed, cudaStream_t s);
void launch_fill_const(int dtype, void* dst, long long n, float v, cudaStream_t s);
// Local column -> global column map of a sharded fill: up to 3 contiguous
// segments, or the packed gate/up interleave of f_loc columns starting at
// global column f_base (gate drawn with seed, up with seed2).
struct ColMap {
    int nseg = 0;
    int lc0[3] = {0, 0, 0}, gc0[3] = {0, 0, 0}, len[3] = {0, 0, 0};
    int gateup = 0, f_loc = 0, f_base = 0;
    uint64_t seed = 0, seed2 = 0;
};
void launch_fill_normal_map(int dtype, void* dst, int K, int ld, const ColMap& m, int row_off, long long n_full,
                            float sd, cudaStream_t s);
// dst[c][r] = src[r][c]  (src: rows x cols, dst leading dimension ldd)
void launch_transpose(int dtype, const void* src, int rows, int cols, void* dst, int ldd, cudaStream_t s);

}  // namespace espec_dev
