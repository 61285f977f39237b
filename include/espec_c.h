/*
 * espec_c.h — C ABI of the B200 EasySpec decode engine (libespec_b200.so).
 *
 * The reference (/root/reference/proj) is a C++20 static library with no
 * FFI; its entry points are C++ functions over espec:: types. This header is
 * the drop-in boundary that replaces them, one entry point per reference
 * interface (cited below). Plain pointers and sizes only; nothing crosses
 * the boundary as an exception: every call returns an espec_status and
 * espec_last_error() carries the message (the reference's exception taxonomy,
 * proj/include/espec/errors.hpp:11-44, maps onto the status codes).
 *
 * Threading: one engine = one in-flight generation; calls on one engine must
 * be serialised (the reference's Generation is likewise single-threaded,
 * proj/src/orchestrator.cpp:138-484). Independent engines may run on
 * different threads.
 */
#ifndef ESPEC_C_H
#define ESPEC_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ESPEC_OK = 0,
    ESPEC_CONFIG = 1,    /* ConfigError    (CLI exit code 1) */
    ESPEC_IO = 2,        /* IoError        (CLI exit code 2) */
    ESPEC_CHECK = 3,     /* CheckError     (CLI exit code 3) */
    ESPEC_SHAPE = 4,     /* ShapeError */
    ESPEC_STRUCTURE = 5, /* StructureError */
    ESPEC_DOMAIN = 6,    /* DomainError */
    ESPEC_CUDA = 7,      /* device / runtime failure (no reference analogue) */
    ESPEC_NCCL = 8
} espec_status;

typedef enum { ESPEC_F32 = 0, ESPEC_BF16 = 1 } espec_dtype;
typedef enum { ESPEC_VANILLA = 0, ESPEC_SD = 1, ESPEC_SD_TREE = 2, ESPEC_EASYSPEC = 3 } espec_algorithm;

/* espec::ModelConfig (proj/include/espec/model.hpp:19-33), extended with the
 * fields real checkpoints need (GQA, rope base, untied head, storage dtypes).
 * n_kv_heads == n_heads, rope_theta 10000, tied_head 1, f32/f32 reproduces
 * the reference model exactly. */
typedef struct {
    int vocab_size;
    int d_model;
    int n_layers;
    int n_heads;
    int n_kv_heads;
    int d_head;
    int d_mlp;
    int max_positions;
    float norm_eps;
    float rope_theta;
    int tied_head;
    int weight_dtype; /* espec_dtype */
    int kv_dtype;     /* espec_dtype */
    uint64_t seed;
} espec_model_cfg;

/* espec::RunConfig (proj/include/espec/orchestrator.hpp:23-38). widths may be
 * NULL (all ones); plan_override may be NULL or "" (plan_groups(L, lp_size)). */
typedef struct {
    int algorithm; /* espec_algorithm */
    int n;
    const int* widths;
    int lp_size;
    const char* plan_override;
    float temperature;
    int max_new_tokens;
    uint64_t seed;
    int calibration;
    /* 1 reproduces the reference's CheckError when a greedy (T = 0) tree's
     * first sibling is rejected with siblings left (verifier.cpp:146-158:
     * the one-hot draft mass is exhausted); 0 (default) accepts the sibling
     * equal to the base argmax instead — identical outputs whenever the
     * reference does not throw. */
    int strict_greedy_tree;
} espec_run_cfg;

/* Devices used by one engine. One engine drives one GPU; a tensor-parallel
 * group of tp_size engines (one per GPU, usually one per process) shards the
 * base Megatron-style and exchanges partial sums over NVLink
 * peer memory. The drafter either follows the same tensor-parallel split
 * (n_lp_devices 0 or 1: every GPU runs a head slice of every layer of a fuzzy
 * group), or takes the paper's layer-parallel placement (n_lp_devices ==
 * tp_size, lp_devices = {0, 1, ..., tp_size - 1}): group slot j runs on rank
 * j with full heads and owns that layer's draft KV, one exchange per group
 * delivers the slots' attention outputs to every rank, and the MLPs / LM head
 * stay tensor-parallel (draft_engine.cpp:89-130, cost_sim.cpp:127-143). */
typedef struct {
    int device;
    int n_lp_devices;
    const int* lp_devices;
    int tp_size;
    int tp_rank;
} espec_device_map;

/* espec::IterationTrace (proj/include/espec/report.hpp:12-28): the *_ms
 * fields are measured device stage times (the reference's *_wall), the *_sim
 * fields the cost model's units (espec_set_cost; orchestrator.cpp:263-386). */
typedef struct {
    int m, n, drafted_nodes, emitted;
    int sequential_forwards, fuzzy_forwards, base_forwards;
    int committed, draft_committed, base_committed;
    int bonus;
    float calibrate_ms, draft_ms, verify_ms;
    double calibrate_sim, draft_sim, verify_sim;
} espec_iteration;

typedef struct espec_engine espec_engine;

/* Generation(...) constructor state: caches, plan and RNG
 * (proj/src/orchestrator.cpp:138-160). Validates both model configs and the
 * run config (ModelConfig::validate proj/src/model.cpp:12-24,
 * validate_run_config proj/src/orchestrator.cpp:95-118). Unlike the
 * reference (proj/src/orchestrator.cpp:114-117) base and drafter may differ
 * in width; they must share the vocabulary. */
espec_status espec_engine_create(const espec_model_cfg* base, const espec_model_cfg* draft,
                                 const espec_run_cfg* run, const espec_device_map* devices,
                                 espec_engine** out);
void espec_engine_destroy(espec_engine* eng);

/* Tensor-parallel wiring (tp_size > 1), before the first forward pass.
 * One process holding all shards: espec_comm_link(engines in rank order).
 * One process per GPU: every rank exports its 64-byte cudaIpcMemHandle_t,
 * the caller all-gathers them (e.g. torch.distributed) and every rank
 * imports the world * 64 bytes in rank order. */
espec_status espec_comm_link(espec_engine** engines, int world);
espec_status espec_comm_export(espec_engine* eng, void* handle64);
/* Shard proxy (measurement only): a tp_size = N engine of rank 0 stands in for
 * the whole group on one GPU — every collective pushes into all N slots of its
 * own receive region — so a single GPU exposes the per-GPU step time of a TP-N
 * deployment (its shard shapes and N-slot collectives). Outputs are not the
 * model's (each sum is N x this shard's partial). */
espec_status espec_comm_loopback(espec_engine* eng);
espec_status espec_comm_import(espec_engine* eng, const void* handles, int world);
const char* espec_last_error(const espec_engine* eng);
/* Error text for a failed espec_engine_create (no engine exists yet). */
const char* espec_create_error(void);

/* init_model(config) (proj/src/model.cpp:38-84). which: 0 drafter, 1 base.
 * parity_mode 1 replays the reference's xoshiro256** stream on the host
 * (bit-identical fp32 weights); 0 draws the same N(0, sd) rules on device
 * (perf mode, any dtype/shape). */
espec_status espec_init_weights_seeded(espec_engine* eng, int which, uint64_t seed, int parity_mode);

/* make_truncated_draft(base, keep) (proj/src/model.cpp:86-99): the drafter
 * aliases the base's first draft->n_layers blocks, embedding and final norm. */
espec_status espec_share_truncated_draft(espec_engine* eng);

/* Load one fp32 host tensor in the reference layout (load_model's manifest,
 * proj/src/model_io.cpp:27-45): "embedding" VxD, "head" DxV (untied),
 * "final_norm_gain" 1xD, per layer "wq" Dx(H*dh), "wk"/"wv" Dx(Hkv*dh),
 * "wo" (H*dh)xD, "w_gate"/"w_up" DxF, "w_down" FxD, "attn_norm_gain",
 * "mlp_norm_gain" 1xD. */
espec_status espec_load_tensor(espec_engine* eng, int which, const char* name, int layer, const float* data,
                               int64_t rows, int64_t cols);
/* Read a tensor back in the same layout (fp32). */
espec_status espec_read_tensor(espec_engine* eng, int which, const char* name, int layer, float* out, int64_t rows,
                               int64_t cols);

/* Replace the run config between generations (RunConfig validation). */
espec_status espec_set_run(espec_engine* eng, const espec_run_cfg* run);

/* generate(base, draft, config, prompt) (proj/src/orchestrator.cpp:488-492):
 * prompt bytes -> BOS + bytes (tokenize_prompt, proj/src/orchestrator.cpp:42-52),
 * run to max_new_tokens. out_tokens needs max_new_tokens entries; traces
 * (optional) needs max_new_tokens entries; *n_iters receives the count. */
espec_status espec_generate(espec_engine* eng, const uint8_t* prompt, int prompt_len, int32_t* out_tokens,
                            int* n_out, espec_iteration* traces, int* n_iters);

/* Stage-level API (Generation::run's loop, proj/src/orchestrator.cpp:163-195):
 * begin() takes already-tokenized input; step() runs one iteration —
 * run_iteration_speculative (calibrate -> draft -> verify -> resolve,
 * proj/src/orchestrator.cpp:407-436) or run_iteration_vanilla (438-468) —
 * and returns the tokens it emitted (<= n+1). */
espec_status espec_begin(espec_engine* eng, const int32_t* tokens, int n_tokens);
espec_status espec_step(espec_engine* eng, int32_t* emitted, int* n_emitted, espec_iteration* trace);
int espec_done(const espec_engine* eng);

/* ---- Stage-level API: one speculative iteration driven stage by stage, the
 * split of Generation::run_iteration_speculative (orchestrator.cpp:407-436)
 * into the reference's stages. Order per iteration: calibrate -> draft ->
 * verify -> resolve_draft_cache -> commit_outcome (espec_step runs the same
 * five in one call). Out-of-order calls return ESPEC_STRUCTURE. */
#define ESPEC_MAX_NODES 64

/* espec::DraftTree (draft_engine.hpp:63-84): nodes level by level, siblings
 * contiguous in selection order; parent -1 = child of the committed context;
 * prob_index indexes the draft distributions; cache_row = drafter-cache flat
 * row (-1 for the never-forwarded last level). */
typedef struct {
    uint64_t id; /* iteration the tree belongs to */
    int n_nodes, root_children, n_levels, n_dists;
    int32_t widths[ESPEC_MAX_NODES];
    int32_t token[ESPEC_MAX_NODES], parent[ESPEC_MAX_NODES], depth[ESPEC_MAX_NODES];
    int32_t prob_index[ESPEC_MAX_NODES], cache_row[ESPEC_MAX_NODES];
    int32_t first_child[ESPEC_MAX_NODES], n_children[ESPEC_MAX_NODES];
    /* optional: caller buffer of dist_capacity x vocab floats that receives
     * DraftTree::dists (softmax_temp rows; one-hot at T = 0) */
    float* dists;
    int dist_capacity;
} espec_tree;

/* espec::VerificationOutcome (verifier.hpp:14-21). */
typedef struct {
    uint64_t id;
    int m, n;
    int32_t bonus;
    int32_t accepted_path[ESPEC_MAX_NODES];
    int32_t accepted_tokens[ESPEC_MAX_NODES];
} espec_outcome;

/* Start a generation over token ids and prefill both caches with what the
 * first iteration would (base: every prompt row but the frontier token;
 * drafter: the prompt's whole 256-row chunks). */
espec_status espec_prefill(espec_engine* eng, const int32_t* tokens, int n_tokens);
/* drafter_leading_pass (orchestrator.cpp:256-300): the uncached committed
 * suffix through one precise drafter pass (the bonus calibration that
 * rewrites the draft KV; fuzzy in the no-calibration arm). root_logits
 * (optional, vocab floats) receives the drafter logits of the last row. */
espec_status espec_calibrate(espec_engine* eng, float* root_logits);
/* draft_stage -> draft_tree (orchestrator.cpp:302-331, draft_engine.cpp:188-289):
 * the fuzzy layer-parallel passes. tree (optional) receives the DraftTree. */
espec_status espec_draft(espec_engine* eng, espec_tree* tree);
/* verify_stage + verify_tree (orchestrator.cpp:333-388, verifier.cpp:86-177):
 * one base pass over [frontier + tree], acceptance, base-cache commit. tree
 * NULL verifies the tree as drafted; otherwise it must be this iteration's
 * tree (same id and shape) and its tokens replace the drafted ones. */
espec_status espec_verify(espec_engine* eng, const espec_tree* tree, espec_outcome* outcome);
/* resolve_draft_cache (orchestrator.cpp:390-405): discard the fuzzy rows
 * (calibrated EasySpec) or commit the accepted path's staged rows. outcome
 * NULL = this iteration's; otherwise it must match it. */
espec_status espec_resolve_draft_cache(espec_engine* eng, const espec_outcome* outcome);
/* run_iteration_speculative's tail (orchestrator.cpp:414-428): commit the
 * accepted tokens + bonus, emit min(m + 1, remaining) into emitted. */
espec_status espec_commit_outcome(espec_engine* eng, int32_t* emitted, int* n_emitted, espec_iteration* trace);

/* IterationHook view (proj/include/espec/orchestrator.hpp:46-55): committed
 * token count and K/V rows [row0, row0+n) of one layer of the drafter (0) or
 * base (1) cache, n x (n_kv_heads*d_head) fp32 each. */
espec_status espec_cache_view(espec_engine* eng, int which, int layer, int row0, int n, float* k, float* v,
                              int* committed_len);
espec_status espec_committed(espec_engine* eng, int32_t* tokens, int cap, int* n);

/* Parity probe: one chain pass over `tokens` on a freshly reset cache of one
 * model (forward_sequential, or forward_fuzzy when plan is "lp=N" or a plan
 * string; proj/src/draft_engine.cpp:35-133) -> logits n x V and final hidden
 * n x D (either may be NULL). Ends any generation in progress. */
espec_status espec_forward(espec_engine* eng, int which, const int32_t* tokens, int n, const char* plan,
                           float* logits, float* hidden);

/* Parity probe at decode shapes: prefill `prompt` on a fresh cache of one
 * model, then ONE decode-sized pass over n <= 64 rows forming a tree
 * (parents[j] = -1: child of the prompt tail, else an earlier row j' < j) —
 * the verify_stage / draft_tree pass (orchestrator.cpp:333-388,
 * draft_engine.cpp:235-287) with its tree mask. logits n x V, hidden n x D
 * (either may be NULL). Ends any generation in progress. */
espec_status espec_forward_tree(espec_engine* eng, int which, const int32_t* prompt, int n_prompt,
                                const int32_t* tokens, const int32_t* parents, int n, const char* plan, float* logits,
                                float* hidden);

/* prefix_distribution (proj/src/orchestrator.cpp:494-526): independent
 * generations of the run config's max_new_tokens tokens over `tokens`, run r
 * seeded SplitMix64(seed + 0x9E37 (r + 1)).next() as in the reference, for
 * r = first_run, first_run + run_stride, ... < runs (one host thread's share of
 * the reference's loop; 0 / 1 = all runs). Writes the distinct emitted
 * prefixes in lexicographic order (cap x max_new_tokens int32) and their
 * counts; *n_distinct = how many. */
espec_status espec_prefix_distribution(espec_engine* eng, const int32_t* tokens, int n_tokens, int64_t runs,
                                       int64_t first_run, int64_t run_stride, int32_t* prefixes, int64_t* counts,
                                       int cap, int* n_distinct);
/* total_variation (orchestrator.cpp:528-553) of two prefix distributions
 * (lexicographically sorted, prefixes of `len` tokens); -1 on bad counts. */
double espec_total_variation(const int32_t* pa, const int64_t* ca, int na, const int32_t* pb, const int64_t* cb,
                             int nb, int len, int64_t runs_a, int64_t runs_b);

/* Layer plans (proj/src/layer_plan.cpp:54-128) -> formatted plan string. */
espec_status espec_plan_groups(int n_layers, int lp_size, char* out, int out_len);
espec_status espec_parse_plan(const char* spec, char* out, int out_len);

/* ---- Host-side analysis API ------------------------
 * Calls without an engine report their error text through
 * espec_create_error(). */

/* RunReport's derived metrics (proj/include/espec/report.hpp:40-57) from the
 * engine's iteration traces; stage times are the measured device times. */
typedef struct {
    int n_iterations;
    int has_alpha;             /* vanilla drafts nothing */
    double alpha;              /* sum m / sum n (report.cpp:77-78) */
    int64_t tokens_emitted;
    double mean_accept_len;    /* emitted / iterations */
    double tokens_per_s;       /* emitted / device seconds of the three stages */
    double draft_per_100_s;    /* stage seconds per 100 emitted tokens (report.cpp:80-84) */
    double verify_per_100_s;
    double calibrate_per_100_s;
    double draft_total_per_100_s; /* draft + calibrate (report.cpp:85) */
    double total_s;
    double speedup_vs_vanilla; /* vanilla_baseline_sim / total_sim (report.cpp:87-90), 1 if total_sim is 0 */
    /* the same in the cost model's units (report.cpp:83-87) */
    double draft_per_100_sim, verify_per_100_sim, calibrate_per_100_sim, draft_total_per_100_sim;
    double total_sim;
} espec_report;

/* aggregate(traces, vanilla_baseline_sim) (proj/src/report.cpp:51-95):
 * ESPEC_CONFIG "cannot aggregate an empty trace list" / "traces emitted zero
 * tokens" as the reference throws. vanilla_baseline_sim: the cost model's
 * vanilla generation of the same tokens (espec_cost_eval
 * ESPEC_COST_VANILLA_BASELINE, orchestrator.cpp:72-77). */
espec_status espec_aggregate(const espec_iteration* traces, int n_traces, double vanilla_baseline_sim,
                             espec_report* out);
/* emit_report (report.cpp:97-171): format 0 = JSON (the reference's keys;
 * "sim" in cost-model units, "wall" in measured device seconds; "config" is
 * left empty), 1 = CSV header + row (the sim numbers, as the reference).
 * *len receives the text length; ESPEC_SHAPE if it does not fit in cap bytes
 * (NUL included). */
espec_status espec_report_emit(const espec_report* report, const espec_iteration* traces, int n_traces,
                               const char* algorithm, int n, const int* widths, int n_widths, int lp_size,
                               int format, char* out, int cap, int* len);

/* Cost simulator (proj/include/espec/cost_sim.hpp, proj/src/cost_sim.cpp):
 * the affine device-cost model c_fixed + c_mem (w / tp) + c_comp (w / tp) s
 * (+ t_addi when tp > 1) behind the reports' simulated stage units. Doubles in
 * the reference's order: every number matches the reference bit for bit. */
typedef struct {
    double c_fixed, c_mem, c_comp, t_addi;
    double attn_workload, mlp_workload, base_layer_workload;
    int tp_size_base, tp_size_draft, devices;
} espec_cost_params;
espec_status espec_cost_defaults(espec_cost_params* out); /* CostParams{} */
typedef enum {
    ESPEC_COST_VALIDATE = 0,         /* CostParams::validate; out = 0 */
    ESPEC_COST_T_EXE = 1,            /* t_exe(p, workload a, s b, tp n_layers) */
    ESPEC_COST_GROUP_ATTENTION = 2,  /* group_attention_time(p, group size n_layers, s a) */
    ESPEC_COST_DRAFT_GROUP = 3,      /* simulate_draft_group(p, plan, s a); plan in the reference's grammar */
    ESPEC_COST_SEQUENTIAL_DRAFT = 4, /* sequential_draft_forward_time(p, n_layers, s a) */
    ESPEC_COST_BASE_FORWARD = 5,     /* base_forward_time(p, n_layers, s a) */
    ESPEC_COST_VANILLA_BASELINE = 6  /* vanilla_baseline_sim(p, n_layers, prompt_len a, tokens b) */
} espec_cost_fn;
/* ESPEC_CONFIG with the reference's ConfigError texts on invalid input. */
espec_status espec_cost_eval(const espec_cost_params* params, int what, double a, double b, int n_layers,
                             const char* plan, double* out);
/* total_time_model: ESPEC_DOMAIN at alpha <= 0, ESPEC_CONFIG outside (0, 1] or n < 1. */
espec_status espec_cost_total_time(double n_tokens, double t_draft, double t_base, int n, double alpha, double* out);
/* RunConfig::cost of an engine (validated; default CostParams{}); the stages
 * advance a SimClock per generation (reset by begin / prefill / generate)
 * exactly as Generation does, so traces carry the reference's *_sim values. */
espec_status espec_set_cost(espec_engine* eng, const espec_cost_params* params);
/* GenerateResult::occupancy_csv of the current generation (cost_sim.cpp:102-117). */
espec_status espec_occupancy_csv(espec_engine* eng, char* out, int cap, int* len);

/* ESPEC1 model file (proj/include/espec/model_io.hpp, proj/src/model_io.cpp):
 * "ESPEC1\n", u64 header length, JSON header (config + tensor manifest), raw
 * little-endian fp32 tensors. espec_model_file_config parses and validates a
 * file (every check of load_model, with its IoError texts as ESPEC_IO) and
 * returns its config (MHA, tied head, fp32). */
espec_status espec_model_file_config(const char* path, espec_model_cfg* cfg);
/* load_model into model `which` (0 drafter, 1 base) of an engine whose config
 * matches the file's; save_model of model `which` (reference-representable
 * models: MHA, tied head, rope base 10000). */
espec_status espec_load_model_file(espec_engine* eng, int which, const char* path);
espec_status espec_save_model_file(espec_engine* eng, int which, const char* path);

/* probe_similarity (proj/src/draft_engine.cpp:291-357) on the drafter: for
 * each lp size, one fuzzy and one precise pass over every corpus sequence
 * (token ids; sequence s = tokens[offsets[s] .. offsets[s+1])) on fresh
 * caches, mean cosine similarity (double, matrix.cpp:139-157) of h_in, q, k,
 * v and the attention output over every parallelized layer and row. Ends any
 * generation in progress. */
typedef struct {
    int lp_size;
    double h, q, k, v, attn_out;
} espec_similarity_row;
espec_status espec_probe_similarity(espec_engine* eng, const int* lp_sizes, int n_lp, const int32_t* tokens,
                                    const int* offsets, int n_seqs, espec_similarity_row* rows);

/* generate() over already-tokenized input (the same loop as espec_generate
 * without the byte tokenizer; vocabularies larger than 258). */
espec_status espec_generate_tokens(espec_engine* eng, const int32_t* tokens, int n_tokens, int32_t* out_tokens,
                                   int* n_out, espec_iteration* traces, int* n_iters);

/* The cudaStream_t every kernel of this engine is launched on. */
void* espec_stream(espec_engine* eng);

/* Per-launch CUDA-event timing of one kernel site while enabled: which 0/1
 * (drafter/base, <0 disables), kind 0 QKV GEMV, 1 attention, 2 O GEMV,
 * 3 gate/up GEMV, 4 down GEMV, 5 head GEMV. Stats: launches timed, their total
 * device ms and algorithmic bytes per launch. */
espec_status espec_time_site(espec_engine* eng, int which, int kind);
espec_status espec_site_stats(espec_engine* eng, int* count, double* total_ms, double* bytes_per_launch);
/* Host<->device bytes copied so far (metadata, tokens, outcomes). */
espec_status espec_io_bytes(espec_engine* eng, int64_t* h2d, int64_t* d2h);

/* Instrumentation: kernel launches issued since the last reset. */
int espec_kernel_launches(const espec_engine* eng);
void espec_reset_kernel_launches(espec_engine* eng);
espec_status espec_sync(espec_engine* eng);

/* Instrumentation: time one bf16 decode GEMV shape (K x N, T rows, nprob
 * batched problems, epilogue 0 store / 1 residual / 2 SiLU) in isolation on
 * `device`, weights rotated over > 512 MB so every launch streams from HBM.
 * Returns the mean device time per launch and the weight bytes it reads. */
espec_status espec_bench_gemv(int K, int N, int T, int nprob, int epi, int iters, int device, double* us_per_launch,
                              double* bytes_per_launch);
/* Instrumentation: time the tcgen05 prompt-prefill GEMM (M <= 256 rows). */
espec_status espec_bench_tc(int M, int K, int N, int iters, int device, double* us_per_launch,
                            double* flops_per_launch);
/* Test probe: the prefill GEMM on host fp32 inputs (W logical K x N). */
espec_status espec_probe_tc(int M, int K, int N, const float* x, const float* w, float* out, int device);
/* One decode GEMV (epi 0 store / 1 residual over a zero residual) of T <= 16 rows on host
 * data, x [T][K], w [K][N] (rounded to bf16): the batch-invariance probe (a row's
 * result must not depend on T). */
espec_status espec_probe_gemv(int T, int K, int N, int epi, const float* x, const float* w, float* out, int device);
/* Instrumentation: time the paged bf16 decode/verify attention for T causal
 * query rows at the end of a ctx-row context (nprob layers batched). */
espec_status espec_bench_attn(int T, int n_heads, int n_kv, int d_head, int ctx, int nprob, int iters, int device,
                              double* us_per_launch, double* bytes_per_launch);

#ifdef __cplusplus
}
#endif
#endif /* ESPEC_C_H */
