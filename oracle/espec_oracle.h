/*
 * espec_oracle.h — CPU restatement of the reference EasySpec decode path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 engine: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product path
 * (paper_2502_02493_b200) never links or calls it.
 *
 * Every function restates the algorithm of the reference C++ core under
 * /root/reference/proj (file:line cited at each definition in
 * espec_oracle.c) in plain C11 with the same fp32 operation order, so its
 * tokens, K/V rows and logits are bit-identical to the reference's on the
 * same seeds. That claim is pinned by tests/test_oracle.py against the
 * fixtures in tests/golden/ (written by oracle/_ref/ref_dump, which links
 * the unmodified reference objects).
 */
#ifndef ESPEC_ORACLE_H
#define ESPEC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors espec::ModelConfig (proj/include/espec/model.hpp:19-33). */
typedef struct {
    int vocab_size;
    int d_model;
    int n_layers;
    int n_heads;
    int d_head;
    int d_mlp;
    int max_positions;
    float norm_eps;
    uint64_t seed;
} eo_config;

/* Mirrors espec::RunConfig (proj/include/espec/orchestrator.hpp:23-38). */
enum { EO_VANILLA = 0, EO_SD = 1, EO_SD_TREE = 2, EO_EASYSPEC = 3 };
typedef struct {
    int algorithm;
    int n;
    const int* widths; /* n entries, or NULL for all ones */
    int lp_size;
    const char* plan_override; /* NULL or "" for none */
    float temperature;
    int max_new_tokens;
    uint64_t seed;
    int calibration;
} eo_run;

/* Status codes, one per reference exception type
 * (proj/include/espec/errors.hpp:11-44). */
enum { EO_OK = 0, EO_CONFIG = 1, EO_IO = 2, EO_CHECK = 3, EO_SHAPE = 4, EO_STRUCTURE = 5,
       EO_DOMAIN = 6 };

typedef struct eo_model eo_model;
typedef struct eo_result eo_result;

eo_model* eo_model_init(const eo_config* cfg, int* status);
eo_model* eo_model_truncated(const eo_model* base, int keep_layers, int* status);
void eo_model_free(eo_model* m);
/* name: "embedding", "final_norm_gain", "wq","wk","wv","wo","w_gate","w_up",
 * "w_down","attn_norm_gain","mlp_norm_gain". Returns row-major data. */
const float* eo_model_tensor(const eo_model* m, const char* name, int layer, int* rows, int* cols);

/* One chain pass over `tokens` on a fresh cache: layer-sequential when
 * plan is NULL/"" else fuzzy under the plan (lp form "lp=N" or an override
 * string). Outputs (each may be NULL): hidden n×d, logits n×V,
 * k/v n_layers×n×d. Returns a status code. */
int eo_prefill(const eo_model* m, const char* plan, const int* tokens, int n, float* hidden,
               float* logits, float* k, float* v);

/* Layer plan helpers (proj/src/layer_plan.cpp). Writes the formatted plan. */
int eo_plan_groups(int n_layers, int lp_size, char* out, int out_len);
int eo_parse_plan(const char* spec, char* out, int out_len);

/* Full generation (proj/src/orchestrator.cpp:488-492). */
eo_result* eo_generate(const eo_model* base, const eo_model* draft, const eo_run* run,
                       const uint8_t* prompt, int prompt_len);
int eo_result_status(const eo_result* r);
const char* eo_result_error(const eo_result* r);
const int* eo_result_tokens(const eo_result* r, int* n);
int eo_result_n_iters(const eo_result* r);
/* out[10] = m, n, drafted_nodes, emitted, sequential, fuzzy, base,
 *           committed, draft_committed, base_committed */
void eo_result_iter(const eo_result* r, int i, int* out);
/* n_layers×4 doubles: sum K, sum |K|, sum V, sum |V| of committed rows. */
void eo_result_kvsums(const eo_result* r, int i, int which_base, double* out);
int eo_result_cache_len(const eo_result* r, int which_base);
/* committed rows of one layer of the final cache: len×d each. */
void eo_result_cache_rows(const eo_result* r, int which_base, int layer, float* k, float* v);
void eo_result_free(eo_result* r);

/* Verifier unit entry (proj/src/verifier.cpp:86-177) over explicit trees:
 * n_nodes nodes with token/parent(-1 root)/prob_index, n_dists draft dists
 * (vocab each), base_dists (n_nodes+1)×vocab, widths[n_levels].
 * Outputs m, accepted tokens (≤ n_levels), bonus. rng_seed seeds the
 * stream. Returns a status code. */
int eo_verify_tree(int vocab, int n_nodes, const int* tokens, const int* parents,
                   const int* prob_index, int n_dists, const float* dists,
                   const float* base_dists, int n_levels, const int* widths, float temperature,
                   uint64_t rng_seed, int* m, int* accepted, int* bonus);

/* select_children (proj/src/draft_engine.cpp:141-186). Returns count. */
int eo_select_children(const float* logits, int vocab, int k, float temperature,
                       uint64_t rng_seed, int* out);

/* xoshiro256** stream (proj/include/espec/rng.hpp:24-68): n uniform doubles. */
void eo_rng_uniforms(uint64_t seed, int n, double* out);

#ifdef __cplusplus
}
#endif
#endif
