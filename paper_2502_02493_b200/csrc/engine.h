// Host orchestrator for the B200 EasySpec decode loop.
//
// Mirrors the reference's Generation (proj/src/orchestrator.cpp:138-484):
// the committed token list and every cache's row bookkeeping (committed
// prefix + staged forest, parents, fuzzy flags, rotary positions) live on the
// host exactly as in proj/src/kv_cache.cpp; K/V rows, weights, activations and
// the drafted/accepted token ids live in HBM and never round-trip through the
// host inside an iteration. One host synchronisation per iteration reads the
// verification outcome (m, path, bonus).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.h"

namespace espec {

enum Status : int {
    ST_OK = 0, ST_CONFIG = 1, ST_IO = 2, ST_CHECK = 3, ST_SHAPE = 4, ST_STRUCTURE = 5, ST_DOMAIN = 6,
    ST_CUDA = 7, ST_NCCL = 8
};

struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

enum Algorithm : int { ALG_VANILLA = 0, ALG_SD = 1, ALG_SD_TREE = 2, ALG_EASYSPEC = 3 };

struct ModelCfg {
    int vocab_size = 258, d_model = 64, n_layers = 4, n_heads = 4, n_kv_heads = 4, d_head = 16, d_mlp = 128;
    int max_positions = 512;
    float norm_eps = 1e-5f;
    float rope_theta = 10000.f;
    int tied_head = 1;
    int weight_dtype = espec_dev::DT_F32;
    int kv_dtype = espec_dev::DT_F32;
    uint64_t seed = 0;
    void validate() const;
};

struct RunCfg {
    int algorithm = ALG_EASYSPEC;
    int n = 5;
    std::vector<int> widths;  // empty = all ones
    int lp_size = 4;
    std::string plan_override;
    float temperature = 0.f;
    int max_new_tokens = 64;
    uint64_t seed = 1;
    int calibration = 1;
    int strict_greedy_tree = 0;  // 1: the reference's greedy multi-sibling CheckError (verifier.cpp:146-158)
    std::vector<int> effective_widths() const;
};

// Layer plan (proj/src/layer_plan.cpp).
struct LayerPlan {
    std::vector<std::vector<int>> groups;
    int lp_size = 1;
    int n_layers() const;
    int max_group_size() const;
};
LayerPlan plan_groups(int n_layers, int lp_size);
LayerPlan parse_plan_override(const std::string& spec);
std::string format_plan(const LayerPlan& plan);

struct IterationTrace {
    int m = 0, n = 0, drafted_nodes = 0, emitted = 0;
    int sequential_forwards = 0, fuzzy_forwards = 0, base_forwards = 0;
    int committed = 0, draft_committed = 0, base_committed = 0;
    float calibrate_ms = 0, draft_ms = 0, verify_ms = 0;  // device time (CUDA events)
    int bonus = 0;
    // simulated stage units of the reference's cost model (cost_sim.h;
    // IterationTrace::*_sim, orchestrator.cpp:263-386)
    double calibrate_sim = 0, draft_sim = 0, verify_sim = 0;
};
struct CostParams;

// DraftTree (proj/include/espec/draft_engine.hpp:63-84) as plain arrays.
struct TreeOut {
    uint64_t id = 0;  // iteration the tree was drafted in
    std::vector<int> widths, token, parent, depth, prob_index, cache_row, first_child, n_children;
    int root_children = 0, n_dists = 0;
    std::vector<float> dists;  // [n_dists][V] when requested
};
// VerificationOutcome (proj/include/espec/verifier.hpp:14-21).
struct OutcomeOut {
    uint64_t id = 0;
    int m = 0, n = 0, bonus = 0;
    std::vector<int> path, tokens;
};

// One layer's intermediates of a probed pass (LayerProbe + AttnCapture,
// proj/include/espec/draft_engine.hpp:24-37, model.hpp:67-69): T rows each.
struct LayerCapture {
    std::vector<float> h_in, q, k, v, attn_out;
};

class Engine;
// tp > 1: this engine is shard `rank` of a tensor-parallel group (one per
// GPU); link the group with comm_link (one process) or comm_ipc_* (one
// process per GPU) before loading weights' first use.
// draft_lp: the drafter's layer-parallel placement (group slot j -> rank j,
// full-head attention + KV on the owner, MLP / head tensor-parallel)
std::unique_ptr<Engine> make_engine(const ModelCfg& base, const ModelCfg& draft, const RunCfg& run, int device,
                                    int tp = 1, int rank = 0, bool draft_lp = false);

class Engine {
public:
    virtual ~Engine() = default;
    virtual void init_weights_seeded(int which, uint64_t seed, bool parity) = 0;
    virtual void share_truncated_draft() = 0;  // drafter = first L_d base layers
    virtual void load_tensor(int which, const std::string& name, int layer, const float* data, long long rows,
                             long long cols) = 0;
    virtual void set_run(const RunCfg& run) = 0;
    // RunConfig::cost (orchestrator.hpp:34): the simulated-time model the
    // stages advance; validated; takes effect at the next begin()/prefill()
    virtual void set_cost(const CostParams& cost) = 0;
    virtual std::string occupancy_csv() const = 0;  // GenerateResult::occupancy_csv of the current generation
    // Start a generation over already-tokenized input (BOS + bytes).
    virtual void begin(const std::vector<int>& tokens) = 0;
    virtual bool done() const = 0;
    virtual IterationTrace step(std::vector<int>& emitted) = 0;
    virtual std::vector<int> generate(const std::vector<int>& tokens, std::vector<IterationTrace>* traces) = 0;
    // prefix_distribution (proj/src/orchestrator.cpp:494-526)
    virtual std::map<std::vector<int>, long> prefix_distribution(const std::vector<int>& tokens, long runs,
                                                                 long first = 0, long stride = 1) = 0;
    // Stage-level iteration (run_iteration_speculative split at the
    // reference's stage boundaries, proj/src/orchestrator.cpp:256-428).
    virtual void prefill(const std::vector<int>& tokens) = 0;
    virtual void calibrate(float* root_logits) = 0;
    virtual void draft(TreeOut* out, bool want_dists) = 0;
    virtual void tree(TreeOut& out, bool want_dists) = 0;
    virtual void verify(const TreeOut* caller, OutcomeOut* out) = 0;
    virtual void resolve_draft_cache(const OutcomeOut* outcome) = 0;
    virtual IterationTrace commit_outcome(std::vector<int>& emitted) = 0;
    // Parity probes.
    virtual void forward_chain(int which, const std::vector<int>& tokens, const std::string& plan, float* logits,
                               float* hidden) = 0;
    virtual void forward_tree(int which, const std::vector<int>& prompt, const std::vector<int>& tokens,
                              const std::vector<int>& parents, const std::string& plan, float* logits,
                              float* hidden) = 0;
    virtual void forward_capture(int which, const std::vector<int>& tokens, const std::string& plan,
                                 std::vector<LayerCapture>& out) = 0;
    virtual int cache_rows(int which, int layer, int row0, int n, float* k, float* v) = 0;
    virtual int cache_committed(int which) const = 0;
    virtual const std::vector<int>& committed() const = 0;
    virtual void weight(int which, const std::string& name, int layer, float* out, long long rows,
                        long long cols) = 0;
    virtual void sync() = 0;
    virtual void* stream() = 0;
    virtual long long device_bytes() const = 0;
    virtual int kernel_launches() const = 0;
    virtual void reset_launch_count() = 0;
    // Per-launch CUDA-event timing of one kernel site (which model, kind):
    // kind 0 QKV GEMV, 1 attention, 2 O GEMV, 3 gate/up GEMV, 4 down GEMV, 5 head.
    virtual void time_site(int which, int kind) = 0;  // which < 0 disables
    virtual void site_stats(int* count, double* total_ms, double* bytes_per_launch) = 0;
    virtual void io_bytes(long long* h2d, long long* d2h) const = 0;
    // ---- tensor-parallel group wiring (tp > 1)
    virtual int tp_size() const = 0;
    // one process: give every shard the others' receive regions
    virtual void comm_link(const std::vector<Engine*>& group) = 0;
    // one process per GPU: export this rank's cudaIpcMemHandle_t (64 bytes),
    // then import all ranks' handles in rank order
    virtual void comm_ipc_export(void* handle64) = 0;
    // shard proxy: one engine stands in for all tp_size ranks (timing only)
    virtual void comm_loopback() = 0;
    virtual void comm_ipc_import(const void* handles, int world) = 0;
    // device pointer of this shard's receive region (comm_link)
    virtual void* comm_region() = 0;
};

}  // namespace espec
