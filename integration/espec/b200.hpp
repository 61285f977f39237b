// espec/b200.hpp — the reference-side binding a maintainer of the reference
// (/root/reference/proj) would add to run its decode loop on a B200 through
// libespec_b200.so. Header-only, in the reference's namespace, over its own
// types (Model, RunConfig, GenerateResult, DraftTree, VerificationOutcome).
// Compiled and run against the unmodified reference core by
// oracle/integration_check.cpp (make -C oracle integration).
//
//  * generate_b200(base, draft, cfg, prompt)       ~ espec::generate
//    (proj/include/espec/orchestrator.hpp:66-67)
//  * B200Generation::{leading_pass, draft, verify, resolve_draft_cache,
//    commit}                                          ~ Generation's stages
//    (proj/src/orchestrator.cpp:256-428), returning the reference's
//    DraftTree (draft_engine.hpp:63-84) and VerificationOutcome
//    (verifier.hpp:14-21)
#pragma once
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "espec/draft_engine.hpp"
#include "espec/errors.hpp"
#include "espec/orchestrator.hpp"
#include "espec/verifier.hpp"
extern "C" {
#include "espec_c.h"
}

namespace espec {

inline void b200_check(espec_status st, espec_engine* e) {
    if (st == ESPEC_OK) return;
    const std::string msg = e ? espec_last_error(e) : espec_create_error();
    switch (st) {  // back to the reference taxonomy (errors.hpp:11-44)
        case ESPEC_CONFIG: throw ConfigError(msg);
        case ESPEC_IO: throw IoError(msg);
        case ESPEC_CHECK: throw CheckError(msg);
        case ESPEC_SHAPE: throw ShapeError(msg);
        case ESPEC_STRUCTURE: throw StructureError(msg);
        case ESPEC_DOMAIN: throw DomainError(msg);
        default: throw std::runtime_error("b200: " + msg);
    }
}

inline espec_model_cfg b200_cfg(const ModelConfig& c) {
    // the reference model = MHA, tied head, rope base 10000, fp32 weights and KV
    return {c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.n_heads, c.d_head, c.d_mlp,
            c.max_positions, c.norm_eps, 10000.f, /*tied*/ 1, ESPEC_F32, ESPEC_F32, c.seed};
}

inline void b200_upload(espec_engine* e, int which, const Model& m) {
    auto put = [&](const char* n, int layer, const Matrix& x) {
        b200_check(espec_load_tensor(e, which, n, layer, x.data.data(), x.rows, x.cols), e);
    };
    put("embedding", -1, m.weights.embedding);
    put("final_norm_gain", -1, m.weights.final_norm_gain);
    for (int l = 0; l < m.config.n_layers; ++l) {
        const LayerWeights& w = m.weights.layers[static_cast<std::size_t>(l)];
        put("wq", l, w.wq);
        put("wk", l, w.wk);
        put("wv", l, w.wv);
        put("wo", l, w.wo);
        put("w_gate", l, w.w_gate);
        put("w_up", l, w.w_up);
        put("w_down", l, w.w_down);
        put("attn_norm_gain", l, w.attn_norm_gain);
        put("mlp_norm_gain", l, w.mlp_norm_gain);
    }
}

// One generation on a B200, stage by stage (Generation, orchestrator.cpp:138-484).
class B200Generation {
public:
    B200Generation(const Model& base, const Model& draft, const RunConfig& cfg, int device = 0)
        : widths_(cfg.effective_widths()), plan_(cfg.plan_override.value_or("")), vocab_(base.config.vocab_size) {
        const espec_model_cfg bc = b200_cfg(base.config), dc = b200_cfg(draft.config);
        const espec_run_cfg rc = {static_cast<int>(cfg.algorithm), cfg.n, widths_.data(), cfg.lp_size,
                                  plan_.c_str(), cfg.temperature, cfg.max_new_tokens, cfg.seed,
                                  cfg.calibration ? 1 : 0, /*strict_greedy_tree*/ 1};
        const espec_device_map dm = {device, 1, &device, /*tp_size*/ 1, /*tp_rank*/ 0};
        b200_check(espec_engine_create(&bc, &dc, &rc, &dm, &e_), nullptr);
        try {
            // RunConfig::cost: the engine's stages advance the same simulated clock
            const CostParams& c = cfg.cost;
            const espec_cost_params cp = {c.c_fixed,       c.c_mem,         c.c_comp,        c.t_addi,
                                          c.attn_workload, c.mlp_workload,  c.base_layer_workload,
                                          c.tp_size_base,  c.tp_size_draft, c.devices};
            b200_check(espec_set_cost(e_, &cp), e_);
            b200_upload(e_, 1, base);
            b200_upload(e_, 0, draft);
        } catch (...) {
            espec_engine_destroy(e_);
            throw;
        }
    }
    ~B200Generation() { espec_engine_destroy(e_); }
    B200Generation(const B200Generation&) = delete;
    B200Generation& operator=(const B200Generation&) = delete;

    void prefill(std::span<const Token> tokens) {
        b200_check(espec_prefill(e_, reinterpret_cast<const int32_t*>(tokens.data()), (int)tokens.size()), e_);
    }
    // drafter_leading_pass -> root logits (1 x V)
    Matrix leading_pass() {
        Matrix root(1, vocab_);
        b200_check(espec_calibrate(e_, root.data.data()), e_);
        return root;
    }
    // draft_stage -> DraftTree
    DraftTree draft() {
        espec_tree t{};
        std::vector<float> dists((size_t)(ESPEC_MAX_NODES + 1) * vocab_);
        t.dists = dists.data();
        t.dist_capacity = ESPEC_MAX_NODES + 1;
        b200_check(espec_draft(e_, &t), e_);
        tree_id_ = t.id;
        DraftTree tree;
        tree.widths = widths_;
        tree.root_children = t.root_children;
        for (int j = 0; j < t.n_nodes; ++j)
            tree.nodes.push_back(DraftNode{t.token[j], t.parent[j], t.depth[j], t.prob_index[j], t.cache_row[j],
                                           t.first_child[j], t.n_children[j]});
        for (int d = 0; d < t.n_dists; ++d) {
            ProbVector p(vocab_);
            std::copy(dists.begin() + (size_t)d * vocab_, dists.begin() + (size_t)(d + 1) * vocab_, p.probs.begin());
            tree.dists.push_back(std::move(p));
        }
        return tree;
    }
    // verify_stage + verify_tree -> VerificationOutcome (the tree's tokens
    // may have been edited; its shape must be the drafted one)
    VerificationOutcome verify(const DraftTree& tree) {
        espec_tree t{};
        t.id = tree_id_;
        t.n_nodes = tree.node_count();
        t.root_children = tree.root_children;
        t.n_levels = (int)tree.widths.size();
        for (int j = 0; j < t.n_nodes; ++j) {
            const DraftNode& n = tree.nodes[static_cast<std::size_t>(j)];
            t.token[j] = n.token;
            t.parent[j] = n.parent;
        }
        b200_check(espec_verify(e_, &t, &last_), e_);
        VerificationOutcome o;
        o.m = last_.m;
        o.n = last_.n;
        o.bonus_token = last_.bonus;
        o.accepted_path.assign(last_.accepted_path, last_.accepted_path + last_.m);
        o.accepted_tokens.assign(last_.accepted_tokens, last_.accepted_tokens + last_.m);
        return o;
    }
    void resolve_draft_cache() { b200_check(espec_resolve_draft_cache(e_, &last_), e_); }
    // commit accepted + bonus; returns the emitted tokens
    std::vector<Token> commit() {
        std::vector<int32_t> em(ESPEC_MAX_NODES + 2);
        int n = 0;
        b200_check(espec_commit_outcome(e_, em.data(), &n, nullptr), e_);
        return std::vector<Token>(em.begin(), em.begin() + n);
    }
    bool done() const { return espec_done(e_) != 0; }
    espec_engine* handle() { return e_; }

private:
    espec_engine* e_ = nullptr;
    std::vector<int> widths_;
    std::string plan_;
    int vocab_;
    uint64_t tree_id_ = 0;
    espec_outcome last_{};
};

// Same signature and semantics as espec::generate (orchestrator.cpp:488-492).
// The report comes from the reference's own aggregate() (report.cpp:51-95)
// over the engine's iteration traces: device stage times in the *_wall slots,
// the engine's simulated units (RunConfig::cost) in the *_sim slots, the
// vanilla baseline from vanilla_baseline_sim (orchestrator.cpp:72-77), and the
// engine's SimClock occupancy CSV.
inline GenerateResult generate_b200(const Model& base, const Model& draft, const RunConfig& cfg,
                                    std::span<const std::uint8_t> prompt, int device = 0) {
    B200Generation g(base, draft, cfg, device);
    GenerateResult out;
    out.tokens.resize(static_cast<std::size_t>(cfg.max_new_tokens));
    std::vector<espec_iteration> it(static_cast<std::size_t>(cfg.max_new_tokens));
    int n_out = 0, n_it = 0;
    b200_check(espec_generate(g.handle(), prompt.data(), (int)prompt.size(),
                              reinterpret_cast<int32_t*>(out.tokens.data()), &n_out, it.data(), &n_it),
               g.handle());
    out.tokens.resize(static_cast<std::size_t>(n_out));
    std::vector<IterationTrace> traces;
    for (int i = 0; i < n_it; ++i) {
        const espec_iteration& e = it[static_cast<std::size_t>(i)];
        IterationTrace t;
        t.m = e.m;
        t.n = e.n;
        t.drafted_nodes = e.drafted_nodes;
        t.emitted = e.emitted;
        t.draft_wall = e.draft_ms * 1e-3;
        t.verify_wall = e.verify_ms * 1e-3;
        t.calibrate_wall = e.calibrate_ms * 1e-3;
        t.draft_sim = e.draft_sim;
        t.verify_sim = e.verify_sim;
        t.calibrate_sim = e.calibrate_sim;
        t.fuzzy_forwards = e.fuzzy_forwards;
        t.sequential_forwards = e.sequential_forwards;
        t.base_forwards = e.base_forwards;
        traces.push_back(t);
    }
    const int prompt_len = static_cast<int>(tokenize_prompt(prompt, base.config.vocab_size).size());
    out.report = aggregate(traces, vanilla_baseline_sim(cfg.cost, base.config.n_layers, prompt_len,
                                                        static_cast<long>(out.tokens.size())));
    out.report.algorithm = to_string(cfg.algorithm);
    out.report.n = cfg.algorithm == Algorithm::vanilla ? 0 : cfg.n;
    int len = 0;
    espec_occupancy_csv(g.handle(), nullptr, 0, &len);
    std::string occ(static_cast<std::size_t>(len) + 1, '\0');
    b200_check(espec_occupancy_csv(g.handle(), occ.data(), len + 1, &len), g.handle());
    occ.resize(static_cast<std::size_t>(len));
    out.occupancy_csv = occ;
    return out;
}

}  // namespace espec
