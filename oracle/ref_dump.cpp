// Golden-vector generator. TEST INFRASTRUCTURE ONLY.
//
// Links the unmodified reference core (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/) and writes
// JSON fixtures that pin the C restatement in oracle/espec_oracle.c:
//   * init checksums      -> init_model            proj/src/model.cpp:38-84
//   * the argmax-110 KAT  -> proj/tests/test_model.cpp:61-68
//   * layer plans         -> plan_groups           proj/src/layer_plan.cpp:54-82
//   * forward outputs     -> forward_sequential / forward_fuzzy
//                            proj/src/draft_engine.cpp:35-133
//   * full generations    -> generate()            proj/src/orchestrator.cpp:488-492
//     with per-iteration traces and KV-cache checksums taken through the
//     IterationHook (proj/include/espec/orchestrator.hpp:46-55).
// Nothing here is shipped or measured.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "espec/cost_sim.hpp"
#include "espec/draft_engine.hpp"
#include "espec/errors.hpp"
#include "espec/kv_cache.hpp"
#include "espec/layer_plan.hpp"
#include "espec/model.hpp"
#include "espec/orchestrator.hpp"
#include "espec/verifier.hpp"
#include "espec/model_io.hpp"
#include "espec/report.hpp"

using namespace espec;
using json = nlohmann::ordered_json;

namespace {

ModelConfig tiny(int n_layers, std::uint64_t seed, int d_model = 32, int n_heads = 2, int d_head = 16,
                 int d_mlp = 64, int max_pos = 128) {
    ModelConfig c;
    c.d_model = d_model;
    c.n_heads = n_heads;
    c.d_head = d_head;
    c.d_mlp = d_mlp;
    c.n_layers = n_layers;
    c.max_positions = max_pos;
    c.seed = seed;
    return c;
}

json cfg_json(const ModelConfig& c) {
    return json{{"vocab_size", c.vocab_size}, {"d_model", c.d_model}, {"n_layers", c.n_layers},
                {"n_heads", c.n_heads},       {"d_head", c.d_head},   {"d_mlp", c.d_mlp},
                {"max_positions", c.max_positions}, {"norm_eps", c.norm_eps},
                {"seed", c.seed}};
}

std::vector<Token> bos_bytes(const std::string& s) {
    std::vector<Token> t = {kBosToken};
    for (unsigned char c : s) t.push_back(c);
    return t;
}

std::vector<float> as_vec(const Matrix& m) { return m.data; }

// Chain prefill on a fresh/partial cache (stage + sequential pass).
Matrix prefill(const Model& model, const std::vector<Token>& tokens, KvCache& cache, bool commit) {
    std::vector<int> parents;
    for (std::size_t i = 0; i < tokens.size(); ++i)
        parents.push_back(i == 0 ? kCommittedTail : cache.committed_len() + static_cast<int>(i) - 1);
    ForwardBatch batch;
    batch.flat_rows = cache.stage_append(parents, false);
    for (int r : batch.flat_rows) batch.positions.push_back(cache.position_of(r));
    const TreeMask mask = cache.build_tree_mask();
    batch.mask = &mask;
    Matrix h = forward_sequential(model, embed(model, tokens), cache, batch);
    if (commit) cache.commit_path(batch.flat_rows);
    return h;
}

double tensor_sum(const Matrix& m) {
    double s = 0.0;
    for (float v : m.data) s += v;
    return s;
}

json init_probe(const ModelConfig& cfg) {
    const Model m = init_model(cfg);
    json j;
    j["config"] = cfg_json(cfg);
    j["embedding_sum"] = tensor_sum(m.weights.embedding);
    j["embedding_head"] = std::vector<float>(m.weights.embedding.data.begin(),
                                             m.weights.embedding.data.begin() + 8);
    json layers = json::array();
    for (const auto& lw : m.weights.layers) {
        layers.push_back(json{{"wq", tensor_sum(lw.wq)},
                              {"wk", tensor_sum(lw.wk)},
                              {"wv", tensor_sum(lw.wv)},
                              {"wo", tensor_sum(lw.wo)},
                              {"w_gate", tensor_sum(lw.w_gate)},
                              {"w_up", tensor_sum(lw.w_up)},
                              {"w_down", tensor_sum(lw.w_down)},
                              {"w_down_head", std::vector<float>(lw.w_down.data.begin(),
                                                                 lw.w_down.data.begin() + 4)}});
    }
    j["layers"] = layers;
    return j;
}

// Per-layer checksum of the committed K/V rows of a cache.
json cache_sums(const KvCache& cache) {
    json layers = json::array();
    for (int l = 0; l < cache.n_layers(); ++l) {
        double ks = 0, ka = 0, vs = 0, va = 0;
        for (int r = 0; r < cache.committed_len(); ++r) {
            for (float v : cache.key_row(l, r)) {
                ks += v;
                ka += std::fabs(v);
            }
            for (float v : cache.value_row(l, r)) {
                vs += v;
                va += std::fabs(v);
            }
        }
        layers.push_back(json::array({ks, ka, vs, va}));
    }
    return layers;
}

struct GenCase {
    std::string name;
    ModelConfig base;
    int keep;  // 0 = self-draft (draft is the base model itself)
    RunConfig run;
    std::string prompt;
    // Non-zero: the drafter is an independent init_model with this seed and
    // `keep` layers (the CLI's --draft-seed path, proj/src/cli.cpp:252-257).
    std::uint64_t draft_seed = 0;
};

RunConfig run_cfg(Algorithm a, int n, std::vector<int> widths, int lp, float temp, int max_new,
                  std::uint64_t seed, bool calibration = true) {
    RunConfig r;
    r.algorithm = a;
    r.n = n;
    r.widths = std::move(widths);
    r.lp_size = lp;
    r.temperature = temp;
    r.max_new_tokens = max_new;
    r.seed = seed;
    r.calibration = calibration;
    r.workers = 1;
    return r;
}

json run_case(const GenCase& gc) {
    const Model base = init_model(gc.base);
    Model draft;
    if (gc.draft_seed != 0) {
        ModelConfig dc = gc.base;
        dc.n_layers = gc.keep;
        dc.seed = gc.draft_seed;
        draft = init_model(dc);
    } else {
        draft = gc.keep == 0 ? base : make_truncated_draft(base, gc.keep);
    }
    json iters = json::array();
    const IterationHook hook = [&](const IterationInspection& view) {
        iters.push_back(json{{"committed", static_cast<int>(view.committed.size())},
                             {"draft_committed", view.draft_cache.committed_len()},
                             {"base_committed", view.base_cache.committed_len()},
                             {"draft_kv", cache_sums(view.draft_cache)},
                             {"base_kv", cache_sums(view.base_cache)}});
    };
    json j;
    j["name"] = gc.name;
    j["base"] = cfg_json(gc.base);
    j["keep"] = gc.keep;
    j["draft_seed"] = gc.draft_seed;
    j["run"] = json{{"algorithm", to_string(gc.run.algorithm)},
                    {"n", gc.run.n},
                    {"widths", gc.run.effective_widths()},
                    {"lp_size", gc.run.lp_size},
                    {"plan_override", gc.run.plan_override ? *gc.run.plan_override : std::string()},
                    {"temperature", gc.run.temperature},
                    {"max_new_tokens", gc.run.max_new_tokens},
                    {"seed", gc.run.seed},
                    {"calibration", gc.run.calibration}};
    j["prompt"] = gc.prompt;
    try {
        const GenerateResult res = generate(
            base, draft, gc.run,
            {reinterpret_cast<const std::uint8_t*>(gc.prompt.data()), gc.prompt.size()}, hook);
        j["tokens"] = res.tokens;
        json traces = json::array();
        for (std::size_t i = 0; i < res.report.iterations.size(); ++i) {
            const auto& t = res.report.iterations[i];
            json tj{{"m", t.m},
                    {"n", t.n},
                    {"drafted_nodes", t.drafted_nodes},
                    {"emitted", t.emitted},
                    {"sequential_forwards", t.sequential_forwards},
                    {"fuzzy_forwards", t.fuzzy_forwards},
                    {"base_forwards", t.base_forwards}};
            for (auto& [k, v] : iters[i].items()) tj[k] = v;
            traces.push_back(tj);
        }
        j["iterations"] = traces;
        j["alpha"] = res.report.alpha;
        j["error"] = nullptr;
    } catch (const Error& e) {
        j["error"] = e.what();
    }
    return j;
}

// The reference's speculative iteration re-driven stage by stage through its
// PUBLIC functions (forward_sequential / forward_fuzzy / draft_tree /
// verify_tree / KvCache), restating Generation's private glue
// (stage_suffix, drafter_leading_pass, verify_stage, resolve_draft_cache,
// proj/src/orchestrator.cpp:225-436), so every iteration's DraftTree and
// VerificationOutcome can be dumped. main() checks that the tokens equal
// generate()'s for the same case, which pins the restated glue.
json run_stages(const GenCase& gc) {
    const Model base = init_model(gc.base);
    Model draft;
    if (gc.draft_seed != 0) {
        ModelConfig dc = gc.base;
        dc.n_layers = gc.keep;
        dc.seed = gc.draft_seed;
        draft = init_model(dc);
    } else {
        draft = gc.keep == 0 ? base : make_truncated_draft(base, gc.keep);
    }
    const RunConfig& cfg = gc.run;
    const bool easy = cfg.algorithm == Algorithm::easyspec;
    const LayerPlan plan = !easy ? plan_groups(draft.config.n_layers, 1)
                                 : (cfg.plan_override ? parse_plan_override(*cfg.plan_override)
                                                      : plan_groups(draft.config.n_layers, cfg.lp_size));
    const std::vector<int> widths = cfg.effective_widths();
    KvCache bcache(base.config.n_layers, base.config.d_model), dcache(draft.config.n_layers, draft.config.d_model);
    Xoshiro256ss rng(cfg.seed);
    ForwardCounters counters;
    std::vector<Token> committed = bos_bytes(gc.prompt), generated;
    int draft_cached = 0;
    auto suffix = [&](KvCache& cache, int cached, bool fuzzy, std::vector<Token>& toks) {
        std::vector<int> parents;
        for (int i = cached; i < static_cast<int>(committed.size()); ++i) {
            parents.push_back(parents.empty() ? kCommittedTail
                                              : cache.committed_len() + static_cast<int>(parents.size()) - 1);
            toks.push_back(committed[static_cast<std::size_t>(i)]);
        }
        return cache.stage_append(parents, fuzzy);
    };
    auto batch_for = [](const KvCache& cache, const std::vector<int>& rows, const TreeMask* mask, bool cal) {
        ForwardBatch b;
        b.flat_rows = rows;
        for (int r : rows) b.positions.push_back(cache.position_of(r));
        b.mask = mask;
        b.calibrate_writes = cal;
        return b;
    };
    json iters = json::array();
    json j;
    j["name"] = gc.name;
    try {
        while (static_cast<int>(generated.size()) < cfg.max_new_tokens) {
            // drafter_leading_pass
            const bool calibrated = easy && cfg.calibration, fuzzy_pass = easy && !cfg.calibration;
            std::vector<Token> ctoks;
            const std::vector<int> crow = suffix(dcache, draft_cached, fuzzy_pass, ctoks);
            Matrix hidden;
            {
                const TreeMask mask = dcache.build_tree_mask();
                const ForwardBatch b = batch_for(dcache, crow, &mask, calibrated);
                const Matrix h_in = embed(draft, ctoks);
                hidden = fuzzy_pass ? forward_fuzzy(draft, plan, h_in, dcache, b)
                                    : forward_sequential(draft, h_in, dcache, b);
            }
            dcache.commit_path(crow);
            draft_cached = static_cast<int>(committed.size());
            const Matrix root = lm_logits(draft, Matrix(1, hidden.cols, {hidden.row(hidden.rows - 1).begin(),
                                                                         hidden.row(hidden.rows - 1).end()}));
            // draft_stage
            const DraftTree tree = draft_tree(draft, plan, dcache, root.row(0), widths, cfg.temperature, rng,
                                              counters, easy, nullptr);
            // verify_stage
            std::vector<Token> vtoks;
            const std::vector<int> vchain = suffix(bcache, bcache.committed_len(), false, vtoks);
            const int first_node_row = vchain.back() + 1;
            std::vector<int> tparents;
            for (const auto& nd : tree.nodes) {
                tparents.push_back(nd.parent < 0 ? vchain.back() : first_node_row + nd.parent);
                vtoks.push_back(nd.token);
            }
            const std::vector<int> node_rows = bcache.stage_append(tparents, false);
            std::vector<int> all_rows = vchain;
            all_rows.insert(all_rows.end(), node_rows.begin(), node_rows.end());
            const TreeMask bmask = bcache.build_tree_mask();
            const Matrix logits =
                lm_logits(base, forward_sequential(base, embed(base, vtoks), bcache,
                                                   batch_for(bcache, all_rows, &bmask, false)));
            std::vector<ProbVector> bd;
            const int frontier = static_cast<int>(vchain.size()) - 1;
            for (int i = 0; i <= tree.node_count(); ++i)
                bd.push_back(softmax_temp(logits.row(frontier + i), cfg.temperature));
            const VerificationOutcome out = verify_tree(tree, bd, cfg.temperature, rng);
            std::vector<int> commit_rows = vchain;
            for (int ni : out.accepted_path) commit_rows.push_back(node_rows[static_cast<std::size_t>(ni)]);
            bcache.commit_path(commit_rows);
            // resolve_draft_cache
            if (calibrated) {
                dcache.discard_staged();
            } else {
                std::vector<int> rows;
                for (int ni : out.accepted_path) {
                    const int r = tree.nodes[static_cast<std::size_t>(ni)].cache_row;
                    if (r < 0) break;
                    rows.push_back(r);
                }
                dcache.commit_path(rows);
                draft_cached += static_cast<int>(rows.size());
            }
            for (Token t : out.accepted_tokens) committed.push_back(t);
            committed.push_back(out.bonus_token);
            const int emit = std::min(out.m + 1, cfg.max_new_tokens - static_cast<int>(generated.size()));
            for (int i = 0; i < emit; ++i)
                generated.push_back(committed[committed.size() - static_cast<std::size_t>(out.m + 1) +
                                              static_cast<std::size_t>(i)]);
            json t = json::object(), ids = json::array();
            std::vector<int> tok, par, dep, pi, cr, fc, nc;
            for (const auto& nd : tree.nodes) {
                tok.push_back(nd.token);
                par.push_back(nd.parent);
                dep.push_back(nd.depth);
                pi.push_back(nd.prob_index);
                cr.push_back(nd.cache_row);
                fc.push_back(nd.first_child);
                nc.push_back(nd.n_children);
            }
            t["token"] = tok;
            t["parent"] = par;
            t["depth"] = dep;
            t["prob_index"] = pi;
            t["cache_row"] = cr;
            t["first_child"] = fc;
            t["n_children"] = nc;
            t["root_children"] = tree.root_children;
            t["n_dists"] = static_cast<int>(tree.dists.size());
            // first draft distribution's top entries (pins dists without the full V rows)
            double dsum = 0.0;
            for (const auto& d : tree.dists)
                for (float v : d.probs) dsum += v;
            t["dists_sum"] = dsum;
            iters.push_back(json{{"tree", t},
                                 {"m", out.m},
                                 {"n", out.n},
                                 {"path", out.accepted_path},
                                 {"accepted", out.accepted_tokens},
                                 {"bonus", out.bonus_token},
                                 {"draft_committed", dcache.committed_len()},
                                 {"base_committed", bcache.committed_len()}});
        }
        j["tokens"] = generated;
        j["error"] = nullptr;
    } catch (const Error& e) {
        j["error"] = e.what();
    }
    j["iterations"] = iters;
    return j;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string out_dir = argc > 1 ? argv[1] : ".";

    // ---- init + numerics KATs ------------------------------------------------
    json numerics;
    numerics["init"] = json::array({init_probe(tiny(3, 99)), init_probe(tiny(2, 7, 64, 4, 16, 128))});
    {
        // proj/tests/test_model.cpp:61-68 — golden argmax 110.
        const Model m = init_model(tiny(4, 2024));
        KvCache cache(m.config.n_layers, m.config.d_model);
        const Matrix h = prefill(m, bos_bytes("golden"), cache, false);
        const Matrix logits = lm_logits(m, h);
        const auto last = logits.row(logits.rows - 1);
        numerics["golden_argmax"] = json{{"config", cfg_json(m.config)},
                                         {"prompt", "golden"},
                                         {"argmax", argmax(last)},
                                         {"logits", std::vector<float>(last.begin(), last.end())}};
    }
    {
        // Prefill K/V rows + hidden for a 2-layer d32 model.
        const Model m = init_model(tiny(2, 7));
        KvCache cache(m.config.n_layers, m.config.d_model);
        const Matrix h = prefill(m, bos_bytes("ab"), cache, true);
        json kv = json::array();
        for (int l = 0; l < 2; ++l) {
            std::vector<float> k, v;
            for (int r = 0; r < cache.committed_len(); ++r) {
                auto kr = cache.key_row(l, r);
                auto vr = cache.value_row(l, r);
                k.insert(k.end(), kr.begin(), kr.end());
                v.insert(v.end(), vr.begin(), vr.end());
            }
            kv.push_back(json{{"k", k}, {"v", v}});
        }
        numerics["prefill_kv"] = json{{"config", cfg_json(m.config)},
                                      {"prompt", "ab"},
                                      {"hidden", as_vec(h)},
                                      {"logits", as_vec(lm_logits(m, h))},
                                      {"kv", kv}};
    }
    {
        // proj/tests/test_model.cpp:236-269 — tree-path commit then decode.
        const Model m = init_model(tiny(3, 43));
        KvCache cache(m.config.n_layers, m.config.d_model);
        prefill(m, bos_bytes("tre"), cache, true);
        const auto roots = cache.stage_append(std::vector<int>{kCommittedTail, kCommittedTail}, false);
        const auto kids = cache.stage_append(std::vector<int>{roots[0], roots[0]}, false);
        const std::vector<Token> toks = {'a', 'b', 'c', 'd'};
        ForwardBatch batch;
        batch.flat_rows = roots;
        batch.flat_rows.insert(batch.flat_rows.end(), kids.begin(), kids.end());
        for (int r : batch.flat_rows) batch.positions.push_back(cache.position_of(r));
        const TreeMask mask = cache.build_tree_mask();
        batch.mask = &mask;
        const Matrix tree_h = forward_sequential(m, embed(m, toks), cache, batch);
        cache.commit_path(std::vector<int>{roots[0], kids[0]});
        const Matrix next = prefill(m, {'e'}, cache, false);
        numerics["tree_commit"] = json{{"config", cfg_json(m.config)},
                                       {"tree_logits", as_vec(lm_logits(m, tree_h))},
                                       {"next_logits", as_vec(lm_logits(m, next))}};
    }
    {
        // Fuzzy vs sequential forward on a 4-token chain, 8 layers, lp 3.
        const Model m = init_model(tiny(8, 63));
        const std::vector<Token> toks = {kBosToken, 'f', 'u', 'z'};
        json fz;
        fz["config"] = cfg_json(m.config);
        fz["tokens"] = toks;
        for (int lp : {1, 2, 3, 4}) {
            const LayerPlan plan = plan_groups(8, lp);
            KvCache cache(m.config.n_layers, m.config.d_model);
            std::vector<int> parents = {kCommittedTail, 0, 1, 2};
            ForwardBatch batch;
            batch.flat_rows = cache.stage_append(parents, true);
            for (int r : batch.flat_rows) batch.positions.push_back(cache.position_of(r));
            const TreeMask mask = cache.build_tree_mask();
            batch.mask = &mask;
            const Matrix h = forward_fuzzy(m, plan, embed(m, toks), cache, batch);
            fz["lp" + std::to_string(lp)] =
                json{{"plan", format_plan(plan)}, {"hidden", as_vec(h)}, {"logits", as_vec(lm_logits(m, h))}};
        }
        numerics["fuzzy"] = fz;
    }
    {
        json plans = json::array();
        const int cases[][2] = {{32, 4}, {28, 4}, {28, 8}, {24, 4}, {24, 2}, {24, 1}, {8, 2},
                                {8, 3},  {12, 3}, {5, 2},  {2, 1},  {3, 5},  {80, 8}, {32, 8},
                                {32, 2}, {32, 1}, {9, 4},  {10, 4}, {4, 3},  {6, 6}};
        for (const auto& c : cases) {
            plans.push_back(json{{"n_layers", c[0]}, {"lp", c[1]},
                                 {"plan", format_plan(plan_groups(c[0], c[1]))}});
        }
        numerics["plans"] = plans;
    }
    {
        std::ofstream f(out_dir + "/ref_numerics.json");
        f << numerics.dump() << "\n";
    }

    // ---- generations ----------------------------------------------------------
    std::vector<GenCase> cases;
    const ModelConfig c1 = tiny(12, 7, 64, 4, 16, 128, 512);  // proj/src/cli.cpp:210-218
    const std::vector<int> chain4 = {1, 1, 1, 1};
    for (Algorithm a : {Algorithm::vanilla, Algorithm::sd, Algorithm::sd_tree, Algorithm::easyspec}) {
        cases.push_back({"c1_" + to_string(a), c1, 8, run_cfg(a, 4, chain4, 2, 0.0f, 64, 1),
                         "the quick brown fox"});
    }
    const ModelConfig fa = tiny(12, 21);
    for (Algorithm a : {Algorithm::vanilla, Algorithm::sd, Algorithm::easyspec}) {
        cases.push_back({"fixa_" + to_string(a), fa, 8, run_cfg(a, 4, chain4, 2, 0.0f, 40, 1),
                         "Zq8#k!pL2@xR9&mW"});
    }
    cases.push_back({"fixa_easyspec_nocal", fa, 8,
                     run_cfg(Algorithm::easyspec, 4, chain4, 2, 0.0f, 40, 1, false),
                     "Zq8#k!pL2@xR9&mW"});
    cases.push_back({"fixa_easyspec_lp4", fa, 8,
                     run_cfg(Algorithm::easyspec, 5, {1, 1, 1, 1, 1}, 4, 0.0f, 40, 1),
                     "Zq8#k!pL2@xR9&mW"});
    {
        GenCase g{"fixa_easyspec_override", fa, 8,
                  run_cfg(Algorithm::easyspec, 4, chain4, 3, 0.0f, 40, 1), "Zq8#k!pL2@xR9&mW"};
        g.run.plan_override = "0|1-3|4-6|7";
        cases.push_back(g);
    }
    cases.push_back({"deep_easyspec_lp4", tiny(10, 77), 9,
                     run_cfg(Algorithm::easyspec, 5, {1, 1, 1, 1, 1}, 4, 0.0f, 36, 1),
                     "layer parallel"});
    cases.push_back({"self_greedy", tiny(4, 83), 0,
                     run_cfg(Algorithm::easyspec, 4, chain4, 1, 0.0f, 20, 3), "fixed point"});
    cases.push_back({"cap7", tiny(4, 99), 0,
                     run_cfg(Algorithm::easyspec, 4, chain4, 1, 0.0f, 7, 3), "cap"});
    // Temperature > 0 (RNG-order parity): chains and trees.
    cases.push_back({"t08_chain_easyspec", tiny(6, 97), 4,
                     run_cfg(Algorithm::easyspec, 4, chain4, 2, 0.8f, 16, 3), "ranges"});
    cases.push_back({"t08_chain_sd", tiny(6, 97), 4,
                     run_cfg(Algorithm::sd, 4, chain4, 2, 0.8f, 16, 3), "ranges"});
    cases.push_back({"t08_chain_vanilla", tiny(6, 97), 4,
                     run_cfg(Algorithm::vanilla, 4, chain4, 2, 0.8f, 16, 3), "ranges"});
    cases.push_back({"t08_tree_easyspec", tiny(6, 91), 4,
                     run_cfg(Algorithm::easyspec, 4, {2, 2, 2, 2}, 2, 0.8f, 16, 3), "replay"});
    cases.push_back({"t08_tree_sd_tree", tiny(6, 91), 4,
                     run_cfg(Algorithm::sd_tree, 4, {2, 2, 2, 2}, 2, 0.8f, 16, 3), "replay"});
    cases.push_back({"crit4_easyspec", tiny(7, 33), 5,
                     run_cfg(Algorithm::easyspec, 3, {2, 2, 2}, 2, 0.8f, 16, 500), "calibrated"});
    cases.push_back({"crit4_nocal", tiny(7, 33), 5,
                     run_cfg(Algorithm::easyspec, 3, {2, 2, 2}, 2, 0.8f, 16, 500, false),
                     "calibrated"});
    cases.push_back({"t1_tree_wide", tiny(5, 93), 3,
                     run_cfg(Algorithm::easyspec, 3, {3, 2, 1}, 2, 1.0f, 18, 9), "wide tree"});
    // Greedy tree: the reference throws when a first sibling is rejected
    // (proj/src/verifier.cpp:156-157); recorded so the oracle reproduces it.
    cases.push_back({"greedy_tree_throws", tiny(6, 91), 4,
                     run_cfg(Algorithm::easyspec, 4, {2, 2, 2, 2}, 2, 0.0f, 16, 3), "replay"});

    // Cases with rejections (alpha < 1) so the reject/residual paths run.
    cases.push_back({"rej_greedy_d32s21k2", tiny(8, 21, 32, 2, 16, 64, 256), 2,
                     run_cfg(Algorithm::easyspec, 4, chain4, 2, 0.0f, 48, 1), "hello world, again"});
    cases.push_back({"rej_greedy_sd_d32s21k2", tiny(8, 21, 32, 2, 16, 64, 256), 2,
                     run_cfg(Algorithm::sd, 4, chain4, 2, 0.0f, 48, 1), "hello world, again"});
    cases.push_back({"rej_greedy_vanilla_d32s21k2", tiny(8, 21, 32, 2, 16, 64, 256), 2,
                     run_cfg(Algorithm::vanilla, 4, chain4, 2, 0.0f, 48, 1), "hello world, again"});
    cases.push_back({"rej_greedy_d64s11k3", tiny(8, 11, 64, 4, 16, 128, 256), 3,
                     run_cfg(Algorithm::easyspec, 4, chain4, 2, 0.0f, 48, 1), "layer parallel"});
    {
        GenCase g{"indep_greedy_easyspec", tiny(8, 11, 64, 4, 16, 128, 256), 5,
                  run_cfg(Algorithm::easyspec, 5, {1, 1, 1, 1, 1}, 4, 0.0f, 40, 1), "independent"};
        g.draft_seed = 9;
        cases.push_back(g);
        g.name = "indep_greedy_vanilla";
        g.run.algorithm = Algorithm::vanilla;
        cases.push_back(g);
    }
    cases.push_back({"t3_chain_easyspec", tiny(8, 5, 32, 2, 16, 64, 256), 3,
                     run_cfg(Algorithm::easyspec, 4, chain4, 2, 3.0f, 48, 1), "the quick brown fox"});
    cases.push_back({"t3_chain_sd", tiny(8, 5, 32, 2, 16, 64, 256), 3,
                     run_cfg(Algorithm::sd, 4, chain4, 2, 3.0f, 48, 1), "the quick brown fox"});
    cases.push_back({"t15_chain_easyspec_d64", tiny(8, 21, 64, 4, 16, 128, 256), 4,
                     run_cfg(Algorithm::easyspec, 5, {1, 1, 1, 1, 1}, 4, 1.5f, 48, 2), "Zq8#k!pL2@xR9&mW"});
    cases.push_back({"t3_tree_easyspec", tiny(8, 7, 32, 2, 16, 64, 256), 4,
                     run_cfg(Algorithm::easyspec, 4, {2, 2, 1, 1}, 2, 3.0f, 48, 4), "tree search"});
    cases.push_back({"t3_tree_sd_tree", tiny(8, 7, 32, 2, 16, 64, 256), 4,
                     run_cfg(Algorithm::sd_tree, 4, {2, 2, 1, 1}, 2, 3.0f, 48, 4), "tree search"});
    cases.push_back({"t3_tree_nocal", tiny(8, 7, 32, 2, 16, 64, 256), 4,
                     run_cfg(Algorithm::easyspec, 4, {2, 2, 1, 1}, 2, 3.0f, 48, 4, false), "tree search"});

    {
        // A greedy tree whose first sibling IS rejected (independent drafter,
        // alpha < 1): the reference raises CheckError("sibling candidates
        // exhaust the draft distribution", proj/src/verifier.cpp:146-158).
        // Appended last so the earlier fixtures stay byte-identical.
        GenCase g{"greedy_tree_throws_indep", tiny(8, 11, 64, 4, 16, 128, 256), 5,
                  run_cfg(Algorithm::easyspec, 4, {2, 2, 1, 1}, 2, 0.0f, 24, 1), "independent"};
        g.draft_seed = 9;
        cases.push_back(g);
    }
    json gens = json::array();
    for (const auto& gc : cases) gens.push_back(run_case(gc));
    {
        std::ofstream f(out_dir + "/ref_generate.json");
        f << gens.dump() << "\n";
    }
    // criterion 2's configuration (proj/tests/acceptance_main.cpp:156-183):
    // prefix_distribution over 2000 runs of easyspec and vanilla, exact counts
    // (the per-run seeds are deterministic, so a bit-exact engine reproduces
    // every count, not just the law)
    {
        const Model base = init_model(tiny(4, 21));
        const Model draft = make_truncated_draft(base, 3);
        RunConfig rc = run_cfg(Algorithm::easyspec, 3, {2, 2, 2}, 2, 0.8f, 2, 11);
        const char* text = "easyspec";
        const std::span<const std::uint8_t> pr{reinterpret_cast<const std::uint8_t*>(text), 8};
        json pj = json::object();
        pj["runs"] = 2000;
        for (Algorithm a : {Algorithm::easyspec, Algorithm::vanilla}) {
            rc.algorithm = a;
            const auto dist = prefix_distribution(base, draft, rc, pr, 2000, 1);
            json e = json::array();
            for (const auto& [k, v] : dist) e.push_back(json{{"prefix", k}, {"count", v}});
            pj[to_string(a)] = e;
        }
        std::ofstream f(out_dir + "/ref_prefix.json");
        f << pj.dump() << "\n";
    }
    // per-iteration trees and outcomes of every speculative case, from the
    // stage-by-stage restatement pinned against generate()
    json stages = json::array();
    for (std::size_t i = 0; i < cases.size(); ++i) {
        if (cases[i].run.algorithm == Algorithm::vanilla) continue;
        json st = run_stages(cases[i]);
        const json& g = gens[i];
        if (st["error"] != g["error"] || (g["error"].is_null() && st["tokens"] != g["tokens"])) {
            std::cerr << "stage restatement diverges from generate() on " << cases[i].name << "\n";
            return 1;
        }
        stages.push_back(st);
    }
    {
        std::ofstream f(out_dir + "/ref_stages.json");
        f << stages.dump() << "\n";
    }
    // ---- host-side analysis API -----------------------------------
    //   report aggregation  -> aggregate / emit_report  proj/src/report.cpp:51-173
    //   similarity probe    -> probe_similarity         proj/src/draft_engine.cpp:291-372
    //   ESPEC1 model file   -> save_model / load_model  proj/src/model_io.cpp:76-190
    {
        json host;
        // Report aggregation over real traces of two generations; stage times
        // replaced by k * 2^-10 s (exactly representable as the engine's float
        // milliseconds) so both sides aggregate the same numbers bit for bit.
        json reps = json::array();
        for (const char* nm : {"fixa_easyspec", "t1_tree_wide", "t3_chain_easyspec", "fixa_vanilla"}) {
            const GenCase* gc = nullptr;
            for (const auto& c : cases)
                if (c.name == nm) gc = &c;
            const Model base = init_model(gc->base);
            const Model draft = gc->keep == 0 ? base : make_truncated_draft(base, gc->keep);
            const std::string& text = gc->prompt;
            const auto res = generate(base, draft, gc->run,
                                      std::span<const std::uint8_t>(
                                          reinterpret_cast<const std::uint8_t*>(text.data()), text.size()),
                                      nullptr);
            std::vector<IterationTrace> tr = res.report.iterations;
            json jt = json::array();
            for (std::size_t i = 0; i < tr.size(); ++i) {
                auto& t = tr[i];
                t.draft_wall = t.draft_sim = double((i * 7) % 13 + 1) / 1024.0;
                t.verify_wall = t.verify_sim = double((i * 5) % 11 + 3) / 1024.0;
                t.calibrate_wall = t.calibrate_sim = gc->run.algorithm == Algorithm::vanilla
                                                         ? 0.0
                                                         : double(i % 3 + 1) / 1024.0;
                jt.push_back(json{{"m", t.m}, {"n", t.n}, {"drafted_nodes", t.drafted_nodes},
                                  {"emitted", t.emitted}, {"draft", t.draft_wall}, {"verify", t.verify_wall},
                                  {"calibrate", t.calibrate_wall}, {"sequential_forwards", t.sequential_forwards},
                                  {"fuzzy_forwards", t.fuzzy_forwards}, {"base_forwards", t.base_forwards}});
            }
            const double vanilla = 0.0185546875 * static_cast<double>(res.tokens.size());
            RunReport r = aggregate(tr, vanilla);
            r.algorithm = to_string(gc->run.algorithm);
            r.n = gc->run.n;
            r.widths = gc->run.effective_widths();
            r.lp_size = gc->run.lp_size;
            reps.push_back(json{{"case", nm}, {"algorithm", r.algorithm}, {"n", r.n}, {"widths", r.widths},
                                {"lp_size", r.lp_size}, {"vanilla_baseline", vanilla}, {"traces", jt},
                                {"has_alpha", r.has_alpha}, {"alpha", r.alpha},
                                {"tokens_emitted", r.tokens_emitted},
                                {"tokens_per_s_wall", r.tokens_per_s_wall},
                                {"per100", {r.per100_wall.draft, r.per100_wall.verify, r.per100_wall.calibrate}},
                                {"draft_total_per100", r.draft_total_per100_sim}, {"total", r.total_sim},
                                {"speedup", r.speedup_vs_vanilla}, {"csv", emit_report(r, ReportFormat::csv)}});
        }
        {
            bool threw = false;
            try {
                aggregate(std::vector<IterationTrace>{}, 1.0);
            } catch (const ConfigError& e) {
                threw = true;
                host["empty_error"] = e.what();
            }
            if (!threw) return 1;
            IterationTrace z;
            try {
                aggregate(std::vector<IterationTrace>{z}, 1.0);
            } catch (const ConfigError& e) {
                host["zero_error"] = e.what();
            }
        }
        host["reports"] = reps;
        // Similarity probe (Table 4): a 9-layer drafter, lp 1..4 and an explicit
        // corpus of two sequences.
        {
            const Model dm = init_model(tiny(9, 45));
            const std::vector<std::vector<Token>> corpus = {bos_bytes("layer parallel drafting"),
                                                            bos_bytes("fuzzy")};
            const std::vector<int> lps = {1, 2, 3, 4};
            const auto rows = probe_similarity(dm, lps, corpus);
            json jr = json::array();
            for (const auto& r : rows)
                jr.push_back(json{{"lp_size", r.lp_size}, {"h", r.h}, {"q", r.q}, {"k", r.k}, {"v", r.v},
                                  {"attn_out", r.attn_out}});
            json jc = json::array();
            for (const auto& c : corpus) jc.push_back(c);
            host["similarity"] = json{{"config", cfg_json(dm.config)}, {"lp_sizes", lps}, {"corpus", jc},
                                      {"rows", jr}, {"csv", similarity_csv(rows)}};
        }
        // ESPEC1 file written by the reference's save_model, plus what
        // load_model makes of it (a greedy generation to replay after loading).
        {
            ModelConfig mc = tiny(3, 31, 16, 2, 8, 32, 64);
            const Model m = init_model(mc);
            save_model(m, out_dir + "/ref_tiny.espec1");
            const Model back = load_model(out_dir + "/ref_tiny.espec1");
            const Model dr = make_truncated_draft(back, 2);
            RunConfig rc = run_cfg(Algorithm::easyspec, 3, {2, 1, 1}, 2, 0.8f, 16, 5);
            const std::string text = "espec1";
            const auto res = generate(back, dr, rc,
                                      std::span<const std::uint8_t>(
                                          reinterpret_cast<const std::uint8_t*>(text.data()), text.size()),
                                      nullptr);
            host["model_file"] = json{{"file", "ref_tiny.espec1"}, {"config", cfg_json(mc)},
                                      {"embedding_sum", tensor_sum(back.weights.embedding)},
                                      {"w_down_2_sum", tensor_sum(back.weights.layers[2].w_down)},
                                      {"prompt", text}, {"keep", 2}, {"run", json{{"n", 3}, {"widths", {2, 1, 1}}, {"lp_size", 2},
                                                                  {"temperature", 0.8}, {"max_new_tokens", 16},
                                                                  {"seed", 5}}},
                                      {"tokens", res.tokens}};
        }
        std::ofstream f(out_dir + "/ref_hostapi.json");
        f << host.dump() << "\n";
    }
    // ---- cost simulator -> proj/src/cost_sim.cpp, the sim
    // fields of every generation's traces and report (orchestrator.cpp:72-77,
    // 256-466; report.cpp:51-95)
    {
        json cost;
        auto pj = [](const CostParams& p) {
            return json{{"c_fixed", p.c_fixed}, {"c_mem", p.c_mem}, {"c_comp", p.c_comp}, {"t_addi", p.t_addi},
                        {"attn_workload", p.attn_workload}, {"mlp_workload", p.mlp_workload},
                        {"base_layer_workload", p.base_layer_workload}, {"tp_size_base", p.tp_size_base},
                        {"tp_size_draft", p.tp_size_draft}, {"devices", p.devices}};
        };
        CostParams p0;
        CostParams p1;
        p1.c_fixed = 0.05;
        p1.c_mem = 0.7;
        p1.c_comp = 0.3;
        p1.t_addi = 0.25;
        p1.attn_workload = 0.2;
        p1.mlp_workload = 0.08;
        p1.base_layer_workload = 1.5;
        p1.tp_size_base = 4;
        p1.tp_size_draft = 2;
        p1.devices = 4;
        CostParams p2;
        p2.tp_size_base = 1;
        p2.devices = 1;
        json fns = json::array();
        for (const CostParams* pp : {&p0, &p1, &p2}) {
            const CostParams& p = *pp;
            json f;
            f["params"] = pj(p);
            json te = json::array();
            for (double w : {0.0, 0.15, 2.0})
                for (double sv : {1.0, 3.0, 7.5})
                    for (int tp : {1, 2, 8}) te.push_back(json{w, sv, tp, t_exe(p, w, sv, tp)});
            f["t_exe"] = te;
            json ga = json::array();
            for (int g : {1, 2, 4})
                for (double sv : {1.0, 2.5}) ga.push_back(json{g, sv, group_attention_time(p, g, sv)});
            f["group_attention"] = ga;
            json dg = json::array();
            for (const std::string& pl : {format_plan(plan_groups(32, 4)), format_plan(plan_groups(12, 2)),
                                          format_plan(plan_groups(8, 1)), std::string("0|1-3|4-7|8"),
                                          std::string("0|1-5|6")})
                for (double sv : {1.0, 6.0}) {
                    try {
                        dg.push_back(json{pl, sv, simulate_draft_group(p, parse_plan_override(pl), sv)});
                    } catch (const Error& e) {
                        dg.push_back(json{pl, sv, e.what()});
                    }
                }
            f["draft_group"] = dg;
            json sq = json::array(), bf = json::array(), vb = json::array();
            for (int L : {1, 8, 32})
                for (double sv : {1.0, 5.0}) {
                    sq.push_back(json{L, sv, sequential_draft_forward_time(p, L, sv)});
                    bf.push_back(json{L, sv, base_forward_time(p, L, sv)});
                }
            for (int pl : {0, 1, 20})
                for (long tk : {0L, 1L, 48L}) vb.push_back(json{12, pl, tk, vanilla_baseline_sim(p, 12, pl, tk)});
            f["sequential"] = sq;
            f["base"] = bf;
            f["vanilla_baseline"] = vb;
            fns.push_back(f);
        }
        cost["functions"] = fns;
        json tt = json::array();
        for (double al : {0.25, 0.8, 1.0}) tt.push_back(json{128.0, 0.3, 2.5, 5, al, total_time_model(128.0, 0.3, 2.5, 5, al)});
        cost["total_time"] = tt;
        // error texts
        json errs;
        auto catch_text = [](auto&& f) -> std::string {
            try {
                f();
            } catch (const Error& e) {
                return e.what();
            }
            return std::string();
        };
        {
            CostParams b = p0;
            b.c_mem = -1.0;
            errs["negative"] = catch_text([&] { b.validate(); });
            CostParams c = p0;
            c.tp_size_base = 0;
            errs["tp_zero"] = catch_text([&] { c.validate(); });
            CostParams d = p0;
            d.tp_size_draft = 9;
            errs["tp_over"] = catch_text([&] { d.validate(); });
            errs["t_exe_s"] = catch_text([&] { t_exe(p0, 0.1, 0.5, 1); });
            errs["group_zero"] = catch_text([&] { group_attention_time(p0, 0, 1.0); });
            errs["plan_over"] = catch_text([&] { simulate_draft_group(p1, parse_plan_override("0|1-5|6"), 1.0); });
            errs["alpha_zero"] = catch_text([&] { total_time_model(10, 1, 1, 2, 0.0); });
            errs["alpha_over"] = catch_text([&] { total_time_model(10, 1, 1, 2, 1.5); });
            errs["n_zero"] = catch_text([&] { total_time_model(10, 1, 1, 0, 0.5); });
        }
        cost["errors"] = errs;
        // every generation case's simulated stage units, occupancy and report,
        // at the default cost and (three cases) at p1
        json runs = json::array();
        for (const auto& gc : cases) {
            for (int variant = 0; variant < 2; ++variant) {
                if (variant == 1 && gc.name != "fixa_easyspec" && gc.name != "t3_chain_easyspec" &&
                    gc.name != "fixa_sd")
                    continue;
                const Model base = init_model(gc.base);
                Model draft;
                if (gc.draft_seed != 0) {
                    ModelConfig dc = gc.base;
                    dc.n_layers = gc.keep;
                    dc.seed = gc.draft_seed;
                    draft = init_model(dc);
                } else {
                    draft = gc.keep == 0 ? base : make_truncated_draft(base, gc.keep);
                }
                RunConfig rc = gc.run;
                if (variant == 1) rc.cost = p1;
                json r{{"name", gc.name}, {"cost", pj(rc.cost)}};
                try {
                    const GenerateResult res = generate(
                        base, draft, rc, {reinterpret_cast<const std::uint8_t*>(gc.prompt.data()), gc.prompt.size()},
                        nullptr);
                    json sims = json::array();
                    for (const auto& t : res.report.iterations)
                        sims.push_back(json{t.calibrate_sim, t.draft_sim, t.verify_sim});
                    const int prompt_len = static_cast<int>(tokenize_prompt(
                        {reinterpret_cast<const std::uint8_t*>(gc.prompt.data()), gc.prompt.size()},
                        base.config.vocab_size).size());
                    r["sims"] = sims;
                    r["prompt_len"] = prompt_len;
                    r["n_tokens"] = res.tokens.size();
                    r["vanilla_baseline"] = vanilla_baseline_sim(rc.cost, base.config.n_layers, prompt_len,
                                                                 static_cast<long>(res.tokens.size()));
                    r["per100_sim"] = {res.report.per100_sim.draft, res.report.per100_sim.verify,
                                       res.report.per100_sim.calibrate};
                    r["draft_total_per100_sim"] = res.report.draft_total_per100_sim;
                    r["total_sim"] = res.report.total_sim;
                    r["speedup"] = res.report.speedup_vs_vanilla;
                    r["csv"] = emit_report(res.report, ReportFormat::csv);
                    r["occupancy"] = res.occupancy_csv;
                    r["error"] = nullptr;
                } catch (const Error& e) {
                    r["error"] = e.what();
                }
                runs.push_back(r);
            }
        }
        // a plan wider than the simulated device count fails the run
        {
            const GenCase* gc = nullptr;
            for (const auto& c : cases)
                if (c.name == "fixa_easyspec") gc = &c;
            const Model base = init_model(gc->base);
            const Model draft = make_truncated_draft(base, gc->keep);
            RunConfig rc = gc->run;
            rc.cost.devices = 1;
            rc.cost.tp_size_base = 1;
            json r{{"name", "fixa_easyspec"}, {"cost", pj(rc.cost)}};
            r["error"] = catch_text([&] {
                generate(base, draft, rc,
                         {reinterpret_cast<const std::uint8_t*>(gc->prompt.data()), gc->prompt.size()}, nullptr);
            });
            runs.push_back(r);
        }
        cost["runs"] = runs;
        std::ofstream f(out_dir + "/ref_cost.json");
        f << cost.dump() << "\n";
    }
    std::cout << "wrote " << out_dir << "/ref_numerics.json and ref_generate.json (" << cases.size()
              << " generation cases)\n";
    return 0;
}
