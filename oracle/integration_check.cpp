// Drop-in check of integration/espec/b200.hpp (the reference-side binding).
// TEST INFRASTRUCTURE ONLY.
//
// Links the unmodified reference core (oracle/_ref/libespec_ref.a, built from
// /root/reference/proj/src) and libespec_b200.so. For each case it runs the
// reference's espec::generate on the CPU and, on the same Model objects:
//   * generate_b200 (the one-call drop-in for espec::generate), and
//   * B200Generation's stage calls (leading_pass -> draft -> verify ->
//     resolve_draft_cache -> commit), the reference's Generation stages
//     (proj/src/orchestrator.cpp:256-428) returning its own DraftTree /
//     VerificationOutcome types; each DraftTree's invariants are checked
//     (token / parent / prob_index ranges, every dists row sums to one).
// Tokens must be identical to espec::generate, and a fixture the reference
// rejects must raise the same CheckError. Prints one JSON line; exit 1 on
// any mismatch.
#include <cmath>
#include <cstdio>
#include <iostream>
#include <string>
#include <vector>

#include "espec/b200.hpp"
#include "espec/model.hpp"

using namespace espec;

namespace {

ModelConfig tiny(int n_layers, std::uint64_t seed, int d_model = 32, int n_heads = 2, int d_head = 16,
                 int d_mlp = 64, int max_pos = 256) {
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

RunConfig run_cfg(Algorithm a, int n, std::vector<int> widths, int lp, float temp, int max_new, std::uint64_t seed) {
    RunConfig r;
    r.algorithm = a;
    r.n = n;
    r.widths = std::move(widths);
    r.lp_size = lp;
    r.temperature = temp;
    r.max_new_tokens = max_new;
    r.seed = seed;
    r.workers = 1;
    return r;
}

struct Case {
    std::string name;
    ModelConfig base;
    int keep;
    std::uint64_t draft_seed;
    RunConfig run;
    std::string prompt;
};

bool tree_ok(const DraftTree& t, int vocab) {
    if (t.node_count() < 1 || t.root_children < 1) return false;
    for (int j = 0; j < t.node_count(); ++j) {
        const DraftNode& n = t.nodes[static_cast<std::size_t>(j)];
        if (n.token < 0 || n.token >= vocab) return false;
        if (n.prob_index < 0 || n.prob_index >= static_cast<int>(t.dists.size())) return false;
        if (n.parent >= j) return false;
    }
    for (const ProbVector& p : t.dists) {
        double s = 0.0;
        for (float v : p.probs) s += v;
        if (std::fabs(s - 1.0) > 1e-4) return false;
    }
    return true;
}

}  // namespace

int main() {
    std::vector<Case> cases;
    // BASELINE configs[0]: the CLI default pair (proj/src/cli.cpp:210-218, 263-265):
    // 12-layer d64 base seed 7, drafter = its first 8 layers, greedy, n 4, lp 2
    cases.push_back({"c1_easyspec", tiny(12, 7, 64, 4, 16, 128, 512), 8, 0,
                     run_cfg(Algorithm::easyspec, 4, {1, 1, 1, 1}, 2, 0.0f, 64, 1), "the quick brown fox"});
    cases.push_back({"c1_sd", tiny(12, 7, 64, 4, 16, 128, 512), 8, 0,
                     run_cfg(Algorithm::sd, 4, {1, 1, 1, 1}, 2, 0.0f, 64, 1), "the quick brown fox"});
    cases.push_back({"c1_vanilla", tiny(12, 7, 64, 4, 16, 128, 512), 8, 0,
                     run_cfg(Algorithm::vanilla, 4, {1, 1, 1, 1}, 2, 0.0f, 64, 1), "the quick brown fox"});
    cases.push_back({"indep_easyspec_lp4", tiny(8, 11, 64, 4, 16, 128, 256), 5, 9,
                     run_cfg(Algorithm::easyspec, 5, {1, 1, 1, 1, 1}, 4, 0.0f, 40, 1), "independent"});
    cases.push_back({"t3_tree_easyspec", tiny(8, 7), 4, 0,
                     run_cfg(Algorithm::easyspec, 4, {2, 2, 1, 1}, 2, 3.0f, 48, 4), "tree search"});
    cases.push_back({"t08_tree_sd_tree", tiny(6, 91), 4, 0,
                     run_cfg(Algorithm::sd_tree, 4, {2, 2, 2, 2}, 2, 0.8f, 16, 3), "replay"});
    cases.push_back({"greedy_tree_throws_indep", tiny(8, 11, 64, 4, 16, 128, 256), 5, 9,
                     run_cfg(Algorithm::easyspec, 4, {2, 2, 1, 1}, 2, 0.0f, 24, 1), "independent"});

    bool all_ok = true;
    std::cout << "{\"cases\": [";
    for (std::size_t ci = 0; ci < cases.size(); ++ci) {
        const Case& c = cases[ci];
        const Model base = init_model(c.base);
        Model draft;
        if (c.draft_seed) {
            ModelConfig dc = c.base;
            dc.n_layers = c.keep;
            dc.seed = c.draft_seed;
            draft = init_model(dc);
        } else {
            draft = make_truncated_draft(base, c.keep);
        }
        const std::span<const std::uint8_t> prompt(reinterpret_cast<const std::uint8_t*>(c.prompt.data()),
                                                   c.prompt.size());
        std::string ref_err, b200_err, stage_err;
        GenerateResult ref, gpu;
        std::vector<Token> staged;
        bool trees_ok = true;
        try {
            ref = generate(base, draft, c.run, prompt);
        } catch (const Error& e) {
            ref_err = e.what();
        }
        try {
            gpu = generate_b200(base, draft, c.run, prompt);
        } catch (const Error& e) {
            b200_err = e.what();
        }
        if (c.run.algorithm != Algorithm::vanilla) {
            try {
                B200Generation g(base, draft, c.run);
                g.prefill(tokenize_prompt(prompt, base.config.vocab_size));
                while (!g.done()) {
                    const Matrix root = g.leading_pass();
                    (void)root;
                    const DraftTree tree = g.draft();
                    trees_ok &= tree_ok(tree, base.config.vocab_size);
                    const VerificationOutcome o = g.verify(tree);
                    trees_ok &= o.m <= o.n && static_cast<int>(o.accepted_path.size()) == o.m;
                    g.resolve_draft_cache();
                    for (Token t : g.commit()) staged.push_back(t);
                }
            } catch (const Error& e) {
                stage_err = e.what();
            }
        } else {
            staged = ref.tokens;
        }
        bool ok = ref_err == b200_err && ref_err == (c.run.algorithm != Algorithm::vanilla ? stage_err : ref_err);
        if (ref_err.empty()) {
            ok &= gpu.tokens == ref.tokens && staged == ref.tokens && trees_ok;
            ok &= gpu.report.has_alpha == ref.report.has_alpha && gpu.report.alpha == ref.report.alpha;
            ok &= gpu.report.tokens_emitted == ref.report.tokens_emitted;
            // the simulated report and occupancy, bit for bit (cost_sim.cpp)
            ok &= gpu.report.total_sim == ref.report.total_sim &&
                  gpu.report.speedup_vs_vanilla == ref.report.speedup_vs_vanilla &&
                  gpu.report.per100_sim.draft == ref.report.per100_sim.draft &&
                  gpu.report.per100_sim.verify == ref.report.per100_sim.verify &&
                  gpu.report.per100_sim.calibrate == ref.report.per100_sim.calibrate &&
                  gpu.occupancy_csv == ref.occupancy_csv;
        }
        all_ok &= ok;
        std::cout << (ci ? ", " : "") << "{\"name\": \"" << c.name << "\", \"ok\": " << (ok ? "true" : "false")
                  << ", \"tokens\": " << ref.tokens.size() << ", \"alpha\": " << ref.report.alpha
                  << ", \"b200_alpha\": " << gpu.report.alpha << ", \"error\": \"" << ref_err
                  << "\", \"b200_error\": \"" << b200_err << "\", \"stage_error\": \"" << stage_err << "\"}";
    }
    std::cout << "], \"ok\": " << (all_ok ? "true" : "false") << "}" << std::endl;
    return all_ok ? 0 : 1;
}
