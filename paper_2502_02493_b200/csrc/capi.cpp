// extern "C" boundary (include/espec_c.h) over the C++ engine.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/espec_c.h"
#include "engine.h"
#include "cost_sim.h"
#include "host_api.h"

using namespace espec;

struct espec_engine {
    std::unique_ptr<Engine> impl;
    std::string err;
    int vocab = 0;
    ModelCfg cfg[2];  // drafter, base
};

static thread_local std::string g_create_error;

namespace {

ModelCfg to_model(const espec_model_cfg* c) {
    ModelCfg m;
    m.vocab_size = c->vocab_size;
    m.d_model = c->d_model;
    m.n_layers = c->n_layers;
    m.n_heads = c->n_heads;
    m.n_kv_heads = c->n_kv_heads > 0 ? c->n_kv_heads : c->n_heads;
    m.d_head = c->d_head;
    m.d_mlp = c->d_mlp;
    m.max_positions = c->max_positions;
    m.norm_eps = c->norm_eps;
    m.rope_theta = c->rope_theta > 0 ? c->rope_theta : 10000.f;
    m.tied_head = c->tied_head;
    m.weight_dtype = c->weight_dtype;
    m.kv_dtype = c->kv_dtype;
    m.seed = c->seed;
    return m;
}

RunCfg to_run(const espec_run_cfg* r) {
    RunCfg c;
    c.algorithm = r->algorithm;
    c.n = r->n;
    if (r->widths)
        for (int i = 0; i < r->n; ++i) c.widths.push_back(r->widths[i]);
    c.lp_size = r->lp_size;
    c.plan_override = r->plan_override ? r->plan_override : "";
    c.temperature = r->temperature;
    c.max_new_tokens = r->max_new_tokens;
    c.seed = r->seed;
    c.calibration = r->calibration;
    c.strict_greedy_tree = r->strict_greedy_tree;
    return c;
}

void fill_trace(const IterationTrace& t, espec_iteration* o) {
    o->m = t.m;
    o->n = t.n;
    o->drafted_nodes = t.drafted_nodes;
    o->emitted = t.emitted;
    o->sequential_forwards = t.sequential_forwards;
    o->fuzzy_forwards = t.fuzzy_forwards;
    o->base_forwards = t.base_forwards;
    o->committed = t.committed;
    o->draft_committed = t.draft_committed;
    o->base_committed = t.base_committed;
    o->bonus = t.bonus;
    o->calibrate_ms = t.calibrate_ms;
    o->draft_ms = t.draft_ms;
    o->verify_ms = t.verify_ms;
    o->calibrate_sim = t.calibrate_sim;
    o->draft_sim = t.draft_sim;
    o->verify_sim = t.verify_sim;
}

template <typename F>
espec_status guard(espec_engine* e, F&& f) {
    if (!e) return ESPEC_CONFIG;
    try {
        f();
        e->err.clear();
        return ESPEC_OK;
    } catch (const Error& x) {
        e->err = x.what();
        return (espec_status)x.status;
    } catch (const espec_dev::DevError& x) {
        e->err = x.what();
        return (espec_status)x.code;
    } catch (const std::exception& x) {
        e->err = x.what();
        return ESPEC_CHECK;
    }
}

template <typename F>
espec_status guard_free(F&& f) {
    try {
        f();
        g_create_error.clear();
        return ESPEC_OK;
    } catch (const Error& x) {
        g_create_error = x.what();
        return (espec_status)x.status;
    } catch (const std::exception& x) {
        g_create_error = x.what();
        return ESPEC_CHECK;
    }
}

IterationTrace from_c(const espec_iteration& o) {
    IterationTrace t;
    t.m = o.m;
    t.n = o.n;
    t.drafted_nodes = o.drafted_nodes;
    t.emitted = o.emitted;
    t.sequential_forwards = o.sequential_forwards;
    t.fuzzy_forwards = o.fuzzy_forwards;
    t.base_forwards = o.base_forwards;
    t.committed = o.committed;
    t.draft_committed = o.draft_committed;
    t.base_committed = o.base_committed;
    t.bonus = o.bonus;
    t.calibrate_ms = o.calibrate_ms;
    t.draft_ms = o.draft_ms;
    t.verify_ms = o.verify_ms;
    t.calibrate_sim = o.calibrate_sim;
    t.draft_sim = o.draft_sim;
    t.verify_sim = o.verify_sim;
    return t;
}

espec_status copy_plan(const LayerPlan& p, char* out, int out_len) {
    const std::string s = format_plan(p);
    if ((int)s.size() + 1 > out_len) return ESPEC_SHAPE;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return ESPEC_OK;
}

}  // namespace

extern "C" {

espec_status espec_engine_create(const espec_model_cfg* base, const espec_model_cfg* draft, const espec_run_cfg* run,
                                 const espec_device_map* devices, espec_engine** out) {
    if (!base || !draft || !run || !out) return ESPEC_CONFIG;
    *out = nullptr;
    try {
        const int tp = devices && devices->tp_size > 0 ? devices->tp_size : 1;
        const int rank = devices ? devices->tp_rank : 0;
        // n_lp_devices > 1: the drafter's layer-parallel placement over the
        // group's GPUs (group slot j -> lp_devices[j] = rank j); 0 / 1: the
        // drafter is tensor-parallel like the base
        bool draft_lp = false;
        if (devices && devices->n_lp_devices > 1) {
            if (devices->n_lp_devices != tp)
                throw Error(ST_CONFIG, "layer-parallel placement spans the tensor-parallel group: n_lp_devices must "
                                       "equal tp_size");
            if (!devices->lp_devices) throw Error(ST_CONFIG, "lp_devices is NULL");
            for (int j = 0; j < tp; ++j)
                if (devices->lp_devices[j] != j)
                    throw Error(ST_CONFIG, "lp_devices must list the group's ranks in order (slot j -> rank j)");
            draft_lp = true;
        }
        auto e = new espec_engine();
        try {
            e->impl = make_engine(to_model(base), to_model(draft), to_run(run), devices ? devices->device : 0, tp, rank,
                                  draft_lp);
        } catch (...) {
            delete e;
            throw;
        }
        e->vocab = base->vocab_size;
        e->cfg[0] = to_model(draft);
        e->cfg[1] = to_model(base);
        *out = e;
        g_create_error.clear();
        return ESPEC_OK;
    } catch (const Error& x) {
        g_create_error = x.what();
        return (espec_status)x.status;
    } catch (const espec_dev::DevError& x) {
        g_create_error = x.what();
        return (espec_status)x.code;
    } catch (const std::exception& x) {
        g_create_error = x.what();
        return ESPEC_CHECK;
    }
}

void espec_engine_destroy(espec_engine* eng) { delete eng; }

espec_status espec_comm_link(espec_engine** engines, int world) {
    if (!engines || world < 1) return ESPEC_CONFIG;
    std::vector<Engine*> group;
    for (int i = 0; i < world; ++i) {
        if (!engines[i]) return ESPEC_CONFIG;
        group.push_back(engines[i]->impl.get());
    }
    for (int i = 0; i < world; ++i) {
        const espec_status st = guard(engines[i], [&] { engines[i]->impl->comm_link(group); });
        if (st != ESPEC_OK) return st;
    }
    return ESPEC_OK;
}

espec_status espec_comm_loopback(espec_engine* eng) {
    return guard(eng, [&] { eng->impl->comm_loopback(); });
}

espec_status espec_comm_export(espec_engine* eng, void* handle64) {
    return guard(eng, [&] { eng->impl->comm_ipc_export(handle64); });
}

espec_status espec_comm_import(espec_engine* eng, const void* handles, int world) {
    return guard(eng, [&] { eng->impl->comm_ipc_import(handles, world); });
}
const char* espec_last_error(const espec_engine* eng) { return eng ? eng->err.c_str() : g_create_error.c_str(); }
const char* espec_create_error(void) { return g_create_error.c_str(); }

espec_status espec_init_weights_seeded(espec_engine* eng, int which, uint64_t seed, int parity_mode) {
    return guard(eng, [&] { eng->impl->init_weights_seeded(which, seed, parity_mode != 0); });
}

espec_status espec_share_truncated_draft(espec_engine* eng) {
    return guard(eng, [&] { eng->impl->share_truncated_draft(); });
}

espec_status espec_load_tensor(espec_engine* eng, int which, const char* name, int layer, const float* data,
                               int64_t rows, int64_t cols) {
    return guard(eng, [&] { eng->impl->load_tensor(which, name, layer, data, rows, cols); });
}

espec_status espec_read_tensor(espec_engine* eng, int which, const char* name, int layer, float* out, int64_t rows,
                               int64_t cols) {
    return guard(eng, [&] { eng->impl->weight(which, name, layer, out, rows, cols); });
}

espec_status espec_set_run(espec_engine* eng, const espec_run_cfg* run) {
    return guard(eng, [&] { eng->impl->set_run(to_run(run)); });
}

espec_status espec_generate(espec_engine* eng, const uint8_t* prompt, int prompt_len, int32_t* out_tokens, int* n_out,
                            espec_iteration* traces, int* n_iters) {
    return guard(eng, [&] {
        std::vector<int> toks = {256};  // BOS (proj/src/orchestrator.cpp:42-52)
        for (int i = 0; i < prompt_len; ++i) toks.push_back(prompt[i]);
        std::vector<IterationTrace> tr;
        const std::vector<int> out = eng->impl->generate(toks, &tr);
        for (size_t i = 0; i < out.size(); ++i) out_tokens[i] = out[i];
        if (n_out) *n_out = (int)out.size();
        if (traces)
            for (size_t i = 0; i < tr.size(); ++i) fill_trace(tr[i], &traces[i]);
        if (n_iters) *n_iters = (int)tr.size();
    });
}

espec_status espec_begin(espec_engine* eng, const int32_t* tokens, int n_tokens) {
    return guard(eng, [&] { eng->impl->begin(std::vector<int>(tokens, tokens + n_tokens)); });
}

espec_status espec_step(espec_engine* eng, int32_t* emitted, int* n_emitted, espec_iteration* trace) {
    return guard(eng, [&] {
        std::vector<int> em;
        const IterationTrace t = eng->impl->step(em);
        for (size_t i = 0; i < em.size(); ++i) emitted[i] = em[i];
        if (n_emitted) *n_emitted = (int)em.size();
        if (trace) fill_trace(t, trace);
    });
}

int espec_done(const espec_engine* eng) { return eng && eng->impl->done() ? 1 : 0; }

espec_status espec_cache_view(espec_engine* eng, int which, int layer, int row0, int n, float* k, float* v,
                              int* committed_len) {
    return guard(eng, [&] {
        const int c = n > 0 ? eng->impl->cache_rows(which, layer, row0, n, k, v) : eng->impl->cache_committed(which);
        if (committed_len) *committed_len = c;
    });
}

espec_status espec_committed(espec_engine* eng, int32_t* tokens, int cap, int* n) {
    return guard(eng, [&] {
        const auto& c = eng->impl->committed();
        const int k = std::min<int>(cap, (int)c.size());
        for (int i = 0; i < k; ++i) tokens[i] = c[i];
        if (n) *n = (int)c.size();
    });
}

espec_status espec_forward(espec_engine* eng, int which, const int32_t* tokens, int n, const char* plan, float* logits,
                           float* hidden) {
    return guard(eng, [&] {
        eng->impl->forward_chain(which, std::vector<int>(tokens, tokens + n), plan ? plan : "", logits, hidden);
    });
}

espec_status espec_forward_tree(espec_engine* eng, int which, const int32_t* prompt, int n_prompt,
                                const int32_t* tokens, const int32_t* parents, int n, const char* plan, float* logits,
                                float* hidden) {
    return guard(eng, [&] {
        if (!prompt || !tokens || !parents) throw Error(ST_CONFIG, "forward_tree: null input");
        eng->impl->forward_tree(which, std::vector<int>(prompt, prompt + n_prompt), std::vector<int>(tokens, tokens + n),
                                std::vector<int>(parents, parents + n), plan ? plan : "", logits, hidden);
    });
}

espec_status espec_plan_groups(int n_layers, int lp_size, char* out, int out_len) {
    try {
        return copy_plan(plan_groups(n_layers, lp_size), out, out_len);
    } catch (const Error& x) {
        g_create_error = x.what();
        return (espec_status)x.status;
    }
}

espec_status espec_parse_plan(const char* spec, char* out, int out_len) {
    try {
        return copy_plan(parse_plan_override(spec ? spec : ""), out, out_len);
    } catch (const Error& x) {
        g_create_error = x.what();
        return (espec_status)x.status;
    }
}

int espec_kernel_launches(const espec_engine* eng) { return eng ? eng->impl->kernel_launches() : 0; }
void espec_reset_kernel_launches(espec_engine* eng) {
    if (eng) eng->impl->reset_launch_count();
}
void* espec_stream(espec_engine* eng) { return eng ? eng->impl->stream() : nullptr; }

espec_status espec_time_site(espec_engine* eng, int which, int kind) {
    return guard(eng, [&] { eng->impl->time_site(which, kind); });
}

espec_status espec_site_stats(espec_engine* eng, int* count, double* total_ms, double* bytes_per_launch) {
    return guard(eng, [&] { eng->impl->site_stats(count, total_ms, bytes_per_launch); });
}

espec_status espec_io_bytes(espec_engine* eng, int64_t* h2d, int64_t* d2h) {
    return guard(eng, [&] {
        long long a = 0, b = 0;
        eng->impl->io_bytes(&a, &b);
        *h2d = a;
        *d2h = b;
    });
}

espec_status espec_generate_tokens(espec_engine* eng, const int32_t* tokens, int n_tokens, int32_t* out_tokens,
                                   int* n_out, espec_iteration* traces, int* n_iters) {
    return guard(eng, [&] {
        std::vector<IterationTrace> tr;
        const std::vector<int> out = eng->impl->generate(std::vector<int>(tokens, tokens + n_tokens), &tr);
        for (size_t i = 0; i < out.size(); ++i) out_tokens[i] = out[i];
        if (n_out) *n_out = (int)out.size();
        if (traces)
            for (size_t i = 0; i < tr.size(); ++i) fill_trace(tr[i], &traces[i]);
        if (n_iters) *n_iters = (int)tr.size();
    });
}

espec_status espec_sync(espec_engine* eng) {
    return guard(eng, [&] { eng->impl->sync(); });
}

}  // extern "C"

// ---- stage-level API
namespace {
void tree_to_c(const TreeOut& t, espec_tree* o, int vocab) {
    const int nn = (int)t.token.size();
    if (nn > ESPEC_MAX_NODES) throw Error(ST_SHAPE, "tree exceeds ESPEC_MAX_NODES");
    o->id = t.id;
    o->n_nodes = nn;
    o->root_children = t.root_children;
    o->n_levels = (int)t.widths.size();
    o->n_dists = t.n_dists;
    for (int i = 0; i < o->n_levels && i < ESPEC_MAX_NODES; ++i) o->widths[i] = t.widths[i];
    for (int j = 0; j < nn; ++j) {
        o->token[j] = t.token[j];
        o->parent[j] = t.parent[j];
        o->depth[j] = t.depth[j];
        o->prob_index[j] = t.prob_index[j];
        o->cache_row[j] = t.cache_row[j];
        o->first_child[j] = t.first_child[j];
        o->n_children[j] = t.n_children[j];
    }
    if (o->dists) {
        if (o->dist_capacity < t.n_dists) throw Error(ST_SHAPE, "dist buffer holds fewer rows than the tree's dists");
        std::memcpy(o->dists, t.dists.data(), sizeof(float) * (size_t)t.n_dists * vocab);
    }
}
TreeOut tree_from_c(const espec_tree* c) {
    if (c->n_nodes < 0 || c->n_nodes > ESPEC_MAX_NODES) throw Error(ST_SHAPE, "tree node count out of range");
    TreeOut t;
    t.id = c->id;
    t.token.assign(c->token, c->token + c->n_nodes);
    t.parent.assign(c->parent, c->parent + c->n_nodes);
    return t;
}
}  // namespace

extern "C" {

espec_status espec_prefill(espec_engine* eng, const int32_t* tokens, int n_tokens) {
    return guard(eng, [&] {
        if (!tokens || n_tokens <= 0) throw Error(ST_CONFIG, "empty prompt");
        eng->impl->prefill(std::vector<int>(tokens, tokens + n_tokens));
    });
}

espec_status espec_calibrate(espec_engine* eng, float* root_logits) {
    return guard(eng, [&] { eng->impl->calibrate(root_logits); });
}

espec_status espec_draft(espec_engine* eng, espec_tree* tree) {
    return guard(eng, [&] {
        if (!tree) {
            eng->impl->draft(nullptr, false);
            return;
        }
        TreeOut t;
        eng->impl->draft(&t, tree->dists != nullptr);
        tree_to_c(t, tree, eng->vocab);
    });
}

espec_status espec_verify(espec_engine* eng, const espec_tree* tree, espec_outcome* outcome) {
    return guard(eng, [&] {
        OutcomeOut o;
        if (tree) {
            const TreeOut t = tree_from_c(tree);
            eng->impl->verify(&t, &o);
        } else {
            eng->impl->verify(nullptr, &o);
        }
        if (outcome) {
            outcome->id = o.id;
            outcome->m = o.m;
            outcome->n = o.n;
            outcome->bonus = o.bonus;
            for (int i = 0; i < o.m; ++i) {
                outcome->accepted_path[i] = o.path[i];
                outcome->accepted_tokens[i] = o.tokens[i];
            }
        }
    });
}

espec_status espec_resolve_draft_cache(espec_engine* eng, const espec_outcome* outcome) {
    return guard(eng, [&] {
        if (!outcome) {
            eng->impl->resolve_draft_cache(nullptr);
            return;
        }
        if (outcome->m < 0 || outcome->m > ESPEC_MAX_NODES) throw Error(ST_SHAPE, "outcome m out of range");
        OutcomeOut o;
        o.id = outcome->id;
        o.m = outcome->m;
        o.path.assign(outcome->accepted_path, outcome->accepted_path + outcome->m);
        eng->impl->resolve_draft_cache(&o);
    });
}

espec_status espec_commit_outcome(espec_engine* eng, int32_t* emitted, int* n_emitted, espec_iteration* trace) {
    return guard(eng, [&] {
        std::vector<int> em;
        const IterationTrace t = eng->impl->commit_outcome(em);
        if (emitted)
            for (size_t i = 0; i < em.size(); ++i) emitted[i] = em[i];
        if (n_emitted) *n_emitted = (int)em.size();
        if (trace) fill_trace(t, trace);
    });
}

}  // extern "C"

extern "C" {

espec_status espec_prefix_distribution(espec_engine* eng, const int32_t* tokens, int n_tokens, int64_t runs,
                                       int64_t first_run, int64_t run_stride, int32_t* prefixes, int64_t* counts,
                                       int cap, int* n_distinct) {
    return guard(eng, [&] {
        if (!tokens || n_tokens <= 0) throw Error(ST_CONFIG, "empty prompt");
        const auto dist = eng->impl->prefix_distribution(std::vector<int>(tokens, tokens + n_tokens), (long)runs,
                                                         (long)first_run, (long)run_stride);
        if (n_distinct) *n_distinct = (int)dist.size();
        if ((int)dist.size() > cap) throw Error(ST_SHAPE, "prefix buffer holds fewer entries than distinct prefixes");
        size_t len = 0;
        int i = 0;
        for (const auto& kv : dist) {
            if (i == 0) len = kv.first.size();
            if (kv.first.size() != len) throw Error(ST_CHECK, "prefixes of different lengths");
            for (size_t j = 0; j < len; ++j) prefixes[(size_t)i * len + j] = kv.first[j];
            counts[i++] = kv.second;
        }
    });
}

double espec_total_variation(const int32_t* pa, const int64_t* ca, int na, const int32_t* pb, const int64_t* cb,
                             int nb, int len, int64_t runs_a, int64_t runs_b) {
    // total_variation (orchestrator.cpp:528-553): both lists in lexicographic order
    if (runs_a <= 0 || runs_b <= 0 || len <= 0) return -1.0;
    auto less = [len](const int32_t* x, const int32_t* y) {
        return std::lexicographical_compare(x, x + len, y, y + len);
    };
    double dist = 0.0;
    int i = 0, j = 0;
    while (i < na || j < nb) {
        double a = 0.0, b = 0.0;
        if (j == nb || (i < na && less(pa + (size_t)i * len, pb + (size_t)j * len))) {
            a = (double)ca[i++] / (double)runs_a;
        } else if (i == na || less(pb + (size_t)j * len, pa + (size_t)i * len)) {
            b = (double)cb[j++] / (double)runs_b;
        } else {
            a = (double)ca[i++] / (double)runs_a;
            b = (double)cb[j++] / (double)runs_b;
        }
        dist += a > b ? a - b : b - a;
    }
    return dist / 2.0;
}

espec_status espec_aggregate(const espec_iteration* traces, int n_traces, double vanilla_baseline_sim,
                             espec_report* out) {
    if (!out || (n_traces > 0 && !traces)) return ESPEC_CONFIG;
    return guard_free([&] {
        std::vector<IterationTrace> t;
        for (int i = 0; i < n_traces; ++i) t.push_back(from_c(traces[i]));
        const ReportAgg r = aggregate_traces(t, vanilla_baseline_sim);
        out->n_iterations = r.iterations;
        out->has_alpha = r.has_alpha;
        out->alpha = r.alpha;
        out->tokens_emitted = r.tokens_emitted;
        out->mean_accept_len = r.mean_accept_len;
        out->tokens_per_s = r.tokens_per_s;
        out->draft_per_100_s = r.draft_per100;
        out->verify_per_100_s = r.verify_per100;
        out->calibrate_per_100_s = r.calibrate_per100;
        out->draft_total_per_100_s = r.draft_total_per100;
        out->total_s = r.total;
        out->speedup_vs_vanilla = r.speedup_vs_vanilla;
        out->draft_per_100_sim = r.draft_per100_sim;
        out->verify_per_100_sim = r.verify_per100_sim;
        out->calibrate_per_100_sim = r.calibrate_per100_sim;
        out->draft_total_per_100_sim = r.draft_total_per100_sim;
        out->total_sim = r.total_sim;
    });
}

espec_status espec_report_emit(const espec_report* report, const espec_iteration* traces, int n_traces,
                               const char* algorithm, int n, const int* widths, int n_widths, int lp_size,
                               int format, char* out, int cap, int* len) {
    if (!report || !algorithm || (n_traces > 0 && !traces) || (n_widths > 0 && !widths)) return ESPEC_CONFIG;
    return guard_free([&] {
        ReportAgg r;
        r.iterations = report->n_iterations;
        r.has_alpha = report->has_alpha != 0;
        r.alpha = report->alpha;
        r.tokens_emitted = (long)report->tokens_emitted;
        r.mean_accept_len = report->mean_accept_len;
        r.tokens_per_s = report->tokens_per_s;
        r.draft_per100 = report->draft_per_100_s;
        r.verify_per100 = report->verify_per_100_s;
        r.calibrate_per100 = report->calibrate_per_100_s;
        r.draft_total_per100 = report->draft_total_per_100_s;
        r.total = report->total_s;
        r.speedup_vs_vanilla = report->speedup_vs_vanilla;
        r.draft_per100_sim = report->draft_per_100_sim;
        r.verify_per100_sim = report->verify_per_100_sim;
        r.calibrate_per100_sim = report->calibrate_per_100_sim;
        r.draft_total_per100_sim = report->draft_total_per_100_sim;
        r.total_sim = report->total_sim;
        std::vector<IterationTrace> t;
        for (int i = 0; i < n_traces; ++i) t.push_back(from_c(traces[i]));
        std::string text;
        if (format == 1) text = report_csv(r, algorithm, n, lp_size);
        else if (format == 0) text = report_json(r, t, algorithm, n, std::vector<int>(widths, widths + n_widths), lp_size);
        else throw Error(ST_CONFIG, "report format must be 0 (json) or 1 (csv)");
        if (len) *len = (int)text.size();
        if (!out || (int)text.size() + 1 > cap) throw Error(ST_SHAPE, "report text does not fit the buffer");
        std::memcpy(out, text.c_str(), text.size() + 1);
    });
}

// ---- cost simulator (proj/src/cost_sim.cpp) -------------------------------
namespace {
CostParams cost_from_c(const espec_cost_params* c) {
    CostParams p;
    p.c_fixed = c->c_fixed;
    p.c_mem = c->c_mem;
    p.c_comp = c->c_comp;
    p.t_addi = c->t_addi;
    p.attn_workload = c->attn_workload;
    p.mlp_workload = c->mlp_workload;
    p.base_layer_workload = c->base_layer_workload;
    p.tp_size_base = c->tp_size_base;
    p.tp_size_draft = c->tp_size_draft;
    p.devices = c->devices;
    return p;
}
}  // namespace

espec_status espec_cost_defaults(espec_cost_params* out) {
    if (!out) return ESPEC_CONFIG;
    const CostParams d;
    *out = espec_cost_params{d.c_fixed,      d.c_mem,         d.c_comp,        d.t_addi,  d.attn_workload,
                             d.mlp_workload, d.base_layer_workload, d.tp_size_base, d.tp_size_draft, d.devices};
    return ESPEC_OK;
}

espec_status espec_cost_eval(const espec_cost_params* params, int what, double a, double b, int n_layers,
                             const char* plan, double* out) {
    if (!params || !out) return ESPEC_CONFIG;
    return guard_free([&] {
        const CostParams p = cost_from_c(params);
        switch (what) {
            case ESPEC_COST_VALIDATE: p.validate(); *out = 0.0; break;
            case ESPEC_COST_T_EXE: *out = t_exe(p, a, b, n_layers); break;
            case ESPEC_COST_GROUP_ATTENTION: *out = group_attention_time(p, n_layers, a); break;
            case ESPEC_COST_DRAFT_GROUP: {
                if (!plan) throw Error(ST_CONFIG, "cost: a layer plan is required");
                *out = simulate_draft_group(p, parse_plan_override(plan), a);
                break;
            }
            case ESPEC_COST_SEQUENTIAL_DRAFT: *out = sequential_draft_forward_time(p, n_layers, a); break;
            case ESPEC_COST_BASE_FORWARD: *out = base_forward_time(p, n_layers, a); break;
            case ESPEC_COST_VANILLA_BASELINE: *out = vanilla_baseline_sim(p, n_layers, (int)a, (long)b); break;
            default: throw Error(ST_CONFIG, "cost: unknown function " + std::to_string(what));
        }
    });
}

espec_status espec_cost_total_time(double n_tokens, double t_draft, double t_base, int n, double alpha, double* out) {
    if (!out) return ESPEC_CONFIG;
    return guard_free([&] { *out = total_time_model(n_tokens, t_draft, t_base, n, alpha); });
}

espec_status espec_set_cost(espec_engine* eng, const espec_cost_params* params) {
    if (!params) return ESPEC_CONFIG;
    return guard(eng, [&] { eng->impl->set_cost(cost_from_c(params)); });
}

espec_status espec_occupancy_csv(espec_engine* eng, char* out, int cap, int* len) {
    return guard(eng, [&] {
        const std::string text = eng->impl->occupancy_csv();
        if (len) *len = (int)text.size();
        if (!out || (int)text.size() + 1 > cap) throw Error(ST_SHAPE, "occupancy text does not fit the buffer");
        std::memcpy(out, text.c_str(), text.size() + 1);
    });
}

espec_status espec_model_file_config(const char* path, espec_model_cfg* cfg) {
    if (!path || !cfg) return ESPEC_CONFIG;
    return guard_free([&] {
        const ModelFileInfo info = read_model_file(path, true);
        const ModelCfg& m = info.cfg;
        cfg->vocab_size = m.vocab_size;
        cfg->d_model = m.d_model;
        cfg->n_layers = m.n_layers;
        cfg->n_heads = m.n_heads;
        cfg->n_kv_heads = m.n_kv_heads;
        cfg->d_head = m.d_head;
        cfg->d_mlp = m.d_mlp;
        cfg->max_positions = m.max_positions;
        cfg->norm_eps = m.norm_eps;
        cfg->rope_theta = m.rope_theta;
        cfg->tied_head = 1;
        cfg->weight_dtype = ESPEC_F32;
        cfg->kv_dtype = ESPEC_F32;
        cfg->seed = m.seed;
    });
}

espec_status espec_load_model_file(espec_engine* eng, int which, const char* path) {
    if (!path || which < 0 || which > 1) return ESPEC_CONFIG;
    return guard(eng, [&] { load_model_file(*eng->impl, which, eng->cfg[which], path); });
}

espec_status espec_save_model_file(espec_engine* eng, int which, const char* path) {
    if (!path || which < 0 || which > 1) return ESPEC_CONFIG;
    return guard(eng, [&] { save_model_file(*eng->impl, which, eng->cfg[which], path); });
}

espec_status espec_probe_similarity(espec_engine* eng, const int* lp_sizes, int n_lp, const int32_t* tokens,
                                    const int* offsets, int n_seqs, espec_similarity_row* rows) {
    if (!eng) return ESPEC_CONFIG;
    if ((n_lp > 0 && (!lp_sizes || !rows)) || (n_seqs > 0 && (!tokens || !offsets))) return ESPEC_CONFIG;
    return guard(eng, [&] {
        std::vector<std::vector<int>> corpus;
        for (int s = 0; s < n_seqs; ++s) {
            if (offsets[s + 1] <= offsets[s]) throw Error(ST_CONFIG, "similarity probe sequences must be non-empty");
            corpus.emplace_back(tokens + offsets[s], tokens + offsets[s + 1]);
        }
        const auto r = probe_similarity(*eng->impl, eng->cfg[0].n_layers, std::vector<int>(lp_sizes, lp_sizes + n_lp),
                                        corpus);
        for (size_t i = 0; i < r.size(); ++i) rows[i] = {r[i].lp_size, r[i].h, r[i].q, r[i].k, r[i].v, r[i].attn_out};
    });
}

}  // extern "C"
