// CPU-baseline timer for the unmodified reference core. TEST/BASELINE
// INFRASTRUCTURE ONLY — used by bench.py's cpu_baseline leg and by
// `bench.py --impl reference`; never part of the product path.
//
// The reference cannot hold the BASELINE C2 models (70B fp32 = 282 GB) and
// requires equal base/draft widths (proj/src/orchestrator.cpp:114-117), so
// the large-shape numbers are a bounded sample: the reference's own per-layer
// body — rms_norm -> attention_forward -> add -> rms_norm -> mlp_forward -> add
// (forward_sequential, proj/src/draft_engine.cpp:35-62) plus build_tree_mask
// (proj/src/kv_cache.cpp:43-60) — timed on ONE layer at the real width, T
// rows, a committed context of `ctx` rows, then extrapolated by the caller.
// Weights are filled with a cheap deterministic pattern (timing does not
// depend on values; init_model's Box-Muller would take minutes at this size).
//
//   ref_bench layer <d_model> <n_heads> <d_head> <d_mlp> <T> <ctx> <reps>
//   ref_bench group <d_model> <n_heads> <d_head> <d_mlp> <g> <T> <ctx> <workers> <reps>
//       one fuzzy group of g layers through forward_fuzzy
//       (proj/src/draft_engine.cpp:64-133) with a WorkerPool of `workers`
//       threads (proj/src/worker_pool.cpp:27-50): the reference's own
//       layer-parallel executor
//   ref_bench head  <d_model> <vocab> <T> <reps>
//   ref_bench c1    <algorithm> <max_new_tokens> <reps>
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "espec/draft_engine.hpp"
#include "espec/kv_cache.hpp"
#include "espec/model.hpp"
#include "espec/orchestrator.hpp"
#include "espec/worker_pool.hpp"

using namespace espec;
using Clock = std::chrono::steady_clock;

static double ms_since(Clock::time_point t) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

static void fill(Matrix& m, uint32_t seed, float scale) {
    uint32_t s = seed * 2654435761u + 1u;
    for (float& v : m.data) {
        s ^= s << 13;
        s ^= s >> 17;
        s ^= s << 5;
        v = ((float)(s & 0xffff) / 65535.0f - 0.5f) * scale;
    }
}

static int cmd_layer(int argc, char** argv) {
    if (argc < 9) return 2;
    const int d = atoi(argv[2]), H = atoi(argv[3]), dh = atoi(argv[4]), f = atoi(argv[5]);
    const int T = atoi(argv[6]), ctx = atoi(argv[7]), reps = atoi(argv[8]);
    Model m;
    m.config.d_model = d;
    m.config.n_heads = H;
    m.config.d_head = dh;
    m.config.d_mlp = f;
    m.config.n_layers = 1;
    m.config.max_positions = ctx + T + 8;
    m.weights.layers.resize(1);
    auto& L = m.weights.layers[0];
    const float ps = 2.0f / std::sqrt((float)d);
    L.wq = Matrix(d, d); fill(L.wq, 1, ps);
    L.wk = Matrix(d, d); fill(L.wk, 2, ps);
    L.wv = Matrix(d, d); fill(L.wv, 3, ps);
    L.wo = Matrix(d, d); fill(L.wo, 4, ps);
    L.w_gate = Matrix(d, f); fill(L.w_gate, 5, ps);
    L.w_up = Matrix(d, f); fill(L.w_up, 6, ps);
    L.w_down = Matrix(f, d); fill(L.w_down, 7, 2.0f / std::sqrt((float)f));
    L.attn_norm_gain = Matrix(1, d);
    L.mlp_norm_gain = Matrix(1, d);
    for (float& v : L.attn_norm_gain.data) v = 1.f;
    for (float& v : L.mlp_norm_gain.data) v = 1.f;

    KvCache cache(1, d);
    if (ctx > 0) {
        std::vector<int> parents;
        for (int i = 0; i < ctx; ++i) parents.push_back(i == 0 ? kCommittedTail : i - 1);
        const auto rows = cache.stage_append(parents, false);
        Matrix k(ctx, d), v(ctx, d);
        fill(k, 8, 1.f);
        fill(v, 9, 1.f);
        cache.write_rows(0, rows, k, v);
        cache.commit_path(rows);
    }
    double best_mask = 1e30, best_attn = 1e30, best_mlp = 1e30, best_rest = 1e30;
    for (int r = 0; r < reps; ++r) {
        std::vector<int> parents;
        for (int i = 0; i < T; ++i) parents.push_back(i == 0 ? kCommittedTail : cache.committed_len() + i - 1);
        ForwardBatch batch;
        batch.flat_rows = cache.stage_append(parents, false);
        for (int row : batch.flat_rows) batch.positions.push_back(cache.position_of(row));
        auto t0 = Clock::now();
        const TreeMask mask = cache.build_tree_mask();
        const double t_mask = ms_since(t0);
        batch.mask = &mask;
        Matrix h(T, d);
        fill(h, 10 + r, 1.f);
        t0 = Clock::now();
        const Matrix hn = rms_norm(h, L.attn_norm_gain, 1e-5f);
        double t_rest = ms_since(t0);
        t0 = Clock::now();
        const Matrix attn = attention_forward(m, 0, hn, cache, batch);
        const double t_attn = ms_since(t0);
        t0 = Clock::now();
        Matrix h_mid = h;
        for (size_t i = 0; i < h_mid.data.size(); ++i) h_mid.data[i] += attn.data[i];
        const Matrix mn = rms_norm(h_mid, L.mlp_norm_gain, 1e-5f);
        t_rest += ms_since(t0);
        t0 = Clock::now();
        const Matrix mlp = mlp_forward(m, 0, mn);
        const double t_mlp = ms_since(t0);
        t0 = Clock::now();
        for (size_t i = 0; i < h_mid.data.size(); ++i) h_mid.data[i] += mlp.data[i];
        t_rest += ms_since(t0);
        cache.discard_staged();
        best_mask = std::min(best_mask, t_mask);
        best_attn = std::min(best_attn, t_attn);
        best_mlp = std::min(best_mlp, t_mlp);
        best_rest = std::min(best_rest, t_rest);
    }
    printf("{\"mode\":\"layer\",\"d_model\":%d,\"n_heads\":%d,\"d_head\":%d,\"d_mlp\":%d,\"T\":%d,\"ctx\":%d,"
           "\"mask_ms\":%.4f,\"attn_ms\":%.4f,\"mlp_ms\":%.4f,\"rest_ms\":%.4f}\n",
           d, H, dh, f, T, ctx, best_mask, best_attn, best_mlp, best_rest);
    return 0;
}

static void fill_layer(LayerWeights& L, int d, int f, uint32_t seed) {
    const float ps = 2.0f / std::sqrt((float)d);
    L.wq = Matrix(d, d); fill(L.wq, seed + 1, ps);
    L.wk = Matrix(d, d); fill(L.wk, seed + 2, ps);
    L.wv = Matrix(d, d); fill(L.wv, seed + 3, ps);
    L.wo = Matrix(d, d); fill(L.wo, seed + 4, ps);
    L.w_gate = Matrix(d, f); fill(L.w_gate, seed + 5, ps);
    L.w_up = Matrix(d, f); fill(L.w_up, seed + 6, ps);
    L.w_down = Matrix(f, d); fill(L.w_down, seed + 7, 2.0f / std::sqrt((float)f));
    L.attn_norm_gain = Matrix(1, d);
    L.mlp_norm_gain = Matrix(1, d);
    for (float& v : L.attn_norm_gain.data) v = 1.f;
    for (float& v : L.mlp_norm_gain.data) v = 1.f;
}

static int cmd_group(int argc, char** argv) {
    if (argc < 11) return 2;
    const int d = atoi(argv[2]), H = atoi(argv[3]), dh = atoi(argv[4]), f = atoi(argv[5]);
    const int g = atoi(argv[6]), T = atoi(argv[7]), ctx = atoi(argv[8]), workers = atoi(argv[9]);
    const int reps = atoi(argv[10]);
    Model m;
    m.config.d_model = d;
    m.config.n_heads = H;
    m.config.d_head = dh;
    m.config.d_mlp = f;
    m.config.n_layers = g;
    m.config.max_positions = ctx + T + 8;
    m.weights.layers.resize(g);
    for (int l = 0; l < g; ++l) fill_layer(m.weights.layers[l], d, f, 16u * l);
    LayerPlan plan;
    plan.groups.push_back({});
    for (int l = 0; l < g; ++l) plan.groups[0].push_back(l);
    plan.lp_size = g;
    KvCache cache(g, d);
    if (ctx > 0) {
        std::vector<int> parents;
        for (int i = 0; i < ctx; ++i) parents.push_back(i == 0 ? kCommittedTail : i - 1);
        const auto rows = cache.stage_append(parents, false);
        Matrix k(ctx, d), v(ctx, d);
        fill(k, 8, 1.f);
        fill(v, 9, 1.f);
        for (int l = 0; l < g; ++l) cache.write_rows(l, rows, k, v);
        cache.commit_path(rows);
    }
    WorkerPool pool(workers);
    FuzzyOptions opt;
    opt.pool = &pool;
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        std::vector<int> parents;
        for (int i = 0; i < T; ++i) parents.push_back(i == 0 ? kCommittedTail : cache.committed_len() + i - 1);
        ForwardBatch batch;
        batch.flat_rows = cache.stage_append(parents, true);
        for (int row : batch.flat_rows) batch.positions.push_back(cache.position_of(row));
        Matrix h(T, d);
        fill(h, 10 + r, 1.f);
        const auto t0 = Clock::now();
        const TreeMask mask = cache.build_tree_mask();
        batch.mask = &mask;
        const Matrix out = forward_fuzzy(m, plan, h, cache, batch, opt);
        best = std::min(best, ms_since(t0));
        if (out.data.empty()) return 3;
        cache.discard_staged();
    }
    printf("{\"mode\":\"group\",\"d_model\":%d,\"g\":%d,\"T\":%d,\"ctx\":%d,\"workers\":%d,\"group_ms\":%.4f}\n", d,
           g, T, ctx, pool.worker_count() ? pool.worker_count() : 1, best);
    return 0;
}

static int cmd_head(int argc, char** argv) {
    if (argc < 6) return 2;
    const int d = atoi(argv[2]), V = atoi(argv[3]), T = atoi(argv[4]), reps = atoi(argv[5]);
    Model m;
    m.config.d_model = d;
    m.config.vocab_size = V;
    m.weights.embedding = Matrix(V, d);
    fill(m.weights.embedding, 11, 0.05f);
    m.weights.final_norm_gain = Matrix(1, d);
    for (float& v : m.weights.final_norm_gain.data) v = 1.f;
    Matrix h(T, d);
    fill(h, 12, 1.f);
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = Clock::now();
        const Matrix lg = lm_logits(m, h);
        best = std::min(best, ms_since(t0));
        if (lg.data.empty()) return 3;
    }
    printf("{\"mode\":\"head\",\"d_model\":%d,\"vocab\":%d,\"T\":%d,\"head_ms\":%.4f}\n", d, V, T, best);
    return 0;
}

static int cmd_c1(int argc, char** argv) {
    // BASELINE config 1: the CLI-default pair (proj/src/cli.cpp:210-218).
    if (argc < 5) return 2;
    ModelConfig c;
    c.n_layers = 12;
    c.d_model = 64;
    c.n_heads = 4;
    c.d_head = 16;
    c.d_mlp = 128;
    c.seed = 7;
    const Model base = init_model(c);
    const Model draft = make_truncated_draft(base, 8);
    RunConfig r;
    r.algorithm = algorithm_from_string(argv[2]);
    r.n = 4;
    r.widths = {1, 1, 1, 1};
    r.lp_size = 2;
    r.temperature = 0.f;
    r.max_new_tokens = atoi(argv[3]);
    r.workers = 1;
    const int reps = atoi(argv[4]);
    const char* prompt = "the quick brown fox";
    double best = 1e30;
    GenerateResult res;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = Clock::now();
        res = generate(base, draft, r, {reinterpret_cast<const uint8_t*>(prompt), strlen(prompt)});
        best = std::min(best, ms_since(t0));
    }
    printf("{\"mode\":\"c1\",\"algorithm\":\"%s\",\"tokens\":%zu,\"ms\":%.4f,\"tokens_per_s\":%.3f,\"alpha\":%.4f}\n",
           argv[2], res.tokens.size(), best, res.tokens.size() / (best / 1000.0), res.report.alpha);
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string mode = argv[1];
    if (mode == "layer") return cmd_layer(argc, argv);
    if (mode == "head") return cmd_head(argc, argv);
    if (mode == "group") return cmd_group(argc, argv);
    if (mode == "c1") return cmd_c1(argc, argv);
    return 2;
}
