// Host orchestrator (see engine.h). Reference: proj/src/orchestrator.cpp,
// proj/src/draft_engine.cpp, proj/src/kv_cache.cpp, proj/src/layer_plan.cpp,
// proj/src/model.cpp (init_model order), proj/src/verifier.cpp (acceptance).
#include <algorithm>
#include <array>
#include <initializer_list>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <condition_variable>
#include <map>
#include <mutex>

#include "common.cuh"
#include "cost_sim.h"
#include "engine.h"

namespace espec {
using namespace espec_dev;

#define CUDA_OK(x)                                                                                   \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw Error(ST_CUDA, std::string(#x) + " failed: " + cudaGetErrorString(e_));            \
    } while (0)

static void cfg_fail(const std::string& m) { throw Error(ST_CONFIG, m); }

// ---------------------------------------------------------------------------
// configs and plans
// ---------------------------------------------------------------------------

void ModelCfg::validate() const {
    // ModelConfig::validate (proj/src/model.cpp:12-24), extended with GQA.
    if (vocab_size < 2) cfg_fail("vocab_size must be >= 2");
    if (n_layers < 2) cfg_fail("n_layers must be >= 2");
    if (n_heads < 1 || d_head < 2 || d_head % 2 != 0) cfg_fail("need n_heads >= 1 and an even d_head >= 2");
    if (n_kv_heads < 1 || n_heads % n_kv_heads != 0) cfg_fail("n_heads must be a multiple of n_kv_heads");
    if (d_mlp < 1) cfg_fail("d_mlp must be >= 1");
    if (max_positions < 2) cfg_fail("max_positions must be >= 2");
    if (!(norm_eps > 0.f)) cfg_fail("norm_eps must be positive");
    if (d_model % 8 != 0) cfg_fail("d_model must be a multiple of 8");
    if ((n_heads * d_head) % 8 != 0) cfg_fail("n_heads * d_head must be a multiple of 8");
    if (d_mlp % 16 != 0) cfg_fail("d_mlp must be a multiple of 16");
    if (n_heads / n_kv_heads * 1 > 64) cfg_fail("query heads per kv head must be <= 64");
    if (weight_dtype != DT_F32 && weight_dtype != DT_BF16) cfg_fail("weight dtype must be f32 or bf16");
    if (weight_dtype == DT_BF16 && (d_model % 32 || (n_heads * d_head) % 16 || d_mlp % 16))
        cfg_fail("bf16 weights need d_model % 32 == 0 and n_heads*d_head, d_mlp multiples of 16");
    if (kv_dtype != DT_F32 && kv_dtype != DT_BF16) cfg_fail("kv dtype must be f32 or bf16");
}

std::vector<int> RunCfg::effective_widths() const {
    if (widths.empty()) return std::vector<int>((size_t)std::max(n, 0), 1);
    return widths;
}

int LayerPlan::n_layers() const {
    int c = 0;
    for (auto& g : groups) c += (int)g.size();
    return c;
}
int LayerPlan::max_group_size() const {
    int b = 0;
    for (auto& g : groups) b = std::max(b, (int)g.size());
    return b;
}

static void validate_plan(const LayerPlan& p) {
    // proj/src/layer_plan.cpp:32-52
    if (p.groups.empty()) cfg_fail("layer plan has no groups");
    int expected = 0;
    for (auto& g : p.groups) {
        if (g.empty()) cfg_fail("layer plan contains an empty group");
        for (int l : g) {
            if (l != expected) cfg_fail("layer plan must cover layers contiguously in ascending order");
            ++expected;
        }
    }
    if (p.groups.front().size() != 1 || p.groups.back().size() != 1)
        cfg_fail("first and last layer must be singleton groups");
    if (p.max_group_size() > p.lp_size && p.lp_size > 0) cfg_fail("layer plan group exceeds the layer-parallel size");
}

LayerPlan plan_groups(int n_layers, int lp) {
    // proj/src/layer_plan.cpp:54-82: 0 | 1..N-1 | N..2N-1 | ... | last
    if (n_layers < 2) cfg_fail("layer plan needs at least 2 layers");
    if (lp < 1) cfg_fail("layer-parallel size must be >= 1");
    LayerPlan p;
    p.lp_size = lp;
    p.groups.push_back({0});
    const int last = n_layers - 1;
    for (int next = 1; next < last;) {
        int end = next == 1 ? std::max(lp, 2) : next + lp;
        end = std::min(end, last);
        std::vector<int> g;
        for (int l = next; l < end; ++l) g.push_back(l);
        p.groups.push_back(g);
        next = end;
    }
    p.groups.push_back({last});
    validate_plan(p);
    return p;
}

LayerPlan parse_plan_override(const std::string& spec) {
    // proj/src/layer_plan.cpp:84-114
    LayerPlan p;
    std::stringstream ss(spec);
    std::string tok;
    while (std::getline(ss, tok, '|')) {
        if (tok.empty()) cfg_fail("empty group in plan override '" + spec + "'");
        const auto dash = tok.find('-');
        int lo = 0, hi = 0;
        try {
            if (dash == std::string::npos) lo = hi = std::stoi(tok);
            else {
                lo = std::stoi(tok.substr(0, dash));
                hi = std::stoi(tok.substr(dash + 1));
            }
        } catch (const std::exception&) {
            cfg_fail("unparsable group '" + tok + "' in plan override");
        }
        if (lo < 0 || hi < lo) cfg_fail("invalid layer range '" + tok + "' in plan override");
        std::vector<int> g;
        for (int l = lo; l <= hi; ++l) g.push_back(l);
        p.groups.push_back(g);
    }
    if (!spec.empty() && spec.back() == '|') cfg_fail("empty group in plan override '" + spec + "'");
    p.lp_size = p.max_group_size();
    validate_plan(p);
    return p;
}

std::string format_plan(const LayerPlan& p) {
    std::string out;
    for (size_t i = 0; i < p.groups.size(); ++i) {
        if (i) out += '|';
        out += std::to_string(p.groups[i].front());
        if (p.groups[i].size() > 1) out += "-" + std::to_string(p.groups[i].back());
    }
    return out;
}

// ---------------------------------------------------------------------------
// host RNG (proj/include/espec/rng.hpp) — parity-mode weights and T>0 draws
// ---------------------------------------------------------------------------

struct Xoshiro {
    uint64_t s[4];
    explicit Xoshiro(uint64_t seed) {
        uint64_t st = seed;
        for (auto& w : s) {
            uint64_t z = (st += 0x9E3779B97F4A7C15ULL);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            w = z ^ (z >> 31);
        }
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t next() {
        const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
    float normal() {
        const double u1 = uniform(), u2 = uniform();
        return (float)(std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(6.283185307179586 * u2));
    }
};

// ---------------------------------------------------------------------------
// device model
// ---------------------------------------------------------------------------

static int pad8(int n) { return (n + 7) / 8 * 8; }
// GEMV weight leading dimension: bf16 weights are packed per 32 columns.
static int ldpad(int n, int dt) { return dt == DT_BF16 ? (n + 31) / 32 * 32 : pad8(n); }
static size_t dsize(int dt) { return dt == DT_BF16 ? 2 : 4; }

static uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

struct LayerDev {
    void* wqkv = nullptr;  // [d][qkv_ld]
    void* wo = nullptr;    // [H*dh][d]
    void* wgu = nullptr;   // [d][gu_ld] interleaved per 32 cols: [gate16 | up16]
    void* wd = nullptr;    // [f][d]
    float* ga = nullptr;
    float* gm = nullptr;
};

// One tensor-parallel shard of a model (Megatron split):
// QKV / gate-up column-parallel (this rank's q heads, kv heads and MLP
// columns), O / down row-parallel (partials all-reduced over NVLink), head
// vocab-parallel; embedding and norm gains replicated. tp == 1 is the whole
// model. Weight values depend only on the global (row, column), so any TP
// degree runs the same model.
struct ModelDev {
    ModelCfg c;
    int tp = 1, rank = 0;
    // attention split: atp ranks share each layer's heads (Megatron, = tp), or
    // under the layer-parallel placement (lp, drafter only: the paper layout)
    // atp = 1 and owner[l] is the one rank that runs layer l's attention (full
    // heads) and holds its KV; the MLP and the head stay tensor-parallel
    int atp = 1, arank = 0;
    bool lp = false;
    std::vector<int> owner;
    void* emb = nullptr;   // [V][d] (replicated)
    void* head = nullptr;  // [d][head_ld]: this rank's vocabulary slice
    int head_ld = 0;
    float* fgain = nullptr;
    float2* rope = nullptr;  // [max_positions][d_head/2] (cos, sin) of apply_rope's angles
    std::vector<LayerDev> L;
    std::vector<void*> owned;
    int qh() const { return c.n_heads / atp; }
    int kvh() const { return c.n_kv_heads / atp; }
    int f_loc() const { return c.d_mlp / tp; }
    int V_loc() const { return c.vocab_size / tp; }
    int qkv_N() const { return (qh() + 2 * kvh()) * c.d_head; }
    int qkv_ld() const { return ldpad(qkv_N(), c.weight_dtype); }
    int gu_N() const { return 2 * f_loc(); }
    int gu_ld() const { return ldpad(gu_N(), c.weight_dtype); }
    int qdim() const { return qh() * c.d_head; }
    int kvdim() const { return kvh() * c.d_head; }
    void* alloc(size_t bytes) {
        void* p = nullptr;
        CUDA_OK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        CUDA_OK(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
        owned.push_back(p);
        return p;
    }
    // Rotary table, computed on the host exactly as apply_rope does
    // (proj/src/matrix.cpp:171-186): inv_freq = pow(theta, -2p/dh) and
    // (float)cos / (float)sin of pos * inv_freq in double. The GEMV epilogues
    // read it instead of evaluating double trigonometry per element.
    void build_rope() {
        const int np = c.d_head / 2;
        std::vector<double> inv_freq(np);
        for (int p = 0; p < np; ++p) inv_freq[p] = std::pow((double)c.rope_theta, -2.0 * p / c.d_head);
        std::vector<float2> tab((size_t)c.max_positions * np);
        for (int pos = 0; pos < c.max_positions; ++pos)
            for (int p = 0; p < np; ++p) {
                const double th = (double)pos * inv_freq[p];
                tab[(size_t)pos * np + p] = make_float2((float)std::cos(th), (float)std::sin(th));
            }
        rope = (float2*)alloc(sizeof(float2) * tab.size());
        CUDA_OK(cudaMemcpy(rope, tab.data(), sizeof(float2) * tab.size(), cudaMemcpyHostToDevice));
    }
    void allocate(bool share_layers_from_base, const ModelDev* base) {
        const int d = c.d_model, f = f_loc(), V = c.vocab_size, es = (int)dsize(c.weight_dtype);
        head_ld = ldpad(V_loc(), c.weight_dtype);
        build_rope();
        if (share_layers_from_base) {
            emb = base->emb;
            head = base->head;
            head_ld = base->head_ld;
            fgain = base->fgain;
            L.assign(base->L.begin(), base->L.begin() + c.n_layers);
            return;
        }
        emb = alloc((size_t)V * d * es);
        head = alloc((size_t)d * head_ld * es);  // [d][V]; for a tied head, the transposed embedding
        fgain = (float*)alloc((size_t)d * 4);
        L.resize(c.n_layers);
        for (auto& l : L) {
            l.wqkv = alloc((size_t)d * qkv_ld() * es);
            l.wo = alloc((size_t)qdim() * d * es);
            l.wgu = alloc((size_t)d * gu_ld() * es);
            l.wd = alloc((size_t)f * d * es);
            l.ga = (float*)alloc((size_t)d * 4);
            l.gm = (float*)alloc((size_t)d * 4);
        }
    }
    void release() {
        for (void* p : owned) cudaFree(p);
        owned.clear();
    }
};

// Upload an fp32 host block [rows][cols] into a device matrix with leading
// dimension ld at column offset col0, converting to the weight dtype.
static void upload_block(void* dst, int dt, long long ld, long long col0, const float* src, long long rows,
                         long long cols, cudaStream_t s) {
    const size_t es = dsize(dt);
    std::vector<uint16_t> tmp16;
    const void* h = src;
    if (dt == DT_BF16) {
        tmp16.resize((size_t)rows * cols);
        for (size_t i = 0; i < tmp16.size(); ++i) tmp16[i] = f2bf(src[i]);
        h = tmp16.data();
    }
    CUDA_OK(cudaMemcpy2DAsync((char*)dst + col0 * es, ld * es, h, cols * es, cols * es, rows, cudaMemcpyHostToDevice, s));
    CUDA_OK(cudaStreamSynchronize(s));
}

static void download_block(const void* src, int dt, long long ld, long long col0, float* dst, long long rows,
                           long long cols) {
    const size_t es = dsize(dt);
    std::vector<uint16_t> tmp16((size_t)rows * cols);
    void* h = dt == DT_BF16 ? (void*)tmp16.data() : (void*)dst;
    CUDA_OK(cudaMemcpy2D(h, cols * es, (const char*)src + col0 * es, ld * es, cols * es, rows, cudaMemcpyDeviceToHost));
    if (dt == DT_BF16)
        for (size_t i = 0; i < tmp16.size(); ++i) dst[i] = bf2f(tmp16[i]);
}

// ---------------------------------------------------------------------------
// KV cache: host bookkeeping (proj/src/kv_cache.cpp) + paged device pool
// ---------------------------------------------------------------------------

constexpr int kTail = -1;  // kCommittedTail

struct Staged {
    int parent;
    bool fuzzy;
    int position;
};

struct Cache {
    int n_layers = 0, n_kv = 0, dh = 0, dtype = DT_F32;
    int committed = 0;
    std::vector<Staged> staged;
    // paged device pool
    void* pool = nullptr;
    int page_rows = 64;
    long long page_elems = 0;
    int n_pages = 0;
    std::vector<int> table;        // logical block -> physical page
    std::vector<int> free_pages;
    int* table_dev = nullptr;
    int mapped_blocks = 0;

    int total() const { return committed + (int)staged.size(); }

    void create(const ModelCfg& c, int kv_heads, int capacity_rows) {
        n_layers = c.n_layers;
        n_kv = kv_heads;
        dh = c.d_head;
        dtype = c.kv_dtype;
        page_elems = (long long)n_layers * 2 * n_kv * page_rows * dh;
        n_pages = (capacity_rows + page_rows - 1) / page_rows;
        CUDA_OK(cudaMalloc(&pool, (size_t)n_pages * page_elems * dsize(dtype)));
        CUDA_OK(cudaMemset(pool, 0, (size_t)n_pages * page_elems * dsize(dtype)));
        CUDA_OK(cudaMalloc(&table_dev, sizeof(int) * (size_t)n_pages));
        CUDA_OK(cudaMemset(table_dev, 0, sizeof(int) * (size_t)n_pages));
        table.assign(n_pages, -1);
        free_pages.clear();
        for (int p = n_pages - 1; p >= 0; --p) free_pages.push_back(p);
        mapped_blocks = 0;
    }
    void destroy() {
        if (pool) cudaFree(pool);
        if (table_dev) cudaFree(table_dev);
        pool = nullptr;
        table_dev = nullptr;
    }
    KvView view() const {
        KvView v;
        v.pool = pool;
        v.pool_pages = n_pages;
        v.page_table = table_dev;
        v.page_rows = page_rows;
        v.n_layers = n_layers;
        v.n_kv = n_kv;
        v.dh = dh;
        v.dtype = dtype;
        v.page_elems = page_elems;
        const int cap = n_pages * page_rows;
        v.attn_ppi = attn_pages_per_item(cap);
        // KV pages are read once per pass (then evicted first): measured a
        // small gain, mostly for 1-row passes
        static const int hint = [] {
            const char* e = std::getenv("ESPEC_ATTN_L2");
            return e ? std::atoi(e) : 1;
        }();
        v.l2_hint = hint;
        return v;
    }
    // Map pages so rows [0, rows) are backed.
    void ensure(int rows, cudaStream_t s) {
        const int need = (rows + page_rows - 1) / page_rows;
        if (need > n_pages) throw Error(ST_CONFIG, "kv cache capacity exceeded");
        const int first = mapped_blocks;
        while (mapped_blocks < need) {
            table[mapped_blocks] = free_pages.back();
            free_pages.pop_back();
            ++mapped_blocks;
        }
        if (need > first)
            CUDA_OK(cudaMemcpyAsync(table_dev + first, table.data() + first, sizeof(int) * (size_t)(need - first),
                                    cudaMemcpyHostToDevice, s));
    }
    void reset() {
        committed = 0;
        staged.clear();
    }
    // stage_append (proj/src/kv_cache.cpp:23-41)
    std::vector<int> stage_append(const std::vector<int>& parents, bool fuzzy) {
        std::vector<int> rows;
        for (int par : parents) {
            const int flat = total();
            if (par != kTail && (par < committed || par >= flat))
                throw Error(ST_STRUCTURE, "staged parent must be the committed tail or an earlier staged row");
            const int pos = par == kTail ? committed : staged[par - committed].position + 1;
            staged.push_back({par, fuzzy, pos});
            rows.push_back(flat);
        }
        return rows;
    }
    int position_of(int flat) const { return flat < committed ? flat : staged[flat - committed].position; }
    // commit_path (proj/src/kv_cache.cpp:62-94): returns the row moves.
    void commit_path(const std::vector<int>& path, std::vector<int>& src, std::vector<int>& dst) {
        int expect = kTail;
        for (int flat : path) {
            if (flat < 0 || flat >= total()) throw Error(ST_STRUCTURE, "kv row out of range");
            if (flat < committed) throw Error(ST_STRUCTURE, "commit path entry is already committed");
            if (staged[flat - committed].parent != expect)
                throw Error(ST_STRUCTURE, "commit path is not a root-to-node chain");
            expect = flat;
        }
        src.clear();
        dst.clear();
        for (size_t i = 0; i < path.size(); ++i)
            if (path[i] != committed + (int)i) {
                src.push_back(path[i]);
                dst.push_back(committed + (int)i);
            }
        committed += (int)path.size();
        staged.clear();
    }
    void discard() { staged.clear(); }  // proj/src/kv_cache.cpp:96-102
    bool any_fuzzy() const {
        for (auto& r : staged)
            if (r.fuzzy) return true;
        return false;
    }
};

// ---------------------------------------------------------------------------
// pinned->device staging for per-pass metadata (bump allocator per iteration)
// ---------------------------------------------------------------------------

struct Staging {
    char* host = nullptr;
    char* dev = nullptr;
    size_t cap = 0, off = 0;
    void create(size_t bytes) {
        cap = bytes;
        CUDA_OK(cudaMallocHost(&host, cap));
        CUDA_OK(cudaMalloc(&dev, cap));
    }
    void destroy() {
        if (host) cudaFreeHost(host);
        if (dev) cudaFree(dev);
        host = dev = nullptr;
    }
    long long* h2d_counter = nullptr;
    template <typename T>
    T* push(const T* data, size_t n, cudaStream_t s) {
        const size_t bytes = sizeof(T) * std::max<size_t>(n, 1);
        const size_t aligned = (bytes + 255) / 256 * 256;
        if (off + aligned > cap) throw Error(ST_CONFIG, "pass metadata staging exhausted");
        if (n) std::memcpy(host + off, data, sizeof(T) * n);
        T* d = reinterpret_cast<T*>(dev + off);
        CUDA_OK(cudaMemcpyAsync(d, host + off, bytes, cudaMemcpyHostToDevice, s));
        if (h2d_counter) *h2d_counter += (long long)bytes;
        off += aligned;
        return d;
    }
    void reset() { off = 0; }
};

// ---------------------------------------------------------------------------
// single-device tensor-parallel harness: cross-stream ordering of the
// collectives' push and combine kernels (see CommView::local_sync)
// ---------------------------------------------------------------------------

struct LocalGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<long long> calls;            // collectives each rank has reached
    std::vector<std::array<cudaEvent_t, 2>> ev;  // per rank, per call parity
    explicit LocalGroup(int w) : world(w), calls(w, 0), ev(w) {
        for (auto& e : ev)
            for (auto& x : e) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    }
    ~LocalGroup() {
        for (auto& e : ev)
            for (auto& x : e) cudaEventDestroy(x);
    }
};

static void local_sync_fn(void* ctx, int rank, cudaStream_t s) {
    LocalGroup* g = static_cast<LocalGroup*>(ctx);
    std::unique_lock<std::mutex> lk(g->mu);
    const long long k = g->calls[rank];
    cudaEventRecord(g->ev[rank][k & 1], s);  // this rank's push is issued
    g->calls[rank] = k + 1;
    g->cv.notify_all();
    g->cv.wait(lk, [&] {
        for (long long c : g->calls)
            if (c < k + 1) return false;
        return true;
    });
    for (int p = 0; p < g->world; ++p)
        if (p != rank) cudaStreamWaitEvent(s, g->ev[p][k & 1], 0);
}

// ---------------------------------------------------------------------------
// engine
// ---------------------------------------------------------------------------

constexpr int kChunk = 256;     // max rows per forward pass (prefill is chunked)
constexpr int kAttnQ = 64;      // query rows per attention launch (prefill chunks: 4 launches per 256 rows)
constexpr int kMaxNodes = 64;   // drafted tree nodes per iteration (ancestor bitmask)

struct Workspace {
    float* h = nullptr;       // [kChunk][d]
    float* stats = nullptr;   // [kChunk][tiles]
    float* q = nullptr;       // [G][kChunk][H*dh]
    float* mixed = nullptr;   // [G][kChunk][H*dh]
    float* attn = nullptr;    // [G][kChunk][d]
    float* act = nullptr;     // [kChunk][f]
    // decode passes (bf16 weights, T <= 16): attention output and SiLU output
    // as bf16, the form the O / down GEMVs stage anyway (half the bytes)
    __nv_bfloat16* mixed_b16 = nullptr;  // [G][kChunk][H*dh]
    __nv_bfloat16* act_b16 = nullptr;    // [kChunk][f]
    float* logits = nullptr;  // [8][head_ld] (parity probes)
    float* am_val = nullptr;
    int* am_idx = nullptr;
    float* gemv_part = nullptr;
    size_t gemv_part_slot = 0;
    unsigned* gemv_tickets = nullptr;
    int gemv_ticket_slot = 0;
    float* attn_ws = nullptr;
    size_t attn_ws_slot = 0;
    unsigned* attn_tickets = nullptr;
    int attn_ticket_slot = 0;
    // tensor parallelism
    float* part = nullptr;      // [kChunk][d] row-parallel GEMV partial
    float* best_val = nullptr;  // [kChunk] vocab-slice max per row
    int* best_idx = nullptr;
    float* lg_loc = nullptr;    // [kMaxNodes+1][head_ld] vocab-slice logits
    // prefill (tcgen05 GEMM) workspace
    __nv_bfloat16* tc_xa = nullptr;
    float* tc_rms = nullptr;
    float* tc_part = nullptr;
    unsigned* tc_tickets = nullptr;
    int G = 1;
};

class EngineImpl final : public Engine {
public:
    EngineImpl(const ModelCfg& bc, const ModelCfg& dc, const RunCfg& run, int device, int tp, int rank,
               bool draft_lp)
        : device_(device) {
        bc.validate();
        dc.validate();
        if (bc.vocab_size != dc.vocab_size) cfg_fail("base and draft models must share the vocabulary");
        if (tp < 1 || tp > kMaxTp) cfg_fail("tp_size must lie in [1, 8]");
        if (rank < 0 || rank >= tp) cfg_fail("tp_rank must lie in [0, tp_size)");
        if (draft_lp && tp < 2) cfg_fail("layer-parallel placement needs tp_size > 1 (one GPU per group slot)");
        for (const ModelCfg* c : {&bc, &dc}) {
            if ((c->n_heads % tp || c->n_kv_heads % tp) && !(c == &dc && draft_lp))
                cfg_fail("attention heads must divide by tp_size");
            if (c->d_mlp % (16 * tp)) cfg_fail("d_mlp must be a multiple of 16 * tp_size");
            if (c->vocab_size % tp) cfg_fail("vocab_size must divide by tp_size");
        }
        base_.c = bc;
        draft_.c = dc;
        base_.tp = draft_.tp = tp;
        base_.rank = draft_.rank = rank;
        base_.atp = tp;
        base_.arank = rank;
        draft_.lp = draft_lp;
        draft_.atp = draft_lp ? 1 : tp;
        draft_.arank = draft_lp ? 0 : rank;
        set_run(run);
        CUDA_OK(cudaSetDevice(device));
        if (const char* e = std::getenv("ESPEC_PDL")) set_pdl(std::atoi(e) != 0);
        CUDA_OK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        if (const char* e = std::getenv("ESPEC_WIDE_DRAFT")) wide_draft_ = std::atoi(e);
        if (const char* e = std::getenv("ESPEC_FUSE_ADDS")) fuse_adds_ = std::atoi(e);
        if (const char* e = std::getenv("ESPEC_B16_ACTS")) b16_acts_ = std::atoi(e);
        for (auto& e : ev_) CUDA_OK(cudaEventCreate(&e));
        const int cap_b = bc.max_positions + kMaxNodes + kChunk;
        const int cap_d = dc.max_positions + kMaxNodes + kChunk;
        bcache_.create(bc, base_.kvh(), cap_b);
        dcache_.create(dc, draft_.kvh(), cap_d);
        if (tp > 1) {
            // symmetric receive region for the NVLink collectives: sized for a
            // prefill chunk of hidden rows or the gathered verify logits
            const int dmax = std::max(bc.d_model, dc.d_model);
            comm_.rank = rank;
            comm_.world = tp;
            comm_.debug = std::getenv("ESPEC_TRACE_COMM") ? 1 : 0;
            comm_.slot_floats = std::max<size_t>((size_t)kChunk * dmax, (size_t)(kMaxNodes + 1) * (bc.vocab_size / tp));
            const size_t bytes = sizeof(float) * comm_.slot_floats * 2 * tp + sizeof(uint64_t) * 2 * tp;
            CUDA_OK(cudaMalloc(&comm_mem_, bytes));
            CUDA_OK(cudaMemset(comm_mem_, 0, bytes));
            comm_.recv_local = reinterpret_cast<float*>(comm_mem_);
            comm_.flags_local = reinterpret_cast<uint64_t*>(comm_.recv_local + comm_.slot_floats * 2 * tp);
            CUDA_OK(cudaMalloc(&comm_.ticket, sizeof(unsigned)));
            CUDA_OK(cudaMemset(comm_.ticket, 0, sizeof(unsigned)));
        }
        staging_.create(8 << 20);
        staging_.h2d_counter = &h2d_bytes_;
        for (auto& e : site_ev_) CUDA_OK(cudaEventCreate(&e));
        tree_off_ = std::max(cap_b, cap_d);
        am_off_ = tree_off_ + kMaxNodes;
        out_off_ = am_off_ + kMaxNodes + 1;   // m, bonus, path[kMaxNodes], tokens[kMaxNodes]
        cur_off_ = out_off_ + 2 + 2 * kMaxNodes;  // uniform cursor
        err_off_ = cur_off_ + 1;                   // device error flag
        arena_cap_ = err_off_ + 64;
        CUDA_OK(cudaMalloc(&arena_, sizeof(int) * (size_t)arena_cap_));
        CUDA_OK(cudaMemset(arena_, 0, sizeof(int) * (size_t)arena_cap_));
        comm_.err = arena_ + err_off_;
        CUDA_OK(cudaMalloc(&pool_.dev, sizeof(unsigned) * sgemv_pool_words()));
        sgemv_pool_reset(pool_, stream_);
        CUDA_OK(cudaMallocHost(&outcome_host_, sizeof(int) * (size_t)(err_off_ - out_off_ + 1)));
        // T > 0 / tree-level buffers: logits and dists per drafted row
        const int V = bc.vocab_size;
        const int ldl = std::max(ldpad(V, bc.weight_dtype), ldpad(V, dc.weight_dtype));
        logits_ld_ = ldl;
        CUDA_OK(cudaMalloc(&dlogits_, sizeof(float) * (size_t)(kMaxNodes + 1) * ldl));
        CUDA_OK(cudaMalloc(&blogits_, sizeof(float) * (size_t)(kMaxNodes + 1) * ldl));
        CUDA_OK(cudaMalloc(&ddists_, sizeof(float) * (size_t)(kMaxNodes + 1) * V));
        CUDA_OK(cudaMalloc(&bdists_, sizeof(float) * (size_t)(kMaxNodes + 1) * V));
        CUDA_OK(cudaMalloc(&target_, sizeof(float) * (size_t)V));
        CUDA_OK(cudaMalloc(&unif_dev_, sizeof(double) * kMaxDraws));
        CUDA_OK(cudaMallocHost(&unif_host_, sizeof(double) * kMaxDraws));
        alloc_ws(bws_, base_, 1);
        alloc_ws(dws_, draft_, kMaxGroup);
        base_allocated_ = draft_allocated_ = false;
    }
    ~EngineImpl() override {
        cudaStreamSynchronize(stream_);
        base_.release();
        draft_.release();
        bcache_.destroy();
        dcache_.destroy();
        staging_.destroy();
        for (void* p : ws_owned_) cudaFree(p);
        cudaFree(arena_);
        cudaFree(pool_.dev);
        if (temp_) cudaFree(temp_);
        cudaFreeHost(outcome_host_);
        cudaFree(dlogits_);
        cudaFree(blogits_);
        cudaFree(ddists_);
        cudaFree(bdists_);
        cudaFree(target_);
        cudaFree(unif_dev_);
        cudaFreeHost(unif_host_);
        for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
        if (comm_mem_) cudaFree(comm_mem_);
        if (comm_.ticket) cudaFree(comm_.ticket);
        for (auto& e : ev_) cudaEventDestroy(e);
        for (auto& e : site_ev_) cudaEventDestroy(e);
        cudaStreamDestroy(stream_);
    }

    // ---------------- setup ----------------

    void set_cost(const CostParams& cost) override {
        cost.validate();
        cost_ = cost;
    }
    std::string occupancy_csv() const override { return clock_.occupancy_csv(); }

    void set_run(const RunCfg& run) override {
        run_ = run;
        widths_ = run.effective_widths();
        if (run.algorithm != ALG_EASYSPEC) plan_ = plan_groups(draft_.c.n_layers, 1);
        else if (!run.plan_override.empty()) plan_ = parse_plan_override(run.plan_override);
        else plan_ = plan_groups(draft_.c.n_layers, run.lp_size);
        if (plan_.n_layers() != draft_.c.n_layers)
            cfg_fail("layer plan covers " + std::to_string(plan_.n_layers()) + " layers, drafter has " +
                     std::to_string(draft_.c.n_layers));
        if (plan_.max_group_size() > kMaxGroup) cfg_fail("layer-parallel groups are limited to 8 layers");
        // layer-parallel placement: group slot j -> rank j (mod the group size
        // of GPUs); sequential drafting (sd / vanilla plans) keeps every layer
        // on rank 0, the lead GPU
        draft_.owner.assign(draft_.c.n_layers, 0);
        for (const auto& grp : plan_.groups)
            for (size_t j = 0; j < grp.size(); ++j) draft_.owner[grp[j]] = (int)(j % std::max(1, draft_.tp));
        // validate_run_config (proj/src/orchestrator.cpp:95-118)
        if (run.n < 1) cfg_fail("speculation length must be >= 1");
        if (run.max_new_tokens < 1) cfg_fail("max_new_tokens must be >= 1");
        if (run.temperature < 0.f) cfg_fail("temperature must be >= 0");
        if ((int)widths_.size() != run.n) cfg_fail("widths must list one branching factor per speculation level");
        for (int w : widths_) {
            if (w < 1 || w > draft_.c.vocab_size) cfg_fail("tree widths must lie in [1, vocab]");
            if (run.algorithm == ALG_SD && w != 1) cfg_fail("plain sd requires all tree widths = 1");
        }
        long long nodes = 0, level = 1;
        for (int w : widths_) {
            level *= w;
            nodes += level;
            if (nodes > kMaxNodes) cfg_fail("drafted tree exceeds 64 nodes");
        }
        for (int w : widths_)
            if (w > kMaxWidth) cfg_fail("tree widths above 16 are not supported on device");
    }

    void ensure_allocated(int which) {
        if (which == 1 && !base_allocated_) {
            base_.allocate(false, nullptr);
            base_allocated_ = true;
        }
        if (which == 0 && !draft_allocated_) {
            draft_.allocate(false, nullptr);
            draft_allocated_ = true;
        }
    }

    void share_truncated_draft() override {
        // make_truncated_draft (proj/src/model.cpp:86-99): the drafter reuses the
        // base's embedding, final norm and first L_d blocks (no copy in HBM).
        if (!base_allocated_) throw Error(ST_CONFIG, "initialise the base model first");
        if (draft_.lp)
            cfg_fail("the layer-parallel drafter holds full-head attention while the base is head-sharded: "
                     "initialise it on its own (init_model(keep layers, same seed) is the same truncated model)");
        const ModelCfg& b = base_.c;
        const ModelCfg& d = draft_.c;
        if (d.n_layers < 2 || d.n_layers >= b.n_layers)
            cfg_fail("keep_layers must satisfy 2 <= keep_layers < base layers, got " + std::to_string(d.n_layers));
        if (d.d_model != b.d_model || d.n_heads != b.n_heads || d.n_kv_heads != b.n_kv_heads || d.d_head != b.d_head ||
            d.d_mlp != b.d_mlp || d.weight_dtype != b.weight_dtype || d.tied_head != b.tied_head)
            cfg_fail("truncated drafter must share the base architecture");
        draft_.release();
        draft_.allocate(true, &base_);
        draft_allocated_ = true;
    }

    void init_weights_seeded(int which, uint64_t seed, bool parity) override {
        ModelDev& M = which ? base_ : draft_;
        M.c.seed = seed;
        ensure_allocated(which);
        const ModelCfg& c = M.c;
        const int d = c.d_model, f = c.d_mlp, V = c.vocab_size;
        const float proj_sd = 1.0f / std::sqrt((float)d);
        const float resid = 1.0f / std::sqrt(2.0f * (float)c.n_layers);
        const float down_sd = resid / std::sqrt((float)f);
        const float emb_sd = 3.0f / std::sqrt((float)d);
        if (parity) {
            // init_model (proj/src/model.cpp:38-84): one xoshiro256** stream, fixed order.
            if (c.n_kv_heads != c.n_heads || c.n_heads * c.d_head != d || !c.tied_head)
                cfg_fail("parity init needs the reference architecture (MHA, tied head)");
            Xoshiro rng(seed);
            auto fill = [&](std::vector<float>& v, size_t n, float sd) {
                v.resize(n);
                for (auto& x : v) x = rng.normal() * sd;
            };
            std::vector<float> t;
            fill(t, (size_t)V * d, emb_sd);
            load_tensor(which, "embedding", -1, t.data(), V, d);
            std::vector<float> ones((size_t)d, 1.f);
            load_tensor(which, "final_norm_gain", -1, ones.data(), 1, d);
            for (int l = 0; l < c.n_layers; ++l) {
                fill(t, (size_t)d * d, proj_sd); load_tensor(which, "wq", l, t.data(), d, d);
                fill(t, (size_t)d * d, proj_sd); load_tensor(which, "wk", l, t.data(), d, d);
                fill(t, (size_t)d * d, proj_sd); load_tensor(which, "wv", l, t.data(), d, d);
                fill(t, (size_t)d * d, proj_sd * resid); load_tensor(which, "wo", l, t.data(), d, d);
                fill(t, (size_t)d * f, proj_sd); load_tensor(which, "w_gate", l, t.data(), d, f);
                fill(t, (size_t)d * f, proj_sd); load_tensor(which, "w_up", l, t.data(), d, f);
                fill(t, (size_t)f * d, down_sd); load_tensor(which, "w_down", l, t.data(), f, d);
                load_tensor(which, "attn_norm_gain", l, ones.data(), 1, d);
                load_tensor(which, "mlp_norm_gain", l, ones.data(), 1, d);
            }
            return;
        }
        // Perf mode: same std rules, drawn on device from a counter hash of
        // the GLOBAL (row, column), so a TP shard holds exactly its slice of
        // the one model (logical layout first, padding zeroed, then packed).
        const int dt = c.weight_dtype;
        uint64_t k = seed * 1000003ULL + 17;
        const int H = c.n_heads, Hkv = c.n_kv_heads, dh = c.d_head, r = M.rank;
        const int qh = M.qh(), kvh = M.kvh(), fl = M.f_loc(), Vl = M.V_loc();
        auto seg = [](std::initializer_list<std::array<int, 3>> ss) {
            ColMap m;
            for (auto& x : ss) {
                m.lc0[m.nseg] = x[0];
                m.gc0[m.nseg] = x[1];
                m.len[m.nseg] = x[2];
                ++m.nseg;
            }
            return m;
        };
        launch_fill_normal(dt, M.emb, (long long)V * d, emb_sd, k++, stream_);  // replicated
        launch_fill_const(DT_F32, M.fgain, d, 1.f, stream_);
        if (c.tied_head) {
            void* t = temp((size_t)d * M.head_ld * dsize(dt));
            CUDA_OK(cudaMemsetAsync(t, 0, (size_t)d * M.head_ld * dsize(dt), stream_));
            launch_transpose(dt, (const char*)M.emb + (size_t)r * Vl * d * dsize(dt), Vl, d, t, M.head_ld, stream_);
            finish_logical(M.head, dt, d, M.head_ld, t);
        } else {
            ColMap m = seg({{0, r * Vl, Vl}});
            m.seed = k++;
            mat_fill_map(M.head, dt, d, M.head_ld, m, 0, V, emb_sd);
        }
        for (int l = 0; l < c.n_layers; ++l) {
            LayerDev& L = M.L[l];
            const int ar = M.arank;  // attention heads of this rank (all of them under lp)
            ColMap mq = seg({{0, ar * qh * dh, qh * dh},
                             {qh * dh, H * dh + ar * kvh * dh, kvh * dh},
                             {(qh + kvh) * dh, (H + Hkv) * dh + ar * kvh * dh, kvh * dh}});
            mq.seed = k++;
            mat_fill_map(L.wqkv, dt, d, M.qkv_ld(), mq, 0, (long long)(H + 2 * Hkv) * dh, proj_sd);
            ColMap mo = seg({{0, 0, d}});
            mo.seed = k++;
            mat_fill_map(L.wo, dt, qh * dh, d, mo, ar * qh * dh, d, proj_sd * resid);
            ColMap mg;
            mg.gateup = 1;
            mg.f_loc = fl;
            mg.f_base = r * fl;
            mg.seed = k++;
            mg.seed2 = k++;
            mat_fill_map(L.wgu, dt, d, M.gu_ld(), mg, 0, f, proj_sd);
            ColMap md = seg({{0, 0, d}});
            md.seed = k++;
            mat_fill_map(L.wd, dt, fl, d, md, r * fl, d, down_sd);
            launch_fill_const(DT_F32, L.ga, d, 1.f, stream_);
            launch_fill_const(DT_F32, L.gm, d, 1.f, stream_);
        }
        CUDA_OK(cudaStreamSynchronize(stream_));
        CUDA_OK(cudaGetLastError());
    }

    void mat_fill_map(void* W, int dt, int K, int ld, const ColMap& m, int row_off, long long n_full, float sd) {
        void* t = temp((size_t)K * ld * dsize(dt));
        launch_fill_normal_map(dt, t, K, ld, m, row_off, n_full, sd, stream_);
        finish_logical(W, dt, K, ld, t);
    }

    // ---- weight matrices: fp32 row-major, or bf16 packed in the UMMA canonical K-major layout
    void* temp(size_t bytes) {
        if (bytes > temp_bytes_) {
            if (temp_) cudaFree(temp_);
            CUDA_OK(cudaMalloc(&temp_, bytes));
            temp_bytes_ = bytes;
        }
        return temp_;
    }
    // logical (K x ld, in temp) -> final storage
    void finish_logical(void* W, int dt, int K, int ld, const void* logical) {
        if (dt == DT_BF16) launch_pack(logical, K, ld, W, false, stream_);
        else CUDA_OK(cudaMemcpyAsync(W, logical, (size_t)K * ld * 4, cudaMemcpyDeviceToDevice, stream_));
        CUDA_OK(cudaStreamSynchronize(stream_));
    }
    template <typename Valid>
    void mat_fill(void* W, int dt, int K, int ld, int N, float sd, uint64_t seed, Valid valid) {
        const size_t es = dsize(dt);
        void* t = temp((size_t)K * ld * es);
        launch_fill_normal(dt, t, (long long)K * ld, sd, seed, stream_);
        if (N < ld) CUDA_OK(cudaMemset2DAsync((char*)t + (size_t)N * es, ld * es, 0, (ld - N) * es, K, stream_));
        // zero padded columns inside the interleaved gate/up tiles
        for (int n0 = 0; n0 < std::min(N, ld); n0 += 128) {
            if (!valid(n0 + 127)) {
                int first = n0;
                while (first < n0 + 128 && valid(first)) ++first;
                CUDA_OK(cudaMemset2DAsync((char*)t + (size_t)first * es, ld * es, 0, (n0 + 128 - first) * es, K, stream_));
            }
        }
        finish_logical(W, dt, K, ld, t);
    }
    void mat_write(void* W, int dt, int K, int ld, long long col0, const float* src, long long cols) {
        if (dt != DT_BF16) return upload_block(W, dt, ld, col0, src, K, cols, stream_);
        void* t = temp((size_t)K * ld * 2);
        launch_pack(t, K, ld, W, true, stream_);
        upload_block(t, dt, ld, col0, src, K, cols, stream_);
        finish_logical(W, dt, K, ld, t);
    }
    void mat_read(const void* W, int dt, int K, int ld, long long col0, float* dst, long long cols) {
        if (dt != DT_BF16) return download_block(W, dt, ld, col0, dst, K, cols);
        void* t = temp((size_t)K * ld * 2);
        launch_pack(t, K, ld, const_cast<void*>(W), true, stream_);
        CUDA_OK(cudaStreamSynchronize(stream_));
        download_block(t, dt, ld, col0, dst, K, cols);
    }

    // Full reference-layout tensors in; this shard keeps its slice
    // (column-parallel: wq/wk/wv/w_gate/w_up/head; row-parallel: wo/w_down).
    void load_tensor(int which, const std::string& name, int layer, const float* data, long long rows,
                     long long cols) override {
        ModelDev& M = which ? base_ : draft_;
        ensure_allocated(which);
        const ModelCfg& c = M.c;
        const int d = c.d_model, f = c.d_mlp, V = c.vocab_size, dt = c.weight_dtype;
        const int r = M.rank, fl = M.f_loc(), Vl = M.V_loc();
        auto expect = [&](long long rr, long long cc) {
            if (rows != rr || cols != cc)
                throw Error(ST_SHAPE, "tensor " + name + " expects " + std::to_string(rr) + "x" + std::to_string(cc));
        };
        // columns [c0, c0+n) of a rows x cols host matrix
        auto cslice = [&](long long c0, long long n) {
            std::vector<float> o((size_t)rows * n);
            for (long long i = 0; i < rows; ++i)
                std::memcpy(o.data() + i * n, data + i * cols + c0, sizeof(float) * n);
            return o;
        };
        if (name == "embedding") {
            expect(V, d);
            upload_block(M.emb, dt, d, 0, data, V, d, stream_);
            if (c.tied_head) {
                std::vector<float> t((size_t)d * Vl);
                for (int v = 0; v < Vl; ++v)
                    for (int j = 0; j < d; ++j) t[(size_t)j * Vl + v] = data[(size_t)(r * Vl + v) * d + j];
                mat_write(M.head, dt, d, M.head_ld, 0, t.data(), Vl);
            }
            return;
        }
        if (name == "head") {
            if (c.tied_head) throw Error(ST_CONFIG, "model has a tied head");
            expect(d, V);
            const auto sl = cslice((long long)r * Vl, Vl);
            mat_write(M.head, dt, d, M.head_ld, 0, sl.data(), Vl);
            return;
        }
        if (name == "final_norm_gain") {
            expect(1, d);
            CUDA_OK(cudaMemcpy(M.fgain, data, sizeof(float) * d, cudaMemcpyHostToDevice));
            return;
        }
        if (layer < 0 || layer >= c.n_layers) throw Error(ST_SHAPE, "layer index out of range");
        LayerDev& L = M.L[layer];
        const int qd = M.qdim(), kd = M.kvdim();
        const int qd_full = c.n_heads * c.d_head, kd_full = c.n_kv_heads * c.d_head;
        const int ar = M.arank;  // attention heads of this rank (all of them under lp)
        if (name == "wq") {
            expect(d, qd_full);
            const auto sl = cslice((long long)ar * qd, qd);
            mat_write(L.wqkv, dt, d, M.qkv_ld(), 0, sl.data(), qd);
        } else if (name == "wk") {
            expect(d, kd_full);
            const auto sl = cslice((long long)ar * kd, kd);
            mat_write(L.wqkv, dt, d, M.qkv_ld(), qd, sl.data(), kd);
        } else if (name == "wv") {
            expect(d, kd_full);
            const auto sl = cslice((long long)ar * kd, kd);
            mat_write(L.wqkv, dt, d, M.qkv_ld(), qd + kd, sl.data(), kd);
        } else if (name == "wo") {
            expect(qd_full, d);
            mat_write(L.wo, dt, qd, d, 0, data + (size_t)ar * qd * d, d);
        } else if (name == "w_down") {
            expect(f, d);
            mat_write(L.wd, dt, fl, d, 0, data + (size_t)r * fl * d, d);
        } else if (name == "w_gate" || name == "w_up") {
            // this shard's columns, interleaved per 32 packed columns: [gate16 | up16]
            expect(d, f);
            const int half = name == "w_up" ? 16 : 0;
            std::vector<float> cur((size_t)d * M.gu_N());
            mat_read(L.wgu, dt, d, M.gu_ld(), 0, cur.data(), M.gu_N());
            for (int t = 0; t < fl / 16; ++t)
                for (int i = 0; i < d; ++i)
                    for (int j = 0; j < 16; ++j)
                        cur[(size_t)i * M.gu_N() + t * 32 + half + j] = data[(size_t)i * f + r * fl + t * 16 + j];
            mat_write(L.wgu, dt, d, M.gu_ld(), 0, cur.data(), M.gu_N());
        } else if (name == "attn_norm_gain") {
            expect(1, d);
            CUDA_OK(cudaMemcpy(L.ga, data, sizeof(float) * d, cudaMemcpyHostToDevice));
        } else if (name == "mlp_norm_gain") {
            expect(1, d);
            CUDA_OK(cudaMemcpy(L.gm, data, sizeof(float) * d, cudaMemcpyHostToDevice));
        } else {
            throw Error(ST_CONFIG, "unknown tensor " + name);
        }
    }

    void weight(int which, const std::string& name, int layer, float* out, long long rows, long long cols) override {
        ModelDev& M = which ? base_ : draft_;
        if (M.tp != 1) throw Error(ST_CONFIG, "reading weights back needs tp_size 1");
        const ModelCfg& c = M.c;
        const int d = c.d_model, f = c.d_mlp, dt = c.weight_dtype;
        if (name == "embedding") return download_block(M.emb, dt, d, 0, out, rows, cols);
        if (name == "head") return mat_read(M.head, dt, d, M.head_ld, 0, out, cols);
        if (name == "final_norm_gain") { CUDA_OK(cudaMemcpy(out, M.fgain, 4 * d, cudaMemcpyDeviceToHost)); return; }
        LayerDev& L = M.L.at(layer);
        const int qd = M.qdim(), kd = M.kvdim();
        if (name == "wq") return mat_read(L.wqkv, dt, d, M.qkv_ld(), 0, out, qd);
        if (name == "wk") return mat_read(L.wqkv, dt, d, M.qkv_ld(), qd, out, kd);
        if (name == "wv") return mat_read(L.wqkv, dt, d, M.qkv_ld(), qd + kd, out, kd);
        if (name == "wo") return mat_read(L.wo, dt, qd, d, 0, out, d);
        if (name == "w_down") return mat_read(L.wd, dt, f, d, 0, out, d);
        if (name == "w_gate" || name == "w_up") {
            // one unpack of the interleaved [gate16 | up16] matrix, de-interleaved on the host
            const int half = name == "w_up" ? 16 : 0, ld = M.gu_ld();
            std::vector<float> all((size_t)d * ld);
            mat_read(L.wgu, dt, d, ld, 0, all.data(), ld);
            for (int r = 0; r < d; ++r)
                for (int t = 0; t < f / 16; ++t)
                    for (int j = 0; j < 16; ++j)
                        out[(size_t)r * f + t * 16 + j] = all[(size_t)r * ld + t * 32 + half + j];
            return;
        }
        if (name == "attn_norm_gain") { CUDA_OK(cudaMemcpy(out, L.ga, 4 * d, cudaMemcpyDeviceToHost)); return; }
        if (name == "mlp_norm_gain") { CUDA_OK(cudaMemcpy(out, L.gm, 4 * d, cudaMemcpyDeviceToHost)); return; }
        throw Error(ST_CONFIG, "unknown tensor " + name);
    }

    // ---------------- workspaces ----------------

    void* wsalloc(size_t bytes) {
        void* p = nullptr;
        CUDA_OK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        CUDA_OK(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
        ws_owned_.push_back(p);
        return p;
    }

    void alloc_ws(Workspace& W, const ModelDev& M, int G) {
        const ModelCfg& c = M.c;
        const int d = c.d_model, qd = M.qdim(), f = M.f_loc(), Vl = M.V_loc();
        const int tiles = (d + kStatTile - 1) / kStatTile;
        const int head_ld = M.head_ld ? M.head_ld : ldpad(Vl, c.weight_dtype);
        W.G = G;
        W.h = (float*)wsalloc(sizeof(float) * kChunk * d);
        W.stats = (float*)wsalloc(sizeof(float) * kChunk * tiles);
        W.q = (float*)wsalloc(sizeof(float) * (size_t)G * kChunk * qd);
        W.mixed = (float*)wsalloc(sizeof(float) * (size_t)G * kChunk * qd);
        W.attn = (float*)wsalloc(sizeof(float) * (size_t)G * kChunk * d);
        W.act = (float*)wsalloc(sizeof(float) * (size_t)kChunk * f);
        if (c.weight_dtype == DT_BF16) {
            W.mixed_b16 = (__nv_bfloat16*)wsalloc(sizeof(__nv_bfloat16) * (size_t)G * kChunk * qd);
            W.act_b16 = (__nv_bfloat16*)wsalloc(sizeof(__nv_bfloat16) * (size_t)kChunk * f);
        }
        W.logits = (float*)wsalloc(sizeof(float) * 8 * (size_t)ldpad(c.vocab_size, c.weight_dtype));
        const int dt = c.weight_dtype;
        const int head_tiles = gemv_col_tiles(d, Vl, dt);
        W.am_val = (float*)wsalloc(sizeof(float) * kChunk * head_tiles);
        W.am_idx = (int*)wsalloc(sizeof(int) * kChunk * head_tiles);
        if (M.tp > 1) {
            W.part = (float*)wsalloc(sizeof(float) * kChunk * d);
            W.best_val = (float*)wsalloc(sizeof(float) * kChunk);
            W.best_idx = (int*)wsalloc(sizeof(int) * kChunk);
            W.lg_loc = (float*)wsalloc(sizeof(float) * (size_t)(kMaxNodes + 1) * head_ld);
        }
        size_t part = 0;
        int tick = 0;
        const int shapes[5][2] = {{d, M.qkv_N()}, {qd, d}, {d, 2 * f}, {f, d}, {d, Vl}};
        for (auto& s : shapes) {
            part = std::max(part, gemv_partial_floats(s[0], s[1], dt));
            tick = std::max(tick, gemv_col_tiles(s[0], s[1], dt) + 1);
        }
        W.gemv_part_slot = part;
        W.gemv_ticket_slot = tick;
        if (dt == DT_BF16) {
            const int kmax = std::max(std::max(d, qd), f);
            W.tc_xa = (__nv_bfloat16*)wsalloc(sizeof(__nv_bfloat16) * tc_xa_elems(kChunk, kmax));
            W.tc_rms = (float*)wsalloc(sizeof(float) * kChunk);
            size_t tpf = 0;
            for (auto& sh : shapes) tpf = std::max(tpf, tc_part_floats(sh[0], ldpad(sh[1], dt)));
            if (tpf) {
                W.tc_part = (float*)wsalloc(sizeof(float) * tpf);
                W.tc_tickets = (unsigned*)wsalloc(sizeof(unsigned) * 4096);
            }
        }
        W.gemv_part = (float*)wsalloc(sizeof(float) * part * kMaxProblems);
        W.gemv_tickets = (unsigned*)wsalloc(sizeof(unsigned) * (size_t)tick * kMaxProblems);
        const int cap = c.max_positions + kMaxNodes + kChunk;
        W.attn_ws_slot = attn_ws_floats(kAttnQ, M.qh(), c.d_head, cap);
        W.attn_ticket_slot = (int)attn_tickets(kAttnQ, M.qh(), M.kvh());
        W.attn_ws = (float*)wsalloc(sizeof(float) * W.attn_ws_slot * G);
        W.attn_tickets = (unsigned*)wsalloc(sizeof(unsigned) * (size_t)W.attn_ticket_slot * G);
    }

    // ---------------- forward passes ----------------

    struct Pass {
        PassView view;
        const int* tok_idx = nullptr;
        int T = 0;
    };

    // Stage rows (already appended to the cache bookkeeping) -> device pass.
    // Visibility restates build_tree_mask (proj/src/kv_cache.cpp:43-60)
    // without the dense n x n mask: a staged query sees every committed row,
    // the longest run of leading staged rows that are all its ancestors
    // (vis_end), and any further ancestors as bits of a 64-bit mask over the
    // rows after tree_base (the shortest such run over the pass's queries).
    Pass make_pass(Cache& C, const std::vector<int>& rows, const std::vector<int>& tok_idx) {
        const int T = (int)rows.size();
        const int base = C.committed, S = (int)C.staged.size();
        std::vector<int> pos(T), vis(T), k_run(T, 0);
        std::vector<unsigned long long> anc(T, 0ull);
        std::vector<std::vector<int>> ancestors(T);
        std::vector<char> is_anc(S, 0);
        int k_min = S;
        for (int t = 0; t < T; ++t) {
            const int r = rows[t];
            pos[t] = C.position_of(r);
            if (r < base) {
                vis[t] = r + 1;
                continue;
            }
            std::fill(is_anc.begin(), is_anc.end(), 0);
            for (int node = r; node != kTail; node = C.staged[node - base].parent) {
                is_anc[node - base] = 1;
                ancestors[t].push_back(node);
            }
            int k = 0;
            while (k < S && is_anc[k]) ++k;
            k_run[t] = k;
            vis[t] = base + k;
            k_min = std::min(k_min, k);
        }
        const int tree_base = base + k_min;
        for (int t = 0; t < T; ++t) {
            for (int node : ancestors[t]) {
                if (node < vis[t]) continue;
                const int o = node - tree_base;
                if (o >= 64) throw Error(ST_CONFIG, "tree region exceeds 64 rows");
                anc[t] |= 1ull << o;
            }
        }
        C.ensure(C.total(), stream_);
        Pass p;
        p.T = T;
        p.view.T = T;
        p.view.rows = staging_.push(rows.data(), T, stream_);
        p.view.pos = staging_.push(pos.data(), T, stream_);
        p.view.vis_end = staging_.push(vis.data(), T, stream_);
        p.view.anc = staging_.push(anc.data(), T, stream_);
        p.view.tree_base = tree_base;
        p.view.total = C.total();
        p.view.new_lo = rows.empty() ? 0 : *std::min_element(rows.begin(), rows.end());
        p.tok_idx = staging_.push(tok_idx.data(), T, stream_);
        return p;
    }

    GemvProblem gp(Workspace& W, int slot) {
        GemvProblem p;
        p.partial = W.gemv_part + W.gemv_part_slot * slot;
        p.tickets = W.gemv_tickets + (size_t)W.gemv_ticket_slot * slot;
        p.tc_xa = W.tc_xa;
        p.tc_rms = W.tc_rms;
        p.tc_part = W.tc_part;
        p.tc_tickets = W.tc_tickets;
        return p;
    }

    // ---- per-launch timing of one kernel site (bench roofline evidence)
    template <typename F>
    void site(const ModelDev& M, int kind, double bytes, F&& launch) {
        const int which = &M == &base_ ? 1 : 0;
        const bool on = which == site_which_ && kind == site_kind_ && site_n_ < kSiteEvents;
        if (on) CUDA_OK(cudaEventRecord(site_ev_[2 * site_n_], stream_));
        launch();
        if (on) {
            CUDA_OK(cudaEventRecord(site_ev_[2 * site_n_ + 1], stream_));
            ++site_n_;
            site_bytes_ = bytes;
        }
    }
    void time_site(int which, int kind) override {
        CUDA_OK(cudaStreamSynchronize(stream_));
        site_which_ = which;
        site_kind_ = kind;
        site_n_ = 0;
        site_ms_ = 0;
        site_bytes_ = 0;
    }
    void site_stats(int* count, double* total_ms, double* bytes_per_launch) override {
        CUDA_OK(cudaStreamSynchronize(stream_));
        double tot = 0;
        for (int i = 0; i < site_n_; ++i) {
            float ms = 0;
            CUDA_OK(cudaEventElapsedTime(&ms, site_ev_[2 * i], site_ev_[2 * i + 1]));
            tot += ms;
        }
        *count = site_n_;
        *total_ms = tot;
        *bytes_per_launch = site_bytes_;
    }
    void io_bytes(long long* h2d, long long* d2h) const override {
        *h2d = h2d_bytes_;
        *d2h = d2h_bytes_;
    }
    static int chunks(const ModelDev& M, int T) {
        const int r = gemv_rows_per_launch(M.c.weight_dtype);
        return (T + r - 1) / r;
    }
    static double gemv_bytes(const ModelDev& M, int K, int ldw, int N, int T, int nprob) {
        return (double)nprob * ((double)K * ldw * dsize(M.c.weight_dtype) + 4.0 * T * (K + N));
    }

    // forward_sequential / forward_fuzzy (proj/src/draft_engine.cpp:35-133)
    // Row-parallel projection + residual: h = h + x.W (+ row stats). One GPU:
    // the GEMV's RESID epilogue. Tensor parallel: the GEMV stores this rank's
    // partial, the NVLink all-reduce sums partials in rank order and applies
    // the residual + stats.
    void row_parallel_resid(ModelDev& M, Workspace& W, void* Wm, int K, const float* x, int ldx, int kind, int T,
                            const Pass& ps, const KvView& kv, const float* resid2 = nullptr, int x_bf16 = 0) {
        const int d = M.c.d_model, tiles = (d + kStatTile - 1) / kStatTile, wdt = M.c.weight_dtype;
        GemvBatch b;
        GemvProblem p = gp(W, 0);
        p.W = Wm; p.K = K; p.N = d; p.ldw = d; p.x = x; p.ldx = ldx; p.x_bf16 = x_bf16;
        if (!tp()) {
            p.out = W.h; p.ldo = d; p.resid = W.h; p.ldr = d; p.stats_out = W.stats; p.stat_tiles_out = tiles;
            p.resid2 = resid2; p.ldr2 = d;
            b.p[0] = p;
            g_gemv(M, kind, gemv_bytes(M, K, d, d, T, 1), EPI_RESID, b, 1, T, ps, kv);
            return;
        }
        p.out = W.part; p.ldo = d;
        // bf16 decode GEMV: its epilogue pushes the partial straight into every
        // rank's receive slot (the all-reduce's push fused into the GEMV)
        const bool fused = gemv_fused_push_ok(wdt, T) && (size_t)T * d <= comm_.slot_floats;
        if (fused) set_push(p, 0);
        b.p[0] = p;
        g_gemv(M, kind, gemv_bytes(M, K, d, d, T, 1), EPI_STORE, b, 1, T, ps, kv);
        AllreduceArgs a;
        a.prepushed = fused ? 1 : 0;
        a.rows = T; a.d = d; a.src = W.part; a.ld_src = d; a.mode = AR_RESID;
        a.out = W.h; a.ldo = d; a.resid = W.h; a.ldr = d; a.stats = W.stats; a.stat_tiles = tiles;
        launch_allreduce_rows(comm_, a, stream_);
        ++launches_;
    }

    // GEMV epilogue push targets: every rank's receive slot for the next
    // collective call, rows from `row0` (packed [rows][d])
    void set_push(GemvProblem& p, int row0) {
        p.push_n = comm_.world;
        for (int q = 0; q < comm_.world; ++q) p.push[q] = comm_push_slot(comm_, q) + (size_t)row0 * p.N;
    }

    // forward_sequential / forward_fuzzy (proj/src/draft_engine.cpp:35-133).
    void forward(ModelDev& M, Cache& C, Workspace& W, const LayerPlan* plan, const Pass& ps) {
        forward_body(M, C, W, plan, ps);
    }
    // decode passes whose attention takes the bf16 item path: its output (and
    // the SiLU output) stay bf16 for the O / down GEMVs
    bool attn_b16(const ModelDev& M, int T) const {
        return M.c.weight_dtype == DT_BF16 && M.c.kv_dtype == DT_BF16 && T <= 16 &&
               (M.c.d_head == 64 || M.c.d_head == 128) && b16_acts_;
    }
    std::vector<LayerCapture>* cap_ = nullptr;  // forward_capture in progress

    // ---- launch wrappers
    void g_gemv(ModelDev& M, int kind, double bytes, int epi, const GemvBatch& b, int n, int T, const Pass& ps,
                const KvView& kv) {
        set_sgemv_wide(&M == &draft_ && wide_draft_);
        site(M, kind, bytes, [&] { launch_gemv(epi, M.c.weight_dtype, b, n, T, ps.view, kv, stream_, &pool_); });
        set_sgemv_wide(false);
        launches_ += chunks(M, T);
    }
    void g_embed(ModelDev& M, Workspace& W, const Pass& ps) {
        const int d = M.c.d_model;
        launch_embed(M.c.weight_dtype, M.emb, d, arena_, ps.tok_idx, ps.T, W.h, W.stats, stream_);
        ++launches_;
    }
    void g_add(Workspace& W, const float* a, int d, int T) {
        launch_add_stats(W.h, a, d, T, W.stats, stream_);
        ++launches_;
    }

    void forward_body(ModelDev& M, Cache& C, Workspace& W, const LayerPlan* plan, const Pass& ps) {
        const ModelCfg& c = M.c;
        const int d = c.d_model, T = ps.T, qd = M.qdim(), f = M.f_loc();
        const int tiles = (d + kStatTile - 1) / kStatTile;
        const int wdt = c.weight_dtype;
        const KvView kv = C.view();
        check_comm();
        g_embed(M, W, ps);
        std::vector<std::vector<int>> groups;
        if (plan) groups = plan->groups;
        else
            for (int l = 0; l < c.n_layers; ++l) groups.push_back({l});
        // fuzzy groups: the residual adds h += attn_i ride on the O / down GEMV
        // epilogues (bf16 decode GEMV, one GPU); otherwise separate add kernels
        const bool fuse = wdt == DT_BF16 && !tp() && T <= 16 && fuse_adds_ && !cap_;
        const int b16 = attn_b16(M, T) ? 1 : 0;
        // similarity-probe capture (LayerProbe, proj/include/espec/draft_engine.hpp:24-37):
        // every group takes the unfused path so attn_out exists on its own
        auto grab = [&](std::vector<float>& dst, const float* src, int cols) {
            dst.resize((size_t)T * cols);
            CUDA_OK(cudaMemcpyAsync(dst.data(), src, sizeof(float) * dst.size(), cudaMemcpyDeviceToHost, stream_));
        };
        for (const auto& g : groups) {
            const int n = (int)g.size();
            // layer-parallel placement (the paper layout, ModelDev::lp): this
            // rank runs the attention of the group's layers it owns, full
            // heads, and the group's exchange delivers every slot to every rank
            std::vector<int> sl, sg;  // slots computed here and their layers
            for (int i = 0; i < n; ++i)
                if (!M.lp || M.owner[g[i]] == comm_.rank) {
                    sl.push_back(i);
                    sg.push_back(g[i]);
                }
            const int m = (int)sl.size();
            // attention of every layer in the group reads the group-entry state
            GemvBatch qb;
            for (int j = 0; j < m; ++j) {
                const int i = j;
                GemvProblem p = gp(W, i);
                const LayerDev& L = M.L[sg[j]];
                p.W = L.wqkv; p.K = d; p.N = M.qkv_N(); p.ldw = M.qkv_ld();
                p.x = W.h; p.ldx = d; p.gain = L.ga; p.stats_in = W.stats; p.stat_tiles_in = tiles; p.eps = c.norm_eps;
                p.out = W.q + (size_t)i * kChunk * qd; p.ldo = qd;
                p.n_heads = M.qh(); p.n_kv = M.kvh(); p.dh = c.d_head; p.layer = sg[j]; p.rope = M.rope;
                qb.p[j] = p;
            }
            if (m > 0) {
                g_gemv(M, 0, gemv_bytes(M, d, M.qkv_ld(), M.qkv_N(), T, m), EPI_QKV, qb, m, T, ps, kv);
                if (cap_)
                    for (int i = 0; i < n; ++i) grab((*cap_)[g[i]].q, W.q + (size_t)i * kChunk * qd, qd);
                attention(M, C, W, sg, ps);
            }
            if (n == 1 && !cap_ && !M.lp) {
                row_parallel_resid(M, W, M.L[g[0]].wo, qd, b16 ? (const float*)W.mixed_b16 : W.mixed, qd, 2, T, ps, kv,
                                   nullptr, b16);
            } else {
                // tensor-parallel drafter (not lp): the O partials go straight
                // into the receive slots when one exchange carries the group
                const bool fused = tp() && !M.lp && gemv_fused_push_ok(wdt, T) && (size_t)n * T * d <= comm_.slot_floats;
                if (m > 0) {
                    GemvBatch ob;
                    for (int j = 0; j < m; ++j) {
                        const int i = sl[j];
                        GemvProblem p = gp(W, j);
                        p.W = M.L[sg[j]].wo; p.K = qd; p.N = d; p.ldw = d;
                        p.x = b16 ? (const float*)(W.mixed_b16 + (size_t)j * kChunk * qd) : W.mixed + (size_t)j * kChunk * qd;
                        p.ldx = qd; p.x_bf16 = b16;
                        p.out = W.attn + (size_t)i * kChunk * d; p.ldo = d;
                        if (i == 0 && fuse) {  // h += attn_0 in the epilogue (+ row stats)
                            p.out = W.h; p.resid = W.h; p.ldr = d; p.stats_out = W.stats; p.stat_tiles_out = tiles;
                        }
                        if (fused) set_push(p, i * T);
                        ob.p[j] = p;
                    }
                    g_gemv(M, 2, gemv_bytes(M, qd, d, d, T, m), EPI_STORE, ob, m, T, ps, kv);
                }
                if (cap_)
                    for (int i = 0; i < n; ++i) grab((*cap_)[g[i]].attn_out, W.attn + (size_t)i * kChunk * d, d);
                if (tp()) {
                    // ONE exchange for the whole group's attention outputs: the
                    // sum of the ranks' row-parallel partials (TP), or under the
                    // layer-parallel placement the owners' outputs (every other
                    // rank pushes exact zeros for a slot it does not own)
                    const int per = (size_t)n * T * d <= comm_.slot_floats ? n : 1;
                    for (int i0 = 0; i0 < n; i0 += per) {
                        AllreduceArgs a;
                        a.rows = per * T; a.d = d; a.mode = AR_STORE;
                        a.src = W.attn + (size_t)i0 * kChunk * d; a.ld_src = d;
                        a.out = W.attn + (size_t)i0 * kChunk * d; a.ldo = d;
                        a.rows_per_block = T; a.block_stride = (size_t)kChunk * d;
                        if (M.lp)
                            for (int b = 0; b < per && i0 + b < n; ++b)
                                if (M.owner[g[i0 + b]] != comm_.rank) a.zero_blocks |= 1u << b;
                        a.prepushed = fused ? 1 : 0;
                        launch_allreduce_rows(comm_, a, stream_);
                        ++launches_;
                    }
                }
            }
            // residual / MLP chain stays sequential (proj/src/draft_engine.cpp:112-130)
            for (int i = 0; i < n; ++i) {
                const LayerDev& L = M.L[g[i]];
                // LayerProbe::h_in is the running state before this layer's residual add
                // (proj/src/draft_engine.cpp:112-124)
                if (cap_) grab((*cap_)[g[i]].h_in, W.h, d);
                if ((n > 1 || cap_ || M.lp) && !fuse) {
                    g_add(W, W.attn + (size_t)i * kChunk * d, d, T);
                }
                GemvBatch ub;
                GemvProblem p = gp(W, 0);
                p.W = L.wgu; p.K = d; p.N = M.gu_N(); p.ldw = M.gu_ld();
                p.x = W.h; p.ldx = d; p.gain = L.gm; p.stats_in = W.stats; p.stat_tiles_in = tiles; p.eps = c.norm_eps;
                p.out = b16 ? (float*)W.act_b16 : W.act; p.ldo = f; p.out_bf16 = b16;
                ub.p[0] = p;
                g_gemv(M, 3, gemv_bytes(M, d, M.gu_ld(), 2 * f, T, 1), EPI_SILU, ub, 1, T, ps, kv);
                row_parallel_resid(M, W, L.wd, f, b16 ? (const float*)W.act_b16 : W.act, f, 4, T, ps, kv,
                                   fuse && n > 1 && i + 1 < n ? W.attn + (size_t)(i + 1) * kChunk * d : nullptr, b16);
            }
        }
    }

    void attention(ModelDev& M, Cache& C, Workspace& W, const std::vector<int>& g, const Pass& ps) {
        const int qd = M.qdim();
        const KvView kv = C.view();
        for (int t0 = 0; t0 < ps.T; t0 += kAttnQ) {
            const int tc = std::min(kAttnQ, ps.T - t0);
            PassView v = ps.view;
            v.T = tc;
            v.rows += t0; v.pos += t0; v.vis_end += t0; v.anc += t0;
            AttnBatch ab;
            for (size_t i = 0; i < g.size(); ++i) {
                AttnProblem a;
                a.q = W.q + i * (size_t)kChunk * qd + (size_t)t0 * qd;
                if (attn_b16(M, ps.T)) {
                    a.out = reinterpret_cast<float*>(W.mixed_b16 + i * (size_t)kChunk * qd + (size_t)t0 * qd);
                    a.out_bf16 = 1;
                } else {
                    a.out = W.mixed + i * (size_t)kChunk * qd + (size_t)t0 * qd;
                }
                a.layer = g[i];
                a.ws = W.attn_ws + W.attn_ws_slot * i;
                a.tickets = W.attn_tickets + (size_t)W.attn_ticket_slot * i;
                ab.p[i] = a;
            }
            const double kvb = (double)g.size() * 2.0 * ps.view.total * M.kvdim() * dsize(M.c.kv_dtype);
            site(M, 1, kvb, [&] { launch_attention(ab, (int)g.size(), M.qh(), v, kv, stream_); });
            launches_ += attention_launches(v, kv, M.qh(), (int)g.size());
        }
    }

    // final norm + head over n rows starting at row r0 -> argmax token ids
    // (lm_logits proj/src/model.cpp:212-215, argmax proj/src/matrix.cpp:196-202)
    void head(ModelDev& M, Workspace& W, int r0, int n, int* tok_out, float* logits, int ld_logits = 0) {
        const ModelCfg& c = M.c;
        const int d = c.d_model, tiles = (d + kStatTile - 1) / kStatTile, Vl = M.V_loc();
        if (ld_logits == 0) ld_logits = logits_ld_;
        GemvBatch hb;
        GemvProblem p = gp(W, 0);
        p.W = M.head; p.K = d; p.N = Vl; p.ldw = M.head_ld;
        p.x = W.h + (size_t)r0 * d; p.ldx = d; p.gain = M.fgain; p.stats_in = W.stats + (size_t)r0 * tiles;
        p.stat_tiles_in = tiles; p.eps = c.norm_eps;
        p.vocab = Vl;
        p.am_val = W.am_val; p.am_idx = W.am_idx;
        if (!tp()) {
            p.logits = logits; p.ld_logits = ld_logits; p.tok_out = tok_out;
        } else {
            // vocab-parallel: this rank's slice, then a (max, argmax) gather
            // and, when logits are wanted, a column all-gather over NVLink
            p.logits = logits ? W.lg_loc : nullptr; p.ld_logits = M.head_ld;
            p.tok_out = W.best_idx; p.tok_val = W.best_val; p.col_base = M.rank * Vl;
        }
        hb.p[0] = p;
        PassView none;
        set_sgemv_wide(&M == &draft_ && wide_draft_);
        site(M, 5, gemv_bytes(M, d, M.head_ld, Vl, n, 1),
             [&] { launch_gemv(EPI_ARGMAX, c.weight_dtype, hb, 1, n, none, KvView(), stream_, &pool_); });
        set_sgemv_wide(false);
        launches_ += chunks(M, n);
        if (tp()) {
            launch_allgather_argmax(comm_, n, W.best_val, W.best_idx, tok_out, stream_);
            ++launches_;
            if (logits) {
                GatherColsArgs g;
                g.rows = n; g.cols = Vl; g.src = W.lg_loc; g.ld_src = M.head_ld; g.dst = logits; g.ld_dst = ld_logits;
                launch_allgather_cols(comm_, g, stream_);
                ++launches_;
            }
        }
    }

    // Stage the committed tokens a cache is missing as a chain and run it,
    // in chunks of kChunk rows, committing every chunk but (optionally) the
    // last kept_tail rows. Returns the staged rows of the final chunk.
    std::vector<int> chain_pass(ModelDev& M, Cache& C, Workspace& W, int from, int to, const LayerPlan* plan,
                                bool fuzzy, bool commit_last, int keep_uncommitted) {
        std::vector<int> rows;
        int s = from;
        while (s < to) {
            const int e = std::min(to, s + kChunk);
            const bool last = e == to;
            std::vector<int> parents, tok;
            for (int i = s; i < e; ++i) {
                parents.push_back(i == s ? kTail : C.committed + (i - s) - 1);
                tok.push_back(i);
            }
            rows = C.stage_append(parents, fuzzy);
            Pass ps = make_pass(C, rows, tok);
            // prompt chunks (> 16 rows) run on the tcgen05 prefill GEMM
            set_prefill_mode(e - s > 16);
            forward(M, C, W, plan, ps);
            set_prefill_mode(false);
            if (!last || commit_last) {
                std::vector<int> a, b;
                C.commit_path(rows, a, b);
            }
            s = e;
            (void)keep_uncommitted;
        }
        return rows;
    }

    void begin(const std::vector<int>& tokens) override {
        CUDA_OK(cudaStreamSynchronize(stream_));
        if (!base_allocated_ || !draft_allocated_) throw Error(ST_CONFIG, "models are not initialised");
        for (int t : tokens)
            if (t < 0 || t >= base_.c.vocab_size) cfg_fail("token " + std::to_string(t) + " outside vocabulary");
        if (tokens.empty()) cfg_fail("empty prompt");
        const int needed = (int)tokens.size() + run_.max_new_tokens + run_.n;
        const int room = std::min(base_.c.max_positions, draft_.c.max_positions);
        if (needed > room)
            cfg_fail("prompt plus max_new_tokens exceeds max_positions (" + std::to_string(needed) + " > " +
                     std::to_string(room) + ")");
        committed_ = tokens;
        generated_ = 0;
        it_.phase = 0;
        draft_cached_ = 0;
        clock_ = SimClock(cost_.devices);
        sim_dpre_ = sim_bpre_ = 0;
        rng_ = Xoshiro(run_.seed);  // Generation's RNG (proj/src/orchestrator.cpp:150)
        bcache_.reset();
        dcache_.reset();
        staging_.reset();
        // a launch that ended early (error) may have left claim counters set
        sgemv_pool_reset(pool_, stream_);
        CUDA_OK(cudaMemsetAsync(arena_ + cur_off_, 0, sizeof(int) * 2, stream_));
        CUDA_OK(cudaMemcpyAsync(arena_, committed_.data(), sizeof(int) * committed_.size(), cudaMemcpyHostToDevice,
                                stream_));
        h2d_bytes_ += (long long)(sizeof(int) * committed_.size());
        CUDA_OK(cudaStreamSynchronize(stream_));
    }

    bool done() const override { return generated_ >= run_.max_new_tokens; }

    IterationTrace step(std::vector<int>& emitted) override {
        if (committed_.empty()) throw Error(ST_CONFIG, "call begin() first");
        IterationTrace tr = run_.algorithm == ALG_VANILLA ? step_vanilla(emitted) : step_speculative(emitted);
        tr.committed = (int)committed_.size();
        tr.draft_committed = dcache_.committed;
        tr.base_committed = bcache_.committed;
        return tr;
    }

    // ---- T > 0: the iteration's uniforms, drawn from a copy of the stream;
    // the stream is advanced by what the device consumed (sync_outcome).
    void upload_uniforms(int n) {
        Xoshiro copy = rng_;
        for (int i = 0; i < n; ++i) unif_host_[i] = copy.uniform();
        CUDA_OK(cudaMemcpyAsync(unif_dev_, unif_host_, sizeof(double) * n, cudaMemcpyHostToDevice, stream_));
        h2d_bytes_ += (long long)sizeof(double) * n;
    }
    void reset_flags() {
        CUDA_OK(cudaMemsetAsync(arena_ + cur_off_, 0, sizeof(int) * 2, stream_));
    }
    // read {m, bonus, path, tokens, cursor, err} back (one D2H per iteration)
    void sync_outcome(int n_levels) {
        const int lo = out_off_, n_out = 2 + 2 * n_levels;
        CUDA_OK(cudaMemcpyAsync(outcome_host_, arena_ + lo, sizeof(int) * (size_t)(err_off_ - lo + 1),
                                cudaMemcpyDeviceToHost, stream_));
        d2h_bytes_ += (long long)sizeof(int) * n_out;
        CUDA_OK(cudaEventRecord(ev_[3], stream_));
        CUDA_OK(cudaEventSynchronize(ev_[3]));
        CUDA_OK(cudaGetLastError());
        const int err = outcome_host_[err_off_ - lo];
        static const char* msgs[] = {"", "softmax input contains a non-finite logit",
                                     "draft distribution exhausted before the tree width",
                                     "drafted token carries zero draft probability",
                                     "sibling candidates exhaust the draft distribution",
                                     "sampling from an all-zero distribution"};
        if (err == kCommErrTimeout) throw Error(ST_NCCL, "tensor-parallel collective: a peer never arrived");
        if (err == 1) throw Error(ST_DOMAIN, msgs[1]);
        if (err > 1 && err <= 5) throw Error(ST_CHECK, msgs[err]);
        const int used = outcome_host_[cur_off_ - lo];
        for (int i = 0; i < used; ++i) (void)rng_.next();
    }
    // softmax_temp of `rows` logits rows (row i of src at dist index first+i)
    void softmax(const float* logits, float* dists, int first, int rows, int V) {
        std::vector<int> idx(rows);
        for (int i = 0; i < rows; ++i) idx[i] = first + i;
        SoftmaxArgs a;
        a.logits = logits;
        a.ld_logits = logits_ld_;
        a.src_row = staging_.push(idx.data(), rows, stream_);
        a.dists = dists;
        a.ld_dists = V;
        a.dst_row = a.src_row;
        a.vocab = V;
        a.temperature = run_.temperature;
        a.err = arena_ + err_off_;
        launch_softmax_rows(a, rows, stream_);
        ++launches_;
    }

    // run_iteration_vanilla (proj/src/orchestrator.cpp:438-468)
    IterationTrace step_vanilla(std::vector<int>& emitted) {
        IterationTrace tr;
        staging_.reset();
        const bool sampled = run_.temperature > 0.f;
        if (sampled) {
            upload_uniforms(1);
            reset_flags();
        }
        CUDA_OK(cudaEventRecord(ev_[0], stream_));
        const int n0 = (int)committed_.size();
        {  // sim_base_forward over the uncached suffix (orchestrator.cpp:441-466)
            const double before = clock_.stage_elapsed(SIM_VERIFY);
            sim_base_forward(cost_, base_.c.n_layers, n0 - bcache_.committed + sim_bpre_, clock_, SIM_VERIFY);
            sim_bpre_ = 0;
            tr.verify_sim = clock_.stage_elapsed(SIM_VERIFY) - before;
        }
        // the prompt but its last token is prefilled (tcgen05 when long); the
        // last token always goes through a decode-sized pass, exactly like the
        // frontier row of a speculative verify, so greedy outputs agree
        if (n0 - 1 > bcache_.committed)
            chain_pass(base_, bcache_, bws_, bcache_.committed, n0 - 1, nullptr, false, true, 0);
        std::vector<int> rows = chain_pass(base_, bcache_, bws_, bcache_.committed, n0, nullptr, false, false, 0);
        const int V = base_.c.vocab_size;
        if (!sampled) {
            head(base_, bws_, (int)rows.size() - 1, 1, arena_ + n0, nullptr);
            CUDA_OK(cudaMemcpyAsync(outcome_host_, arena_ + n0, sizeof(int), cudaMemcpyDeviceToHost, stream_));
            d2h_bytes_ += sizeof(int);
            if (tp()) {  // a collective timeout is reported through the error slot
                CUDA_OK(cudaMemcpyAsync(outcome_host_ + (err_off_ - out_off_), arena_ + err_off_, sizeof(int),
                                        cudaMemcpyDeviceToHost, stream_));
                d2h_bytes_ += sizeof(int);
            }
            CUDA_OK(cudaEventRecord(ev_[3], stream_));
            CUDA_OK(cudaEventSynchronize(ev_[3]));
            CUDA_OK(cudaGetLastError());
            if (tp() && outcome_host_[err_off_ - out_off_] == kCommErrTimeout)
                throw Error(ST_NCCL, "tensor-parallel collective: a peer never arrived");
        } else {
            // sample_from(softmax_temp(logits)) (orchestrator.cpp:457-460)
            head(base_, bws_, (int)rows.size() - 1, 1, arena_ + am_off_, blogits_);
            softmax(blogits_, bdists_, 0, 1, V);
            VerifyArgs va;
            va.vocab = V;
            va.n_levels = 0;
            va.tok_arena = arena_;
            va.base_dists = bdists_;
            va.draft_dists = ddists_;
            va.ld_dists = V;
            va.target = target_;
            va.uniforms = unif_dev_;
            va.cursor = arena_ + cur_off_;
            va.outcome = arena_ + out_off_;
            va.tok_arena_w = arena_;
            va.commit_at = n0;
            va.err = arena_ + err_off_;
            launch_verify_sample(va, stream_);
            ++launches_;
            sync_outcome(0);
            outcome_host_[0] = outcome_host_[1];
        }
        std::vector<int> a, b;
        bcache_.commit_path(rows, a, b);
        const int next = outcome_host_[0];
        committed_.push_back(next);
        emitted.push_back(next);
        ++generated_;
        tr.emitted = 1;
        tr.base_forwards = 1;
        tr.bonus = next;
        CUDA_OK(cudaEventElapsedTime(&tr.verify_ms, ev_[0], ev_[3]));
        return tr;
    }

    // ---- one speculative iteration, split into the reference's stages
    // (Generation::run_iteration_speculative, proj/src/orchestrator.cpp:407-436):
    // stage_calibrate = drafter_leading_pass (256-300), stage_draft =
    // draft_stage / draft_tree (302-331), stage_verify = verify_stage +
    // verify_tree (333-388), stage_resolve = resolve_draft_cache (390-405),
    // stage_commit = the commit/emit tail of run_iteration_speculative
    // (414-428). step() runs all five back to back; the C ABI exposes each.
    struct Node { int parent, depth, prob_index, first_child = -1, n_children = 0, cache_row = -1; };
    struct Iter {
        int phase = 0;  // 0 idle, 1 calibrated, 2 drafted, 3 verified, 4 resolved
        uint64_t id = 0;
        IterationTrace tr;
        bool easy = false, calibrated = false, fuzzy_lead = false, sampled = false, need_logits = false;
        int n_comm = 0, lead_T = 0, n_dists = 0;
        std::vector<Node> nodes;
        std::vector<int> chain_rows, node_rows;
        int m = 0, bonus = 0;
        std::vector<int> path, acc_tokens;
    } it_;
    uint64_t iter_seq_ = 0;

    void expect_phase(int want, const char* stage) {
        if (committed_.empty()) throw Error(ST_CONFIG, "call begin() / prefill() first");
        if (run_.algorithm == ALG_VANILLA) throw Error(ST_CONFIG, std::string(stage) + ": vanilla runs no speculative stages");
        if (it_.phase == 5) throw Error(ST_STRUCTURE, std::string(stage) + ": the iteration failed; call begin() / prefill()");
        if (it_.phase != want) {
            static const char* names[] = {"commit_outcome", "calibrate", "draft", "verify", "resolve_draft_cache"};
            throw Error(ST_STRUCTURE, std::string(stage) + " called out of order (after " + names[it_.phase] + ")");
        }
    }

    // drafter_leading_pass (orchestrator.cpp:256-300): the uncached committed
    // suffix (prompt on iteration 0, else accepted + bonus) through one
    // precise pass (fuzzy in the no-calibration arm), committed; root logits
    // = head of its last row. Greedy chains take the level-1 token straight
    // from the head's argmax epilogue (select_children with k = 1).
    void stage_calibrate(float* root_logits_host) {
        expect_phase(0, "calibrate");
        Iter& I = it_;
        I = Iter();
        I.id = ++iter_seq_;
        I.tr.n = run_.n;
        staging_.reset();
        I.easy = run_.algorithm == ALG_EASYSPEC;
        I.calibrated = I.easy && run_.calibration;
        I.fuzzy_lead = I.easy && !run_.calibration;
        I.sampled = run_.temperature > 0.f;
        bool wide = false;
        for (int w : widths_) wide |= w > 1;
        I.need_logits = I.sampled || wide;  // else: argmax straight from the head epilogue
        I.n_comm = (int)committed_.size();
        if (I.sampled) {
            long long nodes = 0, level = 1;
            for (int w : widths_) nodes += (level *= w);
            upload_uniforms((int)std::min<long long>(kMaxDraws, 2 * nodes + 2));
        }
        reset_flags();
        CUDA_OK(cudaEventRecord(ev_[0], stream_));
        std::vector<int> lead_rows = chain_pass(draft_, dcache_, dws_, draft_cached_, I.n_comm,
                                                I.fuzzy_lead ? &plan_ : nullptr, I.fuzzy_lead, true, 0);
        draft_cached_ = I.n_comm;
        if (I.fuzzy_lead) ++I.tr.fuzzy_forwards;
        else ++I.tr.sequential_forwards;
        I.lead_T = (int)lead_rows.size();
        {  // StageSimDelta of drafter_leading_pass (orchestrator.cpp:262-298)
            const int stage = I.calibrated ? SIM_CALIBRATE : SIM_DRAFT;
            const double before = clock_.stage_elapsed(stage);
            const int s_rows = I.lead_T + sim_dpre_;
            sim_dpre_ = 0;
            if (I.fuzzy_lead) sim_fuzzy_draft_forward(cost_, plan_, s_rows, clock_, stage);
            else sim_sequential_draft_forward(cost_, draft_.c.n_layers, s_rows, clock_, stage);
            (I.calibrated ? I.tr.calibrate_sim : I.tr.draft_sim) += clock_.stage_elapsed(stage) - before;
        }
        const bool store = I.need_logits || root_logits_host;
        head(draft_, dws_, I.lead_T - 1, 1, I.need_logits ? arena_ + am_off_ : arena_ + tree_off_,
             store ? dlogits_ : nullptr);
        CUDA_OK(cudaEventRecord(ev_[1], stream_));
        if (root_logits_host) {
            const int V = draft_.c.vocab_size;
            CUDA_OK(cudaMemcpyAsync(root_logits_host, dlogits_, sizeof(float) * V, cudaMemcpyDeviceToHost, stream_));
            d2h_bytes_ += (long long)sizeof(float) * V;
            CUDA_OK(cudaStreamSynchronize(stream_));
        }
        I.phase = 1;
    }

    // draft_tree (proj/src/draft_engine.cpp:188-289): level-1 children from
    // the root row, then n-1 token-parallel passes (fuzzy under the plan for
    // EasySpec), the last level selected but never forwarded. Host tree
    // shape: nodes level by level, siblings contiguous; tokens live on device.
    // Dist index 0 = the root row, then one per forwarded frontier row.
    void stage_draft() {
        expect_phase(1, "draft");
        Iter& I = it_;
        const int V = draft_.c.vocab_size;
        std::vector<Node>& nodes = I.nodes;
        std::vector<int> frontier;
        for (int i = 0; i < widths_[0]; ++i) {
            nodes.push_back({-1, 1, 0});
            frontier.push_back(i);
        }
        I.n_dists = 1;
        if (I.need_logits) select_level(0, 1, {widths_[0]}, {0}, V);
        const double sim_before = clock_.stage_elapsed(SIM_DRAFT);  // draft_stage's StageSimDelta (302-331)
        for (int level = 1; level <= run_.n - 1 && !frontier.empty(); ++level) {
            std::vector<int> parents, tok;
            for (int idx : frontier) {
                const Node& nd = nodes[idx];
                parents.push_back(nd.parent < 0 ? kTail : nodes[nd.parent].cache_row);
                tok.push_back(tree_off_ + idx);
            }
            std::vector<int> rows = dcache_.stage_append(parents, I.easy);
            for (size_t i = 0; i < frontier.size(); ++i) nodes[frontier[i]].cache_row = rows[i];
            Pass ps = make_pass(dcache_, rows, tok);
            forward(draft_, dcache_, dws_, I.easy ? &plan_ : nullptr, ps);
            if (I.easy) ++I.tr.fuzzy_forwards;
            else ++I.tr.sequential_forwards;
            // one simulated forward per forwarded level of frontier-size rows
            if (I.easy) sim_fuzzy_draft_forward(cost_, plan_, (int)frontier.size(), clock_, SIM_DRAFT);
            else sim_sequential_draft_forward(cost_, draft_.c.n_layers, (int)frontier.size(), clock_, SIM_DRAFT);
            std::vector<int> next, first_child, widths;
            const int dist0 = I.n_dists;
            for (size_t i = 0; i < frontier.size(); ++i) {
                const int idx = frontier[i];
                nodes[idx].first_child = (int)nodes.size();
                nodes[idx].n_children = widths_[level];
                first_child.push_back((int)nodes.size());
                widths.push_back(widths_[level]);
                for (int k = 0; k < widths_[level]; ++k) {
                    nodes.push_back({idx, level + 1, dist0 + (int)i});
                    next.push_back((int)nodes.size() - 1);
                }
            }
            const int nf = (int)frontier.size();
            if (!I.need_logits) {
                // width 1: children of consecutive frontier rows are consecutive nodes
                head(draft_, dws_, 0, nf, arena_ + tree_off_ + first_child[0], nullptr);
            } else {
                head(draft_, dws_, 0, nf, arena_ + am_off_, dlogits_ + (size_t)dist0 * logits_ld_);
                select_level(dist0, nf, widths, first_child, V);
            }
            I.n_dists += nf;
            frontier = next;
        }
        I.tr.draft_sim += clock_.stage_elapsed(SIM_DRAFT) - sim_before;
        I.tr.drafted_nodes = (int)nodes.size();
        CUDA_OK(cudaEventRecord(ev_[2], stream_));
        I.phase = 2;
    }

    // The drafted tree as the reference's DraftTree (draft_engine.hpp:63-84).
    // One D2H copy of the node tokens (and, on request, the draft
    // distributions: softmax_temp rows, one-hot at T = 0).
    void read_tree(TreeOut& out, bool want_dists) {
        if (it_.phase < 2) throw Error(ST_STRUCTURE, "no drafted tree (call draft first)");
        const Iter& I = it_;
        const int nn = (int)I.nodes.size(), V = draft_.c.vocab_size;
        out = TreeOut();
        out.id = I.id;
        out.widths = widths_;
        out.token.resize(nn);
        CUDA_OK(cudaMemcpyAsync(out.token.data(), arena_ + tree_off_, sizeof(int) * nn, cudaMemcpyDeviceToHost,
                                stream_));
        d2h_bytes_ += (long long)sizeof(int) * nn;
        out.n_dists = I.n_dists;
        if (want_dists && I.sampled) {
            out.dists.resize((size_t)I.n_dists * V);
            CUDA_OK(cudaMemcpyAsync(out.dists.data(), ddists_, sizeof(float) * out.dists.size(), cudaMemcpyDeviceToHost,
                                    stream_));
            d2h_bytes_ += (long long)sizeof(float) * out.dists.size();
        }
        CUDA_OK(cudaStreamSynchronize(stream_));
        for (int j = 0; j < nn; ++j) {
            const Node& n = I.nodes[j];
            out.parent.push_back(n.parent);
            out.depth.push_back(n.depth);
            out.prob_index.push_back(n.prob_index);
            out.cache_row.push_back(n.cache_row);
            out.first_child.push_back(n.first_child);
            out.n_children.push_back(n.n_children);
            if (n.parent < 0) ++out.root_children;
        }
        if (want_dists && !I.sampled) {
            // T = 0: softmax_temp is a one-hot at the first maximum, i.e. at
            // the row's top-1 child (select_children's first pick)
            out.dists.assign((size_t)I.n_dists * V, 0.f);
            std::vector<int> first(I.n_dists, -1);
            for (int j = 0; j < nn; ++j)
                if (first[I.nodes[j].prob_index] < 0) first[I.nodes[j].prob_index] = j;
            for (int d = 0; d < I.n_dists; ++d)
                if (first[d] >= 0) out.dists[(size_t)d * V + out.token[first[d]]] = 1.f;
        }
    }

    // verify_stage (orchestrator.cpp:333-388) + verify_tree (verifier.cpp:86-177).
    // `caller` (optional) is a tree the caller may have edited: its shape must
    // be the drafted one; its tokens replace the drafted tokens.
    void stage_verify(const TreeOut* caller) {
        expect_phase(2, "verify");
        Iter& I = it_;
        const int nn = (int)I.nodes.size(), V = base_.c.vocab_size;
        if (caller) {
            if (caller->id != I.id) throw Error(ST_STRUCTURE, "tree does not belong to this iteration's draft");
            if ((int)caller->token.size() != nn || (int)caller->parent.size() != nn)
                throw Error(ST_SHAPE, "tree node count differs from the drafted tree");
            for (int j = 0; j < nn; ++j) {
                if (caller->parent[j] != I.nodes[j].parent)
                    throw Error(ST_STRUCTURE, "tree shape differs from the drafted tree");
                if (caller->token[j] < 0 || caller->token[j] >= V) cfg_fail("tree token outside vocabulary");
            }
            CUDA_OK(cudaMemcpyAsync(arena_ + tree_off_, staging_.push(caller->token.data(), nn, stream_),
                                    sizeof(int) * nn, cudaMemcpyDeviceToDevice, stream_));
        }
        const int n_comm = I.n_comm;
        {  // verify_stage's StageSimDelta (orchestrator.cpp:336-386): one base
           // forward over the uncached suffix plus the tree nodes
            const double before = clock_.stage_elapsed(SIM_VERIFY);
            sim_base_forward(cost_, base_.c.n_layers, n_comm - bcache_.committed + sim_bpre_ + nn, clock_, SIM_VERIFY);
            sim_bpre_ = 0;
            I.tr.verify_sim += clock_.stage_elapsed(SIM_VERIFY) - before;
        }
        // committed tokens the base has no rows for: all but the frontier token
        // are prefilled chunk-wise first (equivalent to one pass: causal rows).
        if (n_comm - 1 > bcache_.committed)
            chain_pass(base_, bcache_, bws_, bcache_.committed, n_comm - 1, nullptr, false, true, 0);
        std::vector<int> parents, tok;
        parents.push_back(kTail);
        tok.push_back(n_comm - 1);
        I.chain_rows = bcache_.stage_append(parents, false);
        const int first_node_row = I.chain_rows.back() + 1;
        parents.clear();
        for (int j = 0; j < nn; ++j)
            parents.push_back(I.nodes[j].parent < 0 ? I.chain_rows.back() : first_node_row + I.nodes[j].parent);
        I.node_rows = bcache_.stage_append(parents, false);
        std::vector<int> all_rows = I.chain_rows;
        all_rows.insert(all_rows.end(), I.node_rows.begin(), I.node_rows.end());
        for (int j = 0; j < nn; ++j) tok.push_back(tree_off_ + j);
        Pass ps = make_pass(bcache_, all_rows, tok);
        forward(base_, bcache_, bws_, nullptr, ps);
        ++I.tr.base_forwards;
        head(base_, bws_, 0, 1 + nn, arena_ + am_off_, I.sampled ? blogits_ : nullptr);
        // acceptance on device
        std::vector<int> np(nn), nfc(nn), nnc(nn), nti(nn), npi(nn);
        int root_children = 0;
        for (int j = 0; j < nn; ++j) {
            np[j] = I.nodes[j].parent;
            nfc[j] = I.nodes[j].first_child;
            nnc[j] = I.nodes[j].n_children;
            nti[j] = tree_off_ + j;
            npi[j] = I.nodes[j].prob_index;
            if (I.nodes[j].parent < 0) ++root_children;
        }
        if (!I.sampled) {
            AcceptArgs aa;
            aa.n_nodes = nn;
            aa.n_levels = run_.n;
            aa.root_children = root_children;
            aa.node_parent = staging_.push(np.data(), nn, stream_);
            aa.node_first_child = staging_.push(nfc.data(), nn, stream_);
            aa.node_n_children = staging_.push(nnc.data(), nn, stream_);
            aa.node_tok_idx = staging_.push(nti.data(), nn, stream_);
            aa.tok_arena = arena_;
            aa.base_argmax = arena_ + am_off_;
            aa.outcome = arena_ + out_off_;
            aa.tok_arena_w = arena_;
            aa.commit_at = n_comm;
            aa.strict_siblings = run_.strict_greedy_tree;
            aa.err = arena_ + err_off_;
            launch_accept_greedy(aa, stream_);
        } else {
            softmax(blogits_, bdists_, 0, 1 + nn, V);
            VerifyArgs va;
            va.vocab = V;
            va.n_levels = run_.n;
            va.root_children = root_children;
            va.node_first_child = staging_.push(nfc.data(), nn, stream_);
            va.node_n_children = staging_.push(nnc.data(), nn, stream_);
            va.node_tok_idx = staging_.push(nti.data(), nn, stream_);
            va.node_prob_index = staging_.push(npi.data(), nn, stream_);
            va.tok_arena = arena_;
            va.base_dists = bdists_;
            va.draft_dists = ddists_;
            va.ld_dists = V;
            va.target = target_;
            va.uniforms = unif_dev_;
            va.cursor = arena_ + cur_off_;
            va.outcome = arena_ + out_off_;
            va.tok_arena_w = arena_;
            va.commit_at = n_comm;
            va.err = arena_ + err_off_;
            launch_verify_sample(va, stream_);
        }
        ++launches_;
        try {
            sync_outcome(run_.n);
        } catch (...) {
            // the iteration is void (its rows stay staged): only begin() recovers
            I.phase = 5;
            throw;
        }
        I.m = outcome_host_[0];
        I.bonus = outcome_host_[1];
        I.path.assign(outcome_host_ + 2, outcome_host_ + 2 + I.m);
        I.acc_tokens.assign(outcome_host_ + 2 + run_.n, outcome_host_ + 2 + run_.n + I.m);
        // base keeps the chain + accepted path (orchestrator.cpp:379-383)
        std::vector<int> commit_rows = I.chain_rows;
        for (int ni : I.path) commit_rows.push_back(I.node_rows[ni]);
        std::vector<int> src, dst;
        bcache_.commit_path(commit_rows, src, dst);
        move_rows(bcache_, src, dst);
        I.phase = 3;
    }

    // resolve_draft_cache (orchestrator.cpp:390-405)
    void stage_resolve() {
        expect_phase(3, "resolve_draft_cache");
        Iter& I = it_;
        if (I.calibrated) {
            dcache_.discard();
        } else {
            std::vector<int> drows, src, dst;
            for (int ni : I.path) {
                if (I.nodes[ni].cache_row < 0) break;  // the last level is never staged
                drows.push_back(I.nodes[ni].cache_row);
            }
            dcache_.commit_path(drows, src, dst);
            move_rows(dcache_, src, dst);
            draft_cached_ += (int)drows.size();
        }
        I.phase = 4;
    }

    // run_iteration_speculative's tail (orchestrator.cpp:414-428): commit
    // accepted + bonus, emit min(m + 1, remaining).
    IterationTrace stage_commit(std::vector<int>& emitted) {
        expect_phase(4, "commit_outcome");
        Iter& I = it_;
        for (int t : I.acc_tokens) committed_.push_back(t);
        committed_.push_back(I.bonus);
        const int remaining = run_.max_new_tokens - generated_;
        const int emit = std::min(I.m + 1, remaining);
        for (int i = 0; i < emit; ++i) emitted.push_back(committed_[committed_.size() - (I.m + 1) + i]);
        generated_ += emit;
        IterationTrace tr = I.tr;
        tr.m = I.m;
        tr.emitted = emit;
        tr.bonus = I.bonus;
        float ms = 0;
        CUDA_OK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        if (I.calibrated) tr.calibrate_ms = ms;
        else tr.draft_ms = ms;
        CUDA_OK(cudaEventElapsedTime(&ms, ev_[1], ev_[2]));
        tr.draft_ms += ms;
        CUDA_OK(cudaEventElapsedTime(&tr.verify_ms, ev_[2], ev_[3]));
        tr.committed = (int)committed_.size();
        tr.draft_committed = dcache_.committed;
        tr.base_committed = bcache_.committed;
        I.phase = 0;
        return tr;
    }

    IterationTrace step_speculative(std::vector<int>& emitted) {
        stage_calibrate(nullptr);
        stage_draft();
        stage_verify(nullptr);
        stage_resolve();
        return stage_commit(emitted);
    }

    // ---- Engine stage interface (C ABI espec_prefill ... espec_commit_outcome)
    void prefill(const std::vector<int>& tokens) override {
        begin(tokens);
        const int n = (int)tokens.size();
        // base: every prompt row but the frontier token (verify_stage re-inputs
        // it with the tree); drafter: the whole chunks before the final one, so
        // the leading pass runs exactly the chunk step() would run.
        if (n - 1 > 0) chain_pass(base_, bcache_, bws_, 0, n - 1, nullptr, false, true, 0);
        sim_bpre_ = n - 1;
        const int dpre = ((n - 1) / kChunk) * kChunk;
        if (dpre > 0 && run_.algorithm != ALG_VANILLA) {
            chain_pass(draft_, dcache_, dws_, 0, dpre, nullptr, false, true, 0);
            draft_cached_ = dpre;
            sim_dpre_ = dpre;
        }
        CUDA_OK(cudaStreamSynchronize(stream_));
    }
    void calibrate(float* root_logits) override { stage_calibrate(root_logits); }
    void draft(TreeOut* out, bool want_dists) override {
        stage_draft();
        if (out) read_tree(*out, want_dists);
    }
    void tree(TreeOut& out, bool want_dists) override { read_tree(out, want_dists); }
    void verify(const TreeOut* caller, OutcomeOut* out) override {
        stage_verify(caller);
        if (out) {
            out->m = it_.m;
            out->n = run_.n;
            out->bonus = it_.bonus;
            out->path = it_.path;
            out->tokens = it_.acc_tokens;
            out->id = it_.id;
        }
    }
    void resolve_draft_cache(const OutcomeOut* o) override {
        if (o && (o->id != it_.id || o->m != it_.m || o->path != it_.path))
            throw Error(ST_STRUCTURE, "outcome does not belong to this iteration's verification");
        stage_resolve();
    }
    IterationTrace commit_outcome(std::vector<int>& emitted) override { return stage_commit(emitted); }

    // select_children (proj/src/draft_engine.cpp:141-186) for `rows`
    // frontier rows whose logits sit at dist indices [dist0, dist0+rows):
    // T = 0 top-k of the logits; T > 0 softmax_temp, then draws without
    // replacement consuming the iteration's uniforms in row order.
    void select_level(int dist0, int rows, const std::vector<int>& widths, const std::vector<int>& first_node, int V) {
        const bool sampled = run_.temperature > 0.f;
        if (sampled) softmax(dlogits_, ddists_, dist0, rows, V);
        std::vector<int> idx(rows), child_at(rows);
        for (int i = 0; i < rows; ++i) {
            idx[i] = dist0 + i;
            child_at[i] = tree_off_ + first_node[i];
        }
        SelectArgs a;
        a.rows = rows;
        a.vocab = V;
        a.temperature = run_.temperature;
        a.logits = dlogits_;
        a.ld_logits = logits_ld_;
        a.logit_row = staging_.push(idx.data(), rows, stream_);
        a.dists = ddists_;
        a.ld_dists = V;
        a.dist_row = a.logit_row;
        a.width = staging_.push(widths.data(), rows, stream_);
        a.child_at = staging_.push(child_at.data(), rows, stream_);
        a.tok_arena = arena_;
        a.uniforms = unif_dev_;
        a.cursor = arena_ + cur_off_;
        a.err = arena_ + err_off_;
        launch_select_children(a, stream_);
        ++launches_;
    }

    void move_rows(Cache& C, const std::vector<int>& src, const std::vector<int>& dst) {
        if (src.empty()) return;
        const int* s = staging_.push(src.data(), src.size(), stream_);
        const int* d = staging_.push(dst.data(), dst.size(), stream_);
        launch_kv_move(C.view(), s, d, (int)src.size(), stream_);
        ++launches_;
    }

    std::vector<int> generate(const std::vector<int>& tokens, std::vector<IterationTrace>* traces) override {
        begin(tokens);
        std::vector<int> out;
        while (!done()) {
            IterationTrace t = step(out);
            if (traces) traces->push_back(t);
        }
        return out;
    }

    // prefix_distribution (proj/src/orchestrator.cpp:494-526): `runs`
    // independent generations of run.max_new_tokens tokens; run r is seeded
    // SplitMix64(seed + 0x9E37 (r + 1)).next() exactly as the reference, so
    // the empirical law is comparable run for run. Runs are serial on this
    // engine's stream (the reference spreads them over host threads).
    // first / stride select one host thread's share of the reference's loop
    // (`for r = thread_index; r < runs; r += n_threads`).
    std::map<std::vector<int>, long> prefix_distribution(const std::vector<int>& tokens, long runs, long first,
                                                         long stride) override {
        if (runs <= 0) cfg_fail("prefix_distribution needs runs > 0");
        if (first < 0 || stride < 1) cfg_fail("prefix_distribution: first >= 0 and stride >= 1");
        const RunCfg saved = run_;
        std::map<std::vector<int>, long> out;
        try {
            for (long r = first; r < runs; r += stride) {
                uint64_t z = saved.seed + 0x9E37ULL * (uint64_t)(r + 1) + 0x9E3779B97F4A7C15ULL;
                z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
                z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
                run_.seed = z ^ (z >> 31);
                ++out[generate(tokens, nullptr)];
            }
        } catch (...) {
            run_ = saved;
            throw;
        }
        run_ = saved;
        return out;
    }

    void forward_chain(int which, const std::vector<int>& tokens, const std::string& plan_spec, float* logits,
                       float* hidden) override {
        ModelDev& M = which ? base_ : draft_;
        Cache& C = which ? bcache_ : dcache_;
        Workspace& W = which ? bws_ : dws_;
        CUDA_OK(cudaStreamSynchronize(stream_));
        LayerPlan plan;
        const LayerPlan* pp = nullptr;
        if (!plan_spec.empty()) {
            plan = plan_spec.rfind("lp=", 0) == 0 ? plan_groups(M.c.n_layers, std::stoi(plan_spec.substr(3)))
                                                  : parse_plan_override(plan_spec);
            if (plan.n_layers() != M.c.n_layers) cfg_fail("plan does not cover the model");
            if (plan.max_group_size() > kMaxGroup && which == 0) cfg_fail("group too large");
            pp = &plan;
        }
        if (pp && which == 1 && plan.max_group_size() > 1) cfg_fail("fuzzy probes run on the drafter");
        C.reset();
        staging_.reset();
        const int n = (int)tokens.size();
        if (n > kChunk) cfg_fail("forward_chain probes are limited to 256 tokens");
        CUDA_OK(cudaMemcpyAsync(arena_, tokens.data(), sizeof(int) * n, cudaMemcpyHostToDevice, stream_));
        std::vector<int> parents, tok;
        for (int i = 0; i < n; ++i) {
            parents.push_back(i == 0 ? kTail : i - 1);
            tok.push_back(i);
        }
        std::vector<int> rows = C.stage_append(parents, pp != nullptr);
        Pass ps = make_pass(C, rows, tok);
        set_prefill_mode(n > 16);  // same rule as chain_pass
        forward(M, C, W, pp, ps);
        set_prefill_mode(false);
        const int d = M.c.d_model, V = M.c.vocab_size;
        if (hidden) CUDA_OK(cudaMemcpyAsync(hidden, W.h, sizeof(float) * n * d, cudaMemcpyDeviceToHost, stream_));
        for (int r0 = 0; r0 < n; r0 += 8) {
            const int k = std::min(8, n - r0);
            head(M, W, r0, k, arena_ + out_off_, W.logits, ldpad(M.c.vocab_size, M.c.weight_dtype));
            if (logits)
                CUDA_OK(cudaMemcpy2DAsync(logits + (size_t)r0 * V, sizeof(float) * V, W.logits,
                                          sizeof(float) * ldpad(M.c.vocab_size, M.c.weight_dtype),
                                          sizeof(float) * V, k, cudaMemcpyDeviceToHost, stream_));
        }
        std::vector<int> a, b;
        C.commit_path(rows, a, b);
        CUDA_OK(cudaStreamSynchronize(stream_));
        CUDA_OK(cudaGetLastError());
        committed_.clear();
    }

    // Parity probe at decode shapes: prefill `prompt` (chunked; tcgen05 for
    // > 16-row chunks), then ONE decode-sized pass over T staged rows whose
    // tree is given by `parents` (-1 = child of the committed tail, j = row j
    // of this pass): the verify_stage / draft_tree pass shape
    // (orchestrator.cpp:333-388, draft_engine.cpp:235-287) with its tree mask.
    // Returns the T rows' logits and final hidden states.
    void forward_tree(int which, const std::vector<int>& prompt, const std::vector<int>& tokens,
                      const std::vector<int>& parents, const std::string& plan_spec, float* logits,
                      float* hidden) override {
        ModelDev& M = which ? base_ : draft_;
        Cache& C = which ? bcache_ : dcache_;
        Workspace& W = which ? bws_ : dws_;
        CUDA_OK(cudaStreamSynchronize(stream_));
        const int np = (int)prompt.size(), T = (int)tokens.size();
        if (T < 1 || T > kMaxNodes) cfg_fail("forward_tree: 1..64 tree rows");
        if ((int)parents.size() != T) cfg_fail("forward_tree: one parent per row");
        if (np < 1 || np + T > M.c.max_positions) cfg_fail("forward_tree: prompt + rows exceed max_positions");
        for (int t : prompt)
            if (t < 0 || t >= M.c.vocab_size) cfg_fail("token outside vocabulary");
        for (int t : tokens)
            if (t < 0 || t >= M.c.vocab_size) cfg_fail("token outside vocabulary");
        LayerPlan plan;
        const LayerPlan* pp = nullptr;
        if (!plan_spec.empty()) {
            plan = plan_spec.rfind("lp=", 0) == 0 ? plan_groups(M.c.n_layers, std::stoi(plan_spec.substr(3)))
                                                  : parse_plan_override(plan_spec);
            if (plan.n_layers() != M.c.n_layers) cfg_fail("plan does not cover the model");
            if (which == 1 && plan.max_group_size() > 1) cfg_fail("fuzzy probes run on the drafter");
            pp = &plan;
        }
        C.reset();
        staging_.reset();
        it_.phase = 0;
        std::vector<int> all = prompt;
        all.insert(all.end(), tokens.begin(), tokens.end());
        CUDA_OK(cudaMemcpyAsync(arena_, staging_.push(all.data(), all.size(), stream_), sizeof(int) * all.size(),
                                cudaMemcpyDeviceToDevice, stream_));
        chain_pass(M, C, W, 0, np, nullptr, false, true, 0);
        std::vector<int> prow, tok;
        std::vector<int> rows;
        for (int j = 0; j < T; ++j) {
            if (parents[j] >= j || parents[j] < -1) cfg_fail("forward_tree: parents must precede their rows");
            tok.push_back(np + j);
        }
        // stage level by level in row order (a parent is staged before its child)
        for (int j = 0; j < T; ++j) prow.push_back(parents[j] < 0 ? kTail : C.committed + parents[j]);
        rows = C.stage_append(prow, pp != nullptr);
        Pass ps = make_pass(C, rows, tok);
        set_prefill_mode(false);
        forward(M, C, W, pp, ps);
        const int d = M.c.d_model, V = M.c.vocab_size;
        if (hidden) CUDA_OK(cudaMemcpyAsync(hidden, W.h, sizeof(float) * T * d, cudaMemcpyDeviceToHost, stream_));
        for (int r0 = 0; r0 < T; r0 += 8) {
            const int k = std::min(8, T - r0);
            head(M, W, r0, k, arena_ + out_off_, W.logits, ldpad(M.c.vocab_size, M.c.weight_dtype));
            if (logits)
                CUDA_OK(cudaMemcpy2DAsync(logits + (size_t)r0 * V, sizeof(float) * V, W.logits,
                                          sizeof(float) * ldpad(M.c.vocab_size, M.c.weight_dtype),
                                          sizeof(float) * V, k, cudaMemcpyDeviceToHost, stream_));
        }
        C.discard();
        CUDA_OK(cudaStreamSynchronize(stream_));
        CUDA_OK(cudaGetLastError());
        committed_.clear();
    }

    // forward_chain with every layer's LayerProbe captured (h_in, q, k, v,
    // attn_out; proj/src/draft_engine.cpp:291-330)
    void forward_capture(int which, const std::vector<int>& tokens, const std::string& plan_spec,
                         std::vector<LayerCapture>& out) override {
        if (tp()) cfg_fail("the similarity probe runs on one GPU");
        ModelDev& M = which ? base_ : draft_;
        out.assign(M.c.n_layers, LayerCapture{});
        cap_ = &out;
        try {
            forward_chain(which, tokens, plan_spec, nullptr, nullptr);
        } catch (...) {
            cap_ = nullptr;
            throw;
        }
        cap_ = nullptr;
        const int n = (int)tokens.size(), kvd = M.kvh() * M.c.d_head;
        for (int l = 0; l < M.c.n_layers; ++l) {
            out[l].k.resize((size_t)n * kvd);
            out[l].v.resize((size_t)n * kvd);
            cache_rows(which, l, 0, n, out[l].k.data(), out[l].v.data());
        }
    }

    int cache_rows(int which, int layer, int row0, int n, float* k, float* v) override {
        Cache& C = which ? bcache_ : dcache_;
        CUDA_OK(cudaStreamSynchronize(stream_));
        const int dh = C.dh, nkv = C.n_kv;
        const size_t es = dsize(C.dtype);
        std::vector<char> buf(dh * es);
        for (int r = 0; r < n; ++r) {
            const int row = row0 + r;
            const int page = C.table.at(row / C.page_rows), off = row % C.page_rows;
            for (int kind = 0; kind < 2; ++kind)
                for (int h = 0; h < nkv; ++h) {
                    const long long e = (long long)page * C.page_elems +
                                        ((((long long)layer * 2 + kind) * nkv + h) * C.page_rows + off) * dh;
                    CUDA_OK(cudaMemcpy(buf.data(), (char*)C.pool + e * es, dh * es, cudaMemcpyDeviceToHost));
                    float* o = (kind ? v : k) + (size_t)r * nkv * dh + (size_t)h * dh;
                    for (int i = 0; i < dh; ++i)
                        o[i] = C.dtype == DT_BF16 ? bf2f(((uint16_t*)buf.data())[i]) : ((float*)buf.data())[i];
                }
        }
        return C.committed;
    }

    int cache_committed(int which) const override { return which ? bcache_.committed : dcache_.committed; }
    const std::vector<int>& committed() const override { return committed_; }
    void sync() override { CUDA_OK(cudaStreamSynchronize(stream_)); }
    void* stream() override { return stream_; }
    long long device_bytes() const override {
        size_t f = 0, t = 0;
        cudaMemGetInfo(&f, &t);
        return (long long)(t - f);
    }
    int kernel_launches() const override { return launches_; }

    // ---------------- tensor-parallel wiring ----------------
    int tp_size() const override { return comm_.world; }
    void* comm_region() override { return comm_mem_; }
    void set_peer(int p, void* region) {
        comm_.peer_recv[p] = reinterpret_cast<float*>(region);
        comm_.peer_flags[p] = reinterpret_cast<uint64_t*>(comm_.peer_recv[p] + comm_.slot_floats * 2 * comm_.world);
    }
    void comm_link(const std::vector<Engine*>& group) override {
        if ((int)group.size() != comm_.world) cfg_fail("tensor-parallel group size does not match tp_size");
        for (int p = 0; p < comm_.world; ++p) {
            if (group[p]->tp_size() != comm_.world) cfg_fail("tensor-parallel group members disagree on tp_size");
            set_peer(p, group[p]->comm_region());
        }
        // shards share one GPU: no early PDL trigger, event-ordered phases
        comm_.early_trigger = 0;
        auto* lead = static_cast<EngineImpl*>(group[0]);
        if (!lead->local_group_) lead->local_group_ = std::make_shared<LocalGroup>(comm_.world);
        local_group_ = lead->local_group_;
        comm_.local_sync = &local_sync_fn;
        comm_.local_ctx = local_group_.get();
    }
    // shard proxy: this engine (rank 0 of a TP-N group) stands in for every
    // rank; collectives loop back into its own receive region
    void comm_loopback() override {
        if (comm_.world < 2) cfg_fail("the shard proxy needs tp_size > 1");
        for (int p = 0; p < comm_.world; ++p) set_peer(p, comm_region());
        comm_.loopback = 1;
    }
    void comm_ipc_export(void* handle64) override {
        if (!comm_mem_) cfg_fail("tp_size is 1: nothing to export");
        cudaIpcMemHandle_t h;
        CUDA_OK(cudaSetDevice(device_));
        CUDA_OK(cudaIpcGetMemHandle(&h, comm_mem_));
        std::memcpy(handle64, &h, sizeof(h));
    }
    void comm_ipc_import(const void* handles, int world) override {
        if (world != comm_.world) cfg_fail("tensor-parallel group size does not match tp_size");
        CUDA_OK(cudaSetDevice(device_));
        for (int p = 0; p < world; ++p) {
            if (p == comm_.rank) {
                set_peer(p, comm_mem_);
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, (const char*)handles + 64 * p, sizeof(h));
            void* ptr = nullptr;
            CUDA_OK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            ipc_opened_.push_back(ptr);
            set_peer(p, ptr);
        }
    }
    bool tp() const { return comm_.world > 1; }
    void check_comm() const {
        if (tp())
            for (int p = 0; p < comm_.world; ++p)
                if (!comm_.peer_recv[p]) throw Error(ST_NCCL, "tensor-parallel group not linked (comm_link / ipc import)");
    }
    void reset_launch_count() override { launches_ = 0; }

private:
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev_[4];
    ModelDev base_, draft_;
    bool base_allocated_ = false, draft_allocated_ = false;
    Cache bcache_, dcache_;
    Workspace bws_, dws_;
    std::vector<void*> ws_owned_;
    Staging staging_;
    int* arena_ = nullptr;
    int arena_cap_ = 0, tree_off_ = 0, am_off_ = 0, out_off_ = 0, cur_off_ = 0, err_off_ = 0;
    int* outcome_host_ = nullptr;
    // T > 0 sampling / tree levels
    static constexpr int kMaxDraws = 4 * kMaxNodes + 8;
    float* dlogits_ = nullptr;  // [kMaxNodes+1][logits_ld_] drafted-row logits (row = dist index)
    float* blogits_ = nullptr;  // [kMaxNodes+1][logits_ld_] verify-row logits
    float* ddists_ = nullptr;   // [kMaxNodes+1][V] draft distributions
    float* bdists_ = nullptr;   // [kMaxNodes+1][V] base distributions
    float* target_ = nullptr;   // [V] verify scratch
    int logits_ld_ = 0;
    double* unif_dev_ = nullptr;
    double* unif_host_ = nullptr;
    Xoshiro rng_{1};
    // tensor parallelism
    CommView comm_;
    SgPool pool_;  // decode-GEMV tail-pool counters of this engine's stream
    std::shared_ptr<LocalGroup> local_group_;
    void* comm_mem_ = nullptr;
    std::vector<void*> ipc_opened_;
    void* temp_ = nullptr;
    size_t temp_bytes_ = 0;
    RunCfg run_;
    std::vector<int> widths_;
    LayerPlan plan_;
    // simulated time (RunConfig::cost, Generation::clock_): reset per
    // generation; sim_*pre_ = rows prefill() ran ahead of the reference's
    // schedule (it stages the whole prompt in the first iteration's passes)
    CostParams cost_;
    SimClock clock_{8};
    int sim_dpre_ = 0, sim_bpre_ = 0;
    std::vector<int> committed_;
    int draft_cached_ = 0;
    int generated_ = 0;
    int launches_ = 0;
    static constexpr int kSiteEvents = 4096;
    cudaEvent_t site_ev_[2 * kSiteEvents];
    int site_which_ = -1, site_kind_ = -1, site_n_ = 0;
    double site_ms_ = 0, site_bytes_ = 0;
    long long h2d_bytes_ = 0, d2h_bytes_ = 0;
    int wide_draft_ = 1;  // ESPEC_WIDE_DRAFT=0: drafter on the (K, N)-only GEMV plan too
    int fuse_adds_ = 1;   // ESPEC_FUSE_ADDS=0: fuzzy-group residual adds as separate kernels
    int b16_acts_ = 1;    // ESPEC_B16_ACTS=0: attention / SiLU outputs in fp32
};

std::unique_ptr<Engine> make_engine(const ModelCfg& base, const ModelCfg& draft, const RunCfg& run, int device,
                                    int tp, int rank, bool draft_lp) {
    return std::unique_ptr<Engine>(new EngineImpl(base, draft, run, device, tp, rank, draft_lp));
}

}  // namespace espec
