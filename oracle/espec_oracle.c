/*
 * espec_oracle.c — plain-C restatement of the reference EasySpec decode path.
 *
 * TEST INFRASTRUCTURE ONLY (see espec_oracle.h). Parity is PINNED: the
 * outputs of this file are checked bit-for-bit against fixtures produced by
 * the unmodified reference core (oracle/_ref/ref_dump) in tests/test_oracle.py.
 *
 * Operation order follows the reference exactly (fp32 products and sums in
 * the same sequence, fp64 where the reference uses double), compiled without
 * FMA contraction (x86-64 baseline), so float results are identical.
 */
#include "espec_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KV_TAIL (-1) /* kCommittedTail, proj/include/espec/kv_cache.hpp:12 */
#define BOS_TOKEN 256
#define DEFAULT_VOCAB 258

/* ------------------------------------------------------------------------ */
/* error plumbing                                                            */

typedef struct {
    int status;
    char msg[256];
} eo_err;

static void fail(eo_err* e, int status, const char* fmt, ...) {
    if (e->status != EO_OK) return;
    e->status = status;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(e->msg, sizeof e->msg, fmt, ap);
    va_end(ap);
}

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz);
    if (!p) abort();
    return p;
}

/* ------------------------------------------------------------------------ */
/* RNG: SplitMix64 seeding + xoshiro256** (proj/include/espec/rng.hpp:9-68)  */

typedef struct {
    uint64_t s[4];
} rng_t;

static uint64_t splitmix_step(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static void rng_seed(rng_t* r, uint64_t seed) {
    uint64_t st = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix_step(&st);
}

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t rng_u64(rng_t* r) {
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

static double rng_uniform(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }

/* Box-Muller, cosine branch only (rng.hpp:55-61). */
static float rng_normal(rng_t* r) {
    const double u1 = rng_uniform(r);
    const double u2 = rng_uniform(r);
    const double rad = sqrt(-2.0 * log1p(-u1));
    return (float)(rad * cos(6.283185307179586 * u2));
}

void eo_rng_uniforms(uint64_t seed, int n, double* out) {
    rng_t r;
    rng_seed(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}

/* ------------------------------------------------------------------------ */
/* numerics (proj/src/matrix.cpp)                                            */

/* out[rows×n] = a[rows×k] · b[k×n], i-k-j order (matrix.cpp:38-57). */
static float* mm(const float* a, int rows, int k, const float* b, int n) {
    float* out = xcalloc((size_t)rows * n, sizeof(float));
    for (int i = 0; i < rows; ++i) {
        const float* ar = a + (size_t)i * k;
        float* orow = out + (size_t)i * n;
        for (int kk = 0; kk < k; ++kk) {
            const float aik = ar[kk];
            const float* br = b + (size_t)kk * n;
            for (int j = 0; j < n; ++j) orow[j] += aik * br[j];
        }
    }
    return out;
}

/* out[rows×m] = a[rows×k] · b[m×k]ᵀ (matrix.cpp:59-76). */
static float* mm_nt(const float* a, int rows, int k, const float* b, int m) {
    float* out = xcalloc((size_t)rows * m, sizeof(float));
    for (int i = 0; i < rows; ++i) {
        const float* ar = a + (size_t)i * k;
        for (int j = 0; j < m; ++j) {
            const float* br = b + (size_t)j * k;
            float acc = 0.0f;
            for (int kk = 0; kk < k; ++kk) acc += ar[kk] * br[kk];
            out[(size_t)i * m + j] = acc;
        }
    }
    return out;
}

/* matrix.cpp:118-137 */
static float* rmsnorm(const float* h, int rows, int cols, const float* gain, float eps) {
    float* out = xcalloc((size_t)rows * cols, sizeof(float));
    for (int i = 0; i < rows; ++i) {
        const float* r = h + (size_t)i * cols;
        float ms = 0.0f;
        for (int j = 0; j < cols; ++j) ms += r[j] * r[j];
        ms /= (float)cols;
        const float scale = 1.0f / sqrtf(ms + eps);
        for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = r[j] * scale * gain[j];
    }
    return out;
}

/* rotary in place, pairs (2p, 2p+1), angle in double (matrix.cpp:159-194) */
static void rope(float* x, int rows, int cols, const int* pos, int head_dim) {
    const int n_heads = cols / head_dim, n_pairs = head_dim / 2;
    double* inv = xcalloc((size_t)n_pairs, sizeof(double));
    for (int p = 0; p < n_pairs; ++p) inv[p] = pow(10000.0, -2.0 * p / head_dim);
    for (int r = 0; r < rows; ++r) {
        const double ps = pos[r];
        float* row = x + (size_t)r * cols;
        for (int h = 0; h < n_heads; ++h) {
            float* seg = row + (size_t)h * head_dim;
            for (int p = 0; p < n_pairs; ++p) {
                const double th = ps * inv[p];
                const float c = (float)cos(th), s = (float)sin(th);
                const float x0 = seg[2 * p], x1 = seg[2 * p + 1];
                seg[2 * p] = x0 * c - x1 * s;
                seg[2 * p + 1] = x0 * s + x1 * c;
            }
        }
    }
    free(inv);
}

/* first maximum (matrix.cpp:196-202) */
static int argmax_f(const float* v, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (v[i] > v[best]) best = i;
    return best;
}

/* softmax_temp (matrix.cpp:88-116); writes probs[n]. */
static void softmax_temp(const float* l, int n, float temp, float* probs, eo_err* e) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(l[i])) {
            fail(e, EO_DOMAIN, "softmax input contains a non-finite logit");
            return;
        }
    memset(probs, 0, sizeof(float) * (size_t)n);
    if (temp == 0.0f) {
        probs[argmax_f(l, n)] = 1.0f;
        return;
    }
    float mx = l[0];
    for (int i = 0; i < n; ++i) mx = (mx < l[i]) ? l[i] : mx;
    float sum = 0.0f;
    for (int i = 0; i < n; ++i) {
        const float ex = expf((l[i] - mx) / temp);
        probs[i] = ex;
        sum += ex;
    }
    for (int i = 0; i < n; ++i) probs[i] /= sum;
}

/* ------------------------------------------------------------------------ */
/* model (proj/src/model.cpp)                                                */

typedef struct {
    float *wq, *wk, *wv, *wo, *wg, *wu, *wd, *ga, *gm;
} layer_w;

struct eo_model {
    eo_config c;
    float* emb;
    float* fgain;
    layer_w* L;
    int owns;
};

static int cfg_check(const eo_config* c, eo_err* e) {
    /* ModelConfig::validate, model.cpp:12-24 */
    if (c->vocab_size < 2) fail(e, EO_CONFIG, "vocab_size must be >= 2");
    else if (c->n_layers < 2) fail(e, EO_CONFIG, "n_layers must be >= 2");
    else if (c->n_heads < 1 || c->d_head < 2 || c->d_head % 2 != 0)
        fail(e, EO_CONFIG, "need n_heads >= 1 and an even d_head >= 2");
    else if (c->d_model != c->n_heads * c->d_head)
        fail(e, EO_CONFIG, "d_model must equal n_heads * d_head");
    else if (c->d_mlp < 1) fail(e, EO_CONFIG, "d_mlp must be >= 1");
    else if (c->max_positions < 2) fail(e, EO_CONFIG, "max_positions must be >= 2");
    else if (!(c->norm_eps > 0.0f)) fail(e, EO_CONFIG, "norm_eps must be positive");
    return e->status;
}

static float* normal_tensor(rng_t* r, size_t n, float sd) {
    float* t = xcalloc(n, sizeof(float));
    for (size_t i = 0; i < n; ++i) t[i] = rng_normal(r) * sd;
    return t;
}

static float* ones(size_t n) {
    float* t = xcalloc(n, sizeof(float));
    for (size_t i = 0; i < n; ++i) t[i] = 1.0f;
    return t;
}

/* init_model, model.cpp:38-84: one stream, fixed tensor order. */
eo_model* eo_model_init(const eo_config* cfg, int* status) {
    eo_err e = {0};
    if (cfg_check(cfg, &e)) {
        if (status) *status = e.status;
        return NULL;
    }
    eo_model* m = xcalloc(1, sizeof *m);
    m->c = *cfg;
    m->owns = 1;
    const int d = cfg->d_model, f = cfg->d_mlp;
    rng_t r;
    rng_seed(&r, cfg->seed);
    const float proj_sd = 1.0f / sqrtf((float)d);
    const float resid = 1.0f / sqrtf(2.0f * (float)cfg->n_layers);
    const float down_sd = resid / sqrtf((float)f);
    const float emb_sd = 3.0f / sqrtf((float)d);
    m->emb = normal_tensor(&r, (size_t)cfg->vocab_size * d, emb_sd);
    m->fgain = ones((size_t)d);
    m->L = xcalloc((size_t)cfg->n_layers, sizeof(layer_w));
    for (int l = 0; l < cfg->n_layers; ++l) {
        layer_w* w = &m->L[l];
        w->wq = normal_tensor(&r, (size_t)d * d, proj_sd);
        w->wk = normal_tensor(&r, (size_t)d * d, proj_sd);
        w->wv = normal_tensor(&r, (size_t)d * d, proj_sd);
        w->wo = normal_tensor(&r, (size_t)d * d, proj_sd * resid);
        w->wg = normal_tensor(&r, (size_t)d * f, proj_sd);
        w->wu = normal_tensor(&r, (size_t)d * f, proj_sd);
        w->wd = normal_tensor(&r, (size_t)f * d, down_sd);
        w->ga = ones((size_t)d);
        w->gm = ones((size_t)d);
    }
    if (status) *status = EO_OK;
    return m;
}

/* make_truncated_draft, model.cpp:86-99 (shares the base tensors). */
eo_model* eo_model_truncated(const eo_model* base, int keep, int* status) {
    if (keep < 2 || keep >= base->c.n_layers) {
        if (status) *status = EO_CONFIG;
        return NULL;
    }
    eo_model* m = xcalloc(1, sizeof *m);
    m->c = base->c;
    m->c.n_layers = keep;
    m->emb = base->emb;
    m->fgain = base->fgain;
    m->L = xcalloc((size_t)keep, sizeof(layer_w));
    memcpy(m->L, base->L, sizeof(layer_w) * (size_t)keep);
    m->owns = 0;
    if (status) *status = EO_OK;
    return m;
}

void eo_model_free(eo_model* m) {
    if (!m) return;
    if (m->owns) {
        free(m->emb);
        free(m->fgain);
        for (int l = 0; l < m->c.n_layers; ++l) {
            layer_w* w = &m->L[l];
            free(w->wq); free(w->wk); free(w->wv); free(w->wo);
            free(w->wg); free(w->wu); free(w->wd); free(w->ga); free(w->gm);
        }
    }
    free(m->L);
    free(m);
}

const float* eo_model_tensor(const eo_model* m, const char* name, int layer, int* rows, int* cols) {
    const int d = m->c.d_model, f = m->c.d_mlp;
    if (!strcmp(name, "embedding")) { *rows = m->c.vocab_size; *cols = d; return m->emb; }
    if (!strcmp(name, "final_norm_gain")) { *rows = 1; *cols = d; return m->fgain; }
    if (layer < 0 || layer >= m->c.n_layers) return NULL;
    const layer_w* w = &m->L[layer];
    *rows = d; *cols = d;
    if (!strcmp(name, "wq")) return w->wq;
    if (!strcmp(name, "wk")) return w->wk;
    if (!strcmp(name, "wv")) return w->wv;
    if (!strcmp(name, "wo")) return w->wo;
    *cols = f;
    if (!strcmp(name, "w_gate")) return w->wg;
    if (!strcmp(name, "w_up")) return w->wu;
    *rows = f; *cols = d;
    if (!strcmp(name, "w_down")) return w->wd;
    *rows = 1; *cols = d;
    if (!strcmp(name, "attn_norm_gain")) return w->ga;
    if (!strcmp(name, "mlp_norm_gain")) return w->gm;
    return NULL;
}

/* ------------------------------------------------------------------------ */
/* KV cache (proj/src/kv_cache.cpp): committed prefix + staged forest        */

typedef struct {
    int parent, fuzzy, position;
} srow;

typedef struct {
    int n_layers, d;
    int committed, staged, cap;
    float** k;
    float** v;
    srow* st;
    int st_cap;
} cache_t;

static void cache_init(cache_t* c, int n_layers, int d) {
    memset(c, 0, sizeof *c);
    c->n_layers = n_layers;
    c->d = d;
    c->k = xcalloc((size_t)n_layers, sizeof(float*));
    c->v = xcalloc((size_t)n_layers, sizeof(float*));
}

static void cache_free(cache_t* c) {
    for (int l = 0; l < c->n_layers; ++l) {
        free(c->k[l]);
        free(c->v[l]);
    }
    free(c->k);
    free(c->v);
    free(c->st);
    memset(c, 0, sizeof *c);
}

static int cache_total(const cache_t* c) { return c->committed + c->staged; }

static void cache_reserve(cache_t* c, int rows) {
    if (rows > c->cap) {
        int nc = c->cap ? c->cap : 16;
        while (nc < rows) nc *= 2;
        for (int l = 0; l < c->n_layers; ++l) {
            c->k[l] = realloc(c->k[l], sizeof(float) * (size_t)nc * c->d);
            c->v[l] = realloc(c->v[l], sizeof(float) * (size_t)nc * c->d);
            if (!c->k[l] || !c->v[l]) abort();
        }
        c->cap = nc;
    }
}

/* stage_append, kv_cache.cpp:23-41. Writes new flat indices to rows_out. */
static void cache_stage(cache_t* c, const int* parents, int n, int fuzzy, int* rows_out, eo_err* e) {
    cache_reserve(c, cache_total(c) + n);
    if (c->staged + n > c->st_cap) {
        c->st_cap = (c->staged + n) * 2 + 8;
        c->st = realloc(c->st, sizeof(srow) * (size_t)c->st_cap);
    }
    for (int i = 0; i < n; ++i) {
        const int flat = cache_total(c), par = parents[i];
        if (par != KV_TAIL && (par < c->committed || par >= flat)) {
            fail(e, EO_STRUCTURE, "staged parent must be the committed tail or an earlier staged row");
            return;
        }
        const int pos = par == KV_TAIL ? c->committed : c->st[par - c->committed].position + 1;
        c->st[c->staged].parent = par;
        c->st[c->staged].fuzzy = fuzzy;
        c->st[c->staged].position = pos;
        c->staged++;
        for (int l = 0; l < c->n_layers; ++l) {
            memset(c->k[l] + (size_t)flat * c->d, 0, sizeof(float) * (size_t)c->d);
            memset(c->v[l] + (size_t)flat * c->d, 0, sizeof(float) * (size_t)c->d);
        }
        rows_out[i] = flat;
    }
}

static int cache_position(const cache_t* c, int flat) {
    return flat < c->committed ? flat : c->st[flat - c->committed].position;
}

/* build_tree_mask semantics (kv_cache.cpp:43-60) as a dense bitmap. */
static unsigned char* cache_mask(const cache_t* c) {
    const int n = cache_total(c);
    unsigned char* m = xcalloc((size_t)n * n, 1);
    for (int q = 0; q < c->committed; ++q)
        for (int k = 0; k <= q; ++k) m[(size_t)q * n + k] = 1;
    for (int q = c->committed; q < n; ++q) {
        for (int k = 0; k < c->committed; ++k) m[(size_t)q * n + k] = 1;
        for (int node = q; node != KV_TAIL; node = c->st[node - c->committed].parent)
            m[(size_t)q * n + node] = 1;
    }
    return m;
}

/* commit_path, kv_cache.cpp:62-94 */
static void cache_commit(cache_t* c, const int* path, int n, eo_err* e) {
    int expect = KV_TAIL;
    for (int i = 0; i < n; ++i) {
        const int flat = path[i];
        if (flat < 0 || flat >= cache_total(c)) { fail(e, EO_STRUCTURE, "kv row out of range"); return; }
        if (flat < c->committed) { fail(e, EO_STRUCTURE, "commit path entry is already committed"); return; }
        if (c->st[flat - c->committed].parent != expect) {
            fail(e, EO_STRUCTURE, "commit path is not a root-to-node chain");
            return;
        }
        expect = flat;
    }
    const int base = c->committed;
    for (int l = 0; l < c->n_layers; ++l)
        for (int i = 0; i < n; ++i) {
            const int src = path[i], dst = base + i;
            if (src != dst) {
                memcpy(c->k[l] + (size_t)dst * c->d, c->k[l] + (size_t)src * c->d, sizeof(float) * (size_t)c->d);
                memcpy(c->v[l] + (size_t)dst * c->d, c->v[l] + (size_t)src * c->d, sizeof(float) * (size_t)c->d);
            }
        }
    c->committed = base + n;
    c->staged = 0;
}

static void cache_discard(cache_t* c) { c->staged = 0; } /* kv_cache.cpp:96-102 */

/* ------------------------------------------------------------------------ */
/* forward passes                                                             */

typedef struct {
    const int* rows;
    const int* pos;
    int n;
    const unsigned char* mask; /* total×total */
    int total;
    int calibrate;
} batch_t;

/* attention_forward, model.cpp:114-195. Returns n×d (pre-residual). */
static float* attention(const eo_model* m, int layer, const float* hn, cache_t* c, const batch_t* b,
                        eo_err* e) {
    const eo_config* cf = &m->c;
    const layer_w* w = &m->L[layer];
    const int d = cf->d_model, n = b->n, dh = cf->d_head;
    for (int i = 0; i < n; ++i)
        if (b->pos[i] >= cf->max_positions) {
            fail(e, EO_CONFIG, "position %d exceeds max_positions %d", b->pos[i], cf->max_positions);
            return NULL;
        }
    float* q = mm(hn, n, d, w->wq, d);
    rope(q, n, d, b->pos, dh);
    float* k = mm(hn, n, d, w->wk, d);
    rope(k, n, d, b->pos, dh);
    float* v = mm(hn, n, d, w->wv, d);
    for (int i = 0; i < n; ++i) {
        memcpy(c->k[layer] + (size_t)b->rows[i] * d, k + (size_t)i * d, sizeof(float) * (size_t)d);
        memcpy(c->v[layer] + (size_t)b->rows[i] * d, v + (size_t)i * d, sizeof(float) * (size_t)d);
        if (b->calibrate && b->rows[i] >= c->committed) c->st[b->rows[i] - c->committed].fuzzy = 0;
    }
    const int total = b->total;
    const float inv_sqrt = 1.0f / sqrtf((float)dh);
    float* mixed = xcalloc((size_t)n * d, sizeof(float));
    float* sc = xcalloc((size_t)total, sizeof(float));
    for (int i = 0; i < n; ++i) {
        const int qr = b->rows[i];
        for (int h = 0; h < cf->n_heads; ++h) {
            const int off = h * dh;
            const float* qv = q + (size_t)i * d + off;
            float mx = -INFINITY;
            for (int j = 0; j < total; ++j) {
                if (!b->mask[(size_t)qr * total + j]) {
                    sc[j] = -INFINITY;
                    continue;
                }
                const float* kv = c->k[layer] + (size_t)j * d + off;
                float dot = 0.0f;
                for (int t = 0; t < dh; ++t) dot += qv[t] * kv[t];
                const float s = dot * inv_sqrt;
                sc[j] = s;
                mx = (mx < s) ? s : mx;
            }
            float den = 0.0f;
            for (int j = 0; j < total; ++j) {
                if (isinf(sc[j]) && sc[j] < 0.0f) {
                    sc[j] = 0.0f;
                } else {
                    sc[j] = expf(sc[j] - mx);
                    den += sc[j];
                }
            }
            float* o = mixed + (size_t)i * d + off;
            for (int j = 0; j < total; ++j) {
                const float wgt = sc[j];
                if (wgt == 0.0f) continue;
                const float* vv = c->v[layer] + (size_t)j * d + off;
                const float wn = wgt / den;
                for (int t = 0; t < dh; ++t) o[t] += wn * vv[t];
            }
        }
    }
    float* out = mm(mixed, n, d, w->wo, d);
    free(q); free(k); free(v); free(mixed); free(sc);
    return out;
}

/* mlp_forward, model.cpp:197-210 */
static float* mlp(const eo_model* m, int layer, const float* hn, int n) {
    const layer_w* w = &m->L[layer];
    const int d = m->c.d_model, f = m->c.d_mlp;
    float* g = mm(hn, n, d, w->wg, f);
    float* u = mm(hn, n, d, w->wu, f);
    for (size_t i = 0; i < (size_t)n * f; ++i) {
        const float x = g[i];
        const float s = x / (1.0f + expf(-x));
        g[i] = s * u[i];
    }
    float* out = mm(g, n, f, w->wd, d);
    free(g); free(u);
    return out;
}

static void add_into(float* a, const float* b, size_t n) {
    for (size_t i = 0; i < n; ++i) a[i] += b[i];
}

static float* embed(const eo_model* m, const int* toks, int n, eo_err* e) {
    const int d = m->c.d_model;
    float* h = xcalloc((size_t)n * d, sizeof(float));
    for (int i = 0; i < n; ++i) {
        if (toks[i] < 0 || toks[i] >= m->c.vocab_size) {
            fail(e, EO_CONFIG, "token %d outside vocabulary", toks[i]);
            return h;
        }
        memcpy(h + (size_t)i * d, m->emb + (size_t)toks[i] * d, sizeof(float) * (size_t)d);
    }
    return h;
}

/* one residual/MLP step: h += attn; h += mlp(norm(h)) (draft_engine.cpp:50-54, 112-121) */
static void residual_mlp(const eo_model* m, int layer, float* h, const float* attn, int n) {
    const int d = m->c.d_model;
    add_into(h, attn, (size_t)n * d);
    float* hn = rmsnorm(h, n, d, m->L[layer].gm, m->c.norm_eps);
    float* mo = mlp(m, layer, hn, n);
    add_into(h, mo, (size_t)n * d);
    free(hn);
    free(mo);
}

/* plan: groups as a flat layer list + group starts */
typedef struct {
    int n_groups;
    int start[512];
    int size[512];
    int lp;
} plan_t;

/* forward_sequential (draft_engine.cpp:35-62) when plan == NULL, else
 * forward_fuzzy (draft_engine.cpp:64-133). h is updated in place. */
static void forward(const eo_model* m, const plan_t* plan, float* h, cache_t* c, const batch_t* b,
                    eo_err* e) {
    const int d = m->c.d_model, n = b->n;
    if (!plan) {
        for (int l = 0; l < m->c.n_layers && !e->status; ++l) {
            float* hn = rmsnorm(h, n, d, m->L[l].ga, m->c.norm_eps);
            float* a = attention(m, l, hn, c, b, e);
            free(hn);
            if (!a) return;
            residual_mlp(m, l, h, a, n);
            free(a);
        }
        return;
    }
    for (int g = 0; g < plan->n_groups && !e->status; ++g) {
        const int s0 = plan->start[g], gs = plan->size[g];
        float** outs = xcalloc((size_t)gs, sizeof(float*));
        /* every attention layer of the group reads the entry state */
        for (int i = 0; i < gs; ++i) {
            float* hn = rmsnorm(h, n, d, m->L[s0 + i].ga, m->c.norm_eps);
            outs[i] = attention(m, s0 + i, hn, c, b, e);
            free(hn);
        }
        for (int i = 0; i < gs; ++i) {
            if (outs[i] && !e->status) residual_mlp(m, s0 + i, h, outs[i], n);
            free(outs[i]);
        }
        free(outs);
    }
}

/* lm_logits, model.cpp:212-215 */
static float* lm_logits(const eo_model* m, const float* h, int n) {
    float* hn = rmsnorm(h, n, m->c.d_model, m->fgain, m->c.norm_eps);
    float* lg = mm_nt(hn, n, m->c.d_model, m->emb, m->c.vocab_size);
    free(hn);
    return lg;
}

/* ------------------------------------------------------------------------ */
/* layer plans (proj/src/layer_plan.cpp)                                     */

static int plan_validate(const plan_t* p, eo_err* e) {
    /* validate_plan, layer_plan.cpp:32-52 (groups are contiguous by construction) */
    if (p->n_groups == 0) return fail(e, EO_CONFIG, "layer plan has no groups"), e->status;
    int expect = 0, mx = 0;
    for (int g = 0; g < p->n_groups; ++g) {
        if (p->size[g] < 1) return fail(e, EO_CONFIG, "layer plan contains an empty group"), e->status;
        if (p->start[g] != expect)
            return fail(e, EO_CONFIG, "layer plan must cover layers contiguously in ascending order"), e->status;
        expect += p->size[g];
        if (p->size[g] > mx) mx = p->size[g];
    }
    if (p->size[0] != 1 || p->size[p->n_groups - 1] != 1)
        return fail(e, EO_CONFIG, "first and last layer must be singleton groups"), e->status;
    if (mx > p->lp && p->lp > 0)
        return fail(e, EO_CONFIG, "layer plan group exceeds the layer-parallel size"), e->status;
    return EO_OK;
}

static int plan_total(const plan_t* p) {
    int t = 0;
    for (int g = 0; g < p->n_groups; ++g) t += p->size[g];
    return t;
}

/* plan_groups, layer_plan.cpp:54-82 */
static int plan_make(int n_layers, int lp, plan_t* p, eo_err* e) {
    memset(p, 0, sizeof *p);
    if (n_layers < 2) return fail(e, EO_CONFIG, "layer plan needs at least 2 layers"), e->status;
    if (lp < 1) return fail(e, EO_CONFIG, "layer-parallel size must be >= 1"), e->status;
    p->lp = lp;
    p->start[0] = 0;
    p->size[0] = 1;
    p->n_groups = 1;
    const int last = n_layers - 1;
    int next = 1;
    while (next < last) {
        int end = (next == 1) ? (lp > 2 ? lp : 2) : next + lp;
        if (end > last) end = last;
        p->start[p->n_groups] = next;
        p->size[p->n_groups] = end - next;
        p->n_groups++;
        next = end;
    }
    p->start[p->n_groups] = last;
    p->size[p->n_groups] = 1;
    p->n_groups++;
    return plan_validate(p, e);
}

/* parse_plan_override, layer_plan.cpp:84-114 */
static int plan_parse(const char* spec, plan_t* p, eo_err* e) {
    memset(p, 0, sizeof *p);
    const char* s = spec;
    while (1) {
        const char* bar = strchr(s, '|');
        const size_t len = bar ? (size_t)(bar - s) : strlen(s);
        if (len == 0) return fail(e, EO_CONFIG, "empty group in plan override '%s'", spec), e->status;
        char tok[64];
        if (len >= sizeof tok) return fail(e, EO_CONFIG, "unparsable group in plan override"), e->status;
        memcpy(tok, s, len);
        tok[len] = 0;
        char* dash = strchr(tok, '-');
        char* endp;
        long lo, hi;
        if (!dash) {
            lo = hi = strtol(tok, &endp, 10);
            if (endp == tok) return fail(e, EO_CONFIG, "unparsable group '%s' in plan override", tok), e->status;
        } else {
            *dash = 0;
            lo = strtol(tok, &endp, 10);
            if (endp == tok) return fail(e, EO_CONFIG, "unparsable group in plan override"), e->status;
            char* h = dash + 1;
            hi = strtol(h, &endp, 10);
            if (endp == h) return fail(e, EO_CONFIG, "unparsable group in plan override"), e->status;
        }
        if (lo < 0 || hi < lo) return fail(e, EO_CONFIG, "invalid layer range in plan override"), e->status;
        if (p->n_groups >= 512) return fail(e, EO_CONFIG, "too many groups"), e->status;
        p->start[p->n_groups] = (int)lo;
        p->size[p->n_groups] = (int)(hi - lo + 1);
        p->n_groups++;
        if (!bar) break;
        s = bar + 1;
    }
    int mx = 0;
    for (int g = 0; g < p->n_groups; ++g) mx = p->size[g] > mx ? p->size[g] : mx;
    p->lp = mx;
    return plan_validate(p, e);
}

static void plan_format(const plan_t* p, char* out, int out_len) {
    int pos = 0;
    out[0] = 0;
    for (int g = 0; g < p->n_groups && pos < out_len; ++g) {
        if (p->size[g] > 1)
            pos += snprintf(out + pos, (size_t)(out_len - pos), "%s%d-%d", g ? "|" : "", p->start[g],
                            p->start[g] + p->size[g] - 1);
        else
            pos += snprintf(out + pos, (size_t)(out_len - pos), "%s%d", g ? "|" : "", p->start[g]);
    }
}

int eo_plan_groups(int n_layers, int lp, char* out, int out_len) {
    eo_err e = {0};
    plan_t p;
    if (plan_make(n_layers, lp, &p, &e)) return e.status;
    plan_format(&p, out, out_len);
    return EO_OK;
}

int eo_parse_plan(const char* spec, char* out, int out_len) {
    eo_err e = {0};
    plan_t p;
    if (plan_parse(spec, &p, &e)) return e.status;
    plan_format(&p, out, out_len);
    return EO_OK;
}

/* ------------------------------------------------------------------------ */
/* chain prefill on a fresh cache                                             */

static void chain_parents(const cache_t* c, int n, int* parents) {
    for (int i = 0; i < n; ++i) parents[i] = i == 0 ? KV_TAIL : c->committed + i - 1;
}

int eo_prefill(const eo_model* m, const char* plan_spec, const int* tokens, int n, float* hidden,
               float* logits, float* kout, float* vout) {
    eo_err e = {0};
    plan_t plan;
    const plan_t* pp = NULL;
    if (plan_spec && plan_spec[0]) {
        if (!strncmp(plan_spec, "lp=", 3)) plan_make(m->c.n_layers, atoi(plan_spec + 3), &plan, &e);
        else plan_parse(plan_spec, &plan, &e);
        if (e.status) return e.status;
        pp = &plan;
    }
    cache_t c;
    cache_init(&c, m->c.n_layers, m->c.d_model);
    int* parents = xcalloc((size_t)n, sizeof(int));
    int* rows = xcalloc((size_t)n, sizeof(int));
    int* pos = xcalloc((size_t)n, sizeof(int));
    chain_parents(&c, n, parents);
    cache_stage(&c, parents, n, pp != NULL, rows, &e);
    for (int i = 0; i < n; ++i) pos[i] = cache_position(&c, rows[i]);
    unsigned char* mask = cache_mask(&c);
    batch_t b = {rows, pos, n, mask, cache_total(&c), 0};
    float* h = embed(m, tokens, n, &e);
    if (!e.status) forward(m, pp, h, &c, &b, &e);
    if (!e.status) {
        const int d = m->c.d_model;
        if (hidden) memcpy(hidden, h, sizeof(float) * (size_t)n * d);
        if (logits) {
            float* lg = lm_logits(m, h, n);
            memcpy(logits, lg, sizeof(float) * (size_t)n * m->c.vocab_size);
            free(lg);
        }
        for (int l = 0; l < m->c.n_layers; ++l) {
            if (kout) memcpy(kout + (size_t)l * n * d, c.k[l], sizeof(float) * (size_t)n * d);
            if (vout) memcpy(vout + (size_t)l * n * d, c.v[l], sizeof(float) * (size_t)n * d);
        }
    }
    free(h); free(mask); free(parents); free(rows); free(pos);
    cache_free(&c);
    return e.status;
}

/* ------------------------------------------------------------------------ */
/* drafting (proj/src/draft_engine.cpp:141-289)                              */

/* select_children, draft_engine.cpp:141-186 */
static int select_children(const float* lg, int V, int k, float temp, rng_t* r, int* out, eo_err* e) {
    if (k < 1 || k > V) return fail(e, EO_CONFIG, "tree width must be in [1, vocab]"), 0;
    if (temp == 0.0f) {
        /* top-k by (logit desc, id asc) */
        unsigned char* taken = xcalloc((size_t)V, 1);
        for (int r0 = 0; r0 < k; ++r0) {
            int best = -1;
            for (int t = 0; t < V; ++t) {
                if (taken[t]) continue;
                if (best < 0 || lg[t] > lg[best]) best = t;
            }
            taken[best] = 1;
            out[r0] = best;
        }
        free(taken);
        return k;
    }
    float* p = xcalloc((size_t)V, sizeof(float));
    softmax_temp(lg, V, temp, p, e);
    double* w = xcalloc((size_t)V, sizeof(double));
    double mass = 0.0;
    for (int t = 0; t < V; ++t) w[t] = p[t];
    for (int t = 0; t < V; ++t) mass += w[t];
    int cnt = 0;
    for (int round = 0; round < k && mass > 1e-12; ++round) {
        const double u = rng_uniform(r) * mass;
        double cum = 0.0;
        int chosen = -1;
        for (int t = 0; t < V; ++t) {
            if (w[t] <= 0.0) continue;
            cum += w[t];
            chosen = t;
            if (u < cum) break;
        }
        if (chosen < 0) break;
        out[cnt++] = chosen;
        mass -= w[chosen];
        w[chosen] = 0.0;
    }
    free(p);
    free(w);
    return cnt;
}

int eo_select_children(const float* logits, int vocab, int k, float temperature, uint64_t seed, int* out) {
    eo_err e = {0};
    rng_t r;
    rng_seed(&r, seed);
    const int n = select_children(logits, vocab, k, temperature, &r, out, &e);
    return e.status ? -e.status : n;
}

typedef struct {
    int token, parent, depth, prob_index, cache_row, first_child, n_children;
} node_t;

typedef struct {
    node_t* nodes;
    int n_nodes, cap;
    float* dists; /* n_dists × V */
    int n_dists, dcap;
    int root_children;
    int n_levels;
    const int* widths;
} tree_t;

static void tree_free(tree_t* t) {
    free(t->nodes);
    free(t->dists);
    memset(t, 0, sizeof *t);
}

static int tree_add_node(tree_t* t, node_t nd) {
    if (t->n_nodes == t->cap) {
        t->cap = t->cap ? t->cap * 2 : 16;
        t->nodes = realloc(t->nodes, sizeof(node_t) * (size_t)t->cap);
    }
    t->nodes[t->n_nodes] = nd;
    return t->n_nodes++;
}

static float* tree_add_dist(tree_t* t, int V) {
    if (t->n_dists == t->dcap) {
        t->dcap = t->dcap ? t->dcap * 2 : 8;
        t->dists = realloc(t->dists, sizeof(float) * (size_t)t->dcap * V);
    }
    return t->dists + (size_t)(t->n_dists++) * V;
}

typedef struct {
    long seq, fuzzy, base;
} counters_t;

/* draft_tree, draft_engine.cpp:188-289 */
static void draft_tree(const eo_model* dm, const plan_t* plan, cache_t* c, const float* root_logits,
                       const int* widths, int n_levels, float temp, rng_t* r, counters_t* cnt,
                       int fuzzy_passes, tree_t* t, eo_err* e) {
    const int V = dm->c.vocab_size;
    memset(t, 0, sizeof *t);
    t->widths = widths;
    t->n_levels = n_levels;
    for (int i = 0; i < n_levels; ++i)
        if (widths[i] < 1 || widths[i] > V) { fail(e, EO_CONFIG, "tree width out of range"); return; }
    softmax_temp(root_logits, V, temp, tree_add_dist(t, V), e);
    int* picks = xcalloc((size_t)V, sizeof(int));
    int* frontier = xcalloc(1, sizeof(int));
    int nf = select_children(root_logits, V, widths[0], temp, r, picks, e);
    frontier = realloc(frontier, sizeof(int) * (size_t)(nf ? nf : 1));
    for (int i = 0; i < nf; ++i) {
        node_t nd = {picks[i], -1, 1, 0, -1, -1, 0};
        frontier[i] = tree_add_node(t, nd);
    }
    t->root_children = nf;
    for (int level = 1; level <= n_levels - 1 && !e->status; ++level) {
        if (nf == 0) break;
        int* parents = xcalloc((size_t)nf, sizeof(int));
        int* rows = xcalloc((size_t)nf, sizeof(int));
        int* pos = xcalloc((size_t)nf, sizeof(int));
        int* toks = xcalloc((size_t)nf, sizeof(int));
        for (int i = 0; i < nf; ++i) {
            const node_t* nd = &t->nodes[frontier[i]];
            parents[i] = nd->parent < 0 ? KV_TAIL : t->nodes[nd->parent].cache_row;
        }
        cache_stage(c, parents, nf, fuzzy_passes, rows, e);
        for (int i = 0; i < nf; ++i) {
            t->nodes[frontier[i]].cache_row = rows[i];
            toks[i] = t->nodes[frontier[i]].token;
            pos[i] = cache_position(c, rows[i]);
        }
        unsigned char* mask = cache_mask(c);
        batch_t b = {rows, pos, nf, mask, cache_total(c), 0};
        float* h = embed(dm, toks, nf, e);
        if (!e->status) {
            forward(dm, fuzzy_passes ? plan : NULL, h, c, &b, e);
            if (fuzzy_passes) cnt->fuzzy++;
            else cnt->seq++;
        }
        int* next = NULL;
        int nn = 0;
        if (!e->status) {
            float* lg = lm_logits(dm, h, nf);
            for (int i = 0; i < nf && !e->status; ++i) {
                const int parent_index = frontier[i];
                const float* row = lg + (size_t)i * V;
                softmax_temp(row, V, temp, tree_add_dist(t, V), e);
                const int prob_index = t->n_dists - 1;
                const int kids = select_children(row, V, widths[level], temp, r, picks, e);
                t->nodes[parent_index].first_child = t->n_nodes;
                t->nodes[parent_index].n_children = kids;
                next = realloc(next, sizeof(int) * (size_t)(nn + kids + 1));
                for (int j = 0; j < kids; ++j) {
                    node_t nd = {picks[j], parent_index, level + 1, prob_index, -1, -1, 0};
                    next[nn++] = tree_add_node(t, nd);
                }
            }
            free(lg);
        }
        free(h); free(mask); free(parents); free(rows); free(pos); free(toks);
        free(frontier);
        frontier = next ? next : xcalloc(1, sizeof(int));
        nf = nn;
    }
    free(frontier);
    free(picks);
}

/* ------------------------------------------------------------------------ */
/* verification (proj/src/verifier.cpp)                                      */

#define RESIDUAL_FLOOR 1e-9

/* residual_distribution, verifier.cpp:25-43 (in place into out) */
static void residual(const float* p, const float* pp, int V, float* out) {
    float* tmp = xcalloc((size_t)V, sizeof(float));
    double mass = 0.0;
    for (int t = 0; t < V; ++t) {
        const double diff = (double)p[t] - pp[t];
        if (diff > 0.0) {
            tmp[t] = (float)diff;
            mass += diff;
        }
    }
    if (mass < RESIDUAL_FLOOR) {
        memmove(out, p, sizeof(float) * (size_t)V);
    } else {
        for (int t = 0; t < V; ++t) out[t] = (float)(tmp[t] / mass);
    }
    free(tmp);
}

/* sample_from, verifier.cpp:70-84 */
static int sample_from(const float* dist, int V, rng_t* r, eo_err* e) {
    const double u = rng_uniform(r);
    double cum = 0.0;
    int last = -1;
    for (int t = 0; t < V; ++t) {
        if (dist[t] <= 0.0f) continue;
        cum += dist[t];
        last = t;
        if (u < cum) return t;
    }
    if (last < 0) fail(e, EO_CHECK, "sampling from an all-zero distribution");
    return last < 0 ? 0 : last;
}

/* verify_tree, verifier.cpp:86-177. base_dists: (n_nodes+1)×V. */
static void verify(const tree_t* t, const float* base_dists, int V, float temp, rng_t* r, int* m_out,
                   int* path, int* bonus, eo_err* e) {
    if (t->n_nodes == 0) { fail(e, EO_STRUCTURE, "verifying an empty draft tree"); return; }
    const int greedy = temp == 0.0f;
    float* target = xcalloc((size_t)V, sizeof(float));
    float* clamped = xcalloc((size_t)V, sizeof(float));
    double* ld = xcalloc((size_t)V, sizeof(double));
    memcpy(target, base_dists, sizeof(float) * (size_t)V);
    int parent = -1, m = 0;
    for (int depth = 1; depth <= t->n_levels && !e->status; ++depth) {
        const int first = parent < 0 ? 0 : t->nodes[parent].first_child;
        const int count = parent < 0 ? t->root_children : t->nodes[parent].n_children;
        if (count == 0) break;
        const float* dist = t->dists + (size_t)t->nodes[first].prob_index * V;
        double dm = 0.0;
        for (int x = 0; x < V; ++x) ld[x] = dist[x];
        for (int x = 0; x < V; ++x) dm += ld[x];
        int acc = -1;
        for (int i = 0; i < count; ++i) {
            const int ni = first + i;
            const int tok = t->nodes[ni].token;
            int accept;
            if (greedy) {
                accept = tok == argmax_f(target, V);
            } else {
                const double p_tok = target[tok];
                const double pp_tok = ld[tok] / dm;
                const double u = rng_uniform(r);
                if (!(pp_tok > 0.0)) { fail(e, EO_CHECK, "drafted token carries zero draft probability"); break; }
                const double ratio = p_tok / pp_tok;
                accept = u < (ratio < 1.0 ? ratio : 1.0);
            }
            if (accept) { acc = ni; break; }
            for (int x = 0; x < V; ++x) clamped[x] = (float)(ld[x] / dm);
            residual(target, clamped, V, target);
            dm -= ld[tok];
            ld[tok] = 0.0;
            if (dm <= RESIDUAL_FLOOR && i + 1 < count) {
                fail(e, EO_CHECK, "sibling candidates exhaust the draft distribution");
                break;
            }
        }
        if (acc < 0 || e->status) break;
        path[m++] = acc;
        memcpy(target, base_dists + (size_t)(acc + 1) * V, sizeof(float) * (size_t)V);
        parent = acc;
    }
    if (!e->status) *bonus = greedy ? argmax_f(target, V) : sample_from(target, V, r, e);
    *m_out = m;
    free(target); free(clamped); free(ld);
}

int eo_verify_tree(int V, int n_nodes, const int* tokens, const int* parents, const int* prob_index,
                   int n_dists, const float* dists, const float* base_dists, int n_levels,
                   const int* widths, float temperature, uint64_t seed, int* m, int* accepted, int* bonus) {
    eo_err e = {0};
    tree_t t;
    memset(&t, 0, sizeof t);
    t.widths = widths;
    t.n_levels = n_levels;
    for (int i = 0; i < n_dists; ++i) memcpy(tree_add_dist(&t, V), dists + (size_t)i * V, sizeof(float) * (size_t)V);
    for (int i = 0; i < n_nodes; ++i) {
        node_t nd = {tokens[i], parents[i], 0, prob_index[i], -1, -1, 0};
        tree_add_node(&t, nd);
    }
    /* siblings are contiguous and stored level by level */
    for (int i = 0; i < n_nodes; ++i) {
        const int p = parents[i];
        if (p < 0) t.root_children++;
        else {
            if (t.nodes[p].n_children == 0) t.nodes[p].first_child = i;
            t.nodes[p].n_children++;
        }
    }
    int* path = xcalloc((size_t)(n_levels + 1), sizeof(int));
    int mm_ = 0, b = 0;
    rng_t r;
    rng_seed(&r, seed);
    verify(&t, base_dists, V, temperature, &r, &mm_, path, &b, &e);
    *m = mm_;
    for (int i = 0; i < mm_; ++i) accepted[i] = t.nodes[path[i]].token;
    *bonus = b;
    free(path);
    tree_free(&t);
    return e.status;
}

/* ------------------------------------------------------------------------ */
/* generation loop (proj/src/orchestrator.cpp:138-484)                      */

typedef struct {
    int m, n, drafted, emitted, seq, fuzzy, base, committed, dcommitted, bcommitted;
    double* dsums;
    double* bsums;
} iter_rec;

struct eo_result {
    int status;
    char msg[256];
    int* tokens;
    int n_tokens;
    iter_rec* it;
    int n_it, it_cap;
    int nl_draft, nl_base, d_draft, d_base;
    cache_t dcache, bcache;
};

static double* kv_sums(const cache_t* c) {
    double* s = xcalloc((size_t)c->n_layers * 4, sizeof(double));
    for (int l = 0; l < c->n_layers; ++l) {
        double ks = 0, ka = 0, vs = 0, va = 0;
        for (size_t i = 0; i < (size_t)c->committed * c->d; ++i) {
            const float kv = c->k[l][i], vv = c->v[l][i];
            ks += kv; ka += fabs(kv); vs += vv; va += fabs(vv);
        }
        s[4 * l] = ks; s[4 * l + 1] = ka; s[4 * l + 2] = vs; s[4 * l + 3] = va;
    }
    return s;
}

typedef struct {
    const eo_model *base, *draft;
    eo_run run;
    int* widths;
    plan_t plan;
    cache_t* bc;
    cache_t* dc;
    rng_t rng;
    counters_t cnt;
    int* committed;
    int n_committed, committed_cap;
    int draft_cached;
    eo_err e;
} gen_t;

static void push_committed(gen_t* g, int tok) {
    if (g->n_committed == g->committed_cap) {
        g->committed_cap = g->committed_cap ? g->committed_cap * 2 : 64;
        g->committed = realloc(g->committed, sizeof(int) * (size_t)g->committed_cap);
    }
    g->committed[g->n_committed++] = tok;
}

/* stage_suffix, orchestrator.cpp:228-240. Returns count; rows/toks alloc'd. */
static int stage_suffix(gen_t* g, cache_t* c, int cached, int fuzzy, int** rows, int** toks) {
    const int n = g->n_committed - cached;
    int* parents = xcalloc((size_t)(n > 0 ? n : 1), sizeof(int));
    *rows = xcalloc((size_t)(n > 0 ? n : 1), sizeof(int));
    *toks = xcalloc((size_t)(n > 0 ? n : 1), sizeof(int));
    for (int i = 0; i < n; ++i) {
        parents[i] = i == 0 ? KV_TAIL : c->committed + i - 1;
        (*toks)[i] = g->committed[cached + i];
    }
    cache_stage(c, parents, n, fuzzy, *rows, &g->e);
    free(parents);
    return n;
}

/* drafter_leading_pass, orchestrator.cpp:256-300. Returns root logits (V). */
static float* leading_pass(gen_t* g) {
    const int easy = g->run.algorithm == EO_EASYSPEC;
    const int calibrated = easy && g->run.calibration;
    const int fuzzy = easy && !g->run.calibration;
    int *rows, *toks;
    const int n = stage_suffix(g, g->dc, g->draft_cached, fuzzy, &rows, &toks);
    int* pos = xcalloc((size_t)(n > 0 ? n : 1), sizeof(int));
    for (int i = 0; i < n; ++i) pos[i] = cache_position(g->dc, rows[i]);
    unsigned char* mask = cache_mask(g->dc);
    batch_t b = {rows, pos, n, mask, cache_total(g->dc), calibrated};
    float* h = embed(g->draft, toks, n, &g->e);
    float* root = NULL;
    if (!g->e.status) {
        forward(g->draft, fuzzy ? &g->plan : NULL, h, g->dc, &b, &g->e);
        if (fuzzy) g->cnt.fuzzy++;
        else g->cnt.seq++;
        cache_commit(g->dc, rows, n, &g->e);
        g->draft_cached = g->n_committed;
        root = lm_logits(g->draft, h + (size_t)(n - 1) * g->draft->c.d_model, 1);
    }
    free(h); free(mask); free(rows); free(toks); free(pos);
    return root;
}

/* verify_stage, orchestrator.cpp:333-388 */
static void verify_stage(gen_t* g, const tree_t* t, int* m_out, int* path, int* bonus) {
    const int V = g->base->c.vocab_size;
    int *crow, *ctok;
    const int nc = stage_suffix(g, g->bc, g->bc->committed, 0, &crow, &ctok);
    const int first_node_row = crow[nc - 1] + 1;
    int* tp = xcalloc((size_t)t->n_nodes, sizeof(int));
    int* nrows = xcalloc((size_t)t->n_nodes, sizeof(int));
    for (int j = 0; j < t->n_nodes; ++j)
        tp[j] = t->nodes[j].parent < 0 ? crow[nc - 1] : first_node_row + t->nodes[j].parent;
    cache_stage(g->bc, tp, t->n_nodes, 0, nrows, &g->e);
    const int T = nc + t->n_nodes;
    int* rows = xcalloc((size_t)T, sizeof(int));
    int* toks = xcalloc((size_t)T, sizeof(int));
    int* pos = xcalloc((size_t)T, sizeof(int));
    for (int i = 0; i < nc; ++i) { rows[i] = crow[i]; toks[i] = ctok[i]; }
    for (int j = 0; j < t->n_nodes; ++j) { rows[nc + j] = nrows[j]; toks[nc + j] = t->nodes[j].token; }
    for (int i = 0; i < T; ++i) pos[i] = cache_position(g->bc, rows[i]);
    unsigned char* mask = cache_mask(g->bc);
    batch_t b = {rows, pos, T, mask, cache_total(g->bc), 0};
    float* h = embed(g->base, toks, T, &g->e);
    if (!g->e.status) {
        forward(g->base, NULL, h, g->bc, &b, &g->e);
        g->cnt.base++;
    }
    if (!g->e.status) {
        float* lg = lm_logits(g->base, h, T);
        const int fr = nc - 1;
        float* bd = xcalloc((size_t)(t->n_nodes + 1) * V, sizeof(float));
        for (int i = 0; i <= t->n_nodes && !g->e.status; ++i)
            softmax_temp(lg + (size_t)(fr + i) * V, V, g->run.temperature, bd + (size_t)i * V, &g->e);
        if (!g->e.status) verify(t, bd, V, g->run.temperature, &g->rng, m_out, path, bonus, &g->e);
        if (!g->e.status) {
            int* commit = xcalloc((size_t)(nc + *m_out), sizeof(int));
            for (int i = 0; i < nc; ++i) commit[i] = crow[i];
            for (int i = 0; i < *m_out; ++i) commit[nc + i] = nrows[path[i]];
            cache_commit(g->bc, commit, nc + *m_out, &g->e);
            free(commit);
        }
        free(bd);
        free(lg);
    }
    free(h); free(mask); free(rows); free(toks); free(pos); free(tp); free(nrows); free(crow); free(ctok);
}

/* resolve_draft_cache, orchestrator.cpp:390-405 */
static void resolve_draft(gen_t* g, const tree_t* t, const int* path, int m) {
    if (g->run.algorithm == EO_EASYSPEC && g->run.calibration) {
        cache_discard(g->dc);
        return;
    }
    int* rows = xcalloc((size_t)(m > 0 ? m : 1), sizeof(int));
    int n = 0;
    for (int i = 0; i < m; ++i) {
        const int row = t->nodes[path[i]].cache_row;
        if (row < 0) break;
        rows[n++] = row;
    }
    cache_commit(g->dc, rows, n, &g->e);
    g->draft_cached += n;
    free(rows);
}

static iter_rec* push_iter(eo_result* res) {
    if (res->n_it == res->it_cap) {
        res->it_cap = res->it_cap ? res->it_cap * 2 : 16;
        res->it = realloc(res->it, sizeof(iter_rec) * (size_t)res->it_cap);
    }
    iter_rec* r = &res->it[res->n_it++];
    memset(r, 0, sizeof *r);
    return r;
}

eo_result* eo_generate(const eo_model* base, const eo_model* draft, const eo_run* run,
                       const uint8_t* prompt, int prompt_len) {
    eo_result* res = xcalloc(1, sizeof *res);
    gen_t G;
    memset(&G, 0, sizeof G);
    gen_t* g = &G;
    g->base = base;
    g->draft = draft;
    g->run = *run;
    const int n = run->n;
    g->widths = xcalloc((size_t)(n > 0 ? n : 1), sizeof(int));
    for (int i = 0; i < n; ++i) g->widths[i] = run->widths ? run->widths[i] : 1;
    /* resolve_plan, orchestrator.cpp:120-131 */
    if (run->algorithm != EO_EASYSPEC) plan_make(draft->c.n_layers, 1, &g->plan, &g->e);
    else if (run->plan_override && run->plan_override[0]) plan_parse(run->plan_override, &g->plan, &g->e);
    else plan_make(draft->c.n_layers, run->lp_size, &g->plan, &g->e);
    if (!g->e.status && plan_total(&g->plan) != draft->c.n_layers)
        fail(&g->e, EO_CONFIG, "layer plan covers %d layers, drafter has %d", plan_total(&g->plan),
             draft->c.n_layers);
    /* validate_run_config, orchestrator.cpp:95-118 */
    if (!g->e.status) {
        if (n < 1) fail(&g->e, EO_CONFIG, "speculation length must be >= 1");
        else if (run->max_new_tokens < 1) fail(&g->e, EO_CONFIG, "max_new_tokens must be >= 1");
        else if (run->temperature < 0.0f) fail(&g->e, EO_CONFIG, "temperature must be >= 0");
        for (int i = 0; i < n && !g->e.status; ++i) {
            if (g->widths[i] < 1 || g->widths[i] > draft->c.vocab_size)
                fail(&g->e, EO_CONFIG, "tree widths must lie in [1, vocab]");
            if (run->algorithm == EO_SD && g->widths[i] != 1)
                fail(&g->e, EO_CONFIG, "plain sd requires all tree widths = 1");
        }
        if (!g->e.status && (base->c.vocab_size != draft->c.vocab_size || base->c.d_model != draft->c.d_model))
            fail(&g->e, EO_CONFIG, "base and draft models must share vocabulary and width");
    }
    /* tokenize_prompt, orchestrator.cpp:42-52 */
    if (!g->e.status && base->c.vocab_size < DEFAULT_VOCAB && prompt_len > 0)
        fail(&g->e, EO_CONFIG, "byte prompts need the full 258-token vocabulary");
    push_committed(g, BOS_TOKEN);
    for (int i = 0; i < prompt_len; ++i) push_committed(g, prompt[i]);
    if (!g->e.status) {
        const int needed = g->n_committed + run->max_new_tokens + n;
        const int room = base->c.max_positions < draft->c.max_positions ? base->c.max_positions
                                                                          : draft->c.max_positions;
        if (needed > room) fail(&g->e, EO_CONFIG, "prompt plus max_new_tokens exceeds max_positions (%d > %d)", needed, room);
    }
    res->bcache.n_layers = 0;
    cache_init(&res->bcache, base->c.n_layers, base->c.d_model);
    cache_init(&res->dcache, draft->c.n_layers, draft->c.d_model);
    g->bc = &res->bcache;
    g->dc = &res->dcache;
    rng_seed(&g->rng, run->seed);
    int* generated = xcalloc((size_t)run->max_new_tokens + (size_t)n + 2, sizeof(int));
    int n_gen = 0;
    const int V = base->c.vocab_size;
    /* Generation::run, orchestrator.cpp:163-195 */
    while (!g->e.status && n_gen < run->max_new_tokens) {
        const counters_t before = g->cnt;
        iter_rec rec;
        memset(&rec, 0, sizeof rec);
        if (run->algorithm == EO_VANILLA) {
            /* run_iteration_vanilla, orchestrator.cpp:438-468 */
            int *rows, *toks;
            const int nr = stage_suffix(g, g->bc, g->bc->committed, 0, &rows, &toks);
            int* pos = xcalloc((size_t)nr, sizeof(int));
            for (int i = 0; i < nr; ++i) pos[i] = cache_position(g->bc, rows[i]);
            unsigned char* mask = cache_mask(g->bc);
            batch_t b = {rows, pos, nr, mask, cache_total(g->bc), 0};
            float* h = embed(base, toks, nr, &g->e);
            if (!g->e.status) {
                forward(base, NULL, h, g->bc, &b, &g->e);
                g->cnt.base++;
            }
            if (!g->e.status) {
                float* lg = lm_logits(base, h + (size_t)(nr - 1) * base->c.d_model, 1);
                float* dist = xcalloc((size_t)V, sizeof(float));
                softmax_temp(lg, V, run->temperature, dist, &g->e);
                int next = 0;
                if (!g->e.status)
                    next = run->temperature == 0.0f ? argmax_f(dist, V) : sample_from(dist, V, &g->rng, &g->e);
                cache_commit(g->bc, rows, nr, &g->e);
                push_committed(g, next);
                generated[n_gen++] = next;
                free(dist);
                free(lg);
            }
            rec.emitted = 1;
            free(h); free(mask); free(rows); free(toks); free(pos);
        } else {
            /* run_iteration_speculative, orchestrator.cpp:407-436 */
            rec.n = n;
            float* root = leading_pass(g);
            tree_t t;
            memset(&t, 0, sizeof t);
            int m = 0, bonus = 0;
            int* path = xcalloc((size_t)n + 1, sizeof(int));
            if (!g->e.status) {
                draft_tree(draft, &g->plan, g->dc, root, g->widths, n, run->temperature, &g->rng, &g->cnt,
                           run->algorithm == EO_EASYSPEC, &t, &g->e);
                rec.drafted = t.n_nodes;
            }
            if (!g->e.status) verify_stage(g, &t, &m, path, &bonus);
            if (!g->e.status) resolve_draft(g, &t, path, m);
            if (!g->e.status) {
                for (int i = 0; i < m; ++i) push_committed(g, t.nodes[path[i]].token);
                push_committed(g, bonus);
                const int remaining = run->max_new_tokens - n_gen;
                const int emit = m + 1 < remaining ? m + 1 : remaining;
                for (int i = 0; i < emit; ++i) generated[n_gen++] = g->committed[g->n_committed - (m + 1) + i];
                rec.m = m;
                rec.emitted = emit;
            }
            free(path);
            free(root);
            tree_free(&t);
        }
        if (g->e.status) break;
        rec.seq = (int)(g->cnt.seq - before.seq);
        rec.fuzzy = (int)(g->cnt.fuzzy - before.fuzzy);
        rec.base = (int)(g->cnt.base - before.base);
        rec.committed = g->n_committed;
        rec.dcommitted = g->dc->committed;
        rec.bcommitted = g->bc->committed;
        rec.dsums = kv_sums(g->dc);
        rec.bsums = kv_sums(g->bc);
        *push_iter(res) = rec;
    }
    res->status = g->e.status;
    memcpy(res->msg, g->e.msg, sizeof res->msg);
    res->tokens = generated;
    res->n_tokens = n_gen;
    free(g->widths);
    free(g->committed);
    return res;
}

int eo_result_status(const eo_result* r) { return r->status; }
const char* eo_result_error(const eo_result* r) { return r->msg; }
const int* eo_result_tokens(const eo_result* r, int* n) { *n = r->n_tokens; return r->tokens; }
int eo_result_n_iters(const eo_result* r) { return r->n_it; }

void eo_result_iter(const eo_result* r, int i, int* out) {
    const iter_rec* x = &r->it[i];
    const int v[10] = {x->m, x->n, x->drafted, x->emitted, x->seq, x->fuzzy, x->base, x->committed,
                       x->dcommitted, x->bcommitted};
    memcpy(out, v, sizeof v);
}

void eo_result_kvsums(const eo_result* r, int i, int which_base, double* out) {
    const cache_t* c = which_base ? &r->bcache : &r->dcache;
    memcpy(out, which_base ? r->it[i].bsums : r->it[i].dsums, sizeof(double) * 4 * (size_t)c->n_layers);
}

int eo_result_cache_len(const eo_result* r, int which_base) {
    return which_base ? r->bcache.committed : r->dcache.committed;
}

void eo_result_cache_rows(const eo_result* r, int which_base, int layer, float* k, float* v) {
    const cache_t* c = which_base ? &r->bcache : &r->dcache;
    memcpy(k, c->k[layer], sizeof(float) * (size_t)c->committed * c->d);
    memcpy(v, c->v[layer], sizeof(float) * (size_t)c->committed * c->d);
}

void eo_result_free(eo_result* r) {
    if (!r) return;
    for (int i = 0; i < r->n_it; ++i) {
        free(r->it[i].dsums);
        free(r->it[i].bsums);
    }
    free(r->it);
    free(r->tokens);
    cache_free(&r->dcache);
    cache_free(&r->bcache);
    free(r);
}
