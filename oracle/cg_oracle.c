/*
 * cg_oracle.c -- TEST INFRASTRUCTURE ONLY (see cg_oracle.h).
 *
 * A scalar C restatement of the reference's skip-gram / hierarchical-softmax
 * training path. Arithmetic is IEEE fp32, evaluated in source order with no
 * contraction (build with -ffp-contract=off and no -march flags), which is what
 * the reference's default build produces (CMakeLists.txt:12, vec_ops.hpp:14-18).
 */
#include "cg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_SENTENCE 1000     /* trainer.hpp:185 kMaxSentence */
#define ORC_ALPHA_BATCH 10000 /* trainer.hpp:186 kAlphaBatch */

/* ---- rng.hpp:13-43 ----------------------------------------------------- */
uint64_t orc_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static float rng_unit(uint64_t* s) { /* rng.hpp:25-27: top 24 bits, exact in float */
    return (float)(orc_splitmix_next(s) >> 40) * (1.0f / 16777216.0f);
}

static uint32_t rng_below(uint64_t* s, uint32_t n) { /* rng.hpp:30-32 */
    return (uint32_t)(orc_splitmix_next(s) % (uint64_t)n);
}

uint64_t orc_mix_seed(uint64_t seed, uint64_t stream) {
    uint64_t s = seed ^ (0x632be59bd9b4e019ull * (stream + 1));
    return orc_splitmix_next(&s);
}

/* ---- corpus.hpp:176-181 ------------------------------------------------- */
double orc_keep_probability(int64_t count, int64_t total, double sample) {
    double budget = sample * (double)total;
    double c = (double)count;
    double p = (sqrt(c / budget) + 1.0) * budget / c;
    return p < 1.0 ? p : 1.0;
}

/* ---- trainer.hpp:58-63 -------------------------------------------------- */
float orc_update_alpha(uint64_t done, uint64_t total, float alpha0) {
    double frac = (double)done / ((double)total + 1.0);
    float a = alpha0 * (float)(1.0 - frac);
    float lo = alpha0 * 1e-4f;
    return a > lo ? a : lo;
}

/* ---- model.hpp:84-99 ---------------------------------------------------- */
void orc_sigmoid_table(float* out) {
    const double width = 2.0 * 6.0 / 1000.0;
    for (int i = 0; i < 1000; ++i) {
        double x = -6.0 + (i + 0.5) * width;
        out[i] = (float)(1.0 / (1.0 + exp(-x)));
    }
}

static float table_sigmoid(const float* t, float x) {
    if (x <= -6.0f) return t[0];
    if (x >= 6.0f) return t[999];
    const float scale = 1000.0f / 12.0f; /* kResolution / (2*kDomain), folded in float */
    int32_t idx = (int32_t)((x + 6.0f) * scale);
    if (idx >= 1000) idx = 999;
    return t[idx];
}

static float exact_sigmoid_f(float x) { return (float)(1.0 / (1.0 + exp(-(double)x))); }

/* ---- model.hpp:66-72 ---------------------------------------------------- */
void orc_init_model(int32_t vocab, int32_t dim, uint64_t seed, float* syn0, float* syn1) {
    uint64_t s = orc_mix_seed(seed, 0x1817);
    const float inv = 1.0f / (float)dim;
    const size_t n0 = (size_t)vocab * (size_t)dim;
    for (size_t i = 0; i < n0; ++i) syn0[i] = (rng_unit(&s) - 0.5f) * inv;
    if (syn1) memset(syn1, 0, (size_t)(vocab - 1) * (size_t)dim * sizeof(float));
}

/* ---- huffman.hpp:57-108 -------------------------------------------------
 * Binary min-heap keyed on (count, node id); keys are unique, so the pop
 * sequence equals std::priority_queue<.., std::greater<>> in the reference. */
typedef struct { int64_t c; int32_t id; } hitem;

static int hless(hitem a, hitem b) { return a.c < b.c || (a.c == b.c && a.id < b.id); }

static void hpush(hitem* h, int32_t* n, hitem x) {
    int32_t i = (*n)++;
    h[i] = x;
    while (i > 0) {
        int32_t p = (i - 1) / 2;
        if (!hless(h[i], h[p])) break;
        hitem t = h[i]; h[i] = h[p]; h[p] = t;
        i = p;
    }
}

static hitem hpop(hitem* h, int32_t* n) {
    hitem top = h[0];
    h[0] = h[--(*n)];
    int32_t i = 0;
    for (;;) {
        int32_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && hless(h[l], h[m])) m = l;
        if (r < *n && hless(h[r], h[m])) m = r;
        if (m == i) break;
        hitem t = h[i]; h[i] = h[m]; h[m] = t;
        i = m;
    }
    return top;
}

int orc_build_huffman(const int64_t* counts, int32_t vocab, int64_t* offsets, int32_t* nodes, uint8_t* turns,
                      int64_t* usage, int64_t* n_steps) {
    if (vocab < 2) return -1;
    const int32_t total = 2 * vocab - 1;
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)total);
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)total);
    uint8_t* turn = (uint8_t*)malloc((size_t)total);
    hitem* heap = (hitem*)malloc(sizeof(hitem) * (size_t)vocab);
    int32_t hn = 0;
    for (int32_t w = 0; w < vocab; ++w) {
        cnt[w] = counts[w];
        parent[w] = -1;
        turn[w] = 0;
        hitem it = {counts[w], w};
        hpush(heap, &hn, it);
    }
    for (int32_t nx = vocab; nx < total; ++nx) {
        hitem a = hpop(heap, &hn), b = hpop(heap, &hn);
        cnt[nx] = a.c + b.c;
        parent[nx] = -1;
        parent[a.id] = nx; turn[a.id] = 0;
        parent[b.id] = nx; turn[b.id] = 1;
        hitem m = {a.c + b.c, nx};
        hpush(heap, &hn, m);
    }
    if (usage)
        for (int32_t n = 0; n < vocab - 1; ++n) usage[n] = cnt[vocab + n];
    /* depth pass, then root-first fill (walk leaf->root, write backwards) */
    int64_t steps = 0;
    for (int32_t w = 0; w < vocab; ++w) {
        int32_t d = 0;
        for (int32_t x = w; parent[x] != -1; x = parent[x]) ++d;
        if (offsets) offsets[w] = steps;
        if (nodes) {
            int64_t k = steps + d - 1;
            for (int32_t x = w; parent[x] != -1; x = parent[x], --k) {
                nodes[k] = parent[x] - vocab;
                turns[k] = turn[x];
            }
        }
        steps += d;
    }
    if (offsets) offsets[vocab] = steps;
    if (n_steps) *n_steps = steps;
    free(cnt); free(parent); free(turn); free(heap);
    return 0;
}

/* ---- huffman.hpp:139-159 ------------------------------------------------ */
static const int64_t* g_sort_usage;
static int usage_cmp(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    if (g_sort_usage[x] != g_sort_usage[y]) return g_sort_usage[x] > g_sort_usage[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

int32_t orc_select_cached(const int64_t* usage, int32_t inner, int32_t k, int32_t* hot_nodes, int32_t* slot_of) {
    if (k < 0) return -1;
    int32_t take = k < inner ? k : inner;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(inner > 0 ? inner : 1));
    for (int32_t i = 0; i < inner; ++i) order[i] = i;
    g_sort_usage = usage;
    qsort(order, (size_t)inner, sizeof(int32_t), usage_cmp);
    for (int32_t i = 0; i < inner; ++i) slot_of[i] = -1;
    for (int32_t s = 0; s < take; ++s) {
        hot_nodes[s] = order[s];
        slot_of[order[s]] = s;
    }
    free(order);
    return take;
}

/* ---- corpus.hpp:86-124 over integer tokens ------------------------------ */
static const int64_t* g_vc;
static const int64_t* g_vo;
static int vocab_cmp(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    if (g_vc[x] != g_vc[y]) return g_vc[x] > g_vc[y] ? -1 : 1;
    return g_vo[x] < g_vo[y] ? -1 : (g_vo[x] > g_vo[y]);
}

int32_t orc_vocab_from_ids(const int32_t* raw, int64_t n, int32_t raw_space, int64_t min_count, int32_t* rank_of_raw,
                           int64_t* counts_out, int64_t* total_out) {
    int64_t* c = (int64_t*)calloc((size_t)raw_space, sizeof(int64_t));
    int64_t* first = (int64_t*)malloc(sizeof(int64_t) * (size_t)raw_space);
    for (int32_t i = 0; i < raw_space; ++i) first[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        int32_t r = raw[i];
        if (first[r] < 0) first[r] = i;
        ++c[r];
    }
    int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)raw_space);
    int32_t m = 0;
    for (int32_t r = 0; r < raw_space; ++r)
        if (c[r] >= min_count && c[r] > 0) ord[m++] = r;
    g_vc = c; g_vo = first;
    qsort(ord, (size_t)m, sizeof(int32_t), vocab_cmp);
    for (int32_t r = 0; r < raw_space; ++r) rank_of_raw[r] = -1;
    int64_t tot = 0;
    for (int32_t i = 0; i < m; ++i) {
        rank_of_raw[ord[i]] = i;
        counts_out[i] = c[ord[i]];
        tot += c[ord[i]];
    }
    *total_out = tot;
    free(c); free(first); free(ord);
    return m;
}

/* ---- trainer.hpp:96-124 (NodeCache) and 147-175 (train_center) ---------- */
static float* cache_acquire(int32_t slot, int32_t dim, const float* shared, float* work, float* snap, uint8_t* flag,
                            int32_t* acquired, int32_t* n_acq) {
    float* w = work + (size_t)slot * dim;
    if (!flag[slot]) {
        float* s = snap + (size_t)slot * dim;
        for (int32_t d = 0; d < dim; ++d) w[d] = shared[d];
        for (int32_t d = 0; d < dim; ++d) s[d] = w[d];
        flag[slot] = 1;
        acquired[(*n_acq)++] = slot;
    }
    return w;
}

void orc_cache_flush(int32_t dim, float* syn1, const int32_t* hot_nodes, float* work, const float* snap,
                     uint8_t* flag, const int32_t* acquired, int32_t* n_acq) {
    for (int32_t i = 0; i < *n_acq; ++i) {
        int32_t slot = acquired[i];
        float* sh = syn1 + (size_t)hot_nodes[slot] * dim;
        const float* w = work + (size_t)slot * dim;
        const float* s = snap + (size_t)slot * dim;
        for (int32_t d = 0; d < dim; ++d) {
            float delta = w[d] - s[d];
            sh[d] += delta;
        }
        flag[slot] = 0;
    }
    *n_acq = 0;
}

static const float* g_table; /* set by callers that use sigmoid_mode 0 */

int64_t orc_train_center(int32_t center, const int32_t* sentence, int64_t len, int64_t cpos, int32_t hw, int32_t dim,
                         float* syn0, float* syn1, const int64_t* offsets, const int32_t* nodes, const uint8_t* turns,
                         const int32_t* slot_of, float* work, float* snap, uint8_t* flag, int32_t* acquired,
                         int32_t* n_acq, float alpha, int32_t mode, float sig_const) {
    float table_local[1000];
    const float* table = g_table;
    if (mode == 0 && !table) { orc_sigmoid_table(table_local); table = table_local; }
    float* hidden = (float*)malloc(sizeof(float) * (size_t)dim);
    int64_t evals = 0;
    const int64_t p0 = offsets[center], p1 = offsets[center + 1];
    const int64_t lo = cpos >= hw ? cpos - hw : 0;
    const int64_t hi = (len - 1) < (cpos + hw) ? (len - 1) : (cpos + hw);
    for (int64_t pos = lo; pos <= hi; ++pos) {
        if (pos == cpos) continue;
        float* v = syn0 + (size_t)sentence[pos] * dim;
        for (int32_t d = 0; d < dim; ++d) hidden[d] = 0.0f;
        for (int64_t k = p0; k < p1; ++k) {
            const int32_t node = nodes[k];
            float* u;
            const int32_t slot = slot_of ? slot_of[node] : -1;
            if (slot >= 0)
                u = cache_acquire(slot, dim, syn1 + (size_t)node * dim, work, snap, flag, acquired, n_acq);
            else
                u = syn1 + (size_t)node * dim;
            float acc = 0.0f; /* vec_ops.hpp:14-18, sequential, no FMA */
            for (int32_t d = 0; d < dim; ++d) acc += v[d] * u[d];
            float f = mode == 0 ? table_sigmoid(table, acc) : (mode == 1 ? exact_sigmoid_f(acc) : sig_const);
            ++evals;
            const float g = (1.0f - (float)turns[k] - f) * alpha;
            for (int32_t d = 0; d < dim; ++d) hidden[d] += g * u[d];
            for (int32_t d = 0; d < dim; ++d) u[d] += g * v[d];
        }
        for (int32_t d = 0; d < dim; ++d) v[d] += 1.0f * hidden[d];
    }
    free(hidden);
    return evals;
}

/* ---- trainer.hpp:200-245 (train_worker, worker 0 of 1) ------------------ */
int orc_train_single(const int32_t* ids, int64_t n_ids, int32_t vocab, const int64_t* counts, int64_t total_tokens,
                     const int64_t* offsets, const int32_t* nodes, const uint8_t* turns, const int32_t* hot_nodes,
                     int32_t hot_count, const int32_t* slot_of, const orc_config* cfg, float* syn0, float* syn1,
                     orc_stats* st) {
    const int32_t dim = cfg->dim;
    float table[1000];
    orc_sigmoid_table(table);
    g_table = table;
    float* keep = NULL;
    if (cfg->sample > 0.0) {
        keep = (float*)malloc(sizeof(float) * (size_t)vocab);
        for (int32_t w = 0; w < vocab; ++w) keep[w] = (float)orc_keep_probability(counts[w], total_tokens, cfg->sample);
    }
    const int32_t hc = hot_count > 0 ? hot_count : 1;
    float* work = (float*)malloc(sizeof(float) * (size_t)hc * dim);
    float* snap = (float*)malloc(sizeof(float) * (size_t)hc * dim);
    uint8_t* flag = (uint8_t*)calloc((size_t)hc, 1);
    int32_t* acquired = (int32_t*)malloc(sizeof(int32_t) * (size_t)hc);
    int32_t n_acq = 0;
    int32_t sentence[ORC_SENTENCE];
    const uint64_t total_words = (uint64_t)cfg->iterations * (uint64_t)total_tokens;
    uint64_t rng = orc_mix_seed(cfg->seed, 0);
    uint64_t progress = 0, unreported = 0;
    float alpha = orc_update_alpha(0, total_words, cfg->alpha0);
    int32_t since_flush = 0;
    orc_stats s;
    memset(&s, 0, sizeof s);

    for (int32_t it = 0; it < cfg->iterations; ++it) {
        int64_t pos = 0;
        int live = 1;
        while (live) {
            int64_t len = 0;
            while (len < ORC_SENTENCE && (live = (pos < n_ids))) {
                const int32_t id = ids[pos++];
                if (++unreported >= ORC_ALPHA_BATCH) {
                    progress += unreported;
                    unreported = 0;
                    alpha = orc_update_alpha(progress, total_words, cfg->alpha0);
                }
                if (keep) {
                    const float kp = keep[id];
                    if (kp < 1.0f && rng_unit(&rng) >= kp) continue;
                }
                sentence[len++] = id;
            }
            for (int64_t p = 0; p < len; ++p) {
                const int32_t hw = cfg->window - (int32_t)rng_below(&rng, (uint32_t)cfg->window);
                const int64_t lo = p >= hw ? p - hw : 0;
                const int64_t hi = (len - 1) < (p + hw) ? (len - 1) : (p + hw);
                const int64_t npairs = hi - lo; /* window minus the center itself */
                s.pairs += (uint64_t)npairs;
                s.steps += (uint64_t)(npairs * (offsets[sentence[p] + 1] - offsets[sentence[p]]));
                orc_train_center(sentence[p], sentence, len, p, hw, dim, syn0, syn1, offsets, nodes, turns,
                                 hot_count > 0 ? slot_of : NULL, work, snap, flag, acquired, &n_acq, alpha, 0, 0.0f);
                ++s.centers;
                if (++since_flush >= cfg->flush_interval) {
                    orc_cache_flush(dim, syn1, hot_nodes, work, snap, flag, acquired, &n_acq);
                    since_flush = 0;
                    ++s.flushes;
                }
            }
        }
        orc_cache_flush(dim, syn1, hot_nodes, work, snap, flag, acquired, &n_acq);
        since_flush = 0;
        ++s.flushes;
    }
    progress += unreported;
    s.words_processed = progress;
    if (st) *st = s;
    g_table = NULL;
    free(keep); free(work); free(snap); free(flag); free(acquired);
    return 0;
}

/* ---- harness: HS log-loss (tests/acceptance.cpp:100-110) ---------------- */
double orc_hs_loss(const int32_t* centers, const int32_t* contexts, int64_t n_pairs, int32_t dim, const float* syn0,
                   const float* syn1, const int64_t* offsets, const int32_t* nodes, const uint8_t* turns) {
    double total = 0.0;
    for (int64_t i = 0; i < n_pairs; ++i) {
        const float* v = syn0 + (size_t)contexts[i] * dim;
        double ll = 0.0;
        for (int64_t k = offsets[centers[i]]; k < offsets[centers[i] + 1]; ++k) {
            const float* u = syn1 + (size_t)nodes[k] * dim;
            double x = 0.0;
            for (int32_t d = 0; d < dim; ++d) x += (double)v[d] * (double)u[d];
            /* log(sigmoid(x)) and log(1 - sigmoid(x)) in a numerically safe form */
            const double ls = x >= 0 ? -log1p(exp(-x)) : x - log1p(exp(x));
            const double lns = x >= 0 ? -x - log1p(exp(-x)) : -log1p(exp(x));
            ll += turns[k] == 0 ? ls : lns;
        }
        total += -ll;
    }
    return n_pairs > 0 ? total / (double)n_pairs : 0.0;
}

int64_t orc_sample_pairs(const int32_t* ids, int64_t n_ids, const float* keep, int32_t window, uint64_t seed,
                         int64_t n_pairs, int32_t* centers, int32_t* contexts) {
    uint64_t rng = orc_mix_seed(seed, 0xe7a1);
    /* accept each candidate pair with probability q so the set spans the stream */
    double q = (double)n_pairs / ((double)n_ids * 2.0 + 1.0);
    if (q > 1.0) q = 1.0;
    const uint64_t thresh = (uint64_t)(q * 18446744073709551615.0);
    int64_t got = 0;
    int32_t sentence[ORC_SENTENCE];
    for (int pass = 0; pass < 64 && got < n_pairs; ++pass) {
        int64_t pos = 0;
        while (pos < n_ids && got < n_pairs) {
            int64_t len = 0;
            while (len < ORC_SENTENCE && pos < n_ids) {
                const int32_t id = ids[pos++];
                if (keep && keep[id] < 1.0f && rng_unit(&rng) >= keep[id]) continue;
                sentence[len++] = id;
            }
            for (int64_t p = 0; p < len && got < n_pairs; ++p) {
                const int32_t hw = window - (int32_t)rng_below(&rng, (uint32_t)window);
                const int64_t lo = p >= hw ? p - hw : 0;
                const int64_t hi = (len - 1) < (p + hw) ? (len - 1) : (p + hw);
                for (int64_t x = lo; x <= hi && got < n_pairs; ++x) {
                    if (x == p) continue;
                    if (orc_splitmix_next(&rng) > thresh) continue;
                    centers[got] = sentence[p];
                    contexts[got] = sentence[x];
                    ++got;
                }
            }
        }
    }
    return got;
}


/* ---------------------------------------------------------------- evaluation */
/* vec_ops.hpp:14-18: sum from +0, ascending i, separately rounded mul and add. */
static float orc_dot(const float* a, const float* b, int32_t n) {
    float s = 0.0f;
    for (int32_t i = 0; i < n; ++i) {
        const float p = a[i] * b[i];
        s = s + p;
    }
    return s;
}

/* eval.hpp:91-103 */
void orc_normalize(const float* src, int64_t rows, int32_t dim, float* out) {
    for (int64_t r = 0; r < rows; ++r) {
        const float* x = src + r * dim;
        float* y = out + r * dim;
        const float norm = sqrtf(orc_dot(x, x, dim));
        for (int32_t d = 0; d < dim; ++d) y[d] = norm > 0.0f ? x[d] / norm : 0.0f;
    }
}

/* eval.hpp:117-136: target = (vb - va) + vc; the first candidate seeds `best`, later
 * ones replace it only when strictly greater. */
void orc_analogy(const float* norm, int64_t rows, int32_t dim, const int32_t* abc, int64_t n, int32_t* out) {
    float* t = (float*)malloc(sizeof(float) * (size_t)(dim > 0 ? dim : 1));
    for (int64_t q = 0; q < n; ++q) {
        const int32_t a = abc[3 * q], b = abc[3 * q + 1], c = abc[3 * q + 2];
        for (int32_t d = 0; d < dim; ++d) {
            const float diff = norm[(int64_t)b * dim + d] - norm[(int64_t)a * dim + d];
            t[d] = diff + norm[(int64_t)c * dim + d];
        }
        int32_t best = -1;
        float best_score = 0.0f;
        for (int64_t w = 0; w < rows; ++w) {
            if (w == a || w == b || w == c) continue;
            const float s = orc_dot(t, norm + w * dim, dim);
            if (best < 0 || s > best_score) {
                best = (int32_t)w;
                best_score = s;
            }
        }
        out[q] = best;
    }
    free(t);
}

void orc_topk(const float* norm, int64_t rows, int32_t dim, const int32_t* queries, int64_t n, int32_t k,
              int32_t* ids, float* scores) {
    for (int64_t q = 0; q < n; ++q) {
        int32_t* qi = ids + q * k;
        float* qs = scores + q * k;
        int32_t filled = 0;
        for (int32_t r = 0; r < k; ++r) {
            qi[r] = -1;
            qs[r] = NAN;
        }
        const float* x = norm + (int64_t)queries[q] * dim;
        for (int64_t w = 0; w < rows; ++w) {
            if (w == queries[q]) continue;
            const float s = orc_dot(x, norm + w * dim, dim);
            if (isnan(s)) continue;
            /* insertion: strictly greater moves ahead, so equal scores keep the lower id first */
            int32_t pos = filled;
            while (pos > 0 && s > qs[pos - 1]) --pos;
            if (pos >= k) continue;
            const int32_t last = filled < k ? filled : k - 1;
            for (int32_t r = last; r > pos; --r) {
                qi[r] = qi[r - 1];
                qs[r] = qs[r - 1];
            }
            qi[pos] = (int32_t)w;
            qs[pos] = s;
            if (filled < k) ++filled;
        }
    }
}
