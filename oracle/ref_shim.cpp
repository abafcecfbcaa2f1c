// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNCHANGED reference headers, compiled straight
// from /root/reference/proj/include by oracle/Makefile into oracle/_ref/libcgref.so.
// Nothing from the reference is copied into this repository: this file only calls
// the reference's public API (corpus.hpp, huffman.hpp, model.hpp, trainer.hpp).
// It serves two purposes: pinning the C restatement (oracle/cg_oracle.c) bit for
// bit, and timing the reference CPU path for bench.py's cpu_baseline and
// `--impl reference` legs (kind "reference").
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "cachegram/corpus.hpp"
#include "cachegram/eval.hpp"
#include "cachegram/huffman.hpp"
#include "cachegram/model.hpp"
#include "cachegram/rng.hpp"
#include "cachegram/trainer.hpp"

using namespace cachegram;

namespace {
struct RefHandle {
    Vocabulary vocab;
    HuffmanTree tree;
};

thread_local std::string g_err;

Vocabulary vocab_from_counts(const int64_t* counts, int32_t v) {
    std::vector<VocabEntry> entries;
    int64_t total = 0;
    for (int32_t i = 0; i < v; ++i) {
        entries.push_back({"w" + std::to_string(i), counts[i]});
        total += counts[i];
    }
    return Vocabulary(std::move(entries), total);
}
}  // namespace

extern "C" {
#pragma GCC visibility push(default)

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

void ref_rng_stream(uint64_t seed, int64_t n, uint64_t* out_u64, float* out_float, uint32_t below, uint32_t* out_below) {
    Rng a(seed), b(seed), c(seed);
    for (int64_t i = 0; i < n; ++i) {
        out_u64[i] = a.next_u64();
        out_float[i] = b.next_float();
        out_below[i] = c.next_below(below);
    }
}

double ref_keep_probability(int64_t count, int64_t total, double sample) {
    return keep_probability(count, total, sample);
}

float ref_update_alpha(uint64_t done, uint64_t total, float alpha0) { return update_alpha(done, total, alpha0); }

float ref_sigmoid_value(float x) {
    static const SigmoidTable table;
    return table.value(x);
}

void ref_init_model(int32_t v, int32_t d, uint64_t seed, float* syn0, float* syn1) {
    Model m = init_model(v, d, seed);
    std::memcpy(syn0, m.input_matrix().data(), m.input_matrix().size() * sizeof(float));
    std::memcpy(syn1, m.weight_matrix().data(), m.weight_matrix().size() * sizeof(float));
}

int32_t ref_shrink_window(int32_t window, uint64_t seed, int64_t n, int32_t* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = shrink_window(window, rng);
    return 0;
}

// ---- vocabulary + tree handles -------------------------------------------
void* ref_open_file(const char* path, int64_t min_count) {
    try {
        auto* h = new RefHandle{build_vocabulary_file(path, min_count), {}};
        h->tree = build_huffman_tree(h->vocab);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ref_open_counts(const int64_t* counts, int32_t v) {
    try {
        auto* h = new RefHandle{vocab_from_counts(counts, v), {}};
        h->tree = build_huffman_tree(h->vocab);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_close(void* hp) { delete static_cast<RefHandle*>(hp); }

int32_t ref_vocab_size(void* hp) { return static_cast<RefHandle*>(hp)->vocab.size(); }
int64_t ref_total_tokens(void* hp) { return static_cast<RefHandle*>(hp)->vocab.total_tokens(); }

// For "w<raw>" words, the raw number; -1 otherwise.
void ref_vocab_export(void* hp, int64_t* counts, int64_t* raw_ids) {
    auto* h = static_cast<RefHandle*>(hp);
    for (int32_t i = 0; i < h->vocab.size(); ++i) {
        counts[i] = h->vocab.count(i);
        const std::string& w = h->vocab.word(i);
        int64_t r = -1;
        if (w.size() > 1 && w[0] == 'w') {
            r = 0;
            for (size_t k = 1; k < w.size(); ++k) {
                if (w[k] < '0' || w[k] > '9') { r = -1; break; }
                r = r * 10 + (w[k] - '0');
            }
        }
        raw_ids[i] = r;
    }
}

int64_t ref_tree_steps(void* hp) {
    auto* h = static_cast<RefHandle*>(hp);
    int64_t s = 0;
    for (int32_t w = 0; w < h->vocab.size(); ++w) s += static_cast<int64_t>(h->tree.path(w).size());
    return s;
}

void ref_tree_export(void* hp, int64_t* offsets, int32_t* nodes, uint8_t* turns, int64_t* usage) {
    auto* h = static_cast<RefHandle*>(hp);
    int64_t k = 0;
    for (int32_t w = 0; w < h->vocab.size(); ++w) {
        offsets[w] = k;
        for (const PathStep& s : h->tree.path(w)) {
            nodes[k] = s.node;
            turns[k] = s.turn;
            ++k;
        }
    }
    offsets[h->vocab.size()] = k;
    for (int32_t n = 0; n < h->tree.inner_count(); ++n) usage[n] = h->tree.node_usage(n);
}

int32_t ref_select(void* hp, int32_t k, int32_t* hot, int32_t* slot_of) {
    auto* h = static_cast<RefHandle*>(hp);
    CacheSelection sel = select_cached_nodes(h->tree, k);
    for (int32_t s = 0; s < sel.size(); ++s) hot[s] = sel.node_at(s);
    for (int32_t n = 0; n < sel.inner_node_count(); ++n) slot_of[n] = sel.slot_of(n);
    return sel.size();
}

// ---- the hot path: cachegram::train() -----------------------------------
// Returns 0, or 1 for invalid_argument, 2 for IoError, 3 otherwise.
int ref_train(void* hp, const char* corpus_path, int32_t dim, int32_t window, int64_t min_count, double sample,
              float alpha0, int32_t iterations, int32_t workers, int32_t cache_nodes, int32_t flush_interval,
              uint64_t seed, float* syn0_out, float* syn1_out, uint64_t* words_processed, double* wall_seconds) {
    auto* h = static_cast<RefHandle*>(hp);
    try {
        TrainConfig cfg;
        cfg.dim = dim;
        cfg.window = window;
        cfg.min_count = min_count;
        cfg.sample = sample;
        cfg.alpha0 = alpha0;
        cfg.iterations = iterations;
        cfg.workers = workers;
        cfg.cache_nodes = cache_nodes;
        cfg.flush_interval = flush_interval;
        cfg.seed = seed;
        CacheSelection sel = select_cached_nodes(h->tree, cache_nodes);
        TrainStats stats;
        Model m = train(corpus_path, h->vocab, h->tree, sel, cfg, &stats);
        if (syn0_out) std::memcpy(syn0_out, m.input_matrix().data(), m.input_matrix().size() * sizeof(float));
        if (syn1_out) std::memcpy(syn1_out, m.weight_matrix().data(), m.weight_matrix().size() * sizeof(float));
        if (words_processed) *words_processed = stats.words_processed;
        if (wall_seconds) *wall_seconds = stats.wall_seconds;
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// One train_center call (trainer.hpp:147-175) on a counts-built vocabulary, then an
// optional NodeCache::flush. sigmoid_mode: 0 table, 1 exact (testutil ExactSigmoid),
// 2 constant. Returns the number of sigmoid evaluations.
int64_t ref_train_center(const int64_t* counts, int32_t v, int32_t dim, float* syn0, float* syn1, int32_t cache_nodes,
                         int32_t do_flush, int32_t center, const int32_t* sentence, int64_t len, int64_t center_pos,
                         int32_t half_window, float alpha, int32_t sigmoid_mode, float sig_const) {
    Vocabulary vocab = vocab_from_counts(counts, v);
    HuffmanTree tree = build_huffman_tree(vocab);
    Model model(v, dim);
    std::memcpy(model.input_matrix().data(), syn0, model.input_matrix().size() * sizeof(float));
    std::memcpy(model.weight_matrix().data(), syn1, model.weight_matrix().size() * sizeof(float));
    CacheSelection sel = select_cached_nodes(tree, cache_nodes);
    NodeCache cache(sel, dim, 1000000);
    std::vector<float> hidden(static_cast<size_t>(dim));
    int64_t evals = 0;
    std::span<const int32_t> sent(sentence, static_cast<size_t>(len));
    static const SigmoidTable table;
    if (sigmoid_mode == 0) {
        auto fn = [&](float x) { ++evals; return table.value(x); };
        train_center(center, sent, static_cast<size_t>(center_pos), half_window, model, tree, sel, cache, alpha,
                     hidden.data(), fn);
    } else if (sigmoid_mode == 1) {
        auto fn = [&](float x) { ++evals; return static_cast<float>(1.0 / (1.0 + std::exp(-static_cast<double>(x)))); };
        train_center(center, sent, static_cast<size_t>(center_pos), half_window, model, tree, sel, cache, alpha,
                     hidden.data(), fn);
    } else {
        auto fn = [&](float) { ++evals; return sig_const; };
        train_center(center, sent, static_cast<size_t>(center_pos), half_window, model, tree, sel, cache, alpha,
                     hidden.data(), fn);
    }
    if (do_flush) cache.flush(model);
    std::memcpy(syn0, model.input_matrix().data(), model.input_matrix().size() * sizeof(float));
    std::memcpy(syn1, model.weight_matrix().data(), model.weight_matrix().size() * sizeof(float));
    return evals;
}

// ---- evaluation and model files (eval.hpp, model.hpp:107-276) ---------------
namespace {
LoadedEmbeddings embeddings_of(const float* vectors, int32_t rows, int32_t dim) {
    LoadedEmbeddings e;
    e.dim = dim;
    for (int32_t w = 0; w < rows; ++w) e.words.push_back("w" + std::to_string(w));
    e.vectors.assign(vectors, vectors + static_cast<size_t>(rows) * dim);
    return e;
}
}  // namespace

// AnalogySolver(embeddings, restrict_top).answer(a, b, c) for n questions.
int ref_analogy(const float* vectors, int32_t rows, int32_t dim, int32_t restrict_top, const int32_t* abc, int64_t n,
                int32_t* out) {
    try {
        const AnalogySolver solver(embeddings_of(vectors, rows, dim), restrict_top);
        for (int64_t q = 0; q < n; ++q) out[q] = solver.answer(abc[3 * q], abc[3 * q + 1], abc[3 * q + 2]);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// save_text (binary == 0) or save_binary of a model whose words are NUL-separated.
int ref_model_save(const char* path, int32_t binary, const char* words_nul, const float* syn0, int32_t v, int32_t d) {
    try {
        std::vector<VocabEntry> entries;
        const char* p = words_nul;
        for (int32_t i = 0; i < v; ++i) {
            entries.push_back({std::string(p), 1});
            p += std::strlen(p) + 1;
        }
        const Vocabulary vocab(std::move(entries), v);
        Model m(v, d);
        std::memcpy(m.input_matrix().data(), syn0, sizeof(float) * static_cast<size_t>(v) * d);
        if (binary)
            save_binary(m, vocab, path);
        else
            save_text(m, vocab, path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// load_embeddings (format 2), load_embeddings_text (0) or load_embeddings_binary (1).
// Returns 0 and fills rows/dim/vectors (capacity floats) or -1 IoError / -2 ParseError.
int ref_model_load(const char* path, int32_t format, int32_t* rows, int32_t* dim, float* vectors, int64_t capacity) {
    try {
        const LoadedEmbeddings e = format == 0   ? load_embeddings_text(path)
                                   : format == 1 ? load_embeddings_binary(path)
                                                 : load_embeddings(path);
        *rows = e.size();
        *dim = e.dim;
        if (vectors && static_cast<int64_t>(e.vectors.size()) <= capacity)
            std::memcpy(vectors, e.vectors.data(), e.vectors.size() * sizeof(float));
        return 0;
    } catch (const IoError& e) {
        g_err = e.what();
        return -1;
    } catch (const ParseError& e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -3;
    }
}

#pragma GCC visibility pop
}  // extern "C"
