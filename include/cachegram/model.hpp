// cachegram-b200: the two weight matrices and the sigmoid lookup of the drop-in API.
//
// Same layout contract as the reference Model (model.hpp:25-62): row-major fp32,
// syn0 = V x D input vectors, syn1 = (V-1) x D inner-node rows in reference node-id
// order. init_model and SigmoidTable reproduce the reference bits (model.hpp:66-99)
// because the deterministic device mode must start from, and look up, the same floats.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cachegram/corpus.hpp"
#include "cachegram/errors.hpp"
#include "cachegram/rng.hpp"
#include "cachegram_b200.h"

namespace cachegram {

class Model {
public:
    Model(std::int32_t vocab_size, std::int32_t dim) : v_(vocab_size), d_(dim) {
        if (vocab_size < 2) throw std::invalid_argument("model needs a vocabulary of at least two words");
        if (dim < 1) throw std::invalid_argument("vector dimension must be >= 1");
        syn0_.assign(static_cast<std::size_t>(vocab_size) * static_cast<std::size_t>(dim), 0.0f);
        syn1_.assign(static_cast<std::size_t>(vocab_size - 1) * static_cast<std::size_t>(dim), 0.0f);
    }

    std::int32_t vocab_size() const { return v_; }
    std::int32_t node_count() const { return v_ - 1; }
    std::int32_t dim() const { return d_; }

    float* input_vector(std::int32_t w) { return syn0_.data() + offset(w); }
    const float* input_vector(std::int32_t w) const { return syn0_.data() + offset(w); }
    float* node_weight(std::int32_t n) { return syn1_.data() + offset(n); }
    const float* node_weight(std::int32_t n) const { return syn1_.data() + offset(n); }

    std::span<float> input_matrix() { return syn0_; }
    std::span<const float> input_matrix() const { return syn0_; }
    std::span<float> weight_matrix() { return syn1_; }
    std::span<const float> weight_matrix() const { return syn1_; }

private:
    std::size_t offset(std::int32_t row) const { return static_cast<std::size_t>(row) * static_cast<std::size_t>(d_); }
    std::int32_t v_, d_;
    std::vector<float> syn0_, syn1_;
};

// syn0 ~ U[-0.5/D, 0.5/D) from Rng(mix_seed(seed, 0x1817)) in row-major order; syn1 = 0.
inline void init_model_into(std::int32_t vocab_size, std::int32_t dim, std::uint64_t seed, float* syn0) {
    Rng r(mix_seed(seed, 0x1817));
    const float scale = 1.0f / static_cast<float>(dim);
    const std::size_t n = static_cast<std::size_t>(vocab_size) * static_cast<std::size_t>(dim);
    for (std::size_t i = 0; i < n; ++i) syn0[i] = (r.next_float() - 0.5f) * scale;
}

inline Model init_model(std::int32_t vocab_size, std::int32_t dim, std::uint64_t seed) {
    Model m(vocab_size, dim);
    init_model_into(vocab_size, dim, seed, m.input_matrix().data());
    return m;
}

inline double exact_sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

// 1000 bucket-centre samples of the logistic on [-6, 6] (double, stored as float);
// lookup truncates (x + 6) * (1000 / 12.0f) and clamps outside the domain.
class SigmoidTable {
public:
    static constexpr float kDomain = 6.0f;
    static constexpr std::int32_t kResolution = 1000;

    SigmoidTable() : t_(kResolution) {
        const double step = 2.0 * static_cast<double>(kDomain) / kResolution;
        for (std::int32_t i = 0; i < kResolution; ++i)
            t_[static_cast<std::size_t>(i)] = static_cast<float>(exact_sigmoid(-6.0 + (i + 0.5) * step));
    }

    float value(float x) const {
        if (x <= -kDomain) return t_.front();
        if (x >= kDomain) return t_.back();
        const float scale = static_cast<float>(kResolution) / (2.0f * kDomain);
        const std::int32_t i = std::min(static_cast<std::int32_t>((x + kDomain) * scale), kResolution - 1);
        return t_[static_cast<std::size_t>(i)];
    }
    float operator()(float x) const { return value(x); }
    const float* data() const { return t_.data(); }

private:
    std::vector<float> t_;
};

// Full-precision logistic, the reference tests' ExactSigmoid (testutil.hpp:28-30).
struct ExactSigmoid {
    float operator()(float x) const { return static_cast<float>(exact_sigmoid(static_cast<double>(x))); }
};

// ---------------------------------------------------------------------------------
// Model files (model.hpp:107-276 of the reference): the input vectors plus the word
// list, as text ("V D" header, "word v1 ... vD" rows, %.6f) or binary ("word " + raw
// float32 + newline). Implemented in libcachegram_b200 (cg_modelio.cpp): the same bytes
// and the same accepted inputs, with text formatting/parsing spread over host cores.
// ---------------------------------------------------------------------------------
namespace model_detail {
[[noreturn]] inline void rethrow_io(int rc) {
    const std::string msg = cg_last_error();
    switch (rc) {
        case CG_ERR_IO: throw IoError(msg);
        case CG_ERR_PARSE: throw ParseError(msg);
        case CG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}
inline void check_io(int rc) {
    if (rc != CG_OK) rethrow_io(rc);
}
inline std::string joined_words(const Vocabulary& vocab, std::int32_t n) {
    std::string out;
    for (std::int32_t w = 0; w < n; ++w) {
        out += vocab.word(w);
        out.push_back('\0');
    }
    return out;
}
inline void save(const Model& model, const Vocabulary& vocab, const std::string& path, std::int32_t format) {
    const std::string words = joined_words(vocab, model.vocab_size());
    check_io(cg_model_save(path.c_str(), format, words.data(), model.input_matrix().data(), model.vocab_size(),
                           model.dim()));
}
}  // namespace model_detail

inline void save_text(const Model& model, const Vocabulary& vocab, const std::string& path) {
    model_detail::save(model, vocab, path, CG_FORMAT_TEXT);
}

inline void save_binary(const Model& model, const Vocabulary& vocab, const std::string& path) {
    model_detail::save(model, vocab, path, CG_FORMAT_BINARY);
}

// What a model file stores: the word list in id order and the input vectors.
struct LoadedEmbeddings {
    std::int32_t dim = 0;
    std::vector<std::string> words;
    std::vector<float> vectors;  // words.size() x dim, row-major

    std::int32_t size() const { return static_cast<std::int32_t>(words.size()); }
    const float* vector(std::int32_t w) const {
        return vectors.data() + static_cast<std::size_t>(w) * static_cast<std::size_t>(dim);
    }
};

inline LoadedEmbeddings to_embeddings(const Model& model, const Vocabulary& vocab) {
    LoadedEmbeddings out;
    out.dim = model.dim();
    out.words.reserve(static_cast<std::size_t>(vocab.size()));
    for (std::int32_t w = 0; w < vocab.size(); ++w) out.words.push_back(vocab.word(w));
    out.vectors.assign(model.input_matrix().begin(), model.input_matrix().end());
    return out;
}

namespace model_detail {
inline LoadedEmbeddings load(const std::string& path, std::int32_t format) {
    cg_embeddings_file* f = nullptr;
    check_io(cg_model_load(path.c_str(), format, &f));
    struct Closer {
        cg_embeddings_file* f;
        ~Closer() { cg_model_file_close(f); }
    } closer{f};
    std::int32_t v = 0, d = 0;
    std::int64_t word_bytes = 0;
    check_io(cg_model_file_info(f, &v, &d, &word_bytes));
    std::string words(static_cast<std::size_t>(word_bytes), '\0');
    LoadedEmbeddings out;
    out.dim = d;
    out.vectors.resize(static_cast<std::size_t>(v) * static_cast<std::size_t>(d));
    check_io(cg_model_file_export(f, words.data(), out.vectors.data()));
    out.words.reserve(static_cast<std::size_t>(v));
    for (std::size_t p = 0; p < words.size();) {
        const std::size_t e = words.find('\0', p);
        out.words.emplace_back(words, p, e - p);
        p = e + 1;
    }
    return out;
}
}  // namespace model_detail

inline LoadedEmbeddings load_embeddings_binary(const std::string& path) {
    return model_detail::load(path, CG_FORMAT_BINARY);
}
inline LoadedEmbeddings load_embeddings_text(const std::string& path) { return model_detail::load(path, CG_FORMAT_TEXT); }
// Either format: a binary file is recognised by a non-printable byte after the header.
inline LoadedEmbeddings load_embeddings(const std::string& path) { return model_detail::load(path, CG_FORMAT_AUTO); }

}  // namespace cachegram
