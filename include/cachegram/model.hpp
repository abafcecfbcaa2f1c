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
#include <vector>

#include "cachegram/rng.hpp"

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

}  // namespace cachegram
