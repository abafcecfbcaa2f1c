// cachegram-b200: the training API of the drop-in, backed by libcachegram_b200.so.
//
// Same names and signatures as the reference trainer (trainer.hpp:25-316):
// TrainConfig, update_alpha, shrink_window, NodeCache, train_center, TrainStats and
//   Model train(corpus_path, vocab, tree, selection, config, stats = nullptr)
// with the same validation messages and exception types. Training runs on the GPU
// through the C-ABI (include/cachegram_b200.h); there is no CPU training path.
//
// Additions (defaulted, so existing callers compile unchanged):
//   TrainConfig::mode   TrainMode::Auto (default): workers == 1 runs the deterministic
//                       device mode, bit-identical to the reference's single-worker run
//                       (the reference is deterministic exactly then); workers > 1 runs
//                       the Hogwild throughput path on every SM (the reference is Hogwild
//                       then). TrainMode::Hogwild / ::Deterministic force one or the other.
//   ConstantSigmoid     a sigmoid functor the device evaluates itself (like SigmoidTable and
//                       ExactSigmoid); any other SigmoidFn is called back on the host per
//                       path step while the device does the arithmetic (cg_train_center_cb).
#pragma once

#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "cachegram/corpus.hpp"
#include "cachegram/errors.hpp"
#include "cachegram/huffman.hpp"
#include "cachegram/model.hpp"
#include "cachegram/rng.hpp"
#include "cachegram_b200.h"

namespace cachegram {

enum class TrainMode : std::int32_t { Hogwild = CG_MODE_HOGWILD, Deterministic = CG_MODE_DETERMINISTIC, Auto = -1 };

struct TrainConfig {
    std::int32_t dim = 100;
    std::int32_t window = 5;
    std::int64_t min_count = 5;
    double sample = 1e-3;
    float alpha0 = 0.025f;
    std::int32_t iterations = 5;
    std::int32_t workers = 1;
    std::int32_t cache_nodes = 31;
    std::int32_t flush_interval = 10;
    std::uint64_t seed = 1;
    TrainMode mode = TrainMode::Auto;
    // B200 additions: model replicas on GPUs 0..gpus-1 of this process; every sync_words
    // words per replica their deltas are summed over peer memory and applied with the
    // per-row sync scale (Hogwild mode, cg_session_sync_apply).
    std::int32_t gpus = 1;
    std::int64_t sync_words = 1000000;

    TrainMode resolved_mode() const {
        if (mode != TrainMode::Auto) return mode;
        return workers == 1 ? TrainMode::Deterministic : TrainMode::Hogwild;
    }

    void validate() const {
        auto need = [](bool ok, const char* msg) {
            if (!ok) throw std::invalid_argument(msg);
        };
        need(dim >= 1, "dim must be >= 1");
        need(window >= 1, "window must be >= 1");
        need(min_count >= 1, "min-count must be >= 1");
        need(sample >= 0.0, "sample must be >= 0");
        need(alpha0 > 0.0f, "alpha must be > 0");
        need(iterations >= 1, "iterations must be >= 1");
        need(workers >= 1, "workers must be >= 1");
        need(cache_nodes >= 0, "cache-nodes must be >= 0");
        need(flush_interval >= 1, "flush-interval must be >= 1");
        need(gpus >= 1 && gpus <= 8, "gpus must be in [1, 8]");
        need(sync_words >= 1, "sync-words must be >= 1");
    }
};

// Linear decay with floor alpha0 * 1e-4 (trainer.hpp:58-63).
inline float update_alpha(std::uint64_t words_processed, std::uint64_t total_words, float alpha0) {
    const double done = static_cast<double>(words_processed) / (static_cast<double>(total_words) + 1.0);
    const float a = alpha0 * static_cast<float>(1.0 - done);
    const float lo = alpha0 * 1e-4f;
    return a > lo ? a : lo;
}
inline float update_alpha_host(std::uint64_t w, std::uint64_t t, float a0) { return update_alpha(w, t, a0); }

// Half-window uniform in [1, window] (trainer.hpp:66-68).
inline std::int32_t shrink_window(std::int32_t window, Rng& rng) {
    return window - static_cast<std::int32_t>(rng.next_below(static_cast<std::uint32_t>(window)));
}

// Shared progress of the training run (trainer.hpp:52-55): atomic, as the reference's.
struct ProgressCounter {
    std::atomic<std::uint64_t> words_processed{0};
    std::uint64_t total_words = 0;
};

struct TrainStats {
    std::uint64_t words_processed = 0;
    double wall_seconds = 0.0;
    double words_per_second = 0.0;
};

// A sigmoid the device can evaluate: f(x) = value for every x.
struct ConstantSigmoid {
    float value = 0.5f;
    float operator()(float) const { return value; }
};

namespace trainer_detail {
[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = cg_last_error();
    switch (rc) {
        case CG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case CG_ERR_IO: throw IoError(msg);
        case CG_ERR_PARSE: throw ParseError(msg);
        case CG_ERR_NO_TRAINABLE_WORDS: throw NoTrainableWords();
        default: throw std::runtime_error(msg);
    }
}
inline void check(int rc) {
    if (rc != CG_OK) rethrow(rc);
}

// Flat CSR copies of a tree for the C-ABI.
struct TreeArrays {
    std::vector<std::int64_t> off;
    std::vector<std::int32_t> node;
    std::vector<std::uint8_t> turn;
    explicit TreeArrays(const HuffmanTree& t) {
        off.assign(t.offsets().begin(), t.offsets().end());
        node.reserve(t.steps().size());
        turn.reserve(t.steps().size());
        for (const PathStep& s : t.steps()) {
            node.push_back(s.node);
            turn.push_back(s.turn);
        }
    }
};

// The CSR arrays and slot map of the last (tree, selection) pair train_center was called
// with, per thread: rebuilding them (O(V)) on every call made the kernel-level entry
// unusable beyond tests. Trees and selections are immutable once built; the key holds
// their addresses and sizes.
struct CenterArrays {
    const HuffmanTree* tree = nullptr;
    const CacheSelection* selection = nullptr;
    std::size_t steps = 0;
    std::int32_t leaves = 0, slots = 0;
    std::unique_ptr<TreeArrays> ta;
    std::vector<std::int32_t> slot_of;
};
inline const CenterArrays& center_arrays(const HuffmanTree& tree, const CacheSelection& selection) {
    thread_local CenterArrays c;
    if (c.tree != &tree || c.selection != &selection || c.steps != tree.steps().size() ||
        c.leaves != tree.leaf_count() || c.slots != selection.size()) {
        c.ta = std::make_unique<TreeArrays>(tree);
        c.slot_of.resize(static_cast<std::size_t>(selection.inner_node_count()));
        for (std::int32_t n = 0; n < selection.inner_node_count(); ++n) c.slot_of[static_cast<std::size_t>(n)] = selection.slot_of(n);
        c.tree = &tree;
        c.selection = &selection;
        c.steps = tree.steps().size();
        c.leaves = tree.leaf_count();
        c.slots = selection.size();
    }
    return c;
}

template <typename S>
constexpr bool kDeviceSigmoid = std::is_same_v<S, SigmoidTable> || std::is_same_v<S, ExactSigmoid> ||
                                std::is_same_v<S, ConstantSigmoid>;
}  // namespace trainer_detail

// Working copies of the hot node rows (trainer.hpp:75-138). The state lives on the
// host so tests can inspect it; the arithmetic of train_center and flush runs on the
// device (cg_train_center / cg_cache_flush).
class NodeCache {
public:
    NodeCache(const CacheSelection& selection, std::int32_t dim, std::int32_t flush_interval)
        : sel_(&selection),
          dim_(dim),
          interval_(flush_interval),
          work_(static_cast<std::size_t>(selection.size()) * static_cast<std::size_t>(dim)),
          snap_(work_.size()),
          flag_(static_cast<std::size_t>(selection.size()), 0) {}

    bool is_cached(std::int32_t slot) const { return flag_[static_cast<std::size_t>(slot)] != 0; }
    std::int32_t words_since_flush() const { return since_; }
    float* row(std::int32_t slot) { return work_.data() + offset(slot); }
    const float* original(std::int32_t slot) const { return snap_.data() + offset(slot); }

    // First touch copies the shared row into the working row and the snapshot.
    float* acquire(std::int32_t slot, const float* shared_row) {
        if (!is_cached(slot)) {
            std::memcpy(row(slot), shared_row, static_cast<std::size_t>(dim_) * sizeof(float));
            std::memcpy(snap_.data() + offset(slot), shared_row, static_cast<std::size_t>(dim_) * sizeof(float));
            flag_[static_cast<std::size_t>(slot)] = 1;
        }
        return row(slot);
    }

    // shared += work - snap for every acquired row, on the device.
    void flush(Model& model) {
        std::vector<std::int32_t> hot(sel_->hot_nodes().begin(), sel_->hot_nodes().end());
        if (!hot.empty())
            trainer_detail::check(cg_cache_flush(model.vocab_size(), dim_, model.weight_matrix().data(), hot.data(),
                                                 sel_->size(), work_.data(), snap_.data(), flag_.data()));
        since_ = 0;
    }

    bool note_center_trained() { return ++since_ >= interval_; }

    // C-ABI views
    float* work_data() { return work_.data(); }
    float* snap_data() { return snap_.data(); }
    std::uint8_t* flag_data() { return flag_.data(); }

private:
    std::size_t offset(std::int32_t slot) const { return static_cast<std::size_t>(slot) * static_cast<std::size_t>(dim_); }
    const CacheSelection* sel_;
    std::int32_t dim_, interval_;
    std::vector<float> work_, snap_;
    std::vector<std::uint8_t> flag_;
    std::int32_t since_ = 0;
};

// One skip-gram/HS update for a center word (trainer.hpp:147-175) on the device.
// SigmoidTable, ExactSigmoid and ConstantSigmoid are evaluated on the device; any other
// functor (e.g. a test's counting lambda) is called on the host once per path step, in
// path order, while the device computes the dot products and applies the updates.
// `hidden` is unused: the device keeps the hidden accumulator in shared memory.
template <typename SigmoidFn>
inline void train_center(std::int32_t center, std::span<const std::int32_t> sentence, std::size_t center_pos,
                         std::int32_t half_window, Model& model, const HuffmanTree& tree,
                         const CacheSelection& selection, NodeCache& cache, float alpha, float* hidden,
                         const SigmoidFn& sigmoid, std::int64_t* sigmoid_calls = nullptr) {
    (void)hidden;
    const trainer_detail::CenterArrays& arrays = trainer_detail::center_arrays(tree, selection);
    const trainer_detail::TreeArrays& ta = *arrays.ta;
    const std::vector<std::int32_t>& slot_of = arrays.slot_of;
    if constexpr (trainer_detail::kDeviceSigmoid<SigmoidFn>) {
        std::int32_t mode = 0;
        float konst = 0.0f;
        if constexpr (std::is_same_v<SigmoidFn, ExactSigmoid>) mode = 1;
        if constexpr (std::is_same_v<SigmoidFn, ConstantSigmoid>) {
            mode = 2;
            konst = sigmoid.value;
        }
        trainer_detail::check(cg_train_center(
            center, sentence.data(), static_cast<std::int64_t>(sentence.size()), static_cast<std::int64_t>(center_pos),
            half_window, model.vocab_size(), model.dim(), model.input_matrix().data(), model.weight_matrix().data(),
            ta.off.data(), ta.node.data(), ta.turn.data(), slot_of.data(), selection.size(), cache.work_data(),
            cache.snap_data(), cache.flag_data(), alpha, mode, konst, sigmoid_calls));
    } else {
        auto trampoline = [](float x, void* ctx) -> float { return (*static_cast<const SigmoidFn*>(ctx))(x); };
        trainer_detail::check(cg_train_center_cb(
            center, sentence.data(), static_cast<std::int64_t>(sentence.size()), static_cast<std::int64_t>(center_pos),
            half_window, model.vocab_size(), model.dim(), model.input_matrix().data(), model.weight_matrix().data(),
            ta.off.data(), ta.node.data(), ta.turn.data(), slot_of.data(), selection.size(), cache.work_data(),
            cache.snap_data(), cache.flag_data(), alpha, trampoline,
            const_cast<void*>(static_cast<const void*>(&sigmoid)), sigmoid_calls));
    }
}

// cachegram::train (trainer.hpp:254-316) on the GPU.
inline Model train(const std::string& corpus_path, const Vocabulary& vocab, const HuffmanTree& tree,
                   const CacheSelection& selection, const TrainConfig& config, TrainStats* stats = nullptr) {
    config.validate();
    if (vocab.size() != tree.leaf_count()) throw std::invalid_argument("vocabulary and tree sizes disagree");
    if (selection.inner_node_count() != tree.inner_count())
        throw std::invalid_argument("cache selection was built from a different tree");
    const TrainMode mode = config.resolved_mode();
    if (mode == TrainMode::Deterministic && config.workers != 1)
        throw std::invalid_argument("deterministic mode replays the single-worker stream: set workers = 1");

    // The corpus is tokenised on the GPU (cg_train_file): IoError if it cannot be opened.
    std::string words;
    for (std::int32_t w = 0; w < vocab.size(); ++w) {
        words += vocab.word(w);
        words.push_back('\0');
    }
    const trainer_detail::TreeArrays ta(tree);
    std::vector<std::int64_t> counts(static_cast<std::size_t>(vocab.size()));
    for (std::int32_t w = 0; w < vocab.size(); ++w) counts[static_cast<std::size_t>(w)] = vocab.count(w);
    std::vector<std::int32_t> hot(selection.hot_nodes().begin(), selection.hot_nodes().end());

    cg_config c{config.dim,        config.window,  config.min_count,   config.sample,
                config.alpha0,     config.iterations, config.workers, config.cache_nodes,
                config.flush_interval, config.seed};
    cg_model_desc m{};
    m.vocab_size = vocab.size();
    m.counts = counts.data();
    m.total_tokens = vocab.total_tokens();
    m.path_offsets = ta.off.data();
    m.path_nodes = ta.node.data();
    m.path_turns = ta.turn.data();
    m.node_usage = tree.usage().data();
    m.hot_nodes = hot.empty() ? nullptr : hot.data();
    m.hot_count = selection.size();

    Model model(vocab.size(), config.dim);
    cg_train_stats st{};
    // Errors: configuration and consistency problems (std::invalid_argument) and a corpus
    // that cannot be opened (IoError) are raised before training starts, as the
    // reference raises them before its worker threads (trainer.hpp:256-276). Anything
    // that fails during training is a worker failure: with workers > 1 the reference
    // wraps it as runtime_error("worker i failed: ...") (trainer.hpp:297-305); the GPU run
    // is one device-wide worker, reported as worker 0.
    auto check_run = [&](int rc) {
        if (rc == CG_OK) return;
        if (config.workers > 1 && rc != CG_ERR_INVALID_ARGUMENT && rc != CG_ERR_IO) {
            const std::string msg = rc == CG_ERR_NO_TRAINABLE_WORDS ? std::string(NoTrainableWords().what())
                                                                    : std::string(cg_last_error());
            throw std::runtime_error("worker 0 failed: " + msg);
        }
        trainer_detail::rethrow(rc);
    };
    if (config.gpus > 1) {
        if (mode != TrainMode::Hogwild) throw std::invalid_argument("gpus > 1 trains replicas in Hogwild mode");
        std::vector<std::int32_t> devices(static_cast<std::size_t>(config.gpus));
        for (std::int32_t g = 0; g < config.gpus; ++g) devices[static_cast<std::size_t>(g)] = g;
        check_run(cg_train_file_replicas(&c, static_cast<std::int32_t>(mode), &m, corpus_path.c_str(), words.data(),
                                         devices.data(), config.gpus, config.sync_words, model.input_matrix().data(),
                                         model.weight_matrix().data(), &st));
    } else {
        check_run(cg_train_file(&c, static_cast<std::int32_t>(mode), &m, corpus_path.c_str(), words.data(),
                                model.input_matrix().data(), model.weight_matrix().data(), &st));
    }
    if (stats) {
        stats->words_processed = st.words_processed;
        stats->wall_seconds = st.wall_seconds;
        stats->words_per_second = st.words_per_second;
    }
    return model;
}

}  // namespace cachegram
