// C++ drop-in check: a program written against include/cachegram/*.hpp exactly the way
// callers of the reference's headers are written (names and signatures of
// /root/reference/proj/include/cachegram), linked with libcachegram_b200.so instead of
// compiling the CPU trainer. Mirrors the reference's trainer_test.cpp / acceptance.cpp
// properties with plain checks (GTest is not available here).
//
//   dropin_test [dump_dir]   exit code = number of failed checks; with dump_dir, the
//                            deterministic-mode model of the golden case g1 is written
//                            there for tests/test_cpp_dropin.py to compare.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <string>
#include <vector>

#include "cachegram/corpus.hpp"
#include "cachegram/huffman.hpp"
#include "cachegram/model.hpp"
#include "cachegram/rng.hpp"
#include "cachegram/trainer.hpp"

using namespace cachegram;

namespace {

int g_fail = 0;
void check(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++g_fail;
}

// The reference test utility's corpus generator, restated (testutil.hpp:78-101).
std::string zipf_corpus(std::size_t min_bytes, int types, std::uint64_t seed) {
    std::vector<double> cum(static_cast<std::size_t>(types));
    double total = 0;
    for (int i = 0; i < types; ++i) cum[static_cast<std::size_t>(i)] = (total += 1.0 / (i + 3));
    for (double& c : cum) c /= total;
    Rng rng(seed);
    std::string out;
    while (out.size() < min_bytes) {
        const double u = static_cast<double>(rng.next_float());
        int w = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), u) - cum.begin());
        if (w >= types) w = types - 1;
        out += "w" + std::to_string(w) + " ";
    }
    if (!out.empty()) out.pop_back();
    return out;
}

std::string write_tmp(const std::string& name, const std::string& text) {
    const std::string path = "/tmp/cg_dropin_" + name;
    std::ofstream(path, std::ios::binary) << text;
    return path;
}

bool same_bits(const Model& a, const Model& b) {
    return std::memcmp(a.input_matrix().data(), b.input_matrix().data(), a.input_matrix().size() * 4) == 0 &&
           std::memcmp(a.weight_matrix().data(), b.weight_matrix().data(), a.weight_matrix().size() * 4) == 0;
}

double max_rel(const Model& a, const Model& b) {
    double worst = 0;
    auto scan = [&](std::span<const float> x, std::span<const float> y) {
        for (std::size_t i = 0; i < x.size(); ++i) {
            const double den = std::max({std::fabs(double(x[i])), std::fabs(double(y[i])), 1e-2});
            worst = std::max(worst, std::fabs(double(x[i]) - double(y[i])) / den);
        }
    };
    scan(a.input_matrix(), b.input_matrix());
    scan(a.weight_matrix(), b.weight_matrix());
    return worst;
}

TrainConfig small_config() {
    TrainConfig c;
    c.dim = 16;
    c.window = 3;
    c.min_count = 2;
    c.sample = 1e-3;
    c.iterations = 2;
    c.workers = 1;
    c.cache_nodes = 0;
    c.flush_interval = 10;
    c.seed = 7;
    c.mode = TrainMode::Deterministic;
    return c;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string dump_dir = argc > 1 ? argv[1] : "";

    // defaults unchanged (trainer_test.cpp ReferenceDefaults)
    {
        const TrainConfig c;
        check(c.dim == 100 && c.window == 5 && c.min_count == 5 && c.sample == 1e-3 && c.alpha0 == 0.025f &&
                  c.cache_nodes == 31 && c.flush_interval == 10,
              "TrainConfig defaults match the reference");
    }

    // known-answer train_center on the device (trainer_test.cpp GradientScalesWithAlpha...)
    {
        Vocabulary vocab({{"w0", 2}, {"w1", 1}}, 3);
        HuffmanTree tree = build_huffman_tree(vocab);
        Model model(2, 2);
        const std::int32_t center = tree.path(0)[0].turn == 0 ? 0 : 1;
        const std::int32_t context = 1 - center;
        model.input_vector(context)[0] = 0.4f;
        model.input_vector(context)[1] = 0.2f;
        CacheSelection sel = select_cached_nodes(tree, 0);
        NodeCache cache(sel, 2, 10);
        std::vector<float> hidden(2);
        const std::vector<std::int32_t> sentence{context, center};
        std::int64_t calls = 0;
        train_center(center, std::span<const std::int32_t>(sentence), 1, 1, model, tree, sel, cache, 0.025f,
                     hidden.data(), ExactSigmoid{}, &calls);
        check(calls == 1 && std::fabs(model.node_weight(0)[0] - 0.0125f * 0.4f) < 1e-8f &&
                  model.input_vector(context)[0] == 0.4f,
              "train_center: neutral sigmoid gives g = 0.0125 (device kernel)");
    }

    // hot rows bypass the shared row until flush (trainer_test.cpp HotRowsBypass...)
    {
        Vocabulary vocab({{"a", 4}, {"b", 3}, {"c", 2}, {"d", 1}}, 10);
        HuffmanTree tree = build_huffman_tree(vocab);
        Model model = init_model(4, 4, 2);
        CacheSelection sel = select_cached_nodes(tree, 1);
        NodeCache cache(sel, 4, 1000);
        std::vector<float> hidden(4);
        const std::vector<std::int32_t> sentence{0, 3};
        train_center(3, std::span<const std::int32_t>(sentence), 1, 1, model, tree, sel, cache, 0.05f, hidden.data(),
                     ExactSigmoid{});
        const float* root = model.node_weight(tree.root_id());
        bool untouched = true;
        for (int d = 0; d < 4; ++d) untouched &= root[d] == 0.0f;
        cache.flush(model);
        bool moved = false;
        for (int d = 0; d < 4; ++d) moved |= root[d] != 0.0f;
        check(untouched && moved && !cache.is_cached(0), "NodeCache: root untouched until flush, moved after");
    }

    // deterministic train(): reproducible, seed-sensitive, cache-transparent (trainer_test.cpp 362-433)
    const std::string path = write_tmp("c30k.txt", zipf_corpus(30000, 120, 21));
    {
        Vocabulary vocab = build_vocabulary_file(path, 2);
        HuffmanTree tree = build_huffman_tree(vocab);
        for (std::int32_t k : {0, 15}) {
            TrainConfig c = small_config();
            c.cache_nodes = k;
            CacheSelection sel = select_cached_nodes(tree, k);
            Model a = train(path, vocab, tree, sel, c);
            Model b = train(path, vocab, tree, sel, c);
            check(same_bits(a, b), "deterministic train() bit-reproducible, K=" + std::to_string(k));
            if (k == 15 && !dump_dir.empty()) {
                std::ofstream(dump_dir + "/g1_syn0.bin", std::ios::binary)
                    .write(reinterpret_cast<const char*>(a.input_matrix().data()),
                           static_cast<std::streamsize>(a.input_matrix().size() * 4));
                std::ofstream(dump_dir + "/g1_syn1.bin", std::ios::binary)
                    .write(reinterpret_cast<const char*>(a.weight_matrix().data()),
                           static_cast<std::streamsize>(a.weight_matrix().size() * 4));
            }
        }
        TrainConfig c = small_config();
        Model a = train(path, vocab, tree, select_cached_nodes(tree, 0), c);
        c.seed = 8;
        Model b = train(path, vocab, tree, select_cached_nodes(tree, 0), c);
        check(std::memcmp(a.input_matrix().data(), b.input_matrix().data(), a.input_matrix().size() * 4) != 0,
              "seed changes the model");
        TrainConfig cc = small_config();
        cc.cache_nodes = 8;
        cc.flush_interval = 4;
        Model cached = train(path, vocab, tree, select_cached_nodes(tree, 8), cc);
        check(max_rel(a, cached) < 1e-4, "single-worker cache transparency < 1e-4");
    }

    // Hogwild (default mode): every in-vocabulary token counted, finite model
    {
        Vocabulary vocab = build_vocabulary_file(path, 2);
        HuffmanTree tree = build_huffman_tree(vocab);
        TrainConfig c = small_config();
        c.mode = TrainMode::Hogwild;
        c.cache_nodes = 4;
        c.iterations = 3;
        c.workers = 3;
        TrainStats stats;
        Model m = train(path, vocab, tree, select_cached_nodes(tree, 4), c, &stats);
        bool finite = true;
        for (float x : m.input_matrix()) finite &= std::isfinite(x);
        for (float x : m.weight_matrix()) finite &= std::isfinite(x);
        check(stats.words_processed == 3ull * static_cast<std::uint64_t>(vocab.total_tokens()) && finite,
              "hogwild train(): progress counts every occurrence, model finite");
    }

    // co-occurring words end up similar (trainer_test.cpp 457-517), Hogwild on the GPU
    {
        std::string corpus;
        Rng topic(99);
        for (int i = 0; i < 30000; ++i) {
            const std::uint32_t t = topic.next_below(30);
            corpus += "x" + std::to_string(t) + " y" + std::to_string(t) + " ";
        }
        const std::string p2 = write_tmp("pairs.txt", corpus);
        TrainConfig c;
        c.dim = 24;
        c.window = 2;
        c.min_count = 5;
        c.sample = 0.0;
        c.iterations = 3;
        c.cache_nodes = 8;
        c.seed = 4;
        const Vocabulary vocab = build_vocabulary_file(p2, c.min_count);
        const HuffmanTree tree = build_huffman_tree(vocab);
        const Model m = train(p2, vocab, tree, select_cached_nodes(tree, c.cache_nodes), c);
        auto cosine = [&](std::int32_t a, std::int32_t b) {
            const float* va = m.input_vector(a);
            const float* vb = m.input_vector(b);
            double ab = 0, aa = 0, bb = 0;
            for (int d = 0; d < m.dim(); ++d) {
                ab += double(va[d]) * vb[d];
                aa += double(va[d]) * va[d];
                bb += double(vb[d]) * vb[d];
            }
            return ab / std::sqrt(aa * bb);
        };
        double partner = 0, stranger = 0;
        for (int t = 0; t < 30; ++t) {
            partner += cosine(vocab.id_of("x" + std::to_string(t)), vocab.id_of("y" + std::to_string(t)));
            stranger += cosine(vocab.id_of("x" + std::to_string(t)), vocab.id_of("y" + std::to_string((t + 7) % 30)));
        }
        check(vocab.size() == 60 && partner / 30 > stranger / 30 + 0.2, "co-occurring words end up similar (hogwild)");
    }

    // invalid configurations and unreadable corpora raise the reference's exceptions
    {
        const std::string p3 = write_tmp("ab.txt", "a b a b a b a b");
        Vocabulary vocab = build_vocabulary_file(p3, 1);
        HuffmanTree tree = build_huffman_tree(vocab);
        CacheSelection sel = select_cached_nodes(tree, 0);
        auto throws = [&](const std::function<void()>& f, auto tag) {
            try {
                f();
            } catch (const decltype(tag)&) {
                return true;
            } catch (...) {
                return false;
            }
            return false;
        };
        TrainConfig c = small_config();
        c.min_count = 1;
        c.workers = 0;
        check(throws([&] { train(p3, vocab, tree, sel, c); }, std::invalid_argument("")), "workers = 0 rejected");
        c = small_config();
        c.flush_interval = 0;
        check(throws([&] { train(p3, vocab, tree, sel, c); }, std::invalid_argument("")), "flush_interval = 0 rejected");
        c = small_config();
        check(throws([&] { train("/tmp/cg_dropin_missing.txt", vocab, tree, sel, c); }, IoError("")),
              "missing corpus raises IoError");
    }

    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
