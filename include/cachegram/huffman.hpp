// cachegram-b200: Huffman tree, root-first paths and the hot-node selection.
//
// Public API and the exact tree shape of the reference (huffman.hpp:21-159):
// repeatedly merge the two lowest (count, node id) items, first pop gets turn 0,
// inner nodes numbered 0..V-2 in merge order (root = V-2), paths stored root-first.
// Built here with the linear two-queue method: leaves sorted by (count, id) in one
// queue, merged nodes appended to a second queue in creation order. Both queues stay
// sorted by (count, id), so taking the smaller front reproduces the heap's pop order
// exactly (ties go to the lower id, i.e. to the leaf queue).
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <span>
#include <stdexcept>
#include <vector>

#include "cachegram/corpus.hpp"

namespace cachegram {

struct PathStep {
    std::int32_t node;   // inner node id
    std::uint8_t turn;   // 0 = first-merged child, 1 = second
};

class HuffmanTree {
public:
    std::int32_t inner_count() const { return inner_; }
    std::int32_t leaf_count() const { return static_cast<std::int32_t>(offsets_.size()) - 1; }
    std::int32_t root_id() const { return inner_ - 1; }

    std::span<const PathStep> path(std::int32_t word) const {
        const std::size_t b = offsets_[static_cast<std::size_t>(word)];
        const std::size_t e = offsets_[static_cast<std::size_t>(word) + 1];
        return {steps_.data() + b, e - b};
    }
    std::int64_t node_usage(std::int32_t node) const { return usage_[static_cast<std::size_t>(node)]; }
    const std::vector<std::int64_t>& usage() const { return usage_; }

    // CSR view used by the C-ABI (offsets has V+1 entries).
    const std::vector<PathStep>& steps() const { return steps_; }
    const std::vector<std::size_t>& offsets() const { return offsets_; }

    friend HuffmanTree build_huffman_tree(const Vocabulary& vocab);
    friend HuffmanTree huffman_from_counts(const std::int64_t* counts, std::int32_t v);

private:
    std::int32_t inner_ = 0;
    std::vector<std::int64_t> usage_;
    std::vector<PathStep> steps_;
    std::vector<std::size_t> offsets_;
};

inline HuffmanTree huffman_from_counts(const std::int64_t* counts, std::int32_t v) {
    if (v <= 0) throw NoTrainableWords();
    if (v == 1)
        throw std::invalid_argument("hierarchical softmax needs at least two words, got a single-word vocabulary");
    const std::size_t nv = static_cast<std::size_t>(v);
    const std::size_t nall = 2 * nv - 1;
    std::vector<std::int64_t> weight(nall);
    std::vector<std::int32_t> up(nall, -1);
    std::vector<std::uint8_t> side(nall, 0);

    std::vector<std::int32_t> leaves(nv);
    std::iota(leaves.begin(), leaves.end(), 0);
    std::stable_sort(leaves.begin(), leaves.end(),
                     [counts](std::int32_t a, std::int32_t b) { return counts[a] < counts[b]; });
    for (std::size_t i = 0; i < nv; ++i) weight[i] = counts[i];

    std::size_t lq = 0;                // next leaf in `leaves`
    std::size_t iq = nv, made = nv;    // inner queue = node ids [iq, made)
    auto take = [&]() -> std::int32_t {
        const bool leaf_ok = lq < nv;
        const bool inner_ok = iq < made;
        if (leaf_ok && (!inner_ok || weight[static_cast<std::size_t>(leaves[lq])] <= weight[iq])) return leaves[lq++];
        return static_cast<std::int32_t>(iq++);
    };
    for (; made < nall; ++made) {
        const std::int32_t a = take();
        const std::int32_t b = take();
        weight[made] = weight[static_cast<std::size_t>(a)] + weight[static_cast<std::size_t>(b)];
        up[static_cast<std::size_t>(a)] = static_cast<std::int32_t>(made);
        up[static_cast<std::size_t>(b)] = static_cast<std::int32_t>(made);
        side[static_cast<std::size_t>(b)] = 1;
    }

    HuffmanTree t;
    t.inner_ = v - 1;
    t.usage_.assign(weight.begin() + v, weight.end());
    // depth of every node, top-down (parents have larger ids than children)
    std::vector<std::int32_t> depth(nall, 0);
    for (std::size_t n = nall - 1; n-- > 0;) depth[n] = depth[static_cast<std::size_t>(up[n])] + 1;
    t.offsets_.resize(nv + 1);
    std::size_t total = 0;
    for (std::size_t w = 0; w < nv; ++w) {
        t.offsets_[w] = total;
        total += static_cast<std::size_t>(depth[w]);
    }
    t.offsets_[nv] = total;
    t.steps_.resize(total);
    for (std::size_t w = 0; w < nv; ++w) {
        std::size_t k = t.offsets_[w + 1];
        for (std::int32_t x = static_cast<std::int32_t>(w); up[static_cast<std::size_t>(x)] >= 0;
             x = up[static_cast<std::size_t>(x)])
            t.steps_[--k] = {up[static_cast<std::size_t>(x)] - v, side[static_cast<std::size_t>(x)]};
    }
    return t;
}

inline HuffmanTree build_huffman_tree(const Vocabulary& vocab) {
    std::vector<std::int64_t> c(static_cast<std::size_t>(vocab.size()));
    for (std::int32_t w = 0; w < vocab.size(); ++w) c[static_cast<std::size_t>(w)] = vocab.count(w);
    return huffman_from_counts(c.data(), vocab.size());
}

inline const std::vector<std::int64_t>& node_usage_frequency(const HuffmanTree& tree) { return tree.usage(); }

// The min(K, V-1) inner nodes with the highest usage (ties to the lower id); slot 0 is
// the hottest. Usage strictly decreases along every root-to-leaf path, so the selection
// is always a root-containing subtree and hot steps form a prefix of every path.
class CacheSelection {
public:
    CacheSelection() = default;
    std::int32_t size() const { return static_cast<std::int32_t>(hot_.size()); }
    std::span<const std::int32_t> hot_nodes() const { return hot_; }
    std::int32_t node_at(std::int32_t slot) const { return hot_[static_cast<std::size_t>(slot)]; }
    std::int32_t inner_node_count() const { return static_cast<std::int32_t>(slot_.size()); }
    std::int32_t slot_of(std::int32_t node) const { return slot_[static_cast<std::size_t>(node)]; }

    friend CacheSelection select_cached_nodes(const HuffmanTree& tree, std::int32_t k);

private:
    std::vector<std::int32_t> hot_;
    std::vector<std::int32_t> slot_;
};

// Full (usage desc, id asc) ranking of the inner nodes; the device path stores syn1
// rows in this order so that "hot" is simply row < K.
inline std::vector<std::int32_t> usage_rank_order(const HuffmanTree& tree) {
    std::vector<std::int32_t> order(static_cast<std::size_t>(tree.inner_count()));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&tree](std::int32_t a, std::int32_t b) { return tree.node_usage(a) > tree.node_usage(b); });
    return order;
}

inline CacheSelection select_cached_nodes(const HuffmanTree& tree, std::int32_t k) {
    if (k < 0) throw std::invalid_argument("cache node count must be >= 0");
    const std::vector<std::int32_t> order = usage_rank_order(tree);
    const std::size_t take = std::min(static_cast<std::size_t>(k), order.size());
    CacheSelection s;
    s.hot_.assign(order.begin(), order.begin() + static_cast<std::ptrdiff_t>(take));
    s.slot_.assign(order.size(), -1);
    for (std::size_t i = 0; i < take; ++i) s.slot_[static_cast<std::size_t>(s.hot_[i])] = static_cast<std::int32_t>(i);
    return s;
}

}  // namespace cachegram
