// cachegram-b200: corpus ingest for the drop-in API.
//
// Public names, signatures and semantics follow the reference corpus layer
// (corpus.hpp:19-283): whitespace tokenisation, count-ordered vocabulary with
// first-occurrence tie-breaks, the subsampling keep probability, separator-aligned
// byte shards and a resettable shard reader. The implementation is this repo's own.
// New here: read_id_stream(), which turns a corpus file into the int32 id stream
// that the device path consumes (the reference re-tokenises inside every worker
// pass, trainer.hpp:220-222; the GPU path tokenises once on the host).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "cachegram/errors.hpp"

namespace cachegram {

// ' ', \t, \n, \v, \f, \r (corpus.hpp:19-21).
inline bool is_token_separator(char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

inline std::vector<std::string_view> tokenize(std::string_view text) {
    std::vector<std::string_view> out;
    const char* p = text.data();
    const char* end = p + text.size();
    while (p < end) {
        while (p < end && is_token_separator(*p)) ++p;
        const char* b = p;
        while (p < end && !is_token_separator(*p)) ++p;
        if (p > b) out.emplace_back(b, static_cast<std::size_t>(p - b));
    }
    return out;
}

struct VocabEntry {
    std::string word;
    std::int64_t count = 0;
};

namespace corpus_detail {
struct SvHash {
    using is_transparent = void;
    std::size_t operator()(std::string_view s) const noexcept { return std::hash<std::string_view>{}(s); }
};
using WordIndex = std::unordered_map<std::string, std::int32_t, SvHash, std::equal_to<>>;

// Streams a byte range of a file through fixed-size buffers, calling fn(token)
// for every whitespace-delimited token that starts inside [begin, end).
template <typename Fn>
void for_each_token(std::FILE* f, std::uint64_t begin, std::uint64_t end, Fn&& fn) {
    std::vector<char> buf(1 << 18);
    std::string carry;
    std::uint64_t pos = begin;
    if (std::fseek(f, static_cast<long>(begin), SEEK_SET) != 0) return;
    bool in_token = false;
    while (true) {
        const std::size_t got = std::fread(buf.data(), 1, buf.size(), f);
        if (got == 0) break;
        std::size_t i = 0;
        while (i < got) {
            if (!in_token) {
                if (pos + i >= end) {  // no token may start at or past the shard end
                    if (!carry.empty()) fn(std::string_view(carry));
                    return;
                }
                if (is_token_separator(buf[i])) { ++i; continue; }
                in_token = true;
            }
            std::size_t j = i;
            while (j < got && !is_token_separator(buf[j])) ++j;
            carry.append(buf.data() + i, j - i);
            if (j < got) {  // token closed inside this buffer
                fn(std::string_view(carry));
                carry.clear();
                in_token = false;
            }
            i = j;
        }
        pos += got;
    }
    if (!carry.empty()) fn(std::string_view(carry));
}

struct FileCloser {
    void operator()(std::FILE* f) const { if (f) std::fclose(f); }
};
using FilePtr = std::unique_ptr<std::FILE, FileCloser>;

inline FilePtr open_or_throw(const std::string& path) {
    FilePtr f(std::fopen(path.c_str(), "rb"));
    if (!f) throw IoError("cannot open corpus file: " + path);
    return f;
}

inline std::uint64_t file_size(std::FILE* f) {
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    return n < 0 ? 0 : static_cast<std::uint64_t>(n);
}
}  // namespace corpus_detail

// Ids 0..V-1 in non-increasing count order; equal counts keep first-occurrence order.
class Vocabulary {
public:
    static constexpr std::int32_t kNotFound = -1;

    Vocabulary() = default;
    Vocabulary(std::vector<VocabEntry> entries, std::int64_t total) : entries_(std::move(entries)), total_(total) {
        index_.reserve(entries_.size() * 2);
        std::int32_t id = 0;
        for (const VocabEntry& e : entries_) index_.emplace(e.word, id++);
    }

    std::int32_t size() const { return static_cast<std::int32_t>(entries_.size()); }
    std::int64_t total_tokens() const { return total_; }
    const VocabEntry& entry(std::int32_t id) const { return entries_[static_cast<std::size_t>(id)]; }
    const std::string& word(std::int32_t id) const { return entry(id).word; }
    std::int64_t count(std::int32_t id) const { return entry(id).count; }
    std::int32_t id_of(std::string_view w) const {
        const auto hit = index_.find(w);
        return hit != index_.end() ? hit->second : kNotFound;
    }

private:
    std::vector<VocabEntry> entries_;
    corpus_detail::WordIndex index_;
    std::int64_t total_ = 0;
};

class VocabBuilder {
public:
    void add(std::string_view token) {
        const auto hit = slot_.find(token);
        if (hit != slot_.end()) {
            ++counts_[static_cast<std::size_t>(hit->second)];
            return;
        }
        slot_.emplace(std::string(token), static_cast<std::int32_t>(words_.size()));
        words_.emplace_back(token);
        counts_.push_back(1);
    }

    // Survivors (count >= min_count) by descending count; first-seen order on ties.
    Vocabulary finish(std::int64_t min_count) const {
        std::vector<std::int32_t> keep;
        for (std::size_t i = 0; i < counts_.size(); ++i)
            if (counts_[i] >= min_count) keep.push_back(static_cast<std::int32_t>(i));
        if (keep.empty()) throw NoTrainableWords();
        // first-seen order is the insertion order, so a stable sort on count suffices
        std::stable_sort(keep.begin(), keep.end(), [this](std::int32_t a, std::int32_t b) {
            return counts_[static_cast<std::size_t>(a)] > counts_[static_cast<std::size_t>(b)];
        });
        std::vector<VocabEntry> entries(keep.size());
        std::int64_t total = 0;
        for (std::size_t r = 0; r < keep.size(); ++r) {
            const auto i = static_cast<std::size_t>(keep[r]);
            entries[r].word = words_[i];
            entries[r].count = counts_[i];
            total += counts_[i];
        }
        return Vocabulary(std::move(entries), total);
    }

private:
    corpus_detail::WordIndex slot_;
    std::vector<std::string> words_;
    std::vector<std::int64_t> counts_;
};

template <typename Range>
Vocabulary build_vocabulary(const Range& tokens, std::int64_t min_count) {
    VocabBuilder b;
    for (const auto& t : tokens) b.add(std::string_view(t));
    return b.finish(min_count);
}

inline Vocabulary build_vocabulary_file(const std::string& path, std::int64_t min_count) {
    auto f = corpus_detail::open_or_throw(path);
    VocabBuilder b;
    corpus_detail::for_each_token(f.get(), 0, UINT64_MAX, [&b](std::string_view t) { b.add(t); });
    return b.finish(min_count);
}

// min(1, (sqrt(c/(s*T)) + 1) * s*T/c), evaluated in double (corpus.hpp:176-181).
inline double keep_probability(std::int64_t count, std::int64_t total_tokens, double sample) {
    const double st = sample * static_cast<double>(total_tokens);
    const double c = static_cast<double>(count);
    const double p = (std::sqrt(c / st) + 1.0) * st / c;
    return std::min(p, 1.0);
}

struct CorpusShard {
    std::uint64_t byte_start = 0;
    std::uint64_t byte_end = 0;
};

// num_workers near-equal byte ranges; interior cuts move forward to the byte after
// the next separator so no token straddles two shards (corpus.hpp:190-223).
inline std::vector<CorpusShard> shard(const std::string& path, std::int32_t num_workers) {
    auto f = corpus_detail::open_or_throw(path);
    const std::uint64_t size = corpus_detail::file_size(f.get());
    std::vector<std::uint64_t> cut(static_cast<std::size_t>(num_workers) + 1, size);
    cut[0] = 0;
    for (std::int32_t i = 1; i < num_workers; ++i) {
        std::uint64_t p = size * static_cast<std::uint64_t>(i) / static_cast<std::uint64_t>(num_workers);
        if (p > 0) {
            std::fseek(f.get(), static_cast<long>(p - 1), SEEK_SET);
            int c;
            while ((c = std::fgetc(f.get())) != EOF && !is_token_separator(static_cast<char>(c))) ++p;
            if (c == EOF) p = size;
        }
        cut[static_cast<std::size_t>(i)] = std::max(p, cut[static_cast<std::size_t>(i) - 1]);
    }
    std::vector<CorpusShard> out(static_cast<std::size_t>(num_workers));
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = {cut[i], std::max(cut[i], cut[i + 1])};
    return out;
}

// Sequential, resettable token reader over one shard.
class ShardReader {
public:
    ShardReader(const std::string& path, CorpusShard range) : f_(corpus_detail::open_or_throw(path)), range_(range) {
        reset();
    }

    void reset() {
        std::fseek(f_.get(), static_cast<long>(range_.byte_start), SEEK_SET);
        pos_ = range_.byte_start;
        have_ = next_ = 0;
    }

    bool next_token(std::string& token) {
        token.clear();
        int c;
        do {
            if (pos_ >= range_.byte_end) return false;
            if ((c = peek()) < 0) return false;
            if (!is_token_separator(static_cast<char>(c))) break;
            bump();
        } while (true);
        while ((c = peek()) >= 0 && !is_token_separator(static_cast<char>(c))) {
            token.push_back(static_cast<char>(c));
            bump();
        }
        return true;
    }

private:
    int peek() {
        if (next_ == have_) {
            have_ = std::fread(buf_, 1, sizeof buf_, f_.get());
            next_ = 0;
            if (have_ == 0) return -1;
        }
        return static_cast<unsigned char>(buf_[next_]);
    }
    void bump() { ++next_; ++pos_; }

    corpus_detail::FilePtr f_;
    CorpusShard range_;
    std::uint64_t pos_ = 0;
    std::size_t have_ = 0, next_ = 0;
    char buf_[1 << 16];
};

// The in-vocabulary id stream of one shard, in file order (OOV tokens dropped), i.e.
// exactly the sequence train_worker obtains from ShardReader + Vocabulary::id_of.
inline std::vector<std::int32_t> read_id_stream(const std::string& path, const Vocabulary& vocab,
                                                CorpusShard range = {0, UINT64_MAX}) {
    auto f = corpus_detail::open_or_throw(path);
    std::vector<std::int32_t> ids;
    ids.reserve(static_cast<std::size_t>(std::max<std::int64_t>(vocab.total_tokens(), 0)));
    corpus_detail::for_each_token(f.get(), range.byte_start, range.byte_end, [&](std::string_view t) {
        const std::int32_t id = vocab.id_of(t);
        if (id >= 0) ids.push_back(id);
    });
    return ids;
}

}  // namespace cachegram
