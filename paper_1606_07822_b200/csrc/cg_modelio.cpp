// cg_modelio.cpp -- model files: the reference's text and binary
// embedding formats (model.hpp:107-276), behind the C-ABI of cachegram_b200.h.
//
// Text:   "V D\n", then per word "word" + D x " %.6f" + "\n"   (model.hpp:119-130)
// Binary: "V D\n", then per word "word " + D raw float32 + "\n" (model.hpp:132-144)
// Loading mirrors load_embeddings_{binary,text} and the auto-detection of
// load_embeddings (model.hpp:172-276): same accepted inputs, same error classes
// (IoError when a file cannot be opened, ParseError on a format violation).
//
// The output bytes are those of the reference's single-threaded fprintf loop; the row
// formatting (the expensive part: %.6f of V x D doubles, ~300M values at C5) is spread
// over all host cores in row blocks and written in order. Parsing the text format also
// runs row-parallel after one newline scan.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <system_error>
#include <thread>
#include <vector>

#include "cachegram/errors.hpp"
#include "cachegram_b200.h"
#include "cg_host.h"

using cachegram::IoError;
using cachegram::ParseError;

struct cg_embeddings_file {
    int32_t dim = 0;
    std::vector<std::string> words;
    std::vector<float> vectors;
};

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return CG_OK;
    } catch (const ParseError& e) {
        cgint::set_last_error(e.what());
        return CG_ERR_PARSE;
    } catch (const IoError& e) {
        cgint::set_last_error(e.what());
        return CG_ERR_IO;
    } catch (const std::invalid_argument& e) {
        cgint::set_last_error(e.what());
        return CG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        cgint::set_last_error(e.what());
        return CG_ERR_INTERNAL;
    }
}

unsigned host_threads() {
    const unsigned n = std::thread::hardware_concurrency();
    return n ? std::min(n, 64u) : 1u;
}

// Runs body(i) for i in [0, n) on up to host_threads() threads, contiguous ranges.
template <typename F>
void parallel_for(int64_t n, F&& body) {
    const int64_t t = std::min<int64_t>(host_threads(), std::max<int64_t>(n, 1));
    if (t <= 1) {
        for (int64_t i = 0; i < n; ++i) body(i);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t chunk = (n + t - 1) / t;
    for (int64_t k = 0; k < t; ++k) {
        const int64_t b = k * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&body, b, e] {
            for (int64_t i = b; i < e; ++i) body(i);
        });
    }
    for (auto& th : pool) th.join();
}

std::vector<const char*> split_words(const char* words_nul, int32_t n) {
    std::vector<const char*> w(static_cast<size_t>(n));
    const char* p = words_nul;
    for (int32_t i = 0; i < n; ++i) {
        w[static_cast<size_t>(i)] = p;
        p += std::strlen(p) + 1;
    }
    return w;
}

struct File {
    std::FILE* f;
    explicit File(std::FILE* x) : f(x) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

void save(const std::string& path, int32_t format, const char* words_nul, const float* syn0, int32_t V, int32_t D) {
    if (V < 0 || D < 1) throw std::invalid_argument("model file needs V >= 0 and D >= 1");
    std::FILE* raw = std::fopen(path.c_str(), "wb");
    if (!raw) throw IoError("cannot write model file: " + path);
    File f(raw);
    std::fprintf(f.f, "%d %d\n", V, D);
    const auto words = split_words(words_nul, V);
    if (format == CG_FORMAT_BINARY) {
        for (int32_t w = 0; w < V; ++w) {
            std::fputs(words[static_cast<size_t>(w)], f.f);
            std::fputc(' ', f.f);
            std::fwrite(syn0 + static_cast<size_t>(w) * static_cast<size_t>(D), sizeof(float), static_cast<size_t>(D),
                        f.f);
            std::fputc('\n', f.f);
        }
    } else {
        // Row blocks formatted in parallel, written in order.
        constexpr int64_t kRowsPerBlock = 256;
        const int64_t nblocks = (static_cast<int64_t>(V) + kRowsPerBlock - 1) / kRowsPerBlock;
        const int64_t batch = static_cast<int64_t>(host_threads()) * 4;
        std::vector<std::string> buf(static_cast<size_t>(batch));
        for (int64_t b0 = 0; b0 < nblocks; b0 += batch) {
            const int64_t nb = std::min(batch, nblocks - b0);
            parallel_for(nb, [&](int64_t i) {
                std::string& out = buf[static_cast<size_t>(i)];
                out.clear();
                const int64_t r0 = (b0 + i) * kRowsPerBlock, r1 = std::min<int64_t>(V, r0 + kRowsPerBlock);
                char num[512];
                for (int64_t w = r0; w < r1; ++w) {
                    out += words[static_cast<size_t>(w)];
                    const float* row = syn0 + static_cast<size_t>(w) * static_cast<size_t>(D);
                    for (int32_t d = 0; d < D; ++d) {
                        const int len = std::snprintf(num, sizeof(num), " %.6f", static_cast<double>(row[d]));
                        out.append(num, static_cast<size_t>(len));
                    }
                    out.push_back('\n');
                }
            });
            for (int64_t i = 0; i < nb; ++i) std::fwrite(buf[static_cast<size_t>(i)].data(), 1, buf[static_cast<size_t>(i)].size(), f.f);
        }
    }
    std::FILE* done = f.f;
    f.f = nullptr;
    if (std::ferror(done) || std::fclose(done) != 0) throw IoError("cannot write model file: " + path);
}

std::string slurp(const std::string& path) {
    std::FILE* raw = std::fopen(path.c_str(), "rb");
    if (!raw) throw IoError("cannot open model file: " + path);
    File f(raw);
    std::string data;
    char chunk[1 << 16];
    size_t n;
    while ((n = std::fread(chunk, 1, sizeof(chunk), f.f)) > 0) data.append(chunk, n);
    return data;
}

// detail::read_header (model.hpp:152-170): "<vocab> <dim>" on the first line, both > 0.
void read_header(const std::string& data, size_t& pos, const std::string& path, int64_t& vocab, int64_t& dim) {
    if (data.empty()) throw ParseError(path + ": malformed header: empty file");
    size_t nl = data.find('\n');
    if (nl == std::string::npos) nl = data.size();
    const std::string line = data.substr(0, nl);
    pos = nl < data.size() ? nl + 1 : nl;
    const char* b = line.data();
    const char* e = b + line.size();
    auto bad = [&] { return ParseError(path + ": malformed header: expected \"<vocab> <dim>\", got \"" + line + "\""); };
    auto r1 = std::from_chars(b, e, vocab);
    if (r1.ec != std::errc() || r1.ptr == e || *r1.ptr != ' ') throw bad();
    auto r2 = std::from_chars(r1.ptr + 1, e, dim);
    if (r2.ec != std::errc() || r2.ptr != e) throw bad();
    if (vocab <= 0 || dim <= 0) throw ParseError(path + ": malformed header: non-positive sizes in \"" + line + "\"");
}

// load_embeddings_binary (model.hpp:172-199): the word runs to the next space (newlines
// are dropped), then exactly D raw floats.
void load_binary(const std::string& path, cg_embeddings_file& out) {
    const std::string data = slurp(path);
    size_t pos = 0;
    int64_t V = 0, D = 0;
    read_header(data, pos, path, V, D);
    out.dim = static_cast<int32_t>(D);
    out.words.reserve(static_cast<size_t>(V));
    out.vectors.resize(static_cast<size_t>(V) * static_cast<size_t>(D));
    const size_t row_bytes = sizeof(float) * static_cast<size_t>(D);
    for (int64_t w = 0; w < V; ++w) {
        std::string word;
        while (pos < data.size() && data[pos] != ' ') {
            if (data[pos] != '\n') word.push_back(data[pos]);
            ++pos;
        }
        if (pos >= data.size()) throw ParseError(path + ": truncated row " + std::to_string(w) + ": unterminated word");
        ++pos;  // the space
        if (data.size() - pos < row_bytes)
            throw ParseError(path + ": truncated row " + std::to_string(w) + " for word \"" + word + "\"");
        std::memcpy(out.vectors.data() + static_cast<size_t>(w) * static_cast<size_t>(D), data.data() + pos, row_bytes);
        pos += row_bytes;
        out.words.push_back(std::move(word));
    }
}

// load_embeddings_text (model.hpp:201-245): one line per word, "word v1 ... vD", values
// separated by runs of spaces, nothing but spaces after the last one.
void load_text(const std::string& path, cg_embeddings_file& out) {
    const std::string data = slurp(path);
    size_t pos = 0;
    int64_t V = 0, D = 0;
    read_header(data, pos, path, V, D);
    std::vector<size_t> line_begin;
    line_begin.reserve(static_cast<size_t>(V) + 1);
    while (static_cast<int64_t>(line_begin.size()) < V && pos < data.size()) {
        line_begin.push_back(pos);
        const size_t nl = data.find('\n', pos);
        pos = nl == std::string::npos ? data.size() : nl + 1;
    }
    const int64_t lines = static_cast<int64_t>(line_begin.size());
    out.dim = static_cast<int32_t>(D);
    out.words.assign(static_cast<size_t>(V), std::string());
    out.vectors.resize(static_cast<size_t>(V) * static_cast<size_t>(D));
    // Parse rows in parallel; the first failing row (lowest index) is reported, as the
    // reference's sequential reader would.
    std::vector<std::string> err(static_cast<size_t>(lines));
    std::vector<uint8_t> failed(static_cast<size_t>(lines), 0);
    parallel_for(lines, [&](int64_t w) {
        const size_t b = line_begin[static_cast<size_t>(w)];
        size_t e = data.find('\n', b);
        if (e == std::string::npos) e = data.size();
        const char* lb = data.data() + b;
        const char* le = data.data() + e;
        const char* sp = static_cast<const char*>(std::memchr(lb, ' ', static_cast<size_t>(le - lb)));
        if (!sp || sp == lb) {
            failed[static_cast<size_t>(w)] = 1;
            err[static_cast<size_t>(w)] = path + ": row " + std::to_string(w) + ": expected \"word v1 ... vD\"";
            return;
        }
        out.words[static_cast<size_t>(w)].assign(lb, sp);
        float* row = out.vectors.data() + static_cast<size_t>(w) * static_cast<size_t>(D);
        const char* p = sp;
        for (int64_t d = 0; d < D; ++d) {
            while (p != le && *p == ' ') ++p;
            auto r = std::from_chars(p, le, row[d]);
            if (r.ec != std::errc()) {
                failed[static_cast<size_t>(w)] = 1;
                err[static_cast<size_t>(w)] = path + ": row " + std::to_string(w) + ": dimension mismatch: expected " +
                                              std::to_string(D) + " values";
                return;
            }
            p = r.ptr;
        }
        while (p != le && *p == ' ') ++p;
        if (p != le) {
            failed[static_cast<size_t>(w)] = 1;
            err[static_cast<size_t>(w)] =
                path + ": row " + std::to_string(w) + ": dimension mismatch: trailing values beyond " + std::to_string(D);
        }
    });
    for (int64_t w = 0; w < lines; ++w)
        if (failed[static_cast<size_t>(w)]) throw ParseError(err[static_cast<size_t>(w)]);
    if (lines < V) throw ParseError(path + ": truncated row " + std::to_string(lines));
}

// load_embeddings (model.hpp:249-274): binary iff the 512 bytes after the header line
// hold a byte outside printable ASCII other than \n, \r, \t.
bool looks_binary(const std::string& path) {
    std::FILE* raw = std::fopen(path.c_str(), "rb");
    if (!raw) throw IoError("cannot open model file: " + path);
    File f(raw);
    int c;
    while ((c = std::fgetc(f.f)) != EOF && c != '\n') {
    }
    unsigned char probe[512];
    const size_t got = std::fread(probe, 1, sizeof(probe), f.f);
    for (size_t i = 0; i < got; ++i) {
        const unsigned char b = probe[i];
        if (b != '\n' && b != '\r' && b != '\t' && (b < 0x20 || b > 0x7e)) return true;
    }
    return false;
}

}  // namespace

extern "C" {

int cg_model_save(const char* path, int32_t format, const char* words_nul, const float* syn0, int32_t vocab_size,
                  int32_t dim) {
    return guarded([&] {
        if (!path || (!words_nul && vocab_size > 0) || (!syn0 && vocab_size > 0))
            throw std::invalid_argument("cg_model_save: null argument");
        if (format != CG_FORMAT_TEXT && format != CG_FORMAT_BINARY)
            throw std::invalid_argument("cg_model_save: format must be text or binary");
        save(path, format, words_nul, syn0, vocab_size, dim);
    });
}

int cg_model_load(const char* path, int32_t format, cg_embeddings_file** out) {
    return guarded([&] {
        if (!path || !out) throw std::invalid_argument("cg_model_load: null argument");
        *out = nullptr;
        auto f = std::make_unique<cg_embeddings_file>();
        int32_t fmt = format;
        if (fmt == CG_FORMAT_AUTO) fmt = looks_binary(path) ? CG_FORMAT_BINARY : CG_FORMAT_TEXT;
        if (fmt == CG_FORMAT_BINARY)
            load_binary(path, *f);
        else if (fmt == CG_FORMAT_TEXT)
            load_text(path, *f);
        else
            throw std::invalid_argument("cg_model_load: unknown format");
        *out = f.release();
    });
}

int cg_model_file_info(const cg_embeddings_file* f, int32_t* vocab_size, int32_t* dim, int64_t* word_bytes) {
    return guarded([&] {
        if (!f) throw std::invalid_argument("cg_model_file_info: null handle");
        if (vocab_size) *vocab_size = static_cast<int32_t>(f->words.size());
        if (dim) *dim = f->dim;
        if (word_bytes) {
            int64_t n = 0;
            for (const auto& w : f->words) n += static_cast<int64_t>(w.size()) + 1;
            *word_bytes = n;
        }
    });
}

int cg_model_file_export(const cg_embeddings_file* f, char* words_nul, float* vectors) {
    return guarded([&] {
        if (!f) throw std::invalid_argument("cg_model_file_export: null handle");
        if (words_nul) {
            char* p = words_nul;
            for (const auto& w : f->words) {
                std::memcpy(p, w.data(), w.size());
                p += w.size();
                *p++ = '\0';
            }
        }
        if (vectors && !f->vectors.empty()) std::memcpy(vectors, f->vectors.data(), f->vectors.size() * sizeof(float));
    });
}

void cg_model_file_close(cg_embeddings_file* f) { delete f; }

}  // extern "C"
