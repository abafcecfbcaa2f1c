// cg_ingest.cu -- corpus ingest on the GPU.
//
// The reference tokenises the corpus text on the host in every worker pass
// (ShardReader + Vocabulary::id_of, corpus.hpp:228-283, trainer.hpp:220-222) and builds
// the vocabulary with a single-threaded hash map (corpus.hpp:136-170). Here the file is
// streamed through pinned host buffers into HBM in chunks cut at separators, and:
//   * tok_ids:   every token is hashed and looked up in a device open-addressing table
//                of the vocabulary (full byte comparison on hash hits), and the
//                in-vocabulary ids are compacted in file order straight into the
//                training session's id buffer -- exactly the sequence the reference's
//                reader yields (OOV tokens dropped);
//   * tok_count: every token is inserted into a growing device table (warp-aggregated
//                count increments, first-occurrence byte offset by atomicMin, one copy of
//                each distinct word's bytes in a device pool); the host then orders the
//                survivors exactly like VocabBuilder::finish (count descending, first
//                occurrence on ties).
// Separators are the reference's: ' ', \t, \n, \v, \f, \r (corpus.hpp:19-21).
//
// Layout: a chunk is processed in 4 KiB tiles, one 256-thread CTA per tile, 16 bytes per
// thread. A thread owns the tokens that START in its 16 bytes (at most 8) and scans each
// to its end. Tile-local compaction goes to a scratch slot of 2048 ids per tile (the most
// tokens a 4 KiB tile can start), then a scan of the tile counts and a coalesced copy
// place them at the running device-side cursor, so chunks pipeline without host syncs.
// This is HBM/L2-bound byte work: one pass over the bytes, one table probe per token.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

#include <unistd.h>
#include <vector>

#include "cachegram/errors.hpp"
#include "cg_device.cuh"
#include "cg_host.h"
#include "cg_kernels.h"

namespace cgk {
namespace {

using namespace cgdev;

constexpr int kTokThreads = 256;
constexpr int kTokPer = 16;                          // bytes per thread
constexpr int kTokTile = kTokThreads * kTokPer;      // 4096 bytes per CTA
constexpr int kTokCap = kTokTile / 2;                // max tokens starting in a tile
constexpr unsigned long long kEmpty = 0ull;
constexpr unsigned long long kUnpublished = ~0ull;

__host__ __device__ __forceinline__ bool is_sep(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

// FNV-1a 64, never 0 (0 marks an empty slot).
__host__ __device__ __forceinline__ unsigned long long fnv_step(unsigned long long h, unsigned char c) {
    return (h ^ c) * 0x100000001b3ull;
}
constexpr unsigned long long kFnvBasis = 0xcbf29ce484222325ull;
__host__ __device__ __forceinline__ unsigned long long fnv_final(unsigned long long h) { return h ? h : 1ull; }

// Hash of the token starting at i (bytes[i] is not a separator); *len receives its length.
__device__ __forceinline__ unsigned long long token_hash(const unsigned char* b, int64_t n, int64_t i, int* len) {
    unsigned long long h = kFnvBasis;
    int64_t j = i;
    while (j < n) {
        const unsigned char c = b[j];
        if (is_sep(c)) break;
        h = fnv_step(h, c);
        ++j;
    }
    *len = static_cast<int>(j - i);
    return fnv_final(h);
}

__device__ __forceinline__ bool same_bytes(const unsigned char* a, const char* b, int len) {
    for (int k = 0; k < len; ++k)
        if (a[k] != static_cast<unsigned char>(b[k])) return false;
    return true;
}

// Block-wide exclusive scan of one int per thread; returns the block total in *total.
__device__ __forceinline__ int block_excl_scan(int v, int* total) {
    __shared__ int warp_sums[kTokThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < kTokThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kTokThreads / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    const int base = w ? warp_sums[w - 1] : 0;
    *total = warp_sums[kTokThreads / 32 - 1];
    __syncthreads();
    return base + x - v;
}

// Does position i (0 <= i < n) start a token?
__device__ __forceinline__ bool starts_token(const unsigned char* b, int64_t i) {
    return !is_sep(b[i]) && (i == 0 || is_sep(b[i - 1]));
}

// ---------------------------------------------------------------- ids (lookup)
__global__ void __launch_bounds__(kTokThreads) tok_ids_kernel(TokChunk c, WordTableDev t, int32_t* tmp,
                                                              uint32_t* tile_count) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTokTile + threadIdx.x * kTokPer;
    int32_t found[kTokPer / 2];
    int nf = 0;
    for (int k = 0; k < kTokPer; ++k) {
        const int64_t i = base + k;
        if (i >= c.n) break;
        if (!starts_token(c.bytes, i)) continue;
        int len;
        const unsigned long long h = token_hash(c.bytes, c.n, i, &len);
        uint64_t s = h & t.mask;
        int32_t id = -1;
        for (;;) {
            const unsigned long long key = t.keys[s];
            if (key == kEmpty) break;
            if (key == h && t.len[s] == len && same_bytes(c.bytes + i, t.pool + t.off[s], len)) {
                id = t.ids[s];
                break;
            }
            s = (s + 1) & t.mask;
        }
        if (id >= 0) found[nf++] = id;
    }
    int total;
    const int off = block_excl_scan(nf, &total);
    int32_t* out = tmp + static_cast<int64_t>(blockIdx.x) * kTokCap + off;
    for (int k = 0; k < nf; ++k) out[k] = found[k];
    if (threadIdx.x == 0) tile_count[blockIdx.x] = static_cast<uint32_t>(total);
}

// Exclusive scan of tile counts into tile_off (single CTA); tile_off[ntiles] = total.
__global__ void __launch_bounds__(1024) tok_scan_kernel(const uint32_t* cnt, uint64_t* off, int64_t ntiles) {
    __shared__ uint64_t part[1024];
    const int64_t per = (ntiles + 1023) / 1024;
    const int64_t b = threadIdx.x * per, e = min(b + per, ntiles);
    uint64_t s = 0;
    for (int64_t i = b; i < e; ++i) s += cnt[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const uint64_t add = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += add;
        __syncthreads();
    }
    uint64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
    for (int64_t i = b; i < e; ++i) {
        off[i] = run;
        run += cnt[i];
    }
    if (threadIdx.x == 1023) off[ntiles] = part[1023];
}

// Copies each tile's compacted ids to out[*cursor + tile_off[tile] ...]; ids past
// `capacity` are counted but not written (the caller retries with a larger buffer).
__global__ void __launch_bounds__(kTokThreads) tok_scatter_kernel(const int32_t* tmp, const uint32_t* tile_count,
                                                                  const uint64_t* tile_off, const uint64_t* cursor,
                                                                  int32_t* out, uint64_t capacity) {
    const uint64_t base = *cursor + tile_off[blockIdx.x];
    const int n = static_cast<int>(tile_count[blockIdx.x]);
    const int32_t* src = tmp + static_cast<int64_t>(blockIdx.x) * kTokCap;
    for (int k = threadIdx.x; k < n; k += kTokThreads)
        if (base + k < capacity) out[base + k] = src[k];
}

__global__ void tok_advance_kernel(uint64_t* cursor, const uint64_t* tile_off, int64_t ntiles) {
    *cursor += tile_off[ntiles];
}

// ---------------------------------------------------------------- counting
// Insert-or-increment; counts are warp-aggregated over lanes holding the same word.
__global__ void __launch_bounds__(kTokThreads) tok_count_kernel(TokChunk c, CountTableDev t) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTokTile + threadIdx.x * kTokPer;
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < kTokPer; ++k) {
        const int64_t i = base + k;
        const bool start = i < c.n && starts_token(c.bytes, i);
        if (!__any_sync(kFull, start)) continue;
        int len = 0;
        unsigned long long h = 0;
        uint64_t slot = 0;
        if (start) {
            h = token_hash(c.bytes, c.n, i, &len);
            uint64_t s = h & t.mask;
            for (;;) {
                unsigned long long key = t.keys[s];
                if (key == kEmpty) {
                    key = atomicCAS(t.keys + s, kEmpty, h);
                    if (key == kEmpty) {  // claimed: publish one copy of the word's bytes
                        const unsigned long long o = atomicAdd(t.pool_cursor, static_cast<unsigned long long>(len));
                        if (o + len <= t.pool_capacity) {
                            for (int q = 0; q < len; ++q) t.pool[o + q] = static_cast<char>(c.bytes[i + q]);
                        } else {
                            atomicExch(t.overflow, 1);
                        }
                        t.len[s] = len;
                        __threadfence();
                        atomicExch(t.off + s, o);
                        atomicAdd(t.distinct, 1ull);
                        break;
                    }
                }
                if (key == h) {
                    unsigned long long o;
                    while ((o = *reinterpret_cast<volatile unsigned long long*>(t.off + s)) == kUnpublished) {
                    }
                    __threadfence();
                    if (t.len[s] == len && (o + len > t.pool_capacity || same_bytes(c.bytes + i, t.pool + o, len)))
                        break;
                }
                s = (s + 1) & t.mask;
            }
            slot = s;
        }
        // one atomic per distinct slot in the warp
        const unsigned peers = __match_any_sync(kFull, start ? slot : ~0ull);
        if (start) {
            const int leader = __ffs(peers) - 1;
            if (lane == leader) atomicAdd(t.count + slot, static_cast<unsigned long long>(__popc(peers)));
            atomicMin(t.first + slot, static_cast<unsigned long long>(c.global_offset + i));
        }
    }
}

// Re-inserts every live slot of `from` into the (larger, empty) table `to`.
__global__ void table_rehash_kernel(CountTableDev from, CountTableDev to) {
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s <= from.mask;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long h = from.keys[s];
        if (h == kEmpty) continue;
        uint64_t d = h & to.mask;
        while (atomicCAS(to.keys + d, kEmpty, h) != kEmpty) d = (d + 1) & to.mask;
        to.count[d] = from.count[s];
        to.first[d] = from.first[s];
        to.off[d] = from.off[s];
        to.len[d] = from.len[s];
    }
}

// Compacts live slots into entries (order irrelevant: the host sorts).
__global__ void table_export_kernel(CountTableDev t, CountEntry* out, unsigned long long* n_out) {
    for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s <= t.mask;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (t.keys[s] == kEmpty) continue;
        const unsigned long long k = atomicAdd(n_out, 1ull);
        out[k] = CountEntry{t.count[s], t.first[s], t.off[s], t.len[s], 0};
    }
}

__global__ void fill_u64_kernel(unsigned long long* p, uint64_t n, unsigned long long v) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw cgint::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device / pinned buffers come from the library's caching pools: the ingest runs once per
// train(corpus_path) call, and raw cudaMalloc/cudaMallocHost of ~0.5 GB per call would
// cost more than the tokenisation itself.
template <typename T>
void dalloc(T** p, size_t bytes) {
    *p = static_cast<T*>(cgint::DevicePool::get().alloc(bytes));
}
template <typename T>
void dfree(T*& p) {
    cgint::DevicePool::get().free(p);
    p = nullptr;
}

// Chunk size of the file reader; CG_INGEST_CHUNK (bytes, >= 64) overrides it so tests can
// exercise many chunks and the token-longer-than-a-chunk path on small files.
size_t chunk_bytes(size_t dflt) {
    if (const char* e = std::getenv("CG_INGEST_CHUNK")) {
        const long long v = std::atoll(e);
        if (v >= 64) return static_cast<size_t>(v);
    }
    return dflt;
}

unsigned grid_of(uint64_t n) { return static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148ull * 16)); }

// Streams a file through pinned double buffers; each delivered chunk ends at a
// separator (or at EOF) so that no token straddles two chunks.
class ChunkReader {
public:
    // first > 0: the first chunk holds at most `first` bytes and each next one twice the
    // previous, up to `chunk` (a consumer that starts on the first chunk waits less)
    ChunkReader(const char* path, size_t chunk, size_t first = 0) : cap_(chunk), limit_(first ? std::min(first, chunk) : chunk) {
        f_ = std::fopen(path, "rb");
        if (!f_) throw cachegram::IoError(std::string("cannot open corpus file: ") + path);
        for (auto& b : buf_) b = static_cast<unsigned char*>(cgint::PinnedPool::get().alloc(cap_));
    }
    ~ChunkReader() {
        if (f_) std::fclose(f_);
        for (auto* b : buf_) cgint::PinnedPool::get().free(b);
    }
    // Fills buffer `which`; returns the usable length (0 at the end of the file).
    size_t next(int which) {
        unsigned char* b = buf_[which];
        size_t have = carry_.size();
        if (have) std::memcpy(b, carry_.data(), have);
        carry_.clear();
        const size_t lim = std::max(std::min(cap_, limit_), have);
        limit_ = std::min(cap_, limit_ * 2);
        if (!eof_ && have < lim) {
            const size_t got = parallel_read(b + have, lim - have);
            if (got < lim - have) eof_ = true;
            have += got;
        }
        if (eof_ || have == 0) return have;
        size_t cut = have;
        while (cut > 0 && !is_sep(b[cut - 1])) --cut;
        if (cut == 0) {  // one token longer than the chunk: grow and keep reading
            grow(which, have);
            return next_grown(which, have);
        }
        carry_.assign(b + cut, b + have);
        return cut;
    }
    unsigned char* buffer(int which) const { return buf_[which]; }
    size_t capacity() const { return cap_; }

private:
    // Fills dst[0, n) from the file position with up to kReadThreads concurrent pread()s
    // (a single reader is memcpy-bound at ~3 GB/s from the page cache). Returns the bytes
    // read; fewer than n only at the end of the file.
    size_t parallel_read(unsigned char* dst, size_t n) {
        constexpr size_t kPiece = size_t{8} << 20;
        const int fd = fileno(f_);
        const size_t pieces = (n + kPiece - 1) / kPiece;
        const size_t nt = std::min<size_t>(kReadThreads, pieces);
        std::vector<size_t> got(pieces, 0);
        auto work = [&](size_t t) {
            for (size_t p = t; p < pieces; p += nt) {
                const size_t b = p * kPiece, len = std::min(kPiece, n - b);
                size_t done = 0;
                while (done < len) {
                    const ssize_t r = pread(fd, dst + b + done, len - done, static_cast<off_t>(pos_ + b + done));
                    if (r <= 0) break;
                    done += static_cast<size_t>(r);
                }
                got[p] = done;
            }
        };
        std::vector<std::thread> th;
        for (size_t t = 1; t < nt; ++t) th.emplace_back(work, t);
        work(0);
        for (auto& x : th) x.join();
        size_t total = 0;
        for (size_t p = 0; p < pieces; ++p) {  // contiguous prefix
            total += got[p];
            if (got[p] < std::min(kPiece, n - p * kPiece)) break;
        }
        pos_ += total;
        return total;
    }
    static constexpr size_t kReadThreads = 8;
    uint64_t pos_ = 0;

    void grow(int which, size_t have) {
        // the other buffer may still feed an asynchronous H2D copy: let it land first
        cudaDeviceSynchronize();
        const size_t ncap = cap_ * 2;
        for (int k = 0; k < 2; ++k) {
            unsigned char* nb = static_cast<unsigned char*>(cgint::PinnedPool::get().alloc(ncap));
            if (k == which) std::memcpy(nb, buf_[k], have);
            cgint::PinnedPool::get().free(buf_[k]);
            buf_[k] = nb;
        }
        cap_ = ncap;
    }
    size_t next_grown(int which, size_t have) {
        carry_.assign(buf_[which], buf_[which] + have);
        return next(which);
    }

    std::FILE* f_ = nullptr;
    size_t cap_;
    size_t limit_;
    unsigned char* buf_[2] = {nullptr, nullptr};
    std::vector<unsigned char> carry_;
    bool eof_ = false;
};

}  // namespace

unsigned long long host_token_hash(const char* s, size_t len) {
    unsigned long long h = kFnvBasis;
    for (size_t k = 0; k < len; ++k) h = fnv_step(h, static_cast<unsigned char>(s[k]));
    return fnv_final(h);
}

// ---------------------------------------------------------------- host drivers
void WordTableHost::build(const std::vector<std::string>& words) {
    uint64_t cap = 1024;
    while (cap < 2 * static_cast<uint64_t>(words.size()) + 2) cap <<= 1;
    mask = cap - 1;
    keys.assign(cap, 0);
    ids.assign(cap, -1);
    off.assign(cap, 0);
    len.assign(cap, 0);
    pool.clear();
    for (size_t w = 0; w < words.size(); ++w) {
        const std::string& word = words[w];
        const unsigned long long h = host_token_hash(word.data(), word.size());
        uint64_t s = h & mask;
        bool dup = false;
        while (keys[s] != 0) {
            if (keys[s] == h && len[s] == static_cast<int32_t>(word.size()) &&
                std::memcmp(pool.data() + off[s], word.data(), word.size()) == 0) {
                dup = true;  // Vocabulary::id_of keeps the first id of a repeated word
                break;
            }
            s = (s + 1) & mask;
        }
        if (dup) continue;
        keys[s] = h;
        ids[s] = static_cast<int32_t>(w);
        off[s] = static_cast<int64_t>(pool.size());
        len[s] = static_cast<int32_t>(word.size());
        pool.insert(pool.end(), word.begin(), word.end());
    }
}

int64_t ingest_ids(const char* path, const WordTableDev& table, int32_t* out, uint64_t capacity, cudaStream_t st,
                   IngestStats* stats, const IngestProgress* progress) {
    const auto t0 = std::chrono::steady_clock::now();
    // small enough that reading overlaps tokenising (CG_INGEST_CHUNK overrides, for tests)
    // (the first chunks ramp up from 4 MB, so training on them starts sooner)
    ChunkReader rd(path, chunk_bytes(size_t{32} << 20), progress ? chunk_bytes(size_t{4} << 20) : 0);
    unsigned char* dbytes[2] = {nullptr, nullptr};
    int32_t* tmp = nullptr;
    uint32_t* tcount = nullptr;
    uint64_t* toff = nullptr;
    uint64_t* cursor = nullptr;
    cudaEvent_t done[2];
    size_t dcap = 0;
    auto ensure = [&](size_t bytes) {
        if (bytes <= dcap) return;
        check(cudaStreamSynchronize(st), "sync");
        for (auto& p : dbytes) {
            dfree(p);
            dalloc(&p, bytes + 16);
        }
        dfree(tmp);
        dfree(tcount);
        dfree(toff);
        const size_t nt = (bytes + kTokTile - 1) / kTokTile;
        dalloc(&tmp, nt * kTokCap * sizeof(int32_t));
        dalloc(&tcount, nt * sizeof(uint32_t));
        dalloc(&toff, (nt + 1) * sizeof(uint64_t));
        dcap = bytes;
    };
    dalloc(&cursor, sizeof(uint64_t));
    check(cudaMemsetAsync(cursor, 0, sizeof(uint64_t), st), "memset");
    for (auto& e : done) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    bool used[2] = {false, false};
    uint64_t bytes_total = 0;
    int k = 0, chunk = 0;
    try {
        for (;; k ^= 1) {
            if (used[k]) check(cudaEventSynchronize(done[k]), "event sync");  // host buffer k free again
            const size_t n = rd.next(k);
            if (n == 0) break;
            ensure(rd.capacity());
            bytes_total += n;
            check(cudaMemcpyAsync(dbytes[k], rd.buffer(k), n, cudaMemcpyHostToDevice, st), "H2D");
            const int64_t nt = static_cast<int64_t>((n + kTokTile - 1) / kTokTile);
            TokChunk c{dbytes[k], static_cast<int64_t>(n), 0};
            tok_ids_kernel<<<static_cast<unsigned>(nt), kTokThreads, 0, st>>>(c, table, tmp, tcount);
            tok_scan_kernel<<<1, 1024, 0, st>>>(tcount, toff, nt);
            tok_scatter_kernel<<<static_cast<unsigned>(nt), kTokThreads, 0, st>>>(tmp, tcount, toff, cursor, out,
                                                                                capacity);
            tok_advance_kernel<<<1, 1, 0, st>>>(cursor, toff, nt);
            check(cudaGetLastError(), "tokenize launch");
            check(cudaEventRecord(done[k], st), "event");
            used[k] = true;
            if (stats) stats->launches += 4;
            if (progress) {
                uint64_t* w = progress->word(progress->ctx, chunk);
                check(cudaMemcpyAsync(w, cursor, sizeof(uint64_t), cudaMemcpyDeviceToHost, st), "D2H");
                cudaEvent_t ev;
                check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
                check(cudaEventRecord(ev, st), "event");
                progress->on_chunk(progress->ctx, chunk, ev);
            }
            ++chunk;
        }
        uint64_t total = 0;
        check(cudaMemcpyAsync(&total, cursor, sizeof total, cudaMemcpyDeviceToHost, st), "D2H");
        check(cudaStreamSynchronize(st), "sync");
        for (auto& e : done) cudaEventDestroy(e);
        for (auto*& p : dbytes) dfree(p);
        dfree(tmp);
        dfree(tcount);
        dfree(toff);
        dfree(cursor);
        if (stats) {
            stats->bytes = bytes_total;
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        return static_cast<int64_t>(total);
    } catch (...) {
        cudaStreamSynchronize(st);
        for (auto& e : done) cudaEventDestroy(e);
        for (auto*& p : dbytes) dfree(p);
        dfree(tmp);
        dfree(tcount);
        dfree(toff);
        dfree(cursor);
        throw;
    }
}

namespace {
struct DevCountTable {
    CountTableDev t{};
    uint64_t cap = 0;
    void alloc(uint64_t slots, cudaStream_t st) {
        cap = slots;
        t.mask = slots - 1;
        dalloc(&t.keys, slots * 8);
        dalloc(&t.count, slots * 8);
        dalloc(&t.first, slots * 8);
        dalloc(&t.off, slots * 8);
        dalloc(&t.len, slots * 4);
        check(cudaMemsetAsync(t.keys, 0, slots * 8, st), "memset");
        check(cudaMemsetAsync(t.count, 0, slots * 8, st), "memset");
        fill_u64_kernel<<<grid_of(slots), 256, 0, st>>>(t.first, slots, ~0ull);
        fill_u64_kernel<<<grid_of(slots), 256, 0, st>>>(t.off, slots, kUnpublished);
    }
    void release() {
        dfree(t.keys);
        dfree(t.count);
        dfree(t.first);
        dfree(t.off);
        dfree(t.len);
        t.keys = t.count = t.first = t.off = nullptr;
        t.len = nullptr;
    }
};
}  // namespace

std::vector<CountedWord> ingest_count(const char* path, cudaStream_t st, IngestStats* stats) {
    const auto t0 = std::chrono::steady_clock::now();
    ChunkReader rd(path, chunk_bytes(size_t{64} << 20));
    unsigned char* dbytes[2] = {nullptr, nullptr};
    size_t dcap = 0;
    DevCountTable tab;
    unsigned long long* scalars = nullptr;  // [0] pool cursor, [1] distinct, [2] overflow, [3] export count
    char* pool = nullptr;
    uint64_t pool_cap = 0;
    cudaEvent_t done[2];
    for (auto& e : done) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    auto cleanup = [&] {
        cudaStreamSynchronize(st);
        for (auto& e : done) cudaEventDestroy(e);
        for (auto*& p : dbytes) dfree(p);
        tab.release();
        dfree(scalars);
        dfree(pool);
    };
    try {
        dalloc(&scalars, 4 * 8);
        check(cudaMemsetAsync(scalars, 0, 4 * 8, st), "memset");
        uint64_t distinct_bound = 0;  // upper bound on distinct words so far
        uint64_t pool_bound = 0;      // upper bound on pool bytes so far
        bool used[2] = {false, false};
        uint64_t offset = 0;
        int k = 0;
        for (;; k ^= 1) {
            if (used[k]) check(cudaEventSynchronize(done[k]), "event sync");
            const size_t n = rd.next(k);
            if (n == 0) break;
            if (rd.capacity() > dcap) {
                check(cudaStreamSynchronize(st), "sync");
                for (auto& p : dbytes) {
                    dfree(p);
                    dalloc(&p, rd.capacity() + 16);
                }
                dcap = rd.capacity();
            }
            // Keep the load factor <= 1/2 even if every token of this chunk is new, and
            // room in the pool for every byte of it: read the exact distinct count back
            // only when the bound says the table might need to grow.
            const uint64_t new_tokens = n / 2 + 1;
            if (2 * (distinct_bound + new_tokens) > tab.cap || pool_bound + n > pool_cap) {
                check(cudaStreamSynchronize(st), "sync");
                unsigned long long sc[4];
                check(cudaMemcpy(sc, scalars, sizeof sc, cudaMemcpyDeviceToHost), "D2H");
                distinct_bound = sc[1];
                pool_bound = sc[0];
                uint64_t want = 1u << 20;
                while (want < 2 * (distinct_bound + new_tokens)) want <<= 1;
                if (want > tab.cap) {
                    DevCountTable nt;
                    nt.alloc(want, st);
                    if (tab.cap) {
                        table_rehash_kernel<<<grid_of(tab.cap), 256, 0, st>>>(tab.t, nt.t);
                        check(cudaStreamSynchronize(st), "sync");
                        tab.release();
                    }
                    tab = nt;
                }
                if (pool_bound + n > pool_cap) {
                    const uint64_t ncap = std::max<uint64_t>(2 * pool_cap, pool_bound + n + (16u << 20));
                    char* np = nullptr;
                    dalloc(&np, ncap);
                    if (pool_bound) check(cudaMemcpyAsync(np, pool, pool_bound, cudaMemcpyDeviceToDevice, st), "D2D");
                    check(cudaStreamSynchronize(st), "sync");
                    dfree(pool);
                    pool = np;
                    pool_cap = ncap;
                }
            }
            distinct_bound += new_tokens;
            pool_bound += n;
            tab.t.pool = pool;
            tab.t.pool_capacity = pool_cap;
            tab.t.pool_cursor = scalars;
            tab.t.distinct = scalars + 1;
            tab.t.overflow = scalars + 2;
            check(cudaMemcpyAsync(dbytes[k], rd.buffer(k), n, cudaMemcpyHostToDevice, st), "H2D");
            const int64_t nt = static_cast<int64_t>((n + kTokTile - 1) / kTokTile);
            tok_count_kernel<<<static_cast<unsigned>(nt), kTokThreads, 0, st>>>(
                TokChunk{dbytes[k], static_cast<int64_t>(n), offset}, tab.t);
            check(cudaGetLastError(), "count launch");
            check(cudaEventRecord(done[k], st), "event");
            used[k] = true;
            offset += n;
            if (stats) stats->launches += 1;
        }
        check(cudaStreamSynchronize(st), "sync");
        unsigned long long sc[4];
        check(cudaMemcpy(sc, scalars, sizeof sc, cudaMemcpyDeviceToHost), "D2H");
        if (sc[2]) throw std::runtime_error("ingest_count: word pool overflow");
        const uint64_t distinct = sc[1];
        std::vector<CountedWord> out;
        if (distinct) {
            CountEntry* ent = nullptr;
            dalloc(&ent, distinct * sizeof(CountEntry));
            check(cudaMemsetAsync(scalars + 3, 0, 8, st), "memset");
            table_export_kernel<<<grid_of(tab.cap), 256, 0, st>>>(tab.t, ent, scalars + 3);
            std::vector<CountEntry> host(distinct);
            std::vector<char> hpool(sc[0]);
            check(cudaMemcpyAsync(host.data(), ent, distinct * sizeof(CountEntry), cudaMemcpyDeviceToHost, st), "D2H");
            if (sc[0]) check(cudaMemcpyAsync(hpool.data(), pool, sc[0], cudaMemcpyDeviceToHost, st), "D2H");
            check(cudaStreamSynchronize(st), "sync");
            dfree(ent);
            out.resize(distinct);
            for (uint64_t i = 0; i < distinct; ++i) {
                out[i].count = static_cast<int64_t>(host[i].count);
                out[i].first = host[i].first;
                out[i].word.assign(hpool.data() + host[i].off, host[i].len);
            }
        }
        cleanup();
        if (stats) {
            stats->bytes = offset;
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        return out;
    } catch (...) {
        cleanup();
        throw;
    }
}

}  // namespace cgk
