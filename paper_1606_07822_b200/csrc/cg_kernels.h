// cg_kernels.h -- host-side launchers of the sm_100a kernels (internal to the .so).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace cgk {

// ---------------- deterministic single-stream mode (K2) ----------------------
// Reference layout: syn0 [V*D], syn1 [(V-1)*D] in reference node-id order.
struct DetModel {
    float* syn0;
    float* syn1;
    int32_t dim;
    int32_t vocab;
    const int64_t* path_off;   // [V+1]
    const int32_t* path_node;  // reference node ids
    const uint8_t* path_turn;
    const int32_t* slot_of;    // [V-1] or nullptr (no cache)
    const int32_t* hot_nodes;  // [K]
    int32_t hot_count;
    float* cache_work;         // [K*D]
    float* cache_snap;         // [K*D]
    uint8_t* cache_flag;       // [K]
    int32_t* acquired;         // [K] acquire order
    const float* sigmoid;      // [1000]
    float sig_scale;           // (float)1000 / 12.0f, folded on the host
};

// Worker state that carries across passes (trainer.hpp:203-212).
struct DetState {
    uint64_t rng;
    uint64_t progress;    // ProgressCounter::words_processed
    uint64_t unreported;
    float alpha;
    int32_t since_flush;
    int32_t n_acquired;
    int32_t pad;
    uint64_t centers, pairs, steps, words;
};

struct DetPass {
    const int32_t* ids;
    int64_t n_ids;
    const float* keep;     // [V] or nullptr when sample == 0
    int32_t window;
    int32_t flush_interval;
    uint64_t total_words;  // iterations * total_tokens
    float alpha0;
};

void launch_det_pass(const DetModel& m, const DetPass& p, DetState* state, cudaStream_t s);

struct DetCenter {
    int32_t center;
    const int32_t* sentence;
    int64_t len;
    int64_t pos;
    int32_t half_window;
    float alpha;
    int32_t sigmoid_mode;  // 0 table, 1 exact, 2 constant
    float sig_const;
    int32_t* n_acquired;   // device scalar
    unsigned long long* evals;
};
void launch_det_center(const DetModel& m, const DetCenter& c, cudaStream_t s);
void launch_det_flush_flags(const DetModel& m, cudaStream_t s);
// One (center, context) pair with a host-evaluated sigmoid: phase 0 writes the L dots
// into buf, phase 1 reads the L sigmoid values from buf and applies the updates.
void launch_det_pair(const DetModel& m, int32_t center, int32_t context, float alpha, int phase, float* buf,
                     int32_t* n_acquired, cudaStream_t s);

// ---------------- throughput mode: subsampling + pair generation (K3) ---------
constexpr int kSubTile = 2048;  // tokens per subsampling block (256 threads x 8)

struct SubArgs {
    const int32_t* ids;   // range start
    int64_t n;            // tokens in the range
    int64_t index_base;   // global index of ids[0] (decorrelates ranges/replicas)
    const float* keep;    // [V] or nullptr (keep everything)
    uint64_t key;         // subsampling stream key
    uint32_t* tile_count; // [ntiles]
    uint64_t* tile_off;   // [ntiles + 1]
    int32_t* kept;        // [n] compacted kept ids
    float* sent_alpha;    // [ceil(n / 1000) + 1]
    // alpha schedule
    uint64_t progress_base;
    uint32_t progress_mult;
    uint64_t total_words;
    float alpha0;
};
int64_t sub_tiles(int64_t n);
void launch_subsample(const SubArgs& a, cudaStream_t s, int* launches);

// ---------------- throughput mode: Hogwild training (K1) ----------------------
// The paper's per-worker node cache (NodeCache, trainer.hpp:75-138) becomes a per-CTA
// cache of the top `cache_rows` syn1 rows (device rows [0, cache_rows): the
// CacheSelection's rows lead the device row order), held in two tiers:
//   * rows [0, smem_rows): deltas in shared memory, merged under per-row locks;
//   * rows [smem_rows, cache_rows): deltas in a CTA-private slice of `tier2` (global
//     memory, L2-resident for moderate K), merged with red.global.add and drained with
//     an atomic exchange.
// A warp reads a cached row as the base row plus its CTA's pending delta. Every
// `flush_centers` merged centers the CTA drains the rows it touched into syn1, scaled
// per row (row_scale: summing the deltas of rows few CTAs touch, averaging the CTA
// replicas of rows many CTAs touch).
struct HogArgs {
    float* syn0;               // [V * Dp]
    float* syn1;               // [V * Dp]: V-1 rows in device order + one all-zero pad row
    int32_t d4;                // Dp / 4 (row stride in float4)
    const int32_t* path_off;   // [V+1]
    const int32_t* path_code;  // (row << 1) | turn
    const int32_t* kept;
    const uint64_t* n_kept_dev;  // device scalar written by the subsample kernels
    const float* sent_alpha;
    const float* sigmoid;      // [1000]
    float sig_scale;
    int32_t window;
    uint64_t win_key;
    int32_t cache_rows;        // K: syn1 rows [0, K) cached per CTA (both tiers)
    int32_t smem_rows;         // S <= K: rows [0, S) in shared memory
    float* tier2;              // [blocks][K - S][Dp] pending deltas of rows [S, K); all zero between launches
    int32_t ctx_cache_rows;    // syn0 rows [0, K0) -- the most frequent words -- cached per CTA too
    int32_t centers_per_warp;
    float hot_flush_scale;     // multiplier on cached deltas at flush (if row_scale == nullptr)
    const float* row_scale;    // per cached row flush multiplier (syn1 rows [0, K), then syn0 rows), or nullptr
    int32_t flush_centers;     // centers merged into a CTA's cache between flushes
    int32_t dummy_row;         // the all-zero syn1 pad row
    int32_t ctx_batch;         // context rows staged per warp (<= 2 * window)
    int32_t flusher;           // 1 = the block's last warp is a cache flusher (set by the launcher)
    int32_t urows;             // v8: path rows staged per chunk
    int32_t smem_stride;       // v8: shared-memory row stride (halves)
    unsigned long long* counters;  // [0] tile ticket, [1] pairs, [2] steps, [3] centers
};
struct HogGeometry {
    int warps;        // worker warps per block
    int blocks;       // grid
    int cpw;          // centers per ticket
    int cache_rows;   // K (both tiers)
    int smem_rows;    // S
    int ctx_batch;    // contexts staged per warp (v8: min(16, 2W) rows of the 16-row tile)
    int variant;      // 8 = v8 (tensor cores); 1..3 = v5 (FP32, float4 chunks per lane); 0 = generic
    bool specialise;  // use the row-width-specialised instantiation when there is one
    bool flusher;     // one extra (flusher) warp; only when registers leave room for it
    int ctx_rows;     // cached syn0 rows (most frequent context words)
    int urows;        // v8: path rows staged per chunk
    int smem_stride;  // v8: shared-memory row stride (halves)
    size_t smem;
};
// Most frequent words whose syn0 rows K1 caches per CTA (averaged at flush, like the hot
// syn1 rows): thousands of warps otherwise add stale updates to them at once.
constexpr int kCtxCacheRows = 16;
// Longest Huffman path the row-group kernel stages per warp; deeper trees (and rows
// wider than 384 floats) train on the generic kernel.
constexpr int kMaxGroupDepth = 64;
// Upper bound on the cached rows per CTA (touched-row bitmap in shared memory).
constexpr int kMaxCacheRows = 16384;
// Warps per CTA the registers allow for this row width / depth.
int hog_max_warps(int d4, int max_depth);
// Picks the kernel variant and the launch geometry for the device. smem_rows < 0 = default.
HogGeometry hog_plan(int d4, int max_depth, int cache_rows, int smem_rows, int blocks_override, int warps_override,
                     int cpw_override, int window, int64_t tokens, int ctx_rows);
void launch_hogwild(const HogArgs& a, const HogGeometry& g, cudaStream_t s);
// K1 v8 (cg_hog8.cu), the default: each center's products on the tensor cores (mma.sync
// m16n8k16 f16, fp32 accumulation) from fp16-staged rows. Returns false where it does not
// apply (rows wider than 384 floats, or no warp fits).
bool hog8_plan(int d4, int cache_rows, int ctx_rows, int blocks, int warps_override, int cpw_override, int64_t tokens,
               int max_depth, int window, HogGeometry* g);
void launch_hog8(const HogArgs& a, const HogGeometry& g, cudaStream_t s);

// ---------------- evaluation (cg_eval.cu) -----------------------------------------
// Row stride of a normalised table: dim rounded up to the scoring kernels' k-chunk.
int eval_ld(int dim);
// dst[r] = src[r] / sqrtf(dot(src[r], src[r])) (zeros unless the norm is > 0), rows padded to ld.
void launch_normalize(const float* src, int64_t src_ld, float* dst, int ld, int64_t rows, int dim, cudaStream_t s);
// 3CosAdd answers of nq questions abc[3*q..] over the first nw rows of N; T [nq*ld] and
// best [nq] are scratch.
void launch_analogy(const float* N, int ld, int dim, int64_t nw, const int32_t* abc, int64_t nq, float* T,
                    unsigned long long* best, int32_t* out, cudaStream_t s);
// Cosine top-k (k <= 32) of rows qidx[0..nq) against rows [0, nw), self excluded.
void launch_topk(const float* N, int ld, int64_t nw, const int32_t* qidx, int64_t nq, int k, int32_t* ids,
                 float* scores, cudaStream_t s);

// ---------------- corpus ingest (cg_ingest.cu) ------------------------------------
struct TokChunk {
    const unsigned char* bytes;
    int64_t n;
    uint64_t global_offset;  // byte offset of bytes[0] in the file
};
// Vocabulary word -> id, open addressing (linear probing) on FNV-1a 64 hashes.
struct WordTableDev {
    const unsigned long long* keys;
    const int32_t* ids;
    const int64_t* off;
    const int32_t* len;
    const char* pool;
    uint64_t mask;
};
struct WordTableHost {
    std::vector<unsigned long long> keys;
    std::vector<int32_t> ids;
    std::vector<int64_t> off;
    std::vector<int32_t> len;
    std::vector<char> pool;
    uint64_t mask = 0;
    void build(const std::vector<std::string>& words);
};
struct CountTableDev {
    unsigned long long* keys;
    unsigned long long* count;
    unsigned long long* first;  // byte offset of the first occurrence
    unsigned long long* off;    // word bytes in pool
    int32_t* len;
    char* pool;
    uint64_t pool_capacity;
    unsigned long long* pool_cursor;
    unsigned long long* distinct;
    unsigned long long* overflow;
    uint64_t mask;
};
struct CountEntry {
    unsigned long long count, first, off;
    int32_t len, pad;
};
struct CountedWord {
    std::string word;
    int64_t count;
    uint64_t first;
};
struct IngestStats {
    uint64_t bytes = 0;
    double seconds = 0.0;
    int32_t launches = 0;
};
unsigned long long host_token_hash(const char* s, size_t len);
// Tokenises a corpus file on the device; in-vocabulary ids are written in file order to
// out[0..capacity) (device). Returns the number of in-vocabulary tokens (which may exceed
// capacity: then only the first `capacity` were written).
// Per-chunk progress: after chunk j is queued, the number of ids written so far is copied
// (asynchronously) into the pinned host word word(ctx, j) provided by the receiver, and
// on_chunk(ctx, j, ev) hands over an event that completes after that copy (the receiver
// destroys it).
struct IngestProgress {
    uint64_t* (*word)(void* ctx, int chunk);
    void (*on_chunk)(void* ctx, int chunk, cudaEvent_t ev);
    void* ctx;
};
int64_t ingest_ids(const char* path, const WordTableDev& table, int32_t* out, uint64_t capacity, cudaStream_t st,
                   IngestStats* stats, const IngestProgress* progress = nullptr);
// Counts every distinct token of a corpus file on the device (unordered).
std::vector<CountedWord> ingest_count(const char* path, cudaStream_t st, IngestStats* stats);

}  // namespace cgk
