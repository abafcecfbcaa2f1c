/*
 * cachegram_b200.h -- the C-ABI of libcachegram_b200.so.
 *
 * This is the drop-in boundary for the reference's hot path, cachegram::train()
 * (/root/reference/proj/include/cachegram/trainer.hpp:254-316). Plain C types only:
 * pointers, sizes and status codes; no C++ or torch types cross it. The C++ API in
 * include/cachegram/trainer.hpp (same names as the reference) and the Python package
 * (ctypes) are both thin layers over these entry points; INTEGRATION.md shows the
 * binding a maintainer of the reference would add.
 *
 * Status codes map onto the reference's exceptions (trainer.hpp:37-47, 256-260;
 * corpus.hpp:194,232; errors.hpp:12-24): CG_ERR_INVALID_ARGUMENT -> std::invalid_argument,
 * CG_ERR_IO -> IoError, CG_ERR_PARSE -> ParseError, CG_ERR_NO_TRAINABLE_WORDS -> NoTrainableWords, the rest ->
 * std::runtime_error. The message is in cg_last_error() (thread-local).
 *
 * Everything that computes on the training path runs on the GPU; there is no CPU
 * fallback. Without a usable CUDA device the training entry points return CG_ERR_CUDA.
 */
#ifndef CACHEGRAM_B200_H
#define CACHEGRAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CG_ABI_VERSION 3  /* 3: two-tier per-CTA cache honouring K and u; cg_tuning without experiment bits */

/* The library is built with -fvisibility=hidden; only these entry points are exported. */
#if defined(__GNUC__)
#define CG_API __attribute__((visibility("default")))
#else
#define CG_API
#endif

enum cg_status {
    CG_OK = 0,
    CG_ERR_INVALID_ARGUMENT = 1,
    CG_ERR_IO = 2,
    CG_ERR_CUDA = 3,
    CG_ERR_NCCL = 4,
    CG_ERR_NO_TRAINABLE_WORDS = 5,
    CG_ERR_INTERNAL = 6,
    CG_ERR_PARSE = 7 /* a model or question file violates its format -> ParseError */
};

/* Training modes. DETERMINISTIC replays the reference's single-worker stream
 * (trainer.hpp:200-245 with workers == 1: same RNG draws, same sentence chunks, same
 * node-cache flush points, sequential non-fused fp32 arithmetic) on one warp and is
 * bit-identical to the reference. HOGWILD is the throughput path: device-side
 * subsampling and pair generation, thousands of warps updating one device-resident
 * model lock-free, with a per-block shared-memory cache of the hot inner-node rows. */
enum cg_mode { CG_MODE_HOGWILD = 0, CG_MODE_DETERMINISTIC = 1 };

/* Mirrors cachegram::TrainConfig (trainer.hpp:25-35), field for field. */
typedef struct cg_config {
    int32_t dim;
    int32_t window;
    int64_t min_count;
    double sample;
    float alpha0;
    int32_t iterations;
    int32_t workers;        /* reference CPU thread count; the GPU path ignores it */
    int32_t cache_nodes;    /* K: the paper's node cache (trainer.hpp:33). HOGWILD: every CTA caches the K
                               CacheSelection rows -- the hottest (default 8) in shared memory, the
                               rest as CTA-private delta rows in L2 -- plus the stability floor
                               (cg_tuning.min_cache_rows). Flushes add each row's delta scaled by
                               1 / E[#CTAs contributing per flush period]: rows few CTAs touch are
                               summed as in the reference, the CTA replicas of hot rows are
                               averaged. cg_epoch_stats reports the rows cached. */
    int32_t flush_interval; /* u, in trained centers per worker (trainer.hpp:34, 127). HOGWILD: a CTA's
                               cache is drained every u x (its worker warps) merged centers. */
    uint64_t seed;
} cg_config;

/* What train() receives besides the corpus: Vocabulary counts, the HuffmanTree paths
 * (root-first CSR, huffman.hpp:30-52) and the CacheSelection (huffman.hpp:116-134). */
typedef struct cg_model_desc {
    int32_t vocab_size;          /* V >= 2 */
    const int64_t* counts;       /* [V]   Vocabulary::count, ids in vocabulary order */
    int64_t total_tokens;        /* Vocabulary::total_tokens */
    const int64_t* path_offsets; /* [V+1] */
    const int32_t* path_nodes;   /* [path_offsets[V]] inner node ids 0..V-2 */
    const uint8_t* path_turns;   /* [path_offsets[V]] 0/1 */
    const int64_t* node_usage;   /* [V-1] HuffmanTree::node_usage */
    const int32_t* hot_nodes;    /* [hot_count] CacheSelection slot order; may be NULL if hot_count == 0 */
    int32_t hot_count;           /* CacheSelection::size() = min(K, V-1) */
} cg_model_desc;

typedef struct cg_train_stats {
    uint64_t words_processed; /* in-vocabulary tokens read, all iterations (trainer.hpp:178) */
    double wall_seconds;      /* host wall time of the training loop (trainer.hpp:280-307) */
    double words_per_second;
    double kernel_seconds;    /* summed device time of the training kernels (CUDA events) */
    uint64_t centers;         /* kept centers trained */
    uint64_t pairs;           /* (center, context) pairs trained */
    uint64_t steps;           /* pair x path-step updates */
} cg_train_stats;

/* ---- library --------------------------------------------------------------- */
CG_API int cg_abi_version(void);
CG_API const char* cg_last_error(void);
/* Device buffers are pooled across calls (cg_train, sessions); this returns the cached,
 * currently unused ones to the driver. */
CG_API void cg_release_cached_memory(void);
/* Number of visible CUDA devices (0 when none); never falls back. */
CG_API int cg_device_count(void);

/* ---- host pieces of the path (reference algorithms, C-ABI for FFI callers) ---- */
/* corpus.hpp:176-181 */
CG_API double cg_keep_probability(int64_t count, int64_t total_tokens, double sample);
/* trainer.hpp:58-63 */
CG_API float cg_update_alpha(uint64_t words_processed, uint64_t total_words, float alpha0);
/* model.hpp:84-91: out[1000] */
CG_API void cg_sigmoid_table(float* out);
/* model.hpp:66-72: syn0 [V*D] (syn1 is all zeros) */
CG_API int cg_init_model(int32_t vocab_size, int32_t dim, uint64_t seed, float* syn0);
/* huffman.hpp:57-108. Two calls: with path_nodes == NULL only *n_steps is written. */
CG_API int cg_build_huffman(const int64_t* counts, int32_t vocab_size, int64_t* path_offsets, int32_t* path_nodes,
                     uint8_t* path_turns, int64_t* node_usage, int64_t* n_steps);
/* huffman.hpp:139-159. Returns the selection size, or -1 (see cg_last_error). */
CG_API int32_t cg_select_cached_nodes(const int64_t* node_usage, int32_t inner_count, int32_t k, int32_t* hot_nodes,
                               int32_t* slot_of);
/* corpus.hpp:136-170 + trainer.hpp:220-222: vocabulary of a corpus file, then the file as an
 * in-vocabulary id stream. Two-phase: cg_corpus_open -> query/export -> cg_corpus_close. */
typedef struct cg_corpus cg_corpus;
CG_API int cg_corpus_open(const char* path, int64_t min_count, cg_corpus** out);
CG_API int32_t cg_corpus_vocab_size(const cg_corpus* c);
CG_API int64_t cg_corpus_total_tokens(const cg_corpus* c);
CG_API int64_t cg_corpus_word_bytes(const cg_corpus* c); /* sum of word lengths + V (NUL separators) */
CG_API int cg_corpus_export_vocab(const cg_corpus* c, int64_t* counts, char* words_nul_separated);
CG_API int cg_corpus_read_ids(const cg_corpus* c, const char* path, int32_t* ids, int64_t capacity, int64_t* n_ids);
CG_API void cg_corpus_close(cg_corpus* c);

/* ---- the hot path: cachegram::train() (trainer.hpp:254-316) -------------------
 * Host buffers in, host buffers out. `ids` is the in-vocabulary id stream of the corpus
 * (cg_corpus_read_ids). The model starts from init_model(V, dim, seed) exactly as the
 * reference's train() does (trainer.hpp:262). syn0_out [V*dim] and syn1_out [(V-1)*dim]
 * receive the trained matrices in reference layout and node order. Blocking. */
CG_API int cg_train(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const int32_t* ids, int64_t n_ids,
             float* syn0_out, float* syn1_out, cg_train_stats* stats);

/* ---- kernel-level entry: one train_center() call (trainer.hpp:147-175) ---------
 * Runs the deterministic device kernel for a single center on host buffers, with the
 * NodeCache (trainer.hpp:75-138) state passed explicitly: cache_work/cache_snap
 * [hot_count*dim], cache_flag [hot_count] (1 = acquired). slot_of [V-1] may be NULL
 * when hot_count == 0. sigmoid_mode: 0 = SigmoidTable, 1 = exact logistic,
 * 2 = the constant sig_const. *sigmoid_calls receives the number of evaluations. */
CG_API int cg_train_center(int32_t center, const int32_t* sentence, int64_t sentence_len, int64_t center_pos,
                    int32_t half_window, int32_t vocab_size, int32_t dim, float* syn0, float* syn1,
                    const int64_t* path_offsets, const int32_t* path_nodes, const uint8_t* path_turns,
                    const int32_t* slot_of, int32_t hot_count, float* cache_work, float* cache_snap,
                    uint8_t* cache_flag, float alpha, int32_t sigmoid_mode, float sig_const, int64_t* sigmoid_calls);
/* train_center with an arbitrary host sigmoid functor (the reference's SigmoidFn template
 * parameter, e.g. its tests' counting lambdas): per pair the device computes the L exact
 * dot products, fn maps each through the sigmoid on the host (in path order, one call
 * per step like the reference), and the device applies the updates. Same cache contract
 * as cg_train_center. */
typedef float (*cg_sigmoid_fn)(float x, void* ctx);
CG_API int cg_train_center_cb(int32_t center, const int32_t* sentence, int64_t sentence_len, int64_t center_pos,
                              int32_t half_window, int32_t vocab_size, int32_t dim, float* syn0, float* syn1,
                              const int64_t* path_offsets, const int32_t* path_nodes, const uint8_t* path_turns,
                              const int32_t* slot_of, int32_t hot_count, float* cache_work, float* cache_snap,
                              uint8_t* cache_flag, float alpha, cg_sigmoid_fn fn, void* ctx, int64_t* sigmoid_calls);
/* NodeCache::flush (trainer.hpp:110-124) on the device: syn1[hot_nodes[s]] += work - snap
 * for every acquired slot, then clears the flags. */
CG_API int cg_cache_flush(int32_t vocab_size, int32_t dim, float* syn1, const int32_t* hot_nodes, int32_t hot_count,
                   float* cache_work, const float* cache_snap, uint8_t* cache_flag);

/* ---- sessions: device-resident training for benchmarks and multi-GPU -----------
 * A session owns the device copies of the tree, the hot-row selection, the keep
 * probabilities, the id stream and the model (one buffer: syn0 rows then syn1 rows,
 * rows padded to a multiple of 4 floats, syn1 rows in usage-rank order). */
typedef struct cg_session cg_session;

typedef struct cg_epoch_stats {
    uint64_t words;          /* id-stream tokens covered by this call */
    uint64_t kept;           /* centers after subsampling */
    uint64_t pairs;
    uint64_t steps;
    double train_ms;         /* device time of the training kernel(s) */
    double subsample_ms;     /* device time of subsampling + compaction */
    int32_t train_launches;  /* kernels launched by this call */
    int32_t other_launches;
    int32_t cached_rows;     /* hogwild: syn1 rows cached per CTA (both tiers) = max(K, floor_rows) */
    int32_t worker_warps;    /* hogwild: worker warps per CTA */
    int32_t ctx_batch;       /* hogwild: contexts staged per batch */
    int32_t blocks;          /* hogwild: persistent CTAs */
    int32_t smem_rows;       /* hogwild: of cached_rows, those held in shared memory (the rest: L2 tier) */
    int32_t floor_rows;      /* hogwild: the stability floor of this launch (0 when disabled) */
    int32_t flush_centers;   /* hogwild: merged centers per CTA between flushes (u x worker warps) */
    int32_t kernel;          /* hogwild: K1 version run (8, 5; 0 = the generic kernel) */
} cg_epoch_stats;

/* stream: a cudaStream_t (NULL = legacy default stream). device: CUDA ordinal. */
CG_API int cg_session_create(const cg_config* cfg, int32_t mode, const cg_model_desc* model, int32_t device, void* stream,
                      cg_session** out);
CG_API void cg_session_destroy(cg_session* s);
/* Copies the host id stream into device memory owned by the session. */
CG_API int cg_session_upload_ids(cg_session* s, const int32_t* ids, int64_t n_ids);
/* Same from a device buffer (device-to-device copy; ids must already be valid). */
CG_API int cg_session_upload_ids_device(cg_session* s, const int32_t* device_ids, int64_t n_ids);
/* (Re)initialises the model on the device side from init_model(V, dim, seed). */
CG_API int cg_session_reset_model(cg_session* s);
/* Uploads a model given in reference layout (host). */
CG_API int cg_session_set_model(cg_session* s, const float* syn0, const float* syn1);
/* One training pass over ids[tok_begin, tok_end). The learning rate follows
 * update_alpha(progress, iterations * total_tokens) with
 * progress = progress_base + progress_mult * (tokens read in this range so far),
 * i.e. progress_mult = N replicas estimate the global counter.
 * `epoch` decorrelates the counter-based draws of successive passes. Blocking. */
CG_API int cg_session_train_range(cg_session* s, int32_t epoch, int64_t tok_begin, int64_t tok_end, uint64_t progress_base,
                           uint32_t progress_mult, cg_epoch_stats* stats);
/* Whole-run convenience: config.iterations passes over the uploaded ids. */
CG_API int cg_session_train(cg_session* s, cg_train_stats* stats);
CG_API int cg_session_download(cg_session* s, float* syn0_out, float* syn1_out);
/* The device model buffer (for an all-reduce between replicas) and its geometry. */
CG_API int cg_session_model_buffer(cg_session* s, void** device_ptr, size_t* bytes, int32_t* row_stride_floats);
/* ---- replica sync: one model replica per GPU, deltas summed -------------
 * The reference's workers all add into one model (trainer.hpp:72-74, 249-253). Replicas
 * keep that semantics between syncs: each replica trains its shard from the model of the
 * last sync (the snapshot); at a sync every replica's delta (model - snapshot) is summed
 * over the replicas (cg_session_sync_delta exposes it for an NCCL all-reduce with SUM) and
 * applied to the snapshot row by row (cg_session_sync_apply) with the scale
 *     s(row) = min(prior, max(ratio, trust)),
 *     prior = cg_sync_row_scale(q, n, centers),
 *     ratio = clamp(sum_r |delta_r|^2 / |sum_r delta_r|^2, 1/n, 1),
 *     trust = min(1, 0.25 / (rms norm of the other matrix's 1024 hottest rows x |sum_r delta_r|)):
 * the ratio is 1 (the reference's plain sum) for a row one replica touched or whose replicas
 * moved it in orthogonal directions and 1/n (their average) when every replica made the same
 * move from the same snapshot; a summed step small enough to move the row's logits by less
 * than ~0.25 is kept whole (n stale trajectories then add up like one sequential one). */
/* snapshot = model: the start of a sync period (after reset/set_model, before training). */
CG_API int cg_session_sync_begin(cg_session* s);
/* delta = model - snapshot, in a session-owned device buffer of n_floats: the model's layout
 * followed by one squared norm per model row (|delta_r|^2, padded to a multiple of 4
 * floats) and 4 floats holding the squared norms of the syn0 and the syn1 matrix. All-reduce
 * all n_floats with SUM. */
CG_API int cg_session_sync_delta(cg_session* s, void** delta_dev, size_t* n_floats);
/* With the delta buffer holding the sum over n_replicas replicas: model = snapshot +
 * s(row) x delta, snapshot = model. words_per_replica: id-stream tokens each replica
 * trained since the last sync (the sync interval; it sets the prior below). */
CG_API int cg_session_sync_apply(cg_session* s, int32_t n_replicas, uint64_t words_per_replica);
/* The prior of the per-row scale from expected update counts, for a row on a share q of
 * the updates, n_replicas replicas of `centers` kept centers each per sync:
 * min(1, max(1 / (p n), 128 / (n q centers))) with p = 1 - (1 - q)^centers -- 1 for rows few
 * replicas touch, at most 128 stale updates' worth and at least the replicas' average for a
 * row every replica updates. Host-only arithmetic (no device needed). */
CG_API float cg_sync_row_scale(double q, int32_t n_replicas, double centers);

/* Hogwild kernel knobs (zero-initialised = defaults, except smem_cache_rows: -1). */
typedef struct cg_tuning {
    int32_t blocks;           /* 0 = one persistent CTA per SM */
    int32_t warps_per_block;  /* 0 = the variant's maximum */
    int32_t centers_per_warp; /* 0 = auto: consecutive kept centers per work ticket (16, or 8 for small passes) */
    int32_t smem_cache_rows;  /* < 0 = 8: how many of the cached rows live in shared memory (capped at 48 KB of
                                 rows); the others are CTA-private delta rows in L2 */
    float hot_flush_scale;    /* 0 = per-row 1/E[#CTAs contributing per flush] (averaging of overlapping
                                 CTA replicas); > 0 = this multiplier for every cached row */
    int32_t flush_centers;    /* 0 = u x worker warps: merged centers per CTA between flushes */
    int32_t min_cache_rows;   /* the stability floor: 0 = auto, the leading rows whose expected concurrent
                                 updaters (share of paths x warps in flight) reach 256 are cached even when
                                 K is smaller; > 0 = at least this many rows; < 0 = none, K is honoured
                                 literally (K = 0 then diverges on small vocabularies at full-GPU
                                 concurrency) */
    int32_t kernel;           /* 0 = default: v8, each center's products on the tensor cores (mma.sync f16
                                 operands, fp32 accumulation), for D <= 384; 5 = v5, FP32 FMA arithmetic
                                 (packed FFMA2) with a shared-memory tier for the hottest cached rows.
                                 Rows wider than 384 floats train on the generic FP32 kernel. */
} cg_tuning;
CG_API int cg_session_tune(cg_session* s, const cg_tuning* t);

/* ---- corpus ingest on the GPU -----------------------------
 * The corpus file is streamed through pinned buffers into HBM and tokenised there
 * (the reference's separators, corpus.hpp:19-21). cg_corpus_open_gpu counts every
 * distinct token on the device and orders the vocabulary exactly like
 * build_vocabulary_file (count descending, first occurrence on ties); the same handle
 * works with cg_corpus_* above. cg_corpus_read_ids_gpu / cg_session_load_corpus turn a
 * file into the in-vocabulary id stream (what ShardReader + id_of yield), the latter
 * straight into a session's device buffer. words_nul: the session's V words, NUL-
 * terminated, in id order. device < 0 = the calling thread's current device. */
CG_API int cg_corpus_open_gpu(const char* path, int64_t min_count, int32_t device, cg_corpus** out);
CG_API int cg_corpus_read_ids_gpu(const cg_corpus* c, const char* path, int32_t device, int32_t* ids,
                                  int64_t capacity, int64_t* n_ids);
CG_API int cg_session_load_corpus(cg_session* s, const char* path, const char* words_nul, int64_t* n_ids);
/* cg_train with the corpus given as a file: tokenised on the device (no host id stream).
 * stats->wall_seconds covers reading the corpus, like the reference's train(). */
CG_API int cg_train_file(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const char* corpus_path,
                         const char* words_nul, float* syn0_out, float* syn1_out, cg_train_stats* stats);

/* ---- in-process replicas: one model replica per GPU -------------------
 * For C/C++ callers that drive several GPUs from one process. Each replica trains a
 * contiguous shard of the id stream (Hogwild mode); every sync_words words per replica the
 * replicas' deltas since the last sync are summed over peer memory (NVLink/NVSwitch:
 * replica r's GPU sums slice r across all replicas and writes it back to all of them) and
 * applied with the per-row sync scale (cg_session_sync_apply). The learning rate follows
 * n_devices x local progress. devices may repeat an ordinal (several replicas on one GPU:
 * functional testing). The result is replica 0's model (all are equal). */
CG_API int cg_train_replicas(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const int32_t* ids,
                             int64_t n_ids, const int32_t* devices, int32_t n_devices, int64_t sync_words,
                             float* syn0_out, float* syn1_out, cg_train_stats* stats);
/* Same with the corpus as a file, tokenised on devices[0] and sharded device to device. */
CG_API int cg_train_file_replicas(const cg_config* cfg, int32_t mode, const cg_model_desc* model,
                                  const char* corpus_path, const char* words_nul, const int32_t* devices,
                                  int32_t n_devices, int64_t sync_words, float* syn0_out, float* syn1_out,
                                  cg_train_stats* stats);
/* In-place average of n (<= 8) equally sized device buffers over peer memory. */
CG_API int cg_average_buffers(void* const* device_bufs, const int32_t* devices, int32_t n, size_t n_floats);

/* ---- evaluation (eval.hpp:88-238) ---------------------------
 * A device-resident table of unit-normalised rows, built exactly like AnalogySolver
 * (eval.hpp:91-103): row / sqrtf(dot(row, row)), zeros when the norm is not > 0.
 * Scores are the reference's sequential fp32 dot, so answers match it bit for bit. */
typedef struct cg_embeddings cg_embeddings;
/* rows = AnalogySolver::vocab_size() = min(V, restrict_top) (first rows of `vectors`).
 * device < 0 selects the calling thread's current CUDA device. */
CG_API int cg_embeddings_create(const float* vectors, int32_t rows, int32_t dim, int32_t device, cg_embeddings** out);
/* Same from device memory (e.g. a session's syn0, row_stride floats apart); no host copy. */
CG_API int cg_embeddings_create_device(const float* device_vectors, int32_t rows, int32_t dim, int32_t row_stride,
                                       int32_t device, cg_embeddings** out);
CG_API void cg_embeddings_destroy(cg_embeddings* e);
CG_API int32_t cg_embeddings_rows(const cg_embeddings* e);
/* The normalised rows (rows x dim, host). */
CG_API int cg_embeddings_normalized(const cg_embeddings* e, float* out);
/* AnalogySolver::answer (eval.hpp:117-136) for n questions: abc = [a0,b0,c0, a1,b1,c1, ...]
 * (ids < rows), best[i] = argmax_w cos(v(b)-v(a)+v(c), v(w)) over w not in {a,b,c}, ties to
 * the lower id, -1 when no candidate is left. */
CG_API int cg_analogy_answer(cg_embeddings* e, const int32_t* abc, int64_t n, int32_t* best);
/* Cosine top-k neighbours (k <= 32) of the query rows, excluding the query's own row,
 * ranked by the same exact scores with ties to the lower id: the recall@k metric of
 * SURVEY 8(d). ids[i*k + r] = -1 (score NaN) when fewer than k candidates exist. */
CG_API int cg_nearest(cg_embeddings* e, const int32_t* queries, int64_t n, int32_t k, int32_t* ids, float* scores);

/* ---- model files (model.hpp:107-276) ---------------------------------------------
 * Text:   "V D\n" then "word v1 ... vD\n" per word, values as " %.6f".
 * Binary: "V D\n" then "word " + D little-endian float32 + "\n" per word.
 * words_nul: the V words, each NUL-terminated, in id order. Text formatting runs on
 * all host cores; the bytes equal the reference's single-threaded fprintf output. */
enum cg_model_format { CG_FORMAT_TEXT = 0, CG_FORMAT_BINARY = 1, CG_FORMAT_AUTO = 2 };
CG_API int cg_model_save(const char* path, int32_t format, const char* words_nul, const float* syn0, int32_t vocab_size,
                         int32_t dim);
/* Two-call load: open parses the file (format AUTO detects it as load_embeddings does),
 * info reports the sizes, export copies words (NUL-separated) and vectors out. */
typedef struct cg_embeddings_file cg_embeddings_file;
CG_API int cg_model_load(const char* path, int32_t format, cg_embeddings_file** out);
CG_API int cg_model_file_info(const cg_embeddings_file* f, int32_t* vocab_size, int32_t* dim, int64_t* word_bytes);
CG_API int cg_model_file_export(const cg_embeddings_file* f, char* words_nul, float* vectors);
CG_API void cg_model_file_close(cg_embeddings_file* f);

#ifdef __cplusplus
}
#endif
#endif
