// cg_hogwild.cu -- throughput mode: K3 subsampling/compaction and K1 Hogwild training.
//
// K3 (subsample): for every id-stream token, keep it iff keep_prob >= 1 or a counter-based
//   splitmix64 draw (same mixer as rng.hpp:17-22, keyed by (seed, pass, token index)) is
//   below keep_prob -- the reference's rule at trainer.hpp:229-232 with the same draw
//   distribution. Kept ids are compacted in stream order; the kept stream is cut into
//   1000-token sentences exactly like trainer.hpp:219-234, and each sentence gets the
//   learning rate the reference would hold after filling it (trainer.hpp:223-228).
//
// K1 (hogwild): persistent CTAs; worker warps pull chunks of consecutive kept centers
//   from a global ticket counter and train each one (train_center, trainer.hpp:147-175):
//   window b = W - draw % W inside the center's 1000-token sentence, the center's
//   root-first path. One warp of every CTA is the cache flusher.
//   * Rows are 128-bit vectors, lanes own float4 chunks. The dot products of all path
//     steps of one pair are independent (distinct rows, fixed context row), so they are
//     reduced together with a warp transpose-reduce.
//   * Hot rows -- the CacheSelection's top nodes, limited to the kernel's private-prefix
//     depth HMAX -- are the per-CTA cache (the paper's per-worker cache, NodeCache
//     trainer.hpp:75-138): a warp copies its center's hot prefix into registers, trains
//     all pairs of the center on that private copy, and merges the delta into the CTA's
//     shared-memory cache under a per-row lock. The flusher warp drains the cache into
//     syn1 with red.global.add.v4 every `flush_centers` merged centers, scaled by
//     1/n_CTA (model averaging of the CTA replicas, see cg_capi.cu), then fences so this
//     SM's stale L1 copies of the hot rows are dropped.
//   * Every other row is read L2-coherent (ld.global.cg) and updated with
//     red.global.add.v4 (no lost updates) or, optionally, plain stores (the reference's
//     lossy Hogwild, trainer.hpp:249-253).
#include <algorithm>
#include <cstdint>

#include "cg_device.cuh"
#include "cg_kernels.h"


#ifndef CG_W2
#define CG_W2 12  // warps per CTA the D <= 256 variant is compiled for (experiments: tools/ab_build.py)
#endif

namespace cgk {
namespace {

using namespace cgdev;

// ----------------------------------------------------------------------------- K3
constexpr int kSubThreads = 256;
constexpr int kSubPer = kSubTile / kSubThreads;  // 8 tokens per thread, strided

__device__ __forceinline__ bool keep_token(const SubArgs& a, int64_t t, int32_t& id) {
    id = a.ids[t];
    if (!a.keep) return true;
    const float kp = a.keep[id];
    return kp >= 1.0f || unit24(ctr_draw(a.key, static_cast<uint64_t>(a.index_base + t))) < kp;
}

__global__ void __launch_bounds__(kSubThreads) sub_count_kernel(SubArgs a) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kSubTile;
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < kSubPer; ++i) {
        const int64_t t = base + i * kSubThreads + threadIdx.x;
        int32_t id;
        if (t < a.n && keep_token(a, t, id)) ++cnt;
    }
    __shared__ int ws[kSubThreads / 32];
    cnt = __reduce_add_sync(kFull, cnt);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < kSubThreads / 32; ++w) s += ws[w];
        a.tile_count[blockIdx.x] = static_cast<uint32_t>(s);
    }
}

// Single-block exclusive scan of the tile counts; tile_off[ntiles] = total kept.
__global__ void __launch_bounds__(1024) sub_scan_kernel(const uint32_t* cnt, uint64_t* off, int64_t ntiles) {
    __shared__ uint64_t part[1024];
    const int64_t per = (ntiles + 1023) / 1024;
    const int64_t b = threadIdx.x * per, e = min(b + per, ntiles);
    uint64_t s = 0;
    for (int64_t i = b; i < e; ++i) s += cnt[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
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

__device__ __forceinline__ float sentence_alpha(const SubArgs& a, int64_t tokens_read) {
    const uint64_t raw = a.progress_base + static_cast<uint64_t>(a.progress_mult) * static_cast<uint64_t>(tokens_read);
    const uint64_t done = raw / kAlphaBatch * kAlphaBatch;
    return update_alpha(done, a.total_words, a.alpha0);
}

__global__ void __launch_bounds__(kSubThreads) sub_scatter_kernel(SubArgs a) {
    __shared__ int ws[kSubThreads / 32];
    __shared__ int wbase[kSubThreads / 32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kSubTile;
    const uint64_t total = a.tile_off[gridDim.x];
    uint64_t run = a.tile_off[blockIdx.x];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = 0; i < kSubPer; ++i) {
        const int64_t t = base + i * kSubThreads + threadIdx.x;
        int32_t id = 0;
        const bool k = t < a.n && keep_token(a, t, id);
        const unsigned m = __ballot_sync(kFull, k);
        if (lane == 0) ws[w] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int q = 0; q < kSubThreads / 32; ++q) { wbase[q] = s; s += ws[q]; }
            ws[0] = s;  // reuse slot 0 for the round total after wbase is read below
        }
        __syncthreads();
        if (k) {
            const uint64_t r = run + static_cast<uint64_t>(wbase[w] + __popc(m & ((1u << lane) - 1u)));
            a.kept[r] = id;
            // sentence s = r / 1000 closes at its 1000th kept token, or at stream end
            if (r % kSentence == kSentence - 1) a.sent_alpha[r / kSentence] = sentence_alpha(a, t + 1);
            if (r == total - 1 && r % kSentence != kSentence - 1) a.sent_alpha[r / kSentence] = sentence_alpha(a, a.n);
        }
        const int round_total = ws[0];
        __syncthreads();
        run += static_cast<uint64_t>(round_total);
    }
}

// ----------------------------------------------------------------------------- K1
constexpr int kCodeSlots = 80;  // per-warp path codes: L <= 64 plus group padding

// Worker warps train centers; warp `workers` (the last one) is the cache flusher.
//
// Per center the warp runs "row-major": every path row is loaded once, trained against
// all of the center's contexts in order (the row's own update sequence is exactly the
// reference's), and written back with a single delta. G rows are processed together
// (their dot products reduce in one transpose-reduce); the contexts' rows and their
// hidden-layer accumulators h live in a per-warp shared-memory buffer.
template <int DCH, int G, int WORKERS>
__global__ void __launch_bounds__((WORKERS + 1) * 32, 1) hog_kernel(HogArgs a) {
    constexpr int LGG = Log2<G>::v;
    extern __shared__ float4 hsm[];
    float* sig = reinterpret_cast<float*>(hsm);                      // 1024 floats
    int* codes_all = reinterpret_cast<int*>(hsm + 256);              // WORKERS * kCodeSlots
    float4* dblk = hsm + 256 + WORKERS * (kCodeSlots / 4);           // cache_rows * d4
    const int K = a.cache_rows;
    const int d4 = a.d4;
    int* locks = reinterpret_cast<int*>(dblk + K * d4);
    float4* ctx_all = reinterpret_cast<float4*>(locks + ((K + 3) & ~3));  // WORKERS * 2 * NB * d4
    const int NB = a.ctx_batch;
    __shared__ int s_done;
    __shared__ unsigned s_merged;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int workers = (blockDim.x >> 5) - 1;
    for (int i = tid; i < 1000; i += blockDim.x) sig[i] = a.sigmoid[i];
    for (int i = tid; i < K * d4; i += blockDim.x) dblk[i] = f4(0.f);
    for (int i = tid; i < K; i += blockDim.x) locks[i] = 0;
    if (tid == 0) {
        s_done = 0;
        s_merged = 0;
    }
    __syncthreads();

    if (warp == workers) {
        // ---- flusher: drain the block cache into syn1 (scaled), row by row under the
        // row locks, whenever enough centers were merged; never blocks the workers.
        unsigned last = 0;
        for (;;) {
            const bool done = *reinterpret_cast<volatile int*>(&s_done) == workers;
            const unsigned merged = *reinterpret_cast<volatile unsigned*>(&s_merged);
            if (K > 0 && (done || merged - last >= static_cast<unsigned>(a.flush_centers))) {
                last = merged;
                for (int r = 0; r < K; ++r) {
                    if (lane == 0)
                        while (atomicCAS(&locks[r], 0, 1) != 0) {
                        }
                    __syncwarp();
                    __threadfence_block();
                    float4 d[DCH];
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        d[k] = f4(0.f);
                        if (q < d4) {
                            d[k] = dblk[r * d4 + q];
                            dblk[r * d4 + q] = f4(0.f);
                        }
                    }
                    __threadfence_block();
                    __syncwarp();
                    if (lane == 0) atomicExch(&locks[r], 0);
                    const float sc = a.row_scale ? a.row_scale[r] : a.hot_flush_scale;
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (q < d4 && nonzero4(d[k])) red_add4(a.syn1 + 4 * (r * d4 + q), scale4(sc, d[k]));
                    }
                }
                __threadfence();  // publish the flush; also drops this SM's stale L1 lines of hot rows
            }
            if (done) break;
            __nanosleep(2000);
        }
        return;
    }

    // ---- workers
    int* codes = codes_all + warp * kCodeSlots;
    float4* V = ctx_all + static_cast<size_t>(warp) * 2 * NB * d4;  // context rows
    float4* Hs = V + NB * d4;                                        // their h accumulators
    const int dummy_code = a.dummy_row << 1;
    const int64_t n_kept = static_cast<int64_t>(*a.n_kept_dev);
    const int cpw = a.centers_per_warp;
    unsigned long long n_pairs = 0, n_steps = 0, n_centers = 0;

    for (;;) {
        long long c0 = 0;
        if (lane == 0) c0 = static_cast<long long>(atomicAdd(a.counters, static_cast<unsigned long long>(cpw)));
        c0 = __shfl_sync(kFull, c0, 0);
        if (c0 >= n_kept) break;
        const int64_t cend = min(static_cast<int64_t>(c0) + cpw, n_kept);
        for (int64_t ci = c0; ci < cend; ++ci) {
            const int32_t c = a.kept[ci];
            const int64_t s_lo = ci / kSentence * kSentence;
            const int64_t s_hi = min(s_lo + kSentence, n_kept);
            const float alpha = a.sent_alpha[ci / kSentence];
            const int b = a.window - static_cast<int>(ctr_draw(a.win_key, static_cast<uint64_t>(ci)) %
                                                      static_cast<uint64_t>(a.window));
            const int64_t lo = max(s_lo, ci - b), hi = min(s_hi - 1, ci + b);
            ++n_centers;
            const int n = static_cast<int>(hi - lo);  // contexts (the center itself excluded)
            if (n == 0) continue;
            const int p0 = a.path_off[c];
            const int L = a.path_off[c + 1] - p0;
            __syncwarp();
            for (int j = lane; j < kCodeSlots; j += 32) codes[j] = j < L ? a.path_code[p0 + j] : dummy_code;
            bool touched_cache = false;

            for (int q0 = 0; q0 < n; q0 += NB) {
                const int nb = min(NB, n - q0);
                // stage this batch of context rows; h accumulators start at 0
                for (int i = 0; i < nb; ++i) {
                    int64_t pos = lo + q0 + i;
                    pos += pos >= ci;  // skip the center's own position
                    const int xo = a.kept[pos] * d4;
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (q < d4) {
                            V[i * d4 + q] = ld_cg4(a.syn0 + 4 * (xo + q));
                            Hs[i * d4 + q] = f4(0.f);
                        }
                    }
                }
                __syncwarp();
                for (int j0 = 0; j0 < L; j0 += G) {
                    float4 U[G][DCH], S[G][DCH];
                    int row[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        row[g] = codes[j0 + g] >> 1;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            float4 u = f4(0.f);
                            if (q < d4) {
                                const int e = row[g] * d4 + q;
                                u = row[g] < K ? add4(ld_ca4(a.syn1 + 4 * e), dblk[e]) : ld_cg4(a.syn1 + 4 * e);
                            }
                            U[g][k] = u;
                            S[g][k] = u;
                        }
                    }
                    const int jl = j0 + (lane >> (5 - LGG));
                    const float turn = static_cast<float>(codes[jl] & 1);
                    const bool jl_live = jl < L;
                    for (int i = 0; i < nb; ++i) {
                        float4 v[DCH];
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            v[k] = q < d4 ? V[i * d4 + q] : f4(0.f);
                        }
                        float p[G];
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            float acc = 0.f;
#pragma unroll
                            for (int k = 0; k < DCH; ++k) acc = dot4(v[k], U[g][k], acc);
                            p[g] = acc;
                        }
                        const float tot = transpose_reduce<G>(p, lane);
                        const float f = table_sigmoid(sig, tot, a.sig_scale);
                        const float gl = jl_live ? (1.0f - turn - f) * alpha : 0.f;
                        float4 hacc[DCH];
#pragma unroll
                        for (int k = 0; k < DCH; ++k) hacc[k] = f4(0.f);
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const float gg = __shfl_sync(kFull, gl, g << (5 - LGG));
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                hacc[k] = axpy4(gg, U[g][k], hacc[k]);
                                U[g][k] = axpy4(gg, v[k], U[g][k]);
                            }
                        }
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            if (q < d4) Hs[i * d4 + q] = add4(Hs[i * d4 + q], hacc[k]);
                        }
                    }
                    // write back each row's delta once: block cache (locked) or HBM (red)
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (j0 + g >= L) continue;
                        if (row[g] < K) {
                            touched_cache = true;
                            if (lane == 0)
                                while (atomicCAS(&locks[row[g]], 0, 1) != 0) {
                                }
                            __syncwarp();
                            __threadfence_block();
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (q < d4) {
                                    const int e = row[g] * d4 + q;
                                    dblk[e] = add4(dblk[e], make_float4(U[g][k].x - S[g][k].x, U[g][k].y - S[g][k].y,
                                                                        U[g][k].z - S[g][k].z, U[g][k].w - S[g][k].w));
                                }
                            }
                            __threadfence_block();
                            __syncwarp();
                            if (lane == 0) atomicExch(&locks[row[g]], 0);
                        } else if (!(a.probe & 1)) {
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (q < d4)
                                    red_add4(a.syn1 + 4 * (row[g] * d4 + q),
                                             make_float4(U[g][k].x - S[g][k].x, U[g][k].y - S[g][k].y,
                                                         U[g][k].z - S[g][k].z, U[g][k].w - S[g][k].w));
                            }
                        }
                    }
                }
                __syncwarp();
                // the contexts' rows move once, by their accumulated h (trainer.hpp:173)
                if (!(a.probe & 2)) {
                    for (int i = 0; i < nb; ++i) {
                        int64_t pos = lo + q0 + i;
                        pos += pos >= ci;
                        const int xo = a.kept[pos] * d4;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            if (q < d4) red_add4(a.syn0 + 4 * (xo + q), Hs[i * d4 + q]);
                        }
                    }
                }
                __syncwarp();
            }
            n_pairs += static_cast<unsigned long long>(n);
            n_steps += static_cast<unsigned long long>(n) * static_cast<unsigned long long>(L);
            if (lane == 0 && touched_cache) atomicAdd(&s_merged, 1u);
        }
    }
    if (lane == 0) {  // counts are warp-uniform
        atomicAdd(a.counters + 1, n_pairs);
        atomicAdd(a.counters + 2, n_steps);
        atomicAdd(a.counters + 3, n_centers);
        atomicAdd(&s_done, 1);
    }
}

// ---- K1 v4: center-batched row groups ---------------------------------------------
// Lane q = lane + 32 k of chunk k is inside a row of d4 float4: chunks k < DCH - 1 always
// are (the variant is DCH = ceil(d4 / 32)), so only the last chunk needs the predicate.
template <int DCH>
__device__ __forceinline__ bool in_row(int k, int q, int d4) {
    return k < DCH - 1 || q < d4;
}

// Learning signals of CIc contexts (cc .., clamped to the batch) against the G rows in U:
// the CIc*G dot products are reduced together (transpose-reduce), after which the pair
// (ii, g) lives in lane (ii*G + g) << (5 - log2(CIc*G)); that lane evaluates the pair's
// g = (1 - turn - sigmoid(dot)) * alpha (0 for a padded context / row) and stores it at
// sg[ii*G + g], so the update loop fetches a context's G signals with one broadcast load.
template <int DCH, int G, int CIc>
__device__ __forceinline__ void chunk_signal(const float4* V, int d4, int lane, int cc, int nb,
                                             const float4 (&U)[G][DCH], const int* codes, int j0, int L,
                                             const float* sig, float sig_scale, float alpha, float* sg) {
    constexpr int N = CIc * G;
    constexpr int LN = Log2<N>::v, LGG = Log2<G>::v, LS = 5 - LN;
    float p[N];
#pragma unroll
    for (int ii = 0; ii < CIc; ++ii) {
        const int i = min(cc + ii, nb - 1);
        // Lanes past the row end read the neighbouring (finite: the region is zeroed at
        // launch and only ever holds model values) shared-memory data; their U chunk is 0,
        // so they add exact zeros to the reduction. No per-element selects.
        float4 v[DCH];
#pragma unroll
        for (int k = 0; k < DCH; ++k) v[k] = V[i * d4 + lane + 32 * k];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < DCH; ++k) acc = dot4(v[k], U[g][k], acc);
            p[ii * G + g] = acc;
        }
    }
    const float tot = transpose_reduce<N>(p, lane);
    const int vi = lane >> LS;
    const int my_i = vi >> LGG, my_g = vi & (G - 1);
    const int code = codes[j0 + my_g];
    const float f = table_sigmoid(sig, tot, sig_scale);
    const float gl = (j0 + my_g < L && cc + my_i < nb) ? (1.0f - static_cast<float>(code & 1) - f) * alpha : 0.f;
    __syncwarp();  // every lane has read the previous chunk's signals
    if ((lane & ((1 << LS) - 1)) == 0) sg[vi] = gl;
    __syncwarp();
}

// Same persistent/ticket/flusher structure, smem layout and hot-row cache protocol as
// hog_kernel. The difference is the per-row-group schedule: every context of a batch
// takes its dot products against the group's rows as they were loaded (the row state at
// the start of this center's group; within-center staleness of at most 2W updates, far
// below the hot-row cache's own flush delay of ~64 centers), so the L x n dot products
// of a center are independent. They are computed CI = 32/G contexts at a time and
// reduced with one 32-value transpose-reduce (lane k ends up holding dot (k / G, k % G)),
// each lane evaluates one sigmoid, and the updates (h_i += g U, delta += g v) follow as
// pure FMA streams. This removes v3's serial dot -> reduce -> sigmoid -> update chain per
// (context, group), the latency that held issue at ~46% with 12 warps per SM.
// Cache flushes: when the registers leave room for a warp that shared memory cannot feed
// as a worker (C2, D 300), that warp is a dedicated flusher, polling the merge count;
// otherwise (C1, C3: registers are the limit) the worker whose merge completes a batch
// of `flush_centers` merged centers drains the cache itself, and its warp slot is one
// more worker. The last worker to finish drains the cache once more. The polling
// flusher spends ~5% of the issued instructions (__nanosleep returns almost at once;
// sleeping in mbarrier.try_wait measured slower), but inline flushes on the workers'
// path cost more than that where the flusher warp is free (C2 +1.7%, C5 +3.5%).
// D4 > 0 specialises the kernel for rows of exactly D4 float4 (the dims of the benchmark
// configurations): every shared-memory and row offset becomes an immediate and the
// last-chunk predicate a constant lane bound. D4 = 0 takes the row width at run time.
// CTX: the most frequent words' syn0 rows are cached per CTA too (only instantiated into
// the launch when some word's expected concurrent updaters pass the threshold in
// cg_capi.cu; the code is compiled out otherwise, where it measured 3-4% slower).
template <int DCH, int G, int WORKERS, int D4 = 0, bool CTX = false>
__global__ void __launch_bounds__(WORKERS * 32, 1) hog4_kernel(HogArgs a) {
    // WORKERS: warps per block the registers allow (workers, plus the flusher if any)
    static_assert(G == 4, "signals are fetched as one float4 per context");
    static_assert(D4 == 0 || (D4 > 32 * (DCH - 1) && D4 <= 32 * DCH), "D4 must belong to the variant");
    extern __shared__ float4 hsm[];
    float* sig = reinterpret_cast<float*>(hsm);
    int* codes_all = reinterpret_cast<int*>(hsm + 256);
    // The hot-row cache and the context/prefetch rows start on 128-byte boundaries (with
    // 32-byte rows, every staged row is then 32-byte aligned): staging at 16 mod 32 bytes
    // made K1 ~30% slower (profiles/r1_smem_align.jsonl).
    auto align128 = [](float4* p) {
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(p));
        return p + ((128u - (sa & 127u)) & 127u) / 16u;
    };
    float4* dblk = align128(hsm + 256 + WORKERS * (kCodeSlots / 4));
    const int K = a.cache_rows;
    const int d4 = D4 > 0 ? D4 : a.d4;
    int* locks = reinterpret_cast<int*>(dblk + K * d4);
    // the CTA's pending deltas of the most frequent words' syn0 rows (context rows)
    const int K0 = CTX ? a.ctx_cache_rows : 0;
    float4* dblk0 = align128(reinterpret_cast<float4*>(locks + ((K + 3) & ~3)));
    int* locks0 = reinterpret_cast<int*>(dblk0 + K0 * d4);
    float4* ctx_all = align128(reinterpret_cast<float4*>(locks0 + ((K0 + 3) & ~3)));
    const int NB = a.ctx_batch;
    __shared__ int s_done;
    __shared__ unsigned s_merged;
    __shared__ float4 s_sig[WORKERS * 8];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int workers = (blockDim.x >> 5) - a.flusher;
    for (int i = tid; i < 1000; i += blockDim.x) sig[i] = a.sigmoid[i];
    for (int i = tid; i < K * d4; i += blockDim.x) dblk[i] = f4(0.f);
    for (int i = tid; i < K; i += blockDim.x) locks[i] = 0;
    for (int i = tid; i < K0 * d4; i += blockDim.x) dblk0[i] = f4(0.f);
    for (int i = tid; i < K0; i += blockDim.x) locks0[i] = 0;
    {  // context, h and prefetch buffers: zeroed once so out-of-row reads are finite
        const int n4 = workers * (2 * NB + G) * d4;  // exactly the ctx + prefetch allocation
        for (int i = tid; i < n4; i += blockDim.x) ctx_all[i] = f4(0.f);
    }
    if (tid == 0) {
        s_done = 0;
        s_merged = 0;
    }
    __syncthreads();

    // Drain every cached row's delta into syn1 (whole warp): row by row under its lock,
    // scaled per row (averaging of the CTA replicas, see cg_capi.cu), then a fence so
    // the other SMs see the update before this CTA's next flush.
    auto drain_rows = [&](float4* cache, int* lk, int n, float* dst, int scale_base) {
        for (int r = 0; r < n; ++r) {
            if (lane == 0)
                while (atomicCAS(&lk[r], 0, 1) != 0) {
                }
            __syncwarp();
            __threadfence_block();
            float4 d[DCH];
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                d[k] = f4(0.f);
                if (in_row<DCH>(k, q, d4)) {
                    d[k] = cache[r * d4 + q];
                    cache[r * d4 + q] = f4(0.f);
                }
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) atomicExch(&lk[r], 0);
            const float sc = a.row_scale ? a.row_scale[scale_base + r] : a.hot_flush_scale;
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                if (in_row<DCH>(k, q, d4) && nonzero4(d[k])) red_add4(dst + 4 * (r * d4 + q), scale4(sc, d[k]));
            }
        }
    };
    auto flush_cache = [&]() {
        drain_rows(dblk, locks, K, a.syn1, 0);
        if constexpr (CTX) drain_rows(dblk0, locks0, K0, a.syn0, K);
    };

    // Flusher warp: blocked in hardware on named barrier 1 (bar.sync, 64 threads) until a
    // worker warp whose merge completed a batch of flush_centers arrives on it (bar.arrive,
    // non-blocking). Arrivals while the flusher is busy count toward its next wait, so no
    // request is lost; two of them may complete a phase on their own, which only delays
    // one flush. The last worker sets s_done before its final arrival, and the flusher
    // checks s_done before every wait, so it always ends with a flush after all merges.
    if (warp == workers) {
        if (K == 0 && K0 == 0) return;
        for (;;) {
            if (*reinterpret_cast<volatile int*>(&s_done) == workers) {
                flush_cache();
                break;
            }
            named_bar_sync(1, 64);
            flush_cache();
            __threadfence();
        }
        return;
    }

    int* codes = codes_all + warp * kCodeSlots;
    float* sg = reinterpret_cast<float*>(s_sig + warp * 8);
    float4* V = ctx_all + static_cast<size_t>(warp) * 2 * NB * d4;
    float4* Hs = V + NB * d4;
    // per-warp staging of the next row group (cp.async one group ahead of its use)
    float4* Ub = ctx_all + static_cast<size_t>(workers) * 2 * NB * d4 + static_cast<size_t>(warp) * G * d4;
    auto prefetch_group = [&](int j0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int rg = codes[j0 + g] >> 1;
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                if (in_row<DCH>(k, q, d4)) cp_async16(Ub + g * d4 + q, a.syn1 + 4 * (rg * d4 + q));
            }
        }
    };
    const int dummy_code = a.dummy_row << 1;
    const int64_t n_kept = static_cast<int64_t>(*a.n_kept_dev);
    const int cpw = a.centers_per_warp;
    const bool cache_reads = !(a.probe & 8), cold_writes = !(a.probe & 1), ctx_writes = !(a.probe & 2);
    unsigned long long n_pairs = 0, n_steps = 0, n_centers = 0;

    for (;;) {
        long long c0 = 0;
        if (lane == 0) c0 = static_cast<long long>(atomicAdd(a.counters, static_cast<unsigned long long>(cpw)));
        c0 = __shfl_sync(kFull, c0, 0);
        if (c0 >= n_kept) break;
        const int64_t cend = min(static_cast<int64_t>(c0) + cpw, n_kept);
        // the ticket's per-center metadata in two coalesced dependent loads (lane j: center
        // c0 + j) instead of a kept -> path_off chain per center
        int t_p0 = 0, t_len = 0;
        float t_alpha = 0.f;
        if (c0 + lane < cend) {
            const int32_t cj = a.kept[c0 + lane];
            t_alpha = a.sent_alpha[(c0 + lane) / kSentence];
            t_p0 = a.path_off[cj];
            t_len = a.path_off[cj + 1] - t_p0;
        }
        for (int64_t ci = c0; ci < cend; ++ci) {
            const int jt = static_cast<int>(ci - c0);
            const int64_t s_lo = ci / kSentence * kSentence;
            const int64_t s_hi = min(s_lo + kSentence, n_kept);
            const float alpha = __shfl_sync(kFull, t_alpha, jt);
            const int p0 = __shfl_sync(kFull, t_p0, jt);
            const int L = __shfl_sync(kFull, t_len, jt);
            // shrink_window (trainer.hpp:66-68): b = W - draw mod W, with the draw reduced by
            // a 32x32 multiply-high of its top bits (uniform to within W / 2^32; the 64-bit
            // modulo was a ~60-instruction call per center)
            const int b = a.window - static_cast<int>(__umulhi(static_cast<unsigned>(ctr_draw(a.win_key, static_cast<uint64_t>(ci)) >> 32),
                                                               static_cast<unsigned>(a.window)));
            const int64_t lo = max(s_lo, ci - b), hi = min(s_hi - 1, ci + b);
            ++n_centers;
            const int n = static_cast<int>(hi - lo);
            if (n == 0) continue;
            __syncwarp();
            for (int j = lane; j < kCodeSlots; j += 32) codes[j] = j < L ? a.path_code[p0 + j] : dummy_code;
            bool touched_cache = false;

            for (int q0 = 0; q0 < n; q0 += NB) {
                const int nb = min(NB, n - q0);
                // context ids in one coalesced load (lane i: context i), then every row copy
                // of the batch in flight at once (cp.async, no registers held)
                int xid = 0;
                if (lane < nb) {
                    int64_t pos = lo + q0 + lane;
                    pos += pos >= ci;  // skip the center's own position
                    xid = a.kept[pos];
                }
                // contexts whose syn0 row is in the CTA cache (word ids are in count order)
                unsigned hot_ctx = 0;
                if constexpr (CTX) hot_ctx = __ballot_sync(kFull, lane < nb && xid < K0);
                __syncwarp();  // codes visible; Ub free
                prefetch_group(0);
                for (int i = 0; i < nb; ++i) {
                    const int xo = __shfl_sync(kFull, xid, i) * d4;
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (in_row<DCH>(k, q, d4)) {
                            cp_async16(V + i * d4 + q, a.syn0 + 4 * (xo + q));
                            Hs[i * d4 + q] = f4(0.f);
                        }
                    }
                }
                for (int j0 = 0; j0 < L; j0 += G) {
                    cp_async_wait_all();  // this group's rows (and, first time, the contexts)
                    __syncwarp();
                    if (CTX && j0 == 0 && hot_ctx) {  // + this CTA's cached delta of hot context rows
                        for (unsigned m = hot_ctx; m; m &= m - 1) {
                            const int i = __ffs(m) - 1;
                            const int x = __shfl_sync(kFull, xid, i);
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) V[i * d4 + q] = add4(V[i * d4 + q], dblk0[x * d4 + q]);
                            }
                        }
                        __syncwarp();
                    }
                    float4 U[G][DCH], Dl[G][DCH];
                    int row[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        row[g] = codes[j0 + g] >> 1;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            U[g][k] = in_row<DCH>(k, q, d4) ? Ub[g * d4 + q] : f4(0.f);
                            Dl[g][k] = f4(0.f);
                        }
                    }
                    // + this CTA's cached delta; row[g] is warp-uniform, so is the branch
                    if (cache_reads) {
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            if (row[g] < K) {
#pragma unroll
                                for (int k = 0; k < DCH; ++k) {
                                    const int q = lane + 32 * k;
                                    if (in_row<DCH>(k, q, d4)) U[g][k] = add4(U[g][k], dblk[row[g] * d4 + q]);
                                }
                            }
                        }
                    }
                    __syncwarp();  // every lane has its copy: Ub takes the next group
                    if (j0 + G < L) prefetch_group(j0 + G);
                    for (int cc = 0; cc < nb;) {
                        // chunk of 8, 4 or 2 contexts: a center's 2b contexts (b = 1..W) are
                        // covered without computing dots for padding (a fixed 8 wasted ~40%)
                        const int r = nb - cc;
                        constexpr int CIM = 32 / G;  // contexts per full chunk (CIM * G = 32 dots)
                        int cic;
                        if (r >= CIM) {
                            chunk_signal<DCH, G, CIM>(V, d4, lane, cc, nb, U, codes, j0, L, sig, a.sig_scale, alpha, sg);
                            cic = CIM;
                        } else if (r >= CIM / 2) {
                            chunk_signal<DCH, G, CIM / 2>(V, d4, lane, cc, nb, U, codes, j0, L, sig, a.sig_scale, alpha,
                                                          sg);
                            cic = CIM / 2;
                        } else {
                            chunk_signal<DCH, G, CIM / 4>(V, d4, lane, cc, nb, U, codes, j0, L, sig, a.sig_scale, alpha,
                                                          sg);
                            cic = CIM / 4;
                        }
                        // Rolled: unrolled (fully or 2x), the kernel's hot loop
                        // outgrows the instruction cache or the registers (ncu: 21%
                        // no_instruction stalls fully unrolled; 2x: +11% K1 time at D 300).
                        // Lanes past the row end compute on neighbouring data; their hacc
                        // and delta chunks are never written back.
                        const int ni = min(cic, r);
                        if constexpr (DCH < 3) {
#pragma unroll 1
                        for (int ii = 0; ii < ni; ++ii) {
                            const int i = cc + ii;
                            // h accumulates in place: load Hs[i] up front (with v) so the
                            // loads overlap and the FMAs add straight into it
                            float4 v[DCH], hacc[DCH];
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                v[k] = V[i * d4 + lane + 32 * k];
                                hacc[k] = Hs[i * d4 + lane + 32 * k];
                            }
                            // one broadcast load instead of G shuffles: C2 K1 92.2 -> 90.3 ms
                            const float4 g4 = reinterpret_cast<const float4*>(sg)[ii];
                            const float gg[G] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                            for (int g = 0; g < G; ++g) {
#pragma unroll
                                for (int k = 0; k < DCH; ++k) {
                                    hacc[k] = axpy4(gg[g], U[g][k], hacc[k]);
                                    Dl[g][k] = axpy4(gg[g], v[k], Dl[g][k]);
                                }
                            }
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) Hs[i * d4 + q] = hacc[k];
                            }
                        }
                        } else {
                        const float4* sg4 = reinterpret_cast<const float4*>(sg);
                        // D > 256: software-pipelined. The next context's v and signals
                        // are loaded while this one's FMAs run, and the Dl FMAs go first so
                        // the h row loaded at the top arrives before its FMAs (C4 1287 ->
                        // 1241 ms; at D <= 256 it measured slower: C2 72.8 -> 75.6 ms).
                        float4 vn[DCH];
#pragma unroll
                        for (int k = 0; k < DCH; ++k) vn[k] = V[cc * d4 + lane + 32 * k];
                        float4 gn = sg4[0];
#pragma unroll 1
                        for (int ii = 0; ii < ni; ++ii) {
                            const int i = cc + ii;
                            float4 v[DCH], hacc[DCH];
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                v[k] = vn[k];
                                hacc[k] = Hs[i * d4 + lane + 32 * k];
                            }
                            const float gg[G] = {gn.x, gn.y, gn.z, gn.w};
                            const int in = min(ii + 1, ni - 1);
#pragma unroll
                            for (int k = 0; k < DCH; ++k) vn[k] = V[(cc + in) * d4 + lane + 32 * k];
                            gn = sg4[in];
#pragma unroll
                            for (int g = 0; g < G; ++g) {
#pragma unroll
                                for (int k = 0; k < DCH; ++k) Dl[g][k] = axpy4(gg[g], v[k], Dl[g][k]);
                            }
#pragma unroll
                            for (int g = 0; g < G; ++g) {
#pragma unroll
                                for (int k = 0; k < DCH; ++k) hacc[k] = axpy4(gg[g], U[g][k], hacc[k]);
                            }
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) Hs[i * d4 + q] = hacc[k];
                            }
                        }
                        }
                        cc += cic;
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (j0 + g >= L) continue;
                        if (row[g] < K) {
                            touched_cache = true;
                            if (lane == 0)
                                while (atomicCAS(&locks[row[g]], 0, 1) != 0) {
                                }
                            __syncwarp();
                            __threadfence_block();
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) {
                                    const int e = row[g] * d4 + q;
                                    dblk[e] = add4(dblk[e], Dl[g][k]);
                                }
                            }
                            __threadfence_block();
                            __syncwarp();
                            if (lane == 0) atomicExch(&locks[row[g]], 0);
                        } else if (cold_writes) {
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) red_add4(a.syn1 + 4 * (row[g] * d4 + q), Dl[g][k]);
                            }
                        }
                    }
                }
                __syncwarp();
                if (ctx_writes) {
                    for (int i = 0; i < nb; ++i) {
                        const int x = __shfl_sync(kFull, xid, i);
                        if (CTX && ((hot_ctx >> i) & 1u)) {  // merge into the CTA's cached delta
                            touched_cache = true;
                            if (lane == 0)
                                while (atomicCAS(&locks0[x], 0, 1) != 0) {
                                }
                            __syncwarp();
                            __threadfence_block();
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) dblk0[x * d4 + q] = add4(dblk0[x * d4 + q], Hs[i * d4 + q]);
                            }
                            __threadfence_block();
                            __syncwarp();
                            if (lane == 0) atomicExch(&locks0[x], 0);
                            continue;
                        }
                        const int xo = x * d4;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            if (in_row<DCH>(k, q, d4)) red_add4(a.syn0 + 4 * (xo + q), Hs[i * d4 + q]);
                        }
                    }
                }
                __syncwarp();
            }
            n_pairs += static_cast<unsigned long long>(n);
            n_steps += static_cast<unsigned long long>(n) * static_cast<unsigned long long>(L);
            if (touched_cache) {
                unsigned m = 0;
                if (lane == 0) m = atomicAdd(&s_merged, 1u) + 1u;
                m = __shfl_sync(kFull, m, 0);
                if (m % static_cast<unsigned>(a.flush_centers) == 0u) {
                    if (a.flusher) {
                        __syncwarp();
                        named_bar_arrive(1, 64);
                    } else {
                        flush_cache();
                    }
                }
            }
        }
    }
    int last = 0;
    if (lane == 0) {
        atomicAdd(a.counters + 1, n_pairs);
        atomicAdd(a.counters + 2, n_steps);
        atomicAdd(a.counters + 3, n_centers);
        __threadfence_block();  // this warp's merges before its done count
        last = atomicAdd(&s_done, 1) == workers - 1;
    }
    last = __shfl_sync(kFull, last, 0);
    if (a.flusher && last && (K > 0 || K0 > 0)) {  // wake the flusher for its final flush
        __threadfence_block();
        named_bar_arrive(1, 64);
        return;
    }
    // without a flusher warp, the last worker to finish drains what the others merged
    // after their last flush
    if (!a.flusher && last && (K > 0 || K0 > 0)) {
        __threadfence_block();
        flush_cache();
    }
}

// v4 rows per group and worker warps per CTA. G = 8 measured worse: for D <= 128 (C1 K1
// 3.66 -> 4.48 ms, 11 workers: ptxas budgets registers for a multiple of 4 warps, so 13
// workers would get 128 and spill) and for D <= 256 (C2 90 -> 124 ms, 7 workers); G = 2
// with 15 workers (128 registers, context batch 7) is also slower at C2 (116 ms).
template <int DCH>
constexpr int kG4 = 4;
template <int DCH>
constexpr int kW4 = DCH == 1 ? 16 : (DCH == 2 ? CG_W2 : 8);

// Row widths with a specialised K1 (D = 100, 128, 200, 300: the benchmark configurations,
// rows padded to 32 bytes).
template <int DCH, bool CTX>
auto hog4_for(int d4, bool specialise) -> decltype(&hog4_kernel<DCH, kG4<DCH>, kW4<DCH>, 0, CTX>) {
    if (specialise) {
        if constexpr (DCH == 1) {
            if (d4 == 26) return hog4_kernel<1, kG4<1>, kW4<1>, 26, CTX>;
            if (d4 == 32) return hog4_kernel<1, kG4<1>, kW4<1>, 32, CTX>;
        } else if constexpr (DCH == 2) {
            if (d4 == 50) return hog4_kernel<2, kG4<2>, kW4<2>, 50, CTX>;
        } else if constexpr (DCH == 3) {
            if (d4 == 76) return hog4_kernel<3, kG4<3>, kW4<3>, 76, CTX>;
        }
    }
    return hog4_kernel<DCH, kG4<DCH>, kW4<DCH>, 0, CTX>;
}

template <int DCH, int G, int WORKERS>
void launch_variant(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    void (*k)(HogArgs) = g.kernel == 3 ? hog_kernel<DCH, G, WORKERS>
                         : (g.ctx_rows > 0 ? hog4_for<DCH, true>(a.d4, g.specialise) : hog4_for<DCH, false>(a.d4, g.specialise));
    // always opt in: dynamic + static shared memory above 48 KB needs it even when the
    // dynamic part alone is below (a launch without it failed with "invalid argument")
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
    HogArgs b = a;
    b.cache_rows = g.cache_rows;
    b.centers_per_warp = g.cpw;
    b.ctx_batch = g.ctx_batch;
    b.flusher = g.flusher ? 1 : 0;
    k<<<g.blocks, (g.warps + (g.kernel == 3 || g.flusher ? 1 : 0)) * 32, g.smem, s>>>(b);  // + flusher warp
}

// Per-variant shape: float4 chunks per lane (DCH), rows trained together (G) and worker
// warps (the register budget of the launch bounds).
template <int DCH>
struct Variant;
template <>
struct Variant<1> {
    static constexpr int G = 8, WORKERS = 15;
};
template <>
struct Variant<2> {
    static constexpr int G = 4, WORKERS = 11;
};
template <>
struct Variant<3> {
    static constexpr int G = 4, WORKERS = 7;
};

}  // namespace

int64_t sub_tiles(int64_t n) { return (n + kSubTile - 1) / kSubTile; }

void launch_subsample(const SubArgs& a, cudaStream_t s, int* launches) {
    const int64_t nt = sub_tiles(a.n);
    if (nt == 0) {
        cudaMemsetAsync(a.tile_off, 0, sizeof(uint64_t), s);
        if (launches) *launches = 0;
        return;
    }
    sub_count_kernel<<<static_cast<unsigned>(nt), kSubThreads, 0, s>>>(a);
    sub_scan_kernel<<<1, 1024, 0, s>>>(a.tile_count, a.tile_off, nt);
    sub_scatter_kernel<<<static_cast<unsigned>(nt), kSubThreads, 0, s>>>(a);
    if (launches) *launches = 3;
}

// Every hot row can be cached (row-major processing has no private-prefix depth limit).
int hog_hmax(int) { return 1 << 30; }

int hog_max_warps(int d4) {
    const int v = (d4 + 31) / 32;
    return v == 1 ? kW4<1> : (v == 2 ? kW4<2> : kW4<3>);
}

HogGeometry hog_plan(int d4, int cache_rows_wanted, int blocks_override, int warps_override, int cpw_override,
                     int rows_override, int window, int kernel, int64_t tokens, int ctx_rows) {
    HogGeometry g{};
    g.kernel = kernel == 3 ? 3 : 4;
    g.specialise = true;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g.variant = (d4 + 31) / 32;
    const int workers = g.kernel == 4
                            ? (g.variant == 1 ? kW4<1> : (g.variant == 2 ? kW4<2> : kW4<3>))
                            : (g.variant == 1 ? Variant<1>::WORKERS : (g.variant == 2 ? Variant<2>::WORKERS : Variant<3>::WORKERS));
    g.warps = warps_override > 0 ? std::min(warps_override, workers) : workers;
    g.blocks = blocks_override > 0 ? blocks_override : sms;
    g.cpw = std::min(cpw_override > 0 ? cpw_override : 4, 32);  // <= 32: a ticket's metadata is one lane each
    // shared memory: sigmoid table | path codes | hot-row cache (+locks) | context buffers
    const size_t fixed = 4096 + static_cast<size_t>(workers) * kCodeSlots * 4 + 14 * 16;
    const size_t per_row = static_cast<size_t>(d4) * 16 + 4;
    int rows = std::min(cache_rows_wanted, static_cast<int>((48 * 1024) / per_row));
    if (rows_override >= 0 && rows_override < rows) rows = rows_override;
    g.cache_rows = std::max(rows, 0);
    g.ctx_rows = g.kernel == 4 ? std::max(ctx_rows, 0) : 0;
    const size_t cache_bytes = static_cast<size_t>(g.cache_rows) * d4 * 16 + static_cast<size_t>((g.cache_rows + 3) & ~3) * 4 +
                               static_cast<size_t>(g.ctx_rows) * d4 * 16 + static_cast<size_t>((g.ctx_rows + 3) & ~3) * 4 + 128;
    // v4 also stages each warp's next row group (4 rows) in shared memory. A center whose
    // 2b contexts do not fit one context batch re-reads (and re-writes) its whole path per
    // batch: unless the caller fixed the warp count, drop one warp if that lets one batch
    // hold a full window (2W contexts). Dropping more measured slower (C4, W 10: 4 warps
    // x batch 20 took 1577 ms, 7 warps x batch 10 1322 ms).
    const size_t budget = 227 * 1024 - 4096;  // dynamic shared memory; static (signals, counters) <= 4 KB
    auto batch_for = [&](int warps, size_t* smem) {
        const int g4 = g.variant == 1 ? kG4<1> : (g.variant == 2 ? kG4<2> : kG4<3>);
        const size_t prefetch = g.kernel == 4 ? static_cast<size_t>(warps) * g4 * d4 * 16 : 0;
        const size_t per_ctx = static_cast<size_t>(warps) * 2 * d4 * 16;
        const size_t room = budget > fixed + cache_bytes + prefetch ? budget - fixed - cache_bytes - prefetch : 0;
        int nb = static_cast<int>(std::min<size_t>(2 * static_cast<size_t>(window), room / per_ctx));
        nb = std::min(std::max(nb, 1), 32);  // one context id per lane
        *smem = fixed + cache_bytes + prefetch + static_cast<size_t>(nb) * per_ctx;
        return nb;
    };
    g.ctx_batch = batch_for(g.warps, &g.smem);
    if (warps_override <= 0 && g.ctx_batch < 2 * window) {
        for (int w = g.warps - 1; w >= std::max(1, g.warps - 1); --w) {
            size_t sm = 0;
            const int nb = batch_for(w, &sm);
            if (nb >= 2 * window) {
                g.warps = w;
                g.ctx_batch = nb;
                g.smem = sm;
                break;
            }
        }
    }
    // Centers per ticket: 16 when every warp gets >= 2000 tokens (fewer ticket atomics and
    // metadata loads: C2 -1%, C3 -1.2%, C5 -1.4% vs 4), else 8 (the tail of a small pass
    // grows with the ticket: C1 3.33 ms at 8, 3.44 at 32).
    if (cpw_override <= 0) g.cpw = tokens / (static_cast<int64_t>(g.blocks) * g.warps) >= 2000 ? 16 : 8;
    // a warp the registers allow but shared memory cannot feed becomes the cache flusher
    g.flusher = g.kernel == 4 && g.warps < workers && (g.cache_rows > 0 || g.ctx_rows > 0);
    return g;
}

void launch_hogwild(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    switch (g.variant) {
        case 1: launch_variant<1, Variant<1>::G, Variant<1>::WORKERS>(a, g, s); break;
        case 2: launch_variant<2, Variant<2>::G, Variant<2>::WORKERS>(a, g, s); break;
        default: launch_variant<3, Variant<3>::G, Variant<3>::WORKERS>(a, g, s); break;
    }
}

}  // namespace cgk
