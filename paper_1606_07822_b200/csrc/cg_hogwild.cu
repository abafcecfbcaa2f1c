// cg_hogwild.cu -- throughput mode: K3 subsampling/compaction and K1 Hogwild training.
//
// K3 (subsample): for every id-stream token, keep it iff keep_prob >= 1 or a counter-based
//   splitmix64 draw (same mixer as rng.hpp:17-22, keyed by (seed, pass, token index)) is
//   below keep_prob -- the reference's rule at trainer.hpp:229-232 with the same draw
//   distribution. Kept ids are compacted in stream order; the kept stream is cut into
//   1000-token sentences exactly like trainer.hpp:219-234, and each sentence gets the
//   learning rate the reference would hold after filling it (trainer.hpp:223-228).
//
// K1 (hogwild): persistent CTAs; worker warps pull tickets of consecutive kept centers
//   from a global counter and train each one (train_center, trainer.hpp:147-175): window
//   b = W - draw % W inside the center's 1000-token sentence, the center's root-first path.
//   * Rows are 128-bit vectors, lanes own float4 chunks; the arithmetic is packed fp32
//     (FFMA2). The dot products of a center's contexts against a group of 4 path rows
//     are independent, so they are reduced together with a warp transpose-reduce.
//   * Rows reach shared memory by bulk copies (cp.async.bulk, the TMA unit) completing on
//     a per-warp mbarrier.
//   * The paper's per-worker cache (NodeCache, trainer.hpp:75-138) is a per-CTA cache of
//     the top K syn1 rows in two tiers (shared memory; CTA-private delta rows in L2),
//     drained into syn1 every flush_centers merged centers with per-row scaling.
//   * Every other row is read through L2 and updated with red.global.add.v4 (no lost
//     updates).
#include <algorithm>
#include <cstdint>

#include "cg_device.cuh"
#include "cg_kernels.h"


#ifndef CG_W2
#define CG_W2 12  // warps per CTA the D <= 256 variant is compiled for (experiments: tools/ab_build.py)
#endif
#ifndef CG_T2_READ
#define CG_T2_READ 0  // 0: warps read the L2-tier cached rows flushed state (write-combining); 1: + their CTA pending delta
#endif
#ifndef CG_H_BULKRED
#define CG_H_BULKRED 1  // 1: a batch's h rows leave shared memory by bulk reductions (TMA unit, UBLKRED); 0: REDG per lane
#endif
#ifndef CG_STAGE_BULK
#define CG_STAGE_BULK 1  // 1: rows staged by bulk copies (TMA unit, UBLKCP); 0: cp.async (LDGSTS)
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
constexpr int kG = 4;           // path rows trained together (one float4 of signals per context)
constexpr int kCodeSlots = 80;  // per-warp path codes: depth <= kMaxGroupDepth plus group padding

// Dynamic shared-memory layout of K1 (byte offsets from a 128-byte aligned base; every
// region starts on a 128-byte boundary, so every staged 32-byte row is 32-byte aligned:
// staging at 16 mod 32 bytes made K1 ~30% slower, profiles/r1_smem_align.jsonl).
struct K1Smem {
    uint32_t codes, mbar, touch, locks, locks0, dblk, dblk0, ctx, ub, total;
};
__host__ __device__ __forceinline__ K1Smem k1_smem(int workers, int S, int K, int K0, int NB, int d4) {
    auto up = [](uint32_t x) { return (x + 127u) & ~127u; };
    K1Smem L{};
    uint32_t o = 4096;  // sigmoid table
    L.codes = o;
    o = up(o + static_cast<uint32_t>(workers) * kCodeSlots * 4);
    L.mbar = o;
    o = up(o + static_cast<uint32_t>(workers) * 8);
    L.touch = o;
    o = up(o + static_cast<uint32_t>((K + 31) / 32) * 4);
    L.locks = o;
    o = up(o + static_cast<uint32_t>(S) * 4);
    L.locks0 = o;
    o = up(o + static_cast<uint32_t>(K0) * 4);
    L.dblk = o;
    o = up(o + static_cast<uint32_t>(S) * d4 * 16);
    L.dblk0 = o;
    o = up(o + static_cast<uint32_t>(K0) * d4 * 16);
    L.ctx = o;
    o = up(o + static_cast<uint32_t>(workers) * 2 * NB * d4 * 16);
    L.ub = o;
    o = up(o + static_cast<uint32_t>(workers) * kG * d4 * 16);
    // Slack: lanes past a row's end read (never write) up to 32 float4 beyond the last
    // staged row, and the base is aligned up by at most 112 bytes.
    L.total = o + 32 * 16 + 128;
    return L;
}

// Lane q = lane + 32 k of chunk k is inside a row of d4 float4: chunks k < DCH - 1 always
// are (the variant is DCH = ceil(d4 / 32)), so only the last chunk needs the predicate.
template <int DCH>
__device__ __forceinline__ bool in_row(int k, int q, int d4) {
    return k < DCH - 1 || q < d4;
}

__device__ __forceinline__ void lock_row(int* lk) {
    while (atomicCAS(lk, 0, 1) != 0) {
    }
}

// Learning signals of CIc contexts (cc .., clamped to the batch) against the G rows in U:
// the CIc*G dot products are reduced together (transpose-reduce), after which the pair
// (ii, g) lives in lane (ii*G + g) << (5 - log2(CIc*G)); that lane evaluates the pair's
// g = (1 - turn - sigmoid(dot)) * alpha (0 for a padded context / row) and stores it at
// sg[ii*G + g], so the update loop fetches a context's G signals with one broadcast load.
// Each lane's partial dots run as two packed sums (FFMA2: even and odd components).
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
        // Lanes past the row end read neighbouring (finite: zeroed at launch, then only
        // model values) shared memory; their U chunk is 0, so they add exact zeros.
        float4 v[DCH];
#pragma unroll
        for (int k = 0; k < DCH; ++k) v[k] = V[i * d4 + lane + 32 * k];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int k = 0; k < DCH; ++k) acc = dot4(v[k], U[g][k], acc);
            p[ii * G + g] = acc.x + acc.y;
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

// K1 v5: persistent CTAs, one warp per center, row-major over the center's path.
//
// Per center the warp stages the center's context rows (syn0) in shared memory, then
// walks the root-first path in groups of G = 4 rows: every context takes its dot products
// against the group's rows as loaded (the CIc x G dots of a chunk reduce together), each
// lane evaluates one sigmoid, and the updates h_i += g U and delta += g v follow as packed
// FMA streams. Each path row is thus loaded once per center and written back once, with
// one delta (within-center staleness <= 2W updates, far below the cache's flush period).
// Rows are copied into shared memory by the TMA unit (cp.async.bulk, one instruction per
// row, completing on the warp's mbarrier), the next group while the current one computes.
//
// WORKERS: warps per block the registers allow (workers, plus the flusher if any).
// D4 > 0 specialises the kernel for rows of exactly D4 float4 (the benchmark dims).
// CTX: the most frequent words' syn0 rows are cached per CTA too (compiled out unless
// some word's expected concurrent updaters pass the threshold in cg_capi.cu).
template <int DCH, int WORKERS, int D4 = 0, bool CTX = false>
__global__ void __launch_bounds__(WORKERS * 32, 1) hog5_kernel(HogArgs a) {
    constexpr int G = kG;
    static_assert(D4 == 0 || (D4 > 32 * (DCH - 1) && D4 <= 32 * DCH), "D4 must belong to the variant");
    extern __shared__ __align__(16) unsigned char k1_raw[];
    unsigned char* base = k1_raw + ((128u - (smem_u32(k1_raw) & 127u)) & 127u);
    const int d4 = D4 > 0 ? D4 : a.d4;
    const int K = a.cache_rows, S = a.smem_rows, K0 = CTX ? a.ctx_cache_rows : 0, NB = a.ctx_batch;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int workers = (blockDim.x >> 5) - a.flusher;
    const K1Smem Ls = k1_smem(workers, S, K, K0, NB, d4);
    float* sig = reinterpret_cast<float*>(base);
    int* codes_all = reinterpret_cast<int*>(base + Ls.codes);
    uint64_t* mbar_all = reinterpret_cast<uint64_t*>(base + Ls.mbar);
    unsigned* touch = reinterpret_cast<unsigned*>(base + Ls.touch);
    int* locks = reinterpret_cast<int*>(base + Ls.locks);
    int* locks0 = reinterpret_cast<int*>(base + Ls.locks0);
    float4* dblk = reinterpret_cast<float4*>(base + Ls.dblk);
    float4* dblk0 = reinterpret_cast<float4*>(base + Ls.dblk0);
    float4* ctx_all = reinterpret_cast<float4*>(base + Ls.ctx);
    float4* ub_all = reinterpret_cast<float4*>(base + Ls.ub);
    const int nwords = (K + 31) >> 5;
    // this CTA's L2-tier delta rows (cached rows [S, K))
    float* t2 = a.tier2 ? a.tier2 + static_cast<size_t>(blockIdx.x) * static_cast<size_t>(K - S) * d4 * 4 : nullptr;
    __shared__ int s_done;
    __shared__ volatile int s_exit;
    __shared__ unsigned s_merged;
    __shared__ float4 s_sig[WORKERS * 8];

    for (int i = tid; i < 1000; i += blockDim.x) sig[i] = a.sigmoid[i];
    for (int i = tid; i < nwords; i += blockDim.x) touch[i] = 0u;
    for (int i = tid; i < S * d4; i += blockDim.x) dblk[i] = f4(0.f);
    for (int i = tid; i < S; i += blockDim.x) locks[i] = 0;
    for (int i = tid; i < K0 * d4; i += blockDim.x) dblk0[i] = f4(0.f);
    for (int i = tid; i < K0; i += blockDim.x) locks0[i] = 0;
    {  // context, h and row-group buffers: zeroed once so out-of-row reads are finite
        float4* z = ctx_all;
        const int n4 = static_cast<int>((Ls.total - 128 - Ls.ctx) / 16);
        for (int i = tid; i < n4; i += blockDim.x) z[i] = f4(0.f);
    }
    if (tid < workers) mbar_init(mbar_all + tid, 1);
    if (tid == 0) {
        s_done = 0;
        s_exit = 0;
        s_merged = 0;
    }
    fence_proxy_async();  // the zeroed staging is overwritten by bulk copies
    __syncthreads();

    // ---- cache drain (whole warp) --------------------------------------------------
    auto drain_syn1_row = [&](int r) {
        float4 d[DCH];
        if (r < S) {
            if (lane == 0) lock_row(&locks[r]);
            __syncwarp();
            __threadfence_block();
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                d[k] = f4(0.f);
                if (in_row<DCH>(k, q, d4)) {
                    d[k] = dblk[r * d4 + q];
                    dblk[r * d4 + q] = f4(0.f);
                }
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) atomicExch(&locks[r], 0);
        } else {
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                d[k] = in_row<DCH>(k, q, d4) ? atom_take4(t2 + (static_cast<size_t>(r - S) * d4 + q) * 4) : f4(0.f);
            }
        }
        const float sc = a.row_scale ? a.row_scale[r] : a.hot_flush_scale;
#pragma unroll
        for (int k = 0; k < DCH; ++k) {
            const int q = lane + 32 * k;
            if (in_row<DCH>(k, q, d4) && nonzero4(d[k]))
                red_add4(a.syn1 + (static_cast<size_t>(r) * d4 + q) * 4, scale4(sc, d[k]));
        }
    };
    auto drain_syn0_rows = [&]() {
        for (int r = 0; r < K0; ++r) {
            if (lane == 0) lock_row(&locks0[r]);
            __syncwarp();
            __threadfence_block();
            float4 d[DCH];
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                d[k] = f4(0.f);
                if (in_row<DCH>(k, q, d4)) {
                    d[k] = dblk0[r * d4 + q];
                    dblk0[r * d4 + q] = f4(0.f);
                }
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) atomicExch(&locks0[r], 0);
            const float sc = a.row_scale ? a.row_scale[K + r] : a.hot_flush_scale;
#pragma unroll
            for (int k = 0; k < DCH; ++k) {
                const int q = lane + 32 * k;
                if (in_row<DCH>(k, q, d4) && nonzero4(d[k]))
                    red_add4(a.syn0 + (static_cast<size_t>(r) * d4 + q) * 4, scale4(sc, d[k]));
            }
        }
    };
    // Drains the rows touched since the last flush (the NodeCache's acquired slots,
    // trainer.hpp:110-124), or every row (`all`: the launch's final flush, which leaves
    // both tiers empty). A merge sets its row's bit after adding its delta, so a delta is
    // either drained now or its bit is set again for the next flush.
    auto flush_cache = [&](bool all) {
        for (int w0 = 0; w0 < nwords; w0 += 32) {
            const int w = w0 + lane;
            unsigned m = 0;
            if (w < nwords) {
                if (all) {
                    m = w == nwords - 1 && (K & 31) ? (1u << (K & 31)) - 1u : ~0u;
                    touch[w] = 0u;
                } else if (touch[w]) {
                    m = atomicExch(&touch[w], 0u);
                }
            }
            for (unsigned live = __ballot_sync(kFull, m != 0); live; live &= live - 1) {
                const int src = __ffs(live) - 1;
                for (unsigned mm = __shfl_sync(kFull, m, src); mm; mm &= mm - 1)
                    drain_syn1_row(((w0 + src) << 5) + __ffs(mm) - 1);
            }
        }
        if constexpr (CTX) drain_syn0_rows();
        __threadfence();  // the other SMs see this flush before the CTA's next one
    };

    // ---- flusher warp ----------------------------------------------------------------
    // Blocked in hardware on named barrier 1 (bar.sync, 64 threads) until a worker whose
    // merge completed a batch of flush_centers arrives on it (bar.arrive, non-blocking).
    // Two worker arrivals may complete a phase on their own, which only delays a flush.
    // Shutdown: the last worker sets s_done and then keeps arriving until the flusher has
    // exited, so a bar.sync entered after the last regular arrival always gets a partner.
    if (warp == workers) {
        if (K > 0 || K0 > 0) {
            for (;;) {
                if (*reinterpret_cast<volatile int*>(&s_done) == workers) {
                    flush_cache(true);
                    break;
                }
                named_bar_sync(1, 64);
                flush_cache(false);
            }
        }
        __syncwarp();
        if (lane == 0) s_exit = 1;
        return;
    }

    // ---- workers ---------------------------------------------------------------------
    int* codes = codes_all + warp * kCodeSlots;
    uint64_t* mb = mbar_all + warp;
    unsigned phase = 0;
    float* sg = reinterpret_cast<float*>(s_sig + warp * 8);
    float4* V = ctx_all + static_cast<size_t>(warp) * 2 * NB * d4;
    float4* Hs = V + NB * d4;
    float4* Ub = ub_all + static_cast<size_t>(warp) * G * d4;
    const unsigned row_bytes = static_cast<unsigned>(d4) * 16u;
    // Stages the live rows of group j0 into Ub (rows past the path end keep their previous,
    // finite contents: their signals are 0 and their deltas unused). Bulk copies: lane 0
    // arms the warp's mbarrier for them (plus `extra_bytes` copied by other lanes) and
    // issues one UBLKCP per row; cp.async: the whole warp, 16 bytes per lane.
    auto issue_group = [&](int j0, int L, unsigned extra_bytes) {
        const int live = min(G, L - j0);
        if constexpr (CG_STAGE_BULK) {
            if (lane == 0) {
                mbar_expect_tx(mb, static_cast<unsigned>(live) * row_bytes + extra_bytes);
                for (int g = 0; g < live; ++g)
                    bulk_g2s(Ub + g * d4, a.syn1 + static_cast<size_t>(codes[j0 + g] >> 1) * d4 * 4, row_bytes, mb);
            }
        } else {
            for (int g = 0; g < live; ++g) {
                const float* src = a.syn1 + static_cast<size_t>(codes[j0 + g] >> 1) * d4 * 4;
#pragma unroll
                for (int k = 0; k < DCH; ++k) {
                    const int q = lane + 32 * k;
                    if (in_row<DCH>(k, q, d4)) cp_async16(Ub + g * d4 + q, src + 4 * q);
                }
            }
        }
    };
    auto wait_stage = [&]() {
        if constexpr (CG_STAGE_BULK) {
            mbar_wait(mb, phase);
            phase ^= 1u;
        } else {
            cp_async_wait_all();
            __syncwarp();
        }
    };
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
        // the ticket's per-center metadata in two coalesced dependent loads (lane j: center c0 + j)
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
            // a 32x32 multiply-high of its top bits (uniform to within W / 2^32)
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
                // context ids in one coalesced load (lane i: context i)
                int xid = 0;
                if (lane < nb) {
                    int64_t pos = lo + q0 + lane;
                    pos += pos >= ci;  // skip the center's own position
                    xid = a.kept[pos];
                }
                unsigned hot_ctx = 0;  // contexts whose syn0 row is in the CTA cache (ids are in count order)
                if constexpr (CTX) hot_ctx = __ballot_sync(kFull, lane < nb && xid < K0);
                __syncwarp();  // codes visible; V and Ub free
                // one phase of the warp's mbarrier covers the batch's context rows and the
                // path's first row group: lane 0 arms it, lane i copies context row i
                if (CTX && lane == 0) fence_proxy_async();  // V was written by the generic proxy
                issue_group(0, L, static_cast<unsigned>(nb) * row_bytes);
                if constexpr (CG_STAGE_BULK) {
                    __syncwarp();
                    if (lane < nb) bulk_g2s(V + lane * d4, a.syn0 + static_cast<size_t>(xid) * d4 * 4, row_bytes, mb);
                } else {
                    for (int i = 0; i < nb; ++i) {
                        const float* src = a.syn0 + static_cast<size_t>(__shfl_sync(kFull, xid, i)) * d4 * 4;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            if (in_row<DCH>(k, q, d4)) cp_async16(V + i * d4 + q, src + 4 * q);
                        }
                    }
                }
                if constexpr (CG_H_BULKRED) {  // the previous batch's h rows have left Hs
                    bulk_wait_read<0>();
                    __syncwarp();
                }
                for (int i = 0; i < nb; ++i) {
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (in_row<DCH>(k, q, d4)) Hs[i * d4 + q] = f4(0.f);
                    }
                }
                for (int j0 = 0; j0 < L; j0 += G) {
                    wait_stage();  // this group's rows (and, first time, the contexts)
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
                    // + this CTA's pending delta of cached rows; row[g] is warp-uniform
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (row[g] < S) {
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) U[g][k] = add4(U[g][k], dblk[row[g] * d4 + q]);
                            }
                        } else if (CG_T2_READ && row[g] < K) {
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4))
                                    U[g][k] = add4(U[g][k], ld_cg4(t2 + (static_cast<size_t>(row[g] - S) * d4 + q) * 4));
                            }
                        }
                    }
                    __syncwarp();  // every lane has its copy: Ub takes the next group
                    if (j0 + G < L) issue_group(j0 + G, L, 0u);
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
                        // Rolled: unrolled (fully or 2x), the hot loop outgrows the
                        // instruction cache or the registers (ncu: 21% no_instruction stalls
                        // fully unrolled; 2x: +11% K1 time at D 300). Lanes past the row end
                        // compute on neighbouring data; those chunks are never written back.
                        const int ni = min(cic, r);
                        const float4* sg4 = reinterpret_cast<const float4*>(sg);
                        if constexpr (DCH < 3) {
#pragma unroll 1
                            for (int ii = 0; ii < ni; ++ii) {
                                const int i = cc + ii;
                                // h accumulates in place: Hs[i] loaded up front with v
                                float4 v[DCH], hacc[DCH];
#pragma unroll
                                for (int k = 0; k < DCH; ++k) {
                                    v[k] = V[i * d4 + lane + 32 * k];
                                    hacc[k] = Hs[i * d4 + lane + 32 * k];
                                }
                                const float4 g4 = sg4[ii];  // one broadcast load for the G signals
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
                            // D > 256: software-pipelined. The next context's v and signals
                            // load while this one's FMAs run, and the Dl FMAs go first so the
                            // h row loaded at the top arrives before its FMAs (C4 1287 ->
                            // 1241 ms at v4; at D <= 256 it measured slower).
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
                    // write each row's delta back once: shared-memory tier (locked merge),
                    // L2 tier (red into this CTA's delta row) or the model row (red)
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (j0 + g >= L) continue;
                        if (row[g] < S) {
                            touched_cache = true;
                            if (lane == 0) lock_row(&locks[row[g]]);
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
                        } else {
                            float* dst = row[g] < K ? t2 + static_cast<size_t>(row[g] - S) * d4 * 4
                                                    : a.syn1 + static_cast<size_t>(row[g]) * d4 * 4;
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                const int q = lane + 32 * k;
                                if (in_row<DCH>(k, q, d4)) red_add4(dst + 4 * q, Dl[g][k]);
                            }
                            if (row[g] >= K) continue;
                            touched_cache = true;
                        }
                        if (lane == 0) {
                            const unsigned bit = 1u << (row[g] & 31);
                            if (!(touch[row[g] >> 5] & bit)) atomicOr(&touch[row[g] >> 5], bit);
                        }
                    }
                }
                __syncwarp();
                // the contexts' rows move once, by their accumulated h (trainer.hpp:173)
                if constexpr (CG_H_BULKRED) {
                    // one bulk reduction per context row, issued by lane i for row i: the TMA
                    // unit adds the whole row at L2 (no per-lane REDG); Hs is reused once
                    // the reads have completed (bulk_wait_read above)
                    fence_proxy_async();
                    __syncwarp();
                    if (lane < nb && !((hot_ctx >> lane) & 1u))
                        bulk_red_add_f32(a.syn0 + static_cast<size_t>(xid) * d4 * 4, Hs + lane * d4, row_bytes);
                    bulk_commit();
                }
                for (int i = 0; i < nb; ++i) {
                    if (CG_H_BULKRED && !(CTX && ((hot_ctx >> i) & 1u))) continue;
                    const int x = __shfl_sync(kFull, xid, i);
                    if (CTX && ((hot_ctx >> i) & 1u)) {  // merge into the CTA's cached delta
                        touched_cache = true;
                        if (lane == 0) lock_row(&locks0[x]);
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
                    float* dst = a.syn0 + static_cast<size_t>(x) * d4 * 4;
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (in_row<DCH>(k, q, d4)) red_add4(dst + 4 * q, Hs[i * d4 + q]);
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
                        flush_cache(false);
                    }
                }
            }
        }
    }
    if constexpr (CG_H_BULKRED) bulk_wait_read<0>();  // shared memory outlives the last bulk reductions
    int last = 0;
    if (lane == 0) {
        atomicAdd(a.counters + 1, n_pairs);
        atomicAdd(a.counters + 2, n_steps);
        atomicAdd(a.counters + 3, n_centers);
        __threadfence_block();  // this warp's merges before its done count
        last = atomicAdd(&s_done, 1) == workers - 1;
    }
    last = __shfl_sync(kFull, last, 0);
    if (!last || (K == 0 && K0 == 0)) return;
    __threadfence_block();
    if (a.flusher) {
        // wake the flusher for its final flush; keep arriving until it has exited
        while (!s_exit) {
            named_bar_arrive(1, 64);
            __nanosleep(256);
        }
    } else {
        // without a flusher warp the last worker drains what the others merged after
        // their last flush, and empties both tiers
        flush_cache(true);
    }
}

// ---- generic K1: any row width, any tree depth ---------------------------------------
// Rows wider than 384 floats or paths deeper than kMaxGroupDepth. One warp per center in
// the reference's per-pair order (train_center, trainer.hpp:160-173): for each context,
// for each path step, dot -> sigmoid -> h += g u -> u += g v, lanes striding over the
// row's float4 chunks. All cached rows use the L2 tier (the delta rows in `tier2`); the
// worker whose merge completes a batch of flush_centers drains the CTA's touched rows.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) hog_generic_kernel(HogArgs a) {
    extern __shared__ __align__(16) unsigned char kg_raw[];
    const int d4 = a.d4, K = a.cache_rows;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int warps = blockDim.x >> 5;
    float* sig = reinterpret_cast<float*>(kg_raw);
    const int nwords = (K + 31) >> 5;
    unsigned* touch = reinterpret_cast<unsigned*>(kg_raw + 4096);
    float4* bufs = reinterpret_cast<float4*>(kg_raw + 4096 + ((nwords * 4 + 127) & ~127));
    float4* V = bufs + static_cast<size_t>(warp) * 2 * d4;
    float4* Hs = V + d4;
    float* t2 = a.tier2 ? a.tier2 + static_cast<size_t>(blockIdx.x) * static_cast<size_t>(K) * d4 * 4 : nullptr;
    __shared__ int s_done;
    __shared__ unsigned s_merged;
    for (int i = tid; i < 1000; i += blockDim.x) sig[i] = a.sigmoid[i];
    for (int i = tid; i < nwords; i += blockDim.x) touch[i] = 0u;
    if (tid == 0) {
        s_done = 0;
        s_merged = 0;
    }
    __syncthreads();

    auto flush_cache = [&](bool all) {
        for (int w = 0; w < nwords; ++w) {
            unsigned m = 0;
            if (lane == 0) {
                if (all) {
                    m = w == nwords - 1 && (K & 31) ? (1u << (K & 31)) - 1u : ~0u;
                    touch[w] = 0u;
                } else if (touch[w]) {
                    m = atomicExch(&touch[w], 0u);
                }
            }
            for (m = __shfl_sync(kFull, m, 0); m; m &= m - 1) {
                const int r = (w << 5) + __ffs(m) - 1;
                const float sc = a.row_scale ? a.row_scale[r] : a.hot_flush_scale;
                for (int q = lane; q < d4; q += 32) {
                    const float4 d = atom_take4(t2 + (static_cast<size_t>(r) * d4 + q) * 4);
                    if (nonzero4(d)) red_add4(a.syn1 + (static_cast<size_t>(r) * d4 + q) * 4, scale4(sc, d));
                }
            }
        }
        __threadfence();
    };

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
            const int b = a.window - static_cast<int>(__umulhi(static_cast<unsigned>(ctr_draw(a.win_key, static_cast<uint64_t>(ci)) >> 32),
                                                               static_cast<unsigned>(a.window)));
            const int64_t lo = max(s_lo, ci - b), hi = min(s_hi - 1, ci + b);
            ++n_centers;
            const int p0 = a.path_off[c];
            const int L = a.path_off[c + 1] - p0;
            bool touched_cache = false;
            for (int64_t pos = lo; pos <= hi; ++pos) {
                if (pos == ci) continue;
                const int x = a.kept[pos];
                const float* xrow = a.syn0 + static_cast<size_t>(x) * d4 * 4;
                __syncwarp();
                for (int q = lane; q < d4; q += 32) {
                    V[q] = ld_cg4(xrow + 4 * q);
                    Hs[q] = f4(0.f);
                }
                __syncwarp();
                for (int j = 0; j < L; ++j) {
                    const int code = a.path_code[p0 + j];
                    const int row = code >> 1;
                    const bool cached = row < K;
                    const float* urow = a.syn1 + static_cast<size_t>(row) * d4 * 4;
                    float* drow = cached ? t2 + static_cast<size_t>(row) * d4 * 4 : nullptr;
                    float2 acc = make_float2(0.f, 0.f);
                    for (int q = lane; q < d4; q += 32) {
                        float4 u = ld_cg4(urow + 4 * q);
                        if (cached) u = add4(u, ld_cg4(drow + 4 * q));
                        acc = dot4(V[q], u, acc);
                    }
                    float dot = acc.x + acc.y;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(kFull, dot, off);
                    const float f = table_sigmoid(sig, dot, a.sig_scale);
                    const float gl = (1.0f - static_cast<float>(code & 1) - f) * alpha;
                    float* dst = cached ? drow : a.syn1 + static_cast<size_t>(row) * d4 * 4;
                    for (int q = lane; q < d4; q += 32) {
                        float4 u = ld_cg4(urow + 4 * q);
                        if (cached) u = add4(u, ld_cg4(drow + 4 * q));
                        Hs[q] = axpy4(gl, u, Hs[q]);
                        red_add4(dst + 4 * q, scale4(gl, V[q]));
                    }
                    if (cached) {
                        touched_cache = true;
                        if (lane == 0) {
                            const unsigned bit = 1u << (row & 31);
                            if (!(touch[row >> 5] & bit)) atomicOr(&touch[row >> 5], bit);
                        }
                    }
                }
                __syncwarp();
                float* dst = a.syn0 + static_cast<size_t>(x) * d4 * 4;
                for (int q = lane; q < d4; q += 32) red_add4(dst + 4 * q, Hs[q]);
                n_pairs += 1;
                n_steps += static_cast<unsigned long long>(L);
            }
            if (touched_cache) {
                unsigned m = 0;
                if (lane == 0) m = atomicAdd(&s_merged, 1u) + 1u;
                m = __shfl_sync(kFull, m, 0);
                if (m % static_cast<unsigned>(a.flush_centers) == 0u) flush_cache(false);
            }
        }
    }
    int last = 0;
    if (lane == 0) {
        atomicAdd(a.counters + 1, n_pairs);
        atomicAdd(a.counters + 2, n_steps);
        atomicAdd(a.counters + 3, n_centers);
        __threadfence_block();
        last = atomicAdd(&s_done, 1) == warps - 1;
    }
    last = __shfl_sync(kFull, last, 0);
    if (last && K > 0) flush_cache(true);
}

constexpr int kGenericWarps = 8;

// Worker warps per CTA for the row-group kernel (the register budget of its launch
// bounds): 16 (D <= 128), 12 (D <= 256), 8 (D <= 384). G = 8 rows per group and fewer
// warps measured slower at v4 (C1 3.66 -> 4.48 ms, C2 90 -> 124 ms), so did G = 2 with
// 15 warps (C2 116 ms); 11 warps at D <= 256 (C2 72.33 vs 72.09 ms).
template <int DCH>
constexpr int kW5 = DCH == 1 ? 16 : (DCH == 2 ? CG_W2 : 8);

template <int DCH, bool CTX>
auto hog5_for(int d4, bool specialise) -> decltype(&hog5_kernel<DCH, kW5<DCH>, 0, CTX>) {
    if (specialise) {  // the benchmark row widths (D 100, 128, 200, 300, padded to 32 bytes)
        if constexpr (DCH == 1) {
            if (d4 == 26) return hog5_kernel<1, kW5<1>, 26, CTX>;
            if (d4 == 32) return hog5_kernel<1, kW5<1>, 32, CTX>;
        } else if constexpr (DCH == 2) {
            if (d4 == 50) return hog5_kernel<2, kW5<2>, 50, CTX>;
        } else if constexpr (DCH == 3) {
            if (d4 == 76) return hog5_kernel<3, kW5<3>, 76, CTX>;
        }
    }
    return hog5_kernel<DCH, kW5<DCH>, 0, CTX>;
}

template <int DCH>
void launch_variant(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    void (*k)(HogArgs) = g.ctx_rows > 0 ? hog5_for<DCH, true>(a.d4, g.specialise) : hog5_for<DCH, false>(a.d4, g.specialise);
    // always opt in: dynamic + static shared memory above 48 KB needs it even when the
    // dynamic part alone is below (a launch without it failed with "invalid argument")
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
    HogArgs b = a;
    b.cache_rows = g.cache_rows;
    b.smem_rows = g.smem_rows;
    b.ctx_cache_rows = g.ctx_rows;
    b.centers_per_warp = g.cpw;
    b.ctx_batch = g.ctx_batch;
    b.flusher = g.flusher ? 1 : 0;
    k<<<g.blocks, (g.warps + (g.flusher ? 1 : 0)) * 32, g.smem, s>>>(b);
}

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

int hog_max_warps(int d4, int max_depth) {
    if (d4 > 96 || max_depth > kMaxGroupDepth) return kGenericWarps;
    const int v = (d4 + 31) / 32;
    return v == 1 ? kW5<1> : (v == 2 ? kW5<2> : kW5<3>);
}

// Shared-memory rows of the cache by default: the hottest 8 (a cached row in shared
// memory costs a lock and a merge per center, and at D 300 its shared memory costs a
// worker warp; at v4, 8 rows was within 3% of the fastest setting at C1-C5 and 31 rows
// 3-16% slower: profiles/r1_rows_sweep.jsonl). Rows [8, K) go to the L2 tier.
constexpr int kSmemRowsDefault = 8;

HogGeometry hog_plan(int d4, int max_depth, int cache_rows, int smem_rows, int blocks_override, int warps_override,
                     int cpw_override, int window, int64_t tokens, int ctx_rows) {
    HogGeometry g{};
    g.specialise = true;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g.blocks = blocks_override > 0 ? blocks_override : sms;
    g.cache_rows = std::max(0, std::min(cache_rows, kMaxCacheRows));
    if (d4 > 96 || max_depth > kMaxGroupDepth) {  // generic kernel: every cached row in the L2 tier
        g.variant = 0;
        g.warps = warps_override > 0 ? std::min(warps_override, kGenericWarps) : kGenericWarps;
        g.smem_rows = 0;
        g.ctx_rows = 0;
        g.ctx_batch = 1;
        g.flusher = false;
        const size_t touch = ((static_cast<size_t>(g.cache_rows) + 31) / 32 * 4 + 127) & ~size_t{127};
        const size_t budget = 227 * 1024 - 1024;
        while (g.warps > 1 && 4096 + touch + static_cast<size_t>(g.warps) * 2 * d4 * 16 > budget) --g.warps;
        g.smem = 4096 + touch + static_cast<size_t>(g.warps) * 2 * d4 * 16;
        if (g.smem > budget) g.smem = 0;  // caller reports: row too wide for shared memory
        g.cpw = cpw_override > 0 ? std::min(cpw_override, 32) : 4;
        return g;
    }
    g.variant = (d4 + 31) / 32;
    const int workers = hog_max_warps(d4, max_depth);
    g.warps = warps_override > 0 ? std::min(warps_override, workers) : workers;
    g.ctx_rows = std::max(ctx_rows, 0);
    // shared-memory tier: at most 48 KB of rows
    const int smem_cap = static_cast<int>((48 * 1024) / (static_cast<size_t>(d4) * 16 + 4));
    g.smem_rows = std::min({g.cache_rows, smem_rows >= 0 ? smem_rows : kSmemRowsDefault, smem_cap});
    // A center whose 2b contexts do not fit one context batch re-reads (and re-writes)
    // its whole path per batch: unless the caller fixed the warp count, drop one warp if
    // that lets one batch hold a full window (2W contexts). Dropping more measured slower
    // (C4, W 10: 4 warps x batch 20 took 1577 ms, 7 warps x batch 10 1322 ms).
    const size_t budget = 227 * 1024 - 4096;  // dynamic shared memory; static (signals, flags) <= 4 KB
    auto batch_for = [&](int warps, size_t* smem) {
        const K1Smem base = k1_smem(warps, g.smem_rows, g.cache_rows, g.ctx_rows, 0, d4);
        const size_t per_ctx = static_cast<size_t>(warps) * 2 * d4 * 16;
        const size_t room = budget > base.total ? budget - base.total : 0;
        int nb = static_cast<int>(std::min<size_t>(2 * static_cast<size_t>(window), room / per_ctx));
        nb = std::min(std::max(nb, 1), 32);  // one context id per lane
        *smem = k1_smem(warps, g.smem_rows, g.cache_rows, g.ctx_rows, nb, d4).total;
        return nb;
    };
    g.ctx_batch = batch_for(g.warps, &g.smem);
    if (warps_override <= 0 && g.ctx_batch < 2 * window && g.warps > 1) {
        size_t sm = 0;
        const int nb = batch_for(g.warps - 1, &sm);
        if (nb >= 2 * window) {
            g.warps -= 1;
            g.ctx_batch = nb;
            g.smem = sm;
        }
    }
    // Centers per ticket: 16 when every warp gets >= 2000 tokens (fewer ticket atomics and
    // metadata loads: C2 -1%, C3 -1.2%, C5 -1.4% vs 4), else 8 (the tail of a small pass
    // grows with the ticket: C1 3.33 ms at 8, 3.44 at 32).
    g.cpw = cpw_override > 0 ? std::min(cpw_override, 32)
                             : (tokens / (static_cast<int64_t>(g.blocks) * g.warps) >= 2000 ? 16 : 8);
    // a warp the registers allow but shared memory cannot feed becomes the cache flusher
    g.flusher = g.warps < workers && (g.cache_rows > 0 || g.ctx_rows > 0);
    return g;
}

void launch_hogwild(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    switch (g.variant) {
        case 8: launch_hog8(a, g, s); break;
        case 0: {
            auto k = hog_generic_kernel<kGenericWarps>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
            HogArgs b = a;
            b.cache_rows = g.cache_rows;
            b.smem_rows = 0;
            b.ctx_cache_rows = 0;
            b.centers_per_warp = g.cpw;
            b.ctx_batch = 1;
            b.flusher = 0;
            k<<<g.blocks, g.warps * 32, g.smem, s>>>(b);
            break;
        }
        case 1: launch_variant<1>(a, g, s); break;
        case 2: launch_variant<2>(a, g, s); break;
        default: launch_variant<3>(a, g, s); break;
    }
}

}  // namespace cgk
