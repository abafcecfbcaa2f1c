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
template <int DCH, int HMAX, int G, int WORKERS>
__global__ void __launch_bounds__((WORKERS + 1) * 32, 1) hog_kernel(HogArgs a) {
    constexpr int LGH = Log2<HMAX>::v;
    constexpr int LGG = Log2<G>::v;
    extern __shared__ float4 hsm[];
    float* sig = reinterpret_cast<float*>(hsm);                      // 1024 floats
    int* codes_all = reinterpret_cast<int*>(hsm + 256);              // WORKERS * kCodeSlots
    float4* dblk = hsm + 256 + WORKERS * (kCodeSlots / 4);           // cache_rows * d4
    const int K = a.cache_rows;
    const int d4 = a.d4;
    int* locks = reinterpret_cast<int*>(dblk + K * d4);
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
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (q < d4 && nonzero4(d[k])) red_add4(a.syn1 + 4 * (r * d4 + q), scale4(a.hot_flush_scale, d[k]));
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
            if (hi == lo) continue;
            const int p0 = a.path_off[c];
            const int L = a.path_off[c + 1] - p0;
            __syncwarp();
            for (int j = lane; j < kCodeSlots; j += 32) codes[j] = j < L ? a.path_code[p0 + j] : dummy_code;
            __syncwarp();
            const unsigned hm = __ballot_sync(kFull, lane < L && (codes[lane] >> 1) < K);
            const int H = hm == kFull ? 32 : __ffs(~hm) - 1;
            const int Hp = min(H, HMAX);

            // private copy of the cached prefix: U = working rows, Q = this center's delta
            float4 U[HMAX][DCH], Q[HMAX][DCH];
#pragma unroll
            for (int j = 0; j < HMAX; ++j) {
                const int row = codes[j] >> 1;
#pragma unroll
                for (int k = 0; k < DCH; ++k) {
                    const int q = lane + 32 * k;
                    float4 u = f4(0.f);
                    if (j < Hp && q < d4) u = add4(ld_ca4(a.syn1 + 4 * (row * d4 + q)), dblk[row * d4 + q]);
                    U[j][k] = u;
                    Q[j][k] = f4(0.f);
                }
            }

            for (int64_t xi = lo; xi <= hi; ++xi) {
                if (xi == ci) continue;
                const int xo = a.kept[xi] * d4;
                float4 v[DCH], h[DCH];
#pragma unroll
                for (int k = 0; k < DCH; ++k) {
                    const int q = lane + 32 * k;
                    v[k] = q < d4 ? ld_cg4(a.syn0 + 4 * (xo + q)) : f4(0.f);
                    h[k] = f4(0.f);
                }
                // -- phase A: the cached prefix, on the private copy
                if (Hp > 0) {
                    float p[HMAX];
#pragma unroll
                    for (int j = 0; j < HMAX; ++j) {
                        float acc = 0.f;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) acc = dot4(v[k], U[j][k], acc);
                        p[j] = acc;
                    }
                    const float tot = transpose_reduce<HMAX>(p, lane);
                    const int jl = lane >> (5 - LGH);
                    const float f = table_sigmoid(sig, tot, a.sig_scale);
                    const float gl = (1.0f - static_cast<float>(codes[jl] & 1) - f) * alpha;
#pragma unroll
                    for (int j = 0; j < HMAX; ++j) {
                        const float g = __shfl_sync(kFull, gl, j << (5 - LGH));
                        if (j < Hp) {
#pragma unroll
                            for (int k = 0; k < DCH; ++k) {
                                h[k] = axpy4(g, U[j][k], h[k]);
                                U[j][k] = axpy4(g, v[k], U[j][k]);
                                Q[j][k] = axpy4(g, v[k], Q[j][k]);
                            }
                        }
                    }
                }
                // -- phase B: the rest of the path, G steps at a time (padded with a zero row)
                for (int j0 = Hp; j0 < L; j0 += G) {
                    float4 R[G][DCH];
                    int ro[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        ro[g] = (codes[j0 + g] >> 1) * d4;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            R[g][k] = q < d4 ? ld_cg4(a.syn1 + 4 * (ro[g] + q)) : f4(0.f);
                        }
                    }
                    float p[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        float acc = 0.f;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) acc = dot4(v[k], R[g][k], acc);
                        p[g] = acc;
                    }
                    const float tot = transpose_reduce<G>(p, lane);
                    const int jl = j0 + (lane >> (5 - LGG));
                    const float f = table_sigmoid(sig, tot, a.sig_scale);
                    const float gl = jl < L ? (1.0f - static_cast<float>(codes[jl] & 1) - f) * alpha : 0.f;
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float gg = __shfl_sync(kFull, gl, g << (5 - LGG));
                        const bool live = j0 + g < L;
#pragma unroll
                        for (int k = 0; k < DCH; ++k) {
                            const int q = lane + 32 * k;
                            h[k] = axpy4(gg, R[g][k], h[k]);
                            if (live && q < d4) {
                                if (a.probe & 1) {
                                } else if (a.cold_store)
                                    st_cg4(a.syn1 + 4 * (ro[g] + q), axpy4(gg, v[k], R[g][k]));
                                else
                                    red_add4(a.syn1 + 4 * (ro[g] + q), scale4(gg, v[k]));
                            }
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < DCH; ++k) {
                    const int q = lane + 32 * k;
                    if (q < d4 && !(a.probe & 2)) {
                        if (a.cold_store)
                            st_cg4(a.syn0 + 4 * (xo + q), add4(v[k], h[k]));
                        else
                            red_add4(a.syn0 + 4 * (xo + q), h[k]);
                    }
                }
                ++n_pairs;
                n_steps += static_cast<unsigned long long>(L);
            }
            // merge the center's delta into the block cache (row locks) and count it
#pragma unroll
            for (int j = 0; j < HMAX; ++j) {
                if (j < Hp && !(a.probe & 4)) {
                    const int row = codes[j] >> 1;
                    if (lane == 0)
                        while (atomicCAS(&locks[row], 0, 1) != 0) {
                        }
                    __syncwarp();
                    __threadfence_block();
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (q < d4) dblk[row * d4 + q] = add4(dblk[row * d4 + q], Q[j][k]);
                    }
                    __threadfence_block();
                    __syncwarp();
                    if (lane == 0) atomicExch(&locks[row], 0);
                }
            }
            if (lane == 0 && Hp > 0) atomicAdd(&s_merged, 1u);
        }
    }
    if (lane == 0) {  // counts are warp-uniform
        atomicAdd(a.counters + 1, n_pairs);
        atomicAdd(a.counters + 2, n_steps);
        atomicAdd(a.counters + 3, n_centers);
        atomicAdd(&s_done, 1);
    }
}

template <int DCH, int HMAX, int G, int WORKERS>
void launch_variant(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    auto k = hog_kernel<DCH, HMAX, G, WORKERS>;
    if (g.smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
    HogArgs b = a;
    b.cache_rows = g.cache_rows;
    b.centers_per_warp = g.cpw;
    k<<<g.blocks, (g.warps + 1) * 32, g.smem, s>>>(b);
}

// Per-variant shape: float4 chunks per lane (DCH), private cached prefix (HMAX),
// cold-step group (G) and worker warps (register budget of the launch bounds).
template <int DCH>
struct Variant;
template <>
struct Variant<1> {
    static constexpr int HMAX = 8, G = 8, WORKERS = 11;
};
template <>
struct Variant<2> {
    static constexpr int HMAX = 4, G = 4, WORKERS = 11;
};
template <>
struct Variant<3> {
    static constexpr int HMAX = 4, G = 4, WORKERS = 7;
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

int hog_hmax(int d4) {
    switch ((d4 + 31) / 32) {
        case 1: return Variant<1>::HMAX;
        case 2: return Variant<2>::HMAX;
        default: return Variant<3>::HMAX;
    }
}

HogGeometry hog_plan(int d4, int cache_rows_wanted, int blocks_override, int warps_override, int cpw_override,
                     int rows_override) {
    HogGeometry g{};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g.variant = (d4 + 31) / 32;
    const int workers = g.variant == 1 ? Variant<1>::WORKERS : (g.variant == 2 ? Variant<2>::WORKERS : Variant<3>::WORKERS);
    g.warps = warps_override > 0 ? std::min(warps_override, workers) : workers;
    g.blocks = blocks_override > 0 ? blocks_override : sms;
    g.cpw = cpw_override > 0 ? cpw_override : 4;
    const size_t fixed = 4096 + static_cast<size_t>(workers) * kCodeSlots * 4;
    const size_t budget = 110 * 1024;
    const size_t per_row = static_cast<size_t>(d4) * 16 + 4;
    const int fit = static_cast<int>((budget - fixed) / per_row);
    int rows = std::min(cache_rows_wanted, fit);
    if (rows_override >= 0 && rows_override < rows) rows = rows_override;
    g.cache_rows = std::max(rows, 0);
    g.smem = fixed + static_cast<size_t>(g.cache_rows) * per_row + 16;
    return g;
}

void launch_hogwild(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    switch (g.variant) {
        case 1: launch_variant<1, Variant<1>::HMAX, Variant<1>::G, Variant<1>::WORKERS>(a, g, s); break;
        case 2: launch_variant<2, Variant<2>::HMAX, Variant<2>::G, Variant<2>::WORKERS>(a, g, s); break;
        default: launch_variant<3, Variant<3>::HMAX, Variant<3>::G, Variant<3>::WORKERS>(a, g, s); break;
    }
}

}  // namespace cgk
