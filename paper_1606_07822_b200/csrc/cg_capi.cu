// cg_capi.cu -- implementation of the C-ABI declared in include/cachegram_b200.h.
//
// Host side of the path (validation, Huffman/selection/keep-prob precompute, device
// layout, launch sequencing, error mapping) in C++; every training computation is a
// CUDA kernel (cg_det.cu, cg_hogwild.cu). There is no CPU training fallback.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <atomic>
#include <barrier>
#include <condition_variable>
#include <deque>
#include <exception>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "cachegram/corpus.hpp"
#include "cachegram/huffman.hpp"
#include "cachegram/model.hpp"
#include "cachegram/trainer.hpp"
#include "cachegram_b200.h"
#include "cg_device.cuh"
#include "cg_host.h"
#include "cg_kernels.h"

namespace {

thread_local std::string g_error;

struct CgError : std::runtime_error {
    int code;
    CgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CgError(CG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CG_CUDA(call) check_cuda((call), #call)

[[noreturn]] void invalid(const std::string& m) { throw CgError(CG_ERR_INVALID_ARGUMENT, m); }

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return CG_OK;
    } catch (const CgError& e) {
        g_error = e.what();
        return e.code;
    } catch (const cgint::CudaError& e) {
        g_error = e.what();
        return CG_ERR_CUDA;
    } catch (const cachegram::IoError& e) {
        g_error = e.what();
        return CG_ERR_IO;
    } catch (const cachegram::ParseError& e) {
        g_error = e.what();
        return CG_ERR_PARSE;
    } catch (const cachegram::NoTrainableWords& e) {
        g_error = e.what();
        return CG_ERR_NO_TRAINABLE_WORDS;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return CG_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return CG_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_error = e.what();
        return CG_ERR_INTERNAL;
    }
}

// TrainConfig::validate (trainer.hpp:37-47), same messages.
void validate_config(const cg_config& c) {
    if (c.dim < 1) invalid("dim must be >= 1");
    if (c.window < 1) invalid("window must be >= 1");
    if (c.min_count < 1) invalid("min-count must be >= 1");
    if (c.sample < 0.0) invalid("sample must be >= 0");
    if (!(c.alpha0 > 0.0f)) invalid("alpha must be > 0");
    if (c.iterations < 1) invalid("iterations must be >= 1");
    if (c.workers < 1) invalid("workers must be >= 1");
    if (c.cache_nodes < 0) invalid("cache-nodes must be >= 0");
    if (c.flush_interval < 1) invalid("flush-interval must be >= 1");
}

void validate_model(const cg_model_desc& m) {
    if (m.vocab_size < 2) invalid("vocabulary and tree sizes disagree");
    if (!m.counts || !m.path_offsets || !m.path_nodes || !m.path_turns) invalid("model description has null arrays");
    if (m.hot_count < 0 || m.hot_count > m.vocab_size - 1)
        invalid("cache selection was built from a different tree");
    if (m.hot_count > 0 && !m.hot_nodes) invalid("cache selection was built from a different tree");
    if (m.path_offsets[0] != 0) invalid("path offsets must start at 0");
    for (int32_t w = 0; w < m.vocab_size; ++w)
        if (m.path_offsets[w + 1] <= m.path_offsets[w]) invalid("every word needs a non-empty tree path");
    const int64_t steps = m.path_offsets[m.vocab_size];
    for (int64_t k = 0; k < steps; ++k)
        if (m.path_nodes[k] < 0 || m.path_nodes[k] >= m.vocab_size - 1 || m.path_turns[k] > 1)
            invalid("vocabulary and tree sizes disagree");
    std::vector<char> seen(static_cast<size_t>(m.vocab_size - 1), 0);
    for (int32_t s = 0; s < m.hot_count; ++s) {
        if (m.hot_nodes[s] < 0 || m.hot_nodes[s] >= m.vocab_size - 1 || seen[static_cast<size_t>(m.hot_nodes[s])])
            invalid("cache selection was built from a different tree");
        seen[static_cast<size_t>(m.hot_nodes[s])] = 1;
    }
    // HuffmanTree::node_usage orders the device rows and sets the flush scale of every
    // cached row; without it the hot rows' CTA replicas would be summed (divergent).
    if (!m.node_usage) invalid("model description has null arrays");
}


template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { cgint::DevicePool::get().free(p); }
    void alloc(size_t count) {
        cgint::DevicePool::get().free(p);
        p = nullptr;
        n = count;
        if (count) p = static_cast<T*>(cgint::DevicePool::get().alloc(count * sizeof(T)));
    }
    void upload(const T* host, size_t count, cudaStream_t s) {
        alloc(count);
        if (count) CG_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
};

// ---- small device helpers of the layout --------------------------------------
__global__ void path_code_kernel(const int32_t* nodes, const uint8_t* turns, const int32_t* row_of_node, int64_t n,
                                 int32_t* code) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        code[k] = (row_of_node[nodes[k]] << 1) | turns[k];
}

__global__ void init_syn0_kernel(float* out, int64_t rows, int32_t dim, int32_t stride, uint64_t key, float inv_dim) {
    // model.hpp:66-72: value i (row-major, unpadded) = (unit24(draw i) - 0.5f) * (1/D)
    const int64_t n = rows * dim;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / dim, d = i - r * dim;
        const float u = cgdev::unit24(cgdev::ctr_draw(key, static_cast<uint64_t>(i)));
        out[r * stride + d] = __fmul_rn(__fsub_rn(u, 0.5f), inv_dim);
    }
}

// dst[r*ds + d] = src[perm(r)*ss + d]; perm == nullptr means identity. Pads are left alone.
__global__ void gather_rows_kernel(float* dst, int32_t ds, const float* src, int32_t ss, const int32_t* perm,
                                   int64_t rows, int32_t dim) {
    const int64_t n = rows * dim;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / dim, d = i - r * dim;
        const int64_t sr = perm ? perm[r] : r;
        dst[r * ds + d] = src[sr * ss + d];
    }
}
// dst[perm(r)*ds + d] = src[r*ss + d]
__global__ void scatter_rows_kernel(float* dst, int32_t ds, const float* src, int32_t ss, const int32_t* perm,
                                    int64_t rows, int32_t dim) {
    const int64_t n = rows * dim;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / dim, d = i - r * dim;
        const int64_t dr = perm ? perm[r] : r;
        dst[dr * ds + d] = src[r * ss + d];
    }
}

unsigned grid_for(int64_t n) { return static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// ---- replica sync: deltas since the last sync, summed across replicas ----
// The delta buffer: the model's layout, then one squared norm per model row (|delta_r|^2),
// padded to a multiple of 4 floats, then 4 floats of which the first two are the summed
// squared norms of the syn0 and the syn1 rows of the model. One all-reduce sums it all.
// Measured (tools/replica_quality.py, learning ratio against one replica): with no trust
// term C5 split 8 ways learns 1.04 but C1 split 4 ways at 500-word syncs 0.915; with 0.5 over
// the rms of all rows C1 0.974 but C5 0.66-0.76 (the hot vectors that most updates pair with
// are longer than the average row); 0.25 over the 1024 hottest rows gives 1.04 and 0.974.
#ifndef CG_SYNC_TRUST
#define CG_SYNC_TRUST 0.25f
#endif
#ifndef CG_SYNC_HOT
#define CG_SYNC_HOT 1024  // the matrices' rms norms are taken over their first CG_SYNC_HOT (hottest) rows; 0 = all
#endif
constexpr float kSyncTrust = CG_SYNC_TRUST;  // a summed step may move a logit by about this much unscaled
constexpr size_t kSyncHot = CG_SYNC_HOT;
__host__ __device__ inline size_t sync_tail_rows(size_t rows) { return (rows + 3) & ~size_t{3}; }

// One warp per model row: delta = model - snapshot, sumsq[row] = |delta|^2, and the row's own
// squared norm added to its matrix's total.
__global__ void sync_delta_kernel(const float4* model, const float4* snap, float4* delta, float* sumsq, float* totals,
                                  size_t rows, size_t rows0, int32_t row4) {
    const size_t warp = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5;
    const size_t nwarps = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    float own0 = 0.f, own1 = 0.f;
    for (size_t r = warp; r < rows; r += nwarps) {
        float acc = 0.f, own = 0.f;
        for (int q = lane; q < row4; q += 32) {
            const size_t i = r * static_cast<size_t>(row4) + q;
            const float4 m = model[i], b = snap[i];
            const float4 d = make_float4(m.x - b.x, m.y - b.y, m.z - b.z, m.w - b.w);
            delta[i] = d;
            acc += d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
            own += m.x * m.x + m.y * m.y + m.z * m.z + m.w * m.w;
        }
        for (int o = 16; o > 0; o >>= 1) {
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
            own += __shfl_xor_sync(0xffffffffu, own, o);
        }
        if (lane == 0) sumsq[r] = acc;
        const size_t rr = r < rows0 ? r : r - rows0;  // rows are hottest first in both matrices
        if (kSyncHot == 0 || rr < kSyncHot) (r < rows0 ? own0 : own1) += own;
    }
    if (lane == 0) {
        if (own0 != 0.f) atomicAdd(totals, own0);
        if (own1 != 0.f) atomicAdd(totals + 1, own1);
    }
}
// With the buffer summed over the n replicas: model = snapshot + s x delta, snapshot = model,
// one warp per row, s = min(prior[row], max(ratio, trust)):
//  * ratio = clamp(sum_r |delta_r|^2 / |sum_r delta_r|^2, 1 / n, 1) is 1 when the replicas'
//    deltas are orthogonal (or one replica alone touched the row: the reference's plain sum)
//    and 1 / n when they are parallel (every replica made the same move from the same
//    snapshot: their average); with it alone the applied step is never longer than the
//    root-sum-square of the replicas' own steps;
//  * trust = min(1, T / |sum_r delta_r|) with T = kSyncTrust / (rms norm of the other
//    matrix's hottest rows): a summed step that moves the row's logits by less than ~kSyncTrust is in the
//    linear regime, where n stale trajectories add up like one sequential one, and is kept
//    whole however parallel the deltas are (small corpora, early training).
__global__ void sync_apply_kernel(float4* model, float4* snap, const float4* delta, const float* sumsq,
                                  const float* totals, const float* prior, size_t rows, size_t rows0, int32_t row4,
                                  float inv_n) {
    const size_t warp = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5;
    const size_t nwarps = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    // rms row norms of the two matrices (totals are summed over the replicas)
    const size_t cnt0 = kSyncHot ? min(rows0, kSyncHot) : rows0, cnt1 = kSyncHot ? min(rows - rows0, kSyncHot) : rows - rows0;
    const float rms0 = sqrtf(totals[0] * inv_n / static_cast<float>(cnt0));
    const float rms1 = sqrtf(totals[1] * inv_n / static_cast<float>(cnt1));
    for (size_t r = warp; r < rows; r += nwarps) {
        float acc = 0.f;
        for (int q = lane; q < row4; q += 32) {
            const float4 d = delta[r * static_cast<size_t>(row4) + q];
            acc += d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (!(acc > 0.f)) continue;  // nobody moved the row
        const float ratio = fminf(1.0f, fmaxf(inv_n, sumsq[r] / acc));
        const float other = fmaxf(r < rows0 ? rms1 : rms0, 1e-12f);
        const float trust = fminf(1.0f, kSyncTrust / (other * sqrtf(acc)));
        const float sc = fminf(prior[r], fmaxf(ratio, trust));
        for (int q = lane; q < row4; q += 32) {
            const size_t i = r * static_cast<size_t>(row4) + q;
            const float4 b = snap[i], d = delta[i];
            const float4 m = make_float4(b.x + sc * d.x, b.y + sc * d.y, b.z + sc * d.z, b.w + sc * d.w);
            model[i] = m;
            snap[i] = m;
        }
    }
}

}  // namespace

void cgint::set_last_error(const std::string& msg) { g_error = msg; }

// ============================================================================ session
struct cg_session {
    cg_config cfg{};
    int32_t mode = CG_MODE_HOGWILD;
    int32_t device = 0;
    cudaStream_t stream = nullptr;
    int32_t V = 0, D = 0, Dp = 0, K = 0;
    int64_t total_tokens = 0;
    int32_t max_depth = 0;
    int32_t cover_depth = 0;  // path length that covers 90% of the kept centers (v8 stages this many path rows)

    // host layout maps (hogwild): node id -> device row and back
    std::vector<int32_t> row_of_node, node_of_row;

    DevBuf<float> model;  // det: syn0[V*D] syn1[(V-1)*D]; hogwild: padded, permuted
    DevBuf<float> sigmoid, keep, stage;
    DevBuf<int32_t> ids, node_of_row_dev, row_of_node_dev;
    int64_t n_ids = 0;

    // det mode
    DevBuf<int64_t> det_off;
    DevBuf<int32_t> det_node, det_slot, det_hot, det_acq;
    DevBuf<uint8_t> det_turn, det_flag;
    DevBuf<float> det_work, det_snap;
    DevBuf<cgk::DetState> det_state;

    // hogwild mode
    DevBuf<int32_t> hw_off, hw_code, kept;
    DevBuf<float> sent_alpha;
    DevBuf<uint32_t> tile_count;
    DevBuf<uint64_t> tile_off;
    DevBuf<unsigned long long> counters;
    cg_tuning tune{0, 0, 0, -1, 0.0f, 0, 0, 0};
    // hogwild: share of the paths through device row r (usage / root usage), for the first
    // min(V-1, kMaxCacheRows) rows (the cacheable ones; device rows are in usage order
    // after the caller's selection)
    std::vector<double> row_share;
    DevBuf<float> tier2;  // hogwild: the L2 tier of the per-CTA cache (zeroed before each launch)
    // replica sync (hogwild): the model at the start of the sync period, the (summed) delta,
    // and per-row update shares for the sync scale: syn0 row w is updated by the centers
    // whose window holds w, device syn1 row r by the centers whose path holds r
    DevBuf<float> snap, delta, sync_scale;
    std::vector<float> row_q;  // [2V]: syn0 rows, then syn1 rows (device order) and the pad row
    double kept_ratio = 1.0;   // expected kept share of the id stream
    int32_t sync_n = -1;
    uint64_t sync_words = 0;
    std::vector<double> ctx_share;  // hogwild: share of centers with word w (w < kCtxCacheRows) in their window
    DevBuf<float> row_scale;
    int scale_blocks = -1, scale_flush = -1;
    int64_t scale_rows = -1;

    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

    float* syn0() const { return model.p; }
    float* syn1() const { return model.p + static_cast<size_t>(V) * (mode == CG_MODE_DETERMINISTIC ? D : Dp); }
    int32_t stride() const { return mode == CG_MODE_DETERMINISTIC ? D : Dp; }

    ~cg_session() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
    }
};

namespace {

float host_sig_scale() { return static_cast<float>(1000) / (2.0f * 6.0f); }

cgk::DetModel det_model(const cg_session& s) {
    cgk::DetModel m{};
    m.syn0 = s.syn0();
    m.syn1 = s.syn1();
    m.dim = s.D;
    m.vocab = s.V;
    m.path_off = s.det_off.p;
    m.path_node = s.det_node.p;
    m.path_turn = s.det_turn.p;
    m.slot_of = s.K > 0 ? s.det_slot.p : nullptr;
    m.hot_nodes = s.det_hot.p;
    m.hot_count = s.K;
    m.cache_work = s.det_work.p;
    m.cache_snap = s.det_snap.p;
    m.cache_flag = s.det_flag.p;
    m.acquired = s.det_acq.p;
    m.sigmoid = s.sigmoid.p;
    m.sig_scale = host_sig_scale();
    return m;
}

// ---- host <-> device copies for pageable host memory ---------------------------------
// A plain cudaMemcpy from/to pageable memory is staged by the driver at ~5 GB/s (23 ms
// for the C2 model), and fresh user pages fault on first touch. Large pageable copies go
// through two pooled pinned buffers instead, with the host-side memcpy split over
// threads and overlapped with the DMA of the next chunk.
bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

void parallel_memcpy(void* dst, const void* src, size_t n) {
    constexpr size_t kMin = size_t{2} << 20;
    const size_t nt = std::min<size_t>(8, std::max<size_t>(1, n / kMin));
    if (nt <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (n + nt - 1) / nt;
    for (size_t t = 1; t < nt; ++t) {
        const size_t b = t * per, e = std::min(n, b + per);
        if (b < e) th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b); });
    }
    std::memcpy(dst, src, std::min(n, per));
    for (auto& x : th) x.join();
}

constexpr size_t kStageBytes = size_t{16} << 20;

void copy_to_host(void* dst, const void* dev_src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes < (size_t{4} << 20) || is_pinned(dst)) {
        CG_CUDA(cudaMemcpyAsync(dst, dev_src, bytes, cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaStreamSynchronize(st));
        return;
    }
    char* stage[2] = {static_cast<char*>(cgint::PinnedPool::get().alloc(kStageBytes)),
                      static_cast<char*>(cgint::PinnedPool::get().alloc(kStageBytes))};
    cudaEvent_t ev[2];
    for (auto& e : ev) CG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t chunks = (bytes + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t c) {
        const size_t b = c * kStageBytes, n = std::min(kStageBytes, bytes - b);
        CG_CUDA(cudaMemcpyAsync(stage[c & 1], static_cast<const char*>(dev_src) + b, n, cudaMemcpyDeviceToHost, st));
        CG_CUDA(cudaEventRecord(ev[c & 1], st));
    };
    issue(0);
    for (size_t c = 0; c < chunks; ++c) {
        if (c + 1 < chunks) issue(c + 1);  // stage[(c+1)&1] was drained in iteration c-1
        CG_CUDA(cudaEventSynchronize(ev[c & 1]));
        const size_t b = c * kStageBytes;
        parallel_memcpy(static_cast<char*>(dst) + b, stage[c & 1], std::min(kStageBytes, bytes - b));
    }
    for (auto& e : ev) cudaEventDestroy(e);
    for (auto* p : stage) cgint::PinnedPool::get().free(p);
}

void copy_to_device(void* dev_dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return;
    if (bytes < (size_t{4} << 20) || is_pinned(src)) {
        CG_CUDA(cudaMemcpyAsync(dev_dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    char* stage[2] = {static_cast<char*>(cgint::PinnedPool::get().alloc(kStageBytes)),
                      static_cast<char*>(cgint::PinnedPool::get().alloc(kStageBytes))};
    cudaEvent_t ev[2];
    for (auto& e : ev) CG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    bool used[2] = {false, false};
    const size_t chunks = (bytes + kStageBytes - 1) / kStageBytes;
    for (size_t c = 0; c < chunks; ++c) {
        const int k = static_cast<int>(c & 1);
        if (used[k]) CG_CUDA(cudaEventSynchronize(ev[k]));  // its previous DMA has finished
        const size_t b = c * kStageBytes, n = std::min(kStageBytes, bytes - b);
        parallel_memcpy(stage[k], static_cast<const char*>(src) + b, n);
        CG_CUDA(cudaMemcpyAsync(static_cast<char*>(dev_dst) + b, stage[k], n, cudaMemcpyHostToDevice, st));
        CG_CUDA(cudaEventRecord(ev[k], st));
        used[k] = true;
    }
    CG_CUDA(cudaStreamSynchronize(st));
    for (auto& e : ev) cudaEventDestroy(e);
    for (auto* p : stage) cgint::PinnedPool::get().free(p);
}

void session_reset_model(cg_session& s) {
    const uint64_t key = cachegram::mix_seed(s.cfg.seed, 0x1817);
    const int32_t st = s.stride();
    CG_CUDA(cudaMemsetAsync(s.model.p, 0, s.model.n * sizeof(float), s.stream));
    const int64_t n = static_cast<int64_t>(s.V) * s.D;
    init_syn0_kernel<<<grid_for(n), 256, 0, s.stream>>>(s.syn0(), s.V, s.D, st, key, 1.0f / static_cast<float>(s.D));
    CG_CUDA(cudaGetLastError());
    if (s.mode == CG_MODE_DETERMINISTIC) {
        cgk::DetState init{};
        init.rng = cachegram::mix_seed(s.cfg.seed, 0);  // trainer.hpp:203, worker 0
        init.alpha = cachegram::update_alpha_host(0, 0, s.cfg.alpha0);
        CG_CUDA(cudaMemcpyAsync(s.det_state.p, &init, sizeof init, cudaMemcpyHostToDevice, s.stream));
        if (s.K > 0) CG_CUDA(cudaMemsetAsync(s.det_flag.p, 0, s.det_flag.n, s.stream));
    }
}

}  // namespace

extern "C" {

int cg_abi_version(void) { return CG_ABI_VERSION; }

void cg_release_cached_memory(void) {
    cgint::DevicePool::get().release();
    cgint::PinnedPool::get().release();
}
const char* cg_last_error(void) { return g_error.c_str(); }

int cg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

double cg_keep_probability(int64_t count, int64_t total_tokens, double sample) {
    return cachegram::keep_probability(count, total_tokens, sample);
}

float cg_update_alpha(uint64_t words_processed, uint64_t total_words, float alpha0) {
    return cachegram::update_alpha_host(words_processed, total_words, alpha0);
}

void cg_sigmoid_table(float* out) {
    const cachegram::SigmoidTable t;
    std::memcpy(out, t.data(), 1000 * sizeof(float));
}

int cg_init_model(int32_t vocab_size, int32_t dim, uint64_t seed, float* syn0) {
    return guarded([&] {
        if (vocab_size < 2) invalid("model needs a vocabulary of at least two words");
        if (dim < 1) invalid("vector dimension must be >= 1");
        cachegram::init_model_into(vocab_size, dim, seed, syn0);
    });
}

int cg_build_huffman(const int64_t* counts, int32_t vocab_size, int64_t* path_offsets, int32_t* path_nodes,
                     uint8_t* path_turns, int64_t* node_usage, int64_t* n_steps) {
    return guarded([&] {
        const cachegram::HuffmanTree t = cachegram::huffman_from_counts(counts, vocab_size);
        if (n_steps) *n_steps = static_cast<int64_t>(t.steps().size());
        if (path_offsets)
            for (size_t i = 0; i < t.offsets().size(); ++i) path_offsets[i] = static_cast<int64_t>(t.offsets()[i]);
        if (path_nodes)
            for (size_t k = 0; k < t.steps().size(); ++k) {
                path_nodes[k] = t.steps()[k].node;
                path_turns[k] = t.steps()[k].turn;
            }
        if (node_usage)
            for (int32_t n = 0; n < t.inner_count(); ++n) node_usage[n] = t.node_usage(n);
    });
}

int32_t cg_select_cached_nodes(const int64_t* node_usage, int32_t inner_count, int32_t k, int32_t* hot_nodes,
                               int32_t* slot_of) {
    int32_t size = -1;
    const int rc = guarded([&] {
        if (k < 0) invalid("cache node count must be >= 0");
        std::vector<int32_t> order(static_cast<size_t>(inner_count));
        for (int32_t i = 0; i < inner_count; ++i) order[static_cast<size_t>(i)] = i;
        std::stable_sort(order.begin(), order.end(),
                         [node_usage](int32_t a, int32_t b) { return node_usage[a] > node_usage[b]; });
        size = std::min(k, inner_count);
        for (int32_t i = 0; i < inner_count; ++i) slot_of[i] = -1;
        for (int32_t s = 0; s < size; ++s) {
            hot_nodes[s] = order[static_cast<size_t>(s)];
            slot_of[order[static_cast<size_t>(s)]] = s;
        }
    });
    return rc == CG_OK ? size : -1;
}

// ---- corpus -------------------------------------------------------------------
}  // extern "C"

struct cg_corpus {
    cachegram::Vocabulary vocab;
};

extern "C" {

int cg_corpus_open(const char* path, int64_t min_count, cg_corpus** out) {
    return guarded([&] {
        if (min_count < 1) invalid("min-count must be >= 1");
        *out = new cg_corpus{cachegram::build_vocabulary_file(path, min_count)};
    });
}
int32_t cg_corpus_vocab_size(const cg_corpus* c) { return c->vocab.size(); }
int64_t cg_corpus_total_tokens(const cg_corpus* c) { return c->vocab.total_tokens(); }
int64_t cg_corpus_word_bytes(const cg_corpus* c) {
    int64_t n = 0;
    for (int32_t i = 0; i < c->vocab.size(); ++i) n += static_cast<int64_t>(c->vocab.word(i).size()) + 1;
    return n;
}
int cg_corpus_export_vocab(const cg_corpus* c, int64_t* counts, char* words) {
    return guarded([&] {
        for (int32_t i = 0; i < c->vocab.size(); ++i) {
            if (counts) counts[i] = c->vocab.count(i);
            if (words) {
                const std::string& w = c->vocab.word(i);
                std::memcpy(words, w.data(), w.size());
                words += w.size();
                *words++ = '\0';
            }
        }
    });
}
int cg_corpus_read_ids(const cg_corpus* c, const char* path, int32_t* ids, int64_t capacity, int64_t* n_ids) {
    return guarded([&] {
        const std::vector<int32_t> v = cachegram::read_id_stream(path, c->vocab);
        if (n_ids) *n_ids = static_cast<int64_t>(v.size());
        if (ids) {
            if (static_cast<int64_t>(v.size()) > capacity) invalid("id buffer too small");
            std::memcpy(ids, v.data(), v.size() * sizeof(int32_t));
        }
    });
}
void cg_corpus_close(cg_corpus* c) { delete c; }

// ---- sessions -------------------------------------------------------------------
int cg_session_create(const cg_config* cfg, int32_t mode, const cg_model_desc* md, int32_t device, void* stream,
                      cg_session** out) {
    *out = nullptr;
    auto s = std::make_unique<cg_session>();
    const int rc = guarded([&] {
        const auto tp0 = std::chrono::steady_clock::now();
        auto tmark = [&](const char* what) {
            if (std::getenv("CG_PROFILE"))
                std::fprintf(stderr, "  create: %-12s %.2f ms\n", what,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count());
        };
        if (!cfg || !md) invalid("null config or model");
        validate_config(*cfg);
        validate_model(*md);
        if (mode != CG_MODE_HOGWILD && mode != CG_MODE_DETERMINISTIC) invalid("unknown training mode");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw CgError(CG_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
        }
        if (device < 0 || device >= ndev) invalid("device ordinal out of range");
        CG_CUDA(cudaSetDevice(device));
        s->cfg = *cfg;
        s->mode = mode;
        s->device = device;
        s->stream = static_cast<cudaStream_t>(stream);
        s->V = md->vocab_size;
        s->D = cfg->dim;
        // Hogwild rows are padded to 32 bytes (8 floats): every row -- in HBM and in the
        // kernel's shared-memory staging -- then starts on a 32-byte boundary. Rows at
        // 16 mod 32 made K1 ~30% slower (C1/C3, profiles/r1_smem_align.jsonl).
        s->Dp = (cfg->dim + 7) / 8 * 8;
        s->K = md->hot_count;
        s->total_tokens = md->total_tokens;
        const int32_t V = s->V;
        const int64_t steps = md->path_offsets[V];
        for (int32_t w = 0; w < V; ++w)
            s->max_depth = std::max<int32_t>(s->max_depth, static_cast<int32_t>(md->path_offsets[w + 1] - md->path_offsets[w]));
        for (auto& e : s->ev) CG_CUDA(cudaEventCreate(&e));
        tmark("validated");

        const cachegram::SigmoidTable table;
        s->sigmoid.upload(table.data(), 1000, s->stream);
        std::vector<float> kp;
        if (cfg->sample > 0.0) {
            kp.resize(static_cast<size_t>(V));
            for (int32_t w = 0; w < V; ++w)
                kp[static_cast<size_t>(w)] =
                    static_cast<float>(cachegram::keep_probability(md->counts[w], md->total_tokens, cfg->sample));
            s->keep.upload(kp.data(), kp.size(), s->stream);
        }
        {  // expected share of centers whose window holds word w, for the most frequent words:
           // (W + 1) x its share of the kept stream (b is uniform on 1..W: E[2b] = W + 1)
            double kept_total = 0.0;
            std::vector<double> kept(static_cast<size_t>(std::min<int32_t>(V, cgk::kCtxCacheRows)));
            for (int32_t w = 0; w < V; ++w) {
                const double kpw = kp.empty() ? 1.0 : std::min(1.0, static_cast<double>(kp[static_cast<size_t>(w)]));
                const double k = static_cast<double>(md->counts[w]) * kpw;
                kept_total += k;
                if (w < static_cast<int32_t>(kept.size())) kept[static_cast<size_t>(w)] = k;
            }
            for (double k : kept) s->ctx_share.push_back(std::min(1.0, (cfg->window + 1) * k / std::max(kept_total, 1.0)));
            {  // the path length that 90% of the kept centers stay within: v8 stages that many
               // path rows per warp and trains the few deeper paths in a second chunk (measured:
               // C4, deepest path 22, 719 ms with 20 staged rows and 9 warps per SM against 753
               // with 24 and 8; C5, deepest 26, 90% within 24: 2338 ms with 24, 2452 with 20)
                std::vector<double> by_len(static_cast<size_t>(s->max_depth) + 1, 0.0);
                for (int32_t w = 0; w < V; ++w) {
                    const double kpw = kp.empty() ? 1.0 : std::min(1.0, static_cast<double>(kp[static_cast<size_t>(w)]));
                    by_len[static_cast<size_t>(md->path_offsets[w + 1] - md->path_offsets[w])] +=
                        static_cast<double>(md->counts[w]) * kpw;
                }
                double run = 0.0;
                s->cover_depth = s->max_depth;
                for (int32_t len = 0; len <= s->max_depth; ++len) {
                    run += by_len[static_cast<size_t>(len)];
                    if (run >= 0.9 * kept_total) {
                        s->cover_depth = len;
                        break;
                    }
                }
            }
            if (mode == CG_MODE_HOGWILD) {
                s->row_q.assign(2 * static_cast<size_t>(V), 0.0f);
                for (int32_t w = 0; w < V; ++w) {
                    const double kpw = kp.empty() ? 1.0 : std::min(1.0, static_cast<double>(kp[static_cast<size_t>(w)]));
                    s->row_q[static_cast<size_t>(w)] = static_cast<float>(
                        std::min(1.0, (cfg->window + 1) * static_cast<double>(md->counts[w]) * kpw / std::max(kept_total, 1.0)));
                }
                s->kept_ratio = kept_total / std::max(1.0, static_cast<double>(md->total_tokens));
            }
        }

        if (mode == CG_MODE_DETERMINISTIC) {
            s->model.alloc(static_cast<size_t>(V) * s->D + static_cast<size_t>(V - 1) * s->D);
            s->det_off.upload(md->path_offsets, static_cast<size_t>(V) + 1, s->stream);
            s->det_node.upload(md->path_nodes, static_cast<size_t>(steps), s->stream);
            s->det_turn.upload(md->path_turns, static_cast<size_t>(steps), s->stream);
            if (s->K > 0) {
                std::vector<int32_t> slot(static_cast<size_t>(V - 1), -1);
                for (int32_t k = 0; k < s->K; ++k) slot[static_cast<size_t>(md->hot_nodes[k])] = k;
                s->det_slot.upload(slot.data(), slot.size(), s->stream);
                s->det_hot.upload(md->hot_nodes, static_cast<size_t>(s->K), s->stream);
                s->det_work.alloc(static_cast<size_t>(s->K) * s->D);
                s->det_snap.alloc(static_cast<size_t>(s->K) * s->D);
                s->det_flag.alloc(static_cast<size_t>(s->K));
                s->det_acq.alloc(static_cast<size_t>(s->K));
            }
            s->det_state.alloc(1);
        } else {
            if (steps >= (int64_t{1} << 31)) invalid("tree too large for 32-bit path offsets");
            if (V >= (1 << 30)) invalid("vocabulary too large for 30-bit device row ids");
            // Device row order: the CacheSelection's rows in slot order (the per-CTA cache
            // holds device rows [0, K), so "cached" is simply row < K), then every other
            // inner node by (usage desc, id asc); one extra all-zero row pads row groups.
            std::vector<char> placed(static_cast<size_t>(V - 1), 0);
            s->node_of_row.reserve(static_cast<size_t>(V - 1));
            for (int32_t k = 0; k < s->K; ++k) {
                s->node_of_row.push_back(md->hot_nodes[k]);
                placed[static_cast<size_t>(md->hot_nodes[k])] = 1;
            }
            std::vector<int32_t> rest;
            rest.reserve(static_cast<size_t>(V - 1 - s->K));
            for (int32_t n = 0; n < V - 1; ++n)
                if (!placed[static_cast<size_t>(n)]) rest.push_back(n);
            std::sort(rest.begin(), rest.end(), [md](int32_t a, int32_t b) {
                return md->node_usage[a] != md->node_usage[b] ? md->node_usage[a] > md->node_usage[b] : a < b;
            });
            s->node_of_row.insert(s->node_of_row.end(), rest.begin(), rest.end());
            tmark("row order");
            const double root = std::max(1.0, static_cast<double>(md->node_usage[V - 2]));
            const int32_t nshare = std::min<int32_t>(V - 1, cgk::kMaxCacheRows);
            for (int32_t r = 0; r < nshare; ++r)
                s->row_share.push_back(static_cast<double>(md->node_usage[s->node_of_row[static_cast<size_t>(r)]]) / root);
            for (int32_t r = 0; r < V - 1; ++r)
                s->row_q[static_cast<size_t>(V) + static_cast<size_t>(r)] =
                    static_cast<float>(static_cast<double>(md->node_usage[s->node_of_row[static_cast<size_t>(r)]]) / root);
            s->row_of_node.assign(static_cast<size_t>(V - 1), 0);
            for (int32_t r = 0; r < V - 1; ++r) s->row_of_node[static_cast<size_t>(s->node_of_row[static_cast<size_t>(r)])] = r;
            std::vector<int32_t> off(static_cast<size_t>(V) + 1);
            for (int32_t w = 0; w <= V; ++w) off[static_cast<size_t>(w)] = static_cast<int32_t>(md->path_offsets[w]);
            s->hw_off.upload(off.data(), off.size(), s->stream);
            s->node_of_row_dev.upload(s->node_of_row.data(), s->node_of_row.size(), s->stream);
            s->row_of_node_dev.upload(s->row_of_node.data(), s->row_of_node.size(), s->stream);
            // path codes (device row << 1 | turn), translated on the device from the tree's
            // node ids and turns (a host pass over every path step took ~1 ms at C2)
            {
                DevBuf<int32_t> nodes;
                DevBuf<uint8_t> turns;
                nodes.upload(md->path_nodes, static_cast<size_t>(steps), s->stream);
                turns.upload(md->path_turns, static_cast<size_t>(steps), s->stream);
                s->hw_code.alloc(static_cast<size_t>(steps));
                path_code_kernel<<<grid_for(steps), 256, 0, s->stream>>>(nodes.p, turns.p, s->row_of_node_dev.p, steps,
                                                                          s->hw_code.p);
                CG_CUDA(cudaGetLastError());
                CG_CUDA(cudaStreamSynchronize(s->stream));  // before the staging buffers go
            }
            tmark("path codes");
            // syn0 [V rows] then syn1 [V-1 rows + 1 zero pad row]
            s->model.alloc(static_cast<size_t>(V) * s->Dp + static_cast<size_t>(V) * s->Dp);
            s->counters.alloc(4);
        }
        tmark("alloc");
        session_reset_model(*s);
        CG_CUDA(cudaStreamSynchronize(s->stream));
        tmark("reset+sync");
    });
    if (rc == CG_OK) *out = s.release();
    return rc;
}

void cg_session_destroy(cg_session* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    delete s;
}

namespace {
__global__ void id_range_kernel(const int32_t* ids, int64_t n, int32_t V, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (ids[i] < 0 || ids[i] >= V) atomicAdd(bad, 1ull);
}

// Every id must index the vocabulary (checked on the device: a host loop over 10^9 ids
// costs a second of the end-to-end time).
void check_ids_on_device(cg_session* s) {
    DevBuf<unsigned long long> bad;
    bad.alloc(1);
    CG_CUDA(cudaMemsetAsync(bad.p, 0, 8, s->stream));
    if (s->n_ids > 0) id_range_kernel<<<grid_for(s->n_ids), 256, 0, s->stream>>>(s->ids.p, s->n_ids, s->V, bad.p);
    CG_CUDA(cudaGetLastError());
    unsigned long long nbad = 0;
    CG_CUDA(cudaMemcpyAsync(&nbad, bad.p, 8, cudaMemcpyDeviceToHost, s->stream));
    CG_CUDA(cudaStreamSynchronize(s->stream));
    if (nbad) {
        s->n_ids = 0;
        invalid("id out of vocabulary range");
    }
}

void session_alloc_stream(cg_session* s, int64_t n_ids) {
    s->n_ids = n_ids;
    if (s->mode == CG_MODE_HOGWILD) {
        s->kept.alloc(static_cast<size_t>(std::max<int64_t>(n_ids, 1)));
        s->sent_alpha.alloc(static_cast<size_t>(n_ids / cgdev::kSentence + 2));
        const int64_t nt = cgk::sub_tiles(n_ids);
        s->tile_count.alloc(static_cast<size_t>(std::max<int64_t>(nt, 1)));
        s->tile_off.alloc(static_cast<size_t>(nt + 1));
    }
}
}  // namespace

int cg_session_upload_ids(cg_session* s, const int32_t* ids, int64_t n_ids) {
    return guarded([&] {
        if (n_ids < 0) invalid("negative id count");
        CG_CUDA(cudaSetDevice(s->device));
        s->ids.alloc(static_cast<size_t>(n_ids));
        copy_to_device(s->ids.p, ids, static_cast<size_t>(n_ids) * sizeof(int32_t), s->stream);
        session_alloc_stream(s, n_ids);
        check_ids_on_device(s);
    });
}

int cg_session_upload_ids_device(cg_session* s, const int32_t* device_ids, int64_t n_ids) {
    return guarded([&] {
        if (n_ids < 0) invalid("negative id count");
        CG_CUDA(cudaSetDevice(s->device));
        s->ids.alloc(static_cast<size_t>(n_ids));
        if (n_ids)
            CG_CUDA(cudaMemcpyAsync(s->ids.p, device_ids, static_cast<size_t>(n_ids) * 4, cudaMemcpyDeviceToDevice,
                                    s->stream));
        session_alloc_stream(s, n_ids);
        CG_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int cg_session_reset_model(cg_session* s) {
    return guarded([&] {
        CG_CUDA(cudaSetDevice(s->device));
        session_reset_model(*s);
        CG_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int cg_session_set_model(cg_session* s, const float* syn0, const float* syn1) {
    return guarded([&] {
        CG_CUDA(cudaSetDevice(s->device));
        const size_t n0 = static_cast<size_t>(s->V) * s->D, n1 = static_cast<size_t>(s->V - 1) * s->D;
        if (s->mode == CG_MODE_DETERMINISTIC) {
            CG_CUDA(cudaMemcpyAsync(s->syn0(), syn0, n0 * 4, cudaMemcpyHostToDevice, s->stream));
            CG_CUDA(cudaMemcpyAsync(s->syn1(), syn1, n1 * 4, cudaMemcpyHostToDevice, s->stream));
        } else {
            s->stage.alloc(n0 + n1);
            CG_CUDA(cudaMemcpyAsync(s->stage.p, syn0, n0 * 4, cudaMemcpyHostToDevice, s->stream));
            CG_CUDA(cudaMemcpyAsync(s->stage.p + n0, syn1, n1 * 4, cudaMemcpyHostToDevice, s->stream));
            CG_CUDA(cudaMemsetAsync(s->model.p, 0, s->model.n * 4, s->stream));
            scatter_rows_kernel<<<grid_for(static_cast<int64_t>(n0)), 256, 0, s->stream>>>(s->syn0(), s->Dp, s->stage.p, s->D, nullptr, s->V, s->D);
            scatter_rows_kernel<<<grid_for(static_cast<int64_t>(n1)), 256, 0, s->stream>>>(s->syn1(), s->Dp, s->stage.p + n0, s->D, s->row_of_node_dev.p, s->V - 1, s->D);
            CG_CUDA(cudaGetLastError());
        }
        CG_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int cg_session_download(cg_session* s, float* syn0_out, float* syn1_out) {
    return guarded([&] {
        CG_CUDA(cudaSetDevice(s->device));
        const size_t n0 = static_cast<size_t>(s->V) * s->D, n1 = static_cast<size_t>(s->V - 1) * s->D;
        if (s->mode == CG_MODE_DETERMINISTIC) {
            if (syn0_out) copy_to_host(syn0_out, s->syn0(), n0 * 4, s->stream);
            if (syn1_out) copy_to_host(syn1_out, s->syn1(), n1 * 4, s->stream);
        } else {
            if (s->stage.n < n0 + n1) s->stage.alloc(n0 + n1);
            gather_rows_kernel<<<grid_for(static_cast<int64_t>(n0)), 256, 0, s->stream>>>(s->stage.p, s->D, s->syn0(), s->Dp, nullptr, s->V, s->D);
            gather_rows_kernel<<<grid_for(static_cast<int64_t>(n1)), 256, 0, s->stream>>>(s->stage.p + n0, s->D, s->syn1(), s->Dp, s->row_of_node_dev.p, s->V - 1, s->D);
            CG_CUDA(cudaGetLastError());
            if (syn0_out) copy_to_host(syn0_out, s->stage.p, n0 * 4, s->stream);
            if (syn1_out) copy_to_host(syn1_out, s->stage.p + n0, n1 * 4, s->stream);
        }
        CG_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int cg_session_model_buffer(cg_session* s, void** device_ptr, size_t* bytes, int32_t* row_stride_floats) {
    return guarded([&] {
        if (device_ptr) *device_ptr = s->model.p;
        if (bytes) *bytes = s->model.n * sizeof(float);
        if (row_stride_floats) *row_stride_floats = s->stride();
    });
}

// Sync scale of one row whose share of the updates is q when n replicas each train
// `centers` kept centers between syncs. The reference's workers all add
// into one model (trainer.hpp:72-74, 249-253), so deltas are summed across replicas, but
// a row every replica updates from the same snapshot receives n x q x centers stale
// updates per sync: the sum is capped at H = 128 stale updates' worth and never scaled
// below the average of the replicas that touched it (the per-CTA flush rule of K1, with
// replicas for CTAs; replicas see their own updates between syncs, and tolerate 4x the
// staleness of a CTA's write-combined cache rows: profiles/r2_replica*_c1.jsonl).
float cg_sync_row_scale(double q, int32_t n_replicas, double centers) {
    if (n_replicas <= 1) return 1.0f;
    q = std::min(std::max(q, 0.0), 1.0);
    const double n = static_cast<double>(n_replicas);
    const double p = 1.0 - std::pow(1.0 - q, std::max(centers, 0.0));
    const double avg = 1.0 / std::max(1.0, p * n);
    constexpr double H = 128.0;  // stable to 256 at N = 8 on C1; 512 diverged (profiles/r2_replica2_*)
    const double stale = H / std::max(1e-30, n * q * centers);
    return static_cast<float>(std::min(1.0, std::max(avg, stale)));
}

int cg_session_sync_begin(cg_session* s) {
    return guarded([&] {
        if (s->mode != CG_MODE_HOGWILD) invalid("replica sync needs a hogwild session");
        CG_CUDA(cudaSetDevice(s->device));
        if (s->snap.n != s->model.n) s->snap.alloc(s->model.n);
        CG_CUDA(cudaMemcpyAsync(s->snap.p, s->model.p, s->model.n * 4, cudaMemcpyDeviceToDevice, s->stream));
        CG_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int cg_session_sync_delta(cg_session* s, void** delta_dev, size_t* n_floats) {
    return guarded([&] {
        if (s->snap.n != s->model.n) invalid("cg_session_sync_begin was not called");
        CG_CUDA(cudaSetDevice(s->device));
        // the delta in the model's layout, then one squared norm per model row (padded to 4),
        // then the squared norms of the two matrices (4 floats)
        const size_t rows = s->model.n / static_cast<size_t>(s->Dp);
        const size_t tail = sync_tail_rows(rows);
        const size_t total = s->model.n + tail + 4;
        if (s->delta.n != total) s->delta.alloc(total);
        CG_CUDA(cudaMemsetAsync(s->delta.p + s->model.n, 0, (tail + 4) * sizeof(float), s->stream));
        sync_delta_kernel<<<148 * 8, 256, 0, s->stream>>>(
            reinterpret_cast<const float4*>(s->model.p), reinterpret_cast<const float4*>(s->snap.p),
            reinterpret_cast<float4*>(s->delta.p), s->delta.p + s->model.n, s->delta.p + s->model.n + tail, rows,
            static_cast<size_t>(s->V), s->Dp / 4);
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaStreamSynchronize(s->stream));
        if (delta_dev) *delta_dev = s->delta.p;
        if (n_floats) *n_floats = s->delta.n;
    });
}

int cg_session_sync_apply(cg_session* s, int32_t n_replicas, uint64_t words_per_replica) {
    return guarded([&] {
        const size_t rows = s->model.n / static_cast<size_t>(s->Dp);
        const size_t tail = sync_tail_rows(rows);
        if (s->snap.n != s->model.n || s->delta.n != s->model.n + tail + 4)
            invalid("cg_session_sync_delta was not called");
        if (n_replicas < 1) invalid("replica count must be >= 1");
        CG_CUDA(cudaSetDevice(s->device));
        if (s->sync_n != n_replicas || s->sync_words != words_per_replica) {
            const double centers = s->kept_ratio * static_cast<double>(words_per_replica);
            std::vector<float> sc(s->row_q.size());
            for (size_t r = 0; r < sc.size(); ++r) sc[r] = cg_sync_row_scale(s->row_q[r], n_replicas, centers);
            s->sync_scale.upload(sc.data(), sc.size(), s->stream);
            s->sync_n = n_replicas;
            s->sync_words = words_per_replica;
        }
        sync_apply_kernel<<<148 * 8, 256, 0, s->stream>>>(
            reinterpret_cast<float4*>(s->model.p), reinterpret_cast<float4*>(s->snap.p),
            reinterpret_cast<const float4*>(s->delta.p), s->delta.p + s->model.n, s->delta.p + s->model.n + tail,
            s->sync_scale.p, rows, static_cast<size_t>(s->V), s->Dp / 4, 1.0f / static_cast<float>(n_replicas));
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int cg_session_tune(cg_session* s, const cg_tuning* t) {
    return guarded([&] {
        if (!t) invalid("null tuning");
        if (t->smem_cache_rows > cgk::kMaxCacheRows) invalid("smem_cache_rows out of range");
        if (t->kernel != 0 && t->kernel != 5 && t->kernel != 8) invalid("kernel must be 0, 5 or 8");
        s->tune = *t;
    });
}

int cg_session_train_range(cg_session* s, int32_t epoch, int64_t tok_begin, int64_t tok_end, uint64_t progress_base,
                           uint32_t progress_mult, cg_epoch_stats* st) {
    return guarded([&] {
        CG_CUDA(cudaSetDevice(s->device));
        if (tok_begin < 0 || tok_end > s->n_ids || tok_begin > tok_end) invalid("token range out of bounds");
        if (progress_mult < 1) invalid("progress_mult must be >= 1");
        cg_epoch_stats out{};
        const int64_t n = tok_end - tok_begin;
        const uint64_t total_words = static_cast<uint64_t>(s->cfg.iterations) * static_cast<uint64_t>(s->total_tokens);
        out.words = static_cast<uint64_t>(n);
        if (s->mode == CG_MODE_DETERMINISTIC) {
            cgk::DetPass p{};
            p.ids = s->ids.p + tok_begin;
            p.n_ids = n;
            p.keep = s->keep.p;
            p.window = s->cfg.window;
            p.flush_interval = s->cfg.flush_interval;
            p.total_words = total_words;
            p.alpha0 = s->cfg.alpha0;
            cgk::DetState before{};
            CG_CUDA(cudaMemcpyAsync(&before, s->det_state.p, sizeof before, cudaMemcpyDeviceToHost, s->stream));
            CG_CUDA(cudaEventRecord(s->ev[2], s->stream));
            cgk::launch_det_pass(det_model(*s), p, s->det_state.p, s->stream);
            CG_CUDA(cudaGetLastError());
            CG_CUDA(cudaEventRecord(s->ev[3], s->stream));
            cgk::DetState after{};
            CG_CUDA(cudaMemcpyAsync(&after, s->det_state.p, sizeof after, cudaMemcpyDeviceToHost, s->stream));
            CG_CUDA(cudaStreamSynchronize(s->stream));
            float ms = 0.f;
            CG_CUDA(cudaEventElapsedTime(&ms, s->ev[2], s->ev[3]));
            out.train_ms = ms;
            out.kept = after.centers - before.centers;
            out.pairs = after.pairs - before.pairs;
            out.steps = after.steps - before.steps;
            out.train_launches = 1;
        } else {
            cgk::SubArgs a{};
            a.ids = s->ids.p + tok_begin;
            a.n = n;
            a.index_base = tok_begin;
            a.keep = s->keep.p;
            a.key = cgdev::mix64(s->cfg.seed ^ 0x5ab5a3b1e5d00d1full) + 0x100000001b3ull * static_cast<uint64_t>(epoch);
            a.tile_count = s->tile_count.p;
            a.tile_off = s->tile_off.p;
            a.kept = s->kept.p;
            a.sent_alpha = s->sent_alpha.p;
            a.progress_base = progress_base;
            a.progress_mult = progress_mult;
            a.total_words = total_words;
            a.alpha0 = s->cfg.alpha0;
            CG_CUDA(cudaEventRecord(s->ev[0], s->stream));
            int sub_launches = 0;
            cgk::launch_subsample(a, s->stream, &sub_launches);
            CG_CUDA(cudaGetLastError());
            CG_CUDA(cudaMemsetAsync(s->counters.p, 0, 4 * sizeof(unsigned long long), s->stream));
            CG_CUDA(cudaEventRecord(s->ev[1], s->stream));
            cgk::HogArgs h{};
            h.syn0 = s->syn0();
            h.syn1 = s->syn1();
            h.d4 = s->Dp / 4;
            h.path_off = s->hw_off.p;
            h.path_code = s->hw_code.p;
            h.kept = s->kept.p;
            h.n_kept_dev = s->tile_off.p + cgk::sub_tiles(n);
            h.sent_alpha = s->sent_alpha.p;
            h.sigmoid = s->sigmoid.p;
            h.sig_scale = host_sig_scale();
            h.window = s->cfg.window;
            h.win_key = cgdev::mix64(s->cfg.seed ^ 0x77696e646f77ull) + 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(epoch + 1);
            h.counters = s->counters.p;
            // ---- the per-CTA cache (NodeCache, trainer.hpp:75-138) at GPU concurrency ----
            // K = cache_nodes rows are cached: the CacheSelection's rows, which lead the
            // device row order. K1 runs ~1500 warps at once, and a row on the paths of a
            // share q of the centers then has ~q x 1500 concurrent updaters; uncached, the
            // top-of-tree rows (q ~ 1) take ~10^3 stale updates at once and training
            // diverges. So on top of K the cache always holds the leading rows
            // whose expected concurrent updaters reach kHotUpdaters (the stability floor,
            // cg_tuning.min_cache_rows; < 0 disables it, which honours K = 0 literally).
            constexpr double kHotUpdaters = 256.0;
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
            const int blocks = s->tune.blocks > 0 ? s->tune.blocks : sms;
            // K1 version: v8 (tensor cores) or v5; the warps in flight set the stability floor
            cgk::HogGeometry g{};
            // v8 (tensor cores) unless the caller asked for v5 (FP32 FMA) or the rows are too wide
            auto plan_tc = [&](int32_t rows, int32_t ctx) {
                return s->tune.kernel != 5 && cgk::hog8_plan(s->Dp / 4, rows, ctx, blocks, s->tune.warps_per_block,
                                                             s->tune.centers_per_warp, n, s->cover_depth, s->cfg.window, &g);
            };
            bool v8 = plan_tc(std::min<int32_t>(s->K, cgk::kMaxCacheRows), 0);
            const double inflight =
                static_cast<double>(blocks) * (v8 ? g.warps : cgk::hog_max_warps(s->Dp / 4, s->max_depth));
            int32_t floor_rows = 0;
            if (s->tune.min_cache_rows == 0) {
                for (int32_t r = 0; r < static_cast<int32_t>(s->row_share.size()); ++r)
                    if (s->row_share[static_cast<size_t>(r)] * inflight >= kHotUpdaters) floor_rows = r + 1;
            } else if (s->tune.min_cache_rows > 0) {
                floor_rows = s->tune.min_cache_rows;
            }
            const int32_t want_rows = std::min<int32_t>({std::max(s->K, floor_rows), s->V - 1, cgk::kMaxCacheRows});
            // The most frequent words' syn0 rows are cached too when their expected number of
            // concurrent updaters -- the share of centers with the word in their window x the
            // warps training at once -- reaches kHotUpdaters. Without subsampling (sample 0)
            // the top words of C1/C2 reach ~1400 and summed stale updates diverged; cached
            // and averaged, the loss matches the reference's (6.6130 vs 6.6128 at C1). With
            // subsampling no word of C1-C5 gets there, and averaging would slow their learning.
            int32_t ctx_rows = 0;
            while (ctx_rows < static_cast<int32_t>(s->ctx_share.size()) &&
                   s->ctx_share[static_cast<size_t>(ctx_rows)] * inflight >= kHotUpdaters)
                ++ctx_rows;
            h.dummy_row = s->V - 1;
            if (v8) v8 = plan_tc(want_rows, ctx_rows);
            if (!v8)
                g = cgk::hog_plan(h.d4, s->max_depth, want_rows, s->tune.smem_cache_rows, s->tune.blocks,
                                  s->tune.warps_per_block, s->tune.centers_per_warp, s->cfg.window, n, ctx_rows);
            if (g.smem == 0) invalid("dim too large for the generic kernel's shared-memory row buffers");
            // flush_interval u (trainer.hpp:127): each worker warp flushes every u of its
            // centers in the reference; here a CTA's workers share one cache, so it is
            // drained every u x (worker warps) merged centers.
            h.flush_centers = s->tune.flush_centers > 0 ? s->tune.flush_centers
                                                          : std::max(1, s->cfg.flush_interval * g.warps);
            // The L2 tier: rows [S, K) of every CTA's cache, zeroed before each launch (the
            // kernel leaves it zero; re-zeroing keeps an aborted launch from leaking deltas).
            const size_t t2n = static_cast<size_t>(g.blocks) *
                               static_cast<size_t>(g.cache_rows - g.smem_rows + (g.variant >= 7 ? g.ctx_rows : 0)) * s->Dp;
            h.tier2 = nullptr;
            if (t2n > 0) {
                if (s->tier2.n < t2n) s->tier2.alloc(t2n);
                CG_CUDA(cudaMemsetAsync(s->tier2.p, 0, t2n * sizeof(float), s->stream));
                h.tier2 = s->tier2.p;
            }
            // Each CTA trains its own replica of the cached rows between flushes. The paper
            // sums the workers' deltas (trainer.hpp:116-119); at GPU concurrency that sum is a
            // step computed from one stale snapshot by every contributing CTA. A row on the
            // paths of a share q of the centers gets, per flush period of F merged centers per
            // CTA, about n_CTA x q x F such updates: for the root (q = 1) ~10^4, and summed they
            // overshoot and diverge. The flush therefore scales each row's delta
            // by s = min(1, max(1 / (p n_CTA), H / (q (n_CTA F + warps in flight)))): at most
            // H = 32 stale updates' worth per flush (8x below where C1 diverged,
            // profiles/r2_rule3_c1.jsonl), never
            // less than the average of the p n_CTA contributing replicas (p = 1 - (1 - q)^F,
            // the chance that a CTA touches the row in a period), and the plain sum of the
            // reference for rows few CTAs touch.
            h.hot_flush_scale = s->tune.hot_flush_scale > 0.0f ? s->tune.hot_flush_scale : 1.0f / static_cast<float>(g.blocks);
            h.row_scale = nullptr;
            if (s->tune.hot_flush_scale <= 0.0f && (g.cache_rows > 0 || g.ctx_rows > 0)) {
                if (s->scale_blocks != g.blocks || s->scale_flush != h.flush_centers ||
                    s->scale_rows != static_cast<int64_t>(g.cache_rows) * 4096 + g.ctx_rows) {
                    // syn1 cached rows [0, cache_rows), then the cached syn0 rows [0, ctx_rows)
                    std::vector<float> sc(static_cast<size_t>(g.cache_rows + g.ctx_rows));
                    constexpr double kStaleUpdates = 32.0;
                    // warps in flight besides the CTA replicas: a flush lands while the other
                    // CTAs' warps are mid-center on the old value (dominant for small F)
                    const double inflight_w = static_cast<double>(g.blocks) * g.warps;
                    auto scale_of = [&](double q) {
                        q = std::min(std::max(q, 0.0), 1.0);
                        const double p = 1.0 - std::pow(1.0 - q, static_cast<double>(h.flush_centers));
                        const double avg = 1.0 / std::max(1.0, p * g.blocks);
                        const double stale =
                            kStaleUpdates / std::max(1e-30, q * (static_cast<double>(g.blocks) * h.flush_centers + inflight_w));
                        return static_cast<float>(std::min(1.0, std::max(avg, stale)));
                    };
                    for (int32_t r = 0; r < g.cache_rows; ++r)
                        sc[static_cast<size_t>(r)] =
                            scale_of(r < static_cast<int32_t>(s->row_share.size()) ? s->row_share[static_cast<size_t>(r)] : 0.0);
                    for (int32_t r = 0; r < g.ctx_rows; ++r)
                        sc[static_cast<size_t>(g.cache_rows + r)] =
                            scale_of(r < static_cast<int32_t>(s->ctx_share.size()) ? s->ctx_share[static_cast<size_t>(r)] : 0.0);
                    s->row_scale.upload(sc.data(), sc.size(), s->stream);
                    s->scale_blocks = g.blocks;
                    s->scale_flush = h.flush_centers;
                    s->scale_rows = static_cast<int64_t>(g.cache_rows) * 4096 + g.ctx_rows;
                }
                h.row_scale = s->row_scale.p;
            }
            CG_CUDA(cudaEventRecord(s->ev[2], s->stream));
            cgk::launch_hogwild(h, g, s->stream);
            CG_CUDA(cudaGetLastError());
            CG_CUDA(cudaEventRecord(s->ev[3], s->stream));
            unsigned long long cnt[4] = {0, 0, 0, 0};
            uint64_t kept = 0;
            CG_CUDA(cudaMemcpyAsync(cnt, s->counters.p, sizeof cnt, cudaMemcpyDeviceToHost, s->stream));
            CG_CUDA(cudaMemcpyAsync(&kept, h.n_kept_dev, sizeof kept, cudaMemcpyDeviceToHost, s->stream));
            CG_CUDA(cudaStreamSynchronize(s->stream));
            float sub_ms = 0.f, tr_ms = 0.f;
            CG_CUDA(cudaEventElapsedTime(&sub_ms, s->ev[0], s->ev[1]));
            CG_CUDA(cudaEventElapsedTime(&tr_ms, s->ev[2], s->ev[3]));
            out.subsample_ms = sub_ms;
            out.train_ms = tr_ms;
            out.kept = kept;
            out.pairs = cnt[1];
            out.steps = cnt[2];
            out.train_launches = 1;
            out.other_launches = sub_launches;
            out.cached_rows = g.cache_rows;
            out.smem_rows = g.smem_rows;
            out.floor_rows = floor_rows;
            out.flush_centers = h.flush_centers;
            out.kernel = g.variant == 8 ? 8 : (g.variant == 0 ? 0 : 5);
            out.worker_warps = g.warps;
            out.ctx_batch = g.ctx_batch;
            out.blocks = g.blocks;
            if (cnt[3] != kept) throw CgError(CG_ERR_INTERNAL, "hogwild kernel did not cover every kept center");
        }
        if (st) *st = out;
    });
}

int cg_session_train(cg_session* s, cg_train_stats* st) {
    return guarded([&] {
        cg_train_stats out{};
        const auto t0 = std::chrono::steady_clock::now();
        for (int32_t it = 0; it < s->cfg.iterations; ++it) {
            cg_epoch_stats e{};
            const int rc = cg_session_train_range(s, it, 0, s->n_ids,
                                                  static_cast<uint64_t>(it) * static_cast<uint64_t>(s->n_ids), 1, &e);
            if (rc != CG_OK) throw CgError(rc, g_error);
            out.kernel_seconds += (e.train_ms + e.subsample_ms) * 1e-3;
            out.centers += e.kept;
            out.pairs += e.pairs;
            out.steps += e.steps;
            out.words_processed += e.words;
        }
        out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out.words_per_second = out.wall_seconds > 0 ? static_cast<double>(out.words_processed) / out.wall_seconds : 0.0;
        if (st) *st = out;
    });
}

}  // extern "C"

namespace {
// cg_train's Hogwild path for long id streams: the first pass trains chunk by chunk while
// the ids are still crossing PCIe. A producer thread copies chunk c into the session's id
// buffer on its own stream, checks its ids on the device and records an event; the caller's
// thread waits for the event and trains the chunk (the draws are keyed by the global token
// index, so only the sentence cuts at chunk edges differ from one launch, as in
// train_file_pipelined). Chunks ramp up from 4M ids so training starts early.
constexpr int64_t kPipelineMinIds = int64_t{32} << 20;
// CG_PIPELINE_MIN_IDS / CG_PIPELINE_FIRST override the threshold and the first chunk (tests).
int64_t env_ids(const char* name, int64_t fallback) {
    const char* e = std::getenv(name);
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? static_cast<int64_t>(v) : fallback;
}
void train_ids_pipelined(cg_session* s, const int32_t* ids, int64_t n, cg_train_stats* out) {
    CG_CUDA(cudaSetDevice(s->device));
    s->ids.alloc(static_cast<size_t>(n));
    session_alloc_stream(s, n);
    std::vector<int64_t> cut{0};
    for (int64_t len = env_ids("CG_PIPELINE_FIRST", int64_t{4} << 20); cut.back() < n;
         len = std::min<int64_t>(len * 2, int64_t{64} << 20))
        cut.push_back(std::min(n, cut.back() + len));
    const int chunks = static_cast<int>(cut.size()) - 1;
    cudaStream_t cst = nullptr;
    CG_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(static_cast<size_t>(chunks));
    for (auto& e : ev) CG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    auto* flags = static_cast<unsigned long long*>(cgint::PinnedPool::get().alloc(static_cast<size_t>(chunks) * 8));
    DevBuf<unsigned long long> bad;
    bad.alloc(1);
    CG_CUDA(cudaMemsetAsync(bad.p, 0, 8, cst));
    std::mutex mu;
    std::condition_variable cv;
    int ready = 0;
    std::exception_ptr perr;
    std::thread producer([&] {
        try {
            CG_CUDA(cudaSetDevice(s->device));
            for (int c = 0; c < chunks; ++c) {
                const int64_t a = cut[static_cast<size_t>(c)], len = cut[static_cast<size_t>(c) + 1] - a;
                copy_to_device(s->ids.p + a, ids + a, static_cast<size_t>(len) * sizeof(int32_t), cst);
                id_range_kernel<<<grid_for(len), 256, 0, cst>>>(s->ids.p + a, len, s->V, bad.p);
                CG_CUDA(cudaGetLastError());
                CG_CUDA(cudaMemcpyAsync(flags + c, bad.p, 8, cudaMemcpyDeviceToHost, cst));
                CG_CUDA(cudaEventRecord(ev[static_cast<size_t>(c)], cst));
                {
                    std::lock_guard<std::mutex> g(mu);
                    ready = c + 1;
                }
                cv.notify_one();
            }
        } catch (...) {
            perr = std::current_exception();
            {
                std::lock_guard<std::mutex> g(mu);
                ready = chunks + 1;  // wakes the trainer; perr tells it why
            }
            cv.notify_one();
        }
    });
    cg_train_stats st{};
    std::string err;
    int err_rc = CG_OK;
    auto add = [&st](const cg_epoch_stats& e) {
        st.kernel_seconds += (e.train_ms + e.subsample_ms) * 1e-3;
        st.centers += e.kept;
        st.pairs += e.pairs;
        st.steps += e.steps;
        st.words_processed += e.words;
    };
    for (int c = 0; c < chunks && err_rc == CG_OK; ++c) {
        {
            std::unique_lock<std::mutex> g(mu);
            cv.wait(g, [&] { return ready > c; });
            if (ready > chunks) break;  // the producer failed
        }
        CG_CUDA(cudaEventSynchronize(ev[static_cast<size_t>(c)]));
        if (flags[c]) {
            err_rc = CG_ERR_INVALID_ARGUMENT;
            err = "id out of vocabulary range";
            break;
        }
        cg_epoch_stats e{};
        const int64_t a = cut[static_cast<size_t>(c)], b = cut[static_cast<size_t>(c) + 1];
        const int rc = cg_session_train_range(s, 0, a, b, static_cast<uint64_t>(a), 1, &e);
        if (rc != CG_OK) {
            err_rc = rc;
            err = g_error;
            break;
        }
        add(e);
    }
    producer.join();
    cudaStreamSynchronize(cst);
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(cst);
    cgint::PinnedPool::get().free(flags);
    if (perr) std::rethrow_exception(perr);
    if (err_rc != CG_OK) {
        s->n_ids = 0;
        throw CgError(err_rc, err);
    }
    for (int32_t it = 1; it < s->cfg.iterations; ++it) {
        cg_epoch_stats e{};
        const int rc = cg_session_train_range(s, it, 0, n, static_cast<uint64_t>(it) * static_cast<uint64_t>(n), 1, &e);
        if (rc != CG_OK) throw CgError(rc, g_error);
        add(e);
    }
    *out = st;
}
}  // namespace

extern "C" {

int cg_train(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const int32_t* ids, int64_t n_ids,
             float* syn0_out, float* syn1_out, cg_train_stats* stats) {
    cg_session* s = nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    const auto tc = std::chrono::steady_clock::now();
    int rc = cg_session_create(cfg, mode, model, dev, nullptr, &s);
    if (rc != CG_OK) return rc;
    const auto t0 = std::chrono::steady_clock::now();
    cg_train_stats st{};
    auto t1 = t0;
    if (mode == CG_MODE_HOGWILD && ids && n_ids >= env_ids("CG_PIPELINE_MIN_IDS", kPipelineMinIds) &&
        !std::getenv("CG_NO_PIPELINE")) {
        rc = guarded([&] { train_ids_pipelined(s, ids, n_ids, &st); });
    } else {
        rc = cg_session_upload_ids(s, ids, n_ids);
        t1 = std::chrono::steady_clock::now();
        if (rc == CG_OK) rc = cg_session_train(s, &st);
    }
    const auto t2 = std::chrono::steady_clock::now();
    if (rc == CG_OK) rc = cg_session_download(s, syn0_out, syn1_out);
    const auto t3 = std::chrono::steady_clock::now();
    st.wall_seconds = std::chrono::duration<double>(t3 - t0).count();
    if (std::getenv("CG_PROFILE")) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "cg_train: create %.2f ms, upload %.2f ms, train %.2f ms (kernels %.2f), download %.2f ms\n",
                     ms(tc, t0), ms(t0, t1), ms(t1, t2), st.kernel_seconds * 1e3, ms(t2, t3));
    }
    st.words_per_second = st.wall_seconds > 0 ? static_cast<double>(st.words_processed) / st.wall_seconds : 0.0;
    if (stats) *stats = st;
    cg_session_destroy(s);
    return rc;
}

// ---- kernel-level entries ---------------------------------------------------------
}  // extern "C"

namespace {
// Device copies of one train_center call's operands (kernel-level entries; tests).
struct CenterCall {
    DevBuf<float> d0, d1, work, snap, sig, buf;
    DevBuf<int64_t> off;
    DevBuf<int32_t> node, slot, sent, acq, nacq;
    DevBuf<uint8_t> turn, flag;
    DevBuf<unsigned long long> evals;
    cgk::DetModel m{};
    size_t n0 = 0, n1 = 0;
    int32_t hot = 0, dim = 0;

    void up(const int32_t* sentence, int64_t len, int32_t V, int32_t D, float* syn0, float* syn1,
            const int64_t* path_offsets, const int32_t* path_nodes, const uint8_t* path_turns, const int32_t* slot_of,
            int32_t hot_count, float* cache_work, float* cache_snap, uint8_t* cache_flag) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw CgError(CG_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
        }
        hot = hot_count;
        dim = D;
        n0 = static_cast<size_t>(V) * D;
        n1 = static_cast<size_t>(V - 1) * D;
        const int64_t steps = path_offsets[V];
        d0.upload(syn0, n0, nullptr);
        d1.upload(syn1, n1, nullptr);
        off.upload(path_offsets, static_cast<size_t>(V) + 1, nullptr);
        node.upload(path_nodes, static_cast<size_t>(steps), nullptr);
        turn.upload(path_turns, static_cast<size_t>(steps), nullptr);
        sent.upload(sentence, static_cast<size_t>(len), nullptr);
        const cachegram::SigmoidTable table;
        sig.upload(table.data(), 1000, nullptr);
        int32_t zero = 0;
        nacq.upload(&zero, 1, nullptr);
        evals.alloc(1);
        m.syn0 = d0.p;
        m.syn1 = d1.p;
        m.dim = D;
        m.vocab = V;
        m.path_off = off.p;
        m.path_node = node.p;
        m.path_turn = turn.p;
        m.sigmoid = sig.p;
        m.sig_scale = host_sig_scale();
        if (hot_count > 0) {
            slot.upload(slot_of, static_cast<size_t>(V - 1), nullptr);
            work.upload(cache_work, static_cast<size_t>(hot_count) * D, nullptr);
            snap.upload(cache_snap, static_cast<size_t>(hot_count) * D, nullptr);
            flag.upload(cache_flag, static_cast<size_t>(hot_count), nullptr);
            acq.alloc(static_cast<size_t>(hot_count));
            m.slot_of = slot.p;
            m.hot_count = hot_count;
            m.cache_work = work.p;
            m.cache_snap = snap.p;
            m.cache_flag = flag.p;
            m.acquired = acq.p;
        }
    }
    void down(float* syn0, float* syn1, float* cache_work, float* cache_snap, uint8_t* cache_flag) {
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpy(syn0, d0.p, n0 * 4, cudaMemcpyDeviceToHost));
        CG_CUDA(cudaMemcpy(syn1, d1.p, n1 * 4, cudaMemcpyDeviceToHost));
        if (hot > 0) {
            CG_CUDA(cudaMemcpy(cache_work, work.p, static_cast<size_t>(hot) * dim * 4, cudaMemcpyDeviceToHost));
            CG_CUDA(cudaMemcpy(cache_snap, snap.p, static_cast<size_t>(hot) * dim * 4, cudaMemcpyDeviceToHost));
            CG_CUDA(cudaMemcpy(cache_flag, flag.p, static_cast<size_t>(hot), cudaMemcpyDeviceToHost));
        }
    }
};

void check_center_args(int32_t center, int64_t sentence_len, int64_t center_pos, int32_t half_window,
                       int32_t vocab_size, int32_t dim, const int32_t* slot_of, int32_t hot_count, float* cache_work,
                       float* cache_snap, uint8_t* cache_flag) {
    if (vocab_size < 2 || dim < 1) invalid("bad model geometry");
    if (center < 0 || center >= vocab_size) invalid("center out of range");
    if (center_pos < 0 || center_pos >= sentence_len) invalid("center position out of range");
    if (half_window < 0) invalid("half window must be >= 0");
    if (hot_count > 0 && (!slot_of || !cache_work || !cache_snap || !cache_flag)) invalid("cache arrays missing");
}
}  // namespace

extern "C" {

int cg_train_center(int32_t center, const int32_t* sentence, int64_t sentence_len, int64_t center_pos,
                    int32_t half_window, int32_t vocab_size, int32_t dim, float* syn0, float* syn1,
                    const int64_t* path_offsets, const int32_t* path_nodes, const uint8_t* path_turns,
                    const int32_t* slot_of, int32_t hot_count, float* cache_work, float* cache_snap,
                    uint8_t* cache_flag, float alpha, int32_t sigmoid_mode, float sig_const, int64_t* sigmoid_calls) {
    return guarded([&] {
        check_center_args(center, sentence_len, center_pos, half_window, vocab_size, dim, slot_of, hot_count,
                          cache_work, cache_snap, cache_flag);
        if (sigmoid_mode < 0 || sigmoid_mode > 2) invalid("sigmoid_mode must be 0, 1 or 2");
        CenterCall cc;
        cc.up(sentence, sentence_len, vocab_size, dim, syn0, syn1, path_offsets, path_nodes, path_turns, slot_of,
              hot_count, cache_work, cache_snap, cache_flag);
        cgk::DetCenter c{};
        c.center = center;
        c.sentence = cc.sent.p;
        c.len = sentence_len;
        c.pos = center_pos;
        c.half_window = half_window;
        c.alpha = alpha;
        c.sigmoid_mode = sigmoid_mode;
        c.sig_const = sig_const;
        c.n_acquired = cc.nacq.p;
        c.evals = cc.evals.p;
        cgk::launch_det_center(cc.m, c, nullptr);
        cc.down(syn0, syn1, cache_work, cache_snap, cache_flag);
        unsigned long long e = 0;
        CG_CUDA(cudaMemcpy(&e, cc.evals.p, sizeof e, cudaMemcpyDeviceToHost));
        if (sigmoid_calls) *sigmoid_calls = static_cast<int64_t>(e);
    });
}

int cg_train_center_cb(int32_t center, const int32_t* sentence, int64_t sentence_len, int64_t center_pos,
                       int32_t half_window, int32_t vocab_size, int32_t dim, float* syn0, float* syn1,
                       const int64_t* path_offsets, const int32_t* path_nodes, const uint8_t* path_turns,
                       const int32_t* slot_of, int32_t hot_count, float* cache_work, float* cache_snap,
                       uint8_t* cache_flag, float alpha, cg_sigmoid_fn fn, void* ctx, int64_t* sigmoid_calls) {
    return guarded([&] {
        check_center_args(center, sentence_len, center_pos, half_window, vocab_size, dim, slot_of, hot_count,
                          cache_work, cache_snap, cache_flag);
        if (!fn) invalid("null sigmoid callback");
        CenterCall cc;
        cc.up(sentence, sentence_len, vocab_size, dim, syn0, syn1, path_offsets, path_nodes, path_turns, slot_of,
              hot_count, cache_work, cache_snap, cache_flag);
        const int L = static_cast<int>(path_offsets[center + 1] - path_offsets[center]);
        cc.buf.alloc(static_cast<size_t>(L));
        std::vector<float> host(static_cast<size_t>(L));
        const int64_t lo = center_pos >= half_window ? center_pos - half_window : 0;
        const int64_t hi = std::min(sentence_len - 1, center_pos + half_window);
        int64_t calls = 0;
        for (int64_t pos = lo; pos <= hi; ++pos) {
            if (pos == center_pos) continue;
            cgk::launch_det_pair(cc.m, center, sentence[pos], alpha, 0, cc.buf.p, cc.nacq.p, nullptr);
            CG_CUDA(cudaGetLastError());
            CG_CUDA(cudaMemcpy(host.data(), cc.buf.p, host.size() * 4, cudaMemcpyDeviceToHost));
            for (float& x : host) x = fn(x, ctx);  // path order, one call per step
            calls += L;
            CG_CUDA(cudaMemcpy(cc.buf.p, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
            cgk::launch_det_pair(cc.m, center, sentence[pos], alpha, 1, cc.buf.p, cc.nacq.p, nullptr);
        }
        cc.down(syn0, syn1, cache_work, cache_snap, cache_flag);
        if (sigmoid_calls) *sigmoid_calls = calls;
    });
}

int cg_cache_flush(int32_t vocab_size, int32_t dim, float* syn1, const int32_t* hot_nodes, int32_t hot_count,
                   float* cache_work, const float* cache_snap, uint8_t* cache_flag) {
    return guarded([&] {
        if (hot_count <= 0) return;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw CgError(CG_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
        }
        const size_t n1 = static_cast<size_t>(vocab_size - 1) * dim;
        DevBuf<float> d1, work, snap;
        DevBuf<int32_t> hot;
        DevBuf<uint8_t> flag;
        d1.upload(syn1, n1, nullptr);
        work.upload(cache_work, static_cast<size_t>(hot_count) * dim, nullptr);
        snap.upload(cache_snap, static_cast<size_t>(hot_count) * dim, nullptr);
        flag.upload(cache_flag, static_cast<size_t>(hot_count), nullptr);
        hot.upload(hot_nodes, static_cast<size_t>(hot_count), nullptr);
        cgk::DetModel m{};
        m.syn1 = d1.p;
        m.dim = dim;
        m.vocab = vocab_size;
        m.hot_nodes = hot.p;
        m.hot_count = hot_count;
        m.cache_work = work.p;
        m.cache_snap = snap.p;
        m.cache_flag = flag.p;
        cgk::launch_det_flush_flags(m, nullptr);
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpy(syn1, d1.p, n1 * 4, cudaMemcpyDeviceToHost));
        CG_CUDA(cudaMemcpy(cache_flag, flag.p, static_cast<size_t>(hot_count), cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"

// ============================================================================ evaluation
struct cg_embeddings {
    int device = 0;
    int32_t rows = 0, dim = 0, ld = 0;
    DevBuf<float> table;  // rows x ld, unit-normalised, zero-padded
};

namespace {
int require_device(int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw CgError(CG_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
    }
    if (device < 0) {  // the calling thread's current device
        CG_CUDA(cudaGetDevice(&device));
        return device;
    }
    if (device >= ndev) invalid("device ordinal out of range");
    CG_CUDA(cudaSetDevice(device));
    return device;
}

int embeddings_make(const float* src, bool src_on_device, int32_t rows, int32_t dim, int32_t stride, int32_t device,
                    cg_embeddings** out) {
    return guarded([&] {
        if (!out) invalid("cg_embeddings_create: out is null");
        *out = nullptr;
        if (rows < 0) invalid("rows must be >= 0");
        if (dim < 1) invalid("vector dimension must be >= 1");
        if (rows > 0 && !src) invalid("vectors is null");
        auto e = std::make_unique<cg_embeddings>();
        e->device = require_device(device);
        e->rows = rows;
        e->dim = dim;
        e->ld = cgk::eval_ld(dim);
        if (rows > 0) {
            e->table.alloc(static_cast<size_t>(rows) * e->ld);
            DevBuf<float> staged;
            const float* dsrc = src;
            if (!src_on_device) {
                staged.upload(src, static_cast<size_t>(rows) * dim, nullptr);
                dsrc = staged.p;
            }
            cgk::launch_normalize(dsrc, stride, e->table.p, e->ld, rows, dim, nullptr);
            CG_CUDA(cudaGetLastError());
            CG_CUDA(cudaDeviceSynchronize());
        }
        *out = e.release();
    });
}
}  // namespace

extern "C" {

int cg_embeddings_create(const float* vectors, int32_t rows, int32_t dim, int32_t device, cg_embeddings** out) {
    return embeddings_make(vectors, false, rows, dim, dim, device, out);
}

int cg_embeddings_create_device(const float* device_vectors, int32_t rows, int32_t dim, int32_t row_stride,
                                int32_t device, cg_embeddings** out) {
    if (row_stride < dim) {
        g_error = "row_stride must be >= dim";
        return CG_ERR_INVALID_ARGUMENT;
    }
    return embeddings_make(device_vectors, true, rows, dim, row_stride, device, out);
}

void cg_embeddings_destroy(cg_embeddings* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    delete e;
}

int32_t cg_embeddings_rows(const cg_embeddings* e) { return e ? e->rows : 0; }

int cg_embeddings_normalized(const cg_embeddings* e, float* out) {
    return guarded([&] {
        if (!e || (!out && e->rows > 0)) invalid("null argument");
        if (e->rows == 0) return;
        CG_CUDA(cudaSetDevice(e->device));
        CG_CUDA(cudaMemcpy2D(out, static_cast<size_t>(e->dim) * 4, e->table.p, static_cast<size_t>(e->ld) * 4,
                             static_cast<size_t>(e->dim) * 4, static_cast<size_t>(e->rows), cudaMemcpyDeviceToHost));
    });
}

int cg_analogy_answer(cg_embeddings* e, const int32_t* abc, int64_t n, int32_t* best) {
    return guarded([&] {
        if (!e) invalid("null embeddings");
        if (n < 0) invalid("question count must be >= 0");
        if (n == 0) return;
        if (!abc || !best) invalid("null argument");
        for (int64_t i = 0; i < 3 * n; ++i)
            if (abc[i] < 0 || abc[i] >= e->rows) invalid("question word id out of range");
        CG_CUDA(cudaSetDevice(e->device));
        DevBuf<int32_t> q, out;
        DevBuf<float> target;
        DevBuf<unsigned long long> keys;
        q.upload(abc, static_cast<size_t>(3 * n), nullptr);
        out.alloc(static_cast<size_t>(n));
        target.alloc(static_cast<size_t>(n) * e->ld);
        keys.alloc(static_cast<size_t>(n));
        cgk::launch_analogy(e->table.p, e->ld, e->dim, e->rows, q.p, n, target.p, keys.p, out.p, nullptr);
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpy(best, out.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost));
    });
}

int cg_nearest(cg_embeddings* e, const int32_t* queries, int64_t n, int32_t k, int32_t* ids, float* scores) {
    return guarded([&] {
        if (!e) invalid("null embeddings");
        if (n < 0) invalid("query count must be >= 0");
        if (k < 1 || k > 32) invalid("k must be in [1, 32]");
        if (n == 0) return;
        if (!queries || !ids || !scores) invalid("null argument");
        for (int64_t i = 0; i < n; ++i)
            if (queries[i] < 0 || queries[i] >= e->rows) invalid("query id out of range");
        CG_CUDA(cudaSetDevice(e->device));
        DevBuf<int32_t> q, oid;
        DevBuf<float> osc;
        q.upload(queries, static_cast<size_t>(n), nullptr);
        oid.alloc(static_cast<size_t>(n) * k);
        osc.alloc(static_cast<size_t>(n) * k);
        cgk::launch_topk(e->table.p, e->ld, e->rows, q.p, n, k, oid.p, osc.p, nullptr);
        CG_CUDA(cudaGetLastError());
        CG_CUDA(cudaMemcpy(ids, oid.p, static_cast<size_t>(n) * k * 4, cudaMemcpyDeviceToHost));
        CG_CUDA(cudaMemcpy(scores, osc.p, static_cast<size_t>(n) * k * 4, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"

// ============================================================================ GPU ingest
namespace {
std::vector<std::string> split_nul(const char* words_nul, int32_t n) {
    std::vector<std::string> w(static_cast<size_t>(n));
    const char* p = words_nul;
    for (int32_t i = 0; i < n; ++i) {
        w[static_cast<size_t>(i)] = p;
        p += w[static_cast<size_t>(i)].size() + 1;
    }
    return w;
}

struct DevWordTable {
    DevBuf<unsigned long long> keys;
    DevBuf<int32_t> ids, len;
    DevBuf<int64_t> off;
    DevBuf<char> pool;
    cgk::WordTableDev view{};
    void upload(const std::vector<std::string>& words, cudaStream_t st) {
        cgk::WordTableHost h;
        h.build(words);
        keys.upload(h.keys.data(), h.keys.size(), st);
        ids.upload(h.ids.data(), h.ids.size(), st);
        len.upload(h.len.data(), h.len.size(), st);
        off.upload(h.off.data(), h.off.size(), st);
        pool.upload(h.pool.data(), std::max<size_t>(h.pool.size(), 1), st);
        if (h.pool.empty()) pool.alloc(1);
        view = cgk::WordTableDev{keys.p, ids.p, off.p, len.p, pool.p, h.mask};
        CG_CUDA(cudaStreamSynchronize(st));  // the host table goes out of scope
    }
};

// Tokenises `path` on the device into `ids` (grown as needed); returns the id count.
int64_t device_id_stream(const char* path, const std::vector<std::string>& words, int64_t hint, DevBuf<int32_t>& ids,
                         cudaStream_t st, cgk::IngestStats* stats) {
    DevWordTable t;
    t.upload(words, st);
    uint64_t cap = static_cast<uint64_t>(std::max<int64_t>(hint, 0)) + 4096;
    for (;;) {
        ids.alloc(cap);
        const int64_t n = cgk::ingest_ids(path, t.view, ids.p, cap, st, stats);
        if (static_cast<uint64_t>(n) <= cap) return n;
        cap = static_cast<uint64_t>(n);  // the vocabulary undercounted this file: once more, exactly sized
    }
}
}  // namespace

extern "C" {

int cg_session_load_corpus(cg_session* s, const char* path, const char* words_nul, int64_t* n_ids) {
    return guarded([&] {
        if (!path || !words_nul) invalid("null argument");
        CG_CUDA(cudaSetDevice(s->device));
        const std::vector<std::string> words = split_nul(words_nul, s->V);
        cgk::IngestStats ist;
        const int64_t n = device_id_stream(path, words, s->total_tokens, s->ids, s->stream, &ist);
        session_alloc_stream(s, n);
        CG_CUDA(cudaStreamSynchronize(s->stream));
        if (n_ids) *n_ids = n;
    });
}

}  // extern "C"

namespace {
// Hands the ingest's per-chunk progress (an event and a pinned word with the ids written
// so far) from the tokenising thread to the training thread.
struct ChunkQueue {
    static constexpr int kBlock = 1024;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::pair<int, cudaEvent_t>> q;
    std::vector<uint64_t*> blocks;
    bool done = false;
    uint64_t* word(int j) {
        std::lock_guard<std::mutex> g(mu);
        while (static_cast<int>(blocks.size()) * kBlock <= j)
            blocks.push_back(static_cast<uint64_t*>(cgint::PinnedPool::get().alloc(kBlock * sizeof(uint64_t))));
        return blocks[static_cast<size_t>(j / kBlock)] + j % kBlock;
    }
    ~ChunkQueue() {
        for (auto& it : q) cudaEventDestroy(it.second);
        for (uint64_t* b : blocks) cgint::PinnedPool::get().free(b);
    }
};
uint64_t* chunk_word(void* ctx, int j) { return static_cast<ChunkQueue*>(ctx)->word(j); }
void chunk_ready(void* ctx, int j, cudaEvent_t ev) {
    auto* q = static_cast<ChunkQueue*>(ctx);
    {
        std::lock_guard<std::mutex> g(q->mu);
        q->q.emplace_back(j, ev);
    }
    q->cv.notify_one();
}

// train(corpus_path) in Hogwild mode with the first pass overlapped with tokenisation:
// a host thread streams and tokenises the file into the session's id buffer while this
// thread trains every chunk as soon as its ids have landed (K3 + K1 per chunk; the draws
// are keyed by global token index, so only the sentence cuts at chunk edges differ from
// one launch over the whole stream). Later passes run over the whole stream. Returns
// false -- nothing trained that matters -- if the file holds more in-vocabulary tokens
// than the vocabulary counted (then the caller re-runs the sequential path).
bool train_file_pipelined(cg_session* s, const char* path, const std::vector<std::string>& words,
                          cg_train_stats* out) {
    CG_CUDA(cudaSetDevice(s->device));
    DevWordTable table;
    table.upload(words, s->stream);
    const uint64_t cap = static_cast<uint64_t>(std::max<int64_t>(s->total_tokens, 0)) + 4096;
    s->ids.alloc(cap);
    session_alloc_stream(s, static_cast<int64_t>(cap));  // K3 buffers fit any chunk
    ChunkQueue q;
    cgk::IngestProgress prog{chunk_word, chunk_ready, &q};
    cudaStream_t ist = nullptr;
    CG_CUDA(cudaStreamCreateWithFlags(&ist, cudaStreamNonBlocking));
    int64_t total = -1;
    std::exception_ptr perr;
    std::thread producer([&] {
        try {
            CG_CUDA(cudaSetDevice(s->device));
            total = cgk::ingest_ids(path, table.view, s->ids.p, cap, ist, nullptr, &prog);
        } catch (...) {
            perr = std::current_exception();
        }
        {
            std::lock_guard<std::mutex> g(q.mu);
            q.done = true;
        }
        q.cv.notify_one();
    });
    cg_train_stats st{};
    uint64_t trained = 0;
    bool overflow = false;
    std::string err;
    int err_rc = CG_OK;
    for (;;) {
        std::pair<int, cudaEvent_t> item{-1, nullptr};
        {
            std::unique_lock<std::mutex> g(q.mu);
            q.cv.wait(g, [&] { return !q.q.empty() || q.done; });
            if (q.q.empty()) break;
            item = q.q.front();
            q.q.pop_front();
        }
        cudaEventSynchronize(item.second);
        cudaEventDestroy(item.second);
        const uint64_t c = *q.word(item.first);
        if (c > cap) overflow = true;
        if (overflow || err_rc != CG_OK || c <= trained) continue;
        cg_epoch_stats e{};
        const int rc = cg_session_train_range(s, 0, static_cast<int64_t>(trained), static_cast<int64_t>(c), trained, 1, &e);
        if (rc != CG_OK) {
            err_rc = rc;
            err = g_error;
            continue;
        }
        st.kernel_seconds += (e.train_ms + e.subsample_ms) * 1e-3;
        st.centers += e.kept;
        st.pairs += e.pairs;
        st.steps += e.steps;
        st.words_processed += e.words;
        trained = c;
    }
    producer.join();
    cudaStreamDestroy(ist);
    if (perr) std::rethrow_exception(perr);
    if (err_rc != CG_OK) throw CgError(err_rc, err);
    if (overflow || static_cast<uint64_t>(total) > cap) return false;
    s->n_ids = total;
    for (int32_t it = 1; it < s->cfg.iterations; ++it) {
        cg_epoch_stats e{};
        const int rc = cg_session_train_range(s, it, 0, total, static_cast<uint64_t>(it) * static_cast<uint64_t>(total), 1, &e);
        if (rc != CG_OK) throw CgError(rc, g_error);
        st.kernel_seconds += (e.train_ms + e.subsample_ms) * 1e-3;
        st.centers += e.kept;
        st.pairs += e.pairs;
        st.steps += e.steps;
        st.words_processed += e.words;
    }
    *out = st;
    return true;
}
}  // namespace

extern "C" {

int cg_train_file(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const char* corpus_path,
                  const char* words_nul, float* syn0_out, float* syn1_out, cg_train_stats* stats) {
    cg_session* s = nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = 0;
    }
    const auto tc = std::chrono::steady_clock::now();
    int rc = cg_session_create(cfg, mode, model, dev, nullptr, &s);
    if (rc != CG_OK) return rc;
    const auto t0 = std::chrono::steady_clock::now();
    cg_train_stats st{};
    bool done = false;
    if (mode == CG_MODE_HOGWILD && corpus_path && words_nul) {
        rc = guarded([&] { done = train_file_pipelined(s, corpus_path, split_nul(words_nul, s->V), &st); });
        if (rc == CG_OK && !done) rc = cg_session_reset_model(s);  // undercounted vocabulary: start over
    }
    if (rc == CG_OK && !done) {
        rc = cg_session_load_corpus(s, corpus_path, words_nul, nullptr);
        if (rc == CG_OK) rc = cg_session_train(s, &st);
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (rc == CG_OK) rc = cg_session_download(s, syn0_out, syn1_out);
    if (std::getenv("CG_PROFILE")) {
        const auto t2 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "cg_train_file: create %.2f ms, ingest+train %.2f ms (kernels %.2f, %s), download %.2f ms\n",
                     ms(tc, t0), ms(t0, t1), st.kernel_seconds * 1e3, done ? "pipelined" : "sequential", ms(t1, t2));
    }
    // like the reference's, the wall time covers reading the corpus as well as training
    st.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    st.words_per_second = st.wall_seconds > 0 ? static_cast<double>(st.words_processed) / st.wall_seconds : 0.0;
    if (stats) *stats = st;
    cg_session_destroy(s);
    return rc;
}

int cg_corpus_open_gpu(const char* path, int64_t min_count, int32_t device, cg_corpus** out) {
    return guarded([&] {
        if (!path || !out) invalid("null argument");
        if (min_count < 1) invalid("min-count must be >= 1");
        *out = nullptr;
        require_device(device);
        cudaStream_t st = nullptr;
        CG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        std::vector<cgk::CountedWord> words;
        try {
            words = cgk::ingest_count(path, st, nullptr);
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        // VocabBuilder::finish: survivors by descending count, first occurrence on ties
        std::vector<cgk::CountedWord*> keep;
        for (auto& w : words)
            if (w.count >= min_count) keep.push_back(&w);
        if (keep.empty()) throw cachegram::NoTrainableWords();
        std::sort(keep.begin(), keep.end(), [](const cgk::CountedWord* a, const cgk::CountedWord* b) {
            return a->count != b->count ? a->count > b->count : a->first < b->first;
        });
        std::vector<cachegram::VocabEntry> entries(keep.size());
        int64_t total = 0;
        for (size_t r = 0; r < keep.size(); ++r) {
            entries[r].word = std::move(keep[r]->word);
            entries[r].count = keep[r]->count;
            total += keep[r]->count;
        }
        *out = new cg_corpus{cachegram::Vocabulary(std::move(entries), total)};
    });
}

int cg_corpus_read_ids_gpu(const cg_corpus* c, const char* path, int32_t device, int32_t* ids, int64_t capacity,
                           int64_t* n_ids) {
    return guarded([&] {
        if (!c || !path) invalid("null argument");
        require_device(device);
        std::vector<std::string> words(static_cast<size_t>(c->vocab.size()));
        for (int32_t w = 0; w < c->vocab.size(); ++w) words[static_cast<size_t>(w)] = c->vocab.word(w);
        cudaStream_t st = nullptr;
        CG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        DevBuf<int32_t> dev_ids;
        int64_t n = 0;
        try {
            n = device_id_stream(path, words, c->vocab.total_tokens(), dev_ids, st, nullptr);
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        if (n_ids) *n_ids = n;
        if (ids) {
            if (n > capacity) {
                cudaStreamDestroy(st);
                invalid("id buffer too small");
            }
            if (n) CG_CUDA(cudaMemcpyAsync(ids, dev_ids.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, st));
        }
        CG_CUDA(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
    });
}

}  // extern "C"

// ============================================================================ in-process replicas
// One model replica per GPU of this process, for C/C++ callers that do not
// run one process per GPU: each replica trains its shard of the id stream, and every
// `sync_words` words per replica the replicas are averaged in place over peer memory
// (NVLink/NVSwitch): replica r's device averages slice r of the model buffer across all
// replicas and writes the mean back to every replica -- a reduce-scatter and an
// all-gather in one pass, the same bytes per GPU as a ring all-reduce.
namespace {
constexpr int kMaxReplicas = 8;
struct ReplicaPtrs {
    float4* buf[kMaxReplicas];
};

// Slice [begin4, end4) of the n buffers: sum in a fixed order (every replica receives the
// same bits), times inv_n (1 = the sum of the replicas' deltas, 1/n = their average),
// written back to every buffer.
__global__ void replica_avg_kernel(ReplicaPtrs p, int n, size_t begin4, size_t end4, float inv_n) {
    for (size_t i = begin4 + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < end4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float4 s = p.buf[0][i];
        for (int r = 1; r < n; ++r) {  // fixed order: every replica receives the same bits
            const float4 x = p.buf[r][i];
            s.x += x.x;
            s.y += x.y;
            s.z += x.z;
            s.w += x.w;
        }
        s = make_float4(s.x * inv_n, s.y * inv_n, s.z * inv_n, s.w * inv_n);
        for (int r = 0; r < n; ++r) p.buf[r][i] = s;
    }
}

void enable_peers(const int32_t* devices, int32_t n) {
    for (int32_t a = 0; a < n; ++a)
        for (int32_t b = 0; b < n; ++b) {
            if (devices[a] == devices[b]) continue;
            int ok = 0;
            CG_CUDA(cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]));
            if (!ok) throw CgError(CG_ERR_CUDA, "replica devices cannot access each other's memory (no P2P)");
            CG_CUDA(cudaSetDevice(devices[a]));
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CG_CUDA(e);
            cudaGetLastError();
        }
}

// Replica r's share of the reduction: slice r of n4 float4s, launched on devices[r].
void launch_reduce_slice(const ReplicaPtrs& p, int32_t n, int32_t r, size_t n4, int32_t device, cudaStream_t st,
                         bool average) {
    const size_t b = n4 * static_cast<size_t>(r) / static_cast<size_t>(n);
    const size_t e = n4 * static_cast<size_t>(r + 1) / static_cast<size_t>(n);
    if (e <= b) return;
    CG_CUDA(cudaSetDevice(device));
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((e - b + 255) / 256, 148 * 8));
    replica_avg_kernel<<<grid, 256, 0, st>>>(p, n, b, e, average ? 1.0f / static_cast<float>(n) : 1.0f);
    CG_CUDA(cudaGetLastError());
}

void check_replica_devices(const int32_t* devices, int32_t n) {
    if (n < 1 || n > kMaxReplicas) invalid("replica count must be in [1, 8]");
    if (!devices) invalid("null device list");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw CgError(CG_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
    }
    for (int32_t r = 0; r < n; ++r)
        if (devices[r] < 0 || devices[r] >= ndev) invalid("device ordinal out of range");
}

// The shared driver of cg_train_replicas / cg_train_file_replicas. `load(r, s)` fills
// replica r's session with its shard and returns the shard length.
template <typename Load>
void run_replicas(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const int32_t* devices, int32_t n,
                  int64_t sync_words, Load&& load, float* syn0_out, float* syn1_out, cg_train_stats* stats) {
    if (!cfg || !model) invalid("null config or model");
    if (mode != CG_MODE_HOGWILD) invalid("replicas train in Hogwild mode (the deterministic mode is one stream)");
    if (sync_words < 1) invalid("sync_words must be >= 1");
    check_replica_devices(devices, n);
    const auto t0 = std::chrono::steady_clock::now();
    struct Rep {
        cg_session* s = nullptr;
        cudaStream_t st = nullptr;
        int64_t len = 0;
        double kernel_s = 0.0;
        uint64_t centers = 0, pairs = 0, steps = 0, words = 0;
    };
    std::vector<Rep> rep(static_cast<size_t>(n));
    auto cleanup = [&] {
        for (auto& x : rep) {
            if (x.s) cg_session_destroy(x.s);
            if (x.st) cudaStreamDestroy(x.st);
        }
    };
    try {
        for (int32_t r = 0; r < n; ++r) {
            Rep& x = rep[static_cast<size_t>(r)];
            CG_CUDA(cudaSetDevice(devices[r]));
            CG_CUDA(cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking));
            const int rc = cg_session_create(cfg, mode, model, devices[r], x.st, &x.s);
            if (rc != CG_OK) throw CgError(rc, g_error);
            x.len = load(r, x.s);
        }
        enable_peers(devices, n);
        for (auto& x : rep) {
            const int rc = cg_session_sync_begin(x.s);
            if (rc != CG_OK) throw CgError(rc, g_error);
        }
        ReplicaPtrs ptrs{};  // the replicas' delta buffers (allocated by their first sync)
        size_t n4 = 0;
        int64_t max_len = 0;
        for (auto& x : rep) max_len = std::max(max_len, x.len);
        const int64_t chunks = (max_len + sync_words - 1) / sync_words;
        std::barrier sync(n);
        std::atomic<int> failed{0};
        std::vector<std::string> errs(static_cast<size_t>(n));
        std::vector<int> codes(static_cast<size_t>(n), CG_OK);
        auto fail = [&](int32_t r, int code, const std::string& m) {
            codes[static_cast<size_t>(r)] = code;
            errs[static_cast<size_t>(r)] = m;
            failed.store(1);
        };
        // Each chunk: train, then the delta reduction -- every replica's delta since the last
        // sync (model - snapshot), summed over replicas slice by slice over peer memory,
        // applied to every replica's snapshot with the per-row sync scale.
        auto worker = [&](int32_t r) {
            Rep& x = rep[static_cast<size_t>(r)];
            for (int32_t it = 0; it < cfg->iterations; ++it) {
                for (int64_t c = 0; c < chunks; ++c) {
                    if (!failed.load()) {
                        const int64_t a = std::min(x.len, c * sync_words), b = std::min(x.len, (c + 1) * sync_words);
                        cg_epoch_stats e{};
                        const uint64_t base = (static_cast<uint64_t>(it) * static_cast<uint64_t>(x.len) + static_cast<uint64_t>(a)) *
                                              static_cast<uint64_t>(n);
                        const int rc = b > a ? cg_session_train_range(x.s, it, a, b, base, static_cast<uint32_t>(n), &e)
                                             : CG_OK;
                        if (rc != CG_OK) fail(r, rc, cg_last_error());
                        x.kernel_s += (e.train_ms + e.subsample_ms) * 1e-3;
                        x.centers += e.kept;
                        x.pairs += e.pairs;
                        x.steps += e.steps;
                        x.words += e.words;
                    }
                    if (n > 1) {
                        if (!failed.load()) {
                            void* d = nullptr;
                            size_t nf = 0;
                            const int rc = cg_session_sync_delta(x.s, &d, &nf);
                            if (rc != CG_OK) fail(r, rc, cg_last_error());
                            ptrs.buf[r] = static_cast<float4*>(d);
                            if (r == 0) n4 = nf / 4;
                        }
                        sync.arrive_and_wait();  // every replica's delta is ready
                        if (!failed.load()) {
                            try {
                                launch_reduce_slice(ptrs, n, r, n4, devices[r], x.st, false);
                                CG_CUDA(cudaStreamSynchronize(x.st));
                            } catch (const std::exception& ex) {
                                fail(r, CG_ERR_CUDA, ex.what());
                            }
                        }
                        sync.arrive_and_wait();  // every slice summed into every replica
                        if (!failed.load()) {
                            const int rc = cg_session_sync_apply(x.s, n, static_cast<uint64_t>(sync_words));
                            if (rc != CG_OK) fail(r, rc, cg_last_error());
                        }
                    }
                    sync.arrive_and_wait();
                }
            }
        };
        std::vector<std::thread> pool;
        for (int32_t r = 1; r < n; ++r) pool.emplace_back(worker, r);
        worker(0);
        for (auto& t : pool) t.join();
        for (int32_t r = 0; r < n; ++r)
            if (codes[static_cast<size_t>(r)] != CG_OK)
                throw CgError(codes[static_cast<size_t>(r)], "replica " + std::to_string(r) + " failed: " + errs[static_cast<size_t>(r)]);
        const int rc = cg_session_download(rep[0].s, syn0_out, syn1_out);
        if (rc != CG_OK) throw CgError(rc, g_error);
        cg_train_stats out{};
        for (auto& x : rep) {
            out.words_processed += x.words;
            out.centers += x.centers;
            out.pairs += x.pairs;
            out.steps += x.steps;
            out.kernel_seconds = std::max(out.kernel_seconds, x.kernel_s);
        }
        out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out.words_per_second = out.wall_seconds > 0 ? static_cast<double>(out.words_processed) / out.wall_seconds : 0.0;
        if (stats) *stats = out;
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}
}  // namespace

extern "C" {

int cg_average_buffers(void* const* device_bufs, const int32_t* devices, int32_t n, size_t n_floats) {
    return guarded([&] {
        if (!device_bufs) invalid("null buffer list");
        check_replica_devices(devices, n);
        if (n_floats % 4) invalid("n_floats must be a multiple of 4");
        enable_peers(devices, n);
        ReplicaPtrs p{};
        for (int32_t r = 0; r < n; ++r) p.buf[r] = static_cast<float4*>(device_bufs[r]);
        for (int32_t r = 0; r < n; ++r) launch_reduce_slice(p, n, r, n_floats / 4, devices[r], nullptr, true);
        for (int32_t r = 0; r < n; ++r) {
            CG_CUDA(cudaSetDevice(devices[r]));
            CG_CUDA(cudaDeviceSynchronize());
        }
    });
}

int cg_train_replicas(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const int32_t* ids, int64_t n_ids,
                      const int32_t* devices, int32_t n_devices, int64_t sync_words, float* syn0_out, float* syn1_out,
                      cg_train_stats* stats) {
    return guarded([&] {
        if (n_ids < 0 || (n_ids > 0 && !ids)) invalid("bad id stream");
        run_replicas(cfg, mode, model, devices, n_devices, sync_words,
                     [&](int32_t r, cg_session* s) -> int64_t {
                         // contiguous near-equal shards (corpus.hpp:192-223 on the id stream)
                         const int64_t a = n_ids * r / n_devices, b = n_ids * (r + 1) / n_devices;
                         const int rc = cg_session_upload_ids(s, ids + a, b - a);
                         if (rc != CG_OK) throw CgError(rc, g_error);
                         return b - a;
                     },
                     syn0_out, syn1_out, stats);
    });
}

int cg_train_file_replicas(const cg_config* cfg, int32_t mode, const cg_model_desc* model, const char* corpus_path,
                           const char* words_nul, const int32_t* devices, int32_t n_devices, int64_t sync_words,
                           float* syn0_out, float* syn1_out, cg_train_stats* stats) {
    return guarded([&] {
        if (!corpus_path || !words_nul || !model) invalid("null argument");
        check_replica_devices(devices, n_devices);
        // tokenise once on the first replica's GPU, then hand each replica its shard
        CG_CUDA(cudaSetDevice(devices[0]));
        const std::vector<std::string> words = split_nul(words_nul, model->vocab_size);
        DevBuf<int32_t> all;
        cudaStream_t st = nullptr;
        CG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        int64_t n_ids = 0;
        try {
            n_ids = device_id_stream(corpus_path, words, model->total_tokens, all, st, nullptr);
            CG_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        run_replicas(cfg, mode, model, devices, n_devices, sync_words,
                     [&](int32_t r, cg_session* s) -> int64_t {
                         const int64_t a = n_ids * r / n_devices, b = n_ids * (r + 1) / n_devices;
                         const int rc = cg_session_upload_ids_device(s, all.p + a, b - a);
                         if (rc != CG_OK) throw CgError(rc, g_error);
                         return b - a;
                     },
                     syn0_out, syn1_out, stats);
    });
}

}  // extern "C"
