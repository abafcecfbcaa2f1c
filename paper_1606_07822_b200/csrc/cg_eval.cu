// cg_eval.cu -- evaluation on the device: unit-normalised
// embedding tables, batched 3CosAdd analogy answering and cosine top-k neighbours.
//
// Exactness contract: every score is the reference's sequential fp32 dot
// (vec_ops.hpp:14-18: sum starts at +0, i ascending, mul then add, no FMA), every
// normalised row is src[d] / sqrtf(dot(src, src)) as in AnalogySolver (eval.hpp:91-103),
// and the 3CosAdd target is (vb - va) + vc (eval.hpp:121-122). So the device answers
// equal the reference's bit for bit, including ties (to the lower id) and NaN rows.
//
// The scoring kernels are GEMM-shaped (queries x words x D) but stay on the FP32 pipe:
// tensor cores would reassociate the sum and change the argmax on near-ties. They are
// register-tiled like an SGEMM (64 queries x 128 words per CTA, 4x8 scores per thread,
// k-major shared-memory tiles): each k step is 3 LDS.128 for 64 separately rounded
// FMUL+FADD. Zero padding of D to a multiple of 16 is exact: the running sum starts at
// +0 and can never be -0, so adding +0 products leaves it unchanged.
#include <cstdint>

#include "cg_device.cuh"
#include "cg_kernels.h"

namespace cgk {
namespace {

using namespace cgdev;

constexpr int kNormRows = 128;
constexpr int BQ = 64, BW = 128, BK = 16;  // CTA tile: queries x words x k-chunk
constexpr int kTileThreads = 256;          // 16 x 16 threads, 4 queries x 8 words each

// One thread per row: the sequential sum of squares over a 32-column shared-memory
// staging tile (coalesced loads, conflict-free column walks), then a coalesced write of
// src / norm (zeros when !(norm > 0), which includes NaN norms, eval.hpp:97-101).
__global__ void __launch_bounds__(kNormRows) normalize_kernel(const float* src, int64_t src_ld, float* dst,
                                                              int ld, int64_t rows, int dim) {
    __shared__ float tile[kNormRows][33];
    __shared__ float norms[kNormRows];
    const int t = threadIdx.x;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kNormRows;
    float acc = 0.0f;
    for (int d0 = 0; d0 < dim; d0 += 32) {
        for (int i = t; i < kNormRows * 32; i += kNormRows) {
            const int r = i >> 5, c = i & 31;
            tile[r][c] = (r0 + r < rows && d0 + c < dim) ? src[(r0 + r) * src_ld + d0 + c] : 0.0f;
        }
        __syncthreads();
        const int n = min(32, dim - d0);
        for (int c = 0; c < n; ++c) acc = __fadd_rn(acc, __fmul_rn(tile[t][c], tile[t][c]));
        __syncthreads();
    }
    norms[t] = __fsqrt_rn(acc);
    __syncthreads();
    for (int r = 0; r < kNormRows; ++r) {
        const int64_t row = r0 + r;
        if (row >= rows) break;
        const float nrm = norms[r];
        for (int d = t; d < ld; d += kNormRows) {
            float v = 0.0f;
            if (d < dim && nrm > 0.0f) v = __fdiv_rn(src[row * src_ld + d], nrm);
            dst[row * ld + d] = v;
        }
    }
}

// target[q] = (N[b] - N[a]) + N[c] (eval.hpp:121-122); pads stay zero.
__global__ void analogy_target_kernel(const float* N, int ld, int dim, const int32_t* abc, int64_t nq, float* T) {
    const int64_t n = nq * ld;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t q = i / ld;
        const int d = static_cast<int>(i - q * ld);
        float v = 0.0f;
        if (d < dim) {
            const int64_t a = abc[3 * q], b = abc[3 * q + 1], c = abc[3 * q + 2];
            v = __fadd_rn(__fsub_rn(N[b * ld + d], N[a * ld + d]), N[c * ld + d]);
        }
        T[i] = v;
    }
}

// Order-preserving key of a non-NaN score (-0 folded onto +0, as `>` treats them equal),
// with the id in the low word so that equal scores rank the lower id higher.
__device__ __forceinline__ unsigned long long score_key(float s, int32_t w) {
    const unsigned u = __float_as_uint(s == 0.0f ? 0.0f : s);
    const unsigned ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return (static_cast<unsigned long long>(ord) << 32) | (0xffffffffu - static_cast<unsigned>(w));
}
__device__ __forceinline__ float key_score(unsigned long long k) {
    const unsigned ord = static_cast<unsigned>(k >> 32);
    const unsigned u = (ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord;
    return __uint_as_float(u);
}
__device__ __forceinline__ int32_t key_id(unsigned long long k) {
    return static_cast<int32_t>(0xffffffffu - static_cast<unsigned>(k & 0xffffffffu));
}
__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m) {
    const unsigned lo = __shfl_xor_sync(kFull, static_cast<unsigned>(v), m);
    const unsigned hi = __shfl_xor_sync(kFull, static_cast<unsigned>(v >> 32), m);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}
__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
    const unsigned lo = __shfl_sync(kFull, static_cast<unsigned>(v), src);
    const unsigned hi = __shfl_sync(kFull, static_cast<unsigned>(v >> 32), src);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}
__device__ __forceinline__ unsigned long long shfl_up_u64(unsigned long long v) {
    const unsigned lo = __shfl_up_sync(kFull, static_cast<unsigned>(v), 1);
    const unsigned hi = __shfl_up_sync(kFull, static_cast<unsigned>(v >> 32), 1);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

struct TileSmem {
    float q[BK][BQ];  // k-major query tile
    float w[BK][BW];  // k-major word tile
};

// acc[i][j] = sequential dot of query row (q0 + 4*tq + i) and word row (w0 + wid(tw, j)),
// wid(tw, j) = 4*tw + j for j < 4 and 64 + 4*tw + (j - 4) otherwise. Rows are padded to
// ld (a multiple of BK) with zeros; rows beyond the tables read as zeros.
__device__ __forceinline__ void score_tile(const float* Q, int64_t nq_rows, const int32_t* q_index, const float* W,
                                           int64_t nw_rows, int ld, int64_t q0, int64_t w0, TileSmem& sm,
                                           float (&acc)[4][8]) {
    const int tid = threadIdx.x, tq = tid >> 4, tw = tid & 15;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    // loader roles: query tile = 64 rows x 16 k = 256 float4; word tile = 512 float4
    const int lq = tid >> 2, lk = (tid & 3) * 4;
    const int64_t qr = q0 + lq;
    const float* qsrc = nullptr;
    if (qr < nq_rows) qsrc = Q + (q_index ? static_cast<int64_t>(q_index[qr]) : qr) * ld;
    const int64_t wr0 = w0 + lq, wr1 = w0 + 64 + lq;
    const float* wsrc0 = wr0 < nw_rows ? W + wr0 * ld : nullptr;
    const float* wsrc1 = wr1 < nw_rows ? W + wr1 * ld : nullptr;
    for (int k0 = 0; k0 < ld; k0 += BK) {
        const float4 a = qsrc ? *reinterpret_cast<const float4*>(qsrc + k0 + lk) : f4(0.f);
        const float4 b0 = wsrc0 ? *reinterpret_cast<const float4*>(wsrc0 + k0 + lk) : f4(0.f);
        const float4 b1 = wsrc1 ? *reinterpret_cast<const float4*>(wsrc1 + k0 + lk) : f4(0.f);
        __syncthreads();  // previous chunk fully consumed
        sm.q[lk + 0][lq] = a.x;
        sm.q[lk + 1][lq] = a.y;
        sm.q[lk + 2][lq] = a.z;
        sm.q[lk + 3][lq] = a.w;
        sm.w[lk + 0][lq] = b0.x;
        sm.w[lk + 1][lq] = b0.y;
        sm.w[lk + 2][lq] = b0.z;
        sm.w[lk + 3][lq] = b0.w;
        sm.w[lk + 0][64 + lq] = b1.x;
        sm.w[lk + 1][64 + lq] = b1.y;
        sm.w[lk + 2][64 + lq] = b1.z;
        sm.w[lk + 3][64 + lq] = b1.w;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            const float4 qa = *reinterpret_cast<const float4*>(&sm.q[k][4 * tq]);
            const float4 wa = *reinterpret_cast<const float4*>(&sm.w[k][4 * tw]);
            const float4 wb = *reinterpret_cast<const float4*>(&sm.w[k][64 + 4 * tw]);
            const float qv[4] = {qa.x, qa.y, qa.z, qa.w};
            const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(qv[i], wv[j]));
        }
    }
}
__device__ __forceinline__ int tile_word(int tw, int j) { return j < 4 ? 4 * tw + j : 64 + 4 * tw + (j - 4); }

// 3CosAdd: per (query tile, word tile) the best non-NaN, non-excluded word of every
// query, merged across word tiles with a 64-bit atomicMax on (score key, ~id).
__global__ void __launch_bounds__(kTileThreads) analogy_score_kernel(const float* T, const float* N, int ld,
                                                                     int64_t nq, int64_t nw, const int32_t* abc,
                                                                     unsigned long long* best) {
    __shared__ TileSmem sm;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * BQ, w0 = static_cast<int64_t>(blockIdx.y) * BW;
    float acc[4][8];
    score_tile(T, nq, nullptr, N, nw, ld, q0, w0, sm, acc);
    const int tq = threadIdx.x >> 4, tw = threadIdx.x & 15;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t q = q0 + 4 * tq + i;
        int32_t a = -1, b = -1, c = -1;
        if (q < nq) {
            a = abc[3 * q];
            b = abc[3 * q + 1];
            c = abc[3 * q + 2];
        }
        unsigned long long k = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t w = w0 + tile_word(tw, j);
            const float s = acc[i][j];
            if (q < nq && w < nw && w != a && w != b && w != c && !isnan(s)) {
                const unsigned long long kk = score_key(s, static_cast<int32_t>(w));
                k = kk > k ? kk : k;
            }
        }
#pragma unroll
        for (int m = 1; m < 16; m <<= 1) {  // the 16 threads of one query row share a half-warp
            const unsigned long long o = shfl_xor_u64(k, m);
            k = o > k ? o : k;
        }
        if (tw == 0 && k != 0) atomicMax(best + q, k);
    }
}

// Final answer per query: the reference keeps its first candidate when that score is NaN
// (nothing compares greater than NaN); otherwise the answer is the first maximum among
// the non-NaN scores, which is what the keys encode.
__global__ void analogy_finish_kernel(const float* T, const float* N, int ld, int dim, int64_t nq, int64_t nw,
                                      const int32_t* abc, const unsigned long long* best, int32_t* out) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= nq) return;
    const int32_t a = abc[3 * q], b = abc[3 * q + 1], c = abc[3 * q + 2];
    int64_t first = 0;
    while (first < nw && (first == a || first == b || first == c)) ++first;
    if (first >= nw) {
        out[q] = -1;
        return;
    }
    float s = 0.0f;
    for (int d = 0; d < dim; ++d) s = __fadd_rn(s, __fmul_rn(T[q * ld + d], N[first * ld + d]));
    if (isnan(s) || best[q] == 0) {
        out[q] = static_cast<int32_t>(first);
        return;
    }
    out[q] = key_id(best[q]);
}

// Cosine top-k (k <= 32) of query rows against all words, excluding the query's own
// word: each CTA owns 64 queries and sweeps every word tile, keeping each query's
// sorted top-k in shared memory; a warp merges 8 queries per tile with a ballot insert.
constexpr int kMaxTopK = 32;
__global__ void __launch_bounds__(kTileThreads) topk_kernel(const float* N, int ld, int64_t nw, const int32_t* qidx,
                                                            int64_t nq, int k, int32_t* out_ids, float* out_scores) {
    __shared__ TileSmem sm;
    extern __shared__ unsigned long long topk_dyn[];
    auto top = reinterpret_cast<unsigned long long(*)[kMaxTopK]>(topk_dyn);            // [BQ][kMaxTopK]
    auto ssc = reinterpret_cast<float(*)[BW + 1]>(topk_dyn + BQ * kMaxTopK);            // [BQ][BW + 1]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tq = tid >> 4, tw = tid & 15;
    const int64_t q0 = static_cast<int64_t>(blockIdx.x) * BQ;
    for (int i = tid; i < BQ * kMaxTopK; i += kTileThreads) top[i / kMaxTopK][i % kMaxTopK] = 0;
    for (int64_t w0 = 0; w0 < nw; w0 += BW) {
        float acc[4][8];
        score_tile(N, nq, qidx, N, nw, ld, q0, w0, sm, acc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) ssc[4 * tq + i][tile_word(tw, j)] = acc[i][j];
        __syncthreads();
        for (int qi = warp * (BQ / 8); qi < (warp + 1) * (BQ / 8); ++qi) {
            const int64_t q = q0 + qi;
            if (q >= nq) break;
            const int64_t self = qidx[q];
            unsigned long long L = lane < k ? top[qi][lane] : 0;
            unsigned long long thr = shfl_u64(L, k - 1);
            unsigned long long cand[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t w = w0 + lane + 32 * i;
                const float s = ssc[qi][lane + 32 * i];
                cand[i] = 0;
                if (w < nw && w != self && !isnan(s)) {
                    const unsigned long long kk = score_key(s, static_cast<int32_t>(w));
                    if (kk > thr) cand[i] = kk;
                }
            }
            for (;;) {
                unsigned long long m = cand[0];
#pragma unroll
                for (int i = 1; i < 4; ++i) m = cand[i] > m ? cand[i] : m;
                if (!__any_sync(kFull, m != 0)) break;
                unsigned long long M = m;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long x = shfl_xor_u64(M, o);
                    M = x > M ? x : M;
                }
                // insert M into the lane-distributed descending list
                const int pos = __popc(__ballot_sync(kFull, lane < k && L > M));
                const unsigned long long up = shfl_up_u64(L);
                if (lane < k) L = lane < pos ? L : (lane == pos ? M : up);
                thr = shfl_u64(L, k - 1);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (cand[i] == M || cand[i] <= thr) cand[i] = 0;
            }
            if (lane < k) top[qi][lane] = L;
        }
        __syncthreads();
    }
    for (int i = tid; i < BQ * k; i += kTileThreads) {
        const int qi = i / k, r = i % k;
        const int64_t q = q0 + qi;
        if (q >= nq) continue;
        const unsigned long long key = top[qi][r];
        out_ids[q * k + r] = key ? key_id(key) : -1;
        out_scores[q * k + r] = key ? key_score(key) : __int_as_float(0x7fc00000);
    }
}

unsigned grid1(int64_t n, int threads) {
    const int64_t b = (n + threads - 1) / threads;
    return static_cast<unsigned>(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace

int eval_ld(int dim) { return (dim + BK - 1) / BK * BK; }

void launch_normalize(const float* src, int64_t src_ld, float* dst, int ld, int64_t rows, int dim, cudaStream_t s) {
    if (rows <= 0) return;
    normalize_kernel<<<static_cast<unsigned>((rows + kNormRows - 1) / kNormRows), kNormRows, 0, s>>>(src, src_ld, dst,
                                                                                                    ld, rows, dim);
}

void launch_analogy(const float* N, int ld, int dim, int64_t nw, const int32_t* abc, int64_t nq, float* T,
                    unsigned long long* best, int32_t* out, cudaStream_t s) {
    if (nq <= 0) return;
    analogy_target_kernel<<<grid1(nq * ld, 256), 256, 0, s>>>(N, ld, dim, abc, nq, T);
    cudaMemsetAsync(best, 0, static_cast<size_t>(nq) * sizeof(unsigned long long), s);
    if (nw > 0) {
        const dim3 grid(static_cast<unsigned>((nq + BQ - 1) / BQ), static_cast<unsigned>((nw + BW - 1) / BW));
        analogy_score_kernel<<<grid, kTileThreads, 0, s>>>(T, N, ld, nq, nw, abc, best);
    }
    analogy_finish_kernel<<<static_cast<unsigned>((nq + 127) / 128), 128, 0, s>>>(T, N, ld, dim, nq, nw, abc, best,
                                                                                 out);
}

void launch_topk(const float* N, int ld, int64_t nw, const int32_t* qidx, int64_t nq, int k, int32_t* ids,
                 float* scores, cudaStream_t s) {
    if (nq <= 0 || k <= 0) return;
    constexpr size_t smem = sizeof(unsigned long long) * BQ * kMaxTopK + sizeof(float) * BQ * (BW + 1);
    cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    topk_kernel<<<static_cast<unsigned>((nq + BQ - 1) / BQ), kTileThreads, smem, s>>>(N, ld, nw, qidx, nq, k, ids,
                                                                                     scores);
}

}  // namespace cgk
