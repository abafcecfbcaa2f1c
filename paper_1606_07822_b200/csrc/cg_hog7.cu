// cg_hog7.cu -- K1 v7: Hogwild skip-gram HS training with each center's products on the
// tensor cores.
//
// For one center c with its batch of contexts x_0..x_{n-1} (syn0 rows v_i) and its root-first
// path rows u_0..u_{L-1} (syn1), train_center (trainer.hpp:147-175) in K1's center-batched
// order (every context's dots against the rows as loaded: within-center staleness of at most
// 2W updates, as in v5) is three small matrix products:
//     S  = V U^T            (n x L)  the dot products            (vec_ops.hpp:14-18)
//     G  = (1 - turn - sigmoid(S)) * alpha, zero outside the real pairs (trainer.hpp:166-167)
//     H  = G U              (n x D)  h_i = sum_j g_ij u_j         (trainer.hpp:168)
//     dU = G^T V            (L x D)  u_j += sum_i g_ij v_i        (trainer.hpp:171)
// then v_i += h_i (trainer.hpp:173). One warp computes them with mma.sync m16n8k8 TF32 (fp32
// accumulation) out of shared memory: contexts are the M dimension of S and H (16 per tile),
// path rows the N dimension of S, the K dimension of H and the M dimension of dU. With S's K
// dimension permuted (k-slot t <-> column 2t, t + 4 <-> 2t + 1) every fragment load is one
// LDS.64 or LDS.32 free of bank conflicts for row strides of 8 or 24 (mod 32) floats. TF32
// operands keep 10 mantissa bits; sums are fp32; the sigmoid is the reference's 1000-bucket
// table (bucket width 0.012), far coarser than the operand rounding.
//
// H and dU leave straight from the accumulator fragments with red.global.add.v2.f32 (no lost
// updates). The per-CTA node cache (NodeCache, trainer.hpp:75-138): the K cached syn1 rows
// (and the most frequent words' syn0 rows) take their updates in CTA-private delta rows in L2
// (`tier2`), which the flush drains with an atomic exchange and adds to the model scaled per
// row; the warps read the cached rows' flushed state (write-combining: a CTA's own pending
// delta joins the row at its flush, like every other CTA's).
#include <algorithm>
#include <cstdint>

#include "cg_device.cuh"
#include "cg_kernels.h"

namespace cgk {
namespace {

using namespace cgdev;

constexpr int kVRows = 16;     // context rows per batch: the M dimension of one mma tile
constexpr int kGtStride = 36;  // G scratch row stride (floats): conflict-free A-fragment loads for H

__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// red.global.add.v2.f32 under a predicate (no branch around it)
__device__ __forceinline__ void red_add2_if(bool pred, float* p, float x, float y) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q red.global.add.v2.f32 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "f"(x), "f"(y), "r"(static_cast<unsigned>(pred))
                 : "memory");
}
__device__ __forceinline__ uint2 lds64(const float* p) { return *reinterpret_cast<const uint2*>(p); }
__device__ __forceinline__ uint32_t ldsu(const float* p) { return __float_as_uint(*p); }

// Shared-memory row stride (floats) of a row of dp floats: the smallest >= dp that is 8 or 24
// (mod 32).
__host__ __device__ constexpr int k7_stride(int dp) {
    int s = dp;
    while (s % 32 != 8 && s % 32 != 24) s += 8;
    return s;
}
// Per warp: G scratch (kVRows x kGtStride) | V (kVRows x ss) | U (urows x ss) | codes (32).
__host__ __device__ constexpr uint32_t k7_warp_floats(int ss, int urows) {
    return static_cast<uint32_t>(kVRows * kGtStride + (kVRows + urows) * ss + 32);
}

// S = V U^T over the row's DP8 k-steps for NT n-tiles; two accumulator sets (even and odd
// k-steps) halve the dependent mma chain. HALF: contexts 8-15 are padding, the tile's
// second half repeats the first (one A load per k-step).
template <int NT, bool HALF, int DP8>
__device__ __forceinline__ void s_phase(const float* V, const float* U, int ss, int dp8, int g, int t,
                                        float (&acc)[4][4]) {
    float ev[NT][4], od[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) ev[n][e] = od[n][e] = 0.f;
    const float* va = V + g * ss + 2 * t;
    const float* vb = V + (g + 8) * ss + 2 * t;
    const float* ub = U + g * ss + 2 * t;
    const int n8 = DP8 > 0 ? DP8 : dp8;
    int s = 0;
#pragma unroll 2
    for (; s + 1 < n8; s += 2) {
        const uint2 x0 = lds64(va + 8 * s), x1 = lds64(va + 8 * s + 8);
        const uint2 y0 = HALF ? x0 : lds64(vb + 8 * s), y1 = HALF ? x1 : lds64(vb + 8 * s + 8);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const uint2 b0 = lds64(ub + 8 * n * ss + 8 * s), b1 = lds64(ub + 8 * n * ss + 8 * s + 8);
            mma_tf32(ev[n], x0.x, y0.x, x0.y, y0.y, b0.x, b0.y);
            mma_tf32(od[n], x1.x, y1.x, x1.y, y1.y, b1.x, b1.y);
        }
    }
    if (s < n8) {
        const uint2 x0 = lds64(va + 8 * s);
        const uint2 y0 = HALF ? x0 : lds64(vb + 8 * s);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const uint2 b0 = lds64(ub + 8 * n * ss + 8 * s);
            mma_tf32(ev[n], x0.x, y0.x, x0.y, y0.y, b0.x, b0.y);
        }
    }
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[n][e] = ev[n][e] + od[n][e];
}

// H = G U (KS k-steps of 8 path rows); each 8-column tile is added to the context rows.
template <int KS, bool HALF, int DP8>
__device__ __forceinline__ void h_phase(const float* GT, const float* U, int ss, int dp8, int g, int t, float* p0,
                                        float* p1, bool w0, bool w1) {
    uint32_t a[KS][4];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        a[kk][0] = ldsu(GT + g * kGtStride + 8 * kk + t);
        a[kk][2] = ldsu(GT + g * kGtStride + 8 * kk + t + 4);
        a[kk][1] = HALF ? 0u : ldsu(GT + (g + 8) * kGtStride + 8 * kk + t);
        a[kk][3] = HALF ? 0u : ldsu(GT + (g + 8) * kGtStride + 8 * kk + t + 4);
    }
    const float* ub = U + t * ss + g;
    const int n8 = DP8 > 0 ? DP8 : dp8;
#pragma unroll 2
    for (int nt = 0; nt < n8; ++nt) {
        const int d0 = 8 * nt;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < KS; ++kk)
            mma_tf32(c, a[kk][0], a[kk][1], a[kk][2], a[kk][3], ldsu(ub + 8 * kk * ss + d0),
                     ldsu(ub + (8 * kk + 4) * ss + d0));
        red_add2_if(w0, p0 + d0 + 2 * t, c[0], c[1]);
        if (!HALF) red_add2_if(w1, p1 + d0 + 2 * t, c[2], c[3]);
    }
}

// dU = G^T V for MT m-tiles of 16 path rows and KC k-steps of 8 contexts.
template <int MT, int KC, int DP8>
__device__ __forceinline__ void u_phase(const float* GT, const float* V, int ss, int dp8, int g, int t,
                                        float* const (&pr)[4], const bool (&pw)[4]) {
    uint32_t a[MT][KC][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
            a[mt][kc][0] = ldsu(GT + (8 * kc + t) * kGtStride + 16 * mt + g);
            a[mt][kc][1] = ldsu(GT + (8 * kc + t) * kGtStride + 16 * mt + g + 8);
            a[mt][kc][2] = ldsu(GT + (8 * kc + t + 4) * kGtStride + 16 * mt + g);
            a[mt][kc][3] = ldsu(GT + (8 * kc + t + 4) * kGtStride + 16 * mt + g + 8);
        }
    const float* vb = V + t * ss + g;
    const int n8 = DP8 > 0 ? DP8 : dp8;
#pragma unroll 2
    for (int nt = 0; nt < n8; ++nt) {
        const int d0 = 8 * nt;
        uint32_t b[KC][2];
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
            b[kc][0] = ldsu(vb + 8 * kc * ss + d0);
            b[kc][1] = ldsu(vb + (8 * kc + 4) * ss + d0);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int kc = 0; kc < KC; ++kc)
                mma_tf32(c, a[mt][kc][0], a[mt][kc][1], a[mt][kc][2], a[mt][kc][3], b[kc][0], b[kc][1]);
            red_add2_if(pw[2 * mt], pr[2 * mt] + d0 + 2 * t, c[0], c[1]);
            red_add2_if(pw[2 * mt + 1], pr[2 * mt + 1] + d0 + 2 * t, c[2], c[3]);
        }
    }
}

// DCH: float4 chunks of a row per lane (staging); WARPS: launch bound; D4 > 0: the row width
// (Dp / 4) of a benchmark configuration, so every loop bound and offset is a constant.
template <int DCH, int WARPS, int D4>
__global__ void __launch_bounds__(WARPS * 32, 1) hog7_kernel(HogArgs a) {
    extern __shared__ __align__(16) unsigned char k7_raw[];
    constexpr int DP8 = D4 / 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int warps = blockDim.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int d4 = D4 > 0 ? D4 : a.d4;
    const int dp = 4 * d4, dp8 = d4 / 2;
    const int ss = D4 > 0 ? k7_stride(4 * D4) : a.smem_stride;
    const int UR = a.urows;
    const int K = a.cache_rows, K0 = a.ctx_cache_rows;
    const int nwords = (K + 31) >> 5;
    unsigned char* base = k7_raw + ((128u - (smem_u32(k7_raw) & 127u)) & 127u);
    float* sig = reinterpret_cast<float*>(base);
    unsigned* touch = reinterpret_cast<unsigned*>(base + 4096);
    float* wbase = reinterpret_cast<float*>(base + 4096 + ((nwords * 4 + 127) & ~127));
    float* GT = wbase + static_cast<size_t>(warp) * k7_warp_floats(ss, UR);
    float* V = GT + kVRows * kGtStride;
    float* U = V + kVRows * ss;
    int* codes = reinterpret_cast<int*>(U + UR * ss);
    // this CTA's pending deltas: cached syn1 rows [0, K), then cached syn0 rows [0, K0)
    float* t2 = a.tier2 ? a.tier2 + static_cast<size_t>(blockIdx.x) * static_cast<size_t>(K + K0) * dp : nullptr;
    float* t2c = t2 ? t2 + static_cast<size_t>(K) * dp : nullptr;
    __shared__ int s_done;
    __shared__ unsigned s_merged;

    for (int i = tid; i < 1000; i += blockDim.x) sig[i] = a.sigmoid[i];
    for (int i = tid; i < nwords; i += blockDim.x) touch[i] = 0u;
    {  // staging zeroed once: padded rows are read (finite) but their results masked
        const int n = warps * static_cast<int>(k7_warp_floats(ss, UR)) + 32 * 4;
        for (int i = tid; i < n; i += blockDim.x) wbase[i] = 0.f;
    }
    if (tid == 0) {
        s_done = 0;
        s_merged = 0;
    }
    __syncthreads();

    // ---- the CTA's cache flush: the touched rows' pending deltas (all of them at the end)
    // are taken with an atomic exchange and added to the model scaled per row.
    auto drain_row = [&](float* src, float* dst, float sc) {
#pragma unroll
        for (int k = 0; k < DCH; ++k) {
            const int q = lane + 32 * k;
            if (k < DCH - 1 || q < d4) {
                const float4 dlt = atom_take4(src + 4 * q);
                if (nonzero4(dlt)) red_add4(dst + 4 * q, scale4(sc, dlt));
            }
        }
    };
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
                for (unsigned mm = __shfl_sync(kFull, m, src); mm; mm &= mm - 1) {
                    const int r = ((w0 + src) << 5) + __ffs(mm) - 1;
                    drain_row(t2 + static_cast<size_t>(r) * dp, a.syn1 + static_cast<size_t>(r) * dp,
                              a.row_scale ? a.row_scale[r] : a.hot_flush_scale);
                }
            }
        }
        for (int r = 0; r < K0; ++r)
            drain_row(t2c + static_cast<size_t>(r) * dp, a.syn0 + static_cast<size_t>(r) * dp,
                      a.row_scale ? a.row_scale[K + r] : a.hot_flush_scale);
        __threadfence();  // the other SMs see this flush before the CTA's next one
    };
    // row `src` (dp floats) -> shared memory, 16 bytes per lane (LDGSTS, through L2)
    auto stage_row = [&](float* dst, const float* src) {
#pragma unroll
        for (int k = 0; k < DCH; ++k) {
            const int q = lane + 32 * k;
            if (k < DCH - 1 || q < d4) cp_async16(dst + 4 * q, src + 4 * q);
        }
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
            // shrink_window (trainer.hpp:66-68): b = W - draw mod W, the draw reduced by a
            // 32x32 multiply-high of its top bits (uniform to within W / 2^32)
            const int b = a.window - static_cast<int>(__umulhi(static_cast<unsigned>(ctr_draw(a.win_key, static_cast<uint64_t>(ci)) >> 32),
                                                               static_cast<unsigned>(a.window)));
            const int64_t lo = max(s_lo, ci - b), hi = min(s_hi - 1, ci + b);
            ++n_centers;
            const int n = static_cast<int>(hi - lo);
            if (n == 0) continue;
            bool touched_cache = false;
            for (int q0 = 0; q0 < n; q0 += kVRows) {
                const int nb = min(kVRows, n - q0);
                int xid = 0;
                if (lane < nb) {
                    int64_t pos = lo + q0 + lane;
                    pos += pos >= ci;  // skip the center's own position
                    xid = a.kept[pos];
                }
                const unsigned hot_ctx = __ballot_sync(kFull, lane < nb && xid < K0);
                // H rows: the context's syn0 row, or the CTA's pending delta of a cached word
                const int x0 = __shfl_sync(kFull, xid, g), x1 = __shfl_sync(kFull, xid, (g + 8) & 31);
                float* pc0 = ((hot_ctx >> g) & 1u ? t2c : a.syn0) + static_cast<size_t>(x0) * dp;
                float* pc1 = ((hot_ctx >> (g + 8)) & 1u ? t2c : a.syn0) + static_cast<size_t>(x1) * dp;
                const bool w0 = g < nb, w1 = g + 8 < nb;
                __syncwarp();  // the previous batch is done with V, U and G
                for (int i = 0; i < nb; ++i) stage_row(V + i * ss, a.syn0 + static_cast<size_t>(__shfl_sync(kFull, xid, i)) * dp);
                for (int jc = 0; jc < L; jc += UR) {
                    const int Lc = min(UR, L - jc);
                    const bool restage = q0 == 0 || L > UR;  // U is kept across the batches of one chunk
                    int code = 0;
                    if (lane < Lc) code = a.path_code[p0 + jc + lane];
                    const int row = code >> 1;
                    if (restage) {
                        if (jc > 0) __syncwarp();  // the previous chunk is done with U and G
                        for (int j = 0; j < Lc; ++j)
                            stage_row(U + j * ss, a.syn1 + static_cast<size_t>(__shfl_sync(kFull, row, j)) * dp);
                        codes[lane] = code;
                    }
                    cp_async_wait_all();
                    __syncwarp();
                    // ---- S = V U^T, then G (masked) into the G scratch ----
                    const int NT = (Lc + 7) >> 3, MT = (Lc + 15) >> 4;
                    float acc[4][4];
#pragma unroll
                    for (int n2 = 0; n2 < 4; ++n2) acc[n2][0] = acc[n2][1] = acc[n2][2] = acc[n2][3] = 0.f;
                    const bool half = nb <= 8;
                    switch (NT * 2 + (half ? 1 : 0)) {
                        case 2: s_phase<1, false, DP8>(V, U, ss, dp8, g, t, acc); break;
                        case 3: s_phase<1, true, DP8>(V, U, ss, dp8, g, t, acc); break;
                        case 4: s_phase<2, false, DP8>(V, U, ss, dp8, g, t, acc); break;
                        case 5: s_phase<2, true, DP8>(V, U, ss, dp8, g, t, acc); break;
                        case 6: s_phase<3, false, DP8>(V, U, ss, dp8, g, t, acc); break;
                        case 7: s_phase<3, true, DP8>(V, U, ss, dp8, g, t, acc); break;
                        case 8: s_phase<4, false, DP8>(V, U, ss, dp8, g, t, acc); break;
                        default: s_phase<4, true, DP8>(V, U, ss, dp8, g, t, acc); break;
                    }
                    // GT[i][j]: i = context (rows g, g + 8), j = path row (columns 2t, 2t + 1 of tile n)
#pragma unroll
                    for (int n2 = 0; n2 < 4; ++n2) {
                        if (n2 >= 2 * MT) break;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int i = g + (e >> 1) * 8, j = 8 * n2 + 2 * t + (e & 1);
                            float gv = 0.f;
                            if (n2 < NT && i < nb && j < Lc)
                                gv = (1.0f - static_cast<float>(codes[j] & 1) - table_sigmoid(sig, acc[n2][e], a.sig_scale)) *
                                     alpha;
                            acc[n2][e] = gv;
                        }
                        *reinterpret_cast<float2*>(GT + g * kGtStride + 8 * n2 + 2 * t) = make_float2(acc[n2][0], acc[n2][1]);
                        *reinterpret_cast<float2*>(GT + (g + 8) * kGtStride + 8 * n2 + 2 * t) = make_float2(acc[n2][2], acc[n2][3]);
                    }
                    __syncwarp();
                    // ---- H = G U -> the context rows (v += h, trainer.hpp:173) ----
                    switch (NT * 2 + (half ? 1 : 0)) {
                        case 2: h_phase<1, false, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        case 3: h_phase<1, true, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        case 4: h_phase<2, false, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        case 5: h_phase<2, true, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        case 6: h_phase<3, false, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        case 7: h_phase<3, true, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        case 8: h_phase<4, false, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                        default: h_phase<4, true, DP8>(GT, U, ss, dp8, g, t, pc0, pc1, w0, w1); break;
                    }
                    // ---- dU = G^T V -> the path rows (syn1, or the CTA's delta of a cached row) ----
                    float* pr[4];
                    bool pw[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j = g + 8 * e;  // rows of m-tile e / 2, halves e % 2
                        const int rj = __shfl_sync(kFull, row, j);
                        pw[e] = j < Lc;
                        pr[e] = (rj < K ? t2 : a.syn1) + static_cast<size_t>(rj) * dp;
                    }
                    if (MT == 1) {
                        if (half) u_phase<1, 1, DP8>(GT, V, ss, dp8, g, t, pr, pw);
                        else u_phase<1, 2, DP8>(GT, V, ss, dp8, g, t, pr, pw);
                    } else {
                        if (half) u_phase<2, 1, DP8>(GT, V, ss, dp8, g, t, pr, pw);
                        else u_phase<2, 2, DP8>(GT, V, ss, dp8, g, t, pr, pw);
                    }
                    const bool cached = lane < Lc && row < K;
                    if (__any_sync(kFull, cached)) {
                        touched_cache = true;
                        if (cached) {
                            const unsigned bit = 1u << (row & 31);
                            if (!(touch[row >> 5] & bit)) atomicOr(&touch[row >> 5], bit);
                        }
                    }
                }
                if (hot_ctx) touched_cache = true;
            }
            n_pairs += static_cast<unsigned long long>(n);
            n_steps += static_cast<unsigned long long>(n) * static_cast<unsigned long long>(L);
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
    if (last && (K > 0 || K0 > 0)) flush_cache(true);
}

constexpr int kV7MaxWarps = 16;

template <int DCH, int D4>
void launch7(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    auto k = hog7_kernel<DCH, kV7MaxWarps, D4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
    k<<<g.blocks, g.warps * 32, g.smem, s>>>(a);
}

}  // namespace

bool hog7_plan(int d4, int cache_rows, int ctx_rows, int blocks, int warps_override, int cpw_override, int64_t tokens,
               int max_depth, HogGeometry* g) {
    if (d4 > 96) return false;
    const int dp = 4 * d4;
    const int ss = k7_stride(dp);
    const int nwords = (cache_rows + 31) / 32;
    const size_t fixed = 4096 + ((static_cast<size_t>(nwords) * 4 + 127) & ~size_t{127}) + 128 + 32 * 16;
    const size_t budget = 227 * 1024 - 1024;
    auto warps_for = [&](int ur) { return static_cast<int>((budget - fixed) / (k7_warp_floats(ss, ur) * 4)); };
    // Path rows staged per chunk: the deepest path when it fits in 32 rows, fewer (more
    // warps) while shared memory would leave fewer than 6 warps; a deeper path is trained
    // in chunks (the context rows stay staged).
    int urows = std::min(32, std::max(8, (max_depth + 7) / 8 * 8));
    while (urows > 16 && warps_for(urows) < 6) urows -= 8;
    int warps = std::min(kV7MaxWarps, warps_for(urows));
    if (warps_override > 0) warps = std::min(warps, warps_override);
    if (warps < 1) return false;
    g->variant = 7;
    g->warps = warps;
    g->blocks = blocks;
    g->cache_rows = cache_rows;
    g->smem_rows = 0;
    g->ctx_rows = ctx_rows;
    g->ctx_batch = kVRows;
    g->flusher = false;
    g->urows = urows;
    g->smem_stride = ss;
    g->specialise = true;
    g->smem = fixed + static_cast<size_t>(warps) * k7_warp_floats(ss, urows) * 4;
    g->cpw = cpw_override > 0 ? std::min(cpw_override, 32)
                              : (tokens / (static_cast<int64_t>(blocks) * warps) >= 2000 ? 16 : 8);
    return true;
}

void launch_hog7(const HogArgs& a0, const HogGeometry& g, cudaStream_t s) {
    HogArgs a = a0;
    a.cache_rows = g.cache_rows;
    a.smem_rows = 0;
    a.ctx_cache_rows = g.ctx_rows;
    a.centers_per_warp = g.cpw;
    a.ctx_batch = kVRows;
    a.flusher = 0;
    a.urows = g.urows;
    a.smem_stride = g.smem_stride;
    const int dch = (a.d4 + 31) / 32;
    switch (a.d4) {  // the benchmark row widths (D 100, 128, 200, 300 padded to 8 floats)
        case 26: launch7<1, 26>(a, g, s); return;
        case 32: launch7<1, 32>(a, g, s); return;
        case 50: launch7<2, 50>(a, g, s); return;
        case 76: launch7<3, 76>(a, g, s); return;
        default: break;
    }
    if (dch == 1) launch7<1, 0>(a, g, s);
    else if (dch == 2) launch7<2, 0>(a, g, s);
    else launch7<3, 0>(a, g, s);
}

}  // namespace cgk
