// cg_hog8.cu -- K1 v8 (the default): Hogwild skip-gram HS training with each center's
// products on the tensor cores.
//
// For one center c with its batch of contexts x_0..x_{n-1} (syn0 rows v_i) and its root-first
// path rows u_0..u_{L-1} (syn1), train_center (trainer.hpp:147-175) in K1's center-batched
// order (every context's dots against the rows as loaded: within-center staleness of at most
// 2W updates, as in v5) is three small matrix products:
//     S  = V U^T            (n x L)  the dot products            (vec_ops.hpp:14-18)
//     G  = (1 - turn - sigmoid(S)) * alpha, zero outside the real pairs (trainer.hpp:166-167)
//     H  = G U              (n x D)  h_i = sum_j g_ij u_j         (trainer.hpp:168)
//     dU = G^T V            (L x D)  u_j += sum_i g_ij v_i        (trainer.hpp:171)
// then v_i += h_i (trainer.hpp:173). One warp computes them with mma.sync m16n8k16 (f16
// operands, fp32 accumulation) out of shared memory: contexts are the M dimension of S and H
// (16 per tile), path rows the N dimension of S, the K dimension of H and the M dimension of
// dU. A center costs ~10x fewer instructions than the FP32 FMA kernel (v5), which spends
// them on per-lane FMAs and the transpose-reduce of the dots.
//
// Operands: the rows are converted to fp16 as they are staged -- 10 mantissa bits, rounded
// to nearest (TF32's operand precision); the fp32 model in HBM is unchanged and every sum
// is fp32; the sigmoid is the reference's 1000-bucket table (bucket width 0.012), far
// coarser than the operand rounding. fp16 staging halves a warp's shared memory against
// fp32 (fp32-staged TF32 operands left 6 and 5 warps per SM at D 200 / 300: v7, measured
// slower than v5 for that reason and removed). Staging goes through registers: every lane
// loads its 16-byte chunks of 4-6 rows at once (ld.global.cg, coherent with the rows'
// red.global updates at L2), converts them to half2 pairs and stores them -- row by row for
// wide rows, as a flat list of (row, chunk) items for rows of at most 32 chunks -- no fp32 ring in
// shared memory, which is what bounds the warps per SM. A warp holds min(16, 2W) context
// rows and `urows` path rows; tile rows beyond them are read from one all-zero row the CTA
// shares (ldmatrix takes a row address per lane). Every fragment load is one ldmatrix --
// m8n8.x4 for the row-major operands, .trans for U as H's B, G^T as dU's A and V as dU's B;
// row strides of 8 (mod 16) halves put the eight 16-byte rows of each matrix in distinct
// banks.
//
// H and dU leave straight from the accumulator fragments with red.global.add.v2.f32 (no
// lost updates). ptxas never predicates a REDG: a lane-divergent guard costs BSSY + BRA
// + BSYNC around each one (29% of the stall samples of the first v8, which guarded every
// REDG per lane). Here an 8-row group of the tile with no real row is skipped by a test the
// compiler knows to be warp-uniform (template parameters HI / FULL), and only the lanes of
// the padding rows inside a partly filled group branch. (Sending the padding rows' zeros to
// a scratch row instead, branch-free, measured 16% slower, and pairing lanes by shuffle for
// 16-byte REDGs 4% slower: C5 2775 and 2502 ms against 2398.) The per-CTA
// node cache (NodeCache, trainer.hpp:75-138): the K cached syn1 rows and the most frequent
// words' syn0 rows take their updates in CTA-private delta rows in L2 (`tier2`), which the
// flush drains by atomic exchange and adds to the model scaled per row; warps read a cached
// row's flushed state (write-combining: a CTA's own pending delta joins the row at its
// flush, like every other CTA's).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include <cuda_fp16.h>

#include "cg_device.cuh"
#include "cg_kernels.h"

namespace cgk {
namespace {

using namespace cgdev;

constexpr int kTileRows = 16;  // M of one mma tile: context rows per batch
constexpr int kGhStride = 40;  // fp16 G scratch [16 contexts][32 path rows], 80-byte rows
#ifndef CG_K8_UNROLL
#define CG_K8_UNROLL 4  // tiles per unrolled step of the S, H and dU loops (1 / 2 / 4 at C5: 2414 / 2338 / 2314 ms)
#endif
#define CG_PRAGMA(x) _Pragma(#x)
#define CG_UNROLL(n) CG_PRAGMA(unroll n)
#ifndef CG_K8_STAGE3
#define CG_K8_STAGE3 6
#endif
// rows a lane has in flight (registers) while staging, by 16-byte chunks per lane and row
__host__ __device__ constexpr int k8_stage(int dch) { return dch >= 3 ? CG_K8_STAGE3 : 4; }
// Rows of at most 32 chunks (D <= 128) stage as a flat list of (row, chunk) items, every lane
// busy and no test per row (C3 75.8 -> 70.9 ms); wider rows stage row by row: the flat
// list's address table costs them a warp of shared memory (C5 2335 -> 2588 ms with it).
__host__ __device__ constexpr bool k8_flat(int dch) { return dch == 1; }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const __half* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const __half* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// red.global.add.v2.f32 (REDG.E.ADD.F32x2) into a model row; a null row is a padding row of
// the tile: its lanes branch around the REDG (ptxas never predicates one), which costs less
// than sending their zeros to L2 (measured: C5 2386 ms against 2775 ms with a scratch row).
__device__ __forceinline__ void red_add2(float* row, int col, float x, float y) {
    if (row == nullptr) return;
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(row + col), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ uint32_t half2_bits(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// fp16 row stride (halves) for rows of dp floats: dp rounded up to 16 (the mma K step),
// plus 8 -- 8 (mod 16) halves, an odd number of 16-byte chunks.
__host__ __device__ constexpr int k8_stride(int dp) { return (dp + 15) / 16 * 16 + 8; }
// Per-warp bytes: G scratch | V (vrows context rows) | U (urows path rows) | codes (32 ints)
// | flat staging: 48 row addresses.
__host__ __device__ constexpr uint32_t k8_warp_bytes(int ssh, int vrows, int urows, int dch) {
    return static_cast<uint32_t>(kTileRows * kGhStride * 2 + (vrows + urows) * ssh * 2 + 32 * 4 + (k8_flat(dch) ? 48 * 8 : 0));
}
// Bytes ahead of the warps' regions: sigmoid table | touched-row bitmap | the all-zero row.
__host__ __device__ constexpr uint32_t k8_fixed_bytes(int ssh, int cache_rows) {
    return 4096u + ((static_cast<uint32_t>((cache_rows + 31) / 32) * 4u + 127u) & ~127u) +
           ((static_cast<uint32_t>(ssh) * 2u + 127u) & ~127u);
}

// S = V U^T for NP pairs of 8-row n-tiles over K16 k-steps of 16 columns. The A fragment of
// each k-step is one ldmatrix.x4 of V (pa: this lane's row of the 16 x 16 tile); the B
// fragments of two n-tiles one ldmatrix.x4 of U (pb[np]: this lane's row of pair np).
template <int NP, int K16>
__device__ __forceinline__ void s_phase(const __half* pa, const __half* const (&pb)[2], int k16, float (&acc)[4][4]) {
    const int n16 = K16 > 0 ? K16 : k16;
CG_UNROLL(CG_K8_UNROLL)
    for (int ks = 0; ks < n16; ++ks) {
        uint32_t a[4];
        ldsm_x4(a, pa + 16 * ks);
#pragma unroll
        for (int np = 0; np < NP; ++np) {
            uint32_t b[4];
            ldsm_x4(b, pb[np] + 16 * ks);
            mma_f16(acc[2 * np], a, b[0], b[1]);
            mma_f16(acc[2 * np + 1], a, b[2], b[3]);
        }
    }
}

// H = G U over KS k-steps of 16 path rows (pb[kk]: this lane's U row of k-step kk); each pair
// of 8-column tiles goes to the context rows g (p0) and, when the batch has more than 8
// contexts (HI), g + 8 (p1). A padding context has a null row.
template <int KS, int K16, bool HI>
__device__ __forceinline__ void h_phase(const __half* GH, const __half* const (&pb)[2], int k16, int dp, int lane, float* p0,
                                        float* p1) {
    const int m = lane >> 3, rr = lane & 7, t = lane & 3;
    uint32_t a[KS][4];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) ldsm_x4(a[kk], GH + (rr + 8 * (m & 1)) * kGhStride + 16 * kk + 8 * (m >> 1));
    const int n16 = K16 > 0 ? K16 : k16;
CG_UNROLL(CG_K8_UNROLL)
    for (int np = 0; np < n16; ++np) {
        float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            uint32_t b[4];
            ldsm_x4_t(b, pb[kk] + 16 * np);
            mma_f16(c0, a[kk], b[0], b[1]);
            mma_f16(c1, a[kk], b[2], b[3]);
        }
        const int d0 = 16 * np + 2 * t;
        const bool second = 16 * np + 8 < dp;  // warp-uniform: dp is a multiple of 8
        red_add2(p0, d0, c0[0], c0[1]);
        if (second) red_add2(p0, d0 + 8, c1[0], c1[1]);
        if constexpr (HI) {
            red_add2(p1, d0, c0[2], c0[3]);
            if (second) red_add2(p1, d0 + 8, c1[2], c1[3]);
        }
    }
}

// dU = G^T V for MT m-tiles of 16 path rows (one k-step: the batch's 16 contexts; pb: this
// lane's V row). pr[e]: the row g + 8 e of this lane (null for padding rows); FULL: the
// last 8-row group of the MT tiles holds a real path row.
template <int MT, int K16, bool FULL>
__device__ __forceinline__ void u_phase(const __half* GH, const __half* pb, int k16, int dp, int lane,
                                        float* const (&pr)[4]) {
    const int m = lane >> 3, rr = lane & 7, t = lane & 3;
    uint32_t a[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) ldsm_x4_t(a[mt], GH + (rr + 8 * (m >> 1)) * kGhStride + 16 * mt + 8 * (m & 1));
    const int n16 = K16 > 0 ? K16 : k16;
CG_UNROLL(CG_K8_UNROLL)
    for (int np = 0; np < n16; ++np) {
        uint32_t b[4];
        ldsm_x4_t(b, pb + 16 * np);
        const int d0 = 16 * np + 2 * t;
        const bool second = 16 * np + 8 < dp;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
            mma_f16(c0, a[mt], b[0], b[1]);
            mma_f16(c1, a[mt], b[2], b[3]);
            red_add2(pr[2 * mt], d0, c0[0], c0[1]);
            if (second) red_add2(pr[2 * mt], d0 + 8, c1[0], c1[1]);
            if (FULL || mt + 1 < MT) {
                red_add2(pr[2 * mt + 1], d0, c0[2], c0[3]);
                if (second) red_add2(pr[2 * mt + 1], d0 + 8, c1[2], c1[3]);
            }
        }
    }
}

// DCH: float4 chunks of a row per lane (staging); WARPS: launch bound; D4 > 0: the row
// width (Dp / 4) of a benchmark configuration (constant loop bounds and offsets).
template <int DCH, int WARPS, int D4>
__global__ void __launch_bounds__(WARPS * 32, 1) hog8_kernel(HogArgs a) {
    extern __shared__ __align__(16) unsigned char k8_raw[];
    constexpr int K16 = D4 > 0 ? (4 * D4 + 15) / 16 : 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int warps = blockDim.x >> 5;
    const int g = lane >> 2;
    const int d4 = D4 > 0 ? D4 : a.d4;
    const int dp = 4 * d4, k16 = (dp + 15) / 16;
    const int ssh = D4 > 0 ? k8_stride(4 * D4) : a.smem_stride;
    const int UR = a.urows, VR = a.ctx_batch;
    const int K = a.cache_rows, K0 = a.ctx_cache_rows;
    const int nwords = (K + 31) >> 5;
    unsigned char* base = k8_raw + ((128u - (smem_u32(k8_raw) & 127u)) & 127u);
    float* sig = reinterpret_cast<float*>(base);
    unsigned* touch = reinterpret_cast<unsigned*>(base + 4096);
    unsigned char* wbase = base + k8_fixed_bytes(ssh, K);
    const __half* zrow = reinterpret_cast<const __half*>(wbase - ((static_cast<uint32_t>(ssh) * 2u + 127u) & ~127u));
    unsigned char* wp = wbase + static_cast<size_t>(warp) * k8_warp_bytes(ssh, VR, UR, DCH);
    __half* GH = reinterpret_cast<__half*>(wp);
    __half* V = GH + kTileRows * kGhStride;
    __half* U = V + VR * ssh;
    int* codes = reinterpret_cast<int*>(U + UR * ssh);
    float* t2 = a.tier2 ? a.tier2 + static_cast<size_t>(blockIdx.x) * static_cast<size_t>(K + K0) * dp : nullptr;
    float* t2c = t2 ? t2 + static_cast<size_t>(K) * dp : nullptr;
    float* const scr = nullptr;  // the row pointer of a padding tile row
    __shared__ int s_done;
    __shared__ unsigned s_merged;

    for (int i = tid; i < 1000; i += blockDim.x) sig[i] = a.sigmoid[i];
    for (int i = tid; i < nwords; i += blockDim.x) touch[i] = 0u;
    {  // zero row and staging zeroed once: the columns past a row and stale rows stay finite
        uint4* z = reinterpret_cast<uint4*>(const_cast<__half*>(zrow));
        const int n = static_cast<int>((((static_cast<uint32_t>(ssh) * 2u + 127u) & ~127u) +
                                        warps * k8_warp_bytes(ssh, VR, UR, DCH)) / 16);
        for (int i = tid; i < n; i += blockDim.x) z[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (tid == 0) {
        s_done = 0;
        s_merged = 0;
    }
    __syncthreads();

    // this lane's ldmatrix rows (tile rows past the staged ones read the zero row)
    const int lm = lane >> 3, lr = lane & 7;
    auto v_row = [&](int r) { return r < VR ? V + r * ssh : zrow; };
    auto u_row = [&](int r) { return r < UR ? U + r * ssh : zrow; };
    const __half* pa_s = v_row(lr + 8 * (lm & 1)) + 8 * (lm >> 1);                       // S: A = V
    const __half* pb_s[2] = {u_row(lr + 8 * (lm >> 1)) + 8 * (lm & 1),                   // S: B = U
                             u_row(16 + lr + 8 * (lm >> 1)) + 8 * (lm & 1)};
    const __half* pb_h[2] = {u_row(lr + 8 * (lm & 1)) + 8 * (lm >> 1),                   // H: B = U (trans)
                             u_row(16 + lr + 8 * (lm & 1)) + 8 * (lm >> 1)};
    const __half* pb_u = v_row(lr + 8 * (lm & 1)) + 8 * (lm >> 1);                       // dU: B = V (trans)

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

    // rows -> fp16 in shared memory through registers: kStage rows in flight per lane
    // (ld.global.cg: through L2, like the rows' red.global updates), each lane converting
    // the 16-byte chunks it loaded to half2 pairs (round to nearest).
    auto stage_rows = [&](int nrows, auto&& src_of, auto&& dst_of) {
        constexpr int kStage = k8_stage(DCH);
        for (int r0 = 0; r0 < nrows; r0 += kStage) {
            float4 buf[kStage][DCH];
#pragma unroll
            for (int r = 0; r < kStage; ++r) {
                const float* src = src_of(min(r0 + r, nrows - 1));  // every lane takes part in the shuffles
                if (r0 + r < nrows) {
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (k < DCH - 1 || q < d4) buf[r][k] = ld_cg4(src + 4 * q);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < kStage; ++r) {
                if (r0 + r < nrows) {
                    __half* d = dst_of(r0 + r);
#pragma unroll
                    for (int k = 0; k < DCH; ++k) {
                        const int q = lane + 32 * k;
                        if (k < DCH - 1 || q < d4)
                            *reinterpret_cast<uint2*>(d + 4 * q) =
                                make_uint2(half2_bits(buf[r][k].x, buf[r][k].y), half2_bits(buf[r][k].z, buf[r][k].w));
                    }
                }
            }
        }
    };

    // Flat staging: the nv context rows (into V) and nu path rows (into U, which follows V)
    // are one list of (row, 16-byte chunk) items; lane l takes items l, l + 32, ... so every
    // lane loads and converts, whatever the row width. Lanes publish their rows' global
    // addresses in the warp's table first (lane i: context i, lane j: path row j).
    unsigned long long* rtab = reinterpret_cast<unsigned long long*>(codes + 32);
    const unsigned rcp = 0xffffffffu / static_cast<unsigned>(d4) + 1u;  // i / d4 = umulhi(i, rcp) for i < 2^25
    auto stage_flat = [&](int nv, int nu, int xid, int row) {
        constexpr int kItems = k8_stage(DCH) * DCH;
        if (lane < nv) rtab[lane] = reinterpret_cast<unsigned long long>(a.syn0 + static_cast<size_t>(xid) * dp);
        if (lane < nu) rtab[nv + lane] = reinterpret_cast<unsigned long long>(a.syn1 + static_cast<size_t>(row) * dp);
        __syncwarp();
        const int total = (nv + nu) * d4, dshift = VR - nv;
        for (int i0 = lane; i0 < total; i0 += 32 * kItems) {
            float4 buf[kItems];
#pragma unroll
            for (int u = 0; u < kItems; ++u) {
                const int i = i0 + 32 * u;
                if (i < total) {
                    const int r = D4 > 0 ? i / D4 : static_cast<int>(__umulhi(static_cast<unsigned>(i), rcp));
                    const int q = i - r * d4;
                    buf[u] = ld_cg4(reinterpret_cast<const float*>(rtab[r]) + 4 * q);
                }
            }
#pragma unroll
            for (int u = 0; u < kItems; ++u) {
                const int i = i0 + 32 * u;
                if (i < total) {
                    const int r = D4 > 0 ? i / D4 : static_cast<int>(__umulhi(static_cast<unsigned>(i), rcp));
                    const int q = i - r * d4;
                    __half* d = V + (r + (r >= nv ? dshift : 0)) * ssh + 4 * q;
                    *reinterpret_cast<uint2*>(d) = make_uint2(half2_bits(buf[u].x, buf[u].y), half2_bits(buf[u].z, buf[u].w));
                }
            }
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
            for (int q0 = 0; q0 < n; q0 += VR) {
                const int nb = min(VR, n - q0);
                int xid = 0;
                if (lane < nb) {
                    int64_t pos = lo + q0 + lane;
                    pos += pos >= ci;  // skip the center's own position
                    xid = a.kept[pos];
                }
                const unsigned hot_ctx = __ballot_sync(kFull, lane < nb && xid < K0);
                const int x0 = __shfl_sync(kFull, xid, g), x1 = __shfl_sync(kFull, xid, (g + 8) & 31);
                // the context rows of this lane's accumulator rows g, g + 8 (null when padding)
                float* pc0 = g < nb ? ((hot_ctx >> g) & 1u ? t2c : a.syn0) + static_cast<size_t>(x0) * dp : scr;
                float* pc1 = g + 8 < nb ? ((hot_ctx >> (g + 8)) & 1u ? t2c : a.syn0) + static_cast<size_t>(x1) * dp : scr;
                for (int jc = 0; jc < L; jc += UR) {
                    const int Lc = min(UR, L - jc);
                    const bool restage = q0 == 0 || L > UR;  // U is kept across the batches of one chunk
                    int code = 0;
                    if (lane < Lc) code = a.path_code[p0 + jc + lane];
                    const int row = code >> 1;
                    __syncwarp();  // the previous chunk / batch is done with V, U and G
                    {  // the batch's context rows (first chunk) and the chunk's path rows, as fp16
                        const int nv = jc == 0 ? nb : 0, nu = restage ? Lc : 0;
                        if constexpr (k8_flat(DCH)) stage_flat(nv, nu, xid, row);
                        else stage_rows(
                            nv + nu,
                            [&](int r) {
                                return r < nv ? a.syn0 + static_cast<size_t>(__shfl_sync(kFull, xid, r)) * dp
                                              : a.syn1 + static_cast<size_t>(__shfl_sync(kFull, row, r - nv)) * dp;
                            },
                            [&](int r) { return r < nv ? V + r * ssh : U + (r - nv) * ssh; });
                        if (restage) codes[lane] = code;
                    }
                    __syncwarp();
                    // ---- S = V U^T, then G (masked, fp16) into the G scratch ----
                    const int NP = (Lc + 15) >> 4;  // pairs of 8-row n-tiles (16 path rows)
                    float acc[4][4];
#pragma unroll
                    for (int n2 = 0; n2 < 4; ++n2) acc[n2][0] = acc[n2][1] = acc[n2][2] = acc[n2][3] = 0.f;
                    if (NP == 1) s_phase<1, K16>(pa_s, pb_s, k16, acc);
                    else s_phase<2, K16>(pa_s, pb_s, k16, acc);
                    const int t = lane & 3;
#pragma unroll
                    for (int n2 = 0; n2 < 4; ++n2) {
                        if (n2 >= 2 * NP) break;
                        float gv[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int i = g + (e >> 1) * 8, j = 8 * n2 + 2 * t + (e & 1);
                            gv[e] = 0.f;
                            if (i < nb && j < Lc)
                                gv[e] = (1.0f - static_cast<float>(codes[j] & 1) - table_sigmoid(sig, acc[n2][e], a.sig_scale)) * alpha;
                        }
                        *reinterpret_cast<uint32_t*>(GH + g * kGhStride + 8 * n2 + 2 * t) = half2_bits(gv[0], gv[1]);
                        *reinterpret_cast<uint32_t*>(GH + (g + 8) * kGhStride + 8 * n2 + 2 * t) = half2_bits(gv[2], gv[3]);
                    }
                    __syncwarp();
                    // ---- H = G U -> the context rows (v += h, trainer.hpp:173) ----
                    if (NP == 1) {
                        if (nb > 8) h_phase<1, K16, true>(GH, pb_h, k16, dp, lane, pc0, pc1);
                        else h_phase<1, K16, false>(GH, pb_h, k16, dp, lane, pc0, pc1);
                    } else {
                        if (nb > 8) h_phase<2, K16, true>(GH, pb_h, k16, dp, lane, pc0, pc1);
                        else h_phase<2, K16, false>(GH, pb_h, k16, dp, lane, pc0, pc1);
                    }
                    // ---- dU = G^T V -> the path rows (syn1, or the CTA's delta of a cached row) ----
                    float* pr[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int j = g + 8 * e;  // m-tile e / 2, rows g and g + 8
                        const int rj = __shfl_sync(kFull, row, j);
                        pr[e] = j < Lc ? (rj < K ? t2 : a.syn1) + static_cast<size_t>(rj) * dp : scr;
                    }
                    const bool full = ((Lc - 1) & 15) >= 8;  // the tiles' last 8-row group has a real row
                    if (NP == 1) {
                        if (full) u_phase<1, K16, true>(GH, pb_u, k16, dp, lane, pr);
                        else u_phase<1, K16, false>(GH, pb_u, k16, dp, lane, pr);
                    } else {
                        if (full) u_phase<2, K16, true>(GH, pb_u, k16, dp, lane, pr);
                        else u_phase<2, K16, false>(GH, pb_u, k16, dp, lane, pr);
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

template <int DCH, int WARPS, int D4>
void launch8(const HogArgs& a, const HogGeometry& g, cudaStream_t s) {
    auto k = hog8_kernel<DCH, WARPS, D4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
    k<<<g.blocks, g.warps * 32, g.smem, s>>>(a);
}

// Warps per CTA each staging width is compiled for (the launch bound sets the register cap:
// 128 at 16 warps, 146 at 14, 204 at 10). Shared memory holds no more than these at the
// benchmark widths anyway (D 200: 14 warps with 24 path rows; D 300: 10).
constexpr int k8_max_warps(int dch) { return dch >= 3 ? 10 : dch == 2 ? 14 : 16; }

}  // namespace

bool hog8_plan(int d4, int cache_rows, int ctx_rows, int blocks, int warps_override, int cpw_override, int64_t tokens,
               int max_depth, int window, HogGeometry* g) {
    if (d4 > 96) return false;
    const int dp = 4 * d4;
    const int ssh = k8_stride(dp);
    const size_t fixed = k8_fixed_bytes(ssh, cache_rows) + 128;
    const size_t budget = 227 * 1024 - 1024;
    // context rows staged per batch: a full window when it fits the 16-row tile
    const int vrows = std::min(kTileRows, std::max(2, 2 * window));
    auto warps_for = [&](int ur) { return static_cast<int>((budget - fixed) / k8_warp_bytes(ssh, vrows, ur, (d4 + 31) / 32)); };
    const int cap = k8_max_warps((d4 + 31) / 32);
    // Path rows staged per chunk (a deeper path trains in chunks, its contexts staying
    // staged; every chunk repeats the H phase): the deepest path rounded up to 4, at least 16
    // and at most 24 -- more rows cost more warps than the second chunk of the few deeper
    // paths (measured, K1 ms at 16 / 20 / 24 / 28 / 32 rows: C5, depth 26: 3109 / 2452 / 2338 /
    // 2424 / 3053; C4, depth 20: 914 / 719 / 763 / 833 / 934). CG_UROWS overrides (experiments).
    int urows = std::min(24, std::max(16, (max_depth + 3) / 4 * 4));
    if (std::min(cap, warps_for(urows)) < 8) urows = 16;
    if (const char* e = std::getenv("CG_UROWS")) {
        const int v = std::atoi(e);
        if (v >= 16 && v <= 32 && v % 4 == 0) urows = v;
    }
    int warps = std::min(cap, warps_for(urows));
    if (warps_override > 0) warps = std::min(warps, warps_override);
    if (warps < 1) return false;
    g->variant = 8;
    g->warps = warps;
    g->blocks = blocks;
    g->cache_rows = cache_rows;
    g->smem_rows = 0;
    g->ctx_rows = ctx_rows;
    g->ctx_batch = vrows;
    g->flusher = false;
    g->urows = urows;
    g->smem_stride = ssh;
    g->specialise = true;
    g->smem = fixed + static_cast<size_t>(warps) * k8_warp_bytes(ssh, vrows, urows, (d4 + 31) / 32);
    g->cpw = cpw_override > 0 ? std::min(cpw_override, 32)
                              : (tokens / (static_cast<int64_t>(blocks) * warps) >= 2000 ? 16 : 8);
    return true;
}

void launch_hog8(const HogArgs& a0, const HogGeometry& g, cudaStream_t s) {
    HogArgs a = a0;
    a.cache_rows = g.cache_rows;
    a.smem_rows = 0;
    a.ctx_cache_rows = g.ctx_rows;
    a.centers_per_warp = g.cpw;
    a.ctx_batch = g.ctx_batch;
    a.flusher = 0;
    a.urows = g.urows;
    a.smem_stride = g.smem_stride;
    const int dch = (a.d4 + 31) / 32;
    switch (a.d4) {  // the benchmark row widths (D 100, 128, 200, 300 padded to 8 floats)
        case 26: launch8<1, k8_max_warps(1), 26>(a, g, s); return;
        case 32: launch8<1, k8_max_warps(1), 32>(a, g, s); return;
        case 50: launch8<2, k8_max_warps(2), 50>(a, g, s); return;
        case 76: launch8<3, k8_max_warps(3), 76>(a, g, s); return;
        default: break;
    }
    if (dch == 1) launch8<1, k8_max_warps(1), 0>(a, g, s);
    else if (dch == 2) launch8<2, k8_max_warps(2), 0>(a, g, s);
    else launch8<3, k8_max_warps(3), 0>(a, g, s);
}

}  // namespace cgk
