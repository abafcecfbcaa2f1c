// cg_device.cuh -- device helpers shared by the sm_100a kernels of libcachegram_b200.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cgdev {

constexpr int kSentence = 1000;      // trainer.hpp:185 kMaxSentence
constexpr uint64_t kAlphaBatch = 10000;  // trainer.hpp:186 kAlphaBatch
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr unsigned kFull = 0xffffffffu;

// splitmix64 finaliser (rng.hpp:19-21). Draw i (0-based) of a stream seeded with s is
// mix64(s + (i+1)*golden), which makes the generator counter-based on the device.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t ctr_draw(uint64_t key, uint64_t index) {
    return mix64(key + (index + 1) * kGolden);
}
// Sequential stream (rng.hpp:17-22), used by the deterministic kernel.
__device__ __forceinline__ uint64_t seq_next(uint64_t& s) {
    s += kGolden;
    return mix64(s);
}
__host__ __device__ __forceinline__ float unit24(uint64_t z) {  // rng.hpp:25-27
    return static_cast<float>(z >> 40) * (1.0f / 16777216.0f);
}

// trainer.hpp:58-63, IEEE double then float, no contraction.
__device__ __forceinline__ float update_alpha(uint64_t done, uint64_t total, float alpha0) {
    const double frac = __ddiv_rn(static_cast<double>(done), __dadd_rn(static_cast<double>(total), 1.0));
    const float a = __fmul_rn(alpha0, static_cast<float>(__dsub_rn(1.0, frac)));
    const float lo = __fmul_rn(alpha0, 1e-4f);
    return a > lo ? a : lo;
}

// SigmoidTable::value (model.hpp:93-99) with the table in shared memory.
__device__ __forceinline__ float table_sigmoid(const float* t, float x, float scale) {
    if (x <= -6.0f) return t[0];
    if (x >= 6.0f) return t[999];
    int idx = __float2int_rz(__fmul_rn(__fadd_rn(x, 6.0f), scale));
    return t[idx > 999 ? 999 : idx];
}

// ---- memory ops -------------------------------------------------------------
// L2-coherent 128-bit load (bypasses L1): rows that other warps update with red.
__device__ __forceinline__ float4 ld_cg4(const float* p) {
    float4 r;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
// L1-allocating 128-bit load: hot-row bases that only change at block flushes.
__device__ __forceinline__ float4 ld_ca4(const float* p) {
    float4 r;
    asm volatile("ld.global.ca.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_cg4(float* p, float4 v) {
    asm volatile("st.global.cg.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
// Asynchronous 16-byte global -> shared copy through L2 (LDGSTS, bypassing L1 like
// ld.global.cg); completes at cp_async_wait_all().
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// Fire-and-forget vector atomic add at L2 (REDG.E.ADD.F32x4).
__device__ __forceinline__ void red_add4(float* p, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// Named barriers (bar.arrive / bar.sync with an explicit thread count): a consumer warp
// blocks in hardware, producers signal without waiting.
__device__ __forceinline__ void named_bar_arrive(int id, int threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ float4 f4(float a) { return make_float4(a, a, a, a); }

// ---- packed fp32 (sm_100: FFMA2 / FADD2 / FMUL2, two lanes of math per instruction) ----
// A float4 lives in four consecutive registers, so .xy and .zw are aligned register pairs
// and every float4 op below is two packed instructions. A scalar operand is broadcast
// by the instruction itself (SASS `R.F32`), so no register pair has to be built for it.
__device__ __forceinline__ float2 lo2(float4 a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ float2 hi2(float4 a) { return make_float2(a.z, a.w); }
__device__ __forceinline__ float4 cat4(float2 l, float2 h) { return make_float4(l.x, l.y, h.x, h.y); }
#ifndef CG_FFMA2
#define CG_FFMA2 1  // 0: scalar FFMA/FADD (same results up to rounding order; experiments: tools/ab_build.py)
#endif
#if CG_FFMA2
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return cat4(__fadd2_rn(lo2(a), lo2(b)), __fadd2_rn(hi2(a), hi2(b)));
}
// a + s*b
__device__ __forceinline__ float4 axpy4(float s, float4 b, float4 a) {
    const float2 ss = make_float2(s, s);
    return cat4(__ffma2_rn(ss, lo2(b), lo2(a)), __ffma2_rn(ss, hi2(b), hi2(a)));
}
__device__ __forceinline__ float4 scale4(float s, float4 b) {
    const float2 ss = make_float2(s, s);
    return cat4(__fmul2_rn(ss, lo2(b)), __fmul2_rn(ss, hi2(b)));
}
// Partial dot product in two interleaved sums (even and odd components); the caller
// adds .x + .y once per dot.
__device__ __forceinline__ float2 dot4(float4 a, float4 b, float2 acc) {
    acc = __ffma2_rn(lo2(a), lo2(b), acc);
    return __ffma2_rn(hi2(a), hi2(b), acc);
}
#else
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 axpy4(float s, float4 b, float4 a) {
    return make_float4(fmaf(s, b.x, a.x), fmaf(s, b.y, a.y), fmaf(s, b.z, a.z), fmaf(s, b.w, a.w));
}
__device__ __forceinline__ float4 scale4(float s, float4 b) { return make_float4(s * b.x, s * b.y, s * b.z, s * b.w); }
__device__ __forceinline__ float2 dot4(float4 a, float4 b, float2 acc) {
    acc.x = fmaf(a.x, b.x, acc.x);
    acc.x = fmaf(a.y, b.y, acc.x);
    acc.x = fmaf(a.z, b.z, acc.x);
    acc.x = fmaf(a.w, b.w, acc.x);
    return acc;
}
#endif
__device__ __forceinline__ bool nonzero4(float4 a) { return a.x != 0.f || a.y != 0.f || a.z != 0.f || a.w != 0.f; }

// ---- atomics, bulk copies and mbarriers ----------------------------------------
// Reads a 16-byte vector and leaves zeros in one atomic step (ATOMG.EXCH.128): drains
// a delta row that other warps keep adding to with red.global without losing an add.
__device__ __forceinline__ float4 atom_take4(float* p) {
    unsigned long long lo, hi;
    asm volatile(
        "{\n\t.reg .b128 d, b;\n\tmov.b128 b, {%2, %2};\n\tatom.global.exch.b128 d, [%3], b;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(lo), "=l"(hi)
        : "l"(0ull), "l"(p)
        : "memory");
    return make_float4(__uint_as_float(static_cast<unsigned>(lo)), __uint_as_float(static_cast<unsigned>(lo >> 32)),
                       __uint_as_float(static_cast<unsigned>(hi)), __uint_as_float(static_cast<unsigned>(hi >> 32)));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
// One arrival that also expects `bytes` of bulk-copy completions in this phase.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
            smem_u32(mb)),
        "r"(parity)
        : "memory");
}
// Global -> shared bulk copy by the TMA unit (UBLKCP), completing on an mbarrier. Goes
// through L2 like cp.async.cg: coherent with the red.global updates of other SMs.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(mb))
                 : "memory");
}
// Shared -> global bulk reduction by the TMA unit (UBLKRED): dst[0..bytes) += src[0..bytes)
// as f32 adds at L2, one instruction per row instead of one REDG per lane and 16 bytes.
// Tracked by the issuing thread's bulk async-group (bulk_commit / bulk_wait_read).
__device__ __forceinline__ void bulk_red_add_f32(float* dst, const void* src, unsigned bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Waits until the sources of this thread's bulk groups (all but the newest N) have been read.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// Orders this thread's generic-proxy shared-memory writes before later bulk copies.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- warp transpose-reduce ---------------------------------------------------
// p[0..N) are per-lane partial sums of N independent dot products (N a power of two,
// N <= 32). Returns the warp total of value index (lane >> (5 - log2 N)); costs
// N - 1 + 5 - log2 N shuffles instead of 5N for N independent butterflies.
template <int N>
struct Log2 {
    static constexpr int v = N <= 1 ? 0 : 1 + Log2<N / 2>::v;
};
template <>
struct Log2<1> {
    static constexpr int v = 0;
};

template <int N>
__device__ __forceinline__ float transpose_reduce(float (&p)[N], int lane) {
    constexpr int LG = Log2<N>::v;
#pragma unroll
    for (int r = 0; r < LG; ++r) {
        const int off = 16 >> r;
        const int n = N >> r;
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const float send = upper ? p[i] : p[i + n / 2];
            const float keep = upper ? p[i + n / 2] : p[i];
            p[i] = keep + __shfl_xor_sync(kFull, send, off);
        }
    }
    float t = p[0];
#pragma unroll
    for (int off = 16 >> LG; off > 0; off >>= 1) t += __shfl_xor_sync(kFull, t, off);
    return t;
}

}  // namespace cgdev
