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
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// a + s*b
__device__ __forceinline__ float4 axpy4(float s, float4 b, float4 a) {
    return make_float4(fmaf(s, b.x, a.x), fmaf(s, b.y, a.y), fmaf(s, b.z, a.z), fmaf(s, b.w, a.w));
}
__device__ __forceinline__ float4 scale4(float s, float4 b) {
    return make_float4(s * b.x, s * b.y, s * b.z, s * b.w);
}
__device__ __forceinline__ float dot4(float4 a, float4 b, float acc) {
    acc = fmaf(a.x, b.x, acc);
    acc = fmaf(a.y, b.y, acc);
    acc = fmaf(a.z, b.z, acc);
    return fmaf(a.w, b.w, acc);
}
__device__ __forceinline__ bool nonzero4(float4 a) { return a.x != 0.f || a.y != 0.f || a.z != 0.f || a.w != 0.f; }

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
