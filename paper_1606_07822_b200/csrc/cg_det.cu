// cg_det.cu -- K2: the deterministic single-stream training kernel.
//
// Replays the reference's single-worker loop (trainer.hpp:200-245) on one warp:
// lane 0 runs the sequential control flow (id stream, alpha batches, splitmix64
// subsampling draws, 1000-kept-token sentences, shrink_window draws), and the warp
// runs train_center (trainer.hpp:147-175) and the NodeCache (trainer.hpp:75-138).
//
// Bit parity with the reference's default x86 build needs its exact fp32 evaluation:
//  * dot (vec_ops.hpp:14-18) is a sequential chain of separately rounded products and
//    sums. Within one (center, context) pair the path rows are distinct and the
//    context row is fixed, so the L dots are independent: lane j runs the chain for
//    step j (__fmul_rn/__fadd_rn, never contracted to FMA).
//  * h += g*u (pre-update u) and u += g*v (vec_ops.hpp:21-23) run sequentially over the
//    path steps for every component, lanes owning components.
//  * flush adds (work - snap) rounded, exactly like trainer.hpp:116-119.
// No atomics (their float forms flush denormals); built without fast-math.
#include <cstdint>

#include "cg_device.cuh"
#include "cg_kernels.h"

namespace cgk {
namespace {

using cgdev::kFull;

struct DetSmem {
    float* sig;      // [1000]
    float* vbuf;     // [D]
    float* hbuf;     // [D]
    float* gbuf;     // [32]
    float** ubuf;    // [32]
};

__device__ __forceinline__ float det_sigmoid(const DetSmem& sm, float x, int mode, float sc, float scale) {
    if (mode == 0) return cgdev::table_sigmoid(sm.sig, x, scale);
    if (mode == 1) return static_cast<float>(1.0 / (1.0 + exp(-static_cast<double>(x))));
    return sc;
}

// NodeCache::acquire for the slot of one path step; returns the working row.
__device__ __forceinline__ float* det_acquire(const DetModel& m, int32_t slot, const float* shared_row, bool& fresh) {
    float* w = m.cache_work + static_cast<size_t>(slot) * m.dim;
    fresh = m.cache_flag[slot] == 0;
    if (fresh) {
        float* s = m.cache_snap + static_cast<size_t>(slot) * m.dim;
        for (int d = 0; d < m.dim; ++d) w[d] = shared_row[d];
        for (int d = 0; d < m.dim; ++d) s[d] = w[d];
        m.cache_flag[slot] = 1;
    }
    return w;
}

// One train_center call on the whole warp. n_acq is warp-uniform.
__device__ uint64_t det_center_warp(const DetModel& m, const DetSmem& sm, int32_t center, const int32_t* sent,
                                    int64_t len, int64_t cpos, int32_t hw, float alpha, int mode, float sc,
                                    int32_t& n_acq) {
    const int lane = threadIdx.x & 31;
    const int D = m.dim;
    const int64_t p0 = m.path_off[center];
    const int L = static_cast<int>(m.path_off[center + 1] - p0);
    const int64_t lo = cpos >= hw ? cpos - hw : 0;
    const int64_t hi = (len - 1) < (cpos + hw) ? (len - 1) : (cpos + hw);
    uint64_t evals = 0;
    for (int64_t pos = lo; pos <= hi; ++pos) {
        if (pos == cpos) continue;
        float* v = m.syn0 + static_cast<size_t>(sent[pos]) * D;
        for (int d = lane; d < D; d += 32) {
            sm.vbuf[d] = v[d];
            sm.hbuf[d] = 0.0f;
        }
        __syncwarp();
        for (int j0 = 0; j0 < L; j0 += 32) {
            const int j = j0 + lane;
            const int nj = min(32, L - j0);
            float g = 0.0f;
            float* u = nullptr;
            bool fresh = false;
            if (j < L) {
                const int32_t node = m.path_node[p0 + j];
                const int32_t slot = m.slot_of ? m.slot_of[node] : -1;
                float* shared_row = m.syn1 + static_cast<size_t>(node) * D;
                u = slot >= 0 ? det_acquire(m, slot, shared_row, fresh) : shared_row;
                float acc = 0.0f;
                for (int d = 0; d < D; ++d) acc = __fadd_rn(acc, __fmul_rn(sm.vbuf[d], u[d]));
                const float f = det_sigmoid(sm, acc, mode, sc, m.sig_scale);
                g = __fmul_rn(__fsub_rn(__fsub_rn(1.0f, static_cast<float>(m.path_turn[p0 + j])), f), alpha);
            }
            // acquire order == path order == lane order (trainer.hpp:103)
            const unsigned fm = __ballot_sync(kFull, fresh);
            if (fresh) m.acquired[n_acq + __popc(fm & ((1u << lane) - 1u))] = m.slot_of[m.path_node[p0 + j]];
            n_acq += __popc(fm);
            sm.gbuf[lane] = g;
            sm.ubuf[lane] = u;
            __syncwarp();
            for (int d = lane; d < D; d += 32) {
                const float vd = sm.vbuf[d];
                float h = sm.hbuf[d];
                for (int k = 0; k < nj; ++k) {
                    float* ur = sm.ubuf[k];
                    const float gk = sm.gbuf[k];
                    const float uo = ur[d];
                    h = __fadd_rn(h, __fmul_rn(gk, uo));
                    ur[d] = __fadd_rn(uo, __fmul_rn(gk, vd));
                }
                sm.hbuf[d] = h;
            }
            __syncwarp();
        }
        for (int d = lane; d < D; d += 32) v[d] = __fadd_rn(sm.vbuf[d], sm.hbuf[d]);
        __syncwarp();
        evals += static_cast<uint64_t>(L);
    }
    return evals;
}

// NodeCache::flush over the acquire list (trainer.hpp:110-124).
__device__ void det_flush_warp(const DetModel& m, int32_t& n_acq) {
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < n_acq; ++i) {
        const int32_t slot = m.acquired[i];
        float* sh = m.syn1 + static_cast<size_t>(m.hot_nodes[slot]) * m.dim;
        const float* w = m.cache_work + static_cast<size_t>(slot) * m.dim;
        const float* s = m.cache_snap + static_cast<size_t>(slot) * m.dim;
        for (int d = lane; d < m.dim; d += 32) sh[d] = __fadd_rn(sh[d], __fsub_rn(w[d], s[d]));
        __syncwarp();
        if (lane == 0) m.cache_flag[slot] = 0;
    }
    __syncwarp();
    n_acq = 0;
}

__device__ DetSmem carve(int D) {
    extern __shared__ float det_smem[];
    DetSmem sm;
    sm.sig = det_smem;
    sm.vbuf = det_smem + 1024;
    sm.hbuf = sm.vbuf + D;
    sm.gbuf = sm.hbuf + D;
    // pointer array after 32 floats, 8-byte aligned
    size_t off = (1024 + 2 * static_cast<size_t>(D) + 32 + 1) & ~static_cast<size_t>(1);
    sm.ubuf = reinterpret_cast<float**>(det_smem + off);
    return sm;
}

__global__ void det_pass_kernel(DetModel m, DetPass p, DetState* state) {
    __shared__ int32_t sent[cgdev::kSentence];
    const int lane = threadIdx.x & 31;
    DetSmem sm = carve(m.dim);
    for (int i = lane; i < 1000; i += 32) sm.sig[i] = m.sigmoid[i];
    DetState st = *state;  // every lane holds a copy; lane 0's control state is authoritative
    __syncwarp();

    int64_t pos = 0;
    bool live = true;
    while (live) {
        int len = 0;
        if (lane == 0) {
            // trainer.hpp:220-234
            while (len < cgdev::kSentence) {
                if (pos >= p.n_ids) { live = false; break; }
                const int32_t id = p.ids[pos++];
                if (++st.unreported >= cgdev::kAlphaBatch) {
                    st.progress += st.unreported;
                    st.unreported = 0;
                    st.alpha = cgdev::update_alpha(st.progress, p.total_words, p.alpha0);
                }
                if (p.keep) {
                    const float kp = p.keep[id];
                    if (kp < 1.0f && cgdev::unit24(cgdev::seq_next(st.rng)) >= kp) continue;
                }
                sent[len++] = id;
            }
        }
        len = __shfl_sync(kFull, len, 0);
        live = __shfl_sync(kFull, live, 0);
        const float alpha = __shfl_sync(kFull, st.alpha, 0);
        __syncwarp();
        for (int c = 0; c < len; ++c) {
            int32_t hw = 0;
            if (lane == 0) hw = p.window - static_cast<int32_t>(cgdev::seq_next(st.rng) % static_cast<uint64_t>(p.window));
            hw = __shfl_sync(kFull, hw, 0);
            const int lo = c >= hw ? c - hw : 0;
            const int hi = (len - 1) < (c + hw) ? (len - 1) : (c + hw);
            const int32_t center = sent[c];
            st.pairs += static_cast<uint64_t>(hi - lo);
            st.steps += static_cast<uint64_t>(hi - lo) * static_cast<uint64_t>(m.path_off[center + 1] - m.path_off[center]);
            det_center_warp(m, sm, center, sent, len, c, hw, alpha, 0, 0.0f, st.n_acquired);
            ++st.centers;
            if (++st.since_flush >= p.flush_interval) {
                det_flush_warp(m, st.n_acquired);
                st.since_flush = 0;
            }
        }
        __syncwarp();
    }
    det_flush_warp(m, st.n_acquired);  // end of pass (trainer.hpp:242)
    st.since_flush = 0;
    st.words += static_cast<uint64_t>(p.n_ids);
    if (lane == 0) *state = st;
}

__global__ void det_center_kernel(DetModel m, DetCenter c) {
    DetSmem sm = carve(m.dim);
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < 1000; i += 32) sm.sig[i] = m.sigmoid[i];
    int32_t n_acq = *c.n_acquired;
    __syncwarp();
    const uint64_t e = det_center_warp(m, sm, c.center, c.sentence, c.len, c.pos, c.half_window, c.alpha,
                                       c.sigmoid_mode, c.sig_const, n_acq);
    if (lane == 0) {
        *c.n_acquired = n_acq;
        *c.evals = e;
    }
}

// Host-callback sigmoid (train_center with an arbitrary SigmoidFn functor): one pair in
// two phases. Phase 0 acquires the path's hot rows (first touch, trainer.hpp:161-165)
// and writes the L exact sequential dot products; the host maps them through the
// functor; phase 1 applies g = ((1 - turn) - f) * alpha, h += g*u, u += g*v, v += h with
// the same rounding as det_center_warp. Exact: the dots of one pair do not depend on
// the pair's own updates (distinct rows, fixed context row).
__global__ void det_pair_kernel(DetModel m, int32_t center, int32_t context, float alpha, int phase, float* buf,
                                int32_t* n_acquired) {
    DetSmem sm = carve(m.dim);
    const int lane = threadIdx.x & 31;
    const int D = m.dim;
    const int64_t p0 = m.path_off[center];
    const int L = static_cast<int>(m.path_off[center + 1] - p0);
    float* v = m.syn0 + static_cast<size_t>(context) * D;
    int32_t n_acq = *n_acquired;
    for (int d = lane; d < D; d += 32) {
        sm.vbuf[d] = v[d];
        sm.hbuf[d] = 0.0f;
    }
    __syncwarp();
    for (int j0 = 0; j0 < L; j0 += 32) {
        const int j = j0 + lane;
        float* u = nullptr;
        bool fresh = false;
        if (j < L) {
            const int32_t node = m.path_node[p0 + j];
            const int32_t slot = m.slot_of ? m.slot_of[node] : -1;
            float* shared_row = m.syn1 + static_cast<size_t>(node) * D;
            if (phase == 0) {
                u = slot >= 0 ? det_acquire(m, slot, shared_row, fresh) : shared_row;
                float acc = 0.0f;
                for (int d = 0; d < D; ++d) acc = __fadd_rn(acc, __fmul_rn(sm.vbuf[d], u[d]));
                buf[j] = acc;
            } else {
                u = slot >= 0 ? m.cache_work + static_cast<size_t>(slot) * D : shared_row;
            }
        }
        if (phase == 0) {
            const unsigned fm = __ballot_sync(kFull, fresh);
            if (fresh) m.acquired[n_acq + __popc(fm & ((1u << lane) - 1u))] = m.slot_of[m.path_node[p0 + j]];
            n_acq += __popc(fm);
            continue;
        }
        const float g = j < L ? __fmul_rn(__fsub_rn(__fsub_rn(1.0f, static_cast<float>(m.path_turn[p0 + j])), buf[j]),
                                          alpha)
                              : 0.0f;
        sm.gbuf[lane] = g;
        sm.ubuf[lane] = u;
        __syncwarp();
        const int nj = min(32, L - j0);
        for (int d = lane; d < D; d += 32) {
            const float vd = sm.vbuf[d];
            float h = sm.hbuf[d];
            for (int k = 0; k < nj; ++k) {
                float* ur = sm.ubuf[k];
                const float uo = ur[d];
                h = __fadd_rn(h, __fmul_rn(sm.gbuf[k], uo));
                ur[d] = __fadd_rn(uo, __fmul_rn(sm.gbuf[k], vd));
            }
            sm.hbuf[d] = h;
        }
        __syncwarp();
    }
    if (phase == 1)
        for (int d = lane; d < D; d += 32) v[d] = __fadd_rn(sm.vbuf[d], sm.hbuf[d]);
    if (lane == 0) *n_acquired = n_acq;
}

// Flush driven by flags (order-free: every acquired slot touches a distinct row).
__global__ void det_flush_flags_kernel(DetModel m) {
    const int lane = threadIdx.x & 31;
    for (int slot = 0; slot < m.hot_count; ++slot) {
        if (!m.cache_flag[slot]) continue;
        float* sh = m.syn1 + static_cast<size_t>(m.hot_nodes[slot]) * m.dim;
        const float* w = m.cache_work + static_cast<size_t>(slot) * m.dim;
        const float* s = m.cache_snap + static_cast<size_t>(slot) * m.dim;
        for (int d = lane; d < m.dim; d += 32) sh[d] = __fadd_rn(sh[d], __fsub_rn(w[d], s[d]));
        __syncwarp();
        if (lane == 0) m.cache_flag[slot] = 0;
        __syncwarp();
    }
}

size_t det_smem_bytes(int D) { return (1024 + 2 * static_cast<size_t>(D) + 32 + 2) * 4 + 32 * sizeof(float*) + 16; }

}  // namespace

void launch_det_pass(const DetModel& m, const DetPass& p, DetState* state, cudaStream_t s) {
    const size_t smem = det_smem_bytes(m.dim);
    cudaFuncSetAttribute(det_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));  // static + dynamic may pass 48 KB
    det_pass_kernel<<<1, 32, smem, s>>>(m, p, state);
}

void launch_det_center(const DetModel& m, const DetCenter& c, cudaStream_t s) {
    const size_t smem = det_smem_bytes(m.dim);
    cudaFuncSetAttribute(det_center_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));  // static + dynamic may pass 48 KB
    det_center_kernel<<<1, 32, smem, s>>>(m, c);
}

void launch_det_flush_flags(const DetModel& m, cudaStream_t s) { det_flush_flags_kernel<<<1, 32, 0, s>>>(m); }

void launch_det_pair(const DetModel& m, int32_t center, int32_t context, float alpha, int phase, float* buf,
                     int32_t* n_acquired, cudaStream_t s) {
    const size_t smem = det_smem_bytes(m.dim);
    cudaFuncSetAttribute(det_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));  // static + dynamic may pass 48 KB
    det_pair_kernel<<<1, 32, smem, s>>>(m, center, context, alpha, phase, buf, n_acquired);
}

}  // namespace cgk
