// mpo.cu -- sm_100a kernels and the C ABI (include/mpo.h) of the residual-compensated 16-bit
// optimizer step of arXiv 2309.12381.  Citation keys as in include/mpo.h.
//
// Kernel design.  The step is an elementwise stream (no contraction, so
// no tensor cores): per element Adam moves 26 B (value 2 + resid 2 + grad 2 + m 4 + v 4 read;
// value, resid, m, v written), SGD-momentum 18 B.  It is HBM-bound on B200, so the kernels
//   * process a "unit" of 8 elements per thread with 128-bit loads/stores of every stream
//     (one uint4 of values, one of residuals, one of 16-bit grads, two float4 of m and of v);
//   * issue all loads of kUnroll units before any arithmetic (memory-level parallelism);
//   * walk a multi-tensor table ("one only stream of values") passed BY VALUE as a
//     __grid_constant__ kernel parameter (no table upload, no host sync), split into tiles of
//     kTileEl elements; a persistent grid of (#SM x resident CTAs) strides over the tiles in
//     order, each CTA advancing a uniform cursor through the table;
//   * handle the ragged tail of a tensor (n % 8) element by element;
//   * use warp shuffles only in the global-norm reduction (clipping).
#include "mpo.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "mpo_device.cuh"

#define MPO_API extern "C" __attribute__((visibility("default")))

namespace mpo {

#ifndef MPO_CW
#define MPO_CW 16            // consumer warps per CTA of the TMA kernel (A/B knob)
#endif
#ifndef MPO_CTAS_PER_SM
#define MPO_CTAS_PER_SM 1    // resident TMA CTAs per SM (A/B knob)
#endif
constexpr int kThreads = 256;
constexpr int kUnitEl = 8;                          // elements per unit (128-bit of 16-bit data)
constexpr int64_t kTileEl = int64_t(MPO_CW) * 32 * kUnitEl;   // 4096 elements: one unit per consumer thread
constexpr int kUnroll = int(kTileEl / (kThreads * kUnitEl));  // LSU kernel: units per thread per tile
static_assert(kUnroll >= 1, "tile smaller than one LSU pass");
constexpr int kNormBlocksMax = 2048;                // partial sums of the norm pre-pass

struct KT {                 // one table entry inside the kernel parameter block
    void* value;
    int16_t* resid;
    const void* grad;
    float* m;
    float* v;
    int64_t n;
    int32_t hp;
    int32_t tile0;          // first tile of this tensor in the launch's tile space
};

template <int MAXT>
struct Table {
    KT t[MAXT];
    int32_t nt;
    int32_t ntiles;
};

template <class K>
struct HP {
    K g[MPO_MAX_HP_GROUPS];
};

// ------------------------------------------------------------------------------------------
// Vector memory helpers: 128-bit streaming (evict-first) loads and stores.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldv(const void* p) { return __ldcs(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ float4 ldf(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void stv(void* p, uint4 x) { __stcs(reinterpret_cast<uint4*>(p), x); }
__device__ __forceinline__ void stf(float* p, float4 x) { __stcs(reinterpret_cast<float4*>(p), x); }

// 8 gradient values of a unit as fp32.
template <int G>
struct GradUnit {
    uint4 a, b;   // 16-bit grads use a only; fp32 grads use a and b (8 floats)
};

template <int G>
__device__ __forceinline__ GradUnit<G> ld_grad(const void* grad, int64_t e) {
    GradUnit<G> u;
    if constexpr (G == kFP32) {
        const float* g = static_cast<const float*>(grad) + e;
        u.a = __ldcs(reinterpret_cast<const uint4*>(g));
        u.b = __ldcs(reinterpret_cast<const uint4*>(g + 4));
    } else {
        u.a = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(grad) + e));
    }
    return u;
}

template <int G>
__device__ __forceinline__ float grad_at(const GradUnit<G>& u, int k) {
    if constexpr (G == kFP32) {
        const uint32_t* w = k < 4 ? &u.a.x : &u.b.x;
        return __uint_as_float(w[k & 3]);
    } else {
        const uint32_t* w = &u.a.x;
        uint32_t x = w[k >> 1];
        return grad_f32_16<G>((k & 1) ? hi16(x) : lo16(x));
    }
}

template <int G>
__device__ __forceinline__ float grad_scalar(const void* grad, int64_t i) {
    if constexpr (G == kFP32) return static_cast<const float*>(grad)[i];
    else return grad_f32_16<G>(static_cast<const uint16_t*>(grad)[i]);
}

// ------------------------------------------------------------------------------------------
// G1 / G2: split and reconstruct.
// ------------------------------------------------------------------------------------------
template <int F>
__global__ void __launch_bounds__(kThreads) split_kernel(const float* __restrict__ w, uint16_t* __restrict__ value,
                                                         int16_t* __restrict__ resid, int64_t n) {
    const int64_t nunits = n / kUnitEl;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        const int64_t e = u * kUnitEl;
        float4 x0 = ldf(w + e), x1 = ldf(w + e + 4);
        uint4 hv, rv;
        split2<F>(x0.x, x0.y, hv.x, rv.x);
        split2<F>(x0.z, x0.w, hv.y, rv.y);
        split2<F>(x1.x, x1.y, hv.z, rv.z);
        split2<F>(x1.z, x1.w, hv.w, rv.w);
        stv(value + e, hv);
        stv(resid + e, rv);
    }
    // ragged tail (n % 8 elements), one thread per element
    const int64_t t = nunits * kUnitEl + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && t < nunits * kUnitEl + kUnitEl) {
        uint32_t hv, rv;
        split2<F>(w[t], 0.0f, hv, rv);
        value[t] = static_cast<uint16_t>(hv & 0xFFFFu);
        resid[t] = static_cast<int16_t>(rv & 0xFFFFu);
    }
}

template <int F>
__global__ void __launch_bounds__(kThreads) reconstruct_kernel(const uint16_t* __restrict__ value,
                                                               const int16_t* __restrict__ resid,
                                                               float* __restrict__ w, int64_t n) {
    const int64_t nunits = n / kUnitEl;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        const int64_t e = u * kUnitEl;
        uint4 hv = ldv(value + e), rv = ldv(resid + e);
        const uint32_t* h = &hv.x;
        const uint32_t* r = &rv.x;
        float o[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            o[2 * j] = reconstruct1<F>(lo16(h[j]), slo16(r[j]));
            o[2 * j + 1] = reconstruct1<F>(hi16(h[j]), shi16(r[j]));
        }
        stf(w + e, make_float4(o[0], o[1], o[2], o[3]));
        stf(w + e + 4, make_float4(o[4], o[5], o[6], o[7]));
    }
    const int64_t t = nunits * kUnitEl + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && t < nunits * kUnitEl + kUnitEl) {
        w[t] = reconstruct1<F>(value[t], resid[t]);
    }
}

// ------------------------------------------------------------------------------------------
// G5: global-norm pre-pass (clipping, R9): per-block fp64 partial sums of (f32(g)*gs)^2, then a
// single-block fixed-order final sum.  Deterministic for a given grid size.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double s, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xFFFFFFFFu, s, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = s;
    __syncthreads();
    s = 0.0;
    if (wid == 0) {
        s = lane < (int(blockDim.x) >> 5) ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xFFFFFFFFu, s, o);
    }
    __syncthreads();
    return s;   // valid in thread 0
}

// The clip pre-pass reads 2 B/param and is issue-bound (widen, scale, F2F.F64, DFMA per element),
// so it uses its own, larger tiles (kSumsqTileEl = 16 units per thread) to amortise the per-tile
// bookkeeping, issues all 16 loads of a tile before any arithmetic, skips the scale multiply when
// it is exactly 1, and keeps 8 independent fp64 accumulators per thread (a single accumulator
// would serialise every DFMA).  Every square of a float is exact in fp64.
constexpr int kSumsqUPT = 16;
constexpr int64_t kSumsqTileEl = int64_t(kThreads) * kSumsqUPT * kUnitEl;   // 32768 elements

template <int MAXT, int G>
__global__ void __launch_bounds__(kThreads) sumsq_kernel(const __grid_constant__ Table<MAXT> tab,
                                                         const __grid_constant__ HP<float> gsc,
                                                         double* __restrict__ partial) {
    __shared__ double sh[32];
    double acc8[kUnitEl];
#pragma unroll
    for (int k = 0; k < kUnitEl; ++k) acc8[k] = 0.0;
    int cur = 0;
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        const float gs = gsc.g[T.hp];
        const int64_t n = T.n;
        const int64_t base = int64_t(tile - T.tile0) * kSumsqTileEl;
        const char* gp = static_cast<const char*>(T.grad);
        if (base + kSumsqTileEl <= n) {
            GradUnit<G> gu[kSumsqUPT];
#pragma unroll
            for (int j = 0; j < kSumsqUPT; ++j)
                gu[j] = ld_grad<G>(T.grad, base + (int64_t(j) * kThreads + threadIdx.x) * kUnitEl);
            if (gs == 1.0f) {
#pragma unroll
                for (int j = 0; j < kSumsqUPT; ++j)
#pragma unroll
                    for (int k = 0; k < kUnitEl; ++k) {
                        const double g = double(grad_at<G>(gu[j], k));
                        acc8[k] = fma(g, g, acc8[k]);
                    }
            } else {
#pragma unroll
                for (int j = 0; j < kSumsqUPT; ++j)
#pragma unroll
                    for (int k = 0; k < kUnitEl; ++k) {
                        const double g = double(grad_at<G>(gu[j], k) * gs);
                        acc8[k] = fma(g, g, acc8[k]);
                    }
            }
        } else {   // partial tile: unit by unit, ragged tail element by element
            (void)gp;
            for (int j = 0; j < kSumsqUPT; ++j) {
                const int64_t e = base + (int64_t(j) * kThreads + threadIdx.x) * kUnitEl;
                if (e + kUnitEl <= n) {
                    const GradUnit<G> u = ld_grad<G>(T.grad, e);
#pragma unroll
                    for (int k = 0; k < kUnitEl; ++k) {
                        const double g = double(grad_at<G>(u, k) * gs);
                        acc8[k] = fma(g, g, acc8[k]);
                    }
                } else if (e < n) {
                    for (int64_t i = e; i < n; ++i) {
                        const double g = double(grad_scalar<G>(T.grad, i) * gs);
                        acc8[0] = fma(g, g, acc8[0]);
                    }
                }
            }
        }
    }
    double acc = ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// Sums nparts partials (fixed order) into out[0].
__global__ void __launch_bounds__(kThreads) sumsq_final_kernel(const double* __restrict__ partial, int nparts,
                                                               double* __restrict__ out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += partial[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) out[0] = acc;
}

// Clip coefficient from the global sum of squares: min(1, max_norm / (sqrt(S) + 1e-6)),
// rounded once to float; a NaN quotient propagates (R9).
__device__ __forceinline__ float clip_coef(const double* sumsq, double max_norm) {
    const double q = max_norm / (sqrt(sumsq[0]) + 1e-6);
    return q > 1.0 ? 1.0f : float(q);
}

// ------------------------------------------------------------------------------------------
// G3 / G4: multi-tensor residual-compensated step.
// ------------------------------------------------------------------------------------------
template <int F, int G>
struct AdamOp {
    using K = AdamK;
    static constexpr bool kHasV = true;
    __device__ __forceinline__ static bool reads_m(const K&) { return true; }
    __device__ __forceinline__ static bool writes_m(const K&) { return true; }
    __device__ __forceinline__ static float apply(float w, float g, float& m, float& v, const K& c) {
        return adam_update(w, g, m, v, c);
    }
    __device__ __forceinline__ static bool unit_fast(float (&w)[8], const float (&g)[8], float (&m)[8], float (&v)[8],
                                                     const K& c) {
        return adam_unit_fast(w, g, m, v, c);
    }
};

template <int F, int G>
struct SgdOp {
    using K = SgdK;
    static constexpr bool kHasV = false;
    // the momentum buffer is read only after the first step (torch clones the grad then)
    __device__ __forceinline__ static bool reads_m(const K& c) { return c.has_mom && !c.first; }
    __device__ __forceinline__ static bool writes_m(const K& c) { return c.has_mom; }
    __device__ __forceinline__ static float apply(float w, float g, float& m, float&, const K& c) {
        return sgd_update(w, g, m, c);
    }
    __device__ __forceinline__ static bool unit_fast(float (&w)[8], const float (&g)[8], float (&m)[8], float (&v)[8],
                                                     const K& c) {
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = apply(w[k], g[k], m[k], v[k], c);
        return true;
    }
};

// One unit (8 consecutive elements): reconstruct -> update -> re-split, registers in and out.
template <int F, int G, class Op, bool CLIP>
__device__ __forceinline__ void process_unit(const uint4& hv, const uint4& rv, const GradUnit<G>& gu, float (&mm)[8],
                                             float (&vv)[8], const typename Op::K& c, float coef, uint4& ho,
                                             uint4& ro) {
    const uint32_t* h = &hv.x;
    const uint32_t* r = &rv.x;
    float w[8], g[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        g[k] = grad_at<G>(gu, k) * c.gs;
        if constexpr (CLIP) g[k] = g[k] * coef;
    }
    const uint32_t special = nonfinite_pair<F>(h[0]) | nonfinite_pair<F>(h[1]) | nonfinite_pair<F>(h[2]) |
                             nonfinite_pair<F>(h[3]);
    bool done = false;
    if (__builtin_expect(special == 0u, 1)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) reconstruct_pair_finite<F>(h[q], r[q], w[2 * q], w[2 * q + 1]);
        done = Op::unit_fast(w, g, mm, vv, c);
    }
    if (__builtin_expect(!done, 0)) {
        // non-finite values, or an operand outside the fast sqrt/div windows: the general path
        // (full IEEE operators; mm/vv are untouched by a failed fast attempt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            w[2 * q] = reconstruct1<F>(lo16(h[q]), slo16(r[q]));
            w[2 * q + 1] = reconstruct1<F>(hi16(h[q]), shi16(r[q]));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = Op::apply(w[k], g[k], mm[k], vv[k], c);
    }
    uint32_t hq[4], rq[4];
    split8<F>(w, hq, rq);
    ho = make_uint4(hq[0], hq[1], hq[2], hq[3]);
    ro = make_uint4(rq[0], rq[1], rq[2], rq[3]);
}

// Ragged tail of one tensor (n % 8 elements): element by element from global memory.
template <int F, int G, class Op, bool CLIP>
__device__ __noinline__ void process_tail(const KT T, int64_t lo, int64_t hi, const typename Op::K c, float coef) {
    uint16_t* val = static_cast<uint16_t*>(T.value);
    const bool need_m = Op::reads_m(c), has_m = Op::writes_m(c);
    for (int64_t i = lo; i < hi; ++i) {
        float g = grad_scalar<G>(T.grad, i) * c.gs;
        if constexpr (CLIP) g = g * coef;
        float w = reconstruct1<F>(val[i], T.resid[i]);
        float mi = need_m ? T.m[i] : 0.0f;
        float vi = 0.0f;
        if constexpr (Op::kHasV) vi = T.v[i];
        w = Op::apply(w, g, mi, vi, c);
        uint32_t ho, ro;
        split2<F>(w, 0.0f, ho, ro);
        val[i] = static_cast<uint16_t>(ho & 0xFFFFu);
        T.resid[i] = static_cast<int16_t>(ro & 0xFFFFu);
        if (has_m) T.m[i] = mi;
        if constexpr (Op::kHasV) T.v[i] = vi;
    }
}

template <class Op>
__device__ __forceinline__ void store_unit(const KT& T, int64_t e, const uint4& ho, const uint4& ro, const float (&mm)[8],
                                           const float (&vv)[8], bool has_m) {
    stv(static_cast<uint16_t*>(T.value) + e, ho);
    stv(T.resid + e, ro);
    if (has_m) {
        stf(T.m + e, make_float4(mm[0], mm[1], mm[2], mm[3]));
        stf(T.m + e + 4, make_float4(mm[4], mm[5], mm[6], mm[7]));
    }
    if constexpr (Op::kHasV) {
        stf(T.v + e, make_float4(vv[0], vv[1], vv[2], vv[3]));
        stf(T.v + e + 4, make_float4(vv[4], vv[5], vv[6], vv[7]));
    }
}

// ---- variant A ("lsu"): every thread loads its own units with 128-bit LDG, computes, stores ----
template <int MAXT, int F, int G, class Op, bool CLIP>
__global__ void __launch_bounds__(kThreads) step_kernel(const __grid_constant__ Table<MAXT> tab,
                                                        const __grid_constant__ HP<typename Op::K> hp,
                                                        const double* __restrict__ sumsq, double max_norm) {
    using K = typename Op::K;
    float coef = 1.0f;
    if constexpr (CLIP) coef = clip_coef(sumsq, max_norm);
    int cur = 0;
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        const K c = hp.g[T.hp];
        const bool need_m = Op::reads_m(c);
        const bool has_m = Op::writes_m(c);
        const int64_t base = int64_t(tile - T.tile0) * kTileEl;
        const int64_t n = T.n;

        uint4 hv[kUnroll], rv[kUnroll];
        GradUnit<G> gu[kUnroll];
        float4 m0[kUnroll], m1[kUnroll], v0[kUnroll], v1[kUnroll];
        // ---- load phase: every 128-bit load of kUnroll units in flight before any math ----
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const int64_t e = base + (int64_t(j) * kThreads + threadIdx.x) * kUnitEl;
            if (e + kUnitEl <= n) {
                hv[j] = ldv(static_cast<uint16_t*>(T.value) + e);
                rv[j] = ldv(T.resid + e);
                gu[j] = ld_grad<G>(T.grad, e);
                if (need_m) {
                    m0[j] = ldf(T.m + e);
                    m1[j] = ldf(T.m + e + 4);
                } else {
                    m0[j] = m1[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                if constexpr (Op::kHasV) {
                    v0[j] = ldf(T.v + e);
                    v1[j] = ldf(T.v + e + 4);
                } else {
                    v0[j] = v1[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
        // ---- compute + store phase ----
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const int64_t e = base + (int64_t(j) * kThreads + threadIdx.x) * kUnitEl;
            if (e + kUnitEl <= n) {
                float mm[8] = {m0[j].x, m0[j].y, m0[j].z, m0[j].w, m1[j].x, m1[j].y, m1[j].z, m1[j].w};
                float vv[8] = {v0[j].x, v0[j].y, v0[j].z, v0[j].w, v1[j].x, v1[j].y, v1[j].z, v1[j].w};
                uint4 ho, ro;
                process_unit<F, G, Op, CLIP>(hv[j], rv[j], gu[j], mm, vv, c, coef, ho, ro);
                store_unit<Op>(T, e, ho, ro, mm, vv, has_m);
            } else if (e < n) {
                process_tail<F, G, Op, CLIP>(T, e, n, c, coef);
            }
        }
    }
}

// ---- variant B ("tma", default): warp-specialised bulk-copy pipeline ----------------------
// One producer warp streams each tile's value / residual / grad / m / v from HBM into a ring of
// shared-memory stages with 1-D TMA bulk copies (cp.async.bulk, mbarrier complete_tx, L2
// evict-first); kCW consumer warps read the stage from shared memory, compute, and store the
// results straight to HBM with 128-bit stores, then release the stage.  Loads are therefore
// issued independently of the arithmetic, several tiles ahead.
constexpr int kCW = MPO_CW;                              // consumer warps per CTA
constexpr int kTmaThreads = (kCW + 1) * 32;              // + 1 producer warp
static_assert(kCW * 32 * kUnitEl == kTileEl, "one unit per consumer thread per tile");
constexpr int kMaxStages = 8;
constexpr int kBarBytes = 2 * kMaxStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Orders this thread's generic-proxy shared-memory reads of a stage before the async-proxy (bulk
// copy) writes that will refill it: without it the producer's next cp.async.bulk can land in the
// stage under a still-pending LDS (seen as wrong value/residual words).
__device__ __forceinline__ void fence_proxy_async_smem() {
#ifndef MPO_NO_PROXY_FENCE   // diagnostic A/B knob only: the fence is required for correctness
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D bulk copy global -> shared, completing `bytes` of transaction on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <int G>
struct GradBytes {
    static constexpr int v = G == kFP32 ? 4 : 2;
};

// bytes of one stage: value 2 + resid 2 + grad gb + m 4 [+ v 4] per element
template <int G, bool HAS_V>
__host__ __device__ constexpr int stage_bytes() {
    return int(kTileEl) * (2 + 2 + GradBytes<G>::v + 4 + (HAS_V ? 4 : 0));
}

template <int MAXT, int F, int G, class Op, bool CLIP>
__global__ void __launch_bounds__(kTmaThreads, MPO_CTAS_PER_SM) step_tma_kernel(const __grid_constant__ Table<MAXT> tab,
                                                                  const __grid_constant__ HP<typename Op::K> hp,
                                                                  const double* __restrict__ sumsq, double max_norm,
                                                                  int stages) {
    using K = typename Op::K;
    constexpr int GB = GradBytes<G>::v;
    constexpr int64_t TE = kTileEl;
    // stage layout: [value TE*2 | resid TE*2 | grad TE*GB | m TE*4 | v TE*4]
    constexpr int OFF_R = int(TE) * 2, OFF_G = int(TE) * 4, OFF_M = int(TE) * (4 + GB), OFF_V = int(TE) * (8 + GB);
    constexpr int SB = stage_bytes<G, Op::kHasV>();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    unsigned char* ring = smem + kBarBytes;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kCW) {
        // ---------------- producer ----------------
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int cur = 0, it = 0;
            for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x, ++it) {
                const int s = it % stages;
                const uint32_t round = uint32_t(it / stages);
                mbar_wait(&empty[s], (round & 1u) ^ 1u);
                while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
                const KT& T = tab.t[cur];
                const K c = hp.g[T.hp];
                const int64_t base = int64_t(tile - T.tile0) * TE;
                const int64_t nvalid = T.n - base < TE ? T.n - base : TE;
                const uint32_t nvec = uint32_t(nvalid) & ~uint32_t(kUnitEl - 1);
                const bool need_m = Op::reads_m(c);
                uint32_t bytes = nvec * (4u + GB);
                if (need_m) bytes += nvec * 4u;
                if constexpr (Op::kHasV) bytes += nvec * 4u;
                unsigned char* st = ring + size_t(s) * SB;
                mbar_arrive_expect_tx(&full[s], bytes);
                if (nvec) {
                    bulk_g2s(st, static_cast<const uint16_t*>(T.value) + base, nvec * 2u, &full[s], pol);
                    bulk_g2s(st + OFF_R, T.resid + base, nvec * 2u, &full[s], pol);
                    bulk_g2s(st + OFF_G, static_cast<const unsigned char*>(T.grad) + base * GB, nvec * GB, &full[s], pol);
                    if (need_m) bulk_g2s(st + OFF_M, T.m + base, nvec * 4u, &full[s], pol);
                    if constexpr (Op::kHasV) bulk_g2s(st + OFF_V, T.v + base, nvec * 4u, &full[s], pol);
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    float coef = 1.0f;
    if constexpr (CLIP) coef = clip_coef(sumsq, max_norm);
    const int ct = threadIdx.x;   // 0 .. kCW*32-1, one unit per tile
    int cur = 0, it = 0;
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x, ++it) {
        const int s = it % stages;
        const uint32_t round = uint32_t(it / stages);
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        const K c = hp.g[T.hp];
        const int64_t base = int64_t(tile - T.tile0) * TE;
        const int64_t nvalid = T.n - base < TE ? T.n - base : TE;
        const int64_t nvec = nvalid & ~int64_t(kUnitEl - 1);
        const int64_t el = int64_t(ct) * kUnitEl;
        mbar_wait(&full[s], round & 1u);
        const bool full_unit = el + kUnitEl <= nvec;
        uint4 hv = make_uint4(0u, 0u, 0u, 0u), rv = hv;
        GradUnit<G> gu;
        gu.a = gu.b = hv;
        float mm[8], vv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mm[k] = vv[k] = 0.0f;
        if (full_unit) {
            const unsigned char* st = ring + size_t(s) * SB;
            hv = *reinterpret_cast<const uint4*>(st + el * 2);
            rv = *reinterpret_cast<const uint4*>(st + OFF_R + el * 2);
            if constexpr (G == kFP32) {
                gu.a = *reinterpret_cast<const uint4*>(st + OFF_G + el * 4);
                gu.b = *reinterpret_cast<const uint4*>(st + OFF_G + el * 4 + 16);
            } else {
                gu.a = *reinterpret_cast<const uint4*>(st + OFF_G + el * 2);
            }
            if (Op::reads_m(c)) {
                const float4 a = *reinterpret_cast<const float4*>(st + OFF_M + el * 4);
                const float4 b = *reinterpret_cast<const float4*>(st + OFF_M + el * 4 + 16);
                mm[0] = a.x; mm[1] = a.y; mm[2] = a.z; mm[3] = a.w; mm[4] = b.x; mm[5] = b.y; mm[6] = b.z; mm[7] = b.w;
            }
            if constexpr (Op::kHasV) {
                const float4 a = *reinterpret_cast<const float4*>(st + OFF_V + el * 4);
                const float4 b = *reinterpret_cast<const float4*>(st + OFF_V + el * 4 + 16);
                vv[0] = a.x; vv[1] = a.y; vv[2] = a.z; vv[3] = a.w; vv[4] = b.x; vv[5] = b.y; vv[6] = b.z; vv[7] = b.w;
            }
        }
#ifdef MPO_RELEASE_EARLY
        // the warp's share of the stage now sits in registers: release the stage to the producer
        // before the arithmetic, so the next bulk copies overlap this tile's compute (the proxy
        // fence orders the reads before the refill).
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#endif
        uint4 ho, ro;
#ifdef MPO_TRIVIAL_MATH
        // roofline experiment only: same bytes moved, trivial arithmetic (not a product path)
        if (full_unit) {
            ho = make_uint4(hv.x ^ gu.a.x, hv.y ^ gu.a.y, hv.z ^ gu.a.z, hv.w ^ gu.a.w);
            ro = make_uint4(rv.x + 1u, rv.y + 1u, rv.z + 1u, rv.w + 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k) { mm[k] = mm[k] * 0.5f; vv[k] = vv[k] * 0.25f; }
        }
#else
        if (full_unit) process_unit<F, G, Op, CLIP>(hv, rv, gu, mm, vv, c, coef, ho, ro);
#endif
#ifndef MPO_RELEASE_EARLY
        // release after the arithmetic has consumed the registers (the proxy fence then waits on
        // nothing still pending from this stage)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#endif
        if (full_unit) {
            store_unit<Op>(T, base + el, ho, ro, mm, vv, Op::writes_m(c));
        } else if (el == nvec && nvec < nvalid) {
            process_tail<F, G, Op, CLIP>(T, base + nvec, base + nvalid, c, coef);
        }
    }
}

// ---- G5 on the bulk-copy pipeline: the clip pre-pass reads only the 16-bit grads (2 B/param),
// so it needs many bytes in flight per SM; a producer warp streams tiles of grads into 8 stages
// while 16 consumer warps square and accumulate (8 independent fp64 accumulators per thread).
template <int MAXT, int G>
__global__ void __launch_bounds__(kTmaThreads, 1) sumsq_tma_kernel(const __grid_constant__ Table<MAXT> tab,
                                                                   const __grid_constant__ HP<float> gsc,
                                                                   double* __restrict__ partial, int stages) {
    constexpr int GB = GradBytes<G>::v;
    constexpr int64_t TE = kTileEl;
    constexpr int SB = int(TE) * GB;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double red[kCW];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    unsigned char* ring = smem + kBarBytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kCW) {
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int cur = 0, it = 0;
            for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x, ++it) {
                const int s = it % stages;
                mbar_wait(&empty[s], (uint32_t(it / stages) & 1u) ^ 1u);
                while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
                const KT& T = tab.t[cur];
                const int64_t base = int64_t(tile - T.tile0) * TE;
                const int64_t nvalid = T.n - base < TE ? T.n - base : TE;
                const uint32_t nvec = uint32_t(nvalid) & ~uint32_t(kUnitEl - 1);
                mbar_arrive_expect_tx(&full[s], nvec * GB);
                if (nvec)
                    bulk_g2s(ring + size_t(s) * SB, static_cast<const unsigned char*>(T.grad) + base * GB, nvec * GB,
                             &full[s], pol);
            }
        }
        return;
    }
    double acc8[kUnitEl];
#pragma unroll
    for (int k = 0; k < kUnitEl; ++k) acc8[k] = 0.0;
    const int64_t el = int64_t(threadIdx.x) * kUnitEl;
    int cur = 0, it = 0;
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x, ++it) {
        const int s = it % stages;
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        const float gs = gsc.g[T.hp];
        const int64_t base = int64_t(tile - T.tile0) * TE;
        const int64_t nvalid = T.n - base < TE ? T.n - base : TE;
        const int64_t nvec = nvalid & ~int64_t(kUnitEl - 1);
        mbar_wait(&full[s], uint32_t(it / stages) & 1u);
        const bool full_unit = el + kUnitEl <= nvec;
        GradUnit<G> gu;
        gu.a = gu.b = make_uint4(0u, 0u, 0u, 0u);
        if (full_unit) {
            const unsigned char* st = ring + size_t(s) * SB;
            gu.a = *reinterpret_cast<const uint4*>(st + el * GB);
            if constexpr (G == kFP32) gu.b = *reinterpret_cast<const uint4*>(st + el * GB + 16);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (full_unit) {
#pragma unroll
            for (int k = 0; k < kUnitEl; ++k) {
                const double g = double(grad_at<G>(gu, k) * gs);
                acc8[k] = fma(g, g, acc8[k]);
            }
        } else if (el == nvec && nvec < nvalid) {
            for (int64_t i = base + nvec; i < base + nvalid; ++i) {
                const double g = double(grad_scalar<G>(T.grad, i) * gs);
                acc8[0] = fma(g, g, acc8[0]);
            }
        }
    }
    double acc = ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0) red[warp] = acc;
    asm volatile("bar.sync 1, %0;" ::"r"(kCW * 32) : "memory");   // consumer warps only
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kCW; ++w) t += red[w];   // fixed order
        partial[blockIdx.x] = t;
    }
}

// ------------------------------------------------------------------------------------------
// Self-check of the branch-free fast sqrt / division against the IEEE operators.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void __launch_bounds__(kThreads) selfcheck_sqrt_kernel(unsigned long long* counts) {
    unsigned long long bad_cnt = 0, fast_cnt = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < (1ull << 32); u += stride) {
        const float x = __uint_as_float(uint32_t(u));
        uint32_t bad = 0;
        const float f = sqrt_rn_fast(x, bad);
        if (!bad) {
            ++fast_cnt;
            if (__float_as_uint(f) != __float_as_uint(sqrtf(x))) ++bad_cnt;
        }
    }
    atomicAdd(&counts[0], bad_cnt);
    atomicAdd(&counts[2], fast_cnt);
}

__global__ void __launch_bounds__(kThreads) selfcheck_div_kernel(int64_t pairs, uint64_t seed, unsigned long long* counts) {
    unsigned long long bad_cnt = 0, fast_cnt = 0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < pairs; i += stride) {
        const uint64_t r = splitmix64(seed ^ splitmix64(uint64_t(i)));
        uint32_t ab = uint32_t(r), bb = uint32_t(r >> 32);
        if (i & 1) {   // half the pairs: exponents inside the accepted window [67, 187]
            ab = (ab & 0x807FFFFFu) | ((67u + (ab >> 23) % 121u) << 23);
            bb = (bb & 0x807FFFFFu) | ((67u + (bb >> 23) % 121u) << 23);
        }
        if ((i & 15) == 2) ab &= 0x80000000u;   // signed zero dividends
        const float a = __uint_as_float(ab), b = __uint_as_float(bb);
        uint32_t bad = 0;
        const float f = div_rn_fast(a, b, bad);
        if (!bad) {
            ++fast_cnt;
            if (__float_as_uint(f) != __float_as_uint(a / b)) ++bad_cnt;
        }
    }
    atomicAdd(&counts[1], bad_cnt);
    atomicAdd(&counts[3], fast_cnt);
}

// ------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------
thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

mpo_status fail(mpo_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

mpo_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MPO_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return MPO_OK;
}

int num_sms() {
    static int sms = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return 148;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
        return v;
    }();
    return sms;
}

template <class Kern>
int resident_blocks(Kern k) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kThreads, 0) != cudaSuccess || b < 1) {
        cudaGetLastError();
        b = 1;
    }
    return b;
}

int64_t grid_for(int64_t work_items, int per_sm) {
    int64_t cap = int64_t(num_sms()) * per_sm;
    int64_t g = work_items < cap ? work_items : cap;
    return g < 1 ? 1 : g;
}

bool finite(double x) { return std::isfinite(x); }

AdamK derive_adam(const mpo_adam_hp& h) {
    AdamK c;
    const double t = double(h.step);
    c.gs = float(h.grad_scale);
    c.b1c = float(1.0 - h.beta1);
    c.omb1c = 1.0f - c.b1c;
    c.b2 = float(h.beta2);
    c.b2c = float(1.0 - h.beta2);
    c.bc2s = float(std::sqrt(1.0 - std::pow(h.beta2, t)));
    c.ss = float(h.lr / (1.0 - std::pow(h.beta1, t)));
    c.eps = float(h.eps);
    c.dec = float(1.0 - h.lr * h.weight_decay);
    c.wd = float(h.weight_decay);
    c.mode = h.adamw ? 1 : (h.weight_decay != 0.0 ? 2 : 0);
    c.lerp_hi = (c.b1c < 0.5f) ? 0 : 1;
    c.dec1 = c.mode == 1 ? c.dec : 1.0f;
    c.wdl2 = c.mode == 2 ? c.wd : 0.0f;
    c.fast_ok = !c.lerp_hi && c.bc2s >= 0x1p-60f && c.bc2s < 0x1p61f;
    c._pad = 0;
    return c;
}

SgdK derive_sgd(const mpo_sgd_hp& h) {
    SgdK c;
    c.gs = float(h.grad_scale);
    c.lr = float(h.lr);
    c.mom = float(h.momentum);
    c.damp1 = float(1.0 - h.dampening);
    c.wd = float(h.weight_decay);
    c.has_wd = h.weight_decay != 0.0;
    c.has_mom = h.momentum != 0.0;
    c.first = h.first_step != 0;
    c.nesterov = h.nesterov != 0;
    c._pad = 0;
    return c;
}

mpo_status check_adam_hp(const mpo_adam_hp* hp, int32_t nhp) {
    if (!hp || nhp < 1 || nhp > MPO_MAX_HP_GROUPS) return fail(MPO_EINVAL, "hyper-parameter group count out of range");
    for (int i = 0; i < nhp; ++i) {
        const mpo_adam_hp& h = hp[i];
        if (!finite(h.lr) || !finite(h.beta1) || !finite(h.beta2) || !finite(h.eps) || !finite(h.weight_decay) ||
            !finite(h.grad_scale) || !finite(h.max_grad_norm))
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": non-finite hyper-parameter");
        if (h.step < 1) return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": step must be >= 1");
        if (h.beta1 < 0.0 || h.beta1 >= 1.0 || h.beta2 < 0.0 || h.beta2 >= 1.0)
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": betas must lie in [0, 1)");
        if (h.max_grad_norm != hp[0].max_grad_norm)
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": max_grad_norm differs from group 0");
    }
    return MPO_OK;
}

mpo_status check_sgd_hp(const mpo_sgd_hp* hp, int32_t nhp) {
    if (!hp || nhp < 1 || nhp > MPO_MAX_HP_GROUPS) return fail(MPO_EINVAL, "hyper-parameter group count out of range");
    for (int i = 0; i < nhp; ++i) {
        const mpo_sgd_hp& h = hp[i];
        if (!finite(h.lr) || !finite(h.momentum) || !finite(h.dampening) || !finite(h.weight_decay) ||
            !finite(h.grad_scale))
            return fail(MPO_EINVAL, "sgd group " + std::to_string(i) + ": non-finite hyper-parameter");
        if (h.nesterov && (h.momentum == 0.0 || h.dampening != 0.0))
            return fail(MPO_EINVAL, "sgd group " + std::to_string(i) + ": nesterov needs momentum > 0, dampening 0");
    }
    return MPO_OK;
}

mpo_status check_dtypes(mpo_dtype vdt, mpo_dtype gdt) {
    if (vdt != MPO_FP16 && vdt != MPO_BF16) return fail(MPO_EDTYPE, "value dtype must be MPO_FP16 or MPO_BF16");
    if (gdt != MPO_FP16 && gdt != MPO_BF16 && gdt != MPO_FP32)
        return fail(MPO_EDTYPE, "grad dtype must be MPO_FP16, MPO_BF16 or MPO_FP32");
    return MPO_OK;
}

mpo_status check_table(const mpo_tensor* t, int32_t nt, int32_t nhp, bool adam, const mpo_sgd_hp* sgd) {
    if (nt < 0 || (nt > 0 && !t)) return fail(MPO_EINVAL, "bad tensor table");
    for (int i = 0; i < nt; ++i) {
        const mpo_tensor& x = t[i];
        const std::string who = "tensor " + std::to_string(i) + ": ";
        if (x.n < 0) return fail(MPO_EINVAL, who + "negative size");
        if (x.hp < 0 || x.hp >= nhp) return fail(MPO_EINVAL, who + "hyper-parameter group index out of range");
        if (x.n == 0) continue;
        const bool need_m = adam || (sgd && sgd[x.hp].momentum != 0.0);
        if (!x.value || !x.resid || !x.grad || (need_m && !x.m) || (adam && !x.v))
            return fail(MPO_EINVAL, who + "NULL array");
        if (!aligned16(x.value) || !aligned16(x.resid) || !aligned16(x.grad) || (need_m && !aligned16(x.m)) ||
            (adam && !aligned16(x.v)))
            return fail(MPO_EALIGN, who + "array base pointer not 16-byte aligned");
    }
    return MPO_OK;
}

// Fill a kernel table from t[lo, hi); returns the tile count.
template <int MAXT>
int64_t fill_table(Table<MAXT>& tab, const mpo_tensor* t, int lo, int hi, bool one_hp, int64_t tile_el = kTileEl) {
    int64_t tiles = 0;
    tab.nt = hi - lo;
    for (int i = lo; i < hi; ++i) {
        KT& k = tab.t[i - lo];
        k.value = t[i].value;
        k.resid = t[i].resid;
        k.grad = t[i].grad;
        k.m = t[i].m;
        k.v = t[i].v;
        k.n = t[i].n;
        k.hp = one_hp ? 0 : t[i].hp;
        k.tile0 = int32_t(tiles);
        tiles += (t[i].n + tile_el - 1) / tile_el;
    }
    tab.ntiles = int32_t(tiles);
    return tiles;
}

constexpr int kSumsqStages = 8;
// The clip pre-pass uses the LSU kernel unless MPO_SUMSQ_KERNEL=tma (A/B knob; see sumsq_kernel).
bool use_tma_sumsq() {
    static const bool tma = [] {
        const char* e = std::getenv("MPO_SUMSQ_KERNEL");
        return e && std::strcmp(e, "tma") == 0;
    }();
    return tma;
}

template <int MAXT, int F, int G>
mpo_status launch_sumsq(const mpo_tensor* t, int lo, int hi, const HP<float>& gsc, double* partial, int nblocks,
                        cudaStream_t s) {
    Table<MAXT> tab;
    fill_table(tab, t, lo, hi, false, use_tma_sumsq() ? kTileEl : kSumsqTileEl);
    if (use_tma_sumsq()) {
        auto kern = sumsq_tma_kernel<MAXT, G>;
        constexpr int smem = kBarBytes + kSumsqStages * int(kTileEl) * GradBytes<G>::v;
        static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (attr != cudaSuccess) return fail(MPO_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr));
        kern<<<nblocks, kTmaThreads, smem, s>>>(tab, gsc, partial, kSumsqStages);
        ++g_launches;
        return check_launch("sumsq_tma_kernel");
    }
    sumsq_kernel<MAXT, G><<<nblocks, kThreads, 0, s>>>(tab, gsc, partial);
    ++g_launches;
    return check_launch("sumsq_kernel");
}

// Kernel variant: "tma" (default, bulk-copy pipeline) or "lsu" (per-thread 128-bit loads), chosen
// once per process from MPO_STEP_KERNEL (A/B evidence for DESIGN.md section 5).
bool use_tma() {
    static const bool tma = [] {
        const char* e = std::getenv("MPO_STEP_KERNEL");
        return !(e && std::strcmp(e, "lsu") == 0);
    }();
    return tma;
}

constexpr int kSmemBudget = (MPO_CTAS_PER_SM == 1 ? 227 * 1024 : (228 * 1024) / MPO_CTAS_PER_SM - 1024);

template <int MAXT, int F, int G, class Op, bool CLIP>
mpo_status launch_step_slice(const mpo_tensor* t, int lo, int hi, const HP<typename Op::K>& hp, bool one_hp,
                             const double* sumsq, double max_norm, cudaStream_t s) {
    Table<MAXT> tab;
    const int64_t tiles = fill_table(tab, t, lo, hi, one_hp);
    if (tiles == 0) return MPO_OK;
    if (tiles > INT32_MAX) return fail(MPO_EINVAL, "table slice too large");
    if (use_tma()) {
        auto kern = step_tma_kernel<MAXT, F, G, Op, CLIP>;
        constexpr int SB = stage_bytes<G, Op::kHasV>();
        constexpr int stages = (kSmemBudget - kBarBytes) / SB < kMaxStages ? (kSmemBudget - kBarBytes) / SB : kMaxStages;
        static_assert(stages >= 2, "need at least two pipeline stages");
        constexpr int smem = kBarBytes + stages * SB;
        static const cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (attr != cudaSuccess) return fail(MPO_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr));
        const int64_t grid = grid_for(tiles, MPO_CTAS_PER_SM);
        kern<<<unsigned(grid), kTmaThreads, smem, s>>>(tab, hp, sumsq, max_norm, stages);
        ++g_launches;
        return check_launch("step_tma_kernel");
    }
    auto kern = step_kernel<MAXT, F, G, Op, CLIP>;
    static int per_sm = resident_blocks(kern);
    const int64_t grid = grid_for(tiles, per_sm);
    kern<<<unsigned(grid), kThreads, 0, s>>>(tab, hp, sumsq, max_norm);
    ++g_launches;
    return check_launch("step_kernel");
}

constexpr int kBigT = 512;    // 512 x 56 B + 16 groups fits the 32 KB kernel-parameter limit
constexpr int kMidT = 32;

template <int F, int G, class Op, bool CLIP>
mpo_status launch_step(const mpo_tensor* t, int nt, const HP<typename Op::K>& hp, bool one_hp, const double* sumsq,
                       double max_norm, cudaStream_t s) {
    for (int lo = 0; lo < nt; lo += kBigT) {
        const int hi = lo + kBigT < nt ? lo + kBigT : nt;
        mpo_status st;
        if (hi - lo == 1) st = launch_step_slice<1, F, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, s);
        else if (hi - lo <= kMidT) st = launch_step_slice<kMidT, F, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, s);
        else st = launch_step_slice<kBigT, F, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, s);
        if (st != MPO_OK) return st;
    }
    return MPO_OK;
}

template <template <int, int> class OpT, bool CLIP>
mpo_status dispatch_step(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int nt,
                         const HP<typename OpT<0, 0>::K>& hp, bool one_hp, const double* sumsq, double max_norm,
                         cudaStream_t s) {
#define MPO_CASE(VF, GF)                                                                                   \
    if (vdt == (VF) && gdt == (GF))                                                                        \
        return launch_step<int(VF), int(GF), OpT<int(VF), int(GF)>, CLIP>(t, nt, hp, one_hp, sumsq, max_norm, s);
    MPO_CASE(MPO_FP16, MPO_FP16)
    MPO_CASE(MPO_FP16, MPO_BF16)
    MPO_CASE(MPO_FP16, MPO_FP32)
    MPO_CASE(MPO_BF16, MPO_FP16)
    MPO_CASE(MPO_BF16, MPO_BF16)
    MPO_CASE(MPO_BF16, MPO_FP32)
#undef MPO_CASE
    return fail(MPO_EDTYPE, "unsupported dtype pair");
}

// Sum of squares of the scaled grads of the whole table into norm_ws[0] (partials in norm_ws[1..]).
mpo_status table_sumsq(mpo_dtype gdt, const mpo_tensor* t, int nt, const float* gs_of_group, int nhp,
                       double* norm_ws, cudaStream_t s) {
    HP<float> gsc;
    for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) gsc.g[i] = i < nhp ? gs_of_group[i] : 1.0f;
    int64_t tiles = 0;
    const int64_t te = use_tma_sumsq() ? kTileEl : kSumsqTileEl;
    for (int i = 0; i < nt; ++i) tiles += (t[i].n + te - 1) / te;
    static const int per_sm = use_tma_sumsq() ? 1 : resident_blocks(sumsq_kernel<kBigT, kBF16>);
    const int64_t g0 = grid_for(tiles, per_sm);
    const int nblocks = int(g0 < kNormBlocksMax ? g0 : kNormBlocksMax);
    double* partial = norm_ws + 1;
    int nparts = 0;
    // every slice writes its own run of partials, summed together at the end (fixed order)
    for (int lo = 0; lo < nt || (nt == 0 && lo == 0); lo += kBigT) {
        const int hi = lo + kBigT < nt ? lo + kBigT : nt;
        const int nb = nt == 0 ? 1 : nblocks;
        if (nparts + nb > kNormBlocksMax) return fail(MPO_EINVAL, "table too large for the norm workspace");
        mpo_status st;
        if (gdt == MPO_FP32) st = launch_sumsq<kBigT, kFP32, kFP32>(t, lo, hi, gsc, partial + nparts, nb, s);
        else if (gdt == MPO_BF16) st = launch_sumsq<kBigT, kBF16, kBF16>(t, lo, hi, gsc, partial + nparts, nb, s);
        else st = launch_sumsq<kBigT, kFP16, kFP16>(t, lo, hi, gsc, partial + nparts, nb, s);
        if (st != MPO_OK) return st;
        nparts += nb;
        if (nt == 0) break;
    }
    sumsq_final_kernel<<<1, kThreads, 0, s>>>(partial, nparts, norm_ws);
    ++g_launches;
    return check_launch("sumsq_final_kernel");
}

// Wrap an NCCL call.
#define MPO_NCCL(call)                                                                             \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess) return fail(MPO_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

ncclDataType_t nccl_dtype(mpo_dtype d) { return d == MPO_BF16 ? ncclBfloat16 : ncclFloat16; }

}  // namespace mpo

using namespace mpo;

// ------------------------------------------------------------------------------------------
// C ABI
// ------------------------------------------------------------------------------------------
MPO_API const char* mpo_last_error(void) { return g_err.c_str(); }

#ifdef MPO_EXACT
MPO_API int32_t mpo_build_exact(void) { return 1; }
#else
MPO_API int32_t mpo_build_exact(void) { return 0; }
#endif

MPO_API int64_t mpo_launch_count(void) { return g_launches.load(); }

MPO_API int64_t mpo_norm_ws_doubles(void) { return 1 + kNormBlocksMax; }

MPO_API mpo_status mpo_selfcheck_fastmath(int64_t pairs, uint64_t seed, unsigned long long* counts,
                                          mpo_stream stream) {
    g_err.clear();
    if (pairs < 0) return fail(MPO_EINVAL, "negative pair count");
    if (!counts) return fail(MPO_EINVAL, "NULL counts");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(counts, 0, 4 * sizeof(unsigned long long), s) != cudaSuccess)
        return check_launch("cudaMemsetAsync");
    const unsigned grid = unsigned(num_sms()) * 8u;
    selfcheck_sqrt_kernel<<<grid, kThreads, 0, s>>>(counts);
    ++g_launches;
    if (check_launch("selfcheck_sqrt_kernel") != MPO_OK) return MPO_ECUDA;
    selfcheck_div_kernel<<<grid, kThreads, 0, s>>>(pairs, seed, counts);
    ++g_launches;
    return check_launch("selfcheck_div_kernel");
}

MPO_API mpo_status mpo_split(mpo_dtype vdt, const float* w, void* value, int16_t* resid, int64_t n,
                             mpo_stream stream) {
    g_err.clear();
    if (vdt != MPO_FP16 && vdt != MPO_BF16) return fail(MPO_EDTYPE, "value dtype must be MPO_FP16 or MPO_BF16");
    if (n < 0) return fail(MPO_EINVAL, "negative size");
    if (n == 0) return MPO_OK;
    if (!w || !value || !resid) return fail(MPO_EINVAL, "NULL array");
    if (!aligned16(w) || !aligned16(value) || !aligned16(resid)) return fail(MPO_EALIGN, "array not 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t grid = grid_for((n / kUnitEl + kThreads - 1) / kThreads + 1, 8);
    if (vdt == MPO_FP16)
        split_kernel<kFP16><<<unsigned(grid), kThreads, 0, s>>>(w, static_cast<uint16_t*>(value), resid, n);
    else
        split_kernel<kBF16><<<unsigned(grid), kThreads, 0, s>>>(w, static_cast<uint16_t*>(value), resid, n);
    ++g_launches;
    return check_launch("split_kernel");
}

MPO_API mpo_status mpo_reconstruct(mpo_dtype vdt, const void* value, const int16_t* resid, float* w, int64_t n,
                                   mpo_stream stream) {
    g_err.clear();
    if (vdt != MPO_FP16 && vdt != MPO_BF16) return fail(MPO_EDTYPE, "value dtype must be MPO_FP16 or MPO_BF16");
    if (n < 0) return fail(MPO_EINVAL, "negative size");
    if (n == 0) return MPO_OK;
    if (!w || !value || !resid) return fail(MPO_EINVAL, "NULL array");
    if (!aligned16(w) || !aligned16(value) || !aligned16(resid)) return fail(MPO_EALIGN, "array not 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t grid = grid_for((n / kUnitEl + kThreads - 1) / kThreads + 1, 8);
    if (vdt == MPO_FP16)
        reconstruct_kernel<kFP16><<<unsigned(grid), kThreads, 0, s>>>(static_cast<const uint16_t*>(value), resid, w, n);
    else
        reconstruct_kernel<kBF16><<<unsigned(grid), kThreads, 0, s>>>(static_cast<const uint16_t*>(value), resid, w, n);
    ++g_launches;
    return check_launch("reconstruct_kernel");
}

MPO_API mpo_status mpo_sgd_step(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const mpo_sgd_hp* hp,
                                int32_t nhp, mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    if ((st = check_sgd_hp(hp, nhp)) != MPO_OK) return st;
    if ((st = check_table(t, nt, nhp, false, hp)) != MPO_OK) return st;
    HP<SgdK> k;
    for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = derive_sgd(hp[i < nhp ? i : 0]);
    return dispatch_step<SgdOp, false>(vdt, gdt, t, nt, k, false, nullptr, 0.0, static_cast<cudaStream_t>(stream));
}

static mpo_status adam_common(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const mpo_adam_hp* hp,
                              int32_t nhp, double* norm_ws, bool one_hp, cudaStream_t s, bool sumsq_ready) {
    HP<AdamK> k;
    for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = derive_adam(hp[i < nhp ? i : 0]);
    const double max_norm = hp[0].max_grad_norm;
    if (max_norm > 0.0) {
        if (!norm_ws) return fail(MPO_EINVAL, "clipping (max_grad_norm > 0) needs a norm workspace");
        if (!sumsq_ready) {
            float gs[MPO_MAX_HP_GROUPS];
            for (int i = 0; i < nhp; ++i) gs[i] = k.g[i].gs;
            mpo_status st = table_sumsq(gdt, t, nt, gs, nhp, norm_ws, s);
            if (st != MPO_OK) return st;
        }
        return dispatch_step<AdamOp, true>(vdt, gdt, t, nt, k, one_hp, norm_ws, max_norm, s);
    }
    return dispatch_step<AdamOp, false>(vdt, gdt, t, nt, k, one_hp, nullptr, 0.0, s);
}

MPO_API mpo_status mpo_adam_step(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt,
                                 const mpo_adam_hp* hp, int32_t nhp, double* norm_ws, mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    if ((st = check_adam_hp(hp, nhp)) != MPO_OK) return st;
    if ((st = check_table(t, nt, nhp, true, nullptr)) != MPO_OK) return st;
    return adam_common(vdt, gdt, t, nt, hp, nhp, norm_ws, false, static_cast<cudaStream_t>(stream), false);
}

MPO_API mpo_status mpo_fused_backward_hook_step(mpo_optim kind, mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* one,
                                                const void* hp, mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if (!one || !hp) return fail(MPO_EINVAL, "NULL tensor or hyper-parameters");
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    mpo_tensor x = *one;
    x.hp = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, 1)) != MPO_OK) return st;
        if (h->max_grad_norm > 0.0)
            return fail(MPO_EINVAL, "global-norm clipping is impossible in the fused backward hook (P:93, P:186)");
        if ((st = check_table(&x, 1, 1, true, nullptr)) != MPO_OK) return st;
        return adam_common(vdt, gdt, &x, 1, h, 1, nullptr, true, s, false);
    }
    if (kind == MPO_SGD) {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, 1)) != MPO_OK) return st;
        if ((st = check_table(&x, 1, 1, false, h)) != MPO_OK) return st;
        HP<SgdK> k;
        for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = derive_sgd(*h);
        return dispatch_step<SgdOp, false>(vdt, gdt, &x, 1, k, true, nullptr, 0.0, s);
    }
    return fail(MPO_EINVAL, "unknown optimizer kind");
}

MPO_API mpo_status mpo_sharded_step(mpo_optim kind, uintptr_t nccl_comm, int32_t rank, int32_t world, mpo_dtype vdt,
                                    void* value_flat, void* grad_flat, int16_t* resid_shard, float* m_shard,
                                    float* v_shard, int64_t n_total, const void* hp, double* norm_ws,
                                    mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if (!nccl_comm) return fail(MPO_EINVAL, "NULL NCCL communicator");
    if (world < 1 || rank < 0 || rank >= world) return fail(MPO_EINVAL, "bad rank / world");
    if (n_total < 0 || n_total % (int64_t(8) * world) != 0)
        return fail(MPO_EINVAL, "n_total must be a non-negative multiple of 8*world");
    if (!hp) return fail(MPO_EINVAL, "NULL hyper-parameters");
    if ((st = check_dtypes(vdt, vdt)) != MPO_OK) return st;
    if (kind != MPO_SGD && kind != MPO_ADAM) return fail(MPO_EINVAL, "unknown optimizer kind");
    if (n_total == 0) return MPO_OK;
    if (!value_flat || !grad_flat) return fail(MPO_EINVAL, "NULL flat buffer");
    if (!aligned16(value_flat) || !aligned16(grad_flat)) return fail(MPO_EALIGN, "flat buffer not 16-byte aligned");
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t shard = n_total / world;
    mpo_tensor x;
    x.value = static_cast<uint16_t*>(value_flat) + rank * shard;
    x.resid = resid_shard;
    x.grad = static_cast<uint16_t*>(grad_flat) + rank * shard;
    x.m = m_shard;
    x.v = v_shard;
    x.n = shard;
    x.hp = 0;
    x._pad = 0;
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, 1)) != MPO_OK) return st;
        if ((st = check_table(&x, 1, 1, true, nullptr)) != MPO_OK) return st;
        if (h->max_grad_norm > 0.0 && !norm_ws) return fail(MPO_EINVAL, "clipping needs a norm workspace");
    } else {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, 1)) != MPO_OK) return st;
        if ((st = check_table(&x, 1, 1, false, h)) != MPO_OK) return st;
    }
    // 1. reduce-scatter of the 16-bit gradients (sum), in place: shard `rank` of grad_flat
    //    (world 1: the reduction of one rank is the identity and the in-place shard is the buffer)
    if (world > 1)
        MPO_NCCL(ncclReduceScatter(grad_flat, const_cast<void*>(x.grad), size_t(shard), nccl_dtype(vdt), ncclSum, comm, s));
    // 2. residual-compensated update of this rank's shard
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if (h->max_grad_norm > 0.0) {
            float gs = float(h->grad_scale);
            if ((st = table_sumsq(vdt, &x, 1, &gs, 1, norm_ws, s)) != MPO_OK) return st;
            if (world > 1) MPO_NCCL(ncclAllReduce(norm_ws, norm_ws, 1, ncclFloat64, ncclSum, comm, s));
        }
        if ((st = adam_common(vdt, vdt, &x, 1, h, 1, norm_ws, true, s, true)) != MPO_OK) return st;
    } else {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        HP<SgdK> k;
        for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = derive_sgd(*h);
        if ((st = dispatch_step<SgdOp, false>(vdt, vdt, &x, 1, k, true, nullptr, 0.0, s)) != MPO_OK) return st;
    }
    // 3. all-gather of the 16-bit values only (residual and state never move)
    if (world > 1) MPO_NCCL(ncclAllGather(x.value, value_flat, size_t(shard), nccl_dtype(vdt), comm, s));
    return MPO_OK;
}
