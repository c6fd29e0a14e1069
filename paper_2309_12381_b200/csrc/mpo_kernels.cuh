// mpo_kernels.cuh -- sm_100a kernels of the residual-compensated 16-bit optimizer step
// (arXiv 2309.12381) and their host launch templates.  Included by mpo.cu (C ABI, clip pre-pass,
// diagnostics) and by mpo_inst.cu, which is compiled once per storage format (-DMPO_SF=...) so the
// format instantiations build in parallel.  Citation keys as in include/mpo.h.
//
// Kernel design.  The step is an elementwise stream (no contraction, so
// no tensor cores): per element Adam moves 26 B (value 2 + resid 2 + grad 2 + m 4 + v 4 read;
// value, resid, m, v written), SGD-momentum 18 B.  It is HBM-bound on B200, so the kernel of
// every launch above 640 tiles (step_tma_kernel) is a persistent warp-specialised pipeline: one
// producer warp streams each 4096-element tile of every stream into shared-memory stages with 1-D
// TMA bulk copies while 16 consumer warps compute one 8-element unit per thread and store with
// 128-bit stores; smaller launches (hook-mode steps, small models) use step_kernel, whose
// per-thread loads avoid the pipeline's fill.  The
// multi-tensor table ("one only stream of values") travels by value as a __grid_constant__
// kernel parameter; ragged tails (n % 8) are handled element by element; warp shuffles appear
// only in the global-norm reduction (clipping).
#pragma once

#include "mpo.h"

#include <cuda_runtime.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "mpo_device.cuh"

#ifndef MPO_CW
#define MPO_CW 16            // consumer warps per CTA of the TMA kernel (A/B knob)
#endif
#ifndef MPO_CTAS_PER_SM
#define MPO_CTAS_PER_SM 1    // resident TMA CTAs per SM (A/B knob)
#endif

namespace mpo {

constexpr int kThreads = 256;
constexpr int kUnitEl = 8;                          // elements per unit (128-bit of 16-bit data)
constexpr int64_t kTileEl = int64_t(MPO_CW) * 32 * kUnitEl;   // 4096 elements: one unit per consumer thread
constexpr int kUnroll = int(kTileEl / (kThreads * kUnitEl));  // LSU kernel: units per thread per tile
static_assert(kUnroll >= 1 && kTileEl % (kThreads * kUnitEl) == 0, "LSU kernel needs whole 2048-element passes");
constexpr int64_t kLsuMaxTiles = 640;   // launches of at most this many tiles use step_kernel (auto)
constexpr int kNormBlocksMax = 2048;                // partial sums of the norm pre-pass
constexpr int kBigT = 512;    // 512 x 56 B + 16 groups fits the 32 KB kernel-parameter limit
constexpr int kMidT = 32;

struct KT {                 // one table entry inside the kernel parameter block
    void* value;
    void* resid;
    const void* grad;
    float* m;
    float* v;
    int64_t n;
    int32_t hps;            // hyper-parameter group (low 4 bits) | stochastic-rounding stream << 4
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

__device__ __forceinline__ int hp_of(const KT& T) { return T.hps & 15; }

// The tensor owning `tile`: the last entry whose first tile is <= tile (empty tensors share
// their successor's tile0 and are skipped), by binary search -- ~log2(nt) parameter-space loads
// instead of a dependent walk from entry 0.
template <int MAXT>
__device__ __forceinline__ int first_tensor(const Table<MAXT>& tab, int tile) {
    int l = 0, h = tab.nt - 1;
    while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (tab.t[mid].tile0 <= tile) l = mid;
        else h = mid - 1;
    }
    return l;
}
__device__ __forceinline__ uint32_t stream_of(const KT& T) { return static_cast<uint32_t>(T.hps) >> 4; }

// ------------------------------------------------------------------------------------------
// Host state shared by the translation units (defined in mpo.cu)
// ------------------------------------------------------------------------------------------
extern thread_local std::string g_err;
// Device copy of the call's derived hyper-parameters (HP<AdamK> / HP<SgdK>) when the step is issued
// by mpo_step_graphed (set around that call only; nullptr otherwise).
extern thread_local const void* g_dev_hp;
extern std::atomic<int64_t> g_launches;
mpo_status fail(mpo_status s, const std::string& msg);
mpo_status check_launch(const char* what);
int num_sms();
int step_kernel_choice();

inline int64_t grid_for(int64_t work_items, int per_sm) {
    int64_t cap = int64_t(num_sms()) * per_sm;
    int64_t g = work_items < cap ? work_items : cap;
    return g < 1 ? 1 : g;
}

template <class Kern>
int resident_blocks(Kern k, int threads = kThreads) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, threads, 0) != cudaSuccess || b < 1) {
        cudaGetLastError();
        b = 1;
    }
    return b;
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
        k.hps = (one_hp ? 0 : (t[i].hp & 15)) | (t[i].sr_stream << 4);
        k.tile0 = int32_t(tiles);
        tiles += (t[i].n + tile_el - 1) / tile_el;
    }
    tab.ntiles = int32_t(tiles);
    return tiles;
}

// ------------------------------------------------------------------------------------------
// Vector memory helpers: 128-bit streaming (evict-first) loads and stores.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldv(const void* p) { return __ldcs(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ float4 ldf(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
#ifdef MPO_ST_DEFAULT   // A/B knob: default (evict-normal) stores instead of streaming ones
__device__ __forceinline__ void stv(void* p, uint4 x) { *reinterpret_cast<uint4*>(p) = x; }
__device__ __forceinline__ void stf(float* p, float4 x) { *reinterpret_cast<float4*>(p) = x; }
#else
__device__ __forceinline__ void stv(void* p, uint4 x) { __stcs(reinterpret_cast<uint4*>(p), x); }
__device__ __forceinline__ void stf(float* p, float4 x) { __stcs(reinterpret_cast<float4*>(p), x); }
#endif
// 8 fp32 of one unit (m, v, reconstructed w): two 128-bit streaming stores.  (sm_100's 256-bit
// st.global.v8.f32 -- SASS STG.E.EF.ENL2.256 -- makes each warp store cover whole sectors instead
// of half sectors at a 32-B thread stride, but measured -0.5 % ResNet-50 / +0.5 % GPT-2 / -2 %
// LLaMA-7B: L2 merges the halves before write-back; profiles/r01_ab13_st256.log.)
__device__ __forceinline__ void stf8(float* p, const float (&x)[8]) {
    stf(p, make_float4(x[0], x[1], x[2], x[3]));
    stf(p + 4, make_float4(x[4], x[5], x[6], x[7]));
}

// 256-bit global store of 8 fp32 (sm_100: st.global.v8.f32): one thread covers a whole 32-B
// sector, so a warp's store is 1 KB contiguous instead of two half-sector passes.
__device__ __forceinline__ void st8f(float* p, const float (&x)[8]) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(x[0]), "f"(x[1]), "f"(x[2]),
                 "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]), "f"(x[7])
                 : "memory");
}

// 8 gradient values of a unit.
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

// 8 residual codes of a unit: 16 bytes (int16 / uint16 schemes) or 8 bytes (X8; in v.x, v.y).
template <int SF>
struct ResidUnit {
    uint4 v;
};

template <int SF>
__device__ __forceinline__ ResidUnit<SF> ld_resid(const void* base, int64_t e) {
    ResidUnit<SF> r;
    if constexpr (Fmt<SF>::rbytes == 2) {
        r.v = ldv(static_cast<const int16_t*>(base) + e);
    } else {
        const uint2 x = __ldcs(reinterpret_cast<const uint2*>(static_cast<const int8_t*>(base) + e));
        r.v = make_uint4(x.x, x.y, 0u, 0u);
    }
    return r;
}

template <int SF>
__device__ __forceinline__ void st_resid(void* base, int64_t e, const ResidUnit<SF>& r) {
    if constexpr (Fmt<SF>::rbytes == 2) stv(static_cast<int16_t*>(base) + e, r.v);
    else __stcs(reinterpret_cast<uint2*>(static_cast<int8_t*>(base) + e), make_uint2(r.v.x, r.v.y));
}

template <int SF>
__device__ __forceinline__ int32_t code_at(const ResidUnit<SF>& r, int k) {
    const uint32_t* w = &r.v.x;
    if constexpr (Fmt<SF>::scheme == kX8Z) {
        return static_cast<int32_t>((w[k >> 2] >> (8 * (k & 3))) & 0xFFu);              // uint8
    } else if constexpr (Fmt<SF>::rbytes == 1) {
        return static_cast<int32_t>(static_cast<int8_t>((w[k >> 2] >> (8 * (k & 3))) & 0xFFu));
    } else if constexpr (Fmt<SF>::scheme == kRTZ) {
        return static_cast<int32_t>((w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu);
    } else {
        return (k & 1) ? shi16(w[k >> 1]) : slo16(w[k >> 1]);
    }
}

// One stored residual code (scalar paths: tails, ragged ends).
template <int SF>
__device__ __forceinline__ int32_t load_code(const void* resid, int64_t i) {
    if constexpr (Fmt<SF>::scheme == kX8Z) return static_cast<const uint8_t*>(resid)[i];
    else if constexpr (Fmt<SF>::rbytes == 1) return static_cast<const int8_t*>(resid)[i];
    else if constexpr (Fmt<SF>::scheme == kRTZ) return static_cast<const uint16_t*>(resid)[i];
    else return static_cast<const int16_t*>(resid)[i];
}

template <int SF>
__device__ __forceinline__ ResidUnit<SF> pack_codes(const int32_t (&c)[8]) {
    ResidUnit<SF> r;
    if constexpr (Fmt<SF>::rbytes == 1) {
        const uint32_t lo = __byte_perm(__byte_perm(uint32_t(c[0]), uint32_t(c[1]), 0x0040),
                                        __byte_perm(uint32_t(c[2]), uint32_t(c[3]), 0x0040), 0x5410);
        const uint32_t hi = __byte_perm(__byte_perm(uint32_t(c[4]), uint32_t(c[5]), 0x0040),
                                        __byte_perm(uint32_t(c[6]), uint32_t(c[7]), 0x0040), 0x5410);
        r.v = make_uint4(lo, hi, 0u, 0u);
    } else {
        r.v = make_uint4(__byte_perm(uint32_t(c[0]), uint32_t(c[1]), 0x5410),
                         __byte_perm(uint32_t(c[2]), uint32_t(c[3]), 0x5410),
                         __byte_perm(uint32_t(c[4]), uint32_t(c[5]), 0x5410),
                         __byte_perm(uint32_t(c[6]), uint32_t(c[7]), 0x5410));
    }
    return r;
}

// RTZ of a pair to fp16 (hardware cvt.rz) / bf16 (pattern truncation), x0 -> low half.
template <int B>
__device__ __forceinline__ uint32_t rtz2(float x0, float x1) {
    if constexpr (B == kBF16) {
        return (__float_as_uint(x0) >> 16) | (__float_as_uint(x1) & 0xFFFF0000u);
    } else {
        uint32_t d;
        asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(x1), "f"(x0));
        return d;
    }
}

// Split a unit under a (deterministic) scheme: one fast branch per unit, general path for units
// with any rounded value Inf/NaN.
template <int SF>
__device__ __forceinline__ void split8_s(const float (&w)[8], uint32_t (&hv)[4], int32_t (&code)[8]) {
    using FM = Fmt<SF>;
    uint32_t p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if constexpr (FM::rtz_value) p[q] = rtz2<FM::base>(w[2 * q], w[2 * q + 1]);
        else p[q] = round2<FM::base>(w[2 * q], w[2 * q + 1]);
    }
    const uint32_t special = nonfinite_pair<FM::base>(p[0]) | nonfinite_pair<FM::base>(p[1]) |
                             nonfinite_pair<FM::base>(p[2]) | nonfinite_pair<FM::base>(p[3]);
    if (__builtin_expect(special == 0u, 1)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            hv[q] = p[q];
            code[2 * q] = resid_code<SF>(w[2 * q], lo16(p[q]));
            code[2 * q + 1] = resid_code<SF>(w[2 * q + 1], hi16(p[q]));
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t h0, h1;
            split1_s<SF>(w[2 * q], 0u, h0, code[2 * q]);
            split1_s<SF>(w[2 * q + 1], 0u, h1, code[2 * q + 1]);
            hv[q] = h0 | (h1 << 16);
        }
    }
}

// ------------------------------------------------------------------------------------------
// G1 / G2: split and reconstruct, any scheme.
// ------------------------------------------------------------------------------------------
template <int SF>
__global__ void __launch_bounds__(kThreads) split_kernel(const float* __restrict__ w, uint16_t* __restrict__ value,
                                                         void* __restrict__ resid, int64_t n, uint64_t seed,
                                                         uint32_t stream) {
    const int64_t nunits = n / kUnitEl;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        const int64_t e = u * kUnitEl;
        // (256-bit loads here: +3 % at 2^24 elements, -1.2 % at 2^28; profiles/r02_ab_conv.log)
        const float4 x0 = ldf(w + e), x1 = ldf(w + e + 4);
        const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        uint32_t hv[4];
        int32_t code[8];
        if constexpr (Fmt<SF>::scheme == kSR) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t h0, h1;
                const uint64_t rr = sr_mix(seed, stream, uint64_t(e + 2 * q) >> 1);   // e is even
                split1_s<SF>(x[2 * q], static_cast<uint32_t>(rr >> 32), h0, code[2 * q]);
                split1_s<SF>(x[2 * q + 1], static_cast<uint32_t>(rr), h1, code[2 * q + 1]);
                hv[q] = h0 | (h1 << 16);
            }
        } else {
            split8_s<SF>(x, hv, code);
        }
        stv(value + e, make_uint4(hv[0], hv[1], hv[2], hv[3]));
        st_resid<SF>(resid, e, pack_codes<SF>(code));
    }
    // ragged tail (n % 8 elements), one thread per element
    const int64_t t = nunits * kUnitEl + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && t < nunits * kUnitEl + kUnitEl) {
        uint32_t h;
        int32_t code;
        split1_s<SF>(w[t], sr_draw(seed, stream, uint64_t(t)), h, code);
        value[t] = static_cast<uint16_t>(h);
        if constexpr (Fmt<SF>::rbytes == 1) static_cast<int8_t*>(resid)[t] = static_cast<int8_t>(code);
        else static_cast<int16_t*>(resid)[t] = static_cast<int16_t>(code);
    }
}

template <int SF>
__global__ void __launch_bounds__(kThreads) reconstruct_kernel(const uint16_t* __restrict__ value,
                                                               const void* __restrict__ resid,
                                                               float* __restrict__ w, int64_t n) {
    const int64_t nunits = n / kUnitEl;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        const int64_t e = u * kUnitEl;
        const uint4 hv = ldv(value + e);
        const ResidUnit<SF> rv = ld_resid<SF>(resid, e);
        const uint32_t* h = &hv.x;
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = reconstruct1_s<SF>((k & 1) ? hi16(h[k >> 1]) : lo16(h[k >> 1]), code_at<SF>(rv, k));
        // one 256-bit store per thread (a whole 32-B sector; a warp writes 1 KB contiguous): +15 % at
        // 2^28 elements over two 128-bit half-sector stores (profiles/r02_ab_conv.log)
        st8f(w + e, o);
    }
    const int64_t t = nunits * kUnitEl + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < n && t < nunits * kUnitEl + kUnitEl) {
        const int32_t code = load_code<SF>(resid, t);
        w[t] = reconstruct1_s<SF>(value[t], code);
    }
}

// Clip coefficient from the global sum of squares: min(1, max_norm / (sqrt(S) + 1e-6)),
// rounded once to float; a NaN quotient propagates (R9).
__device__ __forceinline__ float clip_coef(const double* sumsq, double max_norm) {
    const double q = max_norm / (sqrt(sumsq[0]) + 1e-6);
    return q > 1.0 ? 1.0f : float(q);
}

#ifdef MPO_ABI_TU   // the clip pre-pass is instantiated by mpo.cu only
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
    int cur = first_tensor(tab, int(blockIdx.x));   // not a dependent walk from tensor 0
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        const float gs = gsc.g[hp_of(T)];
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

// Sums nparts partials (fixed order) into out[0] (add_out: out[0] += the sum, mpo_grad_sumsq's
// accumulation over several tables of one step).
__global__ void __launch_bounds__(kThreads) sumsq_final_kernel(const double* __restrict__ partial, int nparts,
                                                               double* __restrict__ out, double* __restrict__ accum,
                                                               int add_out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += partial[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        out[0] = add_out ? out[0] + acc : acc;
        if (accum) accum[0] += acc;   // hook mode: found-inf over a whole backward
    }
}


#endif  // MPO_ABI_TU

// ------------------------------------------------------------------------------------------
// G3 / G4: multi-tensor residual-compensated step.
// ------------------------------------------------------------------------------------------
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

// One unit (8 consecutive elements, the first at tensor index e0): reconstruct -> update ->
// re-split, registers in and out.
template <int SF, int G, class Op, bool CLIP>
__device__ __forceinline__ void process_unit(const uint4& hv, const ResidUnit<SF>& rv, const GradUnit<G>& gu,
                                             float (&mm)[8], float (&vv)[8], const typename Op::K& c, float coef,
                                             uint32_t stream, int64_t e0, uint4& ho, ResidUnit<SF>& ro) {
    using FM = Fmt<SF>;
    const uint32_t* h = &hv.x;
    float w[8], g[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k] = grad_at<G>(gu, k);
    if (c.gs != 1.0f) {   // uniform; g * 1 == g exactly, so skipping it changes nothing
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] = g[k] * c.gs;
    }
    if (c.clip_on) {   // uniform per tensor
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] = clamp_grad(g[k], c.clipv);
    }
    if constexpr (CLIP) {
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] = g[k] * coef;
    }
    const uint32_t special = nonfinite_pair<FM::base>(h[0]) | nonfinite_pair<FM::base>(h[1]) |
                             nonfinite_pair<FM::base>(h[2]) | nonfinite_pair<FM::base>(h[3]);
    bool done = false;
    if (__builtin_expect(special == 0u, 1)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t w1 = FM::base == kBF16 ? (h[q] & 0xFFFF0000u) : widen_bits<FM::base>(hi16(h[q]));
            w[2 * q] = __uint_as_float(widen_bits<FM::base>(lo16(h[q])) + resid_addend<SF>(code_at<SF>(rv, 2 * q)));
            w[2 * q + 1] = __uint_as_float(w1 + resid_addend<SF>(code_at<SF>(rv, 2 * q + 1)));
        }
        done = Op::unit_fast(w, g, mm, vv, c);
    }
    if (__builtin_expect(!done, 0)) {
        // non-finite values, or an operand outside the fast sqrt/div windows: the general path
        // (full IEEE operators; mm/vv are untouched by a failed fast attempt)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            w[k] = reconstruct1_s<SF>((k & 1) ? hi16(h[k >> 1]) : lo16(h[k >> 1]), code_at<SF>(rv, k));
            w[k] = Op::apply(w[k], g[k], mm[k], vv[k], c);
        }
    }
    uint32_t hq[4];
    int32_t code[8];
    if constexpr (FM::scheme == kSR) {
        // Fast unit path when all 8 magnitudes lie in fp16's normal range below the largest finite
        // value, [2^-14, 65504): there t = RTZ(x) is the top 10 mantissa bits, the spacing U is
        // 2^13 binary32 patterns, D = the 13 dropped bits, so sr1's rule "up iff rnd < D*2^32/U"
        // is rnd < D << 19 and the residual is D - up*2^13 -- the same integers as sr1 /
        // resid_code, without their range branches and the 64-bit division kept for subnormals.
        uint32_t a[8];
        bool fast = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a[k] = __float_as_uint(w[k]) & 0x7FFFFFFFu;
            fast &= (a[k] - 0x38800000u) < (0x477FE000u - 0x38800000u);
        }
        if (__builtin_expect(fast, 1)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t rr = sr_mix(c.seed, stream, uint64_t(e0 + 2 * q) >> 1);   // e0 is even
                uint32_t hh[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int k = 2 * q + j;
                    const uint32_t rnd = j == 0 ? static_cast<uint32_t>(rr >> 32) : static_cast<uint32_t>(rr);
                    const uint32_t d = a[k] & 0x1FFFu;
                    const uint32_t up = rnd < (d << 19) ? 1u : 0u;
                    hh[j] = ((__float_as_uint(w[k]) >> 16) & 0x8000u) | ((a[k] >> 13) - 0x1C000u + up);
                    code[k] = static_cast<int32_t>(d) - static_cast<int32_t>(up << 13);
                }
                hq[q] = hh[0] | (hh[1] << 16);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t h0, h1;
                const uint64_t rr = sr_mix(c.seed, stream, uint64_t(e0 + 2 * q) >> 1);   // e0 is even
                split1_s<SF>(w[2 * q], static_cast<uint32_t>(rr >> 32), h0, code[2 * q]);
                split1_s<SF>(w[2 * q + 1], static_cast<uint32_t>(rr), h1, code[2 * q + 1]);
                hq[q] = h0 | (h1 << 16);
            }
        }
    } else {
        split8_s<SF>(w, hq, code);
    }
    ho = make_uint4(hq[0], hq[1], hq[2], hq[3]);
    ro = pack_codes<SF>(code);
}

// Ragged tail of one tensor: element by element from global memory.
template <int SF, int G, class Op, bool CLIP>
__device__ __noinline__ void process_tail(const KT T, int64_t lo, int64_t hi, const typename Op::K c, float coef) {
    using FM = Fmt<SF>;
    uint16_t* val = static_cast<uint16_t*>(T.value);
    const bool need_m = Op::reads_m(c), has_m = Op::writes_m(c);
    for (int64_t i = lo; i < hi; ++i) {
        float g = grad_scalar<G>(T.grad, i) * c.gs;
        if (c.clip_on) g = clamp_grad(g, c.clipv);
        if constexpr (CLIP) g = g * coef;
        int32_t code;
        code = load_code<SF>(T.resid, i);
        float w = reconstruct1_s<SF>(val[i], code);
        float mi = need_m ? T.m[i] : 0.0f;
        float vi = 0.0f;
        if constexpr (Op::kHasV) vi = T.v[i];
        w = Op::apply(w, g, mi, vi, c);
        uint32_t h;
        split1_s<SF>(w, sr_draw(c.seed, stream_of(T), uint64_t(i)), h, code);
        val[i] = static_cast<uint16_t>(h);
        if constexpr (FM::rbytes == 1) static_cast<int8_t*>(T.resid)[i] = static_cast<int8_t>(code);
        else static_cast<int16_t*>(T.resid)[i] = static_cast<int16_t>(code);
        if (has_m) T.m[i] = mi;
        if constexpr (Op::kHasV) T.v[i] = vi;
    }
}

template <int SF, class Op>
__device__ __forceinline__ void store_unit(const KT& T, int64_t e, const uint4& ho, const ResidUnit<SF>& ro,
                                           const float (&mm)[8], const float (&vv)[8], bool has_m) {
    stv(static_cast<uint16_t*>(T.value) + e, ho);
    st_resid<SF>(T.resid, e, ro);
    if (has_m) {
        stf8(T.m + e, mm);
    }
    if constexpr (Op::kHasV) {
        stf8(T.v + e, vv);
    }
}

// ---- variant A ("lsu"): every thread loads its own units with 128-bit LDG, computes, stores.  The
// default for small launches (<= kLsuMaxTiles tiles: hook mode's per-parameter steps, config C1),
// where a grid of several CTAs per SM with every load in flight at once beats the pipeline's fill.
template <int MAXT, int SF, int G, class Op, bool CLIP, bool DHP>
__global__ void __launch_bounds__(kThreads) step_kernel(const __grid_constant__ Table<MAXT> tab,
                                                        const __grid_constant__ HP<typename Op::K> hp,
                                                        const HP<typename Op::K>* __restrict__ dhp,
                                                        const double* __restrict__ sumsq, double max_norm,
                                                        int skip) {
    using K = typename Op::K;
    if (skip && !isfinite(sumsq[0])) return;   // loss-scaling found-inf: no update at all
    float coef = 1.0f;
    if constexpr (CLIP) coef = clip_coef(sumsq, max_norm);
    int cur = first_tensor(tab, int(blockIdx.x));   // not a dependent walk from tensor 0
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        // DHP: a graph-replayed step (mpo_step_graphed) reads its hyper-parameters from the device
        // block; its own instantiation, because a runtime select between the two banks kept both
        // structs in registers (122 -> 156 registers: one CTA per SM instead of two)
        K c;
        if constexpr (DHP) c = dhp->g[hp_of(T)];
        else c = hp.g[hp_of(T)];
        const bool need_m = Op::reads_m(c);
        const bool has_m = Op::writes_m(c);
        const int64_t base = int64_t(tile - T.tile0) * kTileEl;
        const int64_t n = T.n;
        // X8 residual rows are 8 bytes per unit: units must also be 16-element aligned for the
        // vector path; the LSU kernel simply treats the last partial 16-element group as a tail
        const int64_t nvec = Fmt<SF>::rbytes == 1 ? (n & ~int64_t(15)) : (n & ~int64_t(kUnitEl - 1));

        uint4 hv[kUnroll];
        ResidUnit<SF> rv[kUnroll];
        GradUnit<G> gu[kUnroll];
        float4 m0[kUnroll], m1[kUnroll], v0[kUnroll], v1[kUnroll];
        // ---- load phase: every 128-bit load of kUnroll units in flight before any math ----
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const int64_t e = base + (int64_t(j) * kThreads + threadIdx.x) * kUnitEl;
            if (e + kUnitEl <= nvec) {
                hv[j] = ldv(static_cast<uint16_t*>(T.value) + e);
                rv[j] = ld_resid<SF>(T.resid, e);
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
            if (e + kUnitEl <= nvec) {
                float mm[8] = {m0[j].x, m0[j].y, m0[j].z, m0[j].w, m1[j].x, m1[j].y, m1[j].z, m1[j].w};
                float vv[8] = {v0[j].x, v0[j].y, v0[j].z, v0[j].w, v1[j].x, v1[j].y, v1[j].z, v1[j].w};
                uint4 ho;
                ResidUnit<SF> ro;
                process_unit<SF, G, Op, CLIP>(hv[j], rv[j], gu[j], mm, vv, c, coef, stream_of(T), e, ho, ro);
                store_unit<SF, Op>(T, e, ho, ro, mm, vv, has_m);
            } else if (e == nvec && e < n) {
                process_tail<SF, G, Op, CLIP>(T, e, n, c, coef);   // nvec is a multiple of 8
            }
        }
    }
}

// ---- variant B ("tma", default): warp-specialised bulk-copy pipeline ----------------------
// One producer warp streams each tile's value / residual / grad / m / v from HBM into a ring of
// shared-memory stages with 1-D TMA bulk copies (cp.async.bulk, mbarrier complete_tx, L2
// evict-normal); kCW consumer warps read the stage from shared memory, compute, and store the
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
// Wait for the phase of `parity` to complete.  The suspend-time hint lets the hardware park the
// waiting warp until the phase flips (or the hint expires) instead of re-issuing try_wait in a
// tight loop, which would steal issue slots from the producer and the computing warps.
#ifndef MPO_WAIT_HINT_NS
#define MPO_WAIT_HINT_NS 0x989680
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if MPO_WAIT_HINT_NS > 0
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(MPO_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
// L2 policy of the bulk-copy loads.  evict_normal: a loaded line stays until the unit's store
// of the same line (value, residual, m, v are updated in place) hits it in L2; evict_first
// measured 0.2-0.9 % slower (profiles/r01_ab14_cache_policy.log); evict_first for the read-only
// gradient stream alone -0.9 % ResNet-50, -0.7 % GPT-2, +0.4 % LLaMA-7B (r01_ab15_*.log).
__device__ __forceinline__ uint64_t load_policy() {
    uint64_t pol;
#ifdef MPO_LD_EVICT_FIRST   // A/B knob
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#endif
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

#ifdef MPO_BULK_ST
// 1-D bulk copy shared -> global (async proxy, bulk-group completion), the store side of the
// A/B "MPO_BULK_ST": each consumer warp writes its outputs over its inputs in the stage and one
// lane streams them out as four bulk copies instead of 6 x 128-bit STG per thread.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
#endif

#ifdef MPO_L2_PREFETCH
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
#endif

template <int G>
struct GradBytes {
    static constexpr int v = G == kFP32 ? 4 : 2;
};

// the piece a stage holds, published by the producer (tensor index < 0: end of schedule)
struct __align__(16) StageDesc {
    int64_t base;
    int32_t cur;
    int32_t nvalid;
};
constexpr int kDescBytes = kMaxStages * int(sizeof(StageDesc));   // keeps the ring 128-B aligned

// bytes of one stage: value 2 + resid rb + grad gb + m 4 [+ v 4] per element
template <int RB, int G, bool HAS_V>
__host__ __device__ constexpr int stage_bytes() {
    return int(kTileEl) * (2 + RB + GradBytes<G>::v + 4 + (HAS_V ? 4 : 0));
}


template <int MAXT, int SF, int G, class Op, bool CLIP, bool DHP>
__global__ void __launch_bounds__(kTmaThreads, MPO_CTAS_PER_SM) step_tma_kernel(const __grid_constant__ Table<MAXT> tab,
                                                                  const __grid_constant__ HP<typename Op::K> hp,
                                                                  const HP<typename Op::K>* __restrict__ dhp,
                                                                  const double* __restrict__ sumsq, double max_norm,
                                                                  int stages, int skip) {
    using K = typename Op::K;
    if (skip && !isfinite(sumsq[0])) return;   // loss-scaling found-inf: no update, nothing written
    constexpr int GB = GradBytes<G>::v;
    constexpr int RB = Fmt<SF>::rbytes;
    constexpr int64_t TE = kTileEl;
    // bulk copies move multiples of 16 bytes: 8 elements of 16-bit data, 16 of int8 residuals
    constexpr uint32_t kGran = RB == 1 ? 16u : uint32_t(kUnitEl);
    // stage layout: [value TE*2 | resid TE*RB | grad TE*GB | m TE*4 | v TE*4]
    constexpr int OFF_R = int(TE) * 2, OFF_G = int(TE) * (2 + RB), OFF_M = int(TE) * (2 + RB + GB),
                  OFF_V = int(TE) * (6 + RB + GB);
    constexpr int SB = stage_bytes<RB, G, Op::kHasV>();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    StageDesc* desc = reinterpret_cast<StageDesc*>(smem + kBarBytes);
    unsigned char* ring = smem + kBarBytes + kDescBytes;

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
        // ---------------- producer: scheduler + bulk copies ----------------
        // The producer alone walks the schedule and publishes each stage's piece (tensor, offset,
        // length) in the stage descriptor before arming the stage's barrier; the consumers read it
        // after their wait (mbarrier release/acquire orders the shared store), so the 16 consumer
        // warps carry no scheduling arithmetic and no walker registers.
        if (lane == 0) {
            const uint64_t pol = load_policy();
            // stage index and phase advance incrementally (a runtime `it % stages` costs two
            // integer divisions per tile)
            int s = 0;
            uint32_t ph = 0;
            auto issue = [&](int cur, int64_t base, int64_t nvalid) {
                mbar_wait(&empty[s], ph ^ 1u);
                const KT& T = tab.t[cur];
                                K c;   // DHP: graph-replayed step (device block); see step_kernel
                if constexpr (DHP) c = dhp->g[hp_of(T)];
                else c = hp.g[hp_of(T)];
                const uint32_t nvec = uint32_t(nvalid) & ~(kGran - 1u);
                const bool need_m = Op::reads_m(c);
                uint32_t bytes = nvec * (2u + RB + GB);
                if (need_m) bytes += nvec * 4u;
                if constexpr (Op::kHasV) bytes += nvec * 4u;
                unsigned char* st = ring + size_t(s) * SB;
                desc[s] = StageDesc{base, cur, int32_t(nvalid)};
                mbar_arrive_expect_tx(&full[s], bytes);
                if (nvec) {
                    bulk_g2s(st, static_cast<const uint16_t*>(T.value) + base, nvec * 2u, &full[s], pol);
                    bulk_g2s(st + OFF_R, static_cast<const unsigned char*>(T.resid) + base * RB, nvec * RB, &full[s], pol);
                    bulk_g2s(st + OFF_G, static_cast<const unsigned char*>(T.grad) + base * GB, nvec * GB, &full[s], pol);
                    if (need_m) bulk_g2s(st + OFF_M, T.m + base, nvec * 4u, &full[s], pol);
                    if constexpr (Op::kHasV) bulk_g2s(st + OFF_V, T.v + base, nvec * 4u, &full[s], pol);
                }
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            };
            // schedule: tile k of the launch's tile space goes to CTA k mod G, so the grid sweeps
            // memory together (one contiguous window per stream at any moment).  A/B on one box:
            // contiguous per-CTA ranges balanced to 16 elements lost 5 %, a balanced sweep of
            // chunks < 1 tile lost 1-2 % on ResNet-50 (profiles/r01_ab7..10*.log).
            // first tile's tensor by binary search: a linear walk from tensor 0 costs the last
            // CTAs tens of dependent parameter-space loads before their first copy (ResNet-50's
            // first wave spans ~40 tensors); later tiles advance the cursor a few entries at a time
            // First tile's tensor by binary search: a linear walk from tensor 0 costs the last
            // CTAs tens of dependent parameter-space loads (~100+ cycles each) before their first
            // copy -- ResNet-50's first wave spans ~40 tensors; +1.8 % on that step.  Later tiles
            // advance the cursor a few entries at a time while the ring is full.  (A warp-parallel
            // ballot search gave the same on ResNet-50 and cost 0.6 % on the large sets:
            // profiles/r01_ab20_bsearch_start.log, r01_ab21_cursor.log.)
            int cur = first_tensor(tab, int(blockIdx.x));
            for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
                while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
                const int64_t base = int64_t(tile - tab.t[cur].tile0) * TE;
                issue(cur, base, tab.t[cur].n - base < TE ? tab.t[cur].n - base : TE);
#ifdef MPO_L2_PREFETCH
                {   // A/B knob: bulk-prefetch into L2 the tile this CTA loads MPO_L2_PREFETCH rounds later
                    const KT& T = tab.t[cur];
                    const int64_t fb = base + int64_t(MPO_L2_PREFETCH) * gridDim.x * TE;
                    if (fb + TE <= T.n) {
                        l2_prefetch(static_cast<const uint16_t*>(T.value) + fb, uint32_t(TE * 2));
                        l2_prefetch(static_cast<const unsigned char*>(T.resid) + fb * RB, uint32_t(TE * RB));
                        l2_prefetch(static_cast<const unsigned char*>(T.grad) + fb * GB, uint32_t(TE * GB));
                        l2_prefetch(T.m + fb, uint32_t(TE * 4));
                        if constexpr (Op::kHasV) l2_prefetch(T.v + fb, uint32_t(TE * 4));
                    }
                }
#endif
            }
            // end of schedule: a descriptor with no tensor, completed by a plain arrive
            mbar_wait(&empty[s], ph ^ 1u);
            desc[s] = StageDesc{0, -1, 0};
            mbar_arrive(&full[s]);
        }
        return;
    }

    // ---------------- consumers ----------------
    float coef = 1.0f;
    if constexpr (CLIP) coef = clip_coef(sumsq, max_norm);
    const int ct = threadIdx.x;   // 0 .. kCW*32-1, one unit per tile
    const int64_t el = int64_t(ct) * kUnitEl;
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
        mbar_wait(&full[s], ph);
        const StageDesc d = desc[s];
        if (d.cur < 0) break;
        const KT& T = tab.t[d.cur];
                        K c;   // DHP: graph-replayed step (device block); see step_kernel
                if constexpr (DHP) c = dhp->g[hp_of(T)];
                else c = hp.g[hp_of(T)];
        const int64_t base = d.base, nvalid = d.nvalid;
        const int64_t nvec = nvalid & ~int64_t(kGran - 1u);
        const bool full_unit = el + kUnitEl <= nvec;
        uint4 hv;
        ResidUnit<SF> rv;
        GradUnit<G> gu;
        float mm[8], vv[8];
        if (!full_unit) {
            hv = make_uint4(0u, 0u, 0u, 0u);
            rv.v = hv;
            gu.a = gu.b = hv;
#pragma unroll
            for (int k = 0; k < 8; ++k) mm[k] = vv[k] = 0.0f;
        } else {
            const unsigned char* st = ring + size_t(s) * SB;
            hv = *reinterpret_cast<const uint4*>(st + el * 2);
            if constexpr (RB == 2) {
                rv.v = *reinterpret_cast<const uint4*>(st + OFF_R + el * 2);
            } else {
                const uint2 r2 = *reinterpret_cast<const uint2*>(st + OFF_R + el);
                rv.v = make_uint4(r2.x, r2.y, 0u, 0u);
            }
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
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) mm[k] = 0.0f;
            }
            if constexpr (Op::kHasV) {
                const float4 a = *reinterpret_cast<const float4*>(st + OFF_V + el * 4);
                const float4 b = *reinterpret_cast<const float4*>(st + OFF_V + el * 4 + 16);
                vv[0] = a.x; vv[1] = a.y; vv[2] = a.z; vv[3] = a.w; vv[4] = b.x; vv[5] = b.y; vv[6] = b.z; vv[7] = b.w;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) vv[k] = 0.0f;
            }
        }
#ifdef MPO_RELEASE_EARLY
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#endif
        uint4 ho;
        ResidUnit<SF> ro;
#ifdef MPO_TRIVIAL_MATH
        // roofline experiment only: same bytes moved, trivial arithmetic (not a product path)
        if (full_unit) {
            ho = make_uint4(hv.x ^ gu.a.x, hv.y ^ gu.a.y, hv.z ^ gu.a.z, hv.w ^ gu.a.w);
            ro.v = make_uint4(rv.v.x + 1u, rv.v.y + 1u, rv.v.z + 1u, rv.v.w + 1u);
#pragma unroll
            for (int k = 0; k < 8; ++k) { mm[k] = mm[k] * 0.5f; vv[k] = vv[k] * 0.25f; }
        }
#else
        if (full_unit) process_unit<SF, G, Op, CLIP>(hv, rv, gu, mm, vv, c, coef, stream_of(T), base + el, ho, ro);
#endif
#if defined(MPO_BULK_ST)
        {
            // outputs over this thread's own inputs in the stage, then one lane of the warp
            // streams the warp's contiguous 256-element slice out with bulk copies
            unsigned char* st = ring + size_t(s) * SB;
            const bool wm = Op::writes_m(c);
            if (full_unit) {
                *reinterpret_cast<uint4*>(st + el * 2) = ho;
                if constexpr (RB == 2) *reinterpret_cast<uint4*>(st + OFF_R + el * 2) = ro.v;
                else *reinterpret_cast<uint2*>(st + OFF_R + el) = make_uint2(ro.v.x, ro.v.y);
                if (wm) {
                    *reinterpret_cast<float4*>(st + OFF_M + el * 4) = make_float4(mm[0], mm[1], mm[2], mm[3]);
                    *reinterpret_cast<float4*>(st + OFF_M + el * 4 + 16) = make_float4(mm[4], mm[5], mm[6], mm[7]);
                }
                if constexpr (Op::kHasV) {
                    *reinterpret_cast<float4*>(st + OFF_V + el * 4) = make_float4(vv[0], vv[1], vv[2], vv[3]);
                    *reinterpret_cast<float4*>(st + OFF_V + el * 4 + 16) = make_float4(vv[4], vv[5], vv[6], vv[7]);
                }
            }
            fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the bulk copies
            __syncwarp();
            if (lane == 0) {
                const int64_t w0 = int64_t(warp) * 32 * kUnitEl;            // warp slice start in the tile
                const int64_t nw = nvec - w0 < 32 * kUnitEl ? (nvec - w0 > 0 ? nvec - w0 : 0) : 32 * kUnitEl;
                if (nw > 0) {
                    const int64_t g0 = base + w0;
                    bulk_s2g(static_cast<uint16_t*>(T.value) + g0, st + w0 * 2, uint32_t(nw * 2));
                    bulk_s2g(static_cast<unsigned char*>(T.resid) + g0 * RB, st + OFF_R + w0 * RB, uint32_t(nw * RB));
                    if (wm) bulk_s2g(T.m + g0, st + OFF_M + w0 * 4, uint32_t(nw * 4));
                    if constexpr (Op::kHasV) bulk_s2g(T.v + g0, st + OFF_V + w0 * 4, uint32_t(nw * 4));
                    bulk_commit();
                    bulk_wait_read0();      // the stage's smem has been read: it may be refilled
                }
                mbar_arrive(&empty[s]);
            }
            if (!full_unit && nvec < nvalid && el <= nvec && nvec < el + kUnitEl)
                process_tail<SF, G, Op, CLIP>(T, base + nvec, base + nvalid, c, coef);
        }
#else
#ifndef MPO_RELEASE_EARLY
        // release after the arithmetic has consumed the registers (the proxy fence then waits on
        // nothing still pending from this stage)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
#endif
        if (full_unit) {
            store_unit<SF, Op>(T, base + el, ho, ro, mm, vv, Op::writes_m(c));
        } else if (nvec < nvalid && el <= nvec && nvec < el + kUnitEl) {
            process_tail<SF, G, Op, CLIP>(T, base + nvec, base + nvalid, c, coef);
        }
#endif
        if (++s == stages) {
            s = 0;
            ph ^= 1u;
        }
    }
#if defined(MPO_BULK_ST)
    if (lane == 0) bulk_wait0();   // every bulk store of this warp complete before the CTA exits
#endif
}

#ifdef MPO_ABI_TU
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
            const uint64_t pol = load_policy();
            int cur = 0, s = 0;
            uint32_t ph = 0;
            for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
                mbar_wait(&empty[s], ph ^ 1u);
                while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
                const KT& T = tab.t[cur];
                const int64_t base = int64_t(tile - T.tile0) * TE;
                const int64_t nvalid = T.n - base < TE ? T.n - base : TE;
                const uint32_t nvec = uint32_t(nvalid) & ~uint32_t(kUnitEl - 1);
                mbar_arrive_expect_tx(&full[s], nvec * GB);
                if (nvec)
                    bulk_g2s(ring + size_t(s) * SB, static_cast<const unsigned char*>(T.grad) + base * GB, nvec * GB,
                             &full[s], pol);
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    double acc8[kUnitEl];
#pragma unroll
    for (int k = 0; k < kUnitEl; ++k) acc8[k] = 0.0;
    const int64_t el = int64_t(threadIdx.x) * kUnitEl;
    int cur = 0, s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < tab.ntiles; tile += gridDim.x) {
        while (cur + 1 < tab.nt && tile >= tab.t[cur + 1].tile0) ++cur;
        const KT& T = tab.t[cur];
        const float gs = gsc.g[hp_of(T)];
        const int64_t base = int64_t(tile - T.tile0) * TE;
        const int64_t nvalid = T.n - base < TE ? T.n - base : TE;
        const int64_t nvec = nvalid & ~int64_t(kUnitEl - 1);
        mbar_wait(&full[s], ph);
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
        if (++s == stages) {
            s = 0;
            ph ^= 1u;
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

#endif  // MPO_ABI_TU

// ------------------------------------------------------------------------------------------
// G6: the sharded step fused with its collectives over NVLink SHARP.
// Each rank's threads read the SUM of all ranks' 16-bit gradients of their shard with one
// multimem.ld_reduce per 8 elements (the NVSwitch reduces in fp32 and rounds once to 16 bits),
// update value/residual/state exactly like the multi-tensor step, and write the new 16-bit values
// to every rank's replica with multimem.st -- reduce-scatter, update and all-gather in one pass,
// with no intermediate reduced-gradient buffer in HBM.  The caller orders the kernel after every
// rank's backward (grads written) and before any rank's next use of the values (barriers).
// ------------------------------------------------------------------------------------------
template <int B>
__device__ __forceinline__ uint4 multimem_ld_reduce_v4(const void* mc) {
    uint4 r;
    if constexpr (B == kBF16) {
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(mc)
                     : "memory");
    } else {
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(mc)
                     : "memory");
    }
    return r;
}

__device__ __forceinline__ void multimem_st_v4(void* mc, const uint4& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// The kernel reaches the multicast object through an access policy: NvlsMulticast issues the
// real multimem instructions; NvlsEmulated (validation on one device, where no multicast team
// can be created) performs the same two operations with ordinary loads/stores over the ranks'
// unicast buffers -- the sum of every rank's 8 gradients in fp32 in rank order, rounded once to
// the 16-bit format (RNE, canonical NaN), which is what ld_reduce.add.acc::f32 returns whenever
// the fp32 sum does not depend on the order (exact-sum inputs), and a store into every replica.
// Everything else in the kernel (indexing, state streams, update, re-split, fences) is shared.
template <int B>
struct NvlsMulticast {
    static constexpr bool kMulticast = true;
    uint16_t* value_mc;
    const uint16_t* grad_mc;
    __device__ __forceinline__ uint4 grad_sum(int64_t i) const { return multimem_ld_reduce_v4<B>(grad_mc + i); }
    __device__ __forceinline__ void store_value(int64_t i, const uint4& h) const { multimem_st_v4(value_mc + i, h); }
};

constexpr int kMaxPeers = 8;
struct Peers {
    const uint16_t* g[kMaxPeers];
    uint16_t* v[kMaxPeers];
};

template <int B>
struct NvlsEmulated {
    static constexpr bool kMulticast = false;
    Peers P;
    int world;
    __device__ __forceinline__ uint4 grad_sum(int64_t i) const {
        float sum[8];
        GradUnit<B> u;
        u.a = ldv(P.g[0] + i);
#pragma unroll
        for (int j = 0; j < 8; ++j) sum[j] = grad_at<B>(u, j);
        for (int k = 1; k < world; ++k) {
            u.a = ldv(P.g[k] + i);
#pragma unroll
            for (int j = 0; j < 8; ++j) sum[j] = sum[j] + grad_at<B>(u, j);
        }
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t h = round2<B>(sum[2 * j], sum[2 * j + 1]);
            if (sum[2 * j] != sum[2 * j]) h = (h & 0xFFFF0000u) | 0x7FFFu;
            if (sum[2 * j + 1] != sum[2 * j + 1]) h = (h & 0x0000FFFFu) | 0x7FFF0000u;
            w[j] = h;
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
    __device__ __forceinline__ void store_value(int64_t i, const uint4& h) const {
        for (int k = 0; k < world; ++k) stv(P.v[k] + i, h);
    }
};

template <int SF, class Op, class MC>
__global__ void __launch_bounds__(kThreads) nvls_step_kernel(const __grid_constant__ MC mc,
                                                             const uint16_t* __restrict__ value_uc, void* resid,
                                                             float* __restrict__ m, float* __restrict__ v,
                                                             int64_t shard_base, int64_t n, uint32_t stream,
                                                             const __grid_constant__ typename Op::K c) {
    constexpr int B = Fmt<SF>::base;
    const bool need_m = Op::reads_m(c), has_m = Op::writes_m(c);
    const int64_t nunits = n / kUnitEl;
    // kUnroll units per thread per round, every load of the round (the reduced gradients through
    // the switch included) in flight before any arithmetic: a multimem round trip is far longer
    // than an HBM load, so one unit at a time left the kernel latency-bound (ncu on the emulated
    // form: long_scoreboard 61 % of stalls, 52 % of DRAM peak)
    const int64_t per_round = int64_t(gridDim.x) * kThreads * kUnroll;
    for (int64_t u0 = int64_t(blockIdx.x) * kThreads * kUnroll; u0 < nunits; u0 += per_round) {
        GradUnit<B> gu[kUnroll];
        uint4 hv[kUnroll];
        ResidUnit<SF> rv[kUnroll];
        float4 m0[kUnroll], m1[kUnroll], v0[kUnroll], v1[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const int64_t u = u0 + int64_t(j) * kThreads + threadIdx.x;
            if (u < nunits) {
                const int64_t e = u * kUnitEl;                  // index inside the shard
                gu[j].a = mc.grad_sum(shard_base + e);          // reduce-scatter of this unit
                gu[j].b = gu[j].a;
                hv[j] = ldv(value_uc + shard_base + e);
                rv[j] = ld_resid<SF>(resid, e);
                if (need_m) {
                    m0[j] = ldf(m + e);
                    m1[j] = ldf(m + e + 4);
                } else {
                    m0[j] = m1[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                if constexpr (Op::kHasV) {
                    v0[j] = ldf(v + e);
                    v1[j] = ldf(v + e + 4);
                } else {
                    v0[j] = v1[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
            const int64_t u = u0 + int64_t(j) * kThreads + threadIdx.x;
            if (u < nunits) {
                const int64_t e = u * kUnitEl;
                float mm[8] = {m0[j].x, m0[j].y, m0[j].z, m0[j].w, m1[j].x, m1[j].y, m1[j].z, m1[j].w};
                float vv[8] = {v0[j].x, v0[j].y, v0[j].z, v0[j].w, v1[j].x, v1[j].y, v1[j].z, v1[j].w};
                uint4 ho;
                ResidUnit<SF> ro;
                // stochastic-rounding draws keyed like mpo_sharded_step: stream = rank, index in the shard
                process_unit<SF, B, Op, false>(hv[j], rv[j], gu[j], mm, vv, c, 1.0f, stream, e, ho, ro);
                mc.store_value(shard_base + e, ho);             // all-gather: every rank's replica
                st_resid<SF>(resid, e, ro);
                if (has_m) {
                    stf8(m + e, mm);
                }
                if constexpr (Op::kHasV) {
                    stf8(v + e, vv);
                }
            }
        }
    }
    // make the multicast stores visible system-wide, and ordered with later accesses through the
    // unicast alias of the same memory
    if constexpr (MC::kMulticast) asm volatile("fence.proxy.alias;" ::: "memory");
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// ---- sharded step fused with its collectives over NVLink peer memory (P2P loads / stores) ----
// Rank r owns elements [r*S, (r+1)*S) of the flat buffers.  Per 8-element unit of its shard the
// kernel loads the 16-bit gradients of EVERY rank straight from their buffers (NVLink P2P loads;
// rank order, fp32 accumulation: g = ((g_0 + g_1) + g_2) + ..., deterministic and one rounding
// path), runs the same reconstruct -> update -> re-split as every other entry point (the summed
// gradient enters as an fp32 gradient), keeps residual / m / v local, and stores the new 16-bit
// values into EVERY rank's replica (P2P stores).  This is the reduce-scatter + update +
// all-gather of mpo_sharded_step as one kernel: no collective launches, no reduced-gradient
// buffer, and the NVLink transfers overlap the arithmetic unit by unit.

template <int SF, class Op>
__global__ void __launch_bounds__(kThreads) p2p_step_kernel(const __grid_constant__ Peers P, int world, int rank,
                                                            void* resid, float* __restrict__ m, float* __restrict__ v,
                                                            int64_t shard_base, int64_t n,
                                                            const __grid_constant__ typename Op::K c) {
    constexpr int B = Fmt<SF>::base;
    const bool need_m = Op::reads_m(c), has_m = Op::writes_m(c);
    const int64_t nunits = n / kUnitEl;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t u = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; u < nunits; u += stride) {
        const int64_t e = u * kUnitEl;                      // index inside the shard
        uint4 gk[kMaxPeers];
#pragma unroll
        for (int k = 0; k < kMaxPeers; ++k)
            if (k < world) gk[k] = ldv(P.g[k] + shard_base + e);   // all loads in flight first
        float gsum[8];
        GradUnit<B> g0;
        g0.a = gk[0];
#pragma unroll
        for (int i = 0; i < 8; ++i) gsum[i] = grad_at<B>(g0, i);
#pragma unroll
        for (int k = 1; k < kMaxPeers; ++k) {
            if (k < world) {
                GradUnit<B> gx;
                gx.a = gk[k];
#pragma unroll
                for (int i = 0; i < 8; ++i) gsum[i] = gsum[i] + grad_at<B>(gx, i);
            }
        }
        GradUnit<kFP32> gu;
        gu.a = make_uint4(__float_as_uint(gsum[0]), __float_as_uint(gsum[1]), __float_as_uint(gsum[2]),
                          __float_as_uint(gsum[3]));
        gu.b = make_uint4(__float_as_uint(gsum[4]), __float_as_uint(gsum[5]), __float_as_uint(gsum[6]),
                          __float_as_uint(gsum[7]));
        const uint4 hv = ldv(P.v[rank] + shard_base + e);
        const ResidUnit<SF> rv = ld_resid<SF>(resid, e);
        float mm[8], vv[8];
        if (need_m) {
            const float4 a = ldf(m + e), b = ldf(m + e + 4);
            mm[0] = a.x; mm[1] = a.y; mm[2] = a.z; mm[3] = a.w; mm[4] = b.x; mm[5] = b.y; mm[6] = b.z; mm[7] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) mm[k] = 0.0f;
        }
        if constexpr (Op::kHasV) {
            const float4 a = ldf(v + e), b = ldf(v + e + 4);
            vv[0] = a.x; vv[1] = a.y; vv[2] = a.z; vv[3] = a.w; vv[4] = b.x; vv[5] = b.y; vv[6] = b.z; vv[7] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) vv[k] = 0.0f;
        }
        uint4 ho;
        ResidUnit<SF> ro;
        // stochastic-rounding draws keyed like mpo_sharded_step: stream = rank, index in the shard
        process_unit<SF, kFP32, Op, false>(hv, rv, gu, mm, vv, c, 1.0f, uint32_t(rank), e, ho, ro);
#pragma unroll
        for (int k = 0; k < kMaxPeers; ++k)
            if (k < world) stv(P.v[k] + shard_base + e, ho);    // every rank's replica
        st_resid<SF>(resid, e, ro);
        if (has_m) {
            stf8(m + e, mm);
        }
        if constexpr (Op::kHasV) {
            stf8(v + e, vv);
        }
    }
    // peer stores visible system-wide before the caller's cross-rank barrier
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// ---- the same fused P2P step on the bulk-copy pipeline (default; MPO_P2P_KERNEL=lsu selects the
// kernel above).  One producer warp streams, per 2048-element tile of this rank's shard, the local
// value replica / residual / m / v AND the 16-bit gradient slice of every rank (peer addresses)
// into a shared-memory stage with 1-D bulk copies; 8 consumer warps sum the ranks' gradients from
// the stage in rank order (R15), update, and store the new values into every replica (P2P
// stores) and residual / m / v locally.  Tiles are half the step kernel's so that 8 ranks'
// gradients still leave >= 2 stages in half an SM's shared memory (2 CTAs per SM).
constexpr int kP2PCW = 8;
constexpr int64_t kP2PTileEl = int64_t(kP2PCW) * 32 * kUnitEl;   // 2048 elements
constexpr int kP2PThreads = (kP2PCW + 1) * 32;
constexpr int kP2PSmem = 113 * 1024;                              // per CTA, 2 CTAs per SM

// Ragged tail of the shard (X8's 16-element bulk granule): element by element, peers read directly.
template <int SF, class Op>
__device__ __noinline__ void p2p_tail(const Peers& P, int world, int rank, void* resid, float* m, float* v,
                                      int64_t shard_base, int64_t lo, int64_t hi, const typename Op::K c) {
    using FM = Fmt<SF>;
    constexpr int B = FM::base;
    const bool need_m = Op::reads_m(c), has_m = Op::writes_m(c);
    for (int64_t i = lo; i < hi; ++i) {
        float g = grad_f32_16<B>(P.g[0][shard_base + i]);
        for (int k = 1; k < world; ++k) g = g + grad_f32_16<B>(P.g[k][shard_base + i]);
        g = g * c.gs;
        if (c.clip_on) g = clamp_grad(g, c.clipv);
        int32_t code;
        code = load_code<SF>(resid, i);
        float w = reconstruct1_s<SF>(P.v[rank][shard_base + i], code);
        float mi = need_m ? m[i] : 0.0f;
        float vi = 0.0f;
        if constexpr (Op::kHasV) vi = v[i];
        w = Op::apply(w, g, mi, vi, c);
        uint32_t h;
        split1_s<SF>(w, sr_draw(c.seed, uint32_t(rank), uint64_t(i)), h, code);
        for (int k = 0; k < world; ++k) P.v[k][shard_base + i] = static_cast<uint16_t>(h);
        if constexpr (FM::rbytes == 1) static_cast<int8_t*>(resid)[i] = static_cast<int8_t>(code);
        else static_cast<int16_t*>(resid)[i] = static_cast<int16_t>(code);
        if (has_m) m[i] = mi;
        if constexpr (Op::kHasV) v[i] = vi;
    }
}

template <int SF, class Op>
__global__ void __launch_bounds__(kP2PThreads, 2) p2p_tma_kernel(const __grid_constant__ Peers P, int world, int rank,
                                                                  void* resid, float* __restrict__ m,
                                                                  float* __restrict__ v, int64_t shard_base, int64_t n,
                                                                  const __grid_constant__ typename Op::K c, int stages) {
    constexpr int B = Fmt<SF>::base;
    constexpr int RB = Fmt<SF>::rbytes;
    constexpr int64_t TE = kP2PTileEl;
    constexpr uint32_t kGran = RB == 1 ? 16u : uint32_t(kUnitEl);
    // stage layout: [value TE*2 | resid TE*RB | grads of rank 0..world-1, TE*2 each | m TE*4 | v TE*4]
    const int OFF_R = int(TE) * 2, OFF_G = int(TE) * (2 + RB), OFF_M = OFF_G + int(TE) * 2 * world,
              OFF_V = OFF_M + int(TE) * 4;
    const int SB = OFF_V + (Op::kHasV ? int(TE) * 4 : 0);
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kMaxStages;
    unsigned char* ring = smem + kBarBytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool need_m = Op::reads_m(c), has_m = Op::writes_m(c);
    const int64_t ntiles = (n + TE - 1) / TE;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kP2PCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kP2PCW) {
        if (lane == 0) {
            const uint64_t pol = load_policy();
            int s = 0;
            uint32_t ph = 0;
            for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int64_t base = tile * TE;
                const int64_t nvalid = n - base < TE ? n - base : TE;
                const uint32_t nvec = uint32_t(nvalid) & ~(kGran - 1u);
                mbar_wait(&empty[s], ph ^ 1u);
                uint32_t bytes = nvec * (2u + RB + 2u * uint32_t(world));
                if (need_m) bytes += nvec * 4u;
                if constexpr (Op::kHasV) bytes += nvec * 4u;
                unsigned char* st = ring + size_t(s) * SB;
                mbar_arrive_expect_tx(&full[s], bytes);
                if (nvec) {
                    bulk_g2s(st, P.v[rank] + shard_base + base, nvec * 2u, &full[s], pol);
                    bulk_g2s(st + OFF_R, static_cast<const unsigned char*>(resid) + base * RB, nvec * RB, &full[s], pol);
                    for (int k = 0; k < world; ++k)
                        bulk_g2s(st + OFF_G + k * int(TE) * 2, P.g[k] + shard_base + base, nvec * 2u, &full[s], pol);
                    if (need_m) bulk_g2s(st + OFF_M, m + base, nvec * 4u, &full[s], pol);
                    if constexpr (Op::kHasV) bulk_g2s(st + OFF_V, v + base, nvec * 4u, &full[s], pol);
                }
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int64_t el = int64_t(threadIdx.x) * kUnitEl;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * TE;
        const int64_t nvalid = n - base < TE ? n - base : TE;
        const int64_t nvec = nvalid & ~int64_t(kGran - 1u);
        const bool full_unit = el + kUnitEl <= nvec;
        mbar_wait(&full[s], ph);
        uint4 hv = make_uint4(0u, 0u, 0u, 0u);
        ResidUnit<SF> rv;
        rv.v = hv;
        float gsum[8], mm[8], vv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) gsum[k] = mm[k] = vv[k] = 0.0f;
        if (full_unit) {
            const unsigned char* st = ring + size_t(s) * SB;
            hv = *reinterpret_cast<const uint4*>(st + el * 2);
            if constexpr (RB == 2) {
                rv.v = *reinterpret_cast<const uint4*>(st + OFF_R + el * 2);
            } else {
                const uint2 r2 = *reinterpret_cast<const uint2*>(st + OFF_R + el);
                rv.v = make_uint4(r2.x, r2.y, 0u, 0u);
            }
            // the ranks' gradients summed in fp32 in rank order (R15)
            GradUnit<B> g0;
            g0.a = *reinterpret_cast<const uint4*>(st + OFF_G + el * 2);
#pragma unroll
            for (int i = 0; i < 8; ++i) gsum[i] = grad_at<B>(g0, i);
            for (int k = 1; k < world; ++k) {
                GradUnit<B> gx;
                gx.a = *reinterpret_cast<const uint4*>(st + OFF_G + k * int(TE) * 2 + el * 2);
#pragma unroll
                for (int i = 0; i < 8; ++i) gsum[i] = gsum[i] + grad_at<B>(gx, i);
            }
            if (need_m) {
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
        uint4 ho;
        ResidUnit<SF> ro;
        if (full_unit) {
            GradUnit<kFP32> gu;
            gu.a = make_uint4(__float_as_uint(gsum[0]), __float_as_uint(gsum[1]), __float_as_uint(gsum[2]),
                              __float_as_uint(gsum[3]));
            gu.b = make_uint4(__float_as_uint(gsum[4]), __float_as_uint(gsum[5]), __float_as_uint(gsum[6]),
                              __float_as_uint(gsum[7]));
            // stochastic-rounding draws keyed like mpo_sharded_step: stream = rank, index in the shard
            process_unit<SF, kFP32, Op, false>(hv, rv, gu, mm, vv, c, 1.0f, uint32_t(rank), base + el, ho, ro);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (full_unit) {
            const int64_t e = base + el;
            for (int k = 0; k < world; ++k) stv(P.v[k] + shard_base + e, ho);   // every rank's replica
            st_resid<SF>(resid, e, ro);
            if (has_m) stf8(m + e, mm);
            if constexpr (Op::kHasV) stf8(v + e, vv);
        } else if (nvec < nvalid && el <= nvec && nvec < el + kUnitEl) {
            p2p_tail<SF, Op>(P, world, rank, resid, m, v, shard_base, base + nvec, base + nvalid, c);
        }
        if (++s == stages) {
            s = 0;
            ph ^= 1u;
        }
    }
    // peer stores visible system-wide before the caller's cross-rank barrier
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// Host launch templates
// ------------------------------------------------------------------------------------------
constexpr int kSmemBudget = (MPO_CTAS_PER_SM == 1 ? 227 * 1024 : (228 * 1024) / MPO_CTAS_PER_SM - 1024);

// once per kernel (a static per distinct kernel, whatever its function-pointer type)
template <auto KERN>
int resident_per_sm() {
    static const int v = resident_blocks(KERN);
    return v;
}
template <auto KERN, int SMEM>
cudaError_t dyn_smem_attr() {
    static const cudaError_t a = cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    return a;
}

template <int MAXT, int SF, int G, class Op, bool CLIP>
mpo_status launch_step_slice(const mpo_tensor* t, int lo, int hi, const HP<typename Op::K>& hp, bool one_hp,
                             const double* sumsq, double max_norm, int skip, cudaStream_t s) {
    const auto* dhp = static_cast<const HP<typename Op::K>*>(g_dev_hp);
    // A graph-replayed step (mpo_step_graphed) reads its hyper-parameters from the device block:
    // kernels of their own (DHP = true; a runtime select of the two banks held both in registers),
    // instantiated for the largest table only to bound the build
    if constexpr (MAXT != kBigT) {
        if (dhp) return launch_step_slice<kBigT, SF, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, skip, s);
    }
    Table<MAXT> tab;
    const int64_t tiles = fill_table(tab, t, lo, hi, one_hp);
    if (tiles == 0) return MPO_OK;
    if (tiles > INT32_MAX) return fail(MPO_EINVAL, "table slice too large");
    const int choice = step_kernel_choice();
    if (choice == 1 || (choice < 0 && tiles <= kLsuMaxTiles)) {
        constexpr auto k0 = step_kernel<MAXT, SF, G, Op, CLIP, false>;
        if constexpr (MAXT == kBigT) {
            constexpr auto k1 = step_kernel<MAXT, SF, G, Op, CLIP, true>;
            if (dhp) k1<<<unsigned(grid_for(tiles, resident_per_sm<k1>())), kThreads, 0, s>>>(tab, hp, dhp, sumsq, max_norm, skip);
            else k0<<<unsigned(grid_for(tiles, resident_per_sm<k0>())), kThreads, 0, s>>>(tab, hp, nullptr, sumsq, max_norm, skip);
        } else {
            k0<<<unsigned(grid_for(tiles, resident_per_sm<k0>())), kThreads, 0, s>>>(tab, hp, nullptr, sumsq, max_norm, skip);
        }
        ++g_launches;
        return check_launch("step_kernel");
    }
    const int64_t grid = grid_for(tiles, MPO_CTAS_PER_SM);
    constexpr int SB = stage_bytes<Fmt<SF>::rbytes, G, Op::kHasV>();
    constexpr int kFree = kSmemBudget - kBarBytes - kDescBytes;
    constexpr int stages = kFree / SB < kMaxStages ? kFree / SB : kMaxStages;
    static_assert(stages >= 2, "need at least two pipeline stages");
    constexpr int smem = kBarBytes + kDescBytes + stages * SB;
    cudaError_t attr;
    constexpr auto k0 = step_tma_kernel<MAXT, SF, G, Op, CLIP, false>;
    if constexpr (MAXT == kBigT) {
        constexpr auto k1 = step_tma_kernel<MAXT, SF, G, Op, CLIP, true>;
        if (dhp) {
            if ((attr = dyn_smem_attr<k1, smem>()) == cudaSuccess)
                k1<<<unsigned(grid), kTmaThreads, smem, s>>>(tab, hp, dhp, sumsq, max_norm, stages, skip);
        } else if ((attr = dyn_smem_attr<k0, smem>()) == cudaSuccess) {
            k0<<<unsigned(grid), kTmaThreads, smem, s>>>(tab, hp, nullptr, sumsq, max_norm, stages, skip);
        }
    } else if ((attr = dyn_smem_attr<k0, smem>()) == cudaSuccess) {
        k0<<<unsigned(grid), kTmaThreads, smem, s>>>(tab, hp, nullptr, sumsq, max_norm, stages, skip);
    }
    if (attr != cudaSuccess) return fail(MPO_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr));
    ++g_launches;
    return check_launch("step_tma_kernel");
}

template <int SF, int G, class Op, bool CLIP>
mpo_status launch_step(const mpo_tensor* t, int nt, const HP<typename Op::K>& hp, bool one_hp, const double* sumsq,
                       double max_norm, int skip, cudaStream_t s) {
    for (int lo = 0; lo < nt; lo += kBigT) {
        const int hi = lo + kBigT < nt ? lo + kBigT : nt;
        mpo_status st;
        if (hi - lo == 1) st = launch_step_slice<1, SF, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, skip, s);
        else if (hi - lo <= kMidT)
            st = launch_step_slice<kMidT, SF, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, skip, s);
        else st = launch_step_slice<kBigT, SF, G, Op, CLIP>(t, lo, hi, hp, one_hp, sumsq, max_norm, skip, s);
        if (st != MPO_OK) return st;
    }
    return MPO_OK;
}

// Entry points of one storage format, defined in mpo_inst.cu (compiled once per format).
template <int SF>
struct FormatOps {
    static mpo_status sgd(int gdt, const mpo_tensor* t, int nt, const HP<SgdK>& hp, bool one_hp, const double* sumsq,
                          int skip, cudaStream_t s);
    static mpo_status adam(int gdt, const mpo_tensor* t, int nt, const HP<AdamK>& hp, bool one_hp, const double* sumsq,
                           double max_norm, int skip, cudaStream_t s);
    static mpo_status split(const float* w, void* value, void* resid, int64_t n, uint64_t seed, uint32_t stream,
                            cudaStream_t s);
    static mpo_status reconstruct(const void* value, const void* resid, float* w, int64_t n, cudaStream_t s);
    // emu == nullptr: the multicast kernel on value_mc / grad_mc; otherwise the emulated access
    // over emu's `world` peer buffers (value_mc / grad_mc unused)
    static mpo_status nvls(int kind, void* value_mc, const void* value_uc, const void* grad_mc, void* resid, float* m,
                           float* v, int64_t shard_base, int64_t n, const SgdK* sk, const AdamK* ak,
                           const Peers* emu, int world, int rank, cudaStream_t s);
    static mpo_status p2p(int kind, const Peers& peers, int world, int rank, void* resid, float* m, float* v,
                          int64_t shard_base, int64_t n, const SgdK* sk, const AdamK* ak, cudaStream_t s);
};

}  // namespace mpo
