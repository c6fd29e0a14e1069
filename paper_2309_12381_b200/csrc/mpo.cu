// mpo.cu -- the C ABI (include/mpo.h) of the residual-compensated 16-bit optimizer step of
// arXiv 2309.12381: argument validation, host-side derivation of the kernel scalars (R7), the
// global-norm pre-pass (clipping), the NCCL sharded step and diagnostics.  The step kernels
// themselves live in mpo_kernels.cuh and are instantiated per storage format by mpo_inst.cu.
#include <cuda.h>   // driver types only: entry points are fetched with cudaGetDriverEntryPoint
#include <nccl.h>

#include <mutex>
#include <unordered_map>
#include <vector>

#define MPO_ABI_TU
#include "mpo_kernels.cuh"

#define MPO_API extern "C" __attribute__((visibility("default")))

namespace mpo {

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
thread_local const void* g_dev_hp = nullptr;
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

// Step-kernel choice per launch: the bulk-copy pipeline (step_tma_kernel) for large launches, the
// per-thread-load kernel (step_kernel) for launches of at most kLsuMaxTiles tiles, where the
// pipeline's fill and its one-CTA-per-SM grid dominate (device-only, single tensor: 2^20 elements
// 5.7 vs 6.8 us, 2^21 8.9 vs 10.6 us, equal at 2^22, TMA ahead from 2^23; profiles/r02_small_launch_graph.log).
// MPO_STEP_KERNEL=tma|lsu forces one (tests cover both; read at every launch).
int step_kernel_choice() {
    const char* e = std::getenv("MPO_STEP_KERNEL");
    if (e && std::strcmp(e, "lsu") == 0) return 1;
    if (e && std::strcmp(e, "tma") == 0) return 0;
    return -1;
}

bool finite(double x) { return std::isfinite(x); }

// storage formats (mpo_dtype codes) and their properties
bool is_value_format(int f) {
    return f == MPO_FP16 || f == MPO_BF16 || f == MPO_FP16_RTZ || f == MPO_BF16_RTZ || f == MPO_FP16_SR ||
           f == MPO_FP16_X8 || f == MPO_BF16_X8 || f == MPO_FP16_X8Z || f == MPO_BF16_X8Z;
}
int base_of(int f) { return f & 15; }
int resid_bytes(int f) { return ((f >> 4) == kX8 || (f >> 4) == kX8Z) ? 1 : 2; }

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
    c.fast_ok = !c.lerp_hi && c.bc2s >= 0x1p-60f && c.bc2s <= 1.0f && c.eps >= 0.0f && c.eps <= 0x1p59f;
    c._pad = 0;
    c.seed = h.seed;
    c.clip_on = h.clip_value > 0.0;
    c.clipv = float(h.clip_value);
    // v < (bc2s * 2^60)^2 keeps sqrt(v)/bc2s < 2^60, so s = that + eps < 2^61 (rounded down to a
    // float that is still <= the real bound)
    {
        const double vh = double(c.bc2s) * double(c.bc2s) * 0x1p120;
        float f = float(vh < 0x1p122 ? vh : 0x1p122);
        if (double(f) > vh) f = std::nextafter(f, 0.0f);
        c.vhi = f;
    }
    c._pad3 = 0;
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
    c.seed = h.seed;
    c.clip_on = h.clip_value > 0.0;
    c.clipv = float(h.clip_value);
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
        if (!finite(h.clip_value) || h.clip_value < 0.0)
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": clip_value must be finite and >= 0");
        if (h.clip_value > 0.0 && h.max_grad_norm > 0.0)
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": clip_value and max_grad_norm are exclusive");
        if ((h.skip_nonfinite != 0) != (hp[0].skip_nonfinite != 0))
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": skip_nonfinite differs from group 0");
        if ((h.norm_ready != 0) != (hp[0].norm_ready != 0))
            return fail(MPO_EINVAL, "adam group " + std::to_string(i) + ": norm_ready differs from group 0");
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
        if (!finite(h.clip_value) || h.clip_value < 0.0)
            return fail(MPO_EINVAL, "sgd group " + std::to_string(i) + ": clip_value must be finite and >= 0");
        if ((h.skip_nonfinite != 0) != (hp[0].skip_nonfinite != 0))
            return fail(MPO_EINVAL, "sgd group " + std::to_string(i) + ": skip_nonfinite differs from group 0");
        if ((h.norm_ready != 0) != (hp[0].norm_ready != 0))
            return fail(MPO_EINVAL, "sgd group " + std::to_string(i) + ": norm_ready differs from group 0");
    }
    return MPO_OK;
}

mpo_status check_dtypes(mpo_dtype vdt, mpo_dtype gdt) {
    if (!is_value_format(vdt))
        return fail(MPO_EDTYPE, "value dtype must be a storage format (MPO_FP16, MPO_BF16, or a variant)");
    if (gdt != MPO_FP16 && gdt != MPO_BF16 && gdt != MPO_FP32)
        return fail(MPO_EDTYPE, "grad dtype must be MPO_FP16, MPO_BF16 or MPO_FP32");
    if ((vdt >> 4) != kRNE && gdt != MPO_FP32 && gdt != base_of(vdt))
        return fail(MPO_EDTYPE, "variant storage formats take grads of their base dtype or fp32");
    return MPO_OK;
}

mpo_status check_table(const mpo_tensor* t, int32_t nt, int32_t nhp, bool adam, const mpo_sgd_hp* sgd) {
    if (nt < 0 || (nt > 0 && !t)) return fail(MPO_EINVAL, "bad tensor table");
    for (int i = 0; i < nt; ++i) {
        const mpo_tensor& x = t[i];
        // the message is built only on failure (this loop runs on every call, before the launch)
        auto who = [i] { return "tensor " + std::to_string(i) + ": "; };
        if (x.n < 0) return fail(MPO_EINVAL, who() + "negative size");
        if (x.hp < 0 || x.hp >= nhp) return fail(MPO_EINVAL, who() + "hyper-parameter group index out of range");
        if (x.sr_stream < 0 || x.sr_stream >= (1 << 27)) return fail(MPO_EINVAL, who() + "sr_stream out of range");
        if (x.n == 0) continue;
        const bool need_m = adam || (sgd && sgd[x.hp].momentum != 0.0);
        if (!x.value || !x.resid || !x.grad || (need_m && !x.m) || (adam && !x.v))
            return fail(MPO_EINVAL, who() + "NULL array");
        if (!aligned16(x.value) || !aligned16(x.resid) || !aligned16(x.grad) || (need_m && !aligned16(x.m)) ||
            (adam && !aligned16(x.v)))
            return fail(MPO_EALIGN, who() + "array base pointer not 16-byte aligned");
    }
    return MPO_OK;
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

template <int MAXT, int G>
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

// Sum of squares of the scaled grads of the whole table into norm_ws[0] (partials in norm_ws[1..]).
mpo_status table_sumsq(mpo_dtype gdt, const mpo_tensor* t, int nt, const float* gs_of_group, int nhp,
                       double* norm_ws, cudaStream_t s, double* accum = nullptr, int add_out = 0) {
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
        if (gdt == MPO_FP32) st = launch_sumsq<kBigT, kFP32>(t, lo, hi, gsc, partial + nparts, nb, s);
        else if (gdt == MPO_BF16) st = launch_sumsq<kBigT, kBF16>(t, lo, hi, gsc, partial + nparts, nb, s);
        else st = launch_sumsq<kBigT, kFP16>(t, lo, hi, gsc, partial + nparts, nb, s);
        if (st != MPO_OK) return st;
        nparts += nb;
        if (nt == 0) break;
    }
    sumsq_final_kernel<<<1, kThreads, 0, s>>>(partial, nparts, norm_ws, accum, add_out);
    ++g_launches;
    return check_launch("sumsq_final_kernel");
}

// ---- dispatch to the per-format translation units ----
#define MPO_FORMATS(X) X(MPO_FP16) X(MPO_BF16) X(MPO_FP16_RTZ) X(MPO_BF16_RTZ) X(MPO_FP16_SR) X(MPO_FP16_X8) X(MPO_BF16_X8) X(MPO_FP16_X8Z) X(MPO_BF16_X8Z)

mpo_status dispatch_sgd(int vdt, int gdt, const mpo_tensor* t, int nt, const HP<SgdK>& k, bool one_hp,
                        const double* sumsq, int skip, cudaStream_t s) {
#define X(F) if (vdt == F) return FormatOps<F>::sgd(gdt, t, nt, k, one_hp, sumsq, skip, s);
    MPO_FORMATS(X)
#undef X
    return fail(MPO_EDTYPE, "unsupported storage format");
}

mpo_status dispatch_adam(int vdt, int gdt, const mpo_tensor* t, int nt, const HP<AdamK>& k, bool one_hp,
                         const double* sumsq, double max_norm, int skip, cudaStream_t s) {
#define X(F) if (vdt == F) return FormatOps<F>::adam(gdt, t, nt, k, one_hp, sumsq, max_norm, skip, s);
    MPO_FORMATS(X)
#undef X
    return fail(MPO_EDTYPE, "unsupported storage format");
}

mpo_status dispatch_split(int vdt, const float* w, void* value, void* resid, int64_t n, uint64_t seed, uint32_t stream,
                          cudaStream_t s) {
#define X(F) if (vdt == F) return FormatOps<F>::split(w, value, resid, n, seed, stream, s);
    MPO_FORMATS(X)
#undef X
    return fail(MPO_EDTYPE, "unsupported storage format");
}

mpo_status dispatch_reconstruct(int vdt, const void* value, const void* resid, float* w, int64_t n, cudaStream_t s) {
#define X(F) if (vdt == F) return FormatOps<F>::reconstruct(value, resid, w, n, s);
    MPO_FORMATS(X)
#undef X
    return fail(MPO_EDTYPE, "unsupported storage format");
}

// Wrap an NCCL call.
#define MPO_NCCL(call)                                                                             \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess) return fail(MPO_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

ncclDataType_t nccl_dtype(mpo_dtype d) { return base_of(d) == MPO_BF16 ? ncclBfloat16 : ncclFloat16; }

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

MPO_API int64_t mpo_norm_ws_doubles(void) { return 2 + kNormBlocksMax; }

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

MPO_API mpo_status mpo_split(mpo_dtype vdt, const float* w, void* value, void* resid, int64_t n, uint64_t seed,
                             int32_t sr_stream, mpo_stream stream) {
    g_err.clear();
    if (!is_value_format(vdt)) return fail(MPO_EDTYPE, "value dtype must be a storage format");
    if (n < 0) return fail(MPO_EINVAL, "negative size");
    if (sr_stream < 0) return fail(MPO_EINVAL, "negative sr_stream");
    if (n == 0) return MPO_OK;
    if (!w || !value || !resid) return fail(MPO_EINVAL, "NULL array");
    if (!aligned16(w) || !aligned16(value) || !aligned16(resid)) return fail(MPO_EALIGN, "array not 16-byte aligned");
    return dispatch_split(vdt, w, value, resid, n, seed, uint32_t(sr_stream), static_cast<cudaStream_t>(stream));
}

MPO_API mpo_status mpo_reconstruct(mpo_dtype vdt, const void* value, const void* resid, float* w, int64_t n,
                                   mpo_stream stream) {
    g_err.clear();
    if (!is_value_format(vdt)) return fail(MPO_EDTYPE, "value dtype must be a storage format");
    if (n < 0) return fail(MPO_EINVAL, "negative size");
    if (n == 0) return MPO_OK;
    if (!w || !value || !resid) return fail(MPO_EINVAL, "NULL array");
    if (!aligned16(w) || !aligned16(value) || !aligned16(resid)) return fail(MPO_EALIGN, "array not 16-byte aligned");
    return dispatch_reconstruct(vdt, value, resid, w, n, static_cast<cudaStream_t>(stream));
}

// The norm pre-pass of a call when clipping or the found-inf skip needs it.
static mpo_status prepass(mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const float* gs, int32_t nhp,
                          double* norm_ws, cudaStream_t s, double* accum = nullptr) {
    if (!norm_ws) return fail(MPO_EINVAL, "clipping / skip_nonfinite need a norm workspace");
    return table_sumsq(gdt, t, nt, gs, nhp, norm_ws, s, accum);
}

static mpo_status sgd_common(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const mpo_sgd_hp* hp,
                             int32_t nhp, double* norm_ws, bool one_hp, cudaStream_t s, bool sumsq_ready,
                             double* accum = nullptr) {
    HP<SgdK> k;
    for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = i < nhp ? derive_sgd(hp[i]) : k.g[0];
    const int skip = hp[0].skip_nonfinite != 0;
    if (skip && !sumsq_ready && !hp[0].norm_ready) {
        float gs[MPO_MAX_HP_GROUPS];
        for (int i = 0; i < nhp; ++i) gs[i] = k.g[i].gs;
        mpo_status st = prepass(gdt, t, nt, gs, nhp, norm_ws, s, accum);
        if (st != MPO_OK) return st;
    }
    if (skip && !norm_ws) return fail(MPO_EINVAL, "skip_nonfinite needs a norm workspace");
    return dispatch_sgd(vdt, gdt, t, nt, k, one_hp, skip ? norm_ws : nullptr, skip, s);
}

MPO_API mpo_status mpo_sgd_step(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const mpo_sgd_hp* hp,
                                int32_t nhp, double* norm_ws, mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    if ((st = check_sgd_hp(hp, nhp)) != MPO_OK) return st;
    if ((st = check_table(t, nt, nhp, false, hp)) != MPO_OK) return st;
    return sgd_common(vdt, gdt, t, nt, hp, nhp, norm_ws, false, static_cast<cudaStream_t>(stream), false);
}

static mpo_status adam_common(mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const mpo_adam_hp* hp,
                              int32_t nhp, double* norm_ws, bool one_hp, cudaStream_t s, bool sumsq_ready,
                              double* accum = nullptr) {
    HP<AdamK> k;
    for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = i < nhp ? derive_adam(hp[i]) : k.g[0];
    const double max_norm = hp[0].max_grad_norm;
    const int skip = hp[0].skip_nonfinite != 0;
    const bool need = max_norm > 0.0 || skip;
    if (need && !sumsq_ready && !hp[0].norm_ready) {
        float gs[MPO_MAX_HP_GROUPS];
        for (int i = 0; i < nhp; ++i) gs[i] = k.g[i].gs;
        mpo_status st = prepass(gdt, t, nt, gs, nhp, norm_ws, s, accum);
        if (st != MPO_OK) return st;
    }
    if (need && !norm_ws) return fail(MPO_EINVAL, "clipping / skip_nonfinite need a norm workspace");
    return dispatch_adam(vdt, gdt, t, nt, k, one_hp, need ? norm_ws : nullptr, max_norm > 0.0 ? max_norm : 0.0, skip, s);
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

// The per-step block of mpo_step_graphed: the derived scalars of every group, then a 16-B slot whose
// first uint64 is the block's sequence number (written by mpo_hp_block_fill, echoed to the
// caller's acknowledgement word once the device copy has happened).
static size_t hp_part_bytes(mpo_optim kind) { return kind == MPO_ADAM ? sizeof(HP<AdamK>) : sizeof(HP<SgdK>); }

MPO_API int64_t mpo_hp_block_bytes(mpo_optim kind) { return int64_t(hp_part_bytes(kind) + 16); }

MPO_API mpo_status mpo_hp_block_fill(mpo_optim kind, const void* hp, int32_t nhp, uint64_t seq, void* host_block) {
    g_err.clear();
    mpo_status st;
    if (!hp || !host_block) return fail(MPO_EINVAL, "NULL hyper-parameters or block");
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, nhp)) != MPO_OK) return st;
        HP<AdamK> k;
        for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = i < nhp ? derive_adam(h[i]) : k.g[0];
        std::memcpy(host_block, &k, sizeof(k));
    } else if (kind == MPO_SGD) {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, nhp)) != MPO_OK) return st;
        HP<SgdK> k;
        for (int i = 0; i < MPO_MAX_HP_GROUPS; ++i) k.g[i] = i < nhp ? derive_sgd(h[i]) : k.g[0];
        std::memcpy(host_block, &k, sizeof(k));
    } else {
        return fail(MPO_EINVAL, "unknown optimizer kind");
    }
    std::memcpy(static_cast<unsigned char*>(host_block) + hp_part_bytes(kind), &seq, sizeof(seq));
    return MPO_OK;
}

// Echo the device copy's sequence number to the caller's (host-mapped) acknowledgement word: the
// host may refill the block once it reads back the sequence number it wrote.
__global__ void ack_kernel(const uint64_t* __restrict__ seq, volatile unsigned long long* ack) {
    *ack = static_cast<unsigned long long>(*seq);
    __threadfence_system();
}

MPO_API mpo_status mpo_step_graphed(mpo_optim kind, mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* t, int32_t nt,
                                    const void* hp, int32_t nhp, const void* host_block, void* dev_block,
                                    unsigned long long* ack, double* norm_ws, mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if (!host_block || !dev_block) return fail(MPO_EINVAL, "NULL hyper-parameter block");
    if (!aligned16(dev_block)) return fail(MPO_EALIGN, "device hyper-parameter block not 16-byte aligned");
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    if (kind != MPO_SGD && kind != MPO_ADAM) return fail(MPO_EINVAL, "unknown optimizer kind");
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, nhp)) != MPO_OK) return st;
        if ((st = check_table(t, nt, nhp, true, nullptr)) != MPO_OK) return st;
    } else {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, nhp)) != MPO_OK) return st;
        if ((st = check_table(t, nt, nhp, false, h)) != MPO_OK) return st;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the step's derived hyper-parameters travel host block -> device block in stream order, so a
    // CUDA graph that captured this call re-reads the host block (refilled by mpo_hp_block_fill)
    // every time it is replayed
    const cudaError_t ce = cudaMemcpyAsync(dev_block, host_block, size_t(mpo_hp_block_bytes(kind)),
                                           cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) return fail(MPO_ECUDA, std::string("cudaMemcpyAsync: ") + cudaGetErrorString(ce));
    if (ack) {
        ack_kernel<<<1, 1, 0, s>>>(reinterpret_cast<const uint64_t*>(static_cast<unsigned char*>(dev_block) +
                                                                     hp_part_bytes(kind)),
                                   ack);
        ++g_launches;
        if ((st = check_launch("ack_kernel")) != MPO_OK) return st;
    }
    g_dev_hp = dev_block;
    if (kind == MPO_ADAM)
        st = adam_common(vdt, gdt, t, nt, static_cast<const mpo_adam_hp*>(hp), nhp, norm_ws, false, s, false);
    else
        st = sgd_common(vdt, gdt, t, nt, static_cast<const mpo_sgd_hp*>(hp), nhp, norm_ws, false, s, false);
    g_dev_hp = nullptr;
    return st;
}

MPO_API mpo_status mpo_fused_backward_hook_step(mpo_optim kind, mpo_dtype vdt, mpo_dtype gdt, const mpo_tensor* one,
                                                const void* hp, double* norm_ws, mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if (!one || !hp) return fail(MPO_EINVAL, "NULL tensor or hyper-parameters");
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    mpo_tensor x = *one;
    x.hp = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* accum = norm_ws ? norm_ws + (1 + kNormBlocksMax) : nullptr;   // found-inf over the backward
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, 1)) != MPO_OK) return st;
        if (h->max_grad_norm > 0.0)
            return fail(MPO_EINVAL, "global-norm clipping is impossible in the fused backward hook (P:93, P:186)");
        if (h->norm_ready) return fail(MPO_EINVAL, "norm_ready is for multi-tensor calls only");
        if ((st = check_table(&x, 1, 1, true, nullptr)) != MPO_OK) return st;
        return adam_common(vdt, gdt, &x, 1, h, 1, norm_ws, true, s, false, accum);
    }
    if (kind == MPO_SGD) {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, 1)) != MPO_OK) return st;
        if (h->norm_ready) return fail(MPO_EINVAL, "norm_ready is for multi-tensor calls only");
        if ((st = check_table(&x, 1, 1, false, h)) != MPO_OK) return st;
        return sgd_common(vdt, gdt, &x, 1, h, 1, norm_ws, true, s, false, accum);
    }
    return fail(MPO_EINVAL, "unknown optimizer kind");
}

// Asynchronous error of a communicator (ncclInProgress = still initialising: healthy).
static mpo_status comm_status(ncclComm_t comm) {
    ncclResult_t async = ncclSuccess;
    const ncclResult_t r = ncclCommGetAsyncError(comm, &async);
    if (r != ncclSuccess) return fail(MPO_ENCCL, std::string("ncclCommGetAsyncError: ") + ncclGetErrorString(r));
    if (async != ncclSuccess && async != ncclInProgress) {
        const char* last = ncclGetLastError(comm);
        return fail(MPO_ENCCL, std::string("communicator failed asynchronously: ") + ncclGetErrorString(async) +
                                   (last && *last ? std::string(" (") + last + ")" : std::string()));
    }
    return MPO_OK;
}

MPO_API mpo_status mpo_comm_check(uintptr_t nccl_comm) {
    g_err.clear();
    if (!nccl_comm) return fail(MPO_EINVAL, "NULL NCCL communicator");
    return comm_status(reinterpret_cast<ncclComm_t>(nccl_comm));
}

MPO_API mpo_status mpo_grad_sumsq(mpo_dtype gdt, const mpo_tensor* t, int32_t nt, const double* grad_scale,
                                  int32_t nhp, double* norm_ws, int32_t accumulate, mpo_stream stream) {
    g_err.clear();
    if (gdt != MPO_FP16 && gdt != MPO_BF16 && gdt != MPO_FP32)
        return fail(MPO_EDTYPE, "grad dtype must be MPO_FP16, MPO_BF16 or MPO_FP32");
    if (!grad_scale || nhp < 1 || nhp > MPO_MAX_HP_GROUPS) return fail(MPO_EINVAL, "grad_scale group count out of range");
    if (!norm_ws) return fail(MPO_EINVAL, "NULL norm workspace");
    if (nt < 0 || (nt > 0 && !t)) return fail(MPO_EINVAL, "bad tensor table");
    float gs[MPO_MAX_HP_GROUPS];
    for (int i = 0; i < nhp; ++i) {
        if (!std::isfinite(grad_scale[i])) return fail(MPO_EINVAL, "non-finite grad_scale (group " + std::to_string(i) + ")");
        gs[i] = float(grad_scale[i]);
    }
    for (int i = 0; i < nt; ++i) {
        const std::string who = "tensor " + std::to_string(i) + ": ";
        if (t[i].n < 0) return fail(MPO_EINVAL, who + "negative size");
        if (t[i].hp < 0 || t[i].hp >= nhp) return fail(MPO_EINVAL, who + "hyper-parameter group index out of range");
        if (t[i].n == 0) continue;
        if (!t[i].grad) return fail(MPO_EINVAL, who + "NULL gradient");
        if (!aligned16(t[i].grad)) return fail(MPO_EALIGN, who + "gradient not 16-byte aligned");
    }
    return table_sumsq(gdt, t, nt, gs, nhp, norm_ws, static_cast<cudaStream_t>(stream), nullptr, accumulate != 0);
}

// The sharded step over the pieces (segments) of this rank's shard: RS -> [sumsq + AllReduce] ->
// one multi-tensor step over the pieces -> AG.
static mpo_status sharded_common(mpo_optim kind, uintptr_t nccl_comm, int32_t rank, int32_t world, mpo_dtype vdt,
                                 void* value_flat, void* grad_flat, void* resid_shard, float* m_shard, float* v_shard,
                                 int64_t n_total, const mpo_segment* seg, int32_t nseg, const void* hp, int32_t nhp,
                                 double* norm_ws, cudaStream_t s) {
    mpo_status st;
    if (!nccl_comm) return fail(MPO_EINVAL, "NULL NCCL communicator");
    if (world < 1 || rank < 0 || rank >= world) return fail(MPO_EINVAL, "bad rank / world");
    if (n_total < 0 || n_total % (int64_t(8) * world) != 0)
        return fail(MPO_EINVAL, "n_total must be a non-negative multiple of 8*world");
    if (!hp) return fail(MPO_EINVAL, "NULL hyper-parameters");
    const mpo_dtype gdt = mpo_dtype(is_value_format(vdt) ? base_of(vdt) : vdt);
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    if (kind != MPO_SGD && kind != MPO_ADAM) return fail(MPO_EINVAL, "unknown optimizer kind");
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, nhp)) != MPO_OK) return st;
        if (h[0].norm_ready) return fail(MPO_EINVAL, "norm_ready is for multi-tensor calls only");
        if ((h[0].max_grad_norm > 0.0 || h[0].skip_nonfinite) && !norm_ws)
            return fail(MPO_EINVAL, "clipping / skip_nonfinite need a norm workspace");
    } else {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, nhp)) != MPO_OK) return st;
        if (h[0].norm_ready) return fail(MPO_EINVAL, "norm_ready is for multi-tensor calls only");
        if (h[0].skip_nonfinite && !norm_ws) return fail(MPO_EINVAL, "skip_nonfinite needs a norm workspace");
    }
    if (n_total == 0) return MPO_OK;
    if (!value_flat || !grad_flat) return fail(MPO_EINVAL, "NULL flat buffer");
    if (!aligned16(value_flat) || !aligned16(grad_flat)) return fail(MPO_EALIGN, "flat buffer not 16-byte aligned");
    const int64_t shard = n_total / world;
    // the pieces of this rank's shard, as a table (each piece 16-B aligned in every array)
    if (!seg || nseg < 1) return fail(MPO_EINVAL, "need at least one segment");
    if (!resid_shard) return fail(MPO_EINVAL, "NULL residual shard");
    const int64_t gran = resid_bytes(vdt) == 1 ? 16 : 8;
    std::vector<mpo_tensor> tab(static_cast<size_t>(nseg));
    for (int i = 0; i < nseg; ++i) {
        const int64_t a = seg[i].start, b = i + 1 < nseg ? seg[i + 1].start : shard;
        const std::string who = "segment " + std::to_string(i) + ": ";
        if ((i == 0 && a != 0) || a < 0 || b <= a || b > shard)
            return fail(MPO_EINVAL, who + "starts must begin at 0 and increase strictly inside the shard");
        if (a % gran != 0)
            return fail(MPO_EINVAL, who + "start must be a multiple of " + std::to_string(gran) + " elements");
        mpo_tensor& x = tab[size_t(i)];
        x.value = static_cast<uint16_t*>(value_flat) + rank * shard + a;
        x.resid = static_cast<unsigned char*>(resid_shard) + a * resid_bytes(vdt);
        x.grad = static_cast<uint16_t*>(grad_flat) + rank * shard + a;
        x.m = m_shard ? m_shard + a : nullptr;
        x.v = v_shard ? v_shard + a : nullptr;
        x.n = b - a;
        x.hp = seg[i].hp;
        x.sr_stream = seg[i].sr_stream;
    }
    if (kind == MPO_ADAM) {
        if ((st = check_table(tab.data(), nseg, nhp, true, nullptr)) != MPO_OK) return st;
    } else {
        if ((st = check_table(tab.data(), nseg, nhp, false, static_cast<const mpo_sgd_hp*>(hp))) != MPO_OK) return st;
    }
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
    // a communicator that already failed asynchronously is reported instead of hanging
    if ((st = comm_status(comm)) != MPO_OK) return st;
    void* grad_shard = static_cast<uint16_t*>(grad_flat) + rank * shard;
    // 1. reduce-scatter of the 16-bit gradients (sum), in place: shard `rank` of grad_flat.  Issued
    //    at world 1 too: NCCL's single-rank path makes an in-place collective a no-op, and the call
    //    (arguments, communicator, stream) then runs on every one-GPU test
    MPO_NCCL(ncclReduceScatter(grad_flat, grad_shard, size_t(shard), nccl_dtype(vdt), ncclSum, comm, s));
    // 2. residual-compensated update of this rank's pieces
    //    (clipping / found-inf: the shard's sum of squares, all-reduced so every rank agrees)
    const bool need = kind == MPO_ADAM ? (static_cast<const mpo_adam_hp*>(hp)->max_grad_norm > 0.0 ||
                                          static_cast<const mpo_adam_hp*>(hp)->skip_nonfinite != 0)
                                       : static_cast<const mpo_sgd_hp*>(hp)->skip_nonfinite != 0;
    if (need) {
        float gs[MPO_MAX_HP_GROUPS];
        for (int i = 0; i < nhp; ++i)
            gs[i] = float(kind == MPO_ADAM ? static_cast<const mpo_adam_hp*>(hp)[i].grad_scale
                                           : static_cast<const mpo_sgd_hp*>(hp)[i].grad_scale);
        if ((st = prepass(gdt, tab.data(), nseg, gs, nhp, norm_ws, s)) != MPO_OK) return st;
        MPO_NCCL(ncclAllReduce(norm_ws, norm_ws, 1, ncclFloat64, ncclSum, comm, s));
    }
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = adam_common(vdt, gdt, tab.data(), nseg, h, nhp, norm_ws, false, s, true)) != MPO_OK) return st;
    } else {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = sgd_common(vdt, gdt, tab.data(), nseg, h, nhp, norm_ws, false, s, true)) != MPO_OK) return st;
    }
    // 3. all-gather of the 16-bit values only (residual and state never move); in place
    MPO_NCCL(ncclAllGather(static_cast<uint16_t*>(value_flat) + rank * shard, value_flat, size_t(shard),
                           nccl_dtype(vdt), comm, s));
    return MPO_OK;
}

MPO_API mpo_status mpo_sharded_step(mpo_optim kind, uintptr_t nccl_comm, int32_t rank, int32_t world, mpo_dtype vdt,
                                    void* value_flat, void* grad_flat, void* resid_shard, float* m_shard,
                                    float* v_shard, int64_t n_total, const void* hp, double* norm_ws,
                                    mpo_stream stream) {
    g_err.clear();
    const mpo_segment one{0, 0, rank};   // the shard's stochastic-rounding stream is its rank
    return sharded_common(kind, nccl_comm, rank, world, vdt, value_flat, grad_flat, resid_shard, m_shard, v_shard,
                          n_total, &one, 1, hp, 1, norm_ws, static_cast<cudaStream_t>(stream));
}

MPO_API mpo_status mpo_sharded_step_grouped(mpo_optim kind, uintptr_t nccl_comm, int32_t rank, int32_t world,
                                            mpo_dtype vdt, void* value_flat, void* grad_flat, void* resid_shard,
                                            float* m_shard, float* v_shard, int64_t n_total, const mpo_segment* seg,
                                            int32_t nseg, const void* hp, int32_t nhp, double* norm_ws,
                                            mpo_stream stream) {
    g_err.clear();
    return sharded_common(kind, nccl_comm, rank, world, vdt, value_flat, grad_flat, resid_shard, m_shard, v_shard,
                          n_total, seg, nseg, hp, nhp, norm_ws, static_cast<cudaStream_t>(stream));
}


MPO_API mpo_status mpo_p2p_sharded_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt,
                                        void* const* value_peers, const void* const* grad_peers, void* resid_shard,
                                        float* m_shard, float* v_shard, int64_t n_total, const void* hp,
                                        mpo_stream stream) {
    g_err.clear();
    mpo_status st;
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return fail(MPO_EINVAL, "bad rank / world (1 <= world <= 8)");
    if (n_total < 0 || n_total % (int64_t(8) * world) != 0)
        return fail(MPO_EINVAL, "n_total must be a non-negative multiple of 8*world");
    if (!hp) return fail(MPO_EINVAL, "NULL hyper-parameters");
    if (!is_value_format(vdt)) return fail(MPO_EDTYPE, "unsupported storage format");
    const mpo_dtype gdt = mpo_dtype(base_of(vdt));
    if ((st = check_dtypes(vdt, gdt)) != MPO_OK) return st;
    if (kind != MPO_SGD && kind != MPO_ADAM) return fail(MPO_EINVAL, "unknown optimizer kind");
    if (n_total == 0) return MPO_OK;
    if (!value_peers || !grad_peers) return fail(MPO_EINVAL, "NULL peer pointer array");
    Peers peers{};
    for (int k = 0; k < world; ++k) {
        if (!value_peers[k] || !grad_peers[k]) return fail(MPO_EINVAL, "NULL peer buffer (rank " + std::to_string(k) + ")");
        if (!aligned16(value_peers[k]) || !aligned16(grad_peers[k]))
            return fail(MPO_EALIGN, "peer buffer not 16-byte aligned (rank " + std::to_string(k) + ")");
        peers.g[k] = static_cast<const uint16_t*>(grad_peers[k]);
        peers.v[k] = static_cast<uint16_t*>(value_peers[k]);
    }
    const int64_t shard = n_total / world;
    mpo_tensor x;   // this rank's shard, for the common table validation
    x.value = static_cast<uint16_t*>(value_peers[rank]) + rank * shard;
    x.resid = resid_shard;
    x.grad = static_cast<const uint16_t*>(grad_peers[rank]) + rank * shard;
    x.m = m_shard;
    x.v = v_shard;
    x.n = shard;
    x.hp = 0;
    x.sr_stream = rank;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, 1)) != MPO_OK) return st;
        if (h->max_grad_norm > 0.0 || h->skip_nonfinite)
            return fail(MPO_EINVAL, "the P2P step has no norm pre-pass (max_grad_norm / skip_nonfinite)");
        if ((st = check_table(&x, 1, 1, true, nullptr)) != MPO_OK) return st;
        const AdamK k = derive_adam(*h);
#define X(F) \
    if (vdt == F) return FormatOps<F>::p2p(kind, peers, world, rank, resid_shard, m_shard, v_shard, rank * shard, shard, nullptr, &k, s);
        MPO_FORMATS(X)
#undef X
    } else {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, 1)) != MPO_OK) return st;
        if (h->skip_nonfinite) return fail(MPO_EINVAL, "the P2P step has no norm pre-pass (skip_nonfinite)");
        if ((st = check_table(&x, 1, 1, false, h)) != MPO_OK) return st;
        const SgdK k = derive_sgd(*h);
#define X(F) \
    if (vdt == F) return FormatOps<F>::p2p(kind, peers, world, rank, resid_shard, m_shard, nullptr, rank * shard, shard, &k, nullptr, s);
        MPO_FORMATS(X)
#undef X
    }
    return fail(MPO_EDTYPE, "unsupported storage format");
}

// ------------------------------------------------------------------------------------------
// NVLS (NVLink SHARP) fused sharded step and a single-device multicast allocator for tests
// ------------------------------------------------------------------------------------------
namespace {
// Shared validation + dispatch of the NVLS step: `emu` == nullptr launches the multicast kernel,
// otherwise its emulation over `world` peer buffers (mpo_nvls_emulated_step).
mpo_status nvls_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt, void* value_mc, const void* value_uc,
                     const void* grad_mc, const Peers* emu, void* resid_shard, float* m_shard, float* v_shard,
                     int64_t n_total, const void* hp, cudaStream_t s) {
    mpo_status st;
    if (world < 1 || rank < 0 || rank >= world || (emu && world > kMaxPeers)) return fail(MPO_EINVAL, "bad rank / world");
    if (n_total < 0 || n_total % (int64_t(8) * world) != 0)
        return fail(MPO_EINVAL, "n_total must be a non-negative multiple of 8*world");
    if (!is_value_format(vdt)) return fail(MPO_EDTYPE, "unsupported storage format");
    if ((st = check_dtypes(vdt, mpo_dtype(base_of(vdt)))) != MPO_OK) return st;
    if (!hp) return fail(MPO_EINVAL, "NULL hyper-parameters");
    if (n_total == 0) return MPO_OK;
    if ((!emu && (!value_mc || !grad_mc)) || !value_uc || !resid_shard) return fail(MPO_EINVAL, "NULL buffer");
    if ((!emu && (!aligned16(value_mc) || !aligned16(grad_mc))) || !aligned16(value_uc) || !aligned16(resid_shard))
        return fail(MPO_EALIGN, "buffer not 16-byte aligned");
    const int64_t shard = n_total / world;
    if (kind == MPO_ADAM) {
        const mpo_adam_hp* h = static_cast<const mpo_adam_hp*>(hp);
        if ((st = check_adam_hp(h, 1)) != MPO_OK) return st;
        if (h->max_grad_norm > 0.0 || h->skip_nonfinite)
            return fail(MPO_EINVAL, "the NVLS step has no norm pre-pass (max_grad_norm / skip_nonfinite)");
        if (!m_shard || !v_shard || !aligned16(m_shard) || !aligned16(v_shard))
            return fail(MPO_EALIGN, "m/v shards must be non-NULL and 16-byte aligned");
        const AdamK k = derive_adam(*h);
#define X(F)                                                                                                    \
    if (vdt == F)                                                                                               \
        return FormatOps<F>::nvls(kind, value_mc, value_uc, grad_mc, resid_shard, m_shard, v_shard, rank * shard, \
                                  shard, nullptr, &k, emu, world, rank, s);
        MPO_FORMATS(X)
#undef X
    }
    if (kind == MPO_SGD) {
        const mpo_sgd_hp* h = static_cast<const mpo_sgd_hp*>(hp);
        if ((st = check_sgd_hp(h, 1)) != MPO_OK) return st;
        if (h->skip_nonfinite) return fail(MPO_EINVAL, "the NVLS step has no norm pre-pass (skip_nonfinite)");
        if (h->momentum != 0.0 && (!m_shard || !aligned16(m_shard)))
            return fail(MPO_EALIGN, "momentum shard must be non-NULL and 16-byte aligned");
        const SgdK k = derive_sgd(*h);
#define X(F)                                                                                                    \
    if (vdt == F)                                                                                               \
        return FormatOps<F>::nvls(kind, value_mc, value_uc, grad_mc, resid_shard, m_shard, nullptr, rank * shard, \
                                  shard, &k, nullptr, emu, world, rank, s);
        MPO_FORMATS(X)
#undef X
    }
    return fail(MPO_EINVAL, "unknown optimizer kind");
}
}  // namespace

MPO_API mpo_status mpo_nvls_sharded_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt, void* value_mc,
                                         const void* value_uc, const void* grad_mc, void* resid_shard, float* m_shard,
                                         float* v_shard, int64_t n_total, const void* hp, mpo_stream stream) {
    g_err.clear();
    return nvls_step(kind, rank, world, vdt, value_mc, value_uc, grad_mc, nullptr, resid_shard, m_shard, v_shard,
                     n_total, hp, static_cast<cudaStream_t>(stream));
}

MPO_API mpo_status mpo_nvls_emulated_step(mpo_optim kind, int32_t rank, int32_t world, mpo_dtype vdt,
                                          void* const* value_peers, const void* const* grad_peers, void* resid_shard,
                                          float* m_shard, float* v_shard, int64_t n_total, const void* hp,
                                          mpo_stream stream) {
    g_err.clear();
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return fail(MPO_EINVAL, "bad rank / world (1 <= world <= 8)");
    if (!value_peers || !grad_peers) return fail(MPO_EINVAL, "NULL peer pointer array");
    Peers peers{};
    for (int k = 0; k < world; ++k) {
        if (!value_peers[k] || !grad_peers[k]) return fail(MPO_EINVAL, "NULL peer buffer (rank " + std::to_string(k) + ")");
        if (!aligned16(value_peers[k]) || !aligned16(grad_peers[k]))
            return fail(MPO_EALIGN, "peer buffer not 16-byte aligned (rank " + std::to_string(k) + ")");
        peers.g[k] = static_cast<const uint16_t*>(grad_peers[k]);
        peers.v[k] = static_cast<uint16_t*>(value_peers[k]);
    }
    return nvls_step(kind, rank, world, vdt, nullptr, value_peers[rank], nullptr, &peers, resid_shard, m_shard,
                     v_shard, n_total, hp, static_cast<cudaStream_t>(stream));
}

namespace {
struct McAlloc {
    CUmemGenericAllocationHandle mem, mc;
    size_t size;
};
std::mutex g_mc_mu;
std::unordered_map<uintptr_t, McAlloc> g_mc;

template <class F>
F driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<F>(p);
}
}  // namespace

#define MPO_CU(call, what)                                                                                 \
    do {                                                                                                   \
        CUresult r_ = (call);                                                                              \
        if (r_ != CUDA_SUCCESS) return fail(MPO_ECUDA, std::string(what) + " failed: CUresult " + std::to_string(int(r_))); \
    } while (0)

MPO_API mpo_status mpo_nvls_alloc_local(int64_t bytes, void** uc_ptr, void** mc_ptr, int64_t* mapped_bytes) {
    g_err.clear();
    if (bytes <= 0 || !uc_ptr || !mc_ptr || !mapped_bytes) return fail(MPO_EINVAL, "bad arguments");
    auto pGet = driver_fn<CUresult (*)(CUdevice*, int)>("cuDeviceGet");
    auto pGran = driver_fn<CUresult (*)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags)>(
        "cuMulticastGetGranularity");
    auto pMcCreate = driver_fn<CUresult (*)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*)>(
        "cuMulticastCreate");
    auto pMcAdd = driver_fn<CUresult (*)(CUmemGenericAllocationHandle, CUdevice)>("cuMulticastAddDevice");
    auto pCreate = driver_fn<CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                                          unsigned long long)>("cuMemCreate");
    auto pBind = driver_fn<CUresult (*)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                                        size_t, unsigned long long)>("cuMulticastBindMem");
    auto pReserve = driver_fn<CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long)>(
        "cuMemAddressReserve");
    auto pMap = driver_fn<CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long)>(
        "cuMemMap");
    auto pAccess = driver_fn<CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t)>("cuMemSetAccess");
    if (!pGet || !pGran || !pMcCreate || !pMcAdd || !pCreate || !pBind || !pReserve || !pMap || !pAccess)
        return fail(MPO_ECUDA, "driver entry points for multicast are unavailable");
    int devi = 0;
    if (cudaGetDevice(&devi) != cudaSuccess) return check_launch("cudaGetDevice");
    CUdevice dev;
    MPO_CU(pGet(&dev, devi), "cuDeviceGet");
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.size = size_t(bytes);
    size_t gran = 0;
    McAlloc a;
    // the driver may require an exportable handle type on the multicast object: try the POSIX FD,
    // fabric and no-export variants in turn
    const unsigned long long kinds[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC, 0};
    CUresult last = CUDA_ERROR_UNKNOWN;
    size_t size = 0;
    unsigned long long chosen = 0;
    std::string tried;
    const CUmulticastGranularity_flags grans[2] = {CU_MULTICAST_GRANULARITY_MINIMUM, CU_MULTICAST_GRANULARITY_RECOMMENDED};
    for (unsigned long long hk : kinds) {
        for (CUmulticastGranularity_flags gf : grans) {
            mp.handleTypes = hk;
            mp.size = size_t(bytes);
            const CUresult gr = pGran(&gran, &mp, gf);
            if (gr != CUDA_SUCCESS) {
                tried += " [handle " + std::to_string(hk) + " gran " + std::to_string(int(gf)) + ": granularity " +
                         std::to_string(int(gr)) + "]";
                continue;
            }
            size = (size_t(bytes) + gran - 1) / gran * gran;
            mp.size = size;
            last = pMcCreate(&a.mc, &mp);
            tried += " [handle " + std::to_string(hk) + " gran " + std::to_string(gran) + ": create " +
                     std::to_string(int(last)) + "]";
            if (last == CUDA_SUCCESS) {
                chosen = hk;
                break;
            }
        }
        if (last == CUDA_SUCCESS) break;
    }
    if (last != CUDA_SUCCESS) return fail(MPO_ECUDA, "cuMulticastCreate failed:" + tried);
    a.size = size;
    MPO_CU(pMcAdd(a.mc, dev), "cuMulticastAddDevice");
    CUmemAllocationProp ap = {};
    ap.requestedHandleTypes = CUmemAllocationHandleType(chosen);
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = devi;
    MPO_CU(pCreate(&a.mem, size, &ap, 0), "cuMemCreate");
    MPO_CU(pBind(a.mc, 0, a.mem, 0, size, 0), "cuMulticastBindMem");
    CUdeviceptr uc = 0, mc = 0;
    MPO_CU(pReserve(&uc, size, gran, 0, 0), "cuMemAddressReserve(uc)");
    MPO_CU(pMap(uc, size, 0, a.mem, 0), "cuMemMap(uc)");
    MPO_CU(pReserve(&mc, size, gran, 0, 0), "cuMemAddressReserve(mc)");
    MPO_CU(pMap(mc, size, 0, a.mc, 0), "cuMemMap(mc)");
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = devi;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    MPO_CU(pAccess(uc, size, &ad, 1), "cuMemSetAccess(uc)");
    MPO_CU(pAccess(mc, size, &ad, 1), "cuMemSetAccess(mc)");
    {
        std::lock_guard<std::mutex> lk(g_mc_mu);
        g_mc[uintptr_t(uc)] = a;
    }
    *uc_ptr = reinterpret_cast<void*>(uc);
    *mc_ptr = reinterpret_cast<void*>(mc);
    *mapped_bytes = int64_t(size);
    return MPO_OK;
}

MPO_API mpo_status mpo_nvls_free_local(void* uc_ptr, void* mc_ptr, int64_t mapped_bytes) {
    g_err.clear();
    McAlloc a;
    {
        std::lock_guard<std::mutex> lk(g_mc_mu);
        auto it = g_mc.find(uintptr_t(uc_ptr));
        if (it == g_mc.end()) return fail(MPO_EINVAL, "not an mpo_nvls_alloc_local buffer");
        a = it->second;
        g_mc.erase(it);
    }
    auto pUnmap = driver_fn<CUresult (*)(CUdeviceptr, size_t)>("cuMemUnmap");
    auto pFree = driver_fn<CUresult (*)(CUdeviceptr, size_t)>("cuMemAddressFree");
    auto pRelease = driver_fn<CUresult (*)(CUmemGenericAllocationHandle)>("cuMemRelease");
    if (!pUnmap || !pFree || !pRelease) return fail(MPO_ECUDA, "driver entry points unavailable");
    if (cudaDeviceSynchronize() != cudaSuccess) return check_launch("cudaDeviceSynchronize");
    MPO_CU(pUnmap(CUdeviceptr(mc_ptr), a.size), "cuMemUnmap(mc)");
    MPO_CU(pUnmap(CUdeviceptr(uc_ptr), a.size), "cuMemUnmap(uc)");
    MPO_CU(pFree(CUdeviceptr(mc_ptr), a.size), "cuMemAddressFree(mc)");
    MPO_CU(pFree(CUdeviceptr(uc_ptr), a.size), "cuMemAddressFree(uc)");
    MPO_CU(pRelease(a.mc), "cuMemRelease(mc)");
    MPO_CU(pRelease(a.mem), "cuMemRelease(mem)");
    (void)mapped_bytes;
    return MPO_OK;
}
