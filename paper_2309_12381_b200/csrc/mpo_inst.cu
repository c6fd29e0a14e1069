// mpo_inst.cu -- the kernels of ONE storage format (compiled once per format with -DMPO_SF=<code>,
// the code being the C ABI's mpo_dtype value: base | scheme << 4; see mpo_device.cuh Fmt).
#include "mpo_kernels.cuh"

#include <cstdlib>
#include <cstring>

#ifndef MPO_SF
#error "compile with -DMPO_SF=<storage format code>"
#endif

namespace mpo {

namespace {
constexpr int SF = MPO_SF;
constexpr int B = Fmt<SF>::base;
constexpr bool kAllGrads = Fmt<SF>::scheme == kRNE;   // other schemes: grads of the base dtype or fp32
constexpr int kOther = B == kFP16 ? kBF16 : kFP16;

template <class Op, bool CLIP>
mpo_status step_for(int gdt, const mpo_tensor* t, int nt, const HP<typename Op::K>& hp, bool one_hp,
                    const double* sumsq, double max_norm, int skip, cudaStream_t s) {
    if (gdt == B) return launch_step<SF, B, Op, CLIP>(t, nt, hp, one_hp, sumsq, max_norm, skip, s);
    if (gdt == kFP32) return launch_step<SF, kFP32, Op, CLIP>(t, nt, hp, one_hp, sumsq, max_norm, skip, s);
    if constexpr (kAllGrads) {
        if (gdt == kOther) return launch_step<SF, kOther, Op, CLIP>(t, nt, hp, one_hp, sumsq, max_norm, skip, s);
    }
    return fail(MPO_EDTYPE, "unsupported gradient dtype for this storage format");
}
}  // namespace

template <>
mpo_status FormatOps<SF>::sgd(int gdt, const mpo_tensor* t, int nt, const HP<SgdK>& hp, bool one_hp,
                              const double* sumsq, int skip, cudaStream_t s) {
    return step_for<SgdOp, false>(gdt, t, nt, hp, one_hp, sumsq, 0.0, skip, s);
}

template <>
mpo_status FormatOps<SF>::adam(int gdt, const mpo_tensor* t, int nt, const HP<AdamK>& hp, bool one_hp,
                               const double* sumsq, double max_norm, int skip, cudaStream_t s) {
    if (max_norm > 0.0) return step_for<AdamOp, true>(gdt, t, nt, hp, one_hp, sumsq, max_norm, skip, s);
    return step_for<AdamOp, false>(gdt, t, nt, hp, one_hp, sumsq, 0.0, skip, s);
}

template <>
mpo_status FormatOps<SF>::split(const float* w, void* value, void* resid, int64_t n, uint64_t seed, uint32_t stream,
                                cudaStream_t s) {
    const int64_t grid = grid_for((n / kUnitEl + kThreads - 1) / kThreads + 1, 8);
    split_kernel<SF><<<unsigned(grid), kThreads, 0, s>>>(w, static_cast<uint16_t*>(value), resid, n, seed, stream);
    ++g_launches;
    return check_launch("split_kernel");
}

template <>
mpo_status FormatOps<SF>::reconstruct(const void* value, const void* resid, float* w, int64_t n, cudaStream_t s) {
    const int64_t grid = grid_for((n / kUnitEl + kThreads - 1) / kThreads + 1, 8);
    reconstruct_kernel<SF><<<unsigned(grid), kThreads, 0, s>>>(static_cast<const uint16_t*>(value), resid, w, n);
    ++g_launches;
    return check_launch("reconstruct_kernel");
}

template <class Op, class MC>
static void launch_nvls(const MC& mc, const uint16_t* vu, void* resid, float* m, float* v, int64_t shard_base,
                        int64_t n, uint32_t stream, const typename Op::K& k, cudaStream_t s) {
    auto kern = nvls_step_kernel<SF, Op, MC>;
    static const int per_sm = resident_blocks(kern);   // persistent: one wave of resident CTAs
    const int64_t grid = grid_for((n / kUnitEl + kThreads * kUnroll - 1) / (kThreads * kUnroll), per_sm);
    kern<<<unsigned(grid), kThreads, 0, s>>>(mc, vu, resid, m, v, shard_base, n, stream, k);
}

template <>
mpo_status FormatOps<SF>::nvls(int kind, void* value_mc, const void* value_uc, const void* grad_mc, void* resid,
                               float* m, float* v, int64_t shard_base, int64_t n, const SgdK* sk, const AdamK* ak,
                               const Peers* emu, int world, int rank, cudaStream_t s) {
    constexpr int B = Fmt<SF>::base;
    const uint32_t st = uint32_t(rank);
    auto* vu = static_cast<const uint16_t*>(value_uc);
    if (emu) {
        const NvlsEmulated<B> mc{*emu, world};
        if (kind == MPO_ADAM) launch_nvls<AdamOp>(mc, vu, resid, m, v, shard_base, n, st, *ak, s);
        else launch_nvls<SgdOp>(mc, vu, resid, m, v, shard_base, n, st, *sk, s);
    } else {
        const NvlsMulticast<B> mc{static_cast<uint16_t*>(value_mc), static_cast<const uint16_t*>(grad_mc)};
        if (kind == MPO_ADAM) launch_nvls<AdamOp>(mc, vu, resid, m, v, shard_base, n, st, *ak, s);
        else launch_nvls<SgdOp>(mc, vu, resid, m, v, shard_base, n, st, *sk, s);
    }
    ++g_launches;
    return check_launch("nvls_step_kernel");
}

template <>
mpo_status FormatOps<SF>::p2p(int kind, const Peers& peers, int world, int rank, void* resid, float* m, float* v,
                              int64_t shard_base, int64_t n, const SgdK* sk, const AdamK* ak, cudaStream_t s) {
    const char* env = std::getenv("MPO_P2P_KERNEL");   // read per call: tests cover both kernels
    if (env && std::strcmp(env, "lsu") == 0) {   // per-thread 128-bit loads of every stream (round-1 kernel)
        const int64_t grid = grid_for((n / kUnitEl + kThreads - 1) / kThreads, 8);
        if (kind == MPO_ADAM)
            p2p_step_kernel<SF, AdamOp><<<unsigned(grid), kThreads, 0, s>>>(peers, world, rank, resid, m, v, shard_base,
                                                                             n, *ak);
        else
            p2p_step_kernel<SF, SgdOp><<<unsigned(grid), kThreads, 0, s>>>(peers, world, rank, resid, m, v, shard_base,
                                                                            n, *sk);
        ++g_launches;
        return check_launch("p2p_step_kernel");
    }
    // bulk-copy pipeline: stages of [value | resid | world grads | m | v] in 113 KB per CTA
    const bool adam = kind == MPO_ADAM;
    const int sb = int(kP2PTileEl) * (2 + Fmt<SF>::rbytes + 2 * world + 4 + (adam ? 4 : 0));
    int stages = (kP2PSmem - kBarBytes) / sb;
    stages = stages > kMaxStages ? kMaxStages : stages;
    if (stages < 2) return fail(MPO_EINVAL, "P2P step: too many ranks for the shared-memory stages");
    const int smem = kBarBytes + stages * sb;
    const int64_t tiles = (n + kP2PTileEl - 1) / kP2PTileEl;
    const int64_t grid = grid_for(tiles, 2);
    cudaError_t attr;
    if (adam) {
        static const cudaError_t a = cudaFuncSetAttribute(p2p_tma_kernel<SF, AdamOp>,
                                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kP2PSmem);
        attr = a;
    } else {
        static const cudaError_t a = cudaFuncSetAttribute(p2p_tma_kernel<SF, SgdOp>,
                                                          cudaFuncAttributeMaxDynamicSharedMemorySize, kP2PSmem);
        attr = a;
    }
    if (attr != cudaSuccess) return fail(MPO_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr));
    if (adam)
        p2p_tma_kernel<SF, AdamOp><<<unsigned(grid), kP2PThreads, smem, s>>>(peers, world, rank, resid, m, v,
                                                                             shard_base, n, *ak, stages);
    else
        p2p_tma_kernel<SF, SgdOp><<<unsigned(grid), kP2PThreads, smem, s>>>(peers, world, rank, resid, m, v,
                                                                            shard_base, n, *sk, stages);
    ++g_launches;
    return check_launch("p2p_tma_kernel");
}

}  // namespace mpo
