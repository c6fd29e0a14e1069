// Micro-benchmark (sm_100a): what HBM rate does the Adam step's access PATTERN allow, independent
// of the step kernel's pipeline and arithmetic?  Streams of the LLaMA-7B-sized step (n elements):
// value u16, resid u16, grad u16 (read), m f32, v f32 (read), value / resid / m / v written back
// in place -- 26 B/element -- against a plain copy and single-direction sweeps.  Simple grid-stride
// per-thread 128-bit kernels (8 elements per thread per unit, like the step), trivial arithmetic,
// several grid sizes.  GB/s = algorithmic bytes / best-of-5 CUDA-event time.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint4 ld(const void* p) { return __ldcs(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ uint4 ldn(const void* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void st(void* p, uint4 x) { *reinterpret_cast<uint4*>(p) = x; }

// plain copy a -> b (16-bit elements), 8 per unit
__global__ void copy_k(const uint16_t* __restrict__ a, uint16_t* __restrict__ b, int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e < n; e += stride) st(b + e, ldn(a + e));
}
// in-place read-modify-write of one 16-bit stream
__global__ void rmw_k(uint16_t* __restrict__ a, int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e < n; e += stride) {
        uint4 x = ldn(a + e);
        x.x ^= 1u; x.y ^= 1u; x.z ^= 1u; x.w ^= 1u;
        st(a + e, x);
    }
}
// the Adam pattern: 5 reads, 4 in-place writes per 8-element unit (UNROLL units in flight)
template <int UNROLL>
__global__ void adam_pattern_k(uint16_t* __restrict__ h, uint16_t* __restrict__ r, const uint16_t* __restrict__ g,
                               float* __restrict__ m, float* __restrict__ v, int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8 * UNROLL;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x * 8 * UNROLL; base < n; base += stride) {
        uint4 H[UNROLL], R[UNROLL], G[UNROLL], M0[UNROLL], M1[UNROLL], V0[UNROLL], V1[UNROLL];
#pragma unroll
        for (int j = 0; j < UNROLL; ++j) {
            const int64_t e = base + (int64_t(j) * blockDim.x + threadIdx.x) * 8;
            if (e < n) {
                H[j] = ld(h + e); R[j] = ld(r + e); G[j] = ld(g + e);
                M0[j] = ld(m + e); M1[j] = ld(m + e + 4); V0[j] = ld(v + e); V1[j] = ld(v + e + 4);
            }
        }
#pragma unroll
        for (int j = 0; j < UNROLL; ++j) {
            const int64_t e = base + (int64_t(j) * blockDim.x + threadIdx.x) * 8;
            if (e < n) {
                H[j].x ^= G[j].x; R[j].y ^= G[j].y; M0[j].z ^= G[j].z; V1[j].w ^= G[j].w;
                st(h + e, H[j]); st(r + e, R[j]); st(m + e, M0[j]); st(m + e + 4, M1[j]); st(v + e, V0[j]); st(v + e + 4, V1[j]);
            }
        }
    }
}
// 5-stream read only (a checksum per thread to keep the loads live)
__global__ void read5_k(const uint16_t* __restrict__ h, const uint16_t* __restrict__ r, const uint16_t* __restrict__ g,
                        const float* __restrict__ m, const float* __restrict__ v, int64_t n, uint32_t* out) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    uint32_t acc = 0;
    for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e < n; e += stride) {
        const uint4 a = ld(h + e), b = ld(r + e), c = ld(g + e), d0 = ld(m + e), d1 = ld(m + e + 4), f0 = ld(v + e), f1 = ld(v + e + 4);
        acc ^= a.x ^ b.y ^ c.z ^ d0.w ^ d1.x ^ f0.y ^ f1.z;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
// 4-stream write only
__global__ void write4_k(uint16_t* __restrict__ h, uint16_t* __restrict__ r, float* __restrict__ m, float* __restrict__ v,
                         int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    const uint4 z = make_uint4(threadIdx.x, 1u, 2u, 3u);
    for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e < n; e += stride) {
        st(h + e, z); st(r + e, z); st(m + e, z); st(m + e + 4, z); st(v + e, z); st(v + e + 4, z);
    }
}


// the Adam pattern with every access warp-contiguous per instruction: thread t of a warp owns
// elements {4t..4t+3} and {128+4t..128+4t+3} of the warp's 256-element slice, so each 16-bit
// stream moves 8 B per thread (256 B per warp instruction) and each fp32 stream 16 B per thread
// (512 B per warp instruction): full sectors, no half-sector stores
__device__ __forceinline__ uint2 ld2(const void* p) { return __ldcs(reinterpret_cast<const uint2*>(p)); }
__device__ __forceinline__ void st2(void* p, uint2 x) { *reinterpret_cast<uint2*>(p) = x; }
template <bool CS>
__global__ void adam_pattern_coal_k(uint16_t* __restrict__ h, uint16_t* __restrict__ r, const uint16_t* __restrict__ g,
                                    float* __restrict__ m, float* __restrict__ v, int64_t n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    for (int64_t base = (int64_t(blockIdx.x) * (blockDim.x >> 5) + warp) * 256; base < n; base += stride) {
        const int64_t e0 = base + 4 * lane, e1 = e0 + 128;
        uint2 H0 = ld2(h + e0), H1 = ld2(h + e1), R0 = ld2(r + e0), R1 = ld2(r + e1), G0 = ld2(g + e0), G1 = ld2(g + e1);
        uint4 M0 = ld(m + e0), M1 = ld(m + e1), V0 = ld(v + e0), V1 = ld(v + e1);
        H0.x ^= G0.x; H1.y ^= G1.y; R0.x ^= G0.y; M0.z ^= G1.x; V1.w ^= G0.x;
        if (CS) {
            __stcs(reinterpret_cast<uint2*>(h + e0), H0); __stcs(reinterpret_cast<uint2*>(h + e1), H1);
            __stcs(reinterpret_cast<uint2*>(r + e0), R0); __stcs(reinterpret_cast<uint2*>(r + e1), R1);
            __stcs(reinterpret_cast<uint4*>(m + e0), M0); __stcs(reinterpret_cast<uint4*>(m + e1), M1);
            __stcs(reinterpret_cast<uint4*>(v + e0), V0); __stcs(reinterpret_cast<uint4*>(v + e1), V1);
        } else {
            st2(h + e0, H0); st2(h + e1, H1); st2(r + e0, R0); st2(r + e1, R1);
            st(m + e0, M0); st(m + e1, M1); st(v + e0, V0); st(v + e1, V1);
        }
    }
}
// 4-stream write only, warp-contiguous per instruction
__global__ void write4_coal_k(uint16_t* __restrict__ h, uint16_t* __restrict__ r, float* __restrict__ m,
                              float* __restrict__ v, int64_t n) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    const uint4 z = make_uint4(threadIdx.x, 1u, 2u, 3u);
    const uint2 z2 = make_uint2(threadIdx.x, 1u);
    for (int64_t base = (int64_t(blockIdx.x) * (blockDim.x >> 5) + warp) * 256; base < n; base += stride) {
        const int64_t e0 = base + 4 * lane, e1 = e0 + 128;
        st2(h + e0, z2); st2(h + e1, z2); st2(r + e0, z2); st2(r + e1, z2);
        st(m + e0, z); st(m + e1, z); st(v + e0, z); st(v + e1, z);
    }
}

// 256-bit per-thread stores of the fp32 streams (st.global.v8.b32: a whole sector per thread)
__device__ __forceinline__ void st8(void* p, uint4 a, uint4 b) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
                 "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w) : "memory");
}
__global__ void write4_v8_k(uint16_t* __restrict__ h, uint16_t* __restrict__ r, float* __restrict__ m, float* __restrict__ v,
                            int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    const uint4 z = make_uint4(threadIdx.x, 1u, 2u, 3u);
    for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e < n; e += stride) {
        st(h + e, z); st(r + e, z); st8(m + e, z, z); st8(v + e, z, z);
    }
}
__global__ void adam_pattern_v8_k(uint16_t* __restrict__ h, uint16_t* __restrict__ r, const uint16_t* __restrict__ g,
                                  float* __restrict__ m, float* __restrict__ v, int64_t n) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 8;
    for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e < n; e += stride) {
        uint4 H = ld(h + e), R = ld(r + e), G = ld(g + e), M0 = ld(m + e), M1 = ld(m + e + 4), V0 = ld(v + e), V1 = ld(v + e + 4);
        H.x ^= G.x; R.y ^= G.y; M0.z ^= G.z; V1.w ^= G.w;
        st(h + e, H); st(r + e, R); st8(m + e, M0, M1); st8(v + e, V0, V1);
    }
}

template <class F>
float best_ms(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f(); f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : (int64_t(1) << 30);   // elements (1 Gi: 26 GiB per Adam pass)
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint16_t *h, *r, *g, *c; float *m, *v; uint32_t* out;
    CK(cudaMalloc(&h, n * 2)); CK(cudaMalloc(&r, n * 2)); CK(cudaMalloc(&g, n * 2)); CK(cudaMalloc(&c, n * 2));
    CK(cudaMalloc(&m, n * 4)); CK(cudaMalloc(&v, n * 4)); CK(cudaMalloc(&out, 4));
    CK(cudaMemset(h, 1, n * 2)); CK(cudaMemset(r, 2, n * 2)); CK(cudaMemset(g, 3, n * 2)); CK(cudaMemset(c, 0, n * 2));
    CK(cudaMemset(m, 0, n * 4)); CK(cudaMemset(v, 0, n * 4));
    printf("{\"n\": %lld, \"sms\": %d}\n", (long long)n, sms);
    const int T = 256;
    for (int per_sm : {4, 8, 16}) {
        const int grid = sms * per_sm;
        float ms;
        ms = best_ms([&] { copy_k<<<grid, T>>>(h, c, n); });
        printf("{\"kernel\": \"copy 16-bit a->b\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 4.0 * n / ms / 1e6);
        ms = best_ms([&] { rmw_k<<<grid, T>>>(c, n); });
        printf("{\"kernel\": \"in-place rmw 1 stream\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 4.0 * n / ms / 1e6);
        ms = best_ms([&] { adam_pattern_k<1><<<grid, T>>>(h, r, g, m, v, n); });
        printf("{\"kernel\": \"adam pattern 5R+4W in place, unroll 1\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 26.0 * n / ms / 1e6);
        ms = best_ms([&] { adam_pattern_k<2><<<grid, T>>>(h, r, g, m, v, n); });
        printf("{\"kernel\": \"adam pattern 5R+4W in place, unroll 2\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 26.0 * n / ms / 1e6);
        ms = best_ms([&] { read5_k<<<grid, T>>>(h, r, g, m, v, n, out); });
        printf("{\"kernel\": \"5 streams read only\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 14.0 * n / ms / 1e6);
        ms = best_ms([&] { write4_k<<<grid, T>>>(h, r, m, v, n); });
        printf("{\"kernel\": \"4 streams write only\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 12.0 * n / ms / 1e6);
        ms = best_ms([&] { adam_pattern_coal_k<false><<<grid, T>>>(h, r, g, m, v, n); });
        printf("{\"kernel\": \"adam pattern 5R+4W in place, warp-contiguous accesses\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 26.0 * n / ms / 1e6);
        ms = best_ms([&] { adam_pattern_coal_k<true><<<grid, T>>>(h, r, g, m, v, n); });
        printf("{\"kernel\": \"adam pattern 5R+4W in place, warp-contiguous, streaming stores\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 26.0 * n / ms / 1e6);
        ms = best_ms([&] { write4_coal_k<<<grid, T>>>(h, r, m, v, n); });
        printf("{\"kernel\": \"4 streams write only, warp-contiguous\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 12.0 * n / ms / 1e6);
        ms = best_ms([&] { cudaMemsetAsync(h, 0, n * 2); cudaMemsetAsync(r, 0, n * 2); cudaMemsetAsync(m, 0, n * 4); cudaMemsetAsync(v, 0, n * 4); });
        printf("{\"kernel\": \"cudaMemsetAsync x4 (write only)\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 12.0 * n / ms / 1e6);
        ms = best_ms([&] { write4_v8_k<<<grid, T>>>(h, r, m, v, n); });
        printf("{\"kernel\": \"4 streams write only, 256-bit fp32 stores\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 12.0 * n / ms / 1e6);
        ms = best_ms([&] { adam_pattern_v8_k<<<grid, T>>>(h, r, g, m, v, n); });
        printf("{\"kernel\": \"adam pattern 5R+4W in place, 256-bit fp32 stores\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", per_sm, ms, 26.0 * n / ms / 1e6);
    }
    CK(cudaGetLastError());
    return 0;
}
