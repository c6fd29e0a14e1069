// Micro-benchmark: host launch cost vs kernel-parameter size (sm_100a).
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
template <int BYTES> struct P { unsigned char b[BYTES]; };
template <int BYTES> __global__ void k(const __grid_constant__ P<BYTES> p, int* out) { if (threadIdx.x == 0 && p.b[0] == 123) out[0] = p.b[BYTES - 1]; }
template <int BYTES> void run(int* out, cudaStream_t s) {
  P<BYTES> p{}; const int N = 5000;
  for (int i = 0; i < 100; ++i) k<BYTES><<<148, 32, 0, s>>>(p, out);
  cudaStreamSynchronize(s);
  auto t0 = std::chrono::high_resolution_clock::now();
  for (int i = 0; i < N; ++i) k<BYTES><<<148, 32, 0, s>>>(p, out);
  auto t1 = std::chrono::high_resolution_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::high_resolution_clock::now();
  printf("params %6d B: host %.2f us/launch, total %.2f us/launch\n", BYTES,
         std::chrono::duration<double, std::micro>(t1 - t0).count() / N, std::chrono::duration<double, std::micro>(t2 - t0).count() / N);
}
int main() {
  int* out; cudaMalloc(&out, 4); cudaStream_t s; cudaStreamCreate(&s);
  run<256>(out, s); run<1024>(out, s); run<4096>(out, s); run<8192>(out, s); run<16384>(out, s); run<29696>(out, s); run<32000>(out, s);
  return 0;
}
