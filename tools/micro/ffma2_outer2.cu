// FFMA2 outer-product variants from registers: which loop order / tile shape reaches the FFMA2 peak
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int TI, int TJ, int ORDER>
__global__ void __launch_bounds__(256, 2) k(float* out, int iters, unsigned long long seed) {
  unsigned long long acc[TI][TJ];
  unsigned long long av[TI], bv[TJ];
  for (int i = 0; i < TI; ++i) av[i] = seed + i * 3 + threadIdx.x;
  for (int j = 0; j < TJ; ++j) bv[j] = seed * 7 + j + threadIdx.x;
  for (int i = 0; i < TI; ++i)
    for (int j = 0; j < TJ; ++j) acc[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      if (ORDER == 0) {
#pragma unroll
        for (int i = 0; i < TI; ++i)
#pragma unroll
          for (int j = 0; j < TJ; ++j) acc[i][j] = ffma2(av[i], bv[j], acc[i][j]);
      } else {
#pragma unroll
        for (int j = 0; j < TJ; ++j)
#pragma unroll
          for (int i = 0; i < TI; ++i) acc[i][j] = ffma2(av[i], bv[j], acc[i][j]);
      }
      av[kk % TI] += 0x100000001ull;
      bv[kk % TJ] += 0x100000001ull;
    }
  }
  float r = 0;
  for (int i = 0; i < TI; ++i)
    for (int j = 0; j < TJ; ++j) r += __uint_as_float((unsigned)acc[i][j]);
  out[blockIdx.x * 256 + threadIdx.x] = r;
}
template <int TI, int TJ, int ORDER>
void run(float* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000, blocks = 148 * 2;
  float ms;
  k<TI, TJ, ORDER><<<blocks, 256>>>(out, iters, 0x3f8000003f800000ull);
  cudaEventRecord(e0);
  k<TI, TJ, ORDER><<<blocks, 256>>>(out, iters, 0x3f8000003f800000ull);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("tile %dx%d pairs order %d: %.1f TFLOP/s\n", TI, TJ, ORDER,
         2.0 * 2 * TI * TJ * 8 * iters * (double)blocks * 256 / (ms * 1e-3) / 1e12);
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 4 * 256 * 4);
  run<8, 4, 0>(out); run<8, 4, 1>(out); run<4, 4, 0>(out); run<4, 8, 0>(out); run<4, 8, 1>(out);
  run<8, 2, 0>(out); run<2, 8, 1>(out); run<16, 2, 0>(out); run<6, 4, 0>(out);
  return 0;
}
