// FFMA2 outer-product microbenchmark: 8x4 packed accumulators updated from register fragments
// (a) refreshed by a cheap ALU op each step, (b) loaded from shared memory each step.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(float* out, int iters) {
  __shared__ unsigned long long sa[16][128];
  __shared__ float sb[16][128];
  for (int i = threadIdx.x; i < 16 * 128; i += 256) {
    (&sa[0][0])[i] = 0x3f8000003f800000ull + i;
    (&sb[0][0])[i] = 1.0f + i * 1e-7f;
  }
  __syncthreads();
  unsigned long long acc[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  unsigned long long av[8], bv[4];
  for (int i = 0; i < 8; ++i) av[i] = sa[0][ty * 4 + i];
  for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<unsigned long long*>(&sb[0][tx * 4 + 2 * j]);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      if (MODE == 1) {
        const ulonglong2* Ak = reinterpret_cast<const ulonglong2*>(&sa[kk][0]);
        const ulonglong2 a01 = Ak[ty * 2], a23 = Ak[ty * 2 + 1], a45 = Ak[32 + ty * 2], a67 = Ak[32 + ty * 2 + 1];
        av[0] = a01.x; av[1] = a01.y; av[2] = a23.x; av[3] = a23.y; av[4] = a45.x; av[5] = a45.y; av[6] = a67.x; av[7] = a67.y;
        const ulonglong2 b03 = *reinterpret_cast<const ulonglong2*>(&sb[kk][tx * 4]);
        const ulonglong2 b47 = *reinterpret_cast<const ulonglong2*>(&sb[kk][64 + tx * 4]);
        bv[0] = b03.x; bv[1] = b03.y; bv[2] = b47.x; bv[3] = b47.y;
      } else {
        av[kk & 7] ^= 1;  // keep the compiler honest
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(av[i], bv[j], acc[i][j]);
    }
  }
  float r = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) r += __uint_as_float((unsigned)acc[i][j]);
  out[blockIdx.x * 256 + threadIdx.x] = r;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 4 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000, blocks = 148 * 2;
  for (int pass = 0; pass < 2; ++pass) {
    float ms;
    k<0><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e0);
    k<0><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f0 = 2.0 * 64 * 16 * iters * (double)blocks * 256 / (ms * 1e-3) / 1e12;
    k<1><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e0);
    k<1><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f1 = 2.0 * 64 * 16 * iters * (double)blocks * 256 / (ms * 1e-3) / 1e12;
    if (pass) printf("outer product from registers: %.1f TFLOP/s; with smem fragments: %.1f TFLOP/s\n", f0, f1);
  }
  return 0;
}
