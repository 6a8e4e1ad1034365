// FFMA vs packed FFMA2 (fma.rn.f32x2) issue throughput on one B200, for sizing the exact-chain
// (OpenBLAS-bitwise) fp32 GEMM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int NACC>
__global__ void k2(float* out, int iters, float s) {
  unsigned long long acc[NACC];
  unsigned long long a = __float_as_uint(s) | ((unsigned long long)__float_as_uint(s * 1.0001f) << 32);
  unsigned long long b = __float_as_uint(0.999f) | ((unsigned long long)__float_as_uint(0.9991f) << 32);
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = a + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = ffma2(acc[i], b, a);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
// FFMA2 with a scalar broadcast operand (mov.b64 {s, s}: `R.F32` in the SASS), as in the
// k-major exact-chain GEMM
template <int NACC>
__global__ void k3(float* out, int iters, float s) {
  unsigned long long acc[NACC];
  unsigned long long a = __float_as_uint(s) | ((unsigned long long)__float_as_uint(s * 1.0001f) << 32);
  float bs = 0.999f + 1e-7f * threadIdx.x;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = a + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      unsigned long long d;
      asm volatile("{\n\t.reg .b64 bp;\n\tmov.b64 bp, {%1, %1};\n\tfma.rn.f32x2 %0, bp, %2, %3;\n\t}"
                   : "=l"(d) : "f"(bs), "l"(acc[i]), "l"(a));
      acc[i] = d;
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += __uint_as_float((unsigned)acc[i]) + __uint_as_float((unsigned)(acc[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int NACC>
__global__ void k1(float* out, int iters, float s) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = s + i;
  float b = 0.999f, a = s * 1.0001f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fmaf(acc[i], b, a);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int pass = 0; pass < 2; ++pass) {
    for (int threads : {256, 512, 1024}) {
      int blocks = 148 * (1024 / threads) * 2;
      float ms;
      k1<16><<<blocks, threads>>>(out, iters, 1.0f);
      cudaEventRecord(e0);
      k1<16><<<blocks, threads>>>(out, iters, 1.0f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double f1 = 2.0 * 16 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
      k2<16><<<blocks, threads>>>(out, iters, 1.0f);
      cudaEventRecord(e0);
      k2<16><<<blocks, threads>>>(out, iters, 1.0f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double f2 = 4.0 * 16 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
      k3<16><<<blocks, threads>>>(out, iters, 1.0f);
      cudaEventRecord(e0);
      k3<16><<<blocks, threads>>>(out, iters, 1.0f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double f3 = 4.0 * 16 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
      if (pass) printf("threads %d: FFMA %.1f TFLOP/s, FFMA2 %.1f TFLOP/s, FFMA2 broadcast %.1f TFLOP/s\n", threads, f1,
                       f2, f3);
    }
  }
  return 0;
}
