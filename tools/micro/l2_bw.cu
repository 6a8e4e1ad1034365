// L2 read bandwidth of one B200: every SM streams a buffer that fits in L2 (ld.global.cg: cached
// in L2 only, so each load is an L2 hit after the first pass).  The pruning scan's centroid-tail
// reads are served from L2/L1; this is the denominator of its L2 roofline (profiles/l2_peak.json).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ p, long long n4, int passes, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (int r = 0; r < passes; ++r) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
      const float4 v0 = __ldcg(p + i), v1 = __ldcg(p + i + stride), v2 = __ldcg(p + i + 2 * stride),
                   v3 = __ldcg(p + i + 3 * stride);
      acc.x += v0.x + v1.x; acc.y += v0.y + v1.y; acc.z += v2.z + v3.z; acc.w += v2.w + v3.w;
    }
    for (; i < n4; i += stride) {
      const float4 v = __ldcg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (long long mb : {16LL, 32LL, 64LL, 96LL, 8192LL}) {
    const long long bytes = mb << 20, n4 = bytes / 16;
    float4* p;
    float* o;
    cudaMalloc(&p, bytes);
    cudaMalloc(&o, 4);
    cudaMemset(p, 0, bytes);
    const int passes = mb >= 1024 ? 2 : 40;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rd<<<sms * 4, 512>>>(p, n4, 2, o);
    cudaEventRecord(a);
    rd<<<sms * 4, 512>>>(p, n4, passes, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"buffer_mb\": %lld, \"read_gbs\": %.1f}\n", mb, (double)bytes * passes / (ms * 1e-3) / 1e9);
    cudaFree(p);
    cudaFree(o);
  }
  return 0;
}
