// Microbenchmark: ceiling of the lane-per-pair block computation on B200.
// Each lane repeatedly fetches a pseudo-random 256-byte candidate block from an L2-resident
// table (k x nb blocks) and runs the exact 64-dim fp32 chain against an x block in shared
// memory.  Variants: (0) direct LDG.128 x16, (1) per-lane TMA bulk copy double-buffered,
// (2) warp-cooperative LDG (2 blocks per instruction) through shared memory, (3) like 0 but
// two independent pairs per lane (ILP 2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2603_20009_b200/csrc pairblock_bench.cu -o pb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace skm;

__device__ __forceinline__ unsigned hsh(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__device__ __forceinline__ float chain(const float4* xq, int nb, const float4 (&c)[16]) {
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 xv = xq[q * nb];
    const float2 d01 = __fadd2_rn(make_float2(xv.x, xv.y), make_float2(-c[q].x, -c[q].y));
    const float2 d23 = __fadd2_rn(make_float2(xv.z, xv.w), make_float2(-c[q].z, -c[q].w));
    const float2 s01 = __fmul2_rn(d01, d01), s23 = __fmul2_rn(d23, d23);
    acc = __fadd_rn(acc, s01.x); acc = __fadd_rn(acc, s01.y); acc = __fadd_rn(acc, s23.x); acc = __fadd_rn(acc, s23.y);
  }
  return acc;
}

// G rows share each candidate block: one cooperative load, G independent chains per lane
template <int G>
__device__ __forceinline__ void chains(const float* xs, int nb, int slotf, int b, const float4* cq, float (&acc)[G]) {
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.f;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 cv = cq[q];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float4 xv = reinterpret_cast<const float4*>(xs + g * slotf)[q * nb + b];
      const float2 d01 = __fadd2_rn(make_float2(xv.x, xv.y), make_float2(-cv.x, -cv.y));
      const float2 d23 = __fadd2_rn(make_float2(xv.z, xv.w), make_float2(-cv.z, -cv.w));
      const float2 s01 = __fmul2_rn(d01, d01), s23 = __fmul2_rn(d23, d23);
      acc[g] = __fadd_rn(acc[g], s01.x); acc[g] = __fadd_rn(acc[g], s01.y);
      acc[g] = __fadd_rn(acc[g], s23.x); acc[g] = __fadd_rn(acc[g], s23.y);
    }
  }
}

template <int MODE>
__global__ void bench(const float4* __restrict__ tails, int nblk, int nb, int iters, float* out) {
  extern __shared__ __align__(16) float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* xs = sm + warp * (64 * nb);
  float4* stg = reinterpret_cast<float4*>(sm + nw * 64 * nb) + warp * (MODE == 1 ? 2 : 1) * 32 * 17;
  __shared__ uint64_t bars[32][2][32];
  for (int i = lane; i < 64 * nb * ((MODE == 6 || MODE == 8) ? 4 : (MODE == 5 || MODE == 7) ? 2 : 1); i += 32) (MODE >= 5 ? sm + warp * 64 * nb * ((MODE == 6 || MODE == 8) ? 4 : (MODE == 5 || MODE == 7) ? 2 : 1) : xs)[i] = 0.001f * i;
  if (MODE == 1) { mbar_init(&bars[warp][0][lane], 1); mbar_init(&bars[warp][1][lane], 1); fence_mbar_init(); }
  __syncthreads();
  const float4* xq = reinterpret_cast<const float4*>(xs);
  unsigned seed = (blockIdx.x * nw + warp) * 32 + lane;
  float tot = 0.f;
  if (MODE == 0) {
    for (int it = 0; it < iters; ++it) {
      const unsigned blk = hsh(seed + it * 7919u) % nblk;
      const float4* cb = tails + (size_t)blk * 16;
      float4 c[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) c[q] = __ldg(cb + q);
      tot += chain(xq + (blk % nb), nb, c);
    }
  } else if (MODE == 3) {
    for (int it = 0; it < iters; it += 2) {
      const unsigned b0 = hsh(seed + it * 7919u) % nblk, b1 = hsh(seed + (it + 1) * 7919u) % nblk;
      float4 c0[16], c1[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) { c0[q] = __ldg(tails + (size_t)b0 * 16 + q); c1[q] = __ldg(tails + (size_t)b1 * 16 + q); }
      tot += chain(xq + (b0 % nb), nb, c0) + chain(xq + (b1 % nb), nb, c1);
    }
  } else if (MODE == 1) {
    uint32_t ph = 0;
    auto issue = [&](int i, unsigned blk) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[warp][i][lane], 256);
      bulk_g2s(stg + (i * 32 + lane) * 17, tails + (size_t)blk * 16, 256, &bars[warp][i][lane]);
    };
    issue(0, hsh(seed) % nblk);
    for (int it = 0; it < iters; ++it) {
      const int cur = it & 1;
      if (it + 1 < iters) issue(cur ^ 1, hsh(seed + (it + 1) * 7919u) % nblk);
      mbar_wait(&bars[warp][cur][lane], (ph >> cur) & 1); ph ^= 1u << cur;
      const unsigned blk = hsh(seed + it * 7919u) % nblk;
      float4 c[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) c[q] = stg[(cur * 32 + lane) * 17 + q];
      tot += chain(xq + (blk % nb), nb, c);
    }
  } else if (MODE >= 5) {
    constexpr int G = (MODE == 5 || MODE == 7) ? 2 : (MODE == 9 ? 1 : 4);
    const int half = lane >> 4, part = lane & 15;
    float* xg = sm + warp * (G * 64 * nb);
    float4* st = reinterpret_cast<float4*>(sm + nw * G * 64 * nb) + warp * 32 * 17;
    float4 v[16];
    unsigned myblk = hsh(seed) % nblk;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const unsigned blk = __shfl_sync(0xffffffffu, myblk, 2 * i + half);
      v[i] = __ldg(tails + (size_t)blk * 16 + part);
    }
    for (int it = 0; it < iters; ++it) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) st[(2 * i + half) * 17 + part] = v[i];
      __syncwarp();
      const unsigned cur = myblk;
      if (it + 1 < iters) {
        myblk = hsh(seed + (it + 1) * 7919u) % nblk;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const unsigned blk = __shfl_sync(0xffffffffu, myblk, 2 * i + half);
          v[i] = __ldg(tails + (size_t)blk * 16 + part);
        }
      }
      float acc[G];
      chains<G>(xg, nb, 64 * nb, (MODE >= 7 ? it : cur) % nb, st + lane * 17, acc);
#pragma unroll
      for (int g = 0; g < G; ++g) tot += acc[g];
    }
  } else if (MODE == 4) {
    const int half = lane >> 4, part = lane & 15;
    float4 v[16];
    unsigned myblk = hsh(seed) % nblk;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const unsigned blk = __shfl_sync(0xffffffffu, myblk, 2 * i + half);
      v[i] = __ldg(tails + (size_t)blk * 16 + part);
    }
    for (int it = 0; it < iters; ++it) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) stg[(2 * i + half) * 17 + part] = v[i];
      __syncwarp();
      const unsigned cur = myblk;
      if (it + 1 < iters) {
        myblk = hsh(seed + (it + 1) * 7919u) % nblk;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const unsigned blk = __shfl_sync(0xffffffffu, myblk, 2 * i + half);
          v[i] = __ldg(tails + (size_t)blk * 16 + part);
        }
      }
      float4 c[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) c[q] = stg[lane * 17 + q];
      tot += chain(xq + (cur % nb), nb, c);
    }
  } else if (MODE == 2) {
    const int half = lane >> 4, part = lane & 15;
    for (int it = 0; it < iters; ++it) {
      const unsigned myblk = hsh(seed + it * 7919u) % nblk;
      float4 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const unsigned blk = __shfl_sync(0xffffffffu, myblk, 2 * i + half);
        v[i] = __ldg(tails + (size_t)blk * 16 + part);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 16; ++i) stg[(2 * i + half) * 17 + part] = v[i];
      __syncwarp();
      float4 c[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) c[q] = stg[lane * 17 + q];
      tot += chain(xq + (myblk % nb), nb, c);
    }
  }
  if (tot == 12345.f) out[0] = tot;
}

int main() {
  const int k = 4096, nb = 21, nblk = k * nb;
  float4* tails; cudaMalloc(&tails, (size_t)nblk * 256);
  cudaMemset(tails, 0, (size_t)nblk * 256);
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 512;
  for (int mode : {9, 7, 8}) {
    for (int warps : {4, 6, 8, 10, 12, 14}) {
      const int G = (mode == 5 || mode == 7) ? 2 : (mode == 6 || mode == 8) ? 4 : 1;
      const size_t smem = (size_t)warps * G * 64 * nb * 4 + (mode == 1 ? (size_t)warps * 2 * 32 * 17 * 16 : (mode == 2 || mode >= 4) ? (size_t)warps * 32 * 17 * 16 : 0);
      if (smem > 220 * 1024) continue;
      void (*fn)(const float4*, int, int, int, float*) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : mode == 3 ? bench<3> : mode == 4 ? bench<4> : mode == 5 ? bench<5> : mode == 6 ? bench<6> : mode == 7 ? bench<7> : mode == 8 ? bench<8> : bench<9>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      fn<<<sms, warps * 32, smem>>>(tails, nblk, nb, iters, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) fn<<<sms, warps * 32, smem>>>(tails, nblk, nb, iters, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
      cudaError_t err = cudaGetLastError();
      const double pbs = (double)sms * warps * 32 * iters * G;
      printf("mode %d warps/SM %2d: %.3f ms  %.2f Gpb/s  %.1f clk/pb/SM  %s\n", mode, warps, ms, pbs / ms / 1e6,
             (double)sms * 1.965e9 * ms * 1e-3 / pbs, cudaGetErrorString(err));
    }
  }
  return 0;
}
