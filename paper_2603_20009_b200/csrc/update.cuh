// Centroid update (core.py:79-100, _kernels.pyx:106-119) rebuilt for the GPU:
//   1. stable LSD radix sort of row ids by assignment (8-bit digits) -> rows grouped by
//      cluster, ascending row id inside each cluster;
//   2. per-cluster counts + exclusive offsets;
//   3. one thread per (cluster, dim) sums its member rows in ascending row order in
//      double precision -- the same operation order as the reference's serial loop, so
//      the f64 sums are bitwise identical at one GPU -- then divides and rounds to f32
//      (empty clusters keep their previous centroid).
// The sorted row order doubles as the cluster lists used by ETR / IVF probing
// (evaluation.py:78-83) and as a cluster-coherent vector order for the pruning scan.
#pragma once
#include "ptx.cuh"
#include <cstdint>
#include <cuda_runtime.h>

namespace skm {

constexpr int RADIX_THREADS = 256;
constexpr int RADIX_WARPS = RADIX_THREADS / 32;
constexpr int RADIX_ROUNDS = 16;
constexpr int RADIX_TILE = RADIX_THREADS * RADIX_ROUNDS;  // 4096 items per block

__global__ void __launch_bounds__(RADIX_THREADS)
    radix_hist_kernel(const int* __restrict__ keys, int n, int shift, int* __restrict__ hist, int nblocks) {
  __shared__ int cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * RADIX_TILE;
  for (int e = threadIdx.x; e < RADIX_TILE; e += RADIX_THREADS) {
    const int i = base + e;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255], 1);
  }
  __syncthreads();
  hist[threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// In-place exclusive scan of an int array with one block (sizes here are <= a few 1e6).
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(int* __restrict__ a, int n, int* __restrict__ total) {
  __shared__ int part[1024];
  const int tid = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int beg = min(n, tid * per), end = min(n, beg + per);
  int s = 0;
  for (int i = beg; i < end; ++i) s += a[i];
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = part[tid] - s;  // exclusive prefix of this thread's segment
  for (int i = beg; i < end; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  if (tid == 1023 && total) *total = part[1023];
}

__global__ void __launch_bounds__(RADIX_THREADS)
    radix_scatter_kernel(const int* __restrict__ keys_in, const int* __restrict__ vals_in, int* __restrict__ keys_out,
                         int* __restrict__ vals_out, int n, int shift, const int* __restrict__ offs, int nblocks) {
  __shared__ int wcnt[RADIX_WARPS][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < RADIX_WARPS * 256; e += RADIX_THREADS) (&wcnt[0][0])[e] = 0;
  __syncthreads();
  const int base = blockIdx.x * RADIX_TILE + warp * (RADIX_ROUNDS * 32);
  const unsigned lt_mask = (1u << lane) - 1u;
  int k_r[RADIX_ROUNDS], v_r[RADIX_ROUNDS], rank_r[RADIX_ROUNDS];
#pragma unroll
  for (int r = 0; r < RADIX_ROUNDS; ++r) {
    const int i = base + r * 32 + lane;
    const bool ok = i < n;
    const int key = ok ? keys_in[i] : 0;
    const int digit = ok ? ((key >> shift) & 255) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, digit);
    int prior = 0;
    if (ok) prior = wcnt[warp][digit];
    __syncwarp();
    if (ok && (peers & lt_mask) == 0) wcnt[warp][digit] = prior + __popc(peers);
    __syncwarp();
    k_r[r] = key;
    v_r[r] = ok ? vals_in[i] : 0;
    rank_r[r] = ok ? prior + __popc(peers & lt_mask) : -1;
  }
  __syncthreads();
  {  // exclusive prefix over warps for each digit
    const int dgt = threadIdx.x;
    int run = 0;
    for (int w = 0; w < RADIX_WARPS; ++w) {
      const int c = wcnt[w][dgt];
      wcnt[w][dgt] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RADIX_ROUNDS; ++r) {
    if (rank_r[r] >= 0) {
      const int digit = (k_r[r] >> shift) & 255;
      const int pos = offs[digit * nblocks + blockIdx.x] + wcnt[warp][digit] + rank_r[r];
      keys_out[pos] = k_r[r];
      vals_out[pos] = v_r[r];
    }
  }
}

__global__ void count_keys_kernel(const int* __restrict__ keys, int n, int* __restrict__ counts) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(&counts[keys[i]], 1);
}

// Ordered double-precision member sums.  grid = (k, ceil(d / 128)).
// mode 0: finalize into centroids (count>0: f32(sum/count); else keep previous)
// mode 1: write/accumulate raw sums (sums_io holds the running value; used by the parity
//         entry and by the multi-GPU path before the allreduce)
constexpr int SUM_THREADS = 128;
__global__ void __launch_bounds__(SUM_THREADS)
    ordered_cluster_sums_kernel(const float* __restrict__ x, long long ldx, const int* __restrict__ order,
                                const int* __restrict__ offsets, const int* __restrict__ counts, int d,
                                double* __restrict__ sums_io, int accumulate_sums, float* __restrict__ cent,
                                long long ldc, int mode) {
  const int c = blockIdx.x;
  const int col = blockIdx.y * SUM_THREADS + threadIdx.x;
  if (col >= d) return;
  const int beg = offsets[c], cnt = counts[c];
  double s = accumulate_sums ? sums_io[static_cast<long long>(c) * d + col] : 0.0;
  const int* ord = order + beg;
  int m = 0;
  // 8 member rows in flight per thread (the f64 chain itself stays in member order)
  for (; m + 8 <= cnt; m += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(x + static_cast<long long>(__ldg(ord + m + u)) * ldx + col);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, static_cast<double>(v[u]));
  }
  for (; m < cnt; ++m) s = __dadd_rn(s, static_cast<double>(x[static_cast<long long>(ord[m]) * ldx + col]));
  if (mode == 1) {
    sums_io[static_cast<long long>(c) * d + col] = s;
  } else if (cnt > 0) {
    cent[static_cast<long long>(c) * ldc + col] = __double2float_rn(__ddiv_rn(s, static_cast<double>(cnt)));
  }
}

// Same sums, one CTA per cluster: thread = 4 consecutive columns (16-byte aligned rows, ld % 4
// == 0 so the padded columns past d are readable), four f64 chains in member order (bitwise the
// per-column kernel).  A member row is read as one contiguous run by one CTA, and each thread
// keeps SUMV_RING member rows in flight through a private cp.async ring in shared memory (it
// consumes exactly the 16 bytes it copied, so no block barrier): the chain of a large cluster
// is bound by memory latency / ring depth, not by 4 loads per round trip.
constexpr int SUMV_RING = 16;
__device__ __forceinline__ void sumv_add(double (&s)[4], const float4& v) {
  s[0] = __dadd_rn(s[0], static_cast<double>(v.x));
  s[1] = __dadd_rn(s[1], static_cast<double>(v.y));
  s[2] = __dadd_rn(s[2], static_cast<double>(v.z));
  s[3] = __dadd_rn(s[3], static_cast<double>(v.w));
}
__global__ void __launch_bounds__(768)
    ordered_cluster_sums_vec_kernel(const float* __restrict__ x, long long ldx, const int* __restrict__ order,
                                    const int* __restrict__ offsets, const int* __restrict__ counts, int d,
                                    double* __restrict__ sums_io, int accumulate_sums, float* __restrict__ cent,
                                    long long ldc, int mode) {
  extern __shared__ __align__(16) float4 sumv_ring[];  // [SUMV_RING][blockDim.x]
  const int c = blockIdx.x;
  const int beg = offsets[c], cnt = counts[c];
  const int* ord = order + beg;
  const int ng = (d + 3) / 4;
  const int bd = blockDim.x;
  float4* ring = sumv_ring + threadIdx.x;
  for (int g = threadIdx.x; g < ng; g += bd) {
    const int col = 4 * g;
    const long long so = static_cast<long long>(c) * d + col;
    double s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i] = (accumulate_sums && col + i < d) ? sums_io[so + i] : 0.0;
    auto issue = [&](int m) {
      if (m < cnt)
        cp_async_16_zfill(ring + (m % SUMV_RING) * bd, x + static_cast<long long>(__ldg(ord + m)) * ldx + col, 16);
      cp_async_commit();  // empty groups keep the wait count uniform
    };
#pragma unroll 1
    for (int m = 0; m < SUMV_RING - 1; ++m) issue(m);
#pragma unroll 1
    for (int m = 0; m < cnt; ++m) {
      issue(m + SUMV_RING - 1);
      cp_async_wait_group<SUMV_RING - 1>();  // member m has landed
      sumv_add(s, ring[(m % SUMV_RING) * bd]);
    }
    cp_async_wait_all();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (col + i >= d) break;
      if (mode == 1) {
        sums_io[so + i] = s[i];
      } else if (cnt > 0) {
        cent[static_cast<long long>(c) * ldc + col + i] = __double2float_rn(__ddiv_rn(s[i], static_cast<double>(cnt)));
      }
    }
  }
}

// Finalize from (allreduced) sums/counts: count>0 -> f32(sum/count), else keep previous.
__global__ void finalize_centroids_kernel(const double* __restrict__ sums, const long long* __restrict__ counts, int k,
                                          int d, float* __restrict__ cent, long long ldc) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)k * d;
       e += (long long)gridDim.x * blockDim.x) {
    const long long c = e / d;
    const int t = static_cast<int>(e - c * d);
    const long long cnt = counts[c];
    if (cnt > 0) cent[c * ldc + t] = __double2float_rn(__ddiv_rn(sums[e], static_cast<double>(cnt)));
  }
}

__global__ void counts_to_i64_kernel(const int* __restrict__ c32, long long* __restrict__ c64, int k, int accumulate) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
    c64[i] = (accumulate ? c64[i] : 0) + c32[i];
}

}  // namespace skm
