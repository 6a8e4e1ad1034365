// Exact per-row top-k (k smallest by (value, column), lowest column on ties) and the ETR
// recall tally.
//
// Reference semantics: brute_force_topk / etr_probe rank with np.argsort(kind="stable")
// (evaluation.py:53-75, 142-170), i.e. ascending value with ties to the lower index.  Values
// here are squared distances >= +0, so their IEEE bit patterns order like the values.
//
// One CTA per row: 4-pass radix select (8-bit digits, shared-memory histograms) finds the
// k-th key T; elements < T are kept, elements == T are taken in column order until k, then
// the k (key, column) pairs are bitonic-sorted in shared memory.  Memory-bound: 5 streaming
// reads of the row.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace skm {

constexpr int TOPK_THREADS = 512;
constexpr int TOPK_MAX = 2048;

__device__ __forceinline__ unsigned key_of(float v) { return __float_as_uint(v); }

__global__ void __launch_bounds__(TOPK_THREADS)
    topk_rows_kernel(const float* __restrict__ D, long long ld, int cols, int k, int* __restrict__ out_idx,
                     float* __restrict__ out_val, long long out_ld, int col_offset) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long sel[TOPK_MAX];
  __shared__ int s_digit, s_need, s_nsel, s_ties;
  __shared__ int scan_buf[TOPK_THREADS / 32];
  const int row = blockIdx.x;
  const int tid = threadIdx.x;
  const float* d = D + static_cast<long long>(row) * ld;
  const int kk = min(k, cols);
  unsigned prefix = 0, mask = 0;
  int need = kk;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += TOPK_THREADS) hist[i] = 0;
    __syncthreads();
    for (int c = tid; c < cols; c += TOPK_THREADS) {
      const unsigned key = key_of(d[c]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      unsigned cum = 0;
      int dg = 0;
      for (; dg < 256; ++dg) {
        if (cum + hist[dg] >= static_cast<unsigned>(need)) break;
        cum += hist[dg];
      }
      s_digit = dg;
      s_need = need - static_cast<int>(cum);
    }
    __syncthreads();
    prefix |= static_cast<unsigned>(s_digit) << shift;
    mask |= 255u << shift;
    need = s_need;
    __syncthreads();
  }
  // prefix is the k-th key; `need` ties (key == prefix) are taken in column order
  if (tid == 0) {
    s_nsel = 0;
    s_ties = 0;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < cols; c0 += TOPK_THREADS) {
    const int c = c0 + tid;
    unsigned key = 0xffffffffu;
    if (c < cols) key = key_of(d[c]);
    if (c < cols && key < prefix) {
      const int pos = atomicAdd(&s_nsel, 1);
      if (pos < TOPK_MAX) sel[pos] = (static_cast<unsigned long long>(key) << 32) | static_cast<unsigned>(c);
    }
    // ordered tie ranks: block-wide exclusive scan of the tie flags (thread order == column order)
    const bool tie = c < cols && key == prefix;
    const unsigned bal = __ballot_sync(0xffffffffu, tie);
    if (lane == 0) scan_buf[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < TOPK_THREADS / 32; ++w) {
      const int v = scan_buf[w];
      before += (w < warp) ? v : 0;
      total += v;
    }
    const int rank = s_ties + before + __popc(bal & ((1u << lane) - 1u));
    if (tie && rank < need) {
      const int pos = atomicAdd(&s_nsel, 1);
      if (pos < TOPK_MAX) sel[pos] = (static_cast<unsigned long long>(key) << 32) | static_cast<unsigned>(c);
    }
    __syncthreads();
    if (tid == 0) s_ties += total;
    __syncthreads();
  }
  // bitonic sort of the kk selected pairs (padded to a power of two with +inf keys)
  int p2 = 1;
  while (p2 < kk) p2 <<= 1;
  for (int i = kk + tid; i < p2; i += TOPK_THREADS) sel[i] = ~0ull;
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < p2; i += TOPK_THREADS) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const unsigned long long a = sel[i], b = sel[j];
          if ((a > b) == up) {
            sel[i] = b;
            sel[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < kk; i += TOPK_THREADS) {
    const unsigned long long v = sel[i];
    out_idx[static_cast<long long>(row) * out_ld + i] = static_cast<int>(v & 0xffffffffu) + col_offset;
    if (out_val) out_val[static_cast<long long>(row) * out_ld + i] = __uint_as_float(static_cast<unsigned>(v >> 32));
  }
}

// Merge per-shard sorted top-k lists (multi-GPU ground truth): rows x (shards*k) candidates,
// already globally indexed; keeps the k smallest by (value, index).
__global__ void topk_merge_kernel(const int* __restrict__ in_idx, const float* __restrict__ in_val, int shards, int k,
                                  int nrows, int* __restrict__ out_idx, float* __restrict__ out_val) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  // simple k-way merge by repeated selection (k and shards are small)
  int pos[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int o = 0; o < k; ++o) {
    int bs = -1;
    unsigned long long bk = ~0ull;
    for (int s = 0; s < shards && s < 8; ++s) {
      if (pos[s] >= k) continue;
      const long long e = (static_cast<long long>(s) * nrows + row) * k + pos[s];
      const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(in_val[e])) << 32) |
                                     static_cast<unsigned>(in_idx[e]);
      if (key < bk) {
        bk = key;
        bs = s;
      }
    }
    if (bs < 0) break;
    ++pos[bs];
    out_idx[static_cast<long long>(row) * k + o] = static_cast<int>(bk & 0xffffffffu);
    out_val[static_cast<long long>(row) * k + o] = __uint_as_float(static_cast<unsigned>(bk >> 32));
  }
}

// hits[q] = #{ g in gt[q][:top_k] owned by this shard : assign[g - row_lo] in probe[q][:nprobe] }
// (the reference's per-query recall numerator, evaluation.py:163-169, as an integer tally).
__global__ void etr_hits_kernel(const int* __restrict__ gt, int gt_ld, int top_k, const int* __restrict__ probe,
                                int probe_ld, int nprobe, const int* __restrict__ assign, long long row_lo,
                                long long row_hi, int k, int* __restrict__ hits,
                                const int* __restrict__ sizes = nullptr, long long* __restrict__ explored = nullptr) {
  extern __shared__ unsigned bitmap[];
  const int q = blockIdx.x;
  const int words = (k + 31) / 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) bitmap[i] = 0;
  __syncthreads();
  long long ex = 0;  // vectors in the probed clusters (probe_eval's vectors_explored)
  for (int i = threadIdx.x; i < nprobe; i += blockDim.x) {
    const int c = probe[static_cast<long long>(q) * probe_ld + i];
    atomicOr(&bitmap[c >> 5], 1u << (c & 31));
    if (sizes) ex += sizes[c];
  }
  __syncthreads();
  int h = 0;
  for (int i = threadIdx.x; i < top_k; i += blockDim.x) {
    const long long g = gt[static_cast<long long>(q) * gt_ld + i];
    if (g >= row_lo && g < row_hi) {
      const int a = assign[g - row_lo];  // < 0: the row is in no cluster list
      if (a >= 0 && a < k) h += (bitmap[a >> 5] >> (a & 31)) & 1u;
    }
  }
  if (explored) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ex += __shfl_xor_sync(0xffffffffu, ex, o);
    if ((threadIdx.x & 31) == 0 && ex) atomicAdd(reinterpret_cast<unsigned long long*>(explored + q),
                                                 static_cast<unsigned long long>(ex));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  __shared__ int red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) t += red[w];
    hits[q] = t;
  }
}

}  // namespace skm
