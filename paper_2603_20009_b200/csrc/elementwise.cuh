// Memory-bound helper kernels: 3xTF32 operand split, squared norms, row gathers,
// threshold seeding, bit-exact bank scan (parity ABI), portable matmul (parity ABI),
// assignment statistics, split application.
#pragma once
#include "sgemm_chain.cuh"
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace skm {

constexpr float kInf = __builtin_huge_valf();

// x = hi + lo exactly, hi has a 10-bit mantissa (tf32-representable) so the tensor core
// consumes it losslessly whether it truncates or rounds; lo keeps the remaining bits.
__global__ void split_hilo_kernel(const float* __restrict__ x, long long ldx, int rows, int cols,
                                  float* __restrict__ hi, float* __restrict__ lo, long long ldo) {
  const long long total = static_cast<long long>(rows) * ldo;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long r = idx / ldo;
    const int c = static_cast<int>(idx - r * ldo);
    float v = 0.0f;
    if (c < cols) v = x[r * ldx + c];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    if (hi) hi[idx] = h;  // hi == nullptr: lo only (raw fp32 is a valid hi operand)
    lo[idx] = __fsub_rn(v, h);
  }
}

// Vectorised split (16-byte aligned rows, ld multiple of 4): 2-D grid, x over float4 columns,
// y strides over rows -- no per-element integer division.
__global__ void split_hilo_vec_kernel(const float4* __restrict__ x, long long ldx4, int rows, int cols,
                                      float4* __restrict__ hi, float4* __restrict__ lo, long long ldo4) {
  const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c4 >= ldo4) return;
  for (long long r = blockIdx.y; r < rows; r += gridDim.y) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * c4 < cols) v = x[r * ldx4 + c4];
    if (4 * c4 + 3 >= cols) {  // ragged end: zero the padding columns
      if (4 * c4 + 0 >= cols) v.x = 0.f;
      if (4 * c4 + 1 >= cols) v.y = 0.f;
      if (4 * c4 + 2 >= cols) v.z = 0.f;
      if (4 * c4 + 3 >= cols) v.w = 0.f;
    }
    float4 h;
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    if (hi) hi[r * ldo4 + c4] = h;
    lo[r * ldo4 + c4] = make_float4(__fsub_rn(v.x, h.x), __fsub_rn(v.y, h.y), __fsub_rn(v.z, h.z), __fsub_rn(v.w, h.w));
  }
}

// Gate batch gather, one warp per output row: front columns [0, cols) of hi and lo (float4
// when both strides are multiples of 4), plus the row's norm term and gate threshold.
__global__ void gather_front_kernel(const float* __restrict__ hi, const float* __restrict__ lo, long long ldi,
                                    const int* __restrict__ idx, int rows, int cols, float* __restrict__ ohi,
                                    float* __restrict__ olo, long long ldo, const float* __restrict__ xsq,
                                    const float* __restrict__ thr, float* __restrict__ oxsq, float* __restrict__ othr,
                                    const float* __restrict__ s3 = nullptr, float* __restrict__ o3 = nullptr,
                                    const float* __restrict__ s4 = nullptr, float* __restrict__ o4 = nullptr) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const bool vec = ((ldi & 3) == 0) && ((ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(hi) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(lo) & 15) == 0) && ((reinterpret_cast<uintptr_t>(ohi) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(olo) & 15) == 0);
  for (long long r = blockIdx.x * (long long)wpb + (threadIdx.x >> 5); r < rows; r += (long long)gridDim.x * wpb) {
    const long long src = idx[r];
    const float* sh = hi + src * ldi;
    const float* sl = lo + src * ldi;
    float* dh = ohi + r * ldo;
    float* dl = olo + r * ldo;
    int c0 = 0;
    if (vec) {
      const int c4n = cols >> 2;
      for (int c = lane; c < c4n; c += 32) {
        reinterpret_cast<float4*>(dh)[c] = __ldg(reinterpret_cast<const float4*>(sh) + c);
        reinterpret_cast<float4*>(dl)[c] = __ldg(reinterpret_cast<const float4*>(sl) + c);
      }
      c0 = c4n << 2;
    }
    for (int c = c0 + lane; c < cols; c += 32) {
      dh[c] = sh[c];
      dl[c] = sl[c];
    }
    if (lane == 0) {
      oxsq[r] = xsq[src];
      othr[r] = thr[src];
      if (s3) o3[r] = s3[src];
      if (s4) o4[r] = s4[src];
    }
  }
}

// Vector-file ingestion (dataio.py:57-112): one staged chunk of `rows` records starting at
// file row `row0` is validated and scattered into the padded device matrix.  fvecs records are
// [int32 d][d float32] (rec_words = d + 1, header_words = 1); fbin rows are bare (0 / d).
// For every 4096-row reporting chunk the first bad record (declared dim != d) and the first
// non-finite element (flat row-major index) are kept with atomicMin -- the host then reports
// the reference's error for the first reporting chunk holding either (dims take precedence).
constexpr int INGEST_CHUNK_ROWS = 4096;
__global__ void ingest_records_kernel(const uint32_t* __restrict__ raw, long long rows, int d, int rec_words,
                                      int header_words, long long row0, float* __restrict__ out, long long ldo,
                                      unsigned long long* __restrict__ bad_dim, unsigned long long* __restrict__ bad_val) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (long long r = blockIdx.x * (long long)wpb + (threadIdx.x >> 5); r < rows; r += (long long)gridDim.x * wpb) {
    const uint32_t* rec = raw + r * rec_words;
    const long long grow = row0 + r;
    const long long rc = grow / INGEST_CHUNK_ROWS;
    if (header_words && lane == 0 && static_cast<int>(rec[0]) != d)
      atomicMin(bad_dim + rc, static_cast<unsigned long long>(grow));
    const float* v = reinterpret_cast<const float*>(rec + header_words);
    float* o = out + grow * ldo;
    unsigned long long first = ~0ull;
    for (int c = lane; c < d; c += 32) {
      const float x = v[c];
      if (!isfinite(x) && first == ~0ull) first = static_cast<unsigned long long>(grow) * d + c;
      o[c] = x;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, first, s);
      first = o2 < first ? o2 : first;
    }
    if (lane == 0 && first != ~0ull) atomicMin(bad_val + rc, first);
  }
}

// evaluation.wcss (evaluation.py:205-215): sum_i |x_i - c_{a_i}|^2 in double.  Warp per row
// (f64 differences, lanes strided, shuffle tree), then per-block partials reduced in a fixed
// order by wcss_final_kernel: deterministic run to run (the CLI report is compared for
// determinism), equal to the reference's einsum up to f64 summation order.
constexpr int WCSS_THREADS = 256;
__global__ void __launch_bounds__(WCSS_THREADS) wcss_partial_kernel(const float* __restrict__ x, long long ldx,
                                                                    const float* __restrict__ c, long long ldc,
                                                                    const int* __restrict__ assign, long long n,
                                                                    int d, double* __restrict__ part) {
  __shared__ double ws[WCSS_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long beg = per * blockIdx.x, end = min(n, beg + per);
  double acc = 0.0;
  for (long long r = beg + warp; r < end; r += WCSS_THREADS / 32) {
    const float* xr = x + r * ldx;
    const float* cr = c + static_cast<long long>(assign[r]) * ldc;
    double s = 0.0;
    for (int t = lane; t < d; t += 32) {
      const double df = static_cast<double>(xr[t]) - static_cast<double>(cr[t]);
      s += df * df;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    acc += s;
  }
  if (lane == 0) ws[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < WCSS_THREADS / 32; ++w) t += ws[w];
    part[blockIdx.x] = t;
  }
}

__global__ void wcss_final_kernel(const double* __restrict__ part, int parts, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < parts; ++i) t += part[i];
    *out = t;
  }
}

// validate_vector_set's finiteness check (model.py:84-87) on the device: *first = min flat
// row-major index (row * cols + col) of a NaN/Inf among the leading `cols` columns.
__global__ void first_nonfinite_kernel(const float* __restrict__ x, long long ldx, long long rows, int cols,
                                       unsigned long long* __restrict__ first) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (long long r = blockIdx.x * (long long)wpb + (threadIdx.x >> 5); r < rows; r += (long long)gridDim.x * wpb) {
    unsigned long long f = ~0ull;
    for (int c = lane; c < cols; c += 32)
      if (!isfinite(x[r * ldx + c]) && f == ~0ull) f = static_cast<unsigned long long>(r) * cols + c;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, f, s);
      f = o < f ? o : f;
    }
    if (lane == 0 && f != ~0ull) atomicMin(first, f);
  }
}

// Squared row norms over the leading `dims` columns, double accumulation rounded to
// fp32 (preprocess.py:95-101).  One warp per row.
__global__ void row_sq_norms_kernel(const float* __restrict__ x, long long ldx, int rows, int dims,
                                    float* __restrict__ out) {
  const int warps_per_block = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = blockIdx.x * (long long)warps_per_block + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * warps_per_block) {
    const float* row = x + r * ldx;
    double s = 0.0;
    for (int c = lane; c < dims; c += 32) {
      const double v = row[c];
      s += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = static_cast<float>(s);
  }
}

// out[r, :] = in[idx[r], :]  (cols wide, padded leading dims)
__global__ void gather_rows_kernel(const float* __restrict__ in, long long ldi, const long long* __restrict__ idx,
                                   int rows, int cols, float* __restrict__ out, long long ldo) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols;
    const int c = static_cast<int>(e - r * cols);
    out[r * ldo + c] = in[idx[r] * ldi + c];
  }
}

__global__ void gather_rows_i32_kernel(const float* __restrict__ in, long long ldi, const int* __restrict__ idx,
                                       int rows, int cols, float* __restrict__ out, long long ldo) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols;
    const int c = static_cast<int>(e - r * cols);
    out[r * ldo + c] = in[static_cast<long long>(idx[r]) * ldi + c];
  }
}

// tau_i = sum_t (x_it - c_{a_i,t})^2, ascending t, separate mul/add (_kernels.pyx:85-103).
// One thread per row runs its own sequential chain; 32-column chunks of the CTA's 128 rows
// (and of their assigned centroid rows) are loaded coalesced into registers one chunk ahead
// (software pipelining), parked in padded shared memory, then consumed row-wise.
constexpr int SEED_ROWS = 128;
constexpr int SEED_PER = 32;  // elements per thread per chunk (128 rows x 32 cols / 128 threads)
__global__ void __launch_bounds__(SEED_ROWS)
    seed_thresholds_kernel(const float* __restrict__ x, long long ldx, const float* __restrict__ cent, long long ldc,
                           const int* __restrict__ assign, int n, int d, float* __restrict__ out) {
  __shared__ float xs[SEED_ROWS][33];
  __shared__ float cs[SEED_ROWS][33];
  __shared__ int sa[SEED_ROWS];
  const int r0 = blockIdx.x * SEED_ROWS;
  const int tid = threadIdx.x;
  sa[tid] = (r0 + tid < n) ? assign[r0 + tid] : 0;
  __syncthreads();
  // thread tid loads column (tid & 31) of rows (tid >> 5) + 4*m, m < 32
  const int lc = tid & 31, lr = tid >> 5;
  float px[SEED_PER], pc[SEED_PER];
  auto load_chunk = [&](int t0) {
    const int col = t0 + lc;
#pragma unroll
    for (int m = 0; m < SEED_PER; ++m) {
      const int r = lr + 4 * m;
      const int row = r0 + r;
      const bool ok = row < n && col < d;
      px[m] = ok ? __ldg(x + static_cast<long long>(row) * ldx + col) : 0.0f;
      pc[m] = ok ? __ldg(cent + static_cast<long long>(sa[r]) * ldc + col) : 0.0f;
    }
  };
  float acc = 0.0f;
  load_chunk(0);
  for (int t0 = 0; t0 < d; t0 += 32) {
    __syncthreads();
#pragma unroll
    for (int m = 0; m < SEED_PER; ++m) {
      xs[lr + 4 * m][lc] = px[m];
      cs[lr + 4 * m][lc] = pc[m];
    }
    __syncthreads();
    if (t0 + 32 < d) load_chunk(t0 + 32);  // next chunk in flight while this one is consumed
    const int lim = min(32, d - t0);
#pragma unroll 8
    for (int tt = 0; tt < lim; ++tt) {
      const float diff = __fsub_rn(xs[tid][tt], cs[tid][tt]);
      acc = __fadd_rn(acc, __fmul_rn(diff, diff));
    }
  }
  if (r0 + tid < n) out[r0 + tid] = acc;
}

// Same chain as seed_thresholds_kernel, fed by 16-byte zero-filling cp.async copies straight
// into a double-buffered [row][36] shared tile (no register round trip, row pointers hoisted out
// of the chunk loop, LDS.128 reads); the zero-filled columns past d add +0.0 to a non-negative
// running sum, so the result is bitwise the d-column chain.  Needs 16-byte aligned rows.
constexpr int SEEDA_LD = 36;  // padded row (floats): LDS.128 quarter-warps hit 8 distinct bank groups
constexpr int SEEDA_SMEM = 2 * 2 * SEED_ROWS * SEEDA_LD * 4;
// PAIR = 0: seed_thresholds (sub / mul / add chain, _kernels.pyx:97-103).
// PAIR = 1 / 2: the exact squared distance the reference's GEMM + expansion gives the pair
// (row, assign[row]) (distance.py:58-82): the fma (OpenBLAS, K blocks of q) or mul+add
// (portable) inner-product chain of sgemm_chain.cuh, then max(0, fl(fl(-2 ip + xsq) + ysq)).
// Used after the tensor-core argmin of a full pass to give tau its reference bits.
template <int PAIR>
__global__ void __launch_bounds__(SEED_ROWS)
    seed_thresholds_async_kernel(const float* __restrict__ x, long long ldx, const float* __restrict__ cent,
                                 long long ldc, const int* __restrict__ assign, int n, int d,
                                 float* __restrict__ out, const float* __restrict__ xsq = nullptr,
                                 const float* __restrict__ ysq = nullptr, int kq = 0) {
  extern __shared__ __align__(16) float seed_smem[];  // [buf][x|c][row][SEEDA_LD], 73.7 KB
  auto tile = reinterpret_cast<float(*)[2][SEED_ROWS][SEEDA_LD]>(seed_smem);
  const int r0 = blockIdx.x * SEED_ROWS;
  const int tid = threadIdx.x;
  // copy mapping: segment s = tid + 128 i (i < 8) -> row s / 8, 16-byte column group s % 8
  const int q = tid & 7;
  const float* xp[8];
  const float* cp[8];
  int rowq[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (tid >> 3) + 16 * i;
    rowq[i] = r;
    const int row = r0 + r;
    const bool ok = row < n;
    xp[i] = ok ? x + static_cast<long long>(row) * ldx + 4 * q : nullptr;
    cp[i] = ok ? cent + static_cast<long long>(__ldg(assign + row)) * ldc + 4 * q : nullptr;
  }
  auto issue = [&](int t0, int buf) {
    const int rem = d - t0 - 4 * q;  // valid floats from this thread's column group on
    const int bytes = rem >= 4 ? 16 : (rem > 0 ? 4 * rem : 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = xp[i] ? bytes : 0;
      cp_async_16_zfill(&tile[buf][0][rowq[i]][4 * q], b ? xp[i] + t0 : x, b);
      cp_async_16_zfill(&tile[buf][1][rowq[i]][4 * q], b ? cp[i] + t0 : cent, b);
    }
    cp_async_commit();
  };
  const int nchunk = (d + 31) / 32;
  float acc = 0.0f;
  float tot = 0.0f;                                   // PAIR: finished K blocks
  int next_b = PAIR == 1 ? chain_next_boundary(0, d, kq) : d;  // PAIR 1: next K-block boundary
  issue(0, 0);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunk) {
      issue(32 * (ch + 1), buf ^ 1);
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const float4* xr = reinterpret_cast<const float4*>(&tile[buf][0][tid][0]);
    const float4* cr = reinterpret_cast<const float4*>(&tile[buf][1][tid][0]);
    if constexpr (PAIR == 0) {
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const float4 a = xr[v], c = cr[v];
        float df = __fsub_rn(a.x, c.x);
        acc = __fadd_rn(acc, __fmul_rn(df, df));
        df = __fsub_rn(a.y, c.y);
        acc = __fadd_rn(acc, __fmul_rn(df, df));
        df = __fsub_rn(a.z, c.z);
        acc = __fadd_rn(acc, __fmul_rn(df, df));
        df = __fsub_rn(a.w, c.w);
        acc = __fadd_rn(acc, __fmul_rn(df, df));
      }
    } else {
      const int t0 = 32 * ch;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const float4 a = xr[v], c = cr[v];
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if constexpr (PAIR == 1) {
            if (t0 + 4 * v + u == next_b) {  // block boundary (uniform across the CTA)
              tot = __fadd_rn(tot, acc);
              acc = 0.0f;
              next_b = chain_next_boundary(next_b, d, kq);
            }
          }
          // columns past d are zero-filled: fma(0, 0, acc) == acc (acc is never -0)
          acc = chain_scalar_step<PAIR == 1 ? CHAIN_FMA : CHAIN_MULADD>(av[u], cv[u], acc);
        }
      }
    }
    __syncthreads();  // buf is refilled by the next iteration's issue
  }
  if (r0 + tid < n) {
    if constexpr (PAIR == 0) {
      out[r0 + tid] = acc;
    } else {
      const float ip = __fadd_rn(tot, acc);
      const float e = __fadd_rn(__fadd_rn(__fmul_rn(ip, -2.0f), xsq[r0 + tid]), ysq[__ldg(assign + r0 + tid)]);
      out[r0 + tid] = e > 0.0f ? e : 0.0f;
    }
  }
}

// Merge of the ARGMIN epilogue's per-split top-2 records (gemm_tf32x3.cuh): assign = lowest
// column among the smallest tensor-core distances; the row is flagged for an exact re-evaluation
// when the runner-up is within the rigorous error bound of both tensor-core values
// (|p_tc - p_exact| <= kap * (xsq + ysq_max + p)), i.e. when the exact
// chain-based distances could order differently or tie.
__global__ void argmin_merge_kernel(const int4* __restrict__ top, int n_split, int n, const float* __restrict__ xsq,
                                    const float* __restrict__ ysq_max, float kap, int* __restrict__ assign,
                                    float* __restrict__ tau, int* __restrict__ amb_rows,
                                    unsigned int* __restrict__ amb_count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 t = top[i];
  float best = __int_as_float(t.x), second = __int_as_float(t.z);
  int bj = t.y;
  for (int s = 1; s < n_split; ++s) {
    const int4 u = top[static_cast<long long>(s) * n + i];
    const float b1 = __int_as_float(u.x), s1 = __int_as_float(u.z);
    if (b1 < best || (b1 == best && u.y < bj)) {
      second = fminf(best, s1);
      best = b1;
      bj = u.y;
    } else {
      second = fminf(second, b1);
    }
  }
  assign[i] = bj;
  tau[i] = best;
  if (isfinite(second)) {
    const float base = xsq[i] + *ysq_max;
    const float margin = kap * (2.0f * base + best + second);
    if (second - best <= margin) amb_rows[atomicAdd(amb_count, 1u)] = i;
  }
}

// Exact argmin of dense distance rows (lowest column on ties): one warp per row.
__global__ void dense_argmin_kernel(const float* __restrict__ dist, long long ld, int rows, int cols,
                                    const int* __restrict__ row_ids, int* __restrict__ assign,
                                    float* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  for (long long r = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * (blockDim.x >> 5)) {
    const float* p = dist + r * ld;
    float bv = __int_as_float(0x7f800000);
    int bj = 0x7fffffff;
    for (int j = lane; j < cols; j += 32) {
      const float v = p[j];
      if (v < bv) { bv = v; bj = j; }  // ascending j per lane: first occurrence kept
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov < bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
    }
    if (lane == 0) {
      const int g = row_ids[r];
      assign[g] = bj;
      tau[g] = bv;
    }
  }
}

// max over the column norms (one CTA)
__global__ void max_f32_kernel(const float* __restrict__ v, int n, float* __restrict__ out) {
  __shared__ float red[32];
  float m = 0.0f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
  }
}

__device__ __forceinline__ void warp_add_u64(unsigned long long v, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Bit-exact device twin of the reference's bank scan (_kernels.pyx:14-82): one thread per
// vector, PDX tail (dim-major within each block), sequential-tau semantics.  This is the
// parity entry of the kernel protocol; the fused production scan lives in scan.cuh.
__global__ void scan_bank_pdx_kernel(const float* __restrict__ pd, int n, int kb, const float* __restrict__ x,
                                     long long ldx, const float* __restrict__ tail,
                                     const long long* __restrict__ block_offsets, const int* __restrict__ block_dims,
                                     int n_blocks, const float* __restrict__ theta, int d_prime, int bank_offset,
                                     float* __restrict__ tau, int* __restrict__ assign, int sentinel,
                                     unsigned long long* __restrict__ counters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long surv = 0, touched = 0;
  if (i < n) {
    float tcur = tau[i];
    int best = assign[i];
    const float* prow = pd + static_cast<long long>(i) * kb;
    const float* xrow = x + static_cast<long long>(i) * ldx;
    for (int j = 0; j < kb; ++j) {
      float gate = sentinel ? kInf : __fmul_rn(tcur, theta[0]);
      const float p = prow[j];
      if (p > gate) continue;
      ++surv;
      float running = p;
      bool pruned = false;
      int xoff = d_prime;
      for (int b = 0; b < n_blocks; ++b) {
        const int bd = block_dims[b];
        const float* col = tail + block_offsets[b] + j;
        float acc = 0.0f;
        for (int t = 0; t < bd; ++t) {
          const float diff = __fsub_rn(xrow[xoff + t], col[static_cast<long long>(t) * kb]);
          acc = __fadd_rn(acc, __fmul_rn(diff, diff));
        }
        touched += bd;
        running = __fadd_rn(running, acc);
        xoff += bd;
        gate = (sentinel && b < n_blocks - 1) ? kInf : __fmul_rn(tcur, theta[b + 1]);
        if (running > gate) { pruned = true; break; }
      }
      if (!pruned) {
        if (running < tcur) {
          best = bank_offset + j;
          tcur = running;
        } else if (running == tcur && bank_offset + j < best) {
          best = bank_offset + j;
        }
      }
    }
    tau[i] = tcur;
    assign[i] = best;
  }
  warp_add_u64(surv, &counters[0]);
  warp_add_u64(touched, &counters[1]);
}

// out[i, l] = sum_{t<dims} a[i,t] * b[l,t], one thread per cell, ascending t, no FMA:
// bitwise the compiled portable_matmul (_kernels.pyx:122-142, built -ffp-contract=off).
__global__ void portable_matmul_kernel(const float* __restrict__ a, long long lda, const float* __restrict__ b,
                                       long long ldb, int n, int m, int dims, float* __restrict__ out, long long ldo) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * m) return;
  const long long i = e / m;
  const int l = static_cast<int>(e - i * m);
  const float* ar = a + i * lda;
  const float* br = b + static_cast<long long>(l) * ldb;
  float acc = 0.0f;
  for (int t = 0; t < dims; ++t) acc = __fadd_rn(acc, __fmul_rn(ar[t], br[t]));
  out[i * ldo + l] = acc;
}

// keys (dist_bits << 32 | col) -> assign / tau
// Per-block partials of sum(tau) (f64) and count(assign != prev); fixed-order final pass.
constexpr int STAT_THREADS = 256;
__global__ void __launch_bounds__(STAT_THREADS)
    assign_stats_partial_kernel(const float* __restrict__ tau, const int* __restrict__ assign,
                                const int* __restrict__ prev, int n, double* __restrict__ part_sum,
                                unsigned long long* __restrict__ part_cnt) {
  __shared__ double ss[STAT_THREADS];
  __shared__ unsigned long long sc[STAT_THREADS];
  double s = 0.0;
  unsigned long long c = 0;
  const long long per = ((long long)n + gridDim.x - 1) / gridDim.x;
  const long long beg = per * blockIdx.x, end = min((long long)n, beg + per);
  for (long long i = beg + threadIdx.x; i < end; i += STAT_THREADS) {
    s += static_cast<double>(tau[i]);
    if (prev) c += (assign[i] != prev[i]);
  }
  ss[threadIdx.x] = s;
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int o = STAT_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      ss[threadIdx.x] += ss[threadIdx.x + o];
      sc[threadIdx.x] += sc[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part_sum[blockIdx.x] = ss[0];
    part_cnt[blockIdx.x] = sc[0];
  }
}

// wcss = float(np.sum(tau, dtype=np.float64)) (core.py:344), bitwise: NumPy reduces the f32 array
// through 8192-element cast buffers, adding each buffer's pairwise sum (DOUBLE_pairwise_sum:
// blocks of <= 128 with 8 interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// larger spans halved at a multiple of 8) to the running result in buffer order
// (tools/blas_order_probe.py checks this model against np.sum).
constexpr int NP_SUM_BUF = 8192;
__device__ __forceinline__ double np_pairwise_leaf(const float* __restrict__ a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, static_cast<double>(a[i]));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], static_cast<double>(a[i + j]));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, static_cast<double>(a[i]));
  return res;
}

// the recursion pairwise(a, n) = pairwise(a, n2) + pairwise(a + n2, n - n2) for n > 128, evaluated
// with an explicit stack (device recursion overflowed the default per-thread stack)
__device__ double np_pairwise_f32(const float* __restrict__ a, int n) {
  int lo_s[16], n_s[16], stage[16];
  double left[16];
  int top = 0;
  lo_s[0] = 0;
  n_s[0] = n;
  stage[0] = 0;
  double ret = 0.0;
  while (top >= 0) {
    const int m = n_s[top];
    if (m <= 128) {
      ret = np_pairwise_leaf(a + lo_s[top], m);
      --top;
      continue;
    }
    int m2 = m / 2;
    m2 -= m2 % 8;
    if (stage[top] == 0) {  // descend left
      stage[top] = 1;
      lo_s[top + 1] = lo_s[top];
      n_s[top + 1] = m2;
      stage[top + 1] = 0;
      ++top;
    } else if (stage[top] == 1) {  // left done: descend right
      left[top] = ret;
      stage[top] = 2;
      lo_s[top + 1] = lo_s[top] + m2;
      n_s[top + 1] = m - m2;
      stage[top + 1] = 0;
      ++top;
    } else {  // both done
      ret = __dadd_rn(left[top], ret);
      --top;
    }
  }
  return ret;
}

// one CTA of 64 threads per 8192-element buffer: a full buffer's recursion is the balanced tree over
// 64 leaves of 128 (every split is an exact half, a multiple of 8), combined left + right level by
// level; a ragged last buffer takes the general recursion on one thread
__global__ void np_sum_chunks_kernel(const float* __restrict__ v, long long n, double* __restrict__ part) {
  __shared__ double leaf[64];
  const long long c = blockIdx.x;
  const long long lo = c * NP_SUM_BUF;
  const int len = static_cast<int>(min((long long)NP_SUM_BUF, n - lo));
  const int t = threadIdx.x;
  if (len == NP_SUM_BUF) {
    leaf[t] = np_pairwise_leaf(v + lo + 128 * t, 128);
    __syncthreads();
    for (int w = 1; w < 64; w *= 2) {
      if ((t & (2 * w - 1)) == 0) leaf[t] = __dadd_rn(leaf[t], leaf[t + w]);
      __syncthreads();
    }
    if (t == 0) part[c] = leaf[0];
  } else if (t == 0) {
    part[c] = np_pairwise_f32(v + lo, len);
  }
}

// Exact argmin over a row's candidate list (ascending columns, from a tensor-core GATE pass that
// kept every column whose exact distance may tie the best): the reference's chain distance of
// each candidate, smallest value, lowest column on ties.  One warp per row, a lane per candidate.
__global__ void cand_exact_argmin_kernel(const int* __restrict__ rows, int n_rows, const int2* __restrict__ cand,
                                         const int* __restrict__ cand_cnt, int cap, const float* __restrict__ x,
                                         long long ldx, const float* __restrict__ cent, long long ldc, int d,
                                         const float* __restrict__ xsq, const float* __restrict__ ysq, int flavour,
                                         int q, int* __restrict__ assign, float* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows; r += gridDim.x * (blockDim.x >> 5)) {
    const int cnt = cand_cnt[r];
    if (cnt > cap) continue;  // overflow: the caller re-evaluates the whole row
    const int g = rows[r];
    const float* xr = x + static_cast<long long>(g) * ldx;
    float bv = __int_as_float(0x7f800000);
    int bj = 0x7fffffff;
    for (int e = lane; e < cnt; e += 32) {
      const int j = cand[static_cast<long long>(r) * cap + e].x & 0x7fffffff;
      const float* cr = cent + static_cast<long long>(j) * ldc;
      const float ip = flavour == 0 ? exact_dot<CHAIN_FMA>(xr, cr, d, q) : exact_dot<CHAIN_MULADD>(xr, cr, d, 0);
      float v = __fadd_rn(__fadd_rn(__fmul_rn(ip, -2.0f), xsq[g]), ysq[j]);
      v = v > 0.0f ? v : 0.0f;
      if (v < bv || (v == bv && j < bj)) { bv = v; bj = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov < bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
    }
    if (lane == 0) {
      assign[g] = bj;
      tau[g] = bv;
    }
  }
}

// GATE threshold for re-evaluating ambiguous argmin rows: every column whose exact distance may
// be <= the exact best; thr = best~ + 2 kap (xsq + ysq_max + best~ + D) with headroom, rounded up
__global__ void argmin_cand_threshold_kernel(const int* __restrict__ rows, int n_rows, const float* __restrict__ tau,
                                             const float* __restrict__ xsq, const float* __restrict__ ysq_max,
                                             float kap, float* __restrict__ thr, float* __restrict__ xs_out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int g = rows[r];
  const double b = tau[g], base = static_cast<double>(xsq[g]) + *ysq_max;
  const double dl = kap * (base + b);
  thr[r] = __double2float_ru((b + 2.0 * dl + 2.0 * kap * (base + b + 2.0 * dl)) * (1.0 + 0x1p-20));
  xs_out[r] = xsq[g];
}

__global__ void assign_stats_final_kernel(const double* __restrict__ chunk_sum, int chunks,
                                          const unsigned long long* __restrict__ part_cnt, int parts,
                                          double* __restrict__ out_sum, unsigned long long* __restrict__ out_cnt) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int p = 0; p < chunks; ++p) s = __dadd_rn(s, chunk_sum[p]);
    unsigned long long c = 0;
    for (int p = 0; p < parts; ++p) c += part_cnt[p];
    *out_sum = s;
    *out_cnt = c;
  }
}

// Empty-cluster splits decided on the host (core.py:103-128): applied in list order so a
// donor split twice sees its already-shrunk row.  delta = row * eps * (+1,-1,...).
__global__ void apply_splits_kernel(float* __restrict__ cent, long long ldc, int d, const int* __restrict__ empties,
                                    const int* __restrict__ donors, int n_splits, float eps) {
  for (int s = 0; s < n_splits; ++s) {
    const int e = empties[s], dn = donors[s];
    for (int t = threadIdx.x; t < d; t += blockDim.x) {
      const float row = cent[static_cast<long long>(dn) * ldc + t];
      const float sign = (t & 1) ? -1.0f : 1.0f;
      const float delta = __fmul_rn(__fmul_rn(row, eps), sign);
      cent[static_cast<long long>(e) * ldc + t] = __fadd_rn(row, delta);
      cent[static_cast<long long>(dn) * ldc + t] = __fsub_rn(row, delta);
    }
    __syncthreads();
  }
}

__global__ void iota_kernel(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

__global__ void copy_i32_kernel(const int* __restrict__ a, int* __restrict__ b, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}

__global__ void fill_f32_kernel(float* p, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace skm
