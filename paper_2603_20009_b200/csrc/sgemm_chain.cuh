// Exact-chain fp32 GEMM on the CUDA cores: out[i][j] = chain_t A[i][t] * B[j][t], bitwise equal to
// the reference's GEMM backends.
//
// The reference computes every contraction with NumPy `@` -> OpenBLAS sgemm (distance.py:58-59,
// preprocess.py:43,52, evaluation.py:45) or, with gemm_backend="portable", with the Cython
// portable_matmul (_kernels.pyx:122-142).  Measured on the survey container (OpenBLAS 0.3.30,
// SkylakeX kernel, threaded driver; tools/blas_order_probe.py):
//   * each output element is ONE sequential fused-multiply-add chain over ascending t, starting
//     from +0 (the AVX-512 micro-kernel keeps one accumulator per output);
//   * K is blocked by the threaded level-3 driver with GEMM_Q = 448: while more than 2Q remain a
//     block of Q is taken, a remainder in (Q, 2Q) is halved as ceil(m/2), and every block's chain
//     restarts from +0 and is added to the running output with one fp32 add (C += alpha * acc);
//   * portable_matmul: one chain per output with separate rounded multiply and add (the
//     extension is built with -ffp-contract=off), no K blocking.
// A tensor-core product cannot reproduce those roundings (every step rounds the running sum), so
// the contractions whose every output bit matters downstream -- the rotation X.R and C.R^T, the
// ETR distance blocks -- run here; the large distance GEMMs of the Lloyd loop stay on the tensor
// cores and only their decisions near a tie are re-evaluated with the same chain (exact_dot below).
//
// Tiling: 128x128 output tile per 256-thread CTA, 16-deep k tiles double buffered through shared
// memory (A stored as duplicated pairs (a, a) so one 64-bit load feeds a packed f32x2 operand),
// 8x8 outputs per thread as 32 packed pairs: one fma.rn.f32x2 (FFMA2) computes two outputs' chain
// steps, each lane-exact IEEE fma (measured 74 TFLOP/s peak for FFMA2 on B200,
// tools/micro/ffma2_bench.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace skm {

constexpr int CH_BM = 128;
constexpr int CH_BN = 128;
constexpr int CH_BK = 16;
constexpr int CH_THREADS = 256;
constexpr int CH_Q = 448;  // OpenBLAS SkylakeX SGEMM_DEFAULT_Q (threaded driver K blocking)

enum ChainFlavour : int { CHAIN_FMA = 0, CHAIN_MULADD = 1 };
enum ChainMode : int { CHAIN_STORE = 0, CHAIN_DIST = 1 };

struct ChainArgs {
  const float* a;  // row-major, at the K block's first column
  long long lda;
  const float* b;
  long long ldb;
  int M, N, K;       // K: this launch's K block
  float* out;
  long long ldo;
  const float* xsq;  // DIST: per-row norm term
  const float* ysq;  // DIST: per-column norm term
};

// next K-block boundary after `k0` under the threaded OpenBLAS rule (q == 0: no blocking)
__host__ __device__ __forceinline__ int chain_next_boundary(int k0, int K, int q) {
  if (q <= 0) return K;
  const int m = K - k0;
  if (m >= 2 * q) return k0 + q;
  if (m > q) return k0 + (m + 1) / 2;
  return K;
}

__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  return static_cast<unsigned long long>(__float_as_uint(lo)) |
         (static_cast<unsigned long long>(__float_as_uint(hi)) << 32);
}
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float(static_cast<unsigned>(v)); }
__device__ __forceinline__ float f2_hi(unsigned long long v) { return __uint_as_float(static_cast<unsigned>(v >> 32)); }

template <int FLAVOUR>
__device__ __forceinline__ unsigned long long chain_step2(unsigned long long a, unsigned long long b,
                                                          unsigned long long c) {
  unsigned long long d;
  if constexpr (FLAVOUR == CHAIN_FMA) {
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  } else {
    // scalar mul.rn / add.rn: ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (observed in
    // the SASS), which would silently turn the portable chain into the fma chain
    d = f2_pack(__fadd_rn(f2_lo(c), __fmul_rn(f2_lo(a), f2_lo(b))),
                __fadd_rn(f2_hi(c), __fmul_rn(f2_hi(a), f2_hi(b))));
  }
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// One output's chain, scalar: used to re-evaluate single (row, centroid) pairs exactly.
template <int FLAVOUR>
__device__ __forceinline__ float chain_scalar_step(float a, float b, float c) {
  if constexpr (FLAVOUR == CHAIN_FMA) return __fmaf_rn(a, b, c);
  return __fadd_rn(c, __fmul_rn(a, b));
}

template <int FLAVOUR>
__device__ float exact_dot(const float* __restrict__ x, const float* __restrict__ y, int K, int q) {
  float tot = 0.0f;
  int k0 = 0;
  while (k0 < K) {
    const int k1 = chain_next_boundary(k0, K, q);
    float acc = 0.0f;
    int t = k0;
    if ((((reinterpret_cast<uintptr_t>(x + t) | reinterpret_cast<uintptr_t>(y + t)) & 15) == 0)) {
      for (; t + 4 <= k1; t += 4) {
        const float4 u = *reinterpret_cast<const float4*>(x + t);
        const float4 v = *reinterpret_cast<const float4*>(y + t);
        acc = chain_scalar_step<FLAVOUR>(u.x, v.x, acc);
        acc = chain_scalar_step<FLAVOUR>(u.y, v.y, acc);
        acc = chain_scalar_step<FLAVOUR>(u.z, v.z, acc);
        acc = chain_scalar_step<FLAVOUR>(u.w, v.w, acc);
      }
    }
    for (; t < k1; ++t) acc = chain_scalar_step<FLAVOUR>(x[t], y[t], acc);
    tot = __fadd_rn(tot, acc);  // first block: +0 + acc == acc (acc is never -0)
    k0 = k1;
  }
  return tot;
}

// One launch computes one K block of the blocked driver: each output's chain over the block
// starts from +0; ACC = 1 adds it to the previous blocks' sum already in `out` (OpenBLAS's
// C += alpha * A_blk * B_blk with alpha = 1: one fp32 add), so a K-blocked product is a sequence
// of launches -- exactly the reference's association order -- and no block needs a second set of
// accumulator registers (124 registers: two CTAs per SM).
template <int FLAVOUR, int MODE, int ACC>
#ifndef SKM_CHAIN_PREFETCH
#define SKM_CHAIN_PREFETCH 1  // measured 36.2 -> 37.8 TFLOP/s at the c2 rotation shape
#endif
#ifndef SKM_CHAIN_MINB
#define SKM_CHAIN_MINB 2
#endif
__global__ void __launch_bounds__(CH_THREADS, SKM_CHAIN_MINB) sgemm_chain_kernel(const ChainArgs g) {
  extern __shared__ __align__(16) uint8_t ch_smem[];
  // As2[buf][k][m] = (a, a) pairs, Bs[buf][k][n]
  unsigned long long* As2 = reinterpret_cast<unsigned long long*>(ch_smem);
  float* Bs = reinterpret_cast<float*>(ch_smem + 2 * CH_BK * CH_BM * 8);
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * CH_BM, n0 = blockIdx.x * CH_BN;
  const bool vec = ((g.lda | g.ldb) & 3) == 0 && (g.K & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(g.a) | reinterpret_cast<uintptr_t>(g.b)) & 15) == 0;
  // global -> register staging: thread loads 8 k-values of one A row and one B row
  const int lr = tid >> 1, lk = (tid & 1) * 8;
  const long long arow = m0 + lr, brow = n0 + lr;
  float ra[8], rb[8];
  auto gload = [&](int k0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kk = k0 + lk + 4 * h;
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      if (vec) {
        if (arow < g.M && kk < g.K) va = __ldg(reinterpret_cast<const float4*>(g.a + arow * g.lda + kk));
        if (brow < g.N && kk < g.K) vb = __ldg(reinterpret_cast<const float4*>(g.b + brow * g.ldb + kk));
      } else {
        float* pa = &va.x;
        float* pb = &vb.x;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (arow < g.M && kk + u < g.K) pa[u] = g.a[arow * g.lda + kk + u];
          if (brow < g.N && kk + u < g.K) pb[u] = g.b[brow * g.ldb + kk + u];
        }
      }
      ra[4 * h + 0] = va.x; ra[4 * h + 1] = va.y; ra[4 * h + 2] = va.z; ra[4 * h + 3] = va.w;
      rb[4 * h + 0] = vb.x; rb[4 * h + 1] = vb.y; rb[4 * h + 2] = vb.z; rb[4 * h + 3] = vb.w;
    }
  };
  auto sstore = [&](int buf) {
    unsigned long long* A = As2 + buf * CH_BK * CH_BM;
    float* B = Bs + buf * CH_BK * CH_BN;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      A[(lk + u) * CH_BM + lr] = f2_pack(ra[u], ra[u]);
      B[(lk + u) * CH_BN + lr] = rb[u];
    }
  };

  unsigned long long acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;

  const int ntile = (g.K + CH_BK - 1) / CH_BK;
  const int kfull = g.K / CH_BK;  // tiles without a ragged end
  if (ntile > 0) {
    gload(0);
    sstore(0);
  }
  __syncthreads();
  for (int kt = 0; kt < ntile; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ntile) gload((kt + 1) * CH_BK);
    const unsigned long long* A = As2 + buf * CH_BK * CH_BM;
    const float* B = Bs + buf * CH_BK * CH_BN;
    auto step = [&](int kk) {
      const ulonglong2* Ak = reinterpret_cast<const ulonglong2*>(A + kk * CH_BM);
      const ulonglong2 a01 = Ak[ty * 2], a23 = Ak[ty * 2 + 1];
      const ulonglong2 a45 = Ak[32 + ty * 2], a67 = Ak[32 + ty * 2 + 1];
      const unsigned long long av[8] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y, a67.x, a67.y};
      const ulonglong2 b03 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + tx * 4);
      const ulonglong2 b47 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + 64 + tx * 4);
      const unsigned long long bv[4] = {b03.x, b03.y, b47.x, b47.y};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = chain_step2<FLAVOUR>(av[i], bv[j], acc[i][j]);
    };
    if (kt < kfull) {
#if SKM_CHAIN_PREFETCH
      // fragments of step kk + 1 are loaded while step kk's FFMA2s run
      auto lda_ = [&](int kk, unsigned long long* av, unsigned long long* bv) {
        const ulonglong2* Ak = reinterpret_cast<const ulonglong2*>(A + kk * CH_BM);
        const ulonglong2 a01 = Ak[ty * 2], a23 = Ak[ty * 2 + 1];
        const ulonglong2 a45 = Ak[32 + ty * 2], a67 = Ak[32 + ty * 2 + 1];
        av[0] = a01.x; av[1] = a01.y; av[2] = a23.x; av[3] = a23.y;
        av[4] = a45.x; av[5] = a45.y; av[6] = a67.x; av[7] = a67.y;
        const ulonglong2 b03 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + tx * 4);
        const ulonglong2 b47 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + 64 + tx * 4);
        bv[0] = b03.x; bv[1] = b03.y; bv[2] = b47.x; bv[3] = b47.y;
      };
      unsigned long long fa[2][8], fb[2][4];
      lda_(0, fa[0], fb[0]);
#pragma unroll
      for (int kk = 0; kk < CH_BK; ++kk) {
        if (kk + 1 < CH_BK) lda_(kk + 1, fa[(kk + 1) & 1], fb[(kk + 1) & 1]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i][j] = chain_step2<FLAVOUR>(fa[kk & 1][i], fb[kk & 1][j], acc[i][j]);
      }
#else
#pragma unroll
      for (int kk = 0; kk < CH_BK; ++kk) step(kk);
#endif
    } else {
      // ragged last tile: the zero-padded columns past K must not enter the chain
      // (+0 added to a -0 running value would flip its sign)
#pragma unroll 1
      for (int kk = 0; kk < g.K - kt * CH_BK; ++kk) step(kk);
    }
    if (kt + 1 < ntile) sstore(buf ^ 1);
    __syncthreads();
  }
  // epilogue: rows ty*4 + {0..3}, 64 + ty*4 + {0..3}; columns tx*4 + {0..3}, 64 + tx*4 + {0..3}
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (r >= g.M) continue;
    float xs = 0.0f;
    if constexpr (MODE == CHAIN_DIST) xs = g.xsq[r];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c0 = n0 + h * 64 + tx * 4;
      float v[4] = {f2_lo(acc[i][2 * h]), f2_hi(acc[i][2 * h]), f2_lo(acc[i][2 * h + 1]), f2_hi(acc[i][2 * h + 1])};
      float* o = g.out + r * g.ldo + c0;
      const bool vec_o = c0 + 4 <= g.N && ((reinterpret_cast<uintptr_t>(o) & 15) == 0);
      if constexpr (ACC) {  // previous K blocks' sum + this block's chain (one fp32 add)
        if (vec_o) {
          const float4 p = *reinterpret_cast<const float4*>(o);
          v[0] = __fadd_rn(p.x, v[0]); v[1] = __fadd_rn(p.y, v[1]); v[2] = __fadd_rn(p.z, v[2]); v[3] = __fadd_rn(p.w, v[3]);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c0 + u < g.N) v[u] = __fadd_rn(o[u], v[u]);
        }
      }
      if constexpr (MODE == CHAIN_DIST) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (c0 + u < g.N) {
            const float e = __fadd_rn(__fadd_rn(__fmul_rn(v[u], -2.0f), xs), g.ysq[c0 + u]);
            v[u] = e > 0.0f ? e : 0.0f;
          }
        }
      }
      if (vec_o) {
        *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < g.N) o[u] = v[u];
      }
    }
  }
}

// ---- k-major B operand (B[t][j], e.g. the rotation R for x @ R): cp.async pipeline -------------
// Same per-output chains and K-block launches as sgemm_chain_kernel; the B tile is a plain copy of
// B rows (no transpose), so both operands stream through a KN_STAGES-deep cp.async ring without
// register staging, and A stays in its row-major [m][k] layout (read as float2 = 2 chain steps of
// one row).  A's scalar is the broadcast operand of FFMA2 (`R.F32` in the SASS), so it is not
// duplicated in shared memory.
#ifndef SKM_KN_STAGES
#define SKM_KN_STAGES 2
#endif
#ifndef SKM_KN_BK
#define SKM_KN_BK 32
#endif
#ifndef SKM_KN_PREFETCH
#define SKM_KN_PREFETCH 1
#endif
constexpr int KN_STAGES = SKM_KN_STAGES;
constexpr int KN_BK = SKM_KN_BK;   // k depth of one pipeline stage
constexpr int KN_ALD = KN_BK + 4;  // A row stride in floats (80 B: 16-B aligned chunks, rows 4 apart hit other banks)

__device__ __forceinline__ unsigned long long ffma2_bcast(float a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("{\n\t.reg .b64 ap;\n\tmov.b64 ap, {%1, %1};\n\tfma.rn.f32x2 %0, ap, %2, %3;\n\t}"
      : "=l"(d) : "f"(a), "l"(b), "l"(c));
  return d;
}

template <int FLAVOUR>
__device__ __forceinline__ unsigned long long chain_step_bcast(float a, unsigned long long b, unsigned long long c) {
  if constexpr (FLAVOUR == CHAIN_FMA) {
    return ffma2_bcast(a, b, c);
  } else {
    return f2_pack(__fadd_rn(f2_lo(c), __fmul_rn(a, f2_lo(b))), __fadd_rn(f2_hi(c), __fmul_rn(a, f2_hi(b))));
  }
}

inline size_t chain_kn_smem_bytes() { return (size_t)KN_STAGES * (CH_BM * KN_ALD + KN_BK * CH_BN) * 4; }

// requires lda, ldb % 4 == 0 and 16-B aligned a, b (the launcher checks and falls back otherwise)
template <int FLAVOUR, int MODE, int ACC>
__global__ void __launch_bounds__(CH_THREADS, 2) sgemm_chain_kn_kernel(const ChainArgs g) {
  extern __shared__ __align__(16) uint8_t kn_smem[];
  float* As = reinterpret_cast<float*>(kn_smem);                 // [S][BM][KN_ALD]
  float* Bs = As + KN_STAGES * CH_BM * KN_ALD;                    // [S][BK][BN]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * CH_BM, n0 = blockIdx.x * CH_BN;
  const int ntile = (g.K + KN_BK - 1) / KN_BK;
  const int kfull = g.K / KN_BK;
  const bool a_vec = ((reinterpret_cast<uintptr_t>(g.a) & 15) == 0) && (g.lda & 3) == 0;

  auto issue = [&](int kt) {
    const int st = kt % KN_STAGES;
    const int k0 = kt * KN_BK;
#pragma unroll
    for (int h = 0; h < KN_BK / 8; ++h) {
      const int c = tid + h * CH_THREADS;
      // A: row c / (KN_BK / 4), 4-float chunk c % (KN_BK / 4)
      const int ar = c / (KN_BK / 4), ak = (c % (KN_BK / 4)) * 4;
      const long long grow = m0 + ar;
      const int kk = k0 + ak;
      int bytes = 0;
      if (grow < g.M && kk < g.K) bytes = 4 * min(4, g.K - kk);
      const float* src = bytes ? g.a + grow * g.lda + kk : g.a;
      if (a_vec) {
        cp_async_16_zfill(As + (st * CH_BM + ar) * KN_ALD + ak, src, bytes);
      } else {  // K block starting off a 16-byte boundary (odd halves of the blocked driver)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          cp_async_4_zfill(As + (st * CH_BM + ar) * KN_ALD + ak + u, 4 * u < bytes ? src + u : g.a,
                           4 * u < bytes ? 4 : 0);
      }
      // B: k row c >> 5, 4-column chunk c & 31
      const int bk = c >> 5, bn = (c & 31) * 4;
      const int kb = k0 + bk;
      const int col = n0 + bn;
      int bbytes = 0;
      if (kb < g.K && col < g.N) bbytes = 4 * min(4, g.N - col);
      const float* bsrc = bbytes ? g.b + (long long)kb * g.ldb + col : g.b;
      cp_async_16_zfill(Bs + (st * KN_BK + bk) * CH_BN + bn, bsrc, bbytes);
    }
  };

  unsigned long long acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;

#pragma unroll
  for (int s = 0; s < KN_STAGES - 1; ++s) {
    if (s < ntile) issue(s);
    cp_async_commit();
  }
  for (int kt = 0; kt < ntile; ++kt) {
    cp_async_wait_group<KN_STAGES - 2>();
    __syncthreads();
    if (kt + KN_STAGES - 1 < ntile) issue(kt + KN_STAGES - 1);
    cp_async_commit();
    const int st = kt % KN_STAGES;
    const float* A = As + st * CH_BM * KN_ALD;
    const float* B = Bs + st * KN_BK * CH_BN;
    auto bload = [&](int kk, unsigned long long* bv) {
      const ulonglong2 b03 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + tx * 4);
      const ulonglong2 b47 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + 64 + tx * 4);
      bv[0] = b03.x; bv[1] = b03.y; bv[2] = b47.x; bv[3] = b47.y;
    };
    if (kt < kfull) {
#if SKM_KN_PREFETCH
      // fragments of step k2 + 2 are loaded while step k2's FFMA2s run
      float2 fa[2][8];
      unsigned long long fb0[2][4], fb1[2][4];
      auto frag = [&](int k2, float2* av, unsigned long long* b0, unsigned long long* b1) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
          av[i] = *reinterpret_cast<const float2*>(A + r * KN_ALD + k2);
        }
        bload(k2, b0);
        bload(k2 + 1, b1);
      };
      frag(0, fa[0], fb0[0], fb1[0]);
#pragma unroll
      for (int k2 = 0; k2 < KN_BK; k2 += 2) {
        const int cb = (k2 >> 1) & 1;
        if (k2 + 2 < KN_BK) frag(k2 + 2, fa[cb ^ 1], fb0[cb ^ 1], fb1[cb ^ 1]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(fa[cb][i].x, fb0[cb][j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(fa[cb][i].y, fb1[cb][j], acc[i][j]);
      }
#else
#pragma unroll
      for (int k2 = 0; k2 < KN_BK; k2 += 2) {
        float2 av[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
          av[i] = *reinterpret_cast<const float2*>(A + r * KN_ALD + k2);
        }
        unsigned long long b0[4], b1[4];
        bload(k2, b0);
        bload(k2 + 1, b1);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(av[i].x, b0[j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(av[i].y, b1[j], acc[i][j]);
      }
#endif
    } else {
      // ragged last tile: the zero-filled columns past K must not enter the chain
#pragma unroll 1
      for (int kk = 0; kk < g.K - kt * KN_BK; ++kk) {
        unsigned long long bv[4];
        bload(kk, bv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
          const float a = A[r * KN_ALD + kk];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(a, bv[j], acc[i][j]);
        }
      }
    }
  }
  cp_async_wait_all();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const long long r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (r >= g.M) continue;
    float xs = 0.0f;
    if constexpr (MODE == CHAIN_DIST) xs = g.xsq[r];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c0 = n0 + h * 64 + tx * 4;
      float v[4] = {f2_lo(acc[i][2 * h]), f2_hi(acc[i][2 * h]), f2_lo(acc[i][2 * h + 1]), f2_hi(acc[i][2 * h + 1])};
      float* o = g.out + r * g.ldo + c0;
      const bool vec_o = c0 + 4 <= g.N && ((reinterpret_cast<uintptr_t>(o) & 15) == 0);
      if constexpr (ACC) {
        if (vec_o) {
          const float4 p = *reinterpret_cast<const float4*>(o);
          v[0] = __fadd_rn(p.x, v[0]); v[1] = __fadd_rn(p.y, v[1]); v[2] = __fadd_rn(p.z, v[2]); v[3] = __fadd_rn(p.w, v[3]);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c0 + u < g.N) v[u] = __fadd_rn(o[u], v[u]);
        }
      }
      if constexpr (MODE == CHAIN_DIST) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (c0 + u < g.N) {
            const float e = __fadd_rn(__fadd_rn(__fmul_rn(v[u], -2.0f), xs), g.ysq[c0 + u]);
            v[u] = e > 0.0f ? e : 0.0f;
          }
        }
      }
      if (vec_o) {
        *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < g.N) o[u] = v[u];
      }
    }
  }
}

// ---- fused exact-chain distances + per-tile top-k (ETR ground truth, evaluation.py:53-75) -----
// Rows of the collection are the A operand (M = n rows, row-major) and the queries the k-major
// B operand (B[t][q] = query q's column t): the cp.async pipeline of sgemm_chain_kn_kernel with
// 2 stages, EVERY K block of the blocked driver in one launch (each block's chain from +0, added
// to the running sum kept in shared memory with one fp32 add -- the association of the
// launch-per-block kernel), the expansion, and for each query column the k_top smallest
// (distance, row) of the tile, ascending, ties to the lower row:
// out[(query * n_tiles + tile) * k_top + r].  The distance matrix never reaches HBM; a radix top-k
// over the n_tiles * k_top survivors of each query finishes the selection in the same stable
// order (candidates are laid out tile by tile, each tile's in (value, row) order).
constexpr int TOPK_TILE_MAX = 32;
constexpr int KNT_STAGES = 2;
constexpr int KNT_ALD = CH_BK + 4;

struct ChainTopkArgs {
  const float* a;  // collection rows [M][K]
  long long lda;
  const float* b;  // queries, k-major [K][N]
  long long ldb;
  int M, N, K, q;
  const float* xsq;  // per row of a
  const float* ysq;  // per query
  int k_top;
  int n_tiles;       // ceil(M / 128)
  float* out_v;
  int* out_i;
  int col_offset;    // added to the row index
};

inline size_t chain_topk_smem_bytes() {
  return (size_t)KNT_STAGES * (CH_BM * KNT_ALD + CH_BK * CH_BN) * 4 + (size_t)CH_BM * CH_BN * 4;
}

template <int FLAVOUR>
__global__ void __launch_bounds__(CH_THREADS, 2) sgemm_chain_topk_kernel(const ChainTopkArgs g) {
  extern __shared__ __align__(16) uint8_t kt_smem[];
  float* As = reinterpret_cast<float*>(kt_smem);                 // [S][BM][KNT_ALD]
  float* Bs = As + KNT_STAGES * CH_BM * KNT_ALD;                   // [S][BK][BN]
  float* tot = Bs + KNT_STAGES * CH_BK * CH_BN;                   // [BM][BN] running sums
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * CH_BM, n0 = blockIdx.y * CH_BN;
  const bool a_al = ((reinterpret_cast<uintptr_t>(g.a) & 15) == 0) && (g.lda & 3) == 0;
  int k0 = 0;
  bool first = true;
  while (k0 < g.K) {
    const int k1 = chain_next_boundary(k0, g.K, FLAVOUR == CHAIN_FMA ? g.q : 0);
    const int KB = k1 - k0;
    const bool a_vec = a_al && (k0 & 3) == 0;
    const int ntile = (KB + CH_BK - 1) / CH_BK;
    const int kfull = KB / CH_BK;
    auto issue = [&](int kt) {
      const int st = kt % KNT_STAGES;
      const int kb0 = kt * CH_BK;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tid + h * CH_THREADS;
        const int ar = c >> 2, ak = (c & 3) * 4;
        const long long grow = m0 + ar;
        const int kk = kb0 + ak;
        int bytes = 0;
        if (grow < g.M && kk < KB) bytes = 4 * min(4, KB - kk);
        const float* src = bytes ? g.a + grow * g.lda + k0 + kk : g.a;
        if (a_vec) {
          cp_async_16_zfill(As + (st * CH_BM + ar) * KNT_ALD + ak, src, bytes);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            cp_async_4_zfill(As + (st * CH_BM + ar) * KNT_ALD + ak + u, 4 * u < bytes ? src + u : g.a,
                             4 * u < bytes ? 4 : 0);
        }
        const int bk = c >> 5, bn = (c & 31) * 4;
        const int kb = kb0 + bk;
        const int col = n0 + bn;
        int bbytes = 0;
        if (kb < KB && col < g.N) bbytes = 4 * min(4, g.N - col);
        const float* bsrc = bbytes ? g.b + (long long)(k0 + kb) * g.ldb + col : g.b;
        cp_async_16_zfill(Bs + (st * CH_BK + bk) * CH_BN + bn, bsrc, bbytes);
      }
    };
    unsigned long long acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;
    __syncthreads();  // the previous block's last stage reads are complete
#pragma unroll
    for (int s2 = 0; s2 < KNT_STAGES - 1; ++s2) {
      if (s2 < ntile) issue(s2);
      cp_async_commit();
    }
    for (int kt = 0; kt < ntile; ++kt) {
      cp_async_wait_group<KNT_STAGES - 2>();
      __syncthreads();
      if (kt + KNT_STAGES - 1 < ntile) issue(kt + KNT_STAGES - 1);
      cp_async_commit();
      const int st = kt % KNT_STAGES;
      const float* A = As + st * CH_BM * KNT_ALD;
      const float* B = Bs + st * CH_BK * CH_BN;
      auto bload = [&](int kk, unsigned long long* bv) {
        const ulonglong2 b03 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + tx * 4);
        const ulonglong2 b47 = *reinterpret_cast<const ulonglong2*>(B + kk * CH_BN + 64 + tx * 4);
        bv[0] = b03.x; bv[1] = b03.y; bv[2] = b47.x; bv[3] = b47.y;
      };
      if (kt < kfull) {
#pragma unroll
        for (int k2 = 0; k2 < CH_BK; k2 += 2) {
          float2 av[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
            av[i] = *reinterpret_cast<const float2*>(A + r * KNT_ALD + k2);
          }
          unsigned long long b0[4], b1[4];
          bload(k2, b0);
          bload(k2 + 1, b1);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(av[i].x, b0[j], acc[i][j]);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(av[i].y, b1[j], acc[i][j]);
        }
      } else {
#pragma unroll 1
        for (int kk = 0; kk < KB - kt * CH_BK; ++kk) {
          unsigned long long bv[4];
          bload(kk, bv);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
            const float a = A[r * KNT_ALD + kk];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = chain_step_bcast<FLAVOUR>(a, bv[j], acc[i][j]);
          }
        }
      }
    }
    cp_async_wait_all();
    // block chain -> running sum (C += A_blk * B_blk: one fp32 add; the first block is stored)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4* t = reinterpret_cast<float4*>(tot + r * CH_BN + h * 64 + tx * 4);
        float4 v = make_float4(f2_lo(acc[i][2 * h]), f2_hi(acc[i][2 * h]), f2_lo(acc[i][2 * h + 1]),
                               f2_hi(acc[i][2 * h + 1]));
        if (!first) {
          const float4 p = *t;
          v = make_float4(__fadd_rn(p.x, v.x), __fadd_rn(p.y, v.y), __fadd_rn(p.z, v.z), __fadd_rn(p.w, v.w));
        }
        *t = v;
      }
    }
    first = false;
    k0 = k1;
  }
  __syncthreads();
  if (tid < CH_BN && n0 + tid < g.N) {
    const int c = tid;  // query column
    const long long qcol = n0 + c;
    const float ys = g.ysq[qcol];
    const int valid = min(CH_BM, g.M - m0);
    float v[TOPK_TILE_MAX];
    int ix[TOPK_TILE_MAX];
    const int K = g.k_top;
    int cnt = 0;
    for (int r = 0; r < valid; ++r) {
      // expand_to_sq_l2 with the query as the "x" side (evaluation.py:42-50: vals = q . x^T * -2,
      // += q_sq, += x_sq): fl(fl(-2 ip + q_sq) + x_sq)
      const float e = __fadd_rn(__fadd_rn(__fmul_rn(tot[r * CH_BN + c], -2.0f), ys), __ldg(g.xsq + m0 + r));
      const float dv = e > 0.0f ? e : 0.0f;
      if (cnt < K || dv < v[K - 1]) {
        int p = cnt < K ? cnt : K - 1;
        while (p > 0 && v[p - 1] > dv) {
          v[p] = v[p - 1];
          ix[p] = ix[p - 1];
          --p;
        }
        v[p] = dv;
        ix[p] = r;
        if (cnt < K) ++cnt;
      }
    }
    const long long o = (qcol * g.n_tiles + blockIdx.x) * K;
    for (int i = 0; i < K; ++i) {
      g.out_v[o + i] = i < cnt ? v[i] : __int_as_float(0x7f800000);
      g.out_i[o + i] = i < cnt ? m0 + ix[i] + g.col_offset : 0x7fffffff;
    }
  }
}

inline size_t chain_smem_bytes() { return 2 * CH_BK * CH_BM * 8 + 2 * CH_BK * CH_BN * 4; }

// Squared row norms over the leading `dims` columns, bitwise equal to the reference's
// np.einsum("ij,ij->i", m, m, dtype=np.float64).astype(np.float32) (preprocess.py:95-101).
// NumPy's einsum inner loop for two contiguous f64 operands and a 0-stride output
// (sum_of_products_contig_contig_outstride0_two, baseline SSE build: 2 f64 lanes) keeps one
// 2-lane accumulator; its 4x-unrolled body adds the pairs of each 8-element group in the order
// (6,7), (4,5), (2,3), (0,1); the remainder is added pair by pair (zero-padded), and the lanes
// are summed last.  Products of fp32 values are exact in f64, so only the summation order
// matters (verified bitwise on 3000 x {7..1536} random rows and strided column views,
// tools/blas_order_probe.py).  One thread per row; the two lanes are independent chains.
__global__ void row_sq_norms_einsum_kernel(const float* __restrict__ x, long long ldx, int rows, int dims,
                                           float* __restrict__ out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const float* p = x + r * ldx;
    double l0 = 0.0, l1 = 0.0;
    int t = 0;
    const bool al = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    for (; t + 8 <= dims; t += 8) {
      float v[8];
      if (al) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(p + t));
        const float4 w = __ldg(reinterpret_cast<const float4*>(p + t + 4));
        v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[t + u];
      }
#pragma unroll
      for (int pr = 3; pr >= 0; --pr) {
        const double e0 = v[2 * pr], e1 = v[2 * pr + 1];
        l0 = __dadd_rn(l0, e0 * e0);
        l1 = __dadd_rn(l1, e1 * e1);
      }
    }
    for (; t < dims; t += 2) {
      const double e0 = p[t];
      const double e1 = (t + 1 < dims) ? static_cast<double>(p[t + 1]) : 0.0;
      l0 = __dadd_rn(l0, e0 * e0);
      l1 = __dadd_rn(l1, e1 * e1);
    }
    out[r] = static_cast<float>(__dadd_rn(l0, l1));
  }
}

}  // namespace skm
