// fp32-faithful "NT" GEMM on the 5th-gen tensor cores: out[i][j] = sum_t A[i][t] * B[j][t].
//
// Precision: each operand is split x = hi + lo (hi tf32-exact), and every 32-wide k-block
// is computed as 3xTF32 into a FRESH TMEM accumulator -- small products first
// (A_lo*B_hi, A_hi*B_lo), then A_hi*B_hi -- so the tensor core's per-instruction
// accumulator truncation only ever sees one k-block's magnitude.  The epilogue warps add
// the k-block partials into fp32 registers with round-to-nearest.  Measured on B200:
// max rel. error 3.6e-6 at K=1536 (OpenBLAS sgemm: 2.9e-6); a single TMEM accumulator
// over the whole K gives 6.4e-5 (tools/probe_gemm_precision.py).  This is what keeps
// assignments in parity with the reference's sgemm-based distances (distance.py:58-59).
//
// Structure (one CTA per SM, 576 threads, warp-specialised):
//   warp 0      TMA producer: A_hi, A_lo, B_hi, B_lo k-block tiles (SWIZZLE_128B, K-major)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..17 epilogue: warp w reads TMEM lane quadrant (w%4) and column slice (w-2)/4;
//               thread = one output row x BN/4 columns, running sums in registers.
// The 512 TMEM columns hold 512/BN partials in flight (BN = 256: two), each partial KPAIR
// 32-wide k-blocks.  With 128-wide partials two of them span a tile's K at the usual d', so
// the GATE also runs at BN = 256 (2 stages): it reads B from shared memory once per 256
// columns instead of 128 (at N = 128 the MMA is co-limited by its shared-memory operand reads),
// 112 -> 98 ms per c2 fit despite a few spilled registers of the 64 running sums.
// A CTA owns one 128-row M tile and walks a contiguous range of BN-wide N tiles in
// ascending order, so per-row reductions (argmin, candidate emission) see columns in
// ascending index order like the reference's bank loop (core.py:183-190, 243-260).
#pragma once
#include "ptx.cuh"

namespace skm {

enum GemmMode : int {
  GEMM_STORE = 0,    // out = A.B^T (fp32)
  GEMM_DIST = 1,     // out = max(0, fl(fl(-2 acc + xsq_i) + ysq_j))   (distance.py:77-80)
  GEMM_ARGMIN = 2,   // running (min dist, lowest col) + second-smallest dist per row (core.py:183-190)
  GEMM_GATE = 3,     // emit (col, dist) for dist <= thr_i in ascending col order
};

struct GemmArgs {
  int M, N, K;
  int tiles_per_cta;          // N tiles handled by one CTA
  int n_split;                // CTAs per M tile along N; block b -> M tile b / n_split, N range
                              // b % n_split, so one M tile's CTAs run side by side (L2 reuse of A)
  float* out;                 // STORE / DIST
  long long ldo;
  const float* xsq;           // DIST / ARGMIN / GATE: per-row norm term
  const float* ysq;           // per-column norm term
  int4* top;                  // ARGMIN: per (N split, row) {best bits, best col, second bits, 0},
                              // top[split * M + row]; merged by argmin_merge_kernel
  const float* thr;           // GATE: per-row threshold
  int2* cand;                 // GATE: per-row candidate slab [M][cap] of {index, float bits}
  int* cand_cnt;              // GATE: per-row count (may exceed cap -> overflow)
  int cand_cap;
  long long row_offset;       // GATE/ARGMIN: added to the row index when writing outputs
  // GATE, optional "certified block-0 prune" extension: ext_k (64) more columns after K are
  // accumulated into one TMEM partial; a candidate whose distance over K + ext_k columns
  // exceeds thr1 by the GEMM error margin is certainly pruned at tail block 0 (for any tau
  // <= the seed tau) and is emitted with CAND_CERT0 set in its index.
  int ext_k;
  const float* xsq_ext;       // per-row norm over K + ext_k columns
  const float* ysq_ext;       // per-column norm over K + ext_k columns
  const float* thr1;          // per-row fl(tau * F[1])
  float cert_eps;             // margin: eps * (xsq_ext + ysq_ext)
  int dbg;                    // experiments: 1 = GATE drains partials only (no gate phase)
  // grouped columns (ARGMIN / GATE): row i sees columns [row_crange[i].x, row_crange[i].y);
  // M tile t walks the N tiles covering tile_nrange[t] (hierarchical fine phase, one launch
  // for every group: each group's rows against its own centroid block)
  const int2* row_crange;
  const int2* tile_nrange;
  // 1: the extension k-blocks run as one TF32 product (hi x hi) instead of 3xTF32 -- a third
  // of their MMAs and half their TMA bytes -- for a certificate whose margin covers 2^-9 of
  // xsq_ext + ysq_ext (engine.nowin_cert_eps)
  int ext_hi_only;
};
constexpr int CAND_CERT0 = static_cast<int>(0x80000000u);

#ifndef SKM_GATE_LDS
#define SKM_GATE_LDS 1       // GATE reads the staged column norms with explicit ld.shared.v4
#endif
#ifndef SKM_GEMM_KPAIR
#define SKM_GEMM_KPAIR 4     // k-blocks accumulated per TMEM partial
#endif
#ifndef SKM_GATE_PREFETCH
#define SKM_GATE_PREFETCH 1  // GATE loads the next tile's column norms during the drains
#endif

constexpr int GEMM_BM = 128;
constexpr int GEMM_BN = 256;       // STORE / DIST / ARGMIN tile width
#ifndef SKM_GATE_BN
#define SKM_GATE_BN 256
#endif
#ifndef SKM_GATE_STAGES
#define SKM_GATE_STAGES 2
#endif
constexpr int GEMM_BN_GATE = SKM_GATE_BN;  // GATE tile width: 4-deep TMEM partial ring, 32 sums per thread
constexpr int GEMM_BK = 32;        // fp32 elements per 128-byte swizzle row
constexpr int GEMM_EPI_WARPS = 16;
constexpr int GEMM_THREADS = 64 + 32 * GEMM_EPI_WARPS;
constexpr int GEMM_PARTS = GEMM_EPI_WARPS / 4;  // column slices per TMEM lane quadrant
constexpr int GEMM_TMEM_COLS = 512;             // the whole TMEM of the SM (one CTA per SM)

template <int STAGES, int BN>
struct GemmSmem {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 4;
  static constexpr int B_BYTES = BN * GEMM_BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int NBUF = GEMM_TMEM_COLS / BN;  // k-block partials in flight
  static constexpr int HALF = BN / GEMM_PARTS;      // columns per epilogue thread
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 2 * NBUF) + 16;
  // slice exchange (double buffered by tile parity) + column-norm tiles (ysq, ysq_ext; x2)
  static constexpr int XCHG_BYTES = 2 * GEMM_PARTS * GEMM_BM * 4 + 4 * BN * 4;
  static constexpr int TOTAL = 1024 + STAGES * STAGE_BYTES + BAR_BYTES + XCHG_BYTES;
};

__device__ __forceinline__ float expand_dist(float acc, float xs, float ys) {
  // reference op order: vals = inner * -2; vals += x_sq; vals += y_sq; max(vals, 0)
  const float v = __fadd_rn(__fadd_rn(__fmul_rn(acc, -2.0f), xs), ys);
  return v > 0.0f ? v : 0.0f;
}

__device__ __forceinline__ void epi_bar_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * GEMM_EPI_WARPS) : "memory");
}

__device__ __forceinline__ float4 lds_f32x4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ float f4_get(const float4& v, int q) {
  return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

template <int STAGES, int MODE, int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                       const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                       const __grid_constant__ CUtensorMap tE_A_hi, const __grid_constant__ CUtensorMap tE_A_lo,
                       const __grid_constant__ CUtensorMap tE_B_hi, const __grid_constant__ CUtensorMap tE_B_lo,
                       const GemmArgs args) {
  using L = GemmSmem<STAGES, BN>;
  constexpr int NBUF = L::NBUF;
  constexpr int HALF = L::HALF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NBUF);
  int* xchg = reinterpret_cast<int*>(smem + STAGES * L::STAGE_BYTES + L::BAR_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = (blockIdx.x / args.n_split) * GEMM_BM;
  const int n_tiles = (args.N + BN - 1) / BN;
  int t_begin = (blockIdx.x % args.n_split) * args.tiles_per_cta;
  int t_end = min(n_tiles, t_begin + args.tiles_per_cta);
  if (args.tile_nrange) {
    const int2 nr = args.tile_nrange[blockIdx.x];
    t_begin = nr.x / BN;
    t_end = min(n_tiles, (nr.y + BN - 1) / BN);
  }
  const int num_k = (args.K + GEMM_BK - 1) / GEMM_BK;
  // KPAIR 32-wide k-blocks per TMEM partial (4: 128-wide partials): fewer drains, and the GATE's
  // 4-deep partial ring spans a whole tile's K, so the MMA issuer runs a tile ahead of the gate
  // pass.  Every mode uses it, so DIST, ARGMIN and GATE keep identical accumulator bits.  The
  // rigorous bound (engine.tc_kappa, paired) covers it: 48 truncating accumulations per partial
  // cost 6 * 2^-20 of sum |x_t c_t| on top of the 3 * 2^-20 of 3xTF32, inside 2^-16.
  constexpr int KPAIR = SKM_GEMM_KPAIR;  // k-blocks per partial (1, 2 or 4)
  const int num_p = (num_k + KPAIR - 1) / KPAIR;  // main partials per tile
  // extension k-blocks (GATE certification): accumulated into ONE extra TMEM partial per tile
  const int num_e = (MODE == GEMM_GATE) ? (args.ext_k + GEMM_BK - 1) / GEMM_BK : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tA_hi);
    tma_prefetch_desc(&tA_lo);
    tma_prefetch_desc(&tB_hi);
    tma_prefetch_desc(&tB_lo);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NBUF; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], GEMM_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<GEMM_TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && t_begin < t_end && num_k > 0) {
      int s = 0;
      uint32_t ph = 0;
#pragma unroll 1
      for (int t = t_begin; t < t_end; ++t) {
        const int n0 = t * BN;
#pragma unroll 1
        for (int kb = 0; kb < num_k + num_e; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          const bool ext = kb >= num_k;
          const bool hi_only = ext && args.ext_hi_only;
          mbar_arrive_expect_tx(&full[s], hi_only ? L::A_BYTES + L::B_BYTES : L::STAGE_BYTES);
          uint8_t* base = smem + s * L::STAGE_BYTES;
          const int k0 = (ext ? kb - num_k : kb) * GEMM_BK;
          tma_load_2d(base, ext ? &tE_A_hi : &tA_hi, &full[s], k0, m0);
          if (!hi_only) tma_load_2d(base + L::A_BYTES, ext ? &tE_A_lo : &tA_lo, &full[s], k0, m0);
          tma_load_2d(base + 2 * L::A_BYTES, ext ? &tE_B_hi : &tB_hi, &full[s], k0, n0);
          if (!hi_only) tma_load_2d(base + 2 * L::A_BYTES + L::B_BYTES, ext ? &tE_B_lo : &tB_lo, &full[s], k0, n0);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && t_begin < t_end && num_k > 0) {
      constexpr uint32_t idesc = idesc_tf32(GEMM_BM, BN);
      int s = 0;
      uint32_t ph = 0;
      uint32_t kcount = 0;  // global partial counter -> TMEM buffer ring
#pragma unroll 1
      for (int t = t_begin; t < t_end; ++t) {
#pragma unroll 1
        for (int kb = 0; kb < num_k + num_e; ++kb) {
          // extension k-blocks after the first one keep accumulating into the same partial
          const bool main_kb = kb < num_k;
          const bool cont = main_kb ? (kb % KPAIR != 0) : kb > num_k;
          const bool last_of_partial = main_kb ? ((kb % KPAIR == KPAIR - 1) || kb == num_k - 1)
                                               : kb == num_k + num_e - 1;
          const int buf = kcount % NBUF;
          const uint32_t use = kcount / NBUF;
          if (!cont) mbar_wait(&tempty[buf], (use & 1) ^ 1);
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * BN);
          const uint32_t base = smem_u32(smem + s * L::STAGE_BYTES);
          const uint64_t a_hi = sw128_kmajor_desc(base);
          const uint64_t a_lo = sw128_kmajor_desc(base + L::A_BYTES);
          const uint64_t b_hi = sw128_kmajor_desc(base + 2 * L::A_BYTES);
          const uint64_t b_lo = sw128_kmajor_desc(base + 2 * L::A_BYTES + L::B_BYTES);
          if (main_kb || !args.ext_hi_only) {
#pragma unroll
            for (int kk = 0; kk < GEMM_BK / 8; ++kk) {
              const uint64_t adv = static_cast<uint64_t>((kk * 32) >> 4);  // 8 tf32 = 32 bytes
              mma_tf32(d_tmem, a_lo + adv, b_hi + adv, idesc, (kk != 0 || cont) ? 1u : 0u);
              mma_tf32(d_tmem, a_hi + adv, b_lo + adv, idesc, 1u);
            }
#pragma unroll
            for (int kk = 0; kk < GEMM_BK / 8; ++kk) {
              const uint64_t adv = static_cast<uint64_t>((kk * 32) >> 4);
              mma_tf32(d_tmem, a_hi + adv, b_hi + adv, idesc, 1u);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < GEMM_BK / 8; ++kk) {
              const uint64_t adv = static_cast<uint64_t>((kk * 32) >> 4);
              mma_tf32(d_tmem, a_hi + adv, b_hi + adv, idesc, (kk != 0 || cont) ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          if (last_of_partial) {
            mma_commit(&tfull[buf]);
            ++kcount;
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int eq = warp & 3;            // TMEM lane quadrant this warp may access
    const int half = ew >> 2;           // column slice of the tile
    const int r_local = eq * 32 + lane;
    const int row = m0 + r_local;
    const bool row_ok = row < args.M;
    const int e_thr = threadIdx.x - 64;  // epilogue thread index: the first BN stage column norms
    float xs = 0.0f, thr = 0.0f;
    if constexpr (MODE == GEMM_DIST || MODE == GEMM_ARGMIN || MODE == GEMM_GATE) {
      if (row_ok) xs = args.xsq[row];
    }
    int c_lo = 0, c_hi = args.N;  // columns this row may see
    if constexpr (MODE == GEMM_ARGMIN || MODE == GEMM_GATE) {
      if (args.row_crange && row_ok) {
        const int2 cr = args.row_crange[row];
        c_lo = cr.x;
        c_hi = min(cr.y, args.N);
      }
    }
    float xs_e = 0.0f, thr1 = 0.0f;
    if constexpr (MODE == GEMM_GATE) {
      if (row_ok) thr = args.thr[row];
      if (num_e && row_ok) {
        xs_e = args.xsq_ext[row];
        thr1 = args.thr1[row];
      }
    }
    // column norms of the next tile, loaded into registers one tile ahead (the loads are in
    // flight during the tile's k-block drains) and staged in shared memory at the tile end
    float ys_next = 0.0f, ye_next = 0.0f;
    auto load_norms = [&](int t) {
      if (e_thr < BN) {
        const int col = t * BN + e_thr;
        ys_next = col < args.N ? __ldg(args.ysq + col) : 0.0f;
        if (MODE == GEMM_GATE && num_e)
          ye_next = col < args.N ? (1.0f - args.cert_eps) * __ldg(args.ysq_ext + col) : 0.0f;
      }
    };
    // GATE: column norms prefetched one tile ahead; DIST / ARGMIN (measured faster that way)
    // load them at the tile end
    constexpr bool kPrefetchNorms = MODE == GEMM_GATE && SKM_GATE_PREFETCH;
    if constexpr (kPrefetchNorms) {
      if (t_begin < t_end) load_norms(t_begin);
    }
    float best = __int_as_float(0x7f800000);
    float second = __int_as_float(0x7f800000);  // ARGMIN: smallest distance other than the best
    int best_j = 0x7fffffff;
    int cnt = 0;
    const long long out_row = static_cast<long long>(row) + args.row_offset;
    float acc[HALF];
    uint32_t kcount = 0;
#pragma unroll 1
    for (int t = t_begin; t < t_end; ++t) {
      // first k-block of the tile overwrites the sums, the rest add into them (peeled: a
      // branch in the loop body made ptxas spill the 64 sums of the BN = 256 modes)
      auto drain_wait = [&]() -> uint32_t {
        const int buf = kcount % NBUF;
        mbar_wait_sleep(&tfull[buf], (kcount / NBUF) & 1);
        tc_fence_after();
        return tmem_base + (static_cast<uint32_t>(eq * 32) << 16) + static_cast<uint32_t>(buf * BN + half * HALF);
      };
      auto drain_release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[kcount % NBUF]);
        ++kcount;
      };
      if (num_k > 0) {
        const uint32_t tbase = drain_wait();
#pragma unroll
        for (int c = 0; c < HALF / 16; ++c) tmem_ld16_set(tbase + c * 16, *reinterpret_cast<float(*)[16]>(&acc[c * 16]));
        drain_release();
      }
#pragma unroll 1
      for (int kb = 1; kb < num_p; ++kb) {
        const uint32_t tbase = drain_wait();
#pragma unroll
        for (int c = 0; c < HALF / 16; ++c) tmem_ld16_add(tbase + c * 16, *reinterpret_cast<float(*)[16]>(&acc[c * 16]));
        drain_release();
      }
      // ---- tile complete: acc holds columns [col0, col0 + HALF)
      const int col0 = t * BN + half * HALF;
      uint32_t ys_s = 0, ye_s = 0;  // shared addresses of this thread's slice of the norm tiles
      const float* ys_tile = nullptr;
      const float* ye_tile = nullptr;
      if constexpr (MODE != GEMM_STORE) {
        float* yt = reinterpret_cast<float*>(xchg + 2 * GEMM_PARTS * GEMM_BM) + (t & 1) * BN;
        float* ye = yt + 2 * BN;
        if constexpr (!kPrefetchNorms) load_norms(t);
        if (e_thr < BN) {
          yt[e_thr] = ys_next;
          if (MODE == GEMM_GATE && num_e) ye[e_thr] = ye_next;
        }
        if constexpr (kPrefetchNorms) {
          if (t + 1 < t_end) load_norms(t + 1);
        }
        epi_bar_sync();
        ys_s = smem_u32(yt + half * HALF);
        ye_s = smem_u32(ye + half * HALF);
        ys_tile = yt + half * HALF;
        ye_tile = ye + half * HALF;
      }
      if constexpr (MODE == GEMM_STORE || MODE == GEMM_DIST) {
        if (row_ok && col0 < args.N) {
          if constexpr (MODE == GEMM_DIST) {
#pragma unroll
            for (int j = 0; j < HALF; ++j) acc[j] = expand_dist(acc[j], xs, ys_tile[j]);
          }
          float* o = args.out + static_cast<long long>(row) * args.ldo + col0;
          if (col0 + HALF <= args.N && (args.ldo & 3) == 0) {
#pragma unroll
            for (int j = 0; j < HALF; j += 4)
              *reinterpret_cast<float4*>(o + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < HALF; ++j)
              if (col0 + j < args.N) o[j] = acc[j];
          }
        }
      } else if constexpr (MODE == GEMM_ARGMIN) {
        if (row_ok) {
          const int lim = c_hi - col0;  // valid columns in this slice: [lo, lim)
          const int lo = c_lo - col0;
          float bv = best, sv = second;
          int bl = -1;
#pragma unroll
          for (int j = 0; j < HALF; ++j) {
            const float dv = expand_dist(acc[j], xs, ys_tile[j]);
            if (j < lim && j >= lo) {
              // ascending columns: a strictly smaller value takes over (lowest index on ties);
              // every other value, ties included, competes for the second place
              sv = fminf(sv, dv < bv ? bv : dv);
              if (dv < bv) { bv = dv; bl = j; }
            }
          }
          second = sv;
          if (bl >= 0) { best = bv; best_j = col0 + bl; }
        }
      } else if constexpr (MODE == GEMM_GATE) {
        constexpr int W = HALF / 32;  // 32-column mask words per thread
        uint32_t cert[W];
#pragma unroll
        for (int w = 0; w < W; ++w) cert[w] = 0u;
        if (num_e) {
          // certification partial (the ext_k columns after K): consumed first so its TMEM
          // buffer returns to the MMA issuer before the gate pass
          const int buf = kcount % NBUF;
          mbar_wait_sleep(&tfull[buf], (kcount / NBUF) & 1);
          tc_fence_after();
          const uint32_t tb = tmem_base + (static_cast<uint32_t>(eq * 32) << 16) +
                              static_cast<uint32_t>(buf * BN + half * HALF);
          if (args.dbg != 1) {
            // distance over K + ext_k columns minus the margin, folded: (1 - eps)(|x|^2 + |c|^2)
            // - 2 ip > thr1 with the per-column term pre-scaled in shared memory (rounding of
            // the fold is ~1e-7 relative, far inside the 3e-5 margin)
            const float cert_a = thr1 - (1.0f - args.cert_eps) * xs_e;
#pragma unroll
            for (int c = 0; c < HALF / 16; ++c) {
              float e16[16];
              tmem_ld16(tb + c * 16, e16);
#pragma unroll
              for (int j = 0; j < 16; j += 4) {
#if SKM_GATE_LDS
                const float4 y4 = lds_f32x4(ye_s + 4 * (c * 16 + j));
#else
                const float4 y4 = *reinterpret_cast<const float4*>(ye_tile + c * 16 + j);
#endif
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const int jj = c * 16 + j + q;
                  if (fmaf(-2.0f, __fadd_rn(acc[jj], e16[j + q]), f4_get(y4, q)) > cert_a)
                    cert[jj >> 5] |= 1u << (jj & 31);
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
          ++kcount;
        }
        if (args.dbg == 1) continue;
        const int lim = row_ok ? c_hi - col0 : 0;
        const int lo = c_lo - col0;
        uint32_t mask[W];
        int my = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          uint32_t m = 0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
#if SKM_GATE_LDS
            const float4 y4 = lds_f32x4(ys_s + 4 * (w * 32 + j));
#else
            const float4 y4 = *reinterpret_cast<const float4*>(ys_tile + w * 32 + j);
#endif
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int jj = w * 32 + j + q;
              const float dv = expand_dist(acc[jj], xs, f4_get(y4, q));
              acc[jj] = dv;
              m |= (dv > thr ? 0u : 1u) << (j + q);
            }
          }
          const int l = lim - w * 32;
          m &= l >= 32 ? 0xffffffffu : (l <= 0 ? 0u : ((1u << l) - 1u));
          const int l0 = lo - w * 32;  // columns below the row's range (grouped mode)
          m &= l0 <= 0 ? 0xffffffffu : (l0 >= 32 ? 0u : ~((1u << l0) - 1u));
          mask[w] = m;
          my += __popc(m);
        }
        // order the column slices of this row: slice 0 first (exchange double buffered by tile
        // parity, so one barrier per tile orders both the writes and the next tile's reuse)
        int* xc = xchg + (t & 1) * GEMM_PARTS * GEMM_BM;
        xc[half * GEMM_BM + r_local] = my;
        epi_bar_sync();
        int before = 0, total = 0;
#pragma unroll
        for (int q = 0; q < GEMM_PARTS; ++q) {
          const int cq = xc[q * GEMM_BM + r_local];
          before += (q < half) ? cq : 0;
          total += cq;
        }
        int pos = cnt + before;
        if (row_ok && args.dbg != 2) {
          int2* cr = args.cand + out_row * args.cand_cap;  // one 8-byte record per candidate
#pragma unroll
          for (int w = 0; w < W; ++w) {
            // skip empty 4-column groups (about a tenth of the columns pass the gate); static
            // register indices keep acc[] out of local memory
            const uint32_t m = mask[w];
            if (m == 0) continue;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              if (((m >> (4 * g)) & 15u) == 0) continue;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const int j = 4 * g + jj;
                if ((m >> j) & 1u) {
                  if (pos < args.cand_cap) {
                    cr[pos] = make_int2((col0 + w * 32 + j) | (((cert[w] >> j) & 1u) ? CAND_CERT0 : 0),
                                        __float_as_int(acc[w * 32 + j]));
                  }
                  ++pos;
                }
              }
            }
          }
        }
        cnt += total;
      }
    }
    if constexpr (MODE == GEMM_ARGMIN) {
      // combine the column slices lexicographically on (dist, col)
      // (the exchange area holds 2 * GEMM_PARTS * GEMM_BM ints: best | col, then seconds in the
      // column-norm area behind it, which is no longer read)
      float* xf = reinterpret_cast<float*>(xchg);
      float* xs2 = reinterpret_cast<float*>(xchg + 2 * GEMM_PARTS * GEMM_BM);
      epi_bar_sync();  // the last tile's column norms have been consumed by every slice
      xf[half * GEMM_BM + r_local] = best;
      xchg[(GEMM_PARTS + half) * GEMM_BM + r_local] = best_j;
      xs2[half * GEMM_BM + r_local] = second;
      epi_bar_sync();
      if (half == 0 && row_ok && t_begin < t_end) {
#pragma unroll
        for (int q = 1; q < GEMM_PARTS; ++q) {
          const float b1 = xf[q * GEMM_BM + r_local];
          const int j1 = xchg[(GEMM_PARTS + q) * GEMM_BM + r_local];
          const float s1 = xs2[q * GEMM_BM + r_local];
          if (b1 < best || (b1 == best && j1 < best_j)) {
            second = fminf(best, s1);  // the old best is now a runner-up (second >= best)
            best = b1;
            best_j = j1;
          } else {
            second = fminf(second, b1);  // s1 >= b1
          }
        }
        const int split = blockIdx.x % args.n_split;
        args.top[static_cast<long long>(split) * args.M + row] =
            make_int4(__float_as_int(best), best_j, __float_as_int(second), 0);
      }
    }
    if constexpr (MODE == GEMM_GATE) {
      if (row_ok && half == 0) args.cand_cnt[out_row] = cnt;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<GEMM_TMEM_COLS>(tmem_base);
  }
}

}  // namespace skm
