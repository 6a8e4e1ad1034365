// Production pruning scan (ADSampling progressive pruning), exact reference semantics.
//
// Reference behaviour (core.py:230-263 + _kernels.pyx:14-82): for each vector, centroids
// are visited in ascending global index j with a threshold tau that only tightens.
// A candidate survives the gate iff !(p_j > fl(tau*F0)); it then accumulates 64-dim tail
// blocks (each block sum a fresh sequential fp32 chain, no FMA) into `running`, and is
// pruned at the first checkpoint where running > fl(tau*F[b+1]).  A completed candidate
// with running < tau (or == tau and a lower index) becomes the assignment.
//
// GPU formulation (one warp per vector):
//  * candidates arrive in ascending j from the GEMM gate (a superset: the gate used the
//    seed tau, and tau never increases) or, for overflow rows, from a dense distance row;
//  * block sums are independent of tau, so 32 lanes compute them speculatively as
//    8 candidate slots x 4 consecutive blocks per wave, recording every block sum;
//  * slot leaders decide each candidate's exact outcome incrementally, tagged with a tau
//    version; a warp-parallel in-order resolver consumes decided outcomes in O(1) and
//    re-walks (from the recorded sums) only those decided before tau last tightened.
//    This replays the exact sequential semantics from the
//    recorded sums: a speculative evaluation always ran under a tau >= the exact one,
//    so it computed at least the blocks the exact walk needs (the exact walk prunes no
//    later).  Survivor / dims-touched counters therefore match the reference bitwise.
// Centroid tails are stored "PDX-quad" per centroid: T[j][q][b][r] = C[j][d'+64b+4q+r]
// (zero padded in the ragged last block -- adding +0 is exact), so the 4 lanes of a slot
// read 64 contiguous bytes per step.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "sgemm_chain.cuh"

namespace skm {

#ifndef SKM_SCAN_DEPTH
#define SKM_SCAN_DEPTH 4
#endif
#ifndef SKM_SCAN_WARPS
#define SKM_SCAN_WARPS 4
#endif
#ifndef SKM_SCAN_WINDOW
#define SKM_SCAN_WINDOW 64
#endif
constexpr int SCAN_DEPTH = SKM_SCAN_DEPTH;     // consecutive blocks per candidate per wave
constexpr int SCAN_SLOTS = 32 / SCAN_DEPTH;    // candidates in flight per wave
constexpr int SCAN_WINDOW = SKM_SCAN_WINDOW;   // in-flight queue positions per warp
constexpr int SCAN_NB_MAX = 104;               // tail blocks of the default 4-warp CTA (d - d' <= 6656):
                                               // 4 warps x 512 B per block of x tail + records fit in 227 KB
constexpr int SCAN_NB_MAX_WIDE = 432;          // one warp per CTA (longer tails, d - d' <= 27648)
constexpr int SCAN_WARPS = SKM_SCAN_WARPS;     // warps per CTA

struct ScanArgs {
  // candidate source (list mode)
  const int2* cand;  // [rows][cap] {centroid index | CAND_CERT0, float bits of the front distance}
  const int* cand_cnt;
  int cap;
  // candidate source (dense mode): row r reads dense[dense_row[r] * ld_dense + j], j < k
  const float* dense;
  long long ld_dense;
  const int* dense_row;
  int k;
  // rows to process: rows[r] (batch-local index) for r < n_rows; nullptr = identity
  const int* rows;
  int n_rows;
  long long row0;  // global row of batch-local row 0 (when row_map == nullptr)
  const int* row_map;      // optional: global row of batch-local row (cluster-ordered batches)
  unsigned int* work;      // global row-queue counter (zeroed by the launcher)
  const float* x;
  long long ldx;
  const float4* tails;  // [k][16][nb] float4
  int nb;
  int d_prime;
  const float* theta;      // nb + 1 gate factors (sentinel: inf except the last == 1)
  const int* block_dims;   // nb
  float* tau;              // global rows, in/out
  int* assign;             // global rows, in/out
  unsigned long long* counters;  // [0] survivors, [1] dims touched, [2] changed
  unsigned long long* counters_ext;  // optional diagnostics: [0] 64-dim block sums computed
  unsigned long long* prune_hist;  // optional diagnostics: survivors by prune block (nb = complete)
  // Exact re-evaluation of tensor-core partial distances.  kap > 0: a candidate's distance p~
  // comes from the 3xTF32 GEMM and the reference's (chain) value lies in [p~ - D, p~ + D],
  // D = kap * (xsq[row] + *ysq_max + p~).  Decisions are taken on that
  // interval; a decision it cannot settle, and every candidate that may replace the current best
  // (its running sum becomes tau), recomputes p with the reference's chain (exact_dot) first.
  float kap;
  const float* xsq;        // global rows: squared norm over the d' front columns
  const float* ysq;        // centroids: squared norm over d'
  const float* ysq_max;    // device scalar: max_j ysq[j]
  const float* cent;       // centroid rows, row-major (front columns for the exact chain)
  long long ldc;
  int chain_flavour;       // 0 fma chain with K blocks of chain_q (OpenBLAS), 1 mul+add (portable)
  int chain_q;
  // 1: the row's d' front and the centroid fronts of the re-evaluated candidates are staged in the
  // warp's shared memory (scan_dyn_smem(nb, d', true)) and re-evaluated there; 0: from global
  int ex_stage;
  // grouped rows (hierarchical fine phase): counters go to group_counters[3 * row_group[row] + c]
  // instead of counters (each group has its own d' controller and convergence test)
  const int* row_group;
  unsigned long long* group_counters;
  // optional: the row count is read from the device (the flat pass's fallback list length)
  const unsigned int* n_rows_dev;
  // deferred certified entries (exact_work_stats = false, full-d certificate): rows with
  // skip_cert[rl] != 0 leave their CAND_CERT0 entries out of the queue -- such a column never
  // replaces the best -- and record each tau improvement {j, tau bits} in imp[rl][SCAN_IMP_MAX]
  // (count imp_cnt[rl]); deferred_cert_count_kernel then settles the entries' survivor decisions
  // under the tau each would have met (the last improvement at a lower index, else the seed)
  const int* skip_cert;
  int2* imp;
  int* imp_cnt;
};
constexpr int SCAN_IMP_MAX = 32;  // improvements recorded per row (one per lane)

// T[j][q][b][r] = C[j][d' + 64b + 4q + r] (0 beyond d)
__global__ void build_tails_kernel(const float* __restrict__ cent, long long ldc, int k, int d, int d_prime, int nb,
                                   float* __restrict__ tails) {
  const long long per = 64LL * nb;
  const int tail = d - d_prime;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)k * per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / per;
    const int rem = static_cast<int>(e - j * per);
    const int q = rem / (nb * 4);
    const int b = (rem / 4) % nb;
    const int r = rem & 3;
    const int t = 64 * b + 4 * q + r;
    tails[e] = (t < tail) ? cent[j * ldc + d_prime + t] : 0.0f;
  }
}

// thr_i = sentinel ? inf : fl(tau_i * F0); kap > 0: the tensor-core gate's emission threshold,
// a rigorous upper end for every p~ whose exact value may pass fl(tau_i * F0):
// p~ - kap (xsq_i + ysq_max + p~) <= thr  <=>  p~ <= (thr + kap (xsq_i + ysq_max)) / (1 - kap),
// evaluated in f64 and rounded up (plus 2^-20 relative) so no fp32 rounding can drop a candidate.
__global__ void gate_threshold_kernel(const float* __restrict__ tau, int n, float f0, int sentinel,
                                      float* __restrict__ thr, const float* __restrict__ xsq,
                                      const float* __restrict__ ysq_max, float kap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (sentinel) {
    thr[i] = __int_as_float(0x7f800000);
    return;
  }
  const float t0 = __fmul_rn(tau[i], f0);
  if (kap > 0.0f) {
    const double k = kap;
    const double t = (static_cast<double>(t0) + k * (static_cast<double>(xsq[i]) + *ysq_max)) / (1.0 - k);
    thr[i] = __double2float_ru(t * (1.0 + 0x1p-20));
  } else {
    thr[i] = t0;
  }
}

#ifndef SKM_SCAN_TAIL_NOALLOC
#define SKM_SCAN_TAIL_NOALLOC 0
#endif
// centroid tail loads (L2-resident, read once per wave).  A/B variants: 1 = no L1 allocation
// (measured 5 % slower per c2 fit: L1 hits matter), 2 = L1::evict_last
__device__ __forceinline__ float4 scan_tail_load(const float4* p) {
#if SKM_SCAN_TAIL_NOALLOC == 2
  float4 v;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
#elif SKM_SCAN_TAIL_NOALLOC
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

struct ScanWarpSmem {
  // per queue position (ring of SCAN_WINDOW)
  int qj[SCAN_WINDOW];
  float qp[SCAN_WINDOW];
  int qdone[SCAN_WINDOW];   // block sums recorded so far
  int qstat[SCAN_WINDOW];   // 0 pending, 1 not a survivor, 2 pruned (at qpb), 3 complete (qrun)
  int qpb[SCAN_WINDOW];
  float qrun[SCAN_WINDOW];
  int qver[SCAN_WINDOW];    // tau version the outcome was decided under
  float qdl[SCAN_WINDOW];   // error bound of qp (0: exact)
  float qrunhi[SCAN_WINDOW];  // upper end of the final running sum (COMPLETE)
  int sel[32];              // dispatch: lane of the r-th taken position
};

// (a - b)^2 for two lanes with sm_100 packed fp32 ops: sub.rn.f32x2 / mul.rn.f32x2.
__device__ __forceinline__ float2 sq_diff2(float2 a, float2 b) {
  unsigned long long ua, ub, d, q;
  ua = (static_cast<unsigned long long>(__float_as_uint(a.y)) << 32) | __float_as_uint(a.x);
  ub = (static_cast<unsigned long long>(__float_as_uint(b.y)) << 32) | __float_as_uint(b.x);
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(ua), "l"(ub));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(q) : "l"(d));
  return make_float2(__uint_as_float(static_cast<unsigned>(q)), __uint_as_float(static_cast<unsigned>(q >> 32)));
}

// ST_AMBIG: the interval of a tensor-core distance cannot settle the outcome -> exact p needed
#ifndef SKM_EXF
#define SKM_EXF exact_front_dist
#endif
enum : int { ST_PENDING = 0, ST_NOTSURV = 1, ST_PRUNED = 2, ST_COMPLETE = 3, ST_AMBIG = 4 };

// Walk of one recorded candidate under threshold tcur (blocks < nd are available) with its
// distance known to lie in [p - dl, p + dl] (dl == 0: exact).  Adding a block sum is monotone
// under round-to-nearest, so the running sums of the two ends bracket the exact one: a checkpoint
// prunes for certain when the low end exceeds it, and continues for certain when the high end
// does not.  Returns the exact status (NOTSURV / PRUNED at pb / COMPLETE with run in
// [run, run_hi]), ST_AMBIG if some checkpoint was not settled, or ST_PENDING if a block that has
// not been computed yet is needed.  The low-end walk never prunes later than the exact walk
// would, so the blocks recorded for it cover the exact walk.
__device__ __forceinline__ int walk_interval(float p, float dl, const float* rec_row, int nd, int nb, float tcur,
                                             float f0, const float* theta, int& pb, float& run, float& run_hi) {
  const float thr0 = __fmul_rn(tcur, f0);
  if (__fsub_rn(p, dl) > thr0) return ST_NOTSURV;
  bool amb = __fadd_rn(p, dl) > thr0;
  if (nd < 0) {  // GEMM-certified: pruned at block 0 under any tau <= the seed tau
    pb = 0;
    return amb ? ST_AMBIG : ST_PRUNED;
  }
  float lo = fmaxf(__fsub_rn(p, dl), 0.0f), hi = __fadd_rn(p, dl);
  for (int b = 0; b < nb; ++b) {
    if (b >= nd) return ST_PENDING;
    lo = __fadd_rn(lo, rec_row[b]);
    hi = __fadd_rn(hi, rec_row[b]);
    const float thr = __fmul_rn(tcur, theta[b + 1]);
    if (lo > thr) {
      pb = b;
      run = lo;
      return amb ? ST_AMBIG : ST_PRUNED;
    }
    amb = amb || hi > thr;
  }
  run = lo;
  run_hi = hi;
  return amb ? ST_AMBIG : ST_COMPLETE;
}

// The reference's partial distance of (row, j): chain inner product over the d' front columns
// (OpenBLAS / portable bits, sgemm_chain.cuh) + expansion (distance.py:66-82).
__device__ __noinline__ float exact_front_dist(const float* __restrict__ xr, const float* __restrict__ cr, int dp,
                                               int flavour, int q, float xs, float ys) {
  const float ip = flavour == 0 ? exact_dot<CHAIN_FMA>(xr, cr, dp, q) : exact_dot<CHAIN_MULADD>(xr, cr, dp, 0);
  const float e = __fadd_rn(__fadd_rn(__fmul_rn(ip, -2.0f), xs), ys);
  return e > 0.0f ? e : 0.0f;
}

// exact_dot on shared-memory operands: the same chains (K blocks of q, ascending t), with the
// operands of 16 steps loaded ahead of their fma chain so the chain runs at fma latency.
template <int FLAVOUR>
__device__ __forceinline__ float exact_dot_staged(const float* __restrict__ x, const float* __restrict__ y, int K,
                                                  int q) {
  float tot = 0.0f;
  int k0 = 0;
  while (k0 < K) {
    const int k1 = chain_next_boundary(k0, K, q);
    float acc = 0.0f;
    int t = k0;
    if ((k0 & 3) == 0) {
      for (; t + 16 <= k1; t += 16) {
        float4 u[4], v[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          u[h] = *reinterpret_cast<const float4*>(x + t + 4 * h);
          v[h] = *reinterpret_cast<const float4*>(y + t + 4 * h);
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          acc = chain_scalar_step<FLAVOUR>(u[h].x, v[h].x, acc);
          acc = chain_scalar_step<FLAVOUR>(u[h].y, v[h].y, acc);
          acc = chain_scalar_step<FLAVOUR>(u[h].z, v[h].z, acc);
          acc = chain_scalar_step<FLAVOUR>(u[h].w, v[h].w, acc);
        }
      }
    }
    for (; t < k1; ++t) acc = chain_scalar_step<FLAVOUR>(x[t], y[t], acc);
    tot = __fadd_rn(tot, acc);
    k0 = k1;
  }
  return tot;
}

__device__ __noinline__ float exact_front_dist_staged(const float* __restrict__ xr, const float* __restrict__ cr,
                                                      int dp, int flavour, int q, float xs, float ys) {
  const float ip = flavour == 0 ? exact_dot_staged<CHAIN_FMA>(xr, cr, dp, q) : exact_dot_staged<CHAIN_MULADD>(xr, cr, dp, 0);
  const float e = __fadd_rn(__fadd_rn(__fmul_rn(ip, -2.0f), xs), ys);
  return e > 0.0f ? e : 0.0f;
}

constexpr int SCAN_EXS = 2;  // centroid fronts staged per cooperative re-evaluation round

#ifndef SKM_SCAN_MINB
#define SKM_SCAN_MINB 3  // 12 warps per SM: caps registers at 168 (the exact-chain call site raised it to 231)
#endif
// WARPS: warps per CTA.  The default SCAN_WARPS instantiation serves tails up to SCAN_NB_MAX
// blocks; the one-warp instantiation (shared memory of a whole CTA for one row's tail) serves
// longer tails up to SCAN_NB_MAX_WIDE.  The per-row algorithm is the same.
template <bool DENSE, int WARPS = SCAN_WARPS>
__global__ void __launch_bounds__(WARPS * 32, WARPS == SCAN_WARPS ? SKM_SCAN_MINB : 1)
    pruned_scan_kernel(const ScanArgs a) {
  constexpr int NBMAX = WARPS == SCAN_WARPS ? SCAN_NB_MAX : SCAN_NB_MAX_WIDE;
  extern __shared__ float scan_smem[];
  __shared__ ScanWarpSmem wsm[WARPS];
  __shared__ float s_theta[NBMAX + 1];
  __shared__ int s_bdcum[NBMAX + 1];  // dims touched through block b (prefix at b+1)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = a.nb;
  for (int i = threadIdx.x; i <= nb; i += WARPS * 32) s_theta[i] = a.theta[i];
  if (threadIdx.x == 0) {
    int c = 0;
    s_bdcum[0] = 0;
    for (int b = 0; b < nb; ++b) {
      c += a.block_dims[b];
      s_bdcum[b + 1] = c;
    }
  }
  __syncthreads();

  const int dpp = (a.d_prime + 3) & ~3;
  const bool ex_stage = a.ex_stage != 0;
  float* xsm = scan_smem + static_cast<long long>(warp) * (64 * nb + SCAN_WINDOW * nb + (ex_stage ? (1 + SCAN_EXS) * dpp : 0));
  float* rec = xsm + 64 * nb;
  float* xfs = rec + SCAN_WINDOW * nb;  // ex_stage: the row's d' front columns
  float* cfs = xfs + dpp;               // ex_stage: SCAN_EXS staged centroid fronts
  ScanWarpSmem& W = wsm[warp];
  const float4* xsm4 = reinterpret_cast<const float4*>(xsm);
  const int tail_dims = s_bdcum[nb];
  const float f0 = s_theta[0];
  const unsigned FULL = 0xffffffffu;
  const bool x_aligned = ((a.ldx & 3) == 0) && ((a.d_prime & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  const int slot = lane / SCAN_DEPTH, dep = lane % SCAN_DEPTH;
  const bool slot_leader = dep == 0;
  const unsigned leader_mask = (SCAN_DEPTH == 4) ? 0x11111111u : (SCAN_DEPTH == 8) ? 0x01010101u
                              : (SCAN_DEPTH == 2) ? 0x55555555u : 0xffffffffu;  // slot leader lanes

  unsigned long long surv_acc = 0, touched_acc = 0, changed_acc = 0, blocks_acc = 0, waves_acc = 0, exact_acc = 0;
  const int n_rows = a.n_rows_dev ? static_cast<int>(*a.n_rows_dev) : a.n_rows;
  int cur_g = -1;  // grouped mode: group of the accumulated counters
  auto flush_group = [&]() {
    if (cur_g >= 0) {
      unsigned long long* gc = a.group_counters + 3LL * cur_g;
      warp_add_u64(surv_acc, &gc[0]);
      warp_add_u64(touched_acc, &gc[1]);
      warp_add_u64(changed_acc, &gc[2]);
    }
    surv_acc = touched_acc = changed_acc = 0;
  };
  while (true) {
    // rows are handed out in order from a global counter: warps running concurrently work on
    // neighbouring (cluster-sorted) rows, so their candidate centroids' tails stay L2-hot
    int r = 0;
    if (lane == 0) r = static_cast<int>(atomicAdd(a.work, 1u));
    r = __shfl_sync(FULL, r, 0);
    if (r >= n_rows) break;
    const int rl = a.rows ? a.rows[r] : r;
    int n_src;
    if constexpr (DENSE) {
      n_src = a.k;
    } else {
      n_src = a.cand_cnt[rl];
      if (n_src > a.cap) continue;  // overflow row: handled by the dense pass
    }
    const long long row = a.row_map ? static_cast<long long>(a.row_map[rl]) : a.row0 + rl;
    if (a.group_counters) {
      const int g = __ldg(a.row_group + row);
      if (g != cur_g) {
        flush_group();
        cur_g = g;
      }
    }
    // ---- stage the x tail, quad layout (q, b, r): 16-byte async copies (zero-filled past the
    //      tail) whose latency overlaps the row's scalar loads and first queue fill
    const float* xrow = a.x + row * a.ldx + a.d_prime;
    if (x_aligned) {
      for (int c = lane; c < 16 * nb; c += 32) {
        const int b = c >> 4, q = c & 15;
        const int valid = min(4, max(0, tail_dims - 4 * c));
        cp_async_16_zfill(xsm + (q * nb + b) * 4, valid ? xrow + 4 * c : xrow, 4 * valid);
      }
    } else {
      for (int u = lane; u < 64 * nb; u += 32) {
        const int b = u >> 6, t = u & 63;
        xsm[((t >> 2) * nb + b) * 4 + (t & 3)] = (u < tail_dims) ? xrow[u] : 0.0f;
      }
    }
    if (ex_stage) {  // the d' front (read only by exact re-evaluations)
      const float* xf = a.x + row * a.ldx;
      if (x_aligned) {
        for (int c = lane; c < dpp / 4; c += 32) {
          const int valid = min(4, a.d_prime - 4 * c);
          cp_async_16_zfill(xfs + 4 * c, xf + 4 * c, 4 * valid);
        }
      } else {
        for (int u = lane; u < dpp; u += 32) xfs[u] = u < a.d_prime ? xf[u] : 0.0f;
      }
    }
    float tcur = a.tau[row];
    int best = a.assign[row];
    // error-bound base of this row's tensor-core distances: D = kap * (dl_base + p)
    const float dl_base = a.kap > 0.0f ? __ldg(a.xsq + row) + *a.ysq_max : 0.0f;
    const float xs_row = a.kap > 0.0f ? __ldg(a.xsq + row) : 0.0f;
    const int best0 = best;
    const bool skip = !DENSE && a.skip_cert != nullptr && a.skip_cert[rl] != 0;
    int nimp = 0;
    int ver = 0;  // bumped whenever tau tightens
    int src = 0, F = 0, D = 0, R = 0;
    // slot state: all lanes of a slot hold spos/snxt; the leader also walks (srun, sb, sver)
    int spos = -1, snxt = 0, sb = 0, sver = -1;
    float srun = 0.0f, srun_hi = 0.0f;
    bool samb = false;
    const float* dense_row = nullptr;
    const int2* lrec = nullptr;
    if constexpr (DENSE) {
      dense_row = a.dense + static_cast<long long>(a.dense_row[rl]) * a.ld_dense;
    } else {
      lrec = a.cand + static_cast<long long>(rl) * a.cap;
    }
    // candidate records are prefetched one fill batch ahead (their L2 latency then overlaps the
    // wave that precedes the next fill)
    int2 pre = make_int2(0, 0);
    if constexpr (!DENSE) {
      if (lane < n_src) pre = lrec[lane];
    }
    cp_async_wait_all();
    __syncwarp();

    while (true) {
      // ---- 1. fill the queue (gate with the current tau: exact-safe, tau only shrinks)
      while (src < n_src && F - R <= SCAN_WINDOW - 32) {
        const int e = src + lane;
        int j = 0;
        float p = 0.0f;
        bool ok = e < n_src;
        bool cert = false;
        int2 rec = pre;
        if constexpr (!DENSE) {
          if (e + 32 < n_src) pre = lrec[e + 32];
        }
        if (ok) {
          if constexpr (DENSE) {
            j = e;
            p = dense_row[e];
          } else {
            j = rec.x;
            p = __int_as_float(rec.y);
            cert = j < 0;  // CAND_CERT0: certified block-0 prune (gemm_tf32x3.cuh)
            j &= 0x7fffffff;
          }
        }
        const float dl = a.kap * (dl_base + p);
        if (ok) ok = !(__fsub_rn(p, dl) > __fmul_rn(tcur, f0)) && !(skip && cert);
        const unsigned m = __ballot_sync(FULL, ok);
        if (ok) {
          const int qs = (F + __popc(m & ((1u << lane) - 1u))) % SCAN_WINDOW;
          W.qj[qs] = j;
          W.qp[qs] = p;
          W.qdl[qs] = dl;
          W.qdone[qs] = cert ? -1 : 0;  // -1 marks a certified entry: never takes a slot
          W.qstat[qs] = ST_PENDING;
          W.qver[qs] = -1;
        }
        F += __popc(m);
        src += 32;
      }
      __syncwarp();
      if (R == F && src >= n_src) break;  // everything resolved
      // ---- 2. dispatch: free slots take the next positions that still pass the gate under
      //         the current tau; positions failing it are decided (not survivors) on the spot
      {
        const unsigned freem = __ballot_sync(FULL, slot_leader && spos < 0) & leader_mask;
        int nfree = __popc(freem);
        unsigned free_left = freem;
        while (nfree > 0 && D < F && D < R + SCAN_WINDOW) {
          const int lim = min(min(F, R + SCAN_WINDOW) - D, 32);
          const int pp = D + lane;
          bool pass = false, gate = false, gate_hi = false, cert = false;
          if (lane < lim) {
            const float qp = W.qp[pp % SCAN_WINDOW], qd = W.qdl[pp % SCAN_WINDOW];
            const float thr0 = __fmul_rn(tcur, f0);
            gate = !(__fsub_rn(qp, qd) > thr0);      // may pass
            gate_hi = !(__fadd_rn(qp, qd) > thr0);   // passes for certain
            cert = W.qdone[pp % SCAN_WINDOW] < 0;
            pass = gate && !cert;
          }
          const unsigned pm = __ballot_sync(FULL, pass);
          // the first nfree passing positions get slots; cut = positions consumed this round
          int cut = lim;
          if (__popc(pm) >= nfree) {  // past the nfree-th pass (rank by prefix popcount)
            const bool nth = pass && __popc(pm & ((1u << lane) - 1u)) == nfree - 1;
            cut = __ffs(__ballot_sync(FULL, nth));
          }
          if (lane < cut && !pass) {  // decided on the spot: not a survivor, or certified prune
            const int qs = pp % SCAN_WINDOW;
            W.qstat[qs] = !gate ? ST_NOTSURV : (gate_hi ? ST_PRUNED : ST_AMBIG);  // !gate or certified
            W.qpb[qs] = 0;
            W.qver[qs] = ver;
          }
          const unsigned took = pm & ((cut >= 32) ? FULL : ((1u << cut) - 1u));
          // taken positions (ascending) go to the remaining free slots (ascending)
          if ((took >> lane) & 1u) W.sel[__popc(took & ((1u << lane) - 1u))] = lane;
          __syncwarp();
          int newpos = -1;
          if (slot_leader && ((free_left >> lane) & 1u)) {
            const int my_rank = __popc(free_left & ((1u << lane) - 1u));
            if (my_rank < __popc(took)) newpos = D + W.sel[my_rank];
          }
          newpos = __shfl_sync(FULL, newpos, slot * SCAN_DEPTH);
          const unsigned assigned = __ballot_sync(FULL, slot_leader && newpos >= 0);
          if (newpos >= 0) {
            spos = newpos;
            snxt = 0;
            sb = 0;
            sver = -1;
          }
          free_left &= ~assigned;
          nfree -= __popc(took);
          D += cut;
          __syncwarp();
        }
      }
      // ---- 3. issue this wave's tail loads (16 x 16 B per lane); their latency is hidden
      //         behind the in-order resolution of the previous waves' outcomes (step 4)
      ++waves_acc;
      const int myb = snxt + dep;
      const bool active = spos >= 0 && myb < nb;
      float4 c4[16];
      int my_qs = 0;
      if (active) {
        my_qs = spos % SCAN_WINDOW;
        const float4* cb = a.tails + static_cast<long long>(W.qj[my_qs]) * 16 * nb + myb;
#pragma unroll
        for (int q = 0; q < 16; ++q) c4[q] = scan_tail_load(cb + q * nb);
      }
      // ---- 4. in-order resolution, 32 positions per round; outcomes already decided under
      //         the current tau version are O(1), older ones are re-walked from the records
      while (R < D) {
        const int p = R + lane;
        int st = ST_NOTSURV;  // lanes beyond D: neutral
        float run = 0.0f, run_hi = 0.0f;
        int pb = 0, j = 0;
        bool need_exact = false;
        if (p < D) {
          const int qs = p % SCAN_WINDOW;
          st = W.qstat[qs];
          j = W.qj[qs];
          if (st != ST_PENDING) {
            if (W.qver[qs] != ver) {
              st = walk_interval(W.qp[qs], W.qdl[qs], rec + qs * nb, W.qdone[qs], nb, tcur, f0, s_theta, pb, run,
                                 run_hi);
              if (st != ST_PENDING) {
                W.qstat[qs] = st;
                W.qpb[qs] = pb;
                W.qrun[qs] = run;
                W.qrunhi[qs] = run_hi;
                W.qver[qs] = ver;
              }
            } else {
              pb = W.qpb[qs];
              run = W.qrun[qs];
              run_hi = W.qrunhi[qs];
            }
            // an unsettled outcome, or an inexact candidate that may replace the best (its
            // running sum would become tau): recompute p with the reference's chain, walk exactly
            const bool may_improve = st == ST_COMPLETE && (run < tcur || (run == tcur && j < best));
            need_exact = st == ST_AMBIG || (may_improve && W.qdl[qs] > 0.0f);
          }
        }
        float pe = 0.0f;
        if (ex_stage) {
          // warp-cooperative: the fronts of up to SCAN_EXS candidates are copied into the warp's
          // shared memory by all lanes (coalesced), then their lanes run the chains side by side
          unsigned needm = __ballot_sync(FULL, need_exact);
          while (needm) {
            unsigned batch = 0, mm = needm;
#pragma unroll
            for (int s2 = 0; s2 < SCAN_EXS; ++s2) {
              if (mm) {
                batch |= mm & (0u - mm);
                mm &= mm - 1u;
              }
            }
            int slotc = 0;
            for (unsigned bm = batch; bm; bm &= bm - 1u, ++slotc) {
              const int jj = __shfl_sync(FULL, j, __ffs(bm) - 1);
              const float* crow = a.cent + static_cast<long long>(jj) * a.ldc;
              float* dst = cfs + slotc * dpp;
              if (x_aligned && ((a.ldc & 3) == 0)) {
                for (int c = lane; c < dpp / 4; c += 32) {
                  const int valid = min(4, a.d_prime - 4 * c);
                  cp_async_16_zfill(dst + 4 * c, crow + 4 * c, 4 * valid);
                }
              } else {
                for (int u = lane; u < dpp; u += 32) dst[u] = u < a.d_prime ? crow[u] : 0.0f;
              }
            }
            cp_async_wait_all();
            __syncwarp();
            if ((batch >> lane) & 1u) {
              const int my = __popc(batch & ((1u << lane) - 1u));
              pe = exact_front_dist_staged(xfs, cfs + my * dpp, a.d_prime, a.chain_flavour, a.chain_q, xs_row,
                                           __ldg(a.ysq + j));
            }
            __syncwarp();
            needm &= ~batch;
          }
        } else if (need_exact) {
          pe = SKM_EXF(a.x + row * a.ldx, a.cent + static_cast<long long>(j) * a.ldc, a.d_prime, a.chain_flavour,
                       a.chain_q, xs_row, __ldg(a.ysq + j));
        }
        if (need_exact) {
          const int qs = p % SCAN_WINDOW;
          W.qp[qs] = pe;
          W.qdl[qs] = 0.0f;
          st = walk_interval(pe, 0.0f, rec + qs * nb, W.qdone[qs], nb, tcur, f0, s_theta, pb, run, run_hi);
          if (st != ST_PENDING) {
            W.qstat[qs] = st;
            W.qpb[qs] = pb;
            W.qrun[qs] = run;
            W.qrunhi[qs] = run;
            W.qver[qs] = ver;
          }
          ++exact_acc;
        }
        const bool improve = st == ST_COMPLETE && (run < tcur || (run == tcur && j < best));
        const unsigned ev = __ballot_sync(FULL, p < D && (improve || st == ST_PENDING));
        const int limit = ev ? (__ffs(ev) - 1) : 32;  // lanes < limit are final
        const bool counted = p < D && (lane < limit || (lane == limit && improve));
        if (counted && (st == ST_PRUNED || st == ST_COMPLETE)) {
          surv_acc += 1;
          touched_acc += (st == ST_PRUNED) ? s_bdcum[pb + 1] : tail_dims;
          if (a.prune_hist) atomicAdd(&a.prune_hist[st == ST_PRUNED ? pb : nb], 1ull);  // diagnostics only
        }
        const int src_lane = ev ? limit : 0;
        const int ev_improve = __shfl_sync(FULL, (int)improve, src_lane);
        const float ev_run = __shfl_sync(FULL, run, src_lane);
        const int ev_j = __shfl_sync(FULL, j, src_lane);
        __syncwarp();
        if (!ev) {
          R += min(32, D - R);
        } else if (ev_improve) {
          if (skip) {  // at most one improvement per queued (uncertified) entry: <= SCAN_IMP_MAX
            if (lane == 0 && nimp < SCAN_IMP_MAX)
              a.imp[static_cast<long long>(rl) * SCAN_IMP_MAX + nimp] = make_int2(ev_j, __float_as_int(ev_run));
            ++nimp;
          }
          tcur = ev_run;
          best = ev_j;
          ++ver;
          R += limit + 1;
        } else {
          R += limit;
          break;  // stalled on a candidate whose blocks are still being computed
        }
      }
      // ---- 5. the wave's speculative block sums: sequential fp32 chain per (candidate, block)
      float acc = 0.0f;
      if (active) {
        const float4* xb = xsm4 + myb;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 x4 = xb[q * nb];
          // squares of 4 dims with packed FADD2/FMUL2 (per-lane IEEE RN, identical bits),
          // then the sequential fp32 chain in ascending dimension order
          const float2 s01 = sq_diff2(make_float2(x4.x, x4.y), make_float2(c4[q].x, c4[q].y));
          const float2 s23 = sq_diff2(make_float2(x4.z, x4.w), make_float2(c4[q].z, c4[q].w));
          acc = __fadd_rn(acc, s01.x);
          acc = __fadd_rn(acc, s01.y);
          acc = __fadd_rn(acc, s23.x);
          acc = __fadd_rn(acc, s23.y);
        }
        rec[my_qs * nb + myb] = acc;
        ++blocks_acc;
      }
      // ---- 6. slot leaders walk their candidate exactly under the current tau version; the
      //         wave's 4 block sums come from the slot lanes by shuffle
      {
        float blk[SCAN_DEPTH];
#pragma unroll
        for (int i = 0; i < SCAN_DEPTH; ++i) blk[i] = __shfl_sync(FULL, acc, slot * SCAN_DEPTH + i);
        int fin = 0;
        if (spos >= 0 && slot_leader) {
          const int qs = spos % SCAN_WINDOW;
          const int hi = min(nb, snxt + SCAN_DEPTH);
          W.qdone[qs] = hi;
          if (sver != ver) {  // tau tightened since this walk started: restart from the records
            sver = ver;
            sb = 0;
            const float qp = W.qp[qs], qd = W.qdl[qs];
            const float thr0 = __fmul_rn(tcur, f0);
            srun = fmaxf(__fsub_rn(qp, qd), 0.0f);  // low end: prunes only for certain
            srun_hi = __fadd_rn(qp, qd);
            samb = srun_hi > thr0;
            if (__fsub_rn(qp, qd) > thr0) fin = ST_NOTSURV;
          }
          // blocks recorded in earlier waves (only after a restart), then this wave's
          // blocks straight from registers (static indices)
          while (!fin && sb < snxt) {
            srun = __fadd_rn(srun, rec[qs * nb + sb]);
            srun_hi = __fadd_rn(srun_hi, rec[qs * nb + sb]);
            const float thr = __fmul_rn(tcur, s_theta[sb + 1]);
            if (srun > thr) {
              fin = samb ? ST_AMBIG : ST_PRUNED;
              W.qpb[qs] = sb;
            }
            samb = samb || srun_hi > thr;
            ++sb;
          }
          // the wave's checkpoint thresholds fl(tau * theta[b + 1]) do not depend on the running
          // sum: load and scale them ahead of the sequential chain (same values, off the chain)
          float thr_w[SCAN_DEPTH];
#pragma unroll
          for (int i = 0; i < SCAN_DEPTH; ++i) thr_w[i] = __fmul_rn(tcur, s_theta[min(snxt + i + 1, nb)]);
#pragma unroll
          for (int i = 0; i < SCAN_DEPTH; ++i) {
            if (!fin && snxt + i < hi) {
              srun = __fadd_rn(srun, blk[i]);
              srun_hi = __fadd_rn(srun_hi, blk[i]);
              if (srun > thr_w[i]) {
                fin = samb ? ST_AMBIG : ST_PRUNED;
                W.qpb[qs] = snxt + i;
              }
              samb = samb || srun_hi > thr_w[i];
              ++sb;
            }
          }
          if (!fin && sb >= nb) fin = samb ? ST_AMBIG : ST_COMPLETE;
          if (fin) {
            W.qrun[qs] = srun;
            W.qrunhi[qs] = srun_hi;
            W.qver[qs] = ver;
            W.qstat[qs] = fin;
          }
        }
        fin = __shfl_sync(FULL, fin, slot * SCAN_DEPTH);
        if (spos >= 0) {
          snxt += SCAN_DEPTH;
          if (fin) spos = -1;
        }
      }
      __syncwarp();
      // slots whose candidate got resolved are released
      if (spos >= 0 && spos < R) spos = -1;
      __syncwarp();
    }
    if (lane == 0) {
      a.tau[row] = tcur;
      a.assign[row] = best;
      changed_acc += (best != best0);
      if (skip) a.imp_cnt[rl] = nimp;
    }
    __syncwarp();
  }
  if (a.group_counters) {
    flush_group();
  } else {
    warp_add_u64(surv_acc, &a.counters[0]);
    warp_add_u64(touched_acc, &a.counters[1]);
    warp_add_u64(changed_acc, &a.counters[2]);
  }
  if (a.counters_ext) {
    warp_add_u64(blocks_acc, &a.counters_ext[0]);  // speculative block sums computed
    if (lane == 0 && waves_acc) atomicAdd(&a.counters_ext[1], waves_acc);  // warp waves executed
    warp_add_u64(exact_acc, &a.counters_ext[3]);  // candidates re-evaluated with the exact chain
  }
}

// skip[rl] = 1 when row rl's list holds certified entries and at most SCAN_IMP_MAX uncertified
// ones (so its improvements fit the record), 0 otherwise (the scan then queues every entry).
__global__ void defer_cert_flags_kernel(const int2* __restrict__ cand, const int* __restrict__ cand_cnt, int cap,
                                        int n_rows, int* __restrict__ skip) {
  const int rl = static_cast<int>((blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (rl >= n_rows) return;
  const int cnt = cand_cnt[rl];
  int u = 0, c = 0;
  if (cnt <= cap) {
    const int2* row = cand + static_cast<long long>(rl) * cap;
    for (int e = lane; e < cnt; e += 32) {
      const bool cert = row[e].x < 0;
      u += !cert;
      c += cert;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane == 0) skip[rl] = (cnt <= cap && c > 0 && u <= SCAN_IMP_MAX) ? 1 : 0;
}

// The survivor decisions of the entries a skip row left out of its scan, exactly as the scan's
// in-order resolver takes them for a certified entry: under the tau in force at index j (the
// last recorded improvement at a lower index, else the seed tau), p +- D settles the front
// gate fl(tau F0), and an unsettled one takes the reference's chain p.  A survivor is a
// certified block-0 prune: dims touched += block_dims[0].  One warp per batch row.
__global__ void deferred_cert_count_kernel(const ScanArgs a, const float* __restrict__ tau_seed) {
  const int rl = static_cast<int>((blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  if (rl >= a.n_rows || !a.skip_cert[rl]) return;
  const int cnt = a.cand_cnt[rl];
  const long long row = a.row_map ? static_cast<long long>(a.row_map[rl]) : a.row0 + rl;
  const int nimp = a.imp_cnt[rl];
  const int2 im = lane < nimp ? a.imp[static_cast<long long>(rl) * SCAN_IMP_MAX + lane] : make_int2(0x7fffffff, 0);
  const float ts = tau_seed[row];
  const float f0 = __ldg(a.theta);
  const float xs_row = __ldg(a.xsq + row);
  const float dl_base = xs_row + *a.ysq_max;
  const int2* lrec = a.cand + static_cast<long long>(rl) * a.cap;
  int surv = 0;
  for (int e0 = 0; e0 < cnt; e0 += 32) {
    const int e = e0 + lane;
    const int2 r = e < cnt ? lrec[e] : make_int2(0, 0);
    const bool cert = e < cnt && r.x < 0;
    const int j = r.x & 0x7fffffff;
    int c = 0;
    for (int t = 0; t < nimp; ++t) c += __shfl_sync(FULL, im.x, t) < j;
    const float ti = __int_as_float(__shfl_sync(FULL, im.y, c > 0 ? c - 1 : 0));
    if (!cert) continue;
    const float thr0 = __fmul_rn(c > 0 ? ti : ts, f0);
    const float p = __int_as_float(r.y);
    const float dl = a.kap * (dl_base + p);
    if (__fsub_rn(p, dl) > thr0) continue;
    if (!(__fadd_rn(p, dl) > thr0)) {
      ++surv;
      continue;
    }
    const float pe = exact_front_dist(a.x + row * a.ldx, a.cent + static_cast<long long>(j) * a.ldc, a.d_prime,
                                      a.chain_flavour, a.chain_q, xs_row, __ldg(a.ysq + j));
    surv += !(pe > thr0);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) surv += __shfl_xor_sync(FULL, surv, o);
  if (lane == 0 && surv) {
    unsigned long long* ctr = a.group_counters ? a.group_counters + 3LL * __ldg(a.row_group + row) : a.counters;
    atomicAdd(&ctr[0], static_cast<unsigned long long>(surv));
    atomicAdd(&ctr[1], static_cast<unsigned long long>(surv) * static_cast<unsigned long long>(__ldg(a.block_dims)));
  }
}

inline size_t scan_dyn_smem(int nb, int d_prime = 0, bool ex_stage = false, int warps = SCAN_WARPS) {
  const int dpp = (d_prime + 3) & ~3;
  return static_cast<size_t>(warps) * (64 * nb + SCAN_WINDOW * nb + (ex_stage ? (1 + SCAN_EXS) * dpp : 0)) * 4;
}

}  // namespace skm
