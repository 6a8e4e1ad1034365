// Production pruning scan: speculative pair scan with exact multi-round resolution.
//
// Reference semantics (core.py:230-263, _kernels.pyx:14-82): candidates j ascending, a
// threshold tau that starts at the seed tau_s = |x - c_{a0}|^2 (a0 = previous assignment) and
// changes only when a completed candidate beats it (run < tau, or run == tau and j < best);
// every candidate's gate / prune decisions use the tau current at its position.
//
// Segments.  Between two consecutive tau changes ("improvements") every candidate is
// independent of the others: pair (row, j) is a survivor iff !(p_j > fl(tau F0)) and walks
// 64-dim blocks until run > fl(tau F[b+1]).  A round evaluates each of its rows from a known
// state (position P of the last confirmed improvement, its tau and best; P = -1, tau_s, a0 at
// the start) in parallel over all later positions.  The most common tau change -- the row's
// own previous centroid a0, whose walked distance differs from tau_s by GEMM rounding -- is
// taken out of the segment by walking a0 first (row_prep_kernel): positions j < a0 then use
// tau, j > a0 the tau after a0.  The first (lowest-position) other candidate that improves ends
// the segment: the row "freezes" there (dispatch stops, in-flight pairs beyond it are
// cancelled) and the next round resumes it after that position with the improved tau.  A row
// needs one round per assignment change, usually 0 or 1; rows still open after SPEC_ROUNDS go
// to the exact sequential kernel (scan.cuh).
//
// Counters are exact: every position's outcome (dims touched, or -1 for "not a survivor") is
// recorded in `outcome[row][pos]` by the last round that evaluated it; rows that needed more
// than one round sum their records at the end, single-round rows use register totals.
//
// GPU mapping (per warp): lane = one (row, candidate) pair, one 64-dim block per pair per
// step; every lane owns TWO pair contexts that alternate between waves.  A context's next
// 256-byte candidate block (block-major tails T2[j][b][64], L2-resident) is fetched by a TMA
// bulk copy into the lane's shared-memory staging row while the warp computes the other
// context, so the L2 latency is covered by a full wave of work and the loads never touch the
// LSU/L1 path.  x tails of the warp's two in-flight rows are staged asynchronously (cp.async,
// quad layout T[q][b][4]: lanes at different blocks hit different banks, lanes of a row at
// the same block broadcast).  Per-row setup (the a0 walk, list search) is done beforehand by
// row_prep_kernel, and row descriptors / list chunks are prefetched one step ahead.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#include "ptx.cuh"
#include "scan.cuh"

namespace skm {

constexpr int SPEC_WARPS = 12;              // max warps per CTA (launched with as many as smem allows)
constexpr int SPEC_SLOTS = 2;               // rows in flight per warp
constexpr int SPEC_QUEUE = 128;             // dispatch ring (entries of the feeding row)
constexpr int SPEC_ROUNDS = 4;              // speculative rounds before the exact fallback
constexpr int PREP_WARPS = 8;

// T2[j][b][t] = C[j][d' + 64b + t] (0 beyond d): one candidate block = 256 contiguous bytes
__global__ void build_tails_blk_kernel(const float* __restrict__ cent, long long ldc, int k, int d, int d_prime,
                                       int nb, float* __restrict__ tails) {
  const long long per = 64LL * nb;
  const int tail = d - d_prime;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)k * per;
       e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / per;
    const int t = static_cast<int>(e - j * per);
    tails[e] = (t < tail) ? cent[j * ldc + d_prime + t] : 0.0f;
  }
}

struct SpecRound {
  int round;                 // 0: all rows of the batch (a.rows / identity); > 0: in_rows[0 .. *in_cnt)
  const int* in_rows;
  const unsigned int* in_cnt;
  int* out_rows;             // rows frozen this round (batch-local)
  unsigned int* out_cnt;
  int* st_pos;               // per batch-local row: position of the confirmed improvement
  float* st_tau;             //   its walked distance (the new tau)
  int* st_best;              //   its centroid (the new best)
  int* outcome;              // [batch rows][cap] per-position outcome records
};

// One row of a round, prepared by row_prep_kernel (9 words).
struct RowDesc {
  int row;      // global row
  int rl;       // batch-local row (candidate slab index)
  int n;        // candidates in the list; -1: overflow row (dense pass)
  int pos_in;   // first position this round evaluates
  int a0;       // previous assignment
  int best_r;   // best before the segment (a0 in round 0)
  int a0_dims;  // a0's outcome in this segment (-1: not walked / not a survivor)
  float t_lo;   // tau for positions with j < a0
  float t_hi;   // tau for positions with j > a0 (< t_lo iff a0 improved)
};
constexpr int DESC_WORDS = sizeof(RowDesc) / 4;

struct SpecSlot {
  int row, rl, a0, n, busy, frozen, fz_pos, fz_j, best_r, a0_impr;
  float fz_run, t_hi;
};

struct SpecWarpSmem {
  int qj[SPEC_QUEUE];
  float qp[SPEC_QUEUE];
  int qpos[SPEC_QUEUE];
  SpecSlot s[SPEC_SLOTS];
};

struct PairCtx {
  int slot, j, b, pos;
  float run, t;
  int tie;
};

__host__ __device__ inline int spec_slot_floats(int nb) { return 64 * nb + 4; }
// per warp: GENS x PAIRS x 32 lanes x 272-byte staging rows, then the two x-tail slots
__host__ __device__ inline int spec_stage_floats(int gens, int pairs) { return gens * pairs * 32 * 17 * 4; }
__host__ __device__ inline int spec_warp_floats(int nb, int gens, int pairs) {
  return spec_stage_floats(gens, pairs) + SPEC_SLOTS * spec_slot_floats(nb);
}
inline size_t spec_dyn_smem(int nb, int warps, int gens, int pairs) {
  return static_cast<size_t>(warps) * spec_warp_floats(nb, gens, pairs) * 4;
}
inline size_t prep_dyn_smem(int nb) { return static_cast<size_t>(PREP_WARPS) * (2 * 64 * nb + ((nb + 3) & ~3)) * 4; }

// sequential fp32 sum of one 64-dim block: (x - c)^2 per dim, ascending dims, no FMA
__device__ __forceinline__ float block_sum_quad(const float4* __restrict__ xq, int nb, const float4 (&c4)[16]) {
  float acc = 0.0f;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const float4 x4 = xq[q * nb];
    const float2 s01 = sq_diff2(make_float2(x4.x, x4.y), make_float2(c4[q].x, c4[q].y));
    const float2 s23 = sq_diff2(make_float2(x4.z, x4.w), make_float2(c4[q].z, c4[q].w));
    acc = __fadd_rn(acc, s01.x);
    acc = __fadd_rn(acc, s01.y);
    acc = __fadd_rn(acc, s23.x);
    acc = __fadd_rn(acc, s23.y);
  }
  return acc;
}

// Stage a row's tail (contiguous floats src[0 .. tail)) into quad layout dst[(q nb + b) 4 + r],
// zero beyond tail.  Async (cp.async, caller waits) when src is 16-byte aligned.
__device__ __forceinline__ void stage_tail_quad(float* dst, const float* src, int tail, int nb, int lane,
                                                bool aligned) {
  if (aligned) {
    for (int c = lane; c < 16 * nb; c += 32) {
      const int b = c >> 4, q = c & 15;
      const int valid = min(4, max(0, tail - 4 * c));
      cp_async_16_zfill(dst + (q * nb + b) * 4, valid ? src + 4 * c : src, 4 * valid);
    }
  } else {
    for (int u = lane; u < 64 * nb; u += 32) {
      const int b = u >> 6, t = u & 63;
      dst[((t >> 2) * nb + b) * 4 + (t & 3)] = (u < tail) ? src[u] : 0.0f;
    }
  }
}

__device__ __forceinline__ void load_scan_consts(const ScanArgs& a, float* s_theta, int* s_bdcum) {
  const int nb = a.nb;
  if (threadIdx.x <= nb) s_theta[threadIdx.x] = a.theta[threadIdx.x];
  if (threadIdx.x == 0) {
    int c = 0;
    s_bdcum[0] = 0;
    for (int b = 0; b < nb; ++b) {
      c += a.block_dims[b];
      s_bdcum[b + 1] = c;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Per-row setup of a round: locate a0 among the positions the round evaluates, walk it under
// the segment's tau (block sums in parallel, then the sequential chain), record its outcome,
// and write the row descriptor.  One warp per row.
__global__ void __launch_bounds__(PREP_WARPS * 32) row_prep_kernel(const ScanArgs a, const SpecRound R,
                                                                   RowDesc* __restrict__ desc) {
  extern __shared__ __align__(16) float prep_smem[];
  __shared__ float s_theta[SCAN_NB_MAX + 1];
  __shared__ int s_bdcum[SCAN_NB_MAX + 1];
  load_scan_consts(a, s_theta, s_bdcum);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = a.nb, cap = a.cap;
  const int tail_dims = s_bdcum[nb];
  const float f0 = s_theta[0];
  const unsigned FULL = 0xffffffffu;
  float* xq = prep_smem + static_cast<long long>(warp) * (2 * 64 * nb + ((nb + 3) & ~3));
  float* cq = xq + 64 * nb;
  float* rec = cq + 64 * nb;
  const bool x_aligned = ((a.ldx & 3) == 0) && ((a.d_prime & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  const int n_rows = R.round == 0 ? a.n_rows : static_cast<int>(*R.in_cnt);
  unsigned long long blocks_acc = 0;
  for (int r = blockIdx.x * PREP_WARPS + warp; r < n_rows; r += gridDim.x * PREP_WARPS) {
    const int rl = R.round == 0 ? (a.rows ? a.rows[r] : r) : R.in_rows[r];
    const int n_src = a.cand_cnt[rl];
    const long long row = a.row_map ? static_cast<long long>(a.row_map[rl]) : a.row0 + rl;
    RowDesc D;
    D.row = static_cast<int>(row);
    D.rl = rl;
    D.n = n_src;
    D.a0_dims = -1;
    if (n_src > cap) {  // overflow row: the dense pass owns it
      D.n = -1;
      if (lane == 0) desc[r] = D;
      continue;
    }
    const float tseed = a.tau[row];
    const int a0 = a.assign[row];
    D.a0 = a0;
    D.pos_in = 0;
    D.best_r = a0;
    D.t_lo = tseed;
    if (R.round > 0) {
      D.pos_in = R.st_pos[rl] + 1;
      D.t_lo = R.st_tau[rl];
      D.best_r = R.st_best[rl];
    }
    D.t_hi = D.t_lo;
    const int2* lrec = a.cand + static_cast<long long>(rl) * cap;
    int spos = -1;
    for (int e0 = D.pos_in; e0 < n_src; e0 += 32) {
      const int e = e0 + lane;
      const int j = (e < n_src) ? lrec[e].x : 0x7fffffff;
      const unsigned hit = __ballot_sync(FULL, j == a0);
      if (hit) { spos = e0 + __ffs(hit) - 1; break; }
      if (__ballot_sync(FULL, j > a0)) break;
    }
    if (spos >= 0) {
      int* lout = R.outcome + static_cast<long long>(rl) * cap;
      const float p0 = __int_as_float(lrec[spos].y);
      const float t = D.t_lo;
      if (!(p0 > __fmul_rn(t, f0))) {
        __syncwarp();
        stage_tail_quad(xq, a.x + row * a.ldx + a.d_prime, tail_dims, nb, lane, x_aligned);
        stage_tail_quad(cq, reinterpret_cast<const float*>(a.tails_blk + static_cast<long long>(a0) * 16 * nb),
                        64 * nb, nb, lane, true);
        cp_async_wait_all();
        __syncwarp();
        for (int b = lane; b < nb; b += 32) {
          float4 c4[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) c4[q] = reinterpret_cast<const float4*>(cq)[q * nb + b];
          rec[b] = block_sum_quad(reinterpret_cast<const float4*>(xq) + b, nb, c4);
        }
        __syncwarp();
        if (lane == 0) {
          float run = p0;
          int b = 0;
          bool pruned = false;
          for (; b < nb; ++b) {
            run = __fadd_rn(run, rec[b]);
            if (run > __fmul_rn(t, s_theta[b + 1])) { pruned = true; break; }
          }
          D.a0_dims = pruned ? s_bdcum[b + 1] : tail_dims;
          // a tie at a0 cannot improve: best is a0 itself (round 0) or a lower index
          if (!pruned && run < t) D.t_hi = run;
          lout[spos] = D.a0_dims;
          blocks_acc += pruned ? b + 1 : nb;
        }
      } else if (lane == 0) {
        lout[spos] = -1;
      }
    }
    if (lane == 0) desc[r] = D;
    __syncwarp();
  }
  if (a.counters_ext && lane == 0 && blocks_acc) atomicAdd(&a.counters_ext[0], blocks_acc);
}


// ------------------------------------------------------------------------------------------
// P interleaved sequential fp32 block sums (one 64-dim block each), operands in shared memory
// (x quad layout, c linear staging row): (x - c)^2 with packed FADD2/FMUL2 (per-lane IEEE RN,
// identical bits to the scalar ops), each chain ascending in dimension order.
template <int P>
__device__ __forceinline__ void block_sums_smem(const float4* const (&xq)[P], int nb, const float4* const (&cq)[P],
                                                float (&acc)[P]) {
#pragma unroll
  for (int k = 0; k < P; ++k) acc[k] = 0.0f;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const float4 xv = xq[k][q * nb];
      const float4 cv = cq[k][q];
      const float2 d01 = __fadd2_rn(make_float2(xv.x, xv.y), make_float2(-cv.x, -cv.y));
      const float2 d23 = __fadd2_rn(make_float2(xv.z, xv.w), make_float2(-cv.z, -cv.w));
      const float2 s01 = __fmul2_rn(d01, d01);
      const float2 s23 = __fmul2_rn(d23, d23);
      acc[k] = __fadd_rn(acc[k], s01.x);
      acc[k] = __fadd_rn(acc[k], s01.y);
      acc[k] = __fadd_rn(acc[k], s23.x);
      acc[k] = __fadd_rn(acc[k], s23.y);
    }
  }
}

// Warp-uniform state of the warp's two in-flight rows (registers; slot index s is uniform).
struct SlotRegs {
  int busy, row, rl, a0, n, best_r, a0_impr, frozen, fz_pos, fz_j, inflight;
  float t_hi, fz_run;
};

// GENS generations of P pair contexts per lane: wave w computes generation w % GENS (P
// interleaved chains) while the copies of the other generations are in flight.
template <int GENS, int P>
__global__ void __launch_bounds__(SPEC_WARPS * 32, 1)
    spec_scan_kernel(const ScanArgs a, const SpecRound R, const RowDesc* __restrict__ desc) {
  extern __shared__ __align__(16) float spec_smem[];
  __shared__ SpecWarpSmem wsm[SPEC_WARPS];
  __shared__ uint64_t gbar[SPEC_WARPS][GENS];
  __shared__ float s_theta[SCAN_NB_MAX + 1];
  __shared__ int s_bdcum[SCAN_NB_MAX + 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = a.nb;
  load_scan_consts(a, s_theta, s_bdcum);
  const int n_rows = R.round == 0 ? a.n_rows : static_cast<int>(*R.in_cnt);
  if (a.counters_ext && R.round > 0 && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&a.counters_ext[5], static_cast<unsigned long long>(n_rows));
  SpecWarpSmem& W = wsm[warp];
  uint64_t* mbar = gbar[warp];
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < GENS; ++g) mbar_init(&mbar[g], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (lane == 0) {  // complete phase 0 of every generation: the first waves have no data
#pragma unroll
    for (int g = 0; g < GENS; ++g) mbar_arrive(&mbar[g]);
  }
  __syncwarp();

  float* wbase = spec_smem + static_cast<long long>(warp) * spec_warp_floats(nb, GENS, P);
  float4* cstage = reinterpret_cast<float4*>(wbase);  // [GENS][P][32][17]
  float* xslots = wbase + spec_stage_floats(GENS, P);
  const int slot_f = spec_slot_floats(nb);
  const int tail_dims = s_bdcum[nb];
  const float f0 = s_theta[0];
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int cap = a.cap;
  const bool x_aligned = ((a.ldx & 3) == 0) && ((a.d_prime & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  const int* dwords = reinterpret_cast<const int*>(desc);

  // ---- row prefetch: the next row's descriptor words (lanes 0..8) and the row index after it
  int next_r = 0;
  if (lane == 0) next_r = static_cast<int>(atomicAdd(a.work, 1u));
  next_r = __shfl_sync(FULL, next_r, 0);
  int next_dw = (lane < DESC_WORDS && next_r < n_rows) ? dwords[static_cast<long long>(next_r) * DESC_WORDS + lane] : 0;
  int next2_r = 0;  // lane 0 only
  if (lane == 0) next2_r = static_cast<int>(atomicAdd(a.work, 1u));

  SlotRegs S0{}, S1{};
  // ---- feeding row (warp-uniform)
  int fs = -1, f_src = 0, f_n = 0, f_a0 = 0, f_best = 0, f_rl = 0;
  float f_tlo = 0.0f, f_thi = 0.0f;
  int qh = 0, qt = 0;
  bool rows_done = false;
  bool chunk_pending = false;
  int chunk_base = 0, lj = 0;
  float lp = 0.0f;

  PairCtx ctx[GENS][P];
#pragma unroll
  for (int g = 0; g < GENS; ++g)
#pragma unroll
    for (int k = 0; k < P; ++k) ctx[g][k] = PairCtx{-1, 0, 0, 0, 0.0f, 0.0f, 0};
  int cs0 = 0, cs1 = 0, ct0 = 0, ct1 = 0;  // register totals per slot (single-round rows)
  uint32_t phase_bits = 0;                 // bit g: parity of generation g's next wait
  unsigned long long tot_surv = 0, tot_touched = 0, tot_changed = 0, blocks_acc = 0, waves_acc = 0;

  auto finalize = [&](SlotRegs& S, int s) {
    if (S.frozen) {
      if (lane == 0) {
        const unsigned o = atomicAdd(R.out_cnt, 1u);
        R.out_rows[o] = S.rl;
        R.st_pos[S.rl] = S.fz_pos;
        R.st_tau[S.rl] = S.fz_run;
        R.st_best[S.rl] = S.fz_j;
      }
    } else {
      int vs, vt;
      if (R.round == 0) {
        vs = s ? cs1 : cs0;
        vt = s ? ct1 : ct0;
      } else {  // resolved over several rounds: every position's record is final
        const int* lout = R.outcome + static_cast<long long>(S.rl) * cap;
        vs = 0;
        vt = 0;
        for (int e = lane; e < S.n; e += 32) {
          const int v = lout[e];
          if (v >= 0) { vs += 1; vt += v; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        vs += __shfl_xor_sync(FULL, vs, o);
        vt += __shfl_xor_sync(FULL, vt, o);
      }
      if (lane == 0) {
        tot_surv += static_cast<unsigned>(vs);
        tot_touched += static_cast<unsigned>(vt);
        const int best = S.a0_impr ? S.a0 : S.best_r;
        a.tau[S.row] = S.t_hi;
        if (best != S.a0) {
          a.assign[S.row] = best;
          tot_changed += 1;
        }
      }
    }
    if (s) { cs1 = 0; ct1 = 0; } else { cs0 = 0; ct0 = 0; }
    S.busy = 0;
  };

  // freeze slot s at the lowest improving position among the improvers `mine[k]` of gen g
  auto freeze = [&](SlotRegs& S, int s, const PairCtx (&C)[P], const bool (&mine)[P], const float (&imp_run)[P]) {
    unsigned mypos = 0xffffffffu;
    float myrun = 0.0f;
    int myj = 0;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (mine[k] && static_cast<unsigned>(C[k].pos) < mypos) {
        mypos = static_cast<unsigned>(C[k].pos);
        myrun = imp_run[k];
        myj = C[k].j;
      }
    }
    const unsigned pmin = __reduce_min_sync(FULL, mypos);
    const int src = __ffs(__ballot_sync(FULL, mypos == pmin)) - 1;
    const float run = __shfl_sync(FULL, myrun, src);
    const int jmin = __shfl_sync(FULL, myj, src);
    const int P_ = static_cast<int>(pmin);
    if (!S.frozen || P_ < S.fz_pos) {
      S.frozen = 1;
      S.fz_pos = P_;
      S.fz_run = run;
      S.fz_j = jmin;
      // later positions are re-evaluated next round (their copies still land, unused)
      int cancelled = 0;
#pragma unroll
      for (int gg = 0; gg < GENS; ++gg)
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const bool c = ctx[gg][k].slot == s && ctx[gg][k].pos > P_;
          cancelled += __popc(__ballot_sync(FULL, c));
          if (c) ctx[gg][k].slot = -1;
        }
      S.inflight -= cancelled;
      if (s == fs) {
        qh = qt;
        f_src = f_n;
        chunk_pending = false;
      }
    }
  };

  auto wave = [&](auto gc) -> bool {
    constexpr int g = decltype(gc)::value;
    PairCtx (&C)[P] = ctx[g];
    float4* cst = cstage + g * P * 32 * 17;
    // ------------------------------------------------------------ 0. this generation's data
    cp_async_wait_group<GENS - 1>();
    mbar_wait(&mbar[g], (phase_bits >> g) & 1u);
    phase_bits ^= 1u << g;
    __syncwarp();
    // ------------------------------------------------------------ 1. one block per active context
    bool done[P], imp[P];
    float imp_run[P];
    {
      const float4* xq[P];
      const float4* cq[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        xq[k] = reinterpret_cast<const float4*>(xslots + max(C[k].slot, 0) * slot_f) + C[k].b;
        cq[k] = cst + (k * 32 + lane) * 17;
      }
      float acc[P];
      block_sums_smem<P>(xq, nb, cq, acc);
#pragma unroll
      for (int k = 0; k < P; ++k) {
        done[k] = false;
        imp[k] = false;
        imp_run[k] = 0.0f;
        if (C[k].slot >= 0) {
          ++blocks_acc;
          C[k].run = __fadd_rn(C[k].run, acc[k]);
          int dims = -1;
          if (C[k].run > __fmul_rn(C[k].t, s_theta[C[k].b + 1])) {
            dims = s_bdcum[C[k].b + 1];
          } else if (++C[k].b == nb) {
            dims = tail_dims;
            if (C[k].run < C[k].t || (C[k].run == C[k].t && C[k].tie)) {
              imp[k] = true;
              imp_run[k] = C[k].run;
            }
          }
          if (dims >= 0) {
            done[k] = true;
            const int rl = C[k].slot ? S1.rl : S0.rl;
            R.outcome[static_cast<long long>(rl) * cap + C[k].pos] = dims;
            if (C[k].slot) { cs1 += 1; ct1 += dims; } else { cs0 += 1; ct0 += dims; }
          }
        }
      }
    }
    {
      bool any_done = false, m0[P], m1[P];
      bool any_imp = false;
      int d_all = 0, d_one = 0;
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const unsigned dm = __ballot_sync(FULL, done[k]);
        if (dm) {
          any_done = true;
          d_all += __popc(dm);
          d_one += __popc(__ballot_sync(FULL, done[k] && C[k].slot == 1));
        }
        m0[k] = imp[k] && C[k].slot == 0;
        m1[k] = imp[k] && C[k].slot == 1;
        any_imp |= imp[k];
        if (done[k]) C[k].slot = -1;  // finished contexts are never cancelled below
      }
      if (any_done) {
        S1.inflight -= d_one;
        S0.inflight -= d_all - d_one;
      }
      // ------------------------------------------------------ 2. freeze rows at their first improvement
      if (__ballot_sync(FULL, any_imp)) {
        bool a0m = false, a1m = false;
#pragma unroll
        for (int k = 0; k < P; ++k) { a0m |= m0[k]; a1m |= m1[k]; }
        if (__ballot_sync(FULL, a0m)) freeze(S0, 0, C, m0, imp_run);
        if (__ballot_sync(FULL, a1m)) freeze(S1, 1, C, m1, imp_run);
      }
    }
    // ------------------------------------------------------------ 3. finalise drained rows
    if (S0.busy && fs != 0 && S0.inflight == 0) finalize(S0, 0);
    if (S1.busy && fs != 1 && S1.inflight == 0) finalize(S1, 1);
    // ------------------------------------------------------------ 4. admission
    if (fs >= 0 && f_src >= f_n && qh == qt && !chunk_pending) fs = -1;  // fully dispatched: drains
    while (fs < 0 && !rows_done) {
      const int free_s = !S0.busy ? 0 : (!S1.busy ? 1 : -1);
      if (free_s < 0) break;
      if (next_r >= n_rows) { rows_done = true; break; }
      RowDesc D;
      {
        int* dd = reinterpret_cast<int*>(&D);
#pragma unroll
        for (int i = 0; i < DESC_WORDS; ++i) dd[i] = __shfl_sync(FULL, next_dw, i);
      }
      // prefetch the row after (its index was fetched one admission ago)
      next_r = __shfl_sync(FULL, next2_r, 0);
      next_dw = (lane < DESC_WORDS && next_r < n_rows) ? dwords[static_cast<long long>(next_r) * DESC_WORDS + lane] : 0;
      if (lane == 0) next2_r = static_cast<int>(atomicAdd(a.work, 1u));
      if (D.n < 0) continue;  // overflow row: the dense pass owns it
      stage_tail_quad(xslots + free_s * slot_f, a.x + static_cast<long long>(D.row) * a.ldx + a.d_prime, tail_dims,
                      nb, lane, x_aligned);
      SlotRegs& S = free_s ? S1 : S0;
      S.busy = 1;
      S.row = D.row;
      S.rl = D.rl;
      S.a0 = D.a0;
      S.n = D.n;
      S.best_r = D.best_r;
      S.a0_impr = D.t_hi < D.t_lo;
      S.t_hi = D.t_hi;
      S.frozen = 0;
      S.inflight = 0;
      if (lane == 0 && D.a0_dims >= 0) {
        if (free_s) { cs1 += 1; ct1 += D.a0_dims; } else { cs0 += 1; ct0 += D.a0_dims; }
      }
      fs = free_s;
      f_src = D.pos_in;
      f_n = D.n;
      f_a0 = D.a0;
      f_best = D.best_r;
      f_tlo = D.t_lo;
      f_thi = D.t_hi;
      f_rl = D.rl;
      qh = qt = 0;
      chunk_pending = false;
      if (f_src >= f_n) fs = -1;  // nothing to dispatch: finalised once drained
    }
    // ------------------------------------------------------------ 5. queue: insert the chunk loaded last wave, load the next
    unsigned idle[P];
    int n_idle = 0;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      idle[k] = __ballot_sync(FULL, C[k].slot < 0);
      n_idle += __popc(idle[k]);
    }
    int n_act = P * 32 - n_idle;
    if (fs >= 0) {
      if (chunk_pending) {
        const int e = chunk_base + lane;
        bool ok = false;
        if (e < f_n) {
          const float tj = (lj < f_a0) ? f_tlo : f_thi;
          ok = (lj != f_a0) && !(lp > __fmul_rn(tj, f0));
          if (!ok && lj != f_a0) R.outcome[static_cast<long long>(f_rl) * cap + e] = -1;
        }
        const unsigned m = __ballot_sync(FULL, ok);
        if (ok) {
          const int qs = (qt + __popc(m & lt_mask)) & (SPEC_QUEUE - 1);
          W.qj[qs] = lj;
          W.qp[qs] = lp;
          W.qpos[qs] = e;
        }
        qt += __popc(m);
        chunk_pending = false;
      }
      if (f_src < f_n && qt - qh <= SPEC_QUEUE - 32) {
        const int e = f_src + lane;
        if (e < f_n) {
          const int2 rec = a.cand[static_cast<long long>(f_rl) * cap + e];
          lj = rec.x;
          lp = __int_as_float(rec.y);
        }
        chunk_base = f_src;
        f_src += 32;
        chunk_pending = true;
      }
      __syncwarp();
      // -------------------------------------------------------- 6. dispatch to idle contexts of this generation
      const int avail = qt - qh;
      if (n_idle && avail) {
        const int take = min(avail, n_idle);
        int base = 0;
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const int rank = base + __popc(idle[k] & lt_mask);
          if (C[k].slot < 0 && rank < take) {
            const int qs = (qh + rank) & (SPEC_QUEUE - 1);
            C[k].j = W.qj[qs];
            C[k].run = W.qp[qs];
            C[k].pos = W.qpos[qs];
            C[k].slot = fs;
            C[k].b = 0;
            C[k].t = (C[k].j < f_a0) ? f_tlo : f_thi;
            C[k].tie = C[k].j < f_best;
          }
          base += __popc(idle[k]);
        }
        qh += take;
        n_act += take;
        if (fs) S1.inflight += take; else S0.inflight += take;
      }
    }
    // ------------------------------------------------------------ 7. fetch this generation's next blocks (TMA)
    if (n_act) ++waves_acc;
    fence_proxy_async_smem();  // this wave's reads of the staging rows precede the async overwrite
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&mbar[g], 256u * static_cast<unsigned>(n_act));
    __syncwarp();
#pragma unroll
    for (int k = 0; k < P; ++k)
      if (C[k].slot >= 0)
        bulk_g2s(cst + (k * 32 + lane) * 17, a.tails_blk + (static_cast<long long>(C[k].j) * nb + C[k].b) * 16, 256u,
                 &mbar[g]);
    cp_async_commit();
    // ------------------------------------------------------------ exit when nothing is left
    return rows_done && fs < 0 && !S0.busy && !S1.busy;
  };

  static_assert(GENS >= 1 && GENS <= 3, "1..3 generations");
  for (int w = 0;; ++w) {
    bool fin = false;
    const int g = w % GENS;
    if (g == 0) fin = wave(std::integral_constant<int, 0>{});
    else if (g == 1) fin = wave(std::integral_constant<int, (GENS > 1 ? 1 : 0)>{});
    else fin = wave(std::integral_constant<int, (GENS > 2 ? 2 : 0)>{});
    if (fin) {
      // drain the other generations' pending phases (cancelled contexts may have copies in flight)
#pragma unroll
      for (int gg = 0; gg < GENS; ++gg)
        if (gg != g) mbar_wait(&mbar[gg], (phase_bits >> gg) & 1u);
      break;
    }
  }
  cp_async_wait_all();
  if (lane == 0) {
    if (tot_surv) atomicAdd(&a.counters[0], tot_surv);
    if (tot_touched) atomicAdd(&a.counters[1], tot_touched);
    if (tot_changed) atomicAdd(&a.counters[2], tot_changed);
  }
  if (a.counters_ext) {
    warp_add_u64(blocks_acc, &a.counters_ext[0]);
    if (lane == 0 && waves_acc) atomicAdd(&a.counters_ext[1], waves_acc);
  }
}


// ------------------------------------------------------------------------------------------
// pair_scan_kernel<K>: same semantics as spec_scan_kernel, different execution shape.  A lane
// walks its pair through an inner loop of K blocks with no warp-collective operation: per-lane
// mbarriers, block b computed from one staging buffer while block b+1 is already in flight
// into the other (TMA bulk copy, issued one block ahead).  Warp-level control -- freezes,
// finalising drained rows, row admission, queue refill, dispatch to idle lanes -- runs once
// every K blocks.  The next row's x tail is staged (cp.async) while the current row feeds.
__host__ __device__ inline int pair_warp_floats(int nb) { return 2 * 32 * 17 * 4 + SPEC_SLOTS * spec_slot_floats(nb); }
inline size_t pair_dyn_smem(int nb, int warps) { return static_cast<size_t>(warps) * pair_warp_floats(nb) * 4; }

template <int K>
__global__ void __launch_bounds__(SPEC_WARPS * 32, 1)
    pair_scan_kernel(const ScanArgs a, const SpecRound R, const RowDesc* __restrict__ desc) {
  extern __shared__ __align__(16) float spec_smem[];
  __shared__ SpecWarpSmem wsm[SPEC_WARPS];
  __shared__ uint64_t lbar[SPEC_WARPS][2][32];
  __shared__ float s_theta[SCAN_NB_MAX + 1];
  __shared__ int s_bdcum[SCAN_NB_MAX + 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = a.nb;
  load_scan_consts(a, s_theta, s_bdcum);
  const int n_rows = R.round == 0 ? a.n_rows : static_cast<int>(*R.in_cnt);
  if (a.counters_ext && R.round > 0 && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&a.counters_ext[5], static_cast<unsigned long long>(n_rows));
  SpecWarpSmem& W = wsm[warp];
  uint64_t* bar0 = &lbar[warp][0][lane];
  uint64_t* bar1 = &lbar[warp][1][lane];
  mbar_init(bar0, 1);
  mbar_init(bar1, 1);
  fence_mbar_init();
  __syncthreads();

  float* wbase = spec_smem + static_cast<long long>(warp) * pair_warp_floats(nb);
  float4* stg0 = reinterpret_cast<float4*>(wbase) + lane * 17;            // buffer 0 row of this lane
  float4* stg1 = reinterpret_cast<float4*>(wbase) + (32 + lane) * 17;     // buffer 1 row
  float* xslots = wbase + 2 * 32 * 17 * 4;
  const int slot_f = spec_slot_floats(nb);
  const int tail_dims = s_bdcum[nb];
  const float f0 = s_theta[0];
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int cap = a.cap;
  const bool x_aligned = ((a.ldx & 3) == 0) && ((a.d_prime & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  const int* dwords = reinterpret_cast<const int*>(desc);
  const float4* tails = a.tails_blk;

  // ---- row prefetch: the next row's descriptor words (lanes 0..8) and the row index after it
  int next_r = 0;
  if (lane == 0) next_r = static_cast<int>(atomicAdd(a.work, 1u));
  next_r = __shfl_sync(FULL, next_r, 0);
  int next_dw = (lane < DESC_WORDS && next_r < n_rows) ? dwords[static_cast<long long>(next_r) * DESC_WORDS + lane] : 0;
  int next2_r = 0;  // lane 0 only
  if (lane == 0) next2_r = static_cast<int>(atomicAdd(a.work, 1u));

  SlotRegs S0{}, S1{};
  // feeding row state (warp-uniform); `staged` = slot whose x is being staged for the next row
  int fs = -1, staged = -1, f_src = 0, f_n = 0, f_a0 = 0, f_best = 0, f_rl = 0;
  float f_tlo = 0.0f, f_thi = 0.0f;
  int st_pos_in = 0, st_n = 0, st_a0 = 0, st_best = 0, st_rl = 0;
  float st_tlo = 0.0f, st_thi = 0.0f;
  int qh = 0, qt = 0;
  bool rows_done = false;
  bool chunk_pending = false;
  int chunk_base = 0, lj = 0;
  float lp = 0.0f;

  // ---- lane pair state
  int pslot = -1, pj = 0, pb = 0, ppos = 0, cur = 0;
  float prun = 0.0f, pt = 0.0f;
  bool ptie = false;
  uint32_t pend = 0, ph = 0;  // bit i: copy pending on buffer i / parity of buffer i's next wait
  int fin_slot = -1;          // slot of the pair this lane finished since the last control step
  bool imp = false;
  float imp_run = 0.0f;
  int imp_pos = 0, imp_j = 0, imp_slot = -1;
  int cs0 = 0, cs1 = 0, ct0 = 0, ct1 = 0;
  unsigned long long tot_surv = 0, tot_touched = 0, tot_changed = 0, blocks_acc = 0, waves_acc = 0;

  auto wait_buf = [&](int i) {
    mbar_wait(i ? bar1 : bar0, (ph >> i) & 1u);
    ph ^= 1u << i;
    pend &= ~(1u << i);
  };
  auto issue = [&](int i, int j, int b) {
    if ((pend >> i) & 1u) wait_buf(i);  // a wasted prefetch still landing in this buffer
    fence_proxy_async_smem();
    uint64_t* bar = i ? bar1 : bar0;
    mbar_arrive_expect_tx(bar, 256u);
    bulk_g2s(i ? stg1 : stg0, tails + (static_cast<long long>(j) * nb + b) * 16, 256u, bar);
    pend |= 1u << i;
  };

  auto finalize = [&](SlotRegs& S, int s) {
    if (S.frozen) {
      if (lane == 0) {
        const unsigned o = atomicAdd(R.out_cnt, 1u);
        R.out_rows[o] = S.rl;
        R.st_pos[S.rl] = S.fz_pos;
        R.st_tau[S.rl] = S.fz_run;
        R.st_best[S.rl] = S.fz_j;
      }
    } else {
      int vs, vt;
      if (R.round == 0) {
        vs = s ? cs1 : cs0;
        vt = s ? ct1 : ct0;
      } else {  // resolved over several rounds: every position's record is final
        const int* lout = R.outcome + static_cast<long long>(S.rl) * cap;
        vs = 0;
        vt = 0;
        for (int e = lane; e < S.n; e += 32) {
          const int v = lout[e];
          if (v >= 0) { vs += 1; vt += v; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        vs += __shfl_xor_sync(FULL, vs, o);
        vt += __shfl_xor_sync(FULL, vt, o);
      }
      if (lane == 0) {
        tot_surv += static_cast<unsigned>(vs);
        tot_touched += static_cast<unsigned>(vt);
        const int best = S.a0_impr ? S.a0 : S.best_r;
        a.tau[S.row] = S.t_hi;
        if (best != S.a0) {
          a.assign[S.row] = best;
          tot_changed += 1;
        }
      }
    }
    if (s) { cs1 = 0; ct1 = 0; } else { cs0 = 0; ct0 = 0; }
    S.busy = 0;
  };

  auto freeze = [&](SlotRegs& S, int s, bool mine) {
    const unsigned pmin = __reduce_min_sync(FULL, mine ? static_cast<unsigned>(imp_pos) : 0xffffffffu);
    const int src = __ffs(__ballot_sync(FULL, mine && static_cast<unsigned>(imp_pos) == pmin)) - 1;
    const float run = __shfl_sync(FULL, imp_run, src);
    const int jmin = __shfl_sync(FULL, imp_j, src);
    const int P_ = static_cast<int>(pmin);
    if (!S.frozen || P_ < S.fz_pos) {
      S.frozen = 1;
      S.fz_pos = P_;
      S.fz_run = run;
      S.fz_j = jmin;
      // later positions are re-evaluated next round (their pending copies are drained lazily)
      const bool c = pslot == s && ppos > P_;
      S.inflight -= __popc(__ballot_sync(FULL, c));
      if (c) pslot = -1;
      if (s == fs) {
        qh = qt;
        f_src = f_n;
        chunk_pending = false;
      }
    }
  };

  // stage the next row into slot `s` (x copy in flight, descriptor kept in st_*); false: no row
  auto stage_next = [&](int s) -> bool {
    while (true) {
      if (next_r >= n_rows) { rows_done = true; return false; }
      RowDesc D;
      {
        int* dd = reinterpret_cast<int*>(&D);
#pragma unroll
        for (int i = 0; i < DESC_WORDS; ++i) dd[i] = __shfl_sync(FULL, next_dw, i);
      }
      next_r = __shfl_sync(FULL, next2_r, 0);
      next_dw = (lane < DESC_WORDS && next_r < n_rows) ? dwords[static_cast<long long>(next_r) * DESC_WORDS + lane] : 0;
      if (lane == 0) next2_r = static_cast<int>(atomicAdd(a.work, 1u));
      if (D.n < 0) continue;  // overflow row: the dense pass owns it
      stage_tail_quad(xslots + s * slot_f, a.x + static_cast<long long>(D.row) * a.ldx + a.d_prime, tail_dims, nb,
                      lane, x_aligned);
      cp_async_commit();
      SlotRegs& S = s ? S1 : S0;
      S.busy = 1;
      S.row = D.row;
      S.rl = D.rl;
      S.a0 = D.a0;
      S.n = D.n;
      S.best_r = D.best_r;
      S.a0_impr = D.t_hi < D.t_lo;
      S.t_hi = D.t_hi;
      S.frozen = 0;
      S.inflight = 0;
      if (lane == 0 && D.a0_dims >= 0) {
        if (s) { cs1 += 1; ct1 += D.a0_dims; } else { cs0 += 1; ct0 += D.a0_dims; }
      }
      st_pos_in = D.pos_in;
      st_n = D.n;
      st_a0 = D.a0;
      st_best = D.best_r;
      st_tlo = D.t_lo;
      st_thi = D.t_hi;
      st_rl = D.rl;
      staged = s;
      return true;
    }
  };

  while (true) {
    // ================================================================ control step
    {
      // ---- rows: pairs finished since the last control step
      const unsigned fm = __ballot_sync(FULL, fin_slot >= 0);
      if (fm) {
        const int d1 = __popc(__ballot_sync(FULL, fin_slot == 1));
        S1.inflight -= d1;
        S0.inflight -= __popc(fm) - d1;
      }
      if (__ballot_sync(FULL, imp)) {
        const bool m0 = imp && imp_slot == 0, m1 = imp && imp_slot == 1;
        if (__ballot_sync(FULL, m0)) freeze(S0, 0, m0);
        if (__ballot_sync(FULL, m1)) freeze(S1, 1, m1);
      }
      fin_slot = -1;
      imp = false;
      // ---- finalise drained rows (not feeding, not staged, nothing in flight)
      if (S0.busy && fs != 0 && staged != 0 && S0.inflight == 0) finalize(S0, 0);
      if (S1.busy && fs != 1 && staged != 1 && S1.inflight == 0) finalize(S1, 1);
      // ---- feeding row exhausted: the staged row (if any) takes over
      if (fs >= 0 && f_src >= f_n && qh == qt && !chunk_pending) fs = -1;
      while (fs < 0) {
        if (staged < 0) {
          if (rows_done) break;
          const int free_s = !S0.busy ? 0 : (!S1.busy ? 1 : -1);
          if (free_s < 0 || !stage_next(free_s)) break;
        }
        cp_async_wait_all();  // its x tail (issued at least one step ago, normally) has landed
        __syncwarp();
        fs = staged;
        staged = -1;
        f_src = st_pos_in;
        f_n = st_n;
        f_a0 = st_a0;
        f_best = st_best;
        f_tlo = st_tlo;
        f_thi = st_thi;
        f_rl = st_rl;
        qh = qt = 0;
        chunk_pending = false;
        if (f_src >= f_n) fs = -1;  // nothing to dispatch: finalised once drained
      }
      // ---- stage the next row early into the free slot
      if (staged < 0 && !rows_done) {
        const int free_s = !S0.busy ? 0 : (!S1.busy ? 1 : -1);
        if (free_s >= 0) stage_next(free_s);
      }
      // ---- queue: insert the chunk loaded last step, load the next
      const unsigned idle = __ballot_sync(FULL, pslot < 0);
      if (fs >= 0) {
        if (chunk_pending) {
          const int e = chunk_base + lane;
          bool ok = false;
          if (e < f_n) {
            const float tj = (lj < f_a0) ? f_tlo : f_thi;
            ok = (lj != f_a0) && !(lp > __fmul_rn(tj, f0));
            if (!ok && lj != f_a0) R.outcome[static_cast<long long>(f_rl) * cap + e] = -1;
          }
          const unsigned m = __ballot_sync(FULL, ok);
          if (ok) {
            const int qs = (qt + __popc(m & lt_mask)) & (SPEC_QUEUE - 1);
            W.qj[qs] = lj;
            W.qp[qs] = lp;
            W.qpos[qs] = e;
          }
          qt += __popc(m);
          chunk_pending = false;
        }
        if (f_src < f_n && qt - qh <= SPEC_QUEUE - 32) {
          const int e = f_src + lane;
          if (e < f_n) {
            const int2 rec = a.cand[static_cast<long long>(f_rl) * cap + e];
            lj = rec.x;
            lp = __int_as_float(rec.y);
          }
          chunk_base = f_src;
          f_src += 32;
          chunk_pending = true;
        }
        __syncwarp();
        // ---- dispatch to idle lanes: block 0 now, block 1 prefetched
        const int avail = qt - qh;
        if (idle && avail) {
          const int rank = __popc(idle & lt_mask);
          const int take = min(avail, __popc(idle));
          if (pslot < 0 && rank < take) {
            const int qs = (qh + rank) & (SPEC_QUEUE - 1);
            pj = W.qj[qs];
            prun = W.qp[qs];
            ppos = W.qpos[qs];
            pslot = fs;
            pb = 0;
            pt = (pj < f_a0) ? f_tlo : f_thi;
            ptie = pj < f_best;
            issue(cur, pj, 0);
            if (nb > 1) issue(cur ^ 1, pj, 1);
          }
          qh += take;
          if (fs) S1.inflight += take; else S0.inflight += take;
        }
      }
      if (rows_done && fs < 0 && staged < 0 && !S0.busy && !S1.busy) break;
      if (__ballot_sync(FULL, pslot >= 0)) ++waves_acc;
    }
    // ================================================================ K blocks, lane-local
#pragma unroll 1
    for (int it = 0; it < K; ++it) {
      if (pslot >= 0) {
        wait_buf(cur);
        const float4* xq = reinterpret_cast<const float4*>(xslots + pslot * slot_f) + pb;
        const float4* const xqs[1] = {xq};
        const float4* const cqs[1] = {cur ? stg1 : stg0};
        float acc[1];
        block_sums_smem<1>(xqs, nb, cqs, acc);
        ++blocks_acc;
        prun = __fadd_rn(prun, acc[0]);
        int dims = -1;
        if (prun > __fmul_rn(pt, s_theta[pb + 1])) {
          dims = s_bdcum[pb + 1];
        } else if (++pb == nb) {
          dims = tail_dims;
          if (prun < pt || (prun == pt && ptie)) {
            imp = true;
            imp_run = prun;
            imp_pos = ppos;
            imp_j = pj;
            imp_slot = pslot;
          }
        } else {
          // block pb is already landing in the other buffer; prefetch pb + 1 into this one
          if (pb + 1 < nb) issue(cur, pj, pb + 1);
          cur ^= 1;
        }
        if (dims >= 0) {
          const int rl = pslot ? S1.rl : S0.rl;
          R.outcome[static_cast<long long>(rl) * cap + ppos] = dims;
          if (pslot) { cs1 += 1; ct1 += dims; } else { cs0 += 1; ct0 += dims; }
          fin_slot = pslot;
          pslot = -1;
          cur ^= 1;  // the buffer that may still receive a wasted prefetch is drained lazily
        }
      }
      if (fin_slot >= 0) break;  // this lane idles until the next control step
    }
    __syncwarp();
  }
  // drain every copy still landing in this lane's buffers
  if (pend & 1u) wait_buf(0);
  if (pend & 2u) wait_buf(1);
  cp_async_wait_all();
  if (lane == 0) {
    if (tot_surv) atomicAdd(&a.counters[0], tot_surv);
    if (tot_touched) atomicAdd(&a.counters[1], tot_touched);
    if (tot_changed) atomicAdd(&a.counters[2], tot_changed);
  }
  if (a.counters_ext) {
    warp_add_u64(blocks_acc, &a.counters_ext[0]);
    if (lane == 0 && waves_acc) atomicAdd(&a.counters_ext[1], waves_acc);
  }
}

}  // namespace skm
