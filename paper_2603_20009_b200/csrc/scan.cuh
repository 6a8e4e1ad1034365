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
//  * a warp-parallel in-order resolver replays the exact sequential semantics from the
//    recorded sums: a speculative evaluation always ran under a tau >= the exact one,
//    so it computed at least the blocks the exact walk needs (the exact walk prunes no
//    later).  Survivor / dims-touched counters therefore match the reference bitwise.
// Centroid tails are stored "PDX-quad" per centroid: T[j][q][b][r] = C[j][d'+64b+4q+r]
// (zero padded in the ragged last block -- adding +0 is exact), so the 4 lanes of a slot
// read 64 contiguous bytes per step.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace skm {

constexpr int SCAN_SLOTS = 8;
constexpr int SCAN_DEPTH = 4;
constexpr int SCAN_WINDOW = 64;   // in-flight queue positions per warp
constexpr int SCAN_NB_MAX = 40;   // tail blocks supported (d - d' <= 2560)
constexpr int SCAN_WARPS = 4;     // warps per CTA

struct ScanArgs {
  // candidate source (list mode)
  const int* cand_idx;
  const float* cand_val;
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
  long long row0;  // global row of batch-local row 0
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
};

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

// thr_i = sentinel ? inf : fl(tau_i * F0)
__global__ void gate_threshold_kernel(const float* __restrict__ tau, int n, float f0, int sentinel,
                                      float* __restrict__ thr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) thr[i] = sentinel ? __int_as_float(0x7f800000) : __fmul_rn(tau[i], f0);
}

struct ScanWarpSmem {
  // sized at launch: xsm[64*nb] floats, rec[WINDOW*nb] floats
  int qj[SCAN_WINDOW];
  float qp[SCAN_WINDOW];
  int qdone[SCAN_WINDOW];
};

template <bool DENSE>
__global__ void __launch_bounds__(SCAN_WARPS * 32)
    pruned_scan_kernel(const ScanArgs a) {
  extern __shared__ float scan_smem[];
  __shared__ ScanWarpSmem wsm[SCAN_WARPS];
  __shared__ float s_theta[SCAN_NB_MAX + 1];
  __shared__ int s_bdcum[SCAN_NB_MAX + 1];  // dims touched through block b (exclusive prefix at b+1)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  __syncthreads();

  float* xsm = scan_smem + static_cast<long long>(warp) * (64 * nb + SCAN_WINDOW * nb);
  float* rec = xsm + 64 * nb;
  ScanWarpSmem& W = wsm[warp];
  const float4* xsm4 = reinterpret_cast<const float4*>(xsm);
  const int tail_dims = s_bdcum[nb];
  const float f0 = s_theta[0];
  const unsigned FULL = 0xffffffffu;
  const int slot = lane / SCAN_DEPTH, dep = lane % SCAN_DEPTH;
  const bool slot_leader = dep == 0;

  unsigned long long surv_acc = 0, touched_acc = 0, changed_acc = 0;

  for (int r = blockIdx.x * SCAN_WARPS + warp; r < a.n_rows; r += gridDim.x * SCAN_WARPS) {
    const int rl = a.rows ? a.rows[r] : r;
    int n_src;
    if constexpr (DENSE) {
      n_src = a.k;
    } else {
      n_src = a.cand_cnt[rl];
      if (n_src > a.cap) continue;  // overflow row: handled by the dense pass
    }
    const long long row = a.row0 + rl;
    // ---- stage the x tail, quad layout (q, b, r)
    const float* xrow = a.x + row * a.ldx + a.d_prime;
    for (int u = lane; u < 64 * nb; u += 32) {
      const int b = u >> 6, t = u & 63;
      xsm[((t >> 2) * nb + b) * 4 + (t & 3)] = (u < tail_dims) ? xrow[u] : 0.0f;
    }
    float tcur = a.tau[row];
    int best = a.assign[row];
    const int best0 = best;
    int src = 0;        // next source entry to read
    int F = 0;          // queue fill pointer
    int D = 0;          // dispatch pointer
    int R = 0;          // resolve pointer
    // slot state (meaningful in all lanes of the slot; kept identical via shuffles)
    int spos = -1, snxt = 0;
    float srun = 0.0f;
    const float* dense_row = nullptr;
    const int* lidx = nullptr;
    const float* lval = nullptr;
    if constexpr (DENSE) {
      dense_row = a.dense + static_cast<long long>(a.dense_row[rl]) * a.ld_dense;
    } else {
      lidx = a.cand_idx + static_cast<long long>(rl) * a.cap;
      lval = a.cand_val + static_cast<long long>(rl) * a.cap;
    }
    __syncwarp();

    while (true) {
      // ---- 1. fill the queue (gate with the current tau: exact-safe, tau only shrinks)
      while (src < n_src && F - R <= SCAN_WINDOW - 32) {
        const int e = src + lane;
        int j = 0;
        float p = 0.0f;
        bool ok = e < n_src;
        if (ok) {
          if constexpr (DENSE) {
            j = e;
            p = dense_row[e];
          } else {
            j = lidx[e];
            p = lval[e];
          }
          ok = !(p > __fmul_rn(tcur, f0));
        }
        const unsigned m = __ballot_sync(FULL, ok);
        if (ok) {
          const int qpos = (F + __popc(m & ((1u << lane) - 1u))) % SCAN_WINDOW;
          W.qj[qpos] = j;
          W.qp[qpos] = p;
          W.qdone[qpos] = 0;
        }
        F += __popc(m);
        src += 32;
      }
      __syncwarp();
      if (R == F && src >= n_src) break;  // everything resolved
      // ---- 2. dispatch free slots in order
      {
        const unsigned freem = __ballot_sync(FULL, slot_leader && spos < 0);
        // slot s takes the rank-th free position
        if (spos < 0) {
          const unsigned my_leader_bit = 1u << (slot * SCAN_DEPTH);
          const int rank = __popc(freem & (my_leader_bit - 1u));
          const int p = D + rank;
          if (p < F && p < R + SCAN_WINDOW) {
            spos = p;
            snxt = 0;
            srun = W.qp[p % SCAN_WINDOW];
          }
        }
        const int nfree = __popc(freem);
        D = min(min(D + nfree, F), R + SCAN_WINDOW);
      }
      // ---- 3. one wave of speculative block sums
      if (spos >= 0) {
        const int b = snxt + dep;
        if (b < nb) {
          const int qs = spos % SCAN_WINDOW;
          const int j = W.qj[qs];
          const float4* cb = a.tails + static_cast<long long>(j) * 16 * nb + b;
          const float4* xb = xsm4 + b;
          float acc = 0.0f;
#pragma unroll 4
          for (int q = 0; q < 16; ++q) {
            const float4 c4 = __ldg(cb + q * nb);
            const float4 x4 = xb[q * nb];
            float df = __fsub_rn(x4.x, c4.x);
            acc = __fadd_rn(acc, __fmul_rn(df, df));
            df = __fsub_rn(x4.y, c4.y);
            acc = __fadd_rn(acc, __fmul_rn(df, df));
            df = __fsub_rn(x4.z, c4.z);
            acc = __fadd_rn(acc, __fmul_rn(df, df));
            df = __fsub_rn(x4.w, c4.w);
            acc = __fadd_rn(acc, __fmul_rn(df, df));
          }
          rec[qs * nb + b] = acc;
        }
      }
      __syncwarp();
      // ---- 4. slot leaders extend the running sum, mark done / speculatively dead
      {
        int fin_local = 0;
        if (spos >= 0 && slot_leader) {
          const int qs = spos % SCAN_WINDOW;
          const int hi = min(nb, snxt + SCAN_DEPTH);
          for (int b = snxt; b < hi; ++b) {
            srun = __fadd_rn(srun, rec[qs * nb + b]);
            if (srun > __fmul_rn(tcur, s_theta[b + 1])) { fin_local = 1; break; }
          }
          W.qdone[qs] = hi;
          if (hi >= nb) fin_local = 1;
        }
        const int finished = __shfl_sync(FULL, fin_local, slot * SCAN_DEPTH);
        if (spos >= 0) {
          snxt += SCAN_DEPTH;
          if (finished) spos = -1;
        }
      }
      __syncwarp();
      // ---- 5. in-order resolution, 32 positions per round
      while (R < D) {
        const int p = R + lane;
        int outcome = 0;  // 0 none(beyond D), 1 not survivor, 2 pruned, 3 complete, 4 incomplete
        float run = 0.0f;
        int pb = 0, j = 0;
        if (p < D) {
          const int qs = p % SCAN_WINDOW;
          const float pv = W.qp[qs];
          j = W.qj[qs];
          if (pv > __fmul_rn(tcur, f0)) {
            outcome = 1;
          } else {
            const int nd = W.qdone[qs];
            run = pv;
            outcome = 3;
            for (int b = 0; b < nb; ++b) {
              if (b >= nd) { outcome = 4; break; }
              run = __fadd_rn(run, rec[qs * nb + b]);
              if (run > __fmul_rn(tcur, s_theta[b + 1])) { outcome = 2; pb = b; break; }
            }
          }
        }
        const bool improve = outcome == 3 && (run < tcur || (run == tcur && j < best));
        const unsigned ev = __ballot_sync(FULL, improve || outcome == 4);
        const int limit = ev ? (__ffs(ev) - 1) : 32;  // lanes < limit are final
        const bool counted = lane < limit || (lane == limit && improve);
        unsigned long long s_add = 0, t_add = 0;
        if (counted && (outcome == 2 || outcome == 3)) {
          s_add = 1;
          t_add = (outcome == 2) ? s_bdcum[pb + 1] : tail_dims;
        }
        surv_acc += s_add;
        touched_acc += t_add;
        const int src_lane = ev ? limit : 0;
        const int ev_improve = __shfl_sync(FULL, (int)improve, src_lane);
        const float ev_run = __shfl_sync(FULL, run, src_lane);
        const int ev_j = __shfl_sync(FULL, j, src_lane);
        if (!ev) {
          R += min(32, D - R);
        } else if (ev_improve) {
          tcur = ev_run;
          best = ev_j;
          R += limit + 1;
        } else {
          R += limit;
          break;  // stalled on a candidate whose blocks are still being computed
        }
      }
      // slots whose candidate got resolved are released
      if (spos >= 0 && spos < R) spos = -1;
      __syncwarp();
    }
    if (lane == 0) {
      a.tau[row] = tcur;
      a.assign[row] = best;
      changed_acc += (best != best0);
    }
    __syncwarp();
  }
  warp_add_u64(surv_acc, &a.counters[0]);
  warp_add_u64(touched_acc, &a.counters[1]);
  warp_add_u64(changed_acc, &a.counters[2]);
}

inline size_t scan_dyn_smem(int nb) { return static_cast<size_t>(SCAN_WARPS) * (64 * nb + SCAN_WINDOW * nb) * 4; }

}  // namespace skm
