// Flat pruning scan: the exact scan for rows whose threshold only changes at their own centroid.
//
// In the reference's scan (_kernels.pyx:14-82, core.py:230-263) a row's threshold tau starts at
// the seed (the distance to its previous centroid a0) and only changes when a candidate completes
// every checkpoint with a running sum below it.  In a converging fit almost every row keeps a0:
// tau then changes at most once, at a0's own position (a0's running sum, computed in the scan's
// arithmetic, can be below the seed computed in the seed's).  This kernel evaluates a0 first,
// exactly, which fixes the row's whole tau trajectory: tau_seed before a0, tau_after from a0 on.
// Every other candidate is then an independent walk under a known threshold -- no in-order
// resolution, no tau versions, no re-walks -- in 8 slots x 4 blocks per wave like
// pruned_scan_kernel.  The trajectory is correct iff no other candidate "improves" under it:
//   j < a0:  run_j <= tau_seed   (ties at a lower index replace a0),
//   j > a0:  run_j <  tau_after.
// A row where that can happen (its assignment changes, or an interval cannot rule it out) is
// appended to a fallback list and handed, untouched, to pruned_scan_kernel, so every row's
// outcome, survivors and dims touched are the reference's bit for bit.  Decisions on the
// tensor-core front distances use the same rigorous intervals and the same warp-cooperative exact
// chain re-evaluation as pruned_scan_kernel.
#pragma once
#include "scan.cuh"

namespace skm {

inline size_t flat_dyn_smem(int nb, int d_prime) {
  const int dpp = (d_prime + 3) & ~3;
  return static_cast<size_t>(SCAN_WARPS) * (64 * nb + SCAN_SLOTS * nb + (1 + SCAN_EXS) * dpp) * 4;
}

struct FlatWarpSmem {
  int sel[32];
  float blk[SCAN_NB_MAX];  // a0's block sums
};

__global__ void __launch_bounds__(SCAN_WARPS * 32, SKM_SCAN_MINB)
    flat_scan_kernel(const ScanArgs a, int* __restrict__ fb_rows, unsigned int* __restrict__ fb_count) {
  extern __shared__ float flat_smem[];
  __shared__ FlatWarpSmem wsm[SCAN_WARPS];
  __shared__ float s_theta[SCAN_NB_MAX + 1];
  __shared__ int s_bdcum[SCAN_NB_MAX + 1];

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

  const int dpp = (a.d_prime + 3) & ~3;
  float* xsm = flat_smem + static_cast<long long>(warp) * (64 * nb + SCAN_SLOTS * nb + (1 + SCAN_EXS) * dpp);
  const float4* xsm4 = reinterpret_cast<const float4*>(xsm);
  float* srec_all = xsm + 64 * nb;         // [slot][nb] block sums of the slot's candidate
  float* xfs = srec_all + SCAN_SLOTS * nb;  // the row's d' front
  float* cfs = xfs + dpp;                   // SCAN_EXS staged centroid fronts
  FlatWarpSmem& W = wsm[warp];
  const int tail_dims = s_bdcum[nb];
  const float f0 = s_theta[0];
  const unsigned FULL = 0xffffffffu;
  const bool x_aligned = ((a.ldx & 3) == 0) && ((a.d_prime & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  const bool c_aligned = x_aligned && ((a.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.cent) & 15) == 0);
  const int slot = lane / SCAN_DEPTH, dep = lane % SCAN_DEPTH;
  const bool slot_leader = dep == 0;
  const unsigned leader_mask = (SCAN_DEPTH == 4) ? 0x11111111u : (SCAN_DEPTH == 8) ? 0x01010101u
                              : (SCAN_DEPTH == 2) ? 0x55555555u : 0xffffffffu;
  float* srec = srec_all + slot * nb;

  unsigned long long surv_acc = 0, touched_acc = 0;
  int cur_g = -1;
  auto flush_group = [&]() {
    if (cur_g >= 0) {
      unsigned long long* gc = a.group_counters + 3LL * cur_g;
      warp_add_u64(surv_acc, &gc[0]);
      warp_add_u64(touched_acc, &gc[1]);
    }
    surv_acc = touched_acc = 0;
  };

  // warp-cooperative staging of up to SCAN_EXS centroid fronts (lanes in `batch` own one each)
  auto stage_fronts = [&](unsigned batch, int jmine) {
    int sc = 0;
    for (unsigned bm = batch; bm; bm &= bm - 1u, ++sc) {
      const int jj = __shfl_sync(FULL, jmine, __ffs(bm) - 1);
      const float* crow = a.cent + static_cast<long long>(jj) * a.ldc;
      float* dst = cfs + sc * dpp;
      if (c_aligned) {
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
  };

  while (true) {
    int r = 0;
    if (lane == 0) r = static_cast<int>(atomicAdd(a.work, 1u));
    r = __shfl_sync(FULL, r, 0);
    if (r >= a.n_rows) break;
    const int rl = a.rows ? a.rows[r] : r;
    const int n_src = a.cand_cnt[rl];
    if (n_src > a.cap) continue;  // overflow row: the dense pass
    const long long row = a.row_map ? static_cast<long long>(a.row_map[rl]) : a.row0 + rl;
    if (a.group_counters) {
      const int g = __ldg(a.row_group + row);
      if (g != cur_g) {
        flush_group();
        cur_g = g;
      }
    }
    // ---- stage the x tail (quad layout) and the d' front (every lane is done with the previous
    //      row's shared-memory reads first)
    __syncwarp();
    const float* xrow = a.x + row * a.ldx;
    if (x_aligned) {
      for (int c = lane; c < 16 * nb; c += 32) {
        const int b = c >> 4, q = c & 15;
        const int valid = min(4, max(0, tail_dims - 4 * c));
        cp_async_16_zfill(xsm + (q * nb + b) * 4, valid ? xrow + a.d_prime + 4 * c : xrow, 4 * valid);
      }
      for (int c = lane; c < dpp / 4; c += 32) {
        const int valid = min(4, a.d_prime - 4 * c);
        cp_async_16_zfill(xfs + 4 * c, xrow + 4 * c, 4 * valid);
      }
    } else {
      for (int u = lane; u < 64 * nb; u += 32) {
        const int b = u >> 6, t = u & 63;
        xsm[((t >> 2) * nb + b) * 4 + (t & 3)] = (u < tail_dims) ? xrow[a.d_prime + u] : 0.0f;
      }
      for (int u = lane; u < dpp; u += 32) xfs[u] = u < a.d_prime ? xrow[u] : 0.0f;
    }
    const float tau_seed = a.tau[row];
    const int a0 = a.assign[row];
    const float dl_base = __ldg(a.xsq + row) + *a.ysq_max;
    const float xs_row = __ldg(a.xsq + row);
    const int2* lrec = a.cand + static_cast<long long>(rl) * a.cap;
    // a0 needs no lookup: its exact front distance decides the gate, and when it passes, the
    // emission (a superset of every candidate whose exact value may pass) listed it.  The
    // candidate records stream through a 64-entry register window (positions src + lane and
    // src + 32 + lane), so their L2 latency overlaps a0's evaluation and the previous waves.
    int2 cur = make_int2(0, 0), pre = make_int2(0, 0);
    if (lane < n_src) cur = lrec[lane];
    if (32 + lane < n_src) pre = lrec[32 + lane];
    cp_async_wait_all();
    __syncwarp();
    unsigned long long row_surv = 0, row_touch = 0;  // lane partials, committed if the row verifies
    float tau_after = tau_seed;
    // ---- a0 first, exactly (its running sum may become tau)
    {
      stage_fronts(1u, a0);
      float pe = 0.0f;
      if (lane == 0)
        pe = exact_front_dist_staged(xfs, cfs, a.d_prime, a.chain_flavour, a.chain_q, xs_row, __ldg(a.ysq + a0));
      pe = __shfl_sync(FULL, pe, 0);
      if (!(pe > __fmul_rn(tau_seed, f0))) {  // survivor
        {
          for (int b = lane; b < nb; b += 32) {
            const float4* cb = a.tails + static_cast<long long>(a0) * 16 * nb + b;
            float acc = 0.0f;
#pragma unroll 4
            for (int q = 0; q < 16; ++q) {
              const float4 x4 = xsm4[q * nb + b];
              const float4 c4 = __ldg(cb + q * nb);
              const float2 s01 = sq_diff2(make_float2(x4.x, x4.y), make_float2(c4.x, c4.y));
              const float2 s23 = sq_diff2(make_float2(x4.z, x4.w), make_float2(c4.z, c4.w));
              acc = __fadd_rn(acc, s01.x);
              acc = __fadd_rn(acc, s01.y);
              acc = __fadd_rn(acc, s23.x);
              acc = __fadd_rn(acc, s23.y);
            }
            W.blk[b] = acc;
          }
          __syncwarp();
          if (lane == 0) {
            float run = pe;
            int pb = -1;
            for (int b = 0; b < nb; ++b) {
              run = __fadd_rn(run, W.blk[b]);
              if (run > __fmul_rn(tau_seed, s_theta[b + 1])) {
                pb = b;
                break;
              }
            }
            row_surv += 1;
            row_touch += pb >= 0 ? s_bdcum[pb + 1] : tail_dims;
            if (pb < 0 && run < tau_seed) tau_after = run;  // a0 is the best already: strict
          }
          tau_after = __shfl_sync(FULL, tau_after, 0);
          __syncwarp();
        }
      }
    }
    // ---- every other candidate under its known threshold, 8 slots x 4 blocks per wave
    int src = 0;
    int spos = -1, sj = 0, snxt = 0;                 // all lanes of the slot
    float stc = 0.0f;                                // leader: the candidate's threshold
    float slo = 0.0f, shi = 0.0f;                    // leader: running-sum interval
    bool samb = false, sneed = false, scert = false; // leader
    bool failed = false;
    while (true) {
      // 1. dispatch: positions that the gate decides for certain are consumed on the spot
      {
        unsigned free_left = __ballot_sync(FULL, slot_leader && spos < 0) & leader_mask;
        while (free_left && src < n_src) {
          const int e = src + lane;
          const int2 rr = cur;
          const int j = rr.x & 0x7fffffff;
          const bool ok = e < n_src && j != a0;
          const bool cert = rr.x < 0;
          const float p = __int_as_float(rr.y);
          const float tc = j < a0 ? tau_seed : tau_after;
          const float dl = a.kap * (dl_base + p);
          const float thr0 = __fmul_rn(tc, f0);
          const bool gate_fail = __fsub_rn(p, dl) > thr0;     // not a survivor, for certain
          const bool gate_pass = !(__fadd_rn(p, dl) > thr0);  // a survivor, for certain
          const bool decided = ok && !gate_fail && cert && gate_pass;
          const bool need = ok && !gate_fail && !decided;
          const unsigned pm = __ballot_sync(FULL, need);
          const int nfree = __popc(free_left);
          int cut = min(32, n_src - src);
          if (__popc(pm) >= nfree) {
            const bool nth = need && __popc(pm & ((1u << lane) - 1u)) == nfree - 1;
            cut = __ffs(__ballot_sync(FULL, nth));
          }
          {  // slide the record window by cut positions
            const int sl2 = (lane + cut) & 31;
            const bool wrap = lane + cut >= 32;
            const int cx = __shfl_sync(FULL, cur.x, sl2), cy = __shfl_sync(FULL, cur.y, sl2);
            const int px = __shfl_sync(FULL, pre.x, sl2), py = __shfl_sync(FULL, pre.y, sl2);
            cur = wrap ? make_int2(px, py) : make_int2(cx, cy);
            pre = make_int2(px, py);
            if (wrap) {
              const int idx = src + cut + 32 + lane;
              pre = idx < n_src ? lrec[idx] : make_int2(0, 0);
            }
          }
          if (lane < cut && decided) {
            row_surv += 1;
            row_touch += s_bdcum[1];
          }
          const unsigned took = pm & ((cut >= 32) ? FULL : ((1u << cut) - 1u));
          if ((took >> lane) & 1u) W.sel[__popc(took & ((1u << lane) - 1u))] = lane;
          __syncwarp();
          int src_lane = -1;
          if (slot_leader && ((free_left >> lane) & 1u)) {
            const int my_rank = __popc(free_left & ((1u << lane) - 1u));
            if (my_rank < __popc(took)) src_lane = W.sel[my_rank];
          }
          __syncwarp();
          // the taken positions' fields go to their slot leaders, then to the slot's lanes
          const int sl = __shfl_sync(FULL, src_lane, slot * SCAN_DEPTH);
          const int nj = __shfl_sync(FULL, j, sl < 0 ? 0 : sl);
          const float np_ = __shfl_sync(FULL, p, sl < 0 ? 0 : sl);
          const float ndl = __shfl_sync(FULL, dl, sl < 0 ? 0 : sl);
          const float ntc = __shfl_sync(FULL, tc, sl < 0 ? 0 : sl);
          const bool ncert = __shfl_sync(FULL, (int)cert, sl < 0 ? 0 : sl) != 0;
          const bool ngp = __shfl_sync(FULL, (int)gate_pass, sl < 0 ? 0 : sl) != 0;
          const unsigned assigned = __ballot_sync(FULL, slot_leader && sl >= 0);
          if (sl >= 0) {
            spos = src + sl;
            sj = nj;
            snxt = 0;
            stc = ntc;
            scert = ncert;
            slo = fmaxf(__fsub_rn(np_, ndl), 0.0f);
            shi = __fadd_rn(np_, ndl);
            samb = !ngp;            // the gate itself is not settled
            sneed = ncert;          // certified but gate unsettled: exact p decides
          }
          free_left &= ~assigned;
          src += cut;
          __syncwarp();
        }
      }
      if (__ballot_sync(FULL, spos >= 0) == 0 && src >= n_src) break;
      // 2. exact front distances for the slots that need them, then their exact re-walks
      {
        unsigned needm = __ballot_sync(FULL, slot_leader && spos >= 0 && sneed);
        while (needm) {
          unsigned batch = 0, mm = needm;
#pragma unroll
          for (int s2 = 0; s2 < SCAN_EXS; ++s2) {
            if (mm) {
              batch |= mm & (0u - mm);
              mm &= mm - 1u;
            }
          }
          stage_fronts(batch, sj);
          if ((batch >> lane) & 1u) {
            const int my = __popc(batch & ((1u << lane) - 1u));
            const float pe = exact_front_dist_staged(xfs, cfs + my * dpp, a.d_prime, a.chain_flavour, a.chain_q,
                                                     xs_row, __ldg(a.ysq + sj));
            sneed = false;
            samb = false;
            int fin = 0;  // 1 not survivor, 2 pruned (counted), 3 complete -> violation check below
            if (pe > __fmul_rn(stc, f0)) {
              fin = 1;
            } else if (scert) {
              row_surv += 1;
              row_touch += s_bdcum[1];
              fin = 2;
            } else {
              float run = pe;
              for (int b = 0; b < snxt && b < nb; ++b) {
                run = __fadd_rn(run, srec[b]);
                if (run > __fmul_rn(stc, s_theta[b + 1])) {
                  row_surv += 1;
                  row_touch += s_bdcum[b + 1];
                  fin = 2;
                  break;
                }
              }
              slo = shi = run;
              if (!fin && snxt >= nb) {
                fin = 3;
                const bool viol = sj < a0 ? !(run > tau_seed) : run < tau_after;
                if (viol) {
                  failed = true;
                } else {
                  row_surv += 1;
                  row_touch += tail_dims;
                }
              }
            }
            if (fin) spos = -1;
          }
          __syncwarp();
          needm &= ~batch;
        }
        // release the slots resolved above in every lane of the slot
        spos = __shfl_sync(FULL, spos, slot * SCAN_DEPTH);
      }
      if (__any_sync(FULL, failed)) break;
      // 3. this wave's block sums (4 consecutive blocks of each active slot's candidate)
      const int myb = snxt + dep;
      const bool active = spos >= 0 && myb < nb;
      float acc = 0.0f;
      if (active) {
        float4 c4[16];
        const float4* cb = a.tails + static_cast<long long>(sj) * 16 * nb + myb;
#pragma unroll
        for (int q = 0; q < 16; ++q) c4[q] = __ldg(cb + q * nb);
        const float4* xb = xsm4 + myb;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float4 x4 = xb[q * nb];
          const float2 s01 = sq_diff2(make_float2(x4.x, x4.y), make_float2(c4[q].x, c4[q].y));
          const float2 s23 = sq_diff2(make_float2(x4.z, x4.w), make_float2(c4[q].z, c4[q].w));
          acc = __fadd_rn(acc, s01.x);
          acc = __fadd_rn(acc, s01.y);
          acc = __fadd_rn(acc, s23.x);
          acc = __fadd_rn(acc, s23.y);
        }
        srec[myb] = acc;
      }
      // 4. slot leaders walk the wave's blocks on the interval
      float blk[SCAN_DEPTH];
#pragma unroll
      for (int i = 0; i < SCAN_DEPTH; ++i) blk[i] = __shfl_sync(FULL, acc, slot * SCAN_DEPTH + i);
      int fin = 0;
      if (slot_leader && spos >= 0 && !sneed) {
        const int hi = min(nb, snxt + SCAN_DEPTH);
#pragma unroll
        for (int i = 0; i < SCAN_DEPTH; ++i) {
          if (!fin && snxt + i < hi) {
            const int b = snxt + i;
            slo = __fadd_rn(slo, blk[i]);
            shi = __fadd_rn(shi, blk[i]);
            const float thr = __fmul_rn(stc, s_theta[b + 1]);
            if (slo > thr) {
              if (samb) {
                sneed = true;  // an earlier checkpoint (or the gate) was not settled
              } else {
                row_surv += 1;
                row_touch += s_bdcum[b + 1];
                fin = 2;
              }
            }
            samb = samb || shi > thr;
            if (sneed) break;
          }
        }
        if (!fin && !sneed && hi >= nb) {
          // complete: is the row's trajectory still right? (the candidate must not improve)
          const bool viol_lo = sj < a0 ? !(slo > tau_seed) : slo < tau_after;  // possible
          const bool viol_hi = sj < a0 ? !(shi > tau_seed) : shi < tau_after;  // certain
          if (samb || (viol_lo && !viol_hi)) {
            sneed = true;
          } else if (viol_hi) {
            failed = true;
          } else {
            row_surv += 1;
            row_touch += tail_dims;
            fin = 3;
          }
        }
      }
      fin = __shfl_sync(FULL, fin, slot * SCAN_DEPTH);
      if (spos >= 0) {
        snxt = min(nb, snxt + SCAN_DEPTH);
        if (fin) spos = -1;
      }
      if (__any_sync(FULL, failed)) break;
    }
    if (__any_sync(FULL, failed)) {
      if (lane == 0) fb_rows[atomicAdd(fb_count, 1u)] = rl;  // untouched: the exact kernel redoes it
      continue;
    }
    surv_acc += row_surv;
    touched_acc += row_touch;
    if (lane == 0) a.tau[row] = tau_after;  // assignment unchanged (a0 stays the best)
  }
  if (a.group_counters) {
    flush_group();
  } else {
    warp_add_u64(surv_acc, &a.counters[0]);
    warp_add_u64(touched_acc, &a.counters[1]);
  }
}

}  // namespace skm
