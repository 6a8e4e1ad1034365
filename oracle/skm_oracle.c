/*
 * ORACLE -- test / baseline infrastructure only (never linked into the product).
 *
 * Plain-C + OpenMP restatement of the reference's compiled kernel backend so the CPU
 * baseline runs at the speed of the reference's Cython build:
 *   oracle_scan_bank         follows pkg/src/superkmeans/_kernels.pyx:14-82
 *   oracle_seed_thresholds   follows pkg/src/superkmeans/_kernels.pyx:85-103
 *   oracle_accumulate_sums   follows pkg/src/superkmeans/_kernels.pyx:106-119
 * Built with -O3 -fopenmp -ffp-contract=off (the reference's flags, pkg/setup.py:13-15) so
 * the per-element float semantics (no FMA, ascending order) are identical.
 */
#include <math.h>
#include <stdint.h>

void oracle_scan_bank(const float* pd, long n, long kb, const float* x, long ldx, const float* tail,
                      const long long* block_offsets, const int* block_dims, long n_blocks, const float* theta,
                      long d_prime, long bank_offset, float* tau, int* assign, int sentinel, int n_threads,
                      long long* out_counts) {
  long long survivors = 0, touched = 0;
#pragma omp parallel for schedule(dynamic, 8) num_threads(n_threads) reduction(+ : survivors, touched)
  for (long i = 0; i < n; ++i) {
    float tcur = tau[i];
    int best = assign[i];
    for (long j = 0; j < kb; ++j) {
      float gate = sentinel ? INFINITY : tcur * theta[0];
      const float p = pd[i * kb + j];
      if (p > gate) continue;
      survivors += 1;
      float running = p;
      int pruned = 0;
      long xoff = d_prime;
      for (long b = 0; b < n_blocks; ++b) {
        const long bd = block_dims[b];
        const long coff = block_offsets[b] + j;
        float acc = 0.0f;
        for (long t = 0; t < bd; ++t) {
          const float diff = x[i * ldx + xoff + t] - tail[coff + t * kb];
          acc = acc + diff * diff;
        }
        touched += bd;
        running = running + acc;
        xoff += bd;
        gate = (sentinel && b < n_blocks - 1) ? INFINITY : tcur * theta[b + 1];
        if (running > gate) {
          pruned = 1;
          break;
        }
      }
      if (!pruned) {
        if (running < tcur) {
          best = (int)(bank_offset + j);
          tcur = running;
        } else if (running == tcur && bank_offset + j < best) {
          best = (int)(bank_offset + j);
        }
      }
    }
    tau[i] = tcur;
    assign[i] = best;
  }
  out_counts[0] = survivors;
  out_counts[1] = touched;
}

void oracle_seed_thresholds(const float* x, long n, long d, const float* c, const int* assign, float* out,
                            int n_threads) {
#pragma omp parallel for schedule(static) num_threads(n_threads)
  for (long i = 0; i < n; ++i) {
    const float* xr = x + i * d;
    const float* cr = c + (long)assign[i] * d;
    float acc = 0.0f;
    for (long t = 0; t < d; ++t) {
      const float diff = xr[t] - cr[t];
      acc = acc + diff * diff;
    }
    out[i] = acc;
  }
}

void oracle_accumulate_sums(const float* x, long n, long d, const int* assign, double* sums, long long* counts) {
  for (long i = 0; i < n; ++i) {
    const long c = assign[i];
    counts[c] += 1;
    for (long t = 0; t < d; ++t) sums[c * d + t] += (double)x[i * d + t];
  }
}
