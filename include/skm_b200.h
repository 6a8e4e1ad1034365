/*
 * skm_b200.h -- C ABI of libskm_b200.so, the B200 (sm_100a) SuperKMeans hot path.
 *
 * Every entry point is extern "C", takes plain device pointers, element counts and leading
 * dimensions (in elements), plus an opaque cudaStream_t passed as void*.  Calls are
 * stream-ordered and asynchronous; none allocates device memory (scratch comes from the
 * caller through the *_workspace_bytes queries).  Return value: 0 on success, a negative
 * SKM_E* code otherwise; skm_last_error() describes the last failure of the calling thread.
 *
 * Reference interfaces replaced (paths relative to the reference repository root):
 *   skm_scan_bank                <- scan_bank                pkg/src/superkmeans/_kernels.pyx:14-82
 *   skm_seed_thresholds          <- seed_thresholds          pkg/src/superkmeans/_kernels.pyx:85-103
 *   skm_accumulate_centroid_sums <- accumulate_centroid_sums pkg/src/superkmeans/_kernels.pyx:106-119
 *   skm_portable_matmul          <- portable_matmul          pkg/src/superkmeans/_kernels.pyx:122-142
 *   skm_gemm_tf32x3              <- matmul (sgemm `af @ bf.T`) + expand_to_sq_l2
 *                                   pkg/src/superkmeans/distance.py:46-82, apply/unapply_rotation
 *                                   preprocess.py:37-52, full-pass argmin core.py:183-190
 *   skm_row_sq_norms             <- row_sq_norms             pkg/src/superkmeans/preprocess.py:95-101
 *   skm_cluster_sort / skm_cluster_sums / skm_finalize_centroids
 *                                <- update_centroids         pkg/src/superkmeans/core.py:79-100
 *                                   build_cluster_lists      pkg/src/superkmeans/evaluation.py:78-83
 *   skm_apply_splits             <- split_empty_clusters row arithmetic, core.py:119-125
 *   skm_pruned_scan              <- _pruned_assign_pass inner loop, core.py:230-263
 *   skm_etr_*                    <- brute_force_topk / etr_probe, evaluation.py:53-75, 142-170
 */
#ifndef SKM_B200_H
#define SKM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define SKM_OK 0
#define SKM_E_CUDA (-1)
#define SKM_E_ARG (-2)
#define SKM_E_DRIVER (-3)
#define SKM_E_WORKSPACE (-4)

const char* skm_last_error(void);
/* cumulative count of kernels this library has launched (all devices) */
long long skm_kernel_launches(void);
int skm_abi_version(void);

/* ---- layout / preprocessing --------------------------------------------------------- */
/* hi = x with the low 13 mantissa bits cleared, lo = x - hi (exact); pad columns -> 0. */
/* hi may be NULL: lo only.  tcgen05 kind::tf32 truncates raw fp32 operands exactly like the
 * explicit hi (x & 0xFFFFE000; tools/trunc_probe.py: bit-identical products), so the fp32 rows
 * themselves serve as the hi operand and only lo needs storing. */
int skm_split_hilo(const float* x, long long ldx, int rows, int cols, float* hi, float* lo, long long ldo,
                   void* stream);
/* out[r] = f32(sum_{c<dims} (f64)x[r,c]^2) */
int skm_row_sq_norms(const float* x, long long ldx, int rows, int dims, float* out, void* stream);
/* out[r,:cols] = in[idx[r],:cols] */
int skm_gather_rows(const float* in, long long ldi, const long long* idx, int rows, int cols, float* out,
                    long long ldo, void* stream);
/* evaluation.wcss (evaluation.py:205-215): *out = sum_i |x_i - c_{assign_i}|^2 (f64),
 * deterministic; workspace: skm_wcss_workspace_bytes() of device memory. */
long long skm_wcss_workspace_bytes(void);
int skm_wcss(const float* x, long long ldx, const float* centroids, long long ldc, const int* assign, long long n,
             int d, double* out, void* workspace, void* stream);
/* validate_vector_set's finiteness check (model.py:84-87): *first = min row-major flat index
 * (row * cols + col) of a NaN/Inf in the leading cols columns, or ~0 when all finite. */
int skm_first_nonfinite(const float* x, long long ldx, long long rows, int cols, unsigned long long* first,
                        void* stream);
/* Vector-file ingestion (dataio.py:57-112): validate + scatter `rows` staged records (fvecs:
 * rec_words = d + 1, header_words = 1; fbin: d, 0) starting at file row row0 into out (ld ldo).
 * bad_dim / bad_val[row / 4096] = min(bad record row) / min(non-finite flat index). */
int skm_ingest_records(const void* raw, long long rows, int d, int rec_words, int header_words, long long row0,
                       float* out, long long ldo, unsigned long long* bad_dim, unsigned long long* bad_val,
                       void* stream);
/* Gate-batch gather: ohi/olo[r, :cols] = hi/lo[idx[r], :cols], oxsq[r] = xsq[idx[r]],
 * othr[r] = thr[idx[r]] (rows in cluster order for the gate GEMM); optionally (non-NULL) the
 * certification terms oxsq_ext[r] = xsq_ext[idx[r]], othr1[r] = thr1[idx[r]]. */
int skm_gather_front(const float* hi, const float* lo, long long ldi, const int* idx, int rows, int cols, float* ohi,
                     float* olo, long long ldo, const float* xsq, const float* thr, float* oxsq, float* othr,
                     const float* xsq_ext, const float* thr1, float* oxsq_ext, float* othr1, void* stream);
int skm_gather_rows_i32(const float* in, long long ldi, const int* idx, int rows, int cols, float* out,
                        long long ldo, void* stream);
int skm_fill_f32(float* p, long long n, float v, void* stream);
int skm_copy_i32(const int* src, int* dst, int n, void* stream);

/* ---- the reference kernel protocol, on device memory (bitwise parity entries) -------- */
int skm_seed_thresholds(const float* x, long long ldx, const float* centroids, long long ldc, const int* assign,
                        int n, int d, float* out, void* stream);
/* counters: device u64[2] += {survivors, dims_touched} */
int skm_scan_bank(const float* partial_dists, int n, int kb, const float* x, long long ldx, const float* tail,
                  const long long* block_offsets, const int* block_dims, int n_blocks, const float* theta_factors,
                  int d_prime, int bank_offset, float* tau, int* assign, int sentinel,
                  unsigned long long* counters, void* stream);
long long skm_update_workspace_bytes(int n, int k);
int skm_accumulate_centroid_sums(const float* x, long long ldx, const int* assign, int n, int d, int k,
                                 double* sums, long long* counts, void* workspace, long long workspace_bytes,
                                 void* stream);
int skm_portable_matmul(const float* a, long long lda, const float* b, long long ldb, int n, int m, int dims,
                        float* out, long long ldo, void* stream);

/* ---- tensor-core GEMM (3xTF32 on tcgen05/TMEM, TMA-fed) ------------------------------ */
enum skm_gemm_mode { SKM_GEMM_STORE = 0, SKM_GEMM_DIST = 1, SKM_GEMM_ARGMIN = 2, SKM_GEMM_GATE = 3 };
typedef struct skm_gemm_params {
  /* operands: row-major, K contiguous; hi/lo from skm_split_hilo; ld multiple of 4 */
  const float* a_hi; const float* a_lo; long long lda;
  const float* b_hi; const float* b_lo; long long ldb;
  int M, N, K;
  int mode;
  int n_split;                 /* CTAs along N (ARGMIN with n_split>1 goes through keys) */
  float* out; long long ldo;   /* STORE / DIST */
  const float* xsq;            /* per-row norm (DIST/ARGMIN/GATE) */
  const float* ysq;            /* per-column norm */
  int* top;                    /* ARGMIN: int4 records {best bits, best col, second bits, 0} per
                                * (N split, row): top[4 * (split * M + row)]; skm_argmin_merge */
  const float* thr;            /* GATE: per-row threshold (keep iff dist <= thr) */
  int* cand; int* cand_cnt; int cand_cap;  /* cand: [M][cand_cap] records {index, float bits} */
  long long row_offset;        /* ARGMIN/GATE output row offset */
  /* GATE, optional: ext_k (64) more columns after K certify tail-block-0 prunes; certified
   * candidates carry bit 31 in the record's index.  xsq_ext/ysq_ext: norms over K + ext_k columns,
   * thr1: per-row fl(tau * F[1]), cert_eps: margin relative to xsq_ext + ysq_ext. */
  int ext_k; const float* xsq_ext; const float* ysq_ext; const float* thr1; float cert_eps;
  /* grouped columns (hierarchical fine phase, ARGMIN / GATE, n_split 1): row i only sees columns
   * [row_crange[i].x, row_crange[i].y) (its group's centroids); M tile t walks only the N tiles
   * covering [tile_nrange[t].x, tile_nrange[t].y) (the union of its rows' ranges).  Both int2. */
  const int* row_crange; const int* tile_nrange;
  /* GATE extension as one TF32 product (hi x hi): a third of its MMAs, for a certificate whose
   * cert_eps covers 2^-9 of xsq_ext + ysq_ext (exact_work_stats = false) */
  int ext_hi_only;
} skm_gemm_params;
int skm_gemm_tf32x3(const skm_gemm_params* p, void* stream);
/* Merge the ARGMIN top-2 records: assign = lowest index among the smallest distances, tau = its
 * tensor-core distance; rows whose runner-up lies within the rigorous tensor-core error bound
 * (kap * (2 (xsq + *ysq_max) + best + second)) are appended to amb_rows (count in *amb_count,
 * zeroed by the caller) for an exact re-evaluation (core.py:183-190 semantics). */
int skm_argmin_merge(const int* top, int n_split, int n, const float* xsq, const float* ysq_max, float kap,
                     int* assign, float* tau, int* amb_rows, unsigned int* amb_count, void* stream);
/* Exact argmin (lowest column on ties) of dense distance rows; writes assign/tau[row_ids[r]]. */
int skm_dense_argmin(const float* dist, long long ld, int rows, int cols, const int* row_ids, int* assign,
                     float* tau, void* stream);
/* tau[i] = the reference's GEMM + expansion distance of (row i, centroid assign[i]): inner product
 * chain of skm_chain_gemm (flavour, q) over d, then max(0, fl(fl(-2 ip + xsq_i) + ysq_a)). */
int skm_exact_pair_dist(const float* x, long long ldx, const float* centroids, long long ldc, const int* assign,
                        int n, int d, const float* xsq, const float* ysq, int flavour, int q, float* out,
                        void* stream);
/* Ambiguous argmin rows (global indices rows[0..n_rows)): thr[r] = GATE threshold keeping every
 * column whose exact distance may be <= the exact best (tau holds the tensor-core best), xs_out[r] =
 * xsq[rows[r]]; then skm_cand_exact_argmin: exact chain distance of every candidate (cand lists in
 * GATE layout [n_rows][cap]), lowest column among the smallest, into assign/tau[rows[r]]
 * (rows with cand_cnt > cap are skipped: the caller re-evaluates them whole). */
int skm_argmin_candidates(const int* rows, int n_rows, const float* tau, const float* xsq, const float* ysq_max,
                          float kap, float* thr, float* xs_out, void* stream);
int skm_cand_exact_argmin(const int* rows, int n_rows, const int* cand, const int* cand_cnt, int cap, const float* x,
                          long long ldx, const float* centroids, long long ldc, int d, const float* xsq,
                          const float* ysq, int flavour, int q, int* assign, float* tau, void* stream);
/* *out = max(v[0..n)) (>= 0), one CTA */
int skm_max_f32(const float* v, int n, float* out, void* stream);

/* ---- exact-chain fp32 GEMM on the CUDA cores (bitwise the reference's GEMM backends) -------
 * out[i][j] = chain over t < K of a[i][t] * b[j][t]; flavour 0 = fused multiply-add chain with
 * OpenBLAS's threaded K blocking (q = 448: blocks restart from +0 and are added to the output),
 * flavour 1 = separate multiply / add chain (portable_matmul, _kernels.pyx:122-142; q = 0).
 * mode 0 stores the products, mode 1 the clamped squared distances
 * max(0, fl(fl(-2 acc + xsq_i) + ysq_j)) (distance.py:66-82 / evaluation.py:42-50).
 * Replaces: preprocess.py:37-52 (x @ R, C @ R^T), evaluation.py:42-50 (queries @ x.T). */
typedef struct skm_chain_params {
  const float* a; long long lda;
  const float* b; long long ldb;
  int M, N, K;
  int flavour;                 /* 0 fma (OpenBLAS sgemm), 1 mul+add (portable) */
  int q;                       /* K block of the blocked driver (448), 0 = one chain */
  int mode;                    /* 0 store, 1 distance */
  float* out; long long ldo;
  const float* xsq; const float* ysq;
  int b_kmajor;                /* 0: b is [N][K] (b[j][t]); 1: b is [K][N] (b[t][j], e.g. R for x @ R) */
} skm_chain_params;
int skm_chain_gemm(const skm_chain_params* p, void* stream);
/* Fused exact-chain distances + per-tile top-k (the ETR ground truth without the distance matrix).
 * rows: the collection [n][K] (row-major, ldr); queries_t: the queries k-major [K][nq] (ldq % 4 == 0).
 * For query j and 128-row tile t, out_{v,i}[(j * n_tiles + t) * k_top + r] = the k_top smallest
 * max(0, fl(fl(-2 chain(q_j . x_i) + q_sq_j) + row_sq_i)) of the tile's rows with the row index
 * i + col_offset, ascending by (value, row); (+inf, INT_MAX) past the tile's rows.
 * n_tiles = ceil(n / 128), k_top <= 32, chain flavour / q as skm_chain_gemm (all K blocks in one
 * launch, each added to the running sum with one fp32 add).
 * Replaces: evaluation.py:42-75 (distances + argsort of each query's row). */
int skm_chain_topk_tiles(const float* rows, long long ldr, const float* queries_t, long long ldq, int n, int nq, int K,
                         int flavour, int q, const float* row_sq, const float* q_sq, int k_top, float* out_v,
                         int* out_i, int col_offset, void* stream);

/* ---- centroid update ------------------------------------------------------------------ */
/* stable sort of row ids by assignment; counts/offsets int32[k] */
int skm_cluster_sort(const int* assign, int n, int k, int* order, int* counts, int* offsets, void* workspace,
                     long long workspace_bytes, void* stream);
/* mode 0: centroids[c] = f32(sum/count) for count>0 (others untouched); mode 1: sums (f64, k x d) */
int skm_cluster_sums(const float* x, long long ldx, const int* order, const int* offsets, const int* counts, int k,
                     int d, double* sums, int accumulate, float* centroids, long long ldc, int mode, void* stream);
int skm_finalize_centroids(const double* sums, const long long* counts, int k, int d, float* centroids,
                           long long ldc, void* stream);
int skm_counts_to_i64(const int* c32, long long* c64, int k, int accumulate, void* stream);
int skm_apply_splits(float* centroids, long long ldc, int d, const int* empties, const int* donors, int n_splits,
                     float eps, void* stream);
/* stats[0] (f64) = sum(tau), stats[1] (u64) = count(assign != prev) (prev may be NULL) */
long long skm_stats_workspace_bytes(int n);
/* out[c] = NumPy's pairwise sum (f64) of tau[8192 c, 8192 (c + 1)) -- the per-buffer partials of
 * np.sum(tau, dtype=np.float64) (core.py:344); summed in buffer order they give wcss bitwise. */
int skm_tau_chunk_sums(const float* tau, long long n, double* out, void* stream);
int skm_assign_stats(const float* tau, const int* assign, const int* prev, int n, double* out_sum,
                     unsigned long long* out_changed, void* workspace, long long workspace_bytes, void* stream);


/* ---- production pruning scan (fused gate candidates -> exact sequential-tau scan) ---- */
/* tails[j][q][b][r] = C[j][d'+64b+4q+r], zero padded; nb = ceil((d-d')/64) */
int skm_build_tails(const float* centroids, long long ldc, int k, int d, int d_prime, float* tails, void* stream);
/* thr[i] = fl(tau[i] * f0) (inf when sentinel); with kap > 0 the emission threshold of the tensor-core
 * gate instead: every candidate whose exact distance may pass fl(tau * f0) is kept,
 * thr[i] >= (fl(tau f0) + kap (xsq[i] + *ysq_max)) / (1 - kap). */
int skm_gate_threshold(const float* tau, int n, float f0, int sentinel, float* thr, const float* xsq,
                       const float* ysq_max, float kap, void* stream);
typedef struct skm_scan_params {
  const int* cand; const int* cand_cnt; int cap;  /* list mode: [rows][cap] {index, float bits} */
  const float* dense; long long ld_dense; const int* dense_row; int k;       /* dense mode */
  const int* rows; int n_rows; long long row0;  /* batch-local rows to scan (NULL = 0..n_rows-1) */
  const int* row_map;                          /* optional global row of each batch-local row */
  void* work;                                  /* device u32 scratch: dynamic row-queue counter */
  const float* x; long long ldx;
  const float* tails; int nb; int d_prime;
  const float* theta; const int* block_dims;   /* nb+1 factors, nb block widths */
  float* tau; int* assign;                     /* global rows (row0 + local) */
  unsigned long long* counters;                /* += {survivors, dims touched, changed} */
  int dense_mode;
  unsigned long long* counters_ext;            /* optional diagnostics: += {block sums computed, warp waves,
                                                  -, candidates re-evaluated with the exact chain} */
  unsigned long long* prune_hist;              /* optional diagnostics: survivors by prune block */
  /* tensor-core candidate distances (kap > 0): the reference's value lies within
   * kap * (xsq[row] + *ysq_max + p) of p; unsettled decisions and possible new bests recompute it
   * with the exact chain over the d' front columns of x and cent (flavour / q as skm_chain_gemm) */
  float kap; const float* xsq; const float* ysq; const float* ysq_max;
  const float* cent; long long ldc; int chain_flavour; int chain_q;
  /* grouped rows (hierarchical fine phase): with group_counters, the counters of row r go to
   * group_counters[3 * row_group[r] + {0, 1, 2}] (global row r) instead of counters */
  const int* row_group; unsigned long long* group_counters;
  /* flat = 1 (list mode, kap > 0): a first pass resolves every row whose threshold changes only at
   * its own previous centroid (flatscan.cuh); the rest (their batch-local indices appended to
   * fb_rows, count in *fb_count -- both device workspace, fb_rows >= n_rows entries) are then
   * scanned by the exact kernel.  Same outputs as flat = 0. */
  int flat; int* fb_rows; unsigned int* fb_count;
  /* deferred certified entries (exact_work_stats = false, list mode, flat = 0): rows with
   * skip_cert[i] != 0 (skm_defer_cert_flags) leave their CAND_CERT0 entries out of the scan and
   * record each tau improvement {centroid, tau bits} in imp[i * 32 + t] (count imp_cnt[i]);
   * skm_deferred_cert_count then settles those entries' survivor decisions.  Batch-local i. */
  const int* skip_cert; int* imp; int* imp_cnt;
} skm_scan_params;
/* nb <= 104: 4-warp CTAs (flat pass available); 104 < nb <= 432 (d - d' <= 27648): one-warp CTAs
 * with the same results, flat ignored; larger nb returns SKM_E_ARG. */
int skm_pruned_scan(const skm_scan_params* p, void* stream);
/* skip[i] = 1 iff batch row i's candidate list holds certified entries and at most 32 others. */
int skm_defer_cert_flags(const int* cand, const int* cand_cnt, int cap, int n_rows, int* skip, void* stream);
/* After skm_pruned_scan with skip_cert: survivors (+ block_dims[0] dims each) of the deferred
 * entries, taken under the tau each would have met in the in-order walk (tau_seed: the rows'
 * tau before the scan, global rows); counters or group_counters as the scan's. */
int skm_deferred_cert_count(const skm_scan_params* p, const float* tau_seed, void* stream);

/* ---- exact top-k + ETR tally ------------------------------------------------------- */
/* k smallest of each row by (value, column) ascending, ties to the lower column (stable
 * argsort semantics); out_idx = column + col_offset.  k <= 2048. */
int skm_topk_rows(const float* d, long long ld, int rows, int cols, int k, int* out_idx, float* out_val,
                  long long out_ld, int col_offset, void* stream);
/* merge `shards` sorted per-shard top-k lists laid out [shard][row][k] */
int skm_topk_merge(const int* in_idx, const float* in_val, int shards, int k, int rows, int* out_idx, float* out_val,
                   void* stream);
/* hits[q] = #{g in gt[q][:top_k], row_lo <= g < row_hi : assign[g-row_lo] in probe[q][:nprobe]} */
int skm_etr_hits(const int* gt, int gt_ld, int top_k, const int* probe, int probe_ld, int nprobe, const int* assign,
                 long long row_lo, long long row_hi, int k, int nq, int* hits, void* stream);

/* probe_eval tally (evaluation.py:173-203): hits[q] as skm_etr_hits over rows 0..n-1
 * (assign[g] < 0: row in no cluster list) and explored[q] += sum_{c in probe[q]} sizes[c]. */
int skm_probe_tally(const int* gt, int gt_ld, int top_k, const int* probe, int probe_ld, int nprobe, const int* assign,
                    long long n, int k, int nq, const int* sizes, int* hits, long long* explored, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKM_B200_H */
