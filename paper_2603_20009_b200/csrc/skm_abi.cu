#include <atomic>
// extern "C" entry points of libskm_b200.so (declared in include/skm_b200.h).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/skm_b200.h"
#include "elementwise.cuh"
#include "gemm_tf32x3.cuh"
#include "update.cuh"
#include "scan.cuh"
#include "flatscan.cuh"
#include "sgemm_chain.cuh"
#include "topk.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return SKM_E_CUDA;
}
// every kernel launch of the library is counted (skm_kernel_launches: bench.py's gpu_launches)
static std::atomic<long long> g_kernel_launches{0};
#define SKM_COUNT_LAUNCH() g_kernel_launches.fetch_add(1, std::memory_order_relaxed)
#define SKM_LAUNCH_CHECK(where)                         \
  do {                                                  \
    cudaError_t _e = cudaGetLastError();                \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-device "first use" flag for function attributes (cudaFuncSetAttribute is per device): one
// bit per device ordinal in the caller's static mask.
inline bool first_use_on_device(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask & bit) return false;
  mask |= bit;
  return true;
}
inline int grid_for(long long work, int threads, int cap = 148 * 32) {
  long long g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  return static_cast<int>(std::min<long long>(g, cap));
}

// ---------------------------------------------------------------- TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// fp32 row-major [rows x ld], K extent `cols`, box = 32 x box_rows, 128B swizzle.
int make_tmap(CUtensorMap* m, const float* ptr, long long rows, long long cols, long long ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SKM_E_DRIVER, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 4) % 16) return fail(SKM_E_ARG, "TMA operand needs 16B-aligned base and ld%4==0");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld box=%d", (int)r, rows,
             cols, ld, box_rows);
    return fail(SKM_E_DRIVER, buf);
  }
  return SKM_OK;
}

template <int STAGES, int MODE, int BN>
int launch_gemm(const skm_gemm_params* p, cudaStream_t st) {
  using L = skm::GemmSmem<STAGES, BN>;
  CUtensorMap ta_hi, ta_lo, tb_hi, tb_lo;
  int rc;
  if ((rc = make_tmap(&ta_hi, p->a_hi, p->M, p->K, p->lda, skm::GEMM_BM))) return rc;
  if ((rc = make_tmap(&ta_lo, p->a_lo, p->M, p->K, p->lda, skm::GEMM_BM))) return rc;
  if ((rc = make_tmap(&tb_hi, p->b_hi, p->N, p->K, p->ldb, BN))) return rc;
  if ((rc = make_tmap(&tb_lo, p->b_lo, p->N, p->K, p->ldb, BN))) return rc;
  // GATE certification extension: columns [K, K + ext_k) of the same operands
  CUtensorMap te_a_hi = ta_hi, te_a_lo = ta_lo, te_b_hi = tb_hi, te_b_lo = tb_lo;
  const int ext_k = (MODE == skm::GEMM_GATE) ? p->ext_k : 0;
  if (ext_k > 0) {
    if (p->K % 4 || !p->xsq_ext || !p->ysq_ext || !p->thr1) return fail(SKM_E_ARG, "gemm: ext_k needs K%4==0 and ext norms/thr1");
    if ((rc = make_tmap(&te_a_hi, p->a_hi + p->K, p->M, ext_k, p->lda, skm::GEMM_BM))) return rc;
    if ((rc = make_tmap(&te_a_lo, p->a_lo + p->K, p->M, ext_k, p->lda, skm::GEMM_BM))) return rc;
    if ((rc = make_tmap(&te_b_hi, p->b_hi + p->K, p->N, ext_k, p->ldb, BN))) return rc;
    if ((rc = make_tmap(&te_b_lo, p->b_lo + p->K, p->N, ext_k, p->ldb, BN))) return rc;
  }
  auto kern = skm::gemm_tf32x3_kernel<STAGES, MODE, BN>;
  static unsigned long long attr_set_mask = 0;
  if (first_use_on_device(attr_set_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return cuda_fail(e, "gemm smem attribute");
  }
  skm::GemmArgs a{};
  a.M = p->M;
  a.N = p->N;
  a.K = p->K;
  const int n_tiles = (p->N + BN - 1) / BN;
  int split = std::max(1, std::min(p->n_split, n_tiles));
  a.tiles_per_cta = (n_tiles + split - 1) / split;
  split = (n_tiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
  a.n_split = split;
  a.out = p->out;
  a.ldo = p->ldo;
  a.xsq = p->xsq;
  a.ysq = p->ysq;
  a.top = reinterpret_cast<int4*>(p->top);
  a.thr = p->thr;
  a.cand = reinterpret_cast<decltype(a.cand)>(p->cand);
  a.cand_cnt = p->cand_cnt;
  a.cand_cap = p->cand_cap;
  a.row_offset = p->row_offset;
  a.ext_k = ext_k;
  a.xsq_ext = p->xsq_ext;
  a.ysq_ext = p->ysq_ext;
  a.thr1 = p->thr1;
  a.cert_eps = p->cert_eps;
  a.ext_hi_only = ext_k > 0 ? p->ext_hi_only : 0;
  a.row_crange = reinterpret_cast<const int2*>(p->row_crange);
  a.tile_nrange = reinterpret_cast<const int2*>(p->tile_nrange);
  if ((a.row_crange != nullptr) != (a.tile_nrange != nullptr))
    return fail(SKM_E_ARG, "gemm: row_crange and tile_nrange go together");
  if (a.tile_nrange && (MODE == skm::GEMM_STORE || MODE == skm::GEMM_DIST))
    return fail(SKM_E_ARG, "gemm: grouped columns need ARGMIN or GATE");
  if (a.tile_nrange) {  // one CTA per M tile, N range from the table
    split = 1;
    a.n_split = 1;
    a.tiles_per_cta = n_tiles;
  }
  {
    static int dbg = -1;
    if (dbg < 0) { const char* e = getenv("SKM_GEMM_DBG"); dbg = e ? atoi(e) : 0; }
    a.dbg = dbg;
  }
  if (MODE == skm::GEMM_ARGMIN && !p->top) return fail(SKM_E_ARG, "ARGMIN needs the top-2 record buffer");
  if (MODE == skm::GEMM_GATE && split > 1) return fail(SKM_E_ARG, "GATE requires n_split == 1");
  const long long blocks = static_cast<long long>((p->M + skm::GEMM_BM - 1) / skm::GEMM_BM) * split;
  if (blocks > 0x7fffffffLL) return fail(SKM_E_ARG, "gemm: grid too large");
  dim3 grid(static_cast<unsigned>(blocks));
  { kern<<<grid, skm::GEMM_THREADS, L::TOTAL, st>>>(ta_hi, ta_lo, tb_hi, tb_lo, te_a_hi, te_a_lo, te_b_hi, te_b_lo, a); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("gemm_tf32x3 launch");
  return SKM_OK;
}

}  // namespace

// ---------------------------------------------------------------- exact-chain GEMM
namespace {
template <int FL, int MODE, int ACC>
int launch_chain(const skm::ChainArgs& g, cudaStream_t st) {
  auto kern = skm::sgemm_chain_kernel<FL, MODE, ACC>;
  static unsigned long long attr_dev_mask = 0;
  if (first_use_on_device(attr_dev_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(skm::chain_smem_bytes()));
    if (e != cudaSuccess) return cuda_fail(e, "chain_gemm smem attribute");
  }
  dim3 grid((g.N + skm::CH_BN - 1) / skm::CH_BN, (g.M + skm::CH_BM - 1) / skm::CH_BM);
  if (grid.y > 65535) return fail(SKM_E_ARG, "chain_gemm: too many row tiles for one launch");
  { kern<<<grid, skm::CH_THREADS, skm::chain_smem_bytes(), st>>>(g); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("chain_gemm launch");
  return SKM_OK;
}

template <int FL, int MODE, int ACC>
int launch_chain_kn(const skm::ChainArgs& g, cudaStream_t st) {
  auto kern = skm::sgemm_chain_kn_kernel<FL, MODE, ACC>;
  static unsigned long long attr_dev_mask = 0;
  if (first_use_on_device(attr_dev_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(skm::chain_kn_smem_bytes()));
    if (e != cudaSuccess) return cuda_fail(e, "chain_gemm smem attribute");
  }
  dim3 grid((g.N + skm::CH_BN - 1) / skm::CH_BN, (g.M + skm::CH_BM - 1) / skm::CH_BM);
  if (grid.y > 65535) return fail(SKM_E_ARG, "chain_gemm: too many row tiles for one launch");
  { kern<<<grid, skm::CH_THREADS, skm::chain_kn_smem_bytes(), st>>>(g); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("chain_gemm_kn launch");
  return SKM_OK;
}

template <int FL>
int launch_chain_block(const skm::ChainArgs& g, bool dist, bool acc, bool kmajor, cudaStream_t st) {
  if (kmajor) {
    if (dist) return acc ? launch_chain_kn<FL, 1, 1>(g, st) : launch_chain_kn<FL, 1, 0>(g, st);
    return acc ? launch_chain_kn<FL, 0, 1>(g, st) : launch_chain_kn<FL, 0, 0>(g, st);
  }
  if (dist) return acc ? launch_chain<FL, 1, 1>(g, st) : launch_chain<FL, 1, 0>(g, st);
  return acc ? launch_chain<FL, 0, 1>(g, st) : launch_chain<FL, 0, 0>(g, st);
}
}  // namespace

// The blocked driver's association order as a sequence of launches: K block b of every output is
// a fresh chain added to the sum of blocks < b (stored in `out` between launches); the distance
// expansion runs in the last block's epilogue.
extern "C" int skm_chain_gemm(const skm_chain_params* p, void* stream) {
  if (!p || p->M < 0 || p->N < 0 || p->K < 0) return fail(SKM_E_ARG, "chain_gemm: bad shape");
  if ((long long)p->M * p->N == 0) return SKM_OK;
  if (p->mode == 1 && (!p->xsq || !p->ysq)) return fail(SKM_E_ARG, "chain_gemm: distance mode needs xsq/ysq");
  if (p->b_kmajor && ((p->ldb & 3) != 0 || (reinterpret_cast<uintptr_t>(p->b) & 15) != 0))
    return fail(SKM_E_ARG, "chain_gemm: k-major b needs a 16-byte aligned b and ldb % 4 == 0");
  cudaStream_t st = as_stream(stream);
  const int rows_per = 65535 * skm::CH_BM;  // grid.y limit: consecutive launches over row ranges
  for (int r0 = 0; r0 < p->M; r0 += rows_per) {
    int k0 = 0;
    do {
      const int k1 = skm::chain_next_boundary(k0, p->K, p->flavour == 0 ? p->q : 0);
      skm::ChainArgs h{};
      h.M = std::min(rows_per, p->M - r0);
      h.N = p->N;
      h.K = k1 - k0;
      h.a = p->a + (long long)r0 * p->lda + k0;
      h.lda = p->lda;
      h.b = p->b_kmajor ? p->b + (long long)k0 * p->ldb : p->b + k0;
      h.ldb = p->ldb;
      h.out = p->out + (long long)r0 * p->ldo;
      h.ldo = p->ldo;
      h.xsq = p->xsq ? p->xsq + r0 : nullptr;
      h.ysq = p->ysq;
      const bool last = k1 >= p->K;
      const bool dist = last && p->mode == 1;
      const bool acc = k0 > 0;
      int rc = p->flavour == 0 ? launch_chain_block<0>(h, dist, acc, p->b_kmajor != 0, st)
                               : launch_chain_block<1>(h, dist, acc, p->b_kmajor != 0, st);
      if (rc) return rc;
      k0 = k1;
    } while (k0 < p->K);
  }
  return SKM_OK;
}

template <int FL>
static int launch_chain_topk(const skm::ChainTopkArgs& g, cudaStream_t st) {
  auto kern = skm::sgemm_chain_topk_kernel<FL>;
  static unsigned long long attr_dev_mask = 0;
  if (first_use_on_device(attr_dev_mask)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(skm::chain_topk_smem_bytes()));
    if (e != cudaSuccess) return cuda_fail(e, "chain_topk smem attribute");
  }
  dim3 grid(static_cast<unsigned>(g.n_tiles), static_cast<unsigned>((g.N + skm::CH_BN - 1) / skm::CH_BN));
  { kern<<<grid, skm::CH_THREADS, skm::chain_topk_smem_bytes(), st>>>(g); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("chain_topk launch");
  return SKM_OK;
}

extern "C" int skm_chain_topk_tiles(const float* rows, long long ldr, const float* queries_t, long long ldq, int n,
                                    int nq, int K, int flavour, int q, const float* row_sq, const float* q_sq,
                                    int k_top, float* out_v, int* out_i, int col_offset, void* stream) {
  if (n <= 0 || nq <= 0) return SKM_OK;
  if (K <= 0 || k_top < 1 || k_top > skm::TOPK_TILE_MAX) return fail(SKM_E_ARG, "chain_topk: bad K or k_top (1..32)");
  if ((nq + skm::CH_BN - 1) / skm::CH_BN > 65535) return fail(SKM_E_ARG, "chain_topk: too many query tiles");
  if ((ldq & 3) != 0 || (reinterpret_cast<uintptr_t>(queries_t) & 15) != 0)
    return fail(SKM_E_ARG, "chain_topk: k-major queries need 16-byte alignment and ld % 4 == 0");
  skm::ChainTopkArgs g{};
  g.a = rows; g.lda = ldr; g.b = queries_t; g.ldb = ldq;
  g.M = n; g.N = nq; g.K = K; g.q = q;
  g.xsq = row_sq; g.ysq = q_sq;
  g.k_top = k_top;
  g.n_tiles = (n + skm::CH_BM - 1) / skm::CH_BM;
  g.out_v = out_v; g.out_i = out_i; g.col_offset = col_offset;
  cudaStream_t st = as_stream(stream);
  return flavour == 0 ? launch_chain_topk<0>(g, st) : launch_chain_topk<1>(g, st);
}

extern "C" {

const char* skm_last_error(void) { return g_err.c_str(); }
long long skm_kernel_launches(void) { return g_kernel_launches.load(std::memory_order_relaxed); }
int skm_abi_version(void) { return 1; }

int skm_split_hilo(const float* x, long long ldx, int rows, int cols, float* hi, float* lo, long long ldo,
                   void* stream) {
  if (rows <= 0) return SKM_OK;
  if (cols > ldo) return fail(SKM_E_ARG, "split_hilo: cols > ldo");
  if ((ldx & 3) == 0 && (ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(hi) & 15) == 0 && (reinterpret_cast<uintptr_t>(lo) & 15) == 0) {
    const long long ldo4 = ldo / 4;
    dim3 grid(static_cast<unsigned>((ldo4 + 127) / 128), static_cast<unsigned>(std::min(rows, 16384)));
    { skm::split_hilo_vec_kernel<<<grid, 128, 0, as_stream(stream)>>>(reinterpret_cast<const float4*>(x), ldx / 4, rows,
                                                                     cols, reinterpret_cast<float4*>(hi),
                                                                     reinterpret_cast<float4*>(lo), ldo4); SKM_COUNT_LAUNCH(); }
    SKM_LAUNCH_CHECK("split_hilo");
    return SKM_OK;
  }
  { skm::split_hilo_kernel<<<grid_for((long long)rows * ldo, 256), 256, 0, as_stream(stream)>>>(x, ldx, rows, cols, hi,
                                                                                             lo, ldo); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("split_hilo");
  return SKM_OK;
}

int skm_row_sq_norms(const float* x, long long ldx, int rows, int dims, float* out, void* stream) {
  if (rows <= 0) return SKM_OK;
  { skm::row_sq_norms_einsum_kernel<<<grid_for(rows, 128, 148 * 64), 128, 0, as_stream(stream)>>>(x, ldx, rows, dims,
                                                                                                out); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("row_sq_norms");
  return SKM_OK;
}

int skm_gather_rows(const float* in, long long ldi, const long long* idx, int rows, int cols, float* out,
                    long long ldo, void* stream) {
  if (rows <= 0) return SKM_OK;
  { skm::gather_rows_kernel<<<grid_for((long long)rows * cols, 256), 256, 0, as_stream(stream)>>>(in, ldi, idx, rows,
                                                                                              cols, out, ldo); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("gather_rows");
  return SKM_OK;
}

int skm_gather_front(const float* hi, const float* lo, long long ldi, const int* idx, int rows, int cols, float* ohi,
                     float* olo, long long ldo, const float* xsq, const float* thr, float* oxsq, float* othr,
                     const float* xsq_ext, const float* thr1, float* oxsq_ext, float* othr1, void* stream) {
  if (rows <= 0) return SKM_OK;
  if (cols > ldo || cols > ldi) return fail(SKM_E_ARG, "gather_front: cols exceeds a stride");
  { skm::gather_front_kernel<<<grid_for((long long)rows * 32, 256), 256, 0, as_stream(stream)>>>(
      hi, lo, ldi, idx, rows, cols, ohi, olo, ldo, xsq, thr, oxsq, othr, xsq_ext, oxsq_ext, thr1, othr1); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("gather_front");
  return SKM_OK;
}

int skm_ingest_records(const void* raw, long long rows, int d, int rec_words, int header_words, long long row0,
                       float* out, long long ldo, unsigned long long* bad_dim, unsigned long long* bad_val,
                       void* stream) {
  if (rows <= 0) return SKM_OK;
  if (d <= 0 || ldo < d || rec_words < d + header_words) return fail(SKM_E_ARG, "ingest_records: bad shape");
  { skm::ingest_records_kernel<<<grid_for(rows * 32, 256), 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const uint32_t*>(raw), rows, d, rec_words, header_words, row0, out, ldo, bad_dim, bad_val); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("ingest_records");
  return SKM_OK;
}

long long skm_wcss_workspace_bytes() { return 8LL * 1024; }

int skm_wcss(const float* x, long long ldx, const float* centroids, long long ldc, const int* assign, long long n,
             int d, double* out, void* workspace, void* stream) {
  if (n <= 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), as_stream(stream));
    return e == cudaSuccess ? SKM_OK : cuda_fail(e, "wcss zero");
  }
  const int parts = static_cast<int>(std::min<long long>(1024, (n + 7) / 8));
  double* part = reinterpret_cast<double*>(workspace);
  { skm::wcss_partial_kernel<<<parts, skm::WCSS_THREADS, 0, as_stream(stream)>>>(x, ldx, centroids, ldc, assign, n, d,
                                                                               part); SKM_COUNT_LAUNCH(); }
  { skm::wcss_final_kernel<<<1, 32, 0, as_stream(stream)>>>(part, parts, out); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("wcss");
  return SKM_OK;
}

int skm_first_nonfinite(const float* x, long long ldx, long long rows, int cols, unsigned long long* first,
                        void* stream) {
  cudaError_t e = cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "first_nonfinite reset");
  if (rows <= 0 || cols <= 0) return SKM_OK;
  { skm::first_nonfinite_kernel<<<grid_for(rows * 32, 256), 256, 0, as_stream(stream)>>>(x, ldx, rows, cols, first); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("first_nonfinite");
  return SKM_OK;
}

int skm_gather_rows_i32(const float* in, long long ldi, const int* idx, int rows, int cols, float* out,
                        long long ldo, void* stream) {
  if (rows <= 0) return SKM_OK;
  { skm::gather_rows_i32_kernel<<<grid_for((long long)rows * cols, 256), 256, 0, as_stream(stream)>>>(in, ldi, idx, rows,
                                                                                                  cols, out, ldo); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("gather_rows_i32");
  return SKM_OK;
}

int skm_fill_f32(float* p, long long n, float v, void* stream) {
  if (n <= 0) return SKM_OK;
  { skm::fill_f32_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(p, n, v); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("fill_f32");
  return SKM_OK;
}

int skm_copy_i32(const int* src, int* dst, int n, void* stream) {
  if (n <= 0) return SKM_OK;
  { skm::copy_i32_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(src, dst, n); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("copy_i32");
  return SKM_OK;
}

int skm_seed_thresholds(const float* x, long long ldx, const float* centroids, long long ldc, const int* assign,
                        int n, int d, float* out, void* stream) {
  if (n <= 0) return SKM_OK;
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(centroids)) & 15) == 0 &&
                       ldx % 4 == 0 && ldc % 4 == 0;
  if (aligned) {
    static unsigned long long set_mask = 0;
    if (first_use_on_device(set_mask)) {
      cudaError_t e = cudaFuncSetAttribute(skm::seed_thresholds_async_kernel<0>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, skm::SEEDA_SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "seed_thresholds smem attribute");
    }
    { skm::seed_thresholds_async_kernel<0><<<(n + skm::SEED_ROWS - 1) / skm::SEED_ROWS, skm::SEED_ROWS, skm::SEEDA_SMEM,
                                        as_stream(stream)>>>(x, ldx, centroids, ldc, assign, n, d, out); SKM_COUNT_LAUNCH(); }
  } else {
    { skm::seed_thresholds_kernel<<<(n + skm::SEED_ROWS - 1) / skm::SEED_ROWS, skm::SEED_ROWS, 0, as_stream(stream)>>>(
        x, ldx, centroids, ldc, assign, n, d, out); SKM_COUNT_LAUNCH(); }
  }
  SKM_LAUNCH_CHECK("seed_thresholds");
  return SKM_OK;
}

int skm_scan_bank(const float* partial_dists, int n, int kb, const float* x, long long ldx, const float* tail,
                  const long long* block_offsets, const int* block_dims, int n_blocks, const float* theta_factors,
                  int d_prime, int bank_offset, float* tau, int* assign, int sentinel,
                  unsigned long long* counters, void* stream) {
  if (n <= 0) return SKM_OK;
  { skm::scan_bank_pdx_kernel<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(
      partial_dists, n, kb, x, ldx, tail, block_offsets, block_dims, n_blocks, theta_factors, d_prime, bank_offset,
      tau, assign, sentinel, counters); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("scan_bank");
  return SKM_OK;
}

int skm_portable_matmul(const float* a, long long lda, const float* b, long long ldb, int n, int m, int dims,
                        float* out, long long ldo, void* stream) {
  if ((long long)n * m <= 0) return SKM_OK;
  { skm::portable_matmul_kernel<<<(int)(((long long)n * m + 255) / 256), 256, 0, as_stream(stream)>>>(
      a, lda, b, ldb, n, m, dims, out, ldo); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("portable_matmul");
  return SKM_OK;
}

// ---------------------------------------------------------------- sort / update
static int radix_blocks(int n) { return (n + skm::RADIX_TILE - 1) / skm::RADIX_TILE; }
static long long align256(long long b) { return (b + 255) & ~255LL; }

long long skm_update_workspace_bytes(int n, int k) {
  const long long nb = radix_blocks(std::max(n, 1));
  return 3 * align256(4LL * n) + align256(4LL * 256 * nb) + align256(16) + align256(4LL * std::max(k, 1));
}

int skm_cluster_sort(const int* assign, int n, int k, int* order, int* counts, int* offsets, void* workspace,
                     long long workspace_bytes, void* stream) {
  if (n < 0 || k <= 0) return fail(SKM_E_ARG, "cluster_sort: bad n/k");
  if (workspace_bytes < skm_update_workspace_bytes(n, k)) return fail(SKM_E_WORKSPACE, "cluster_sort: workspace too small");
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int) * k, st);
  if (e != cudaSuccess) return cuda_fail(e, "cluster_sort memset");
  if (n == 0) {
    e = cudaMemsetAsync(offsets, 0, sizeof(int) * k, st);
    return e == cudaSuccess ? SKM_OK : cuda_fail(e, "cluster_sort memset");
  }
  char* ws = static_cast<char*>(workspace);
  int* keys_a = reinterpret_cast<int*>(ws);
  int* keys_b = reinterpret_cast<int*>(ws + align256(4LL * n));
  int* vals_a = reinterpret_cast<int*>(ws + 2 * align256(4LL * n));
  const int nb = radix_blocks(n);
  int* hist = reinterpret_cast<int*>(ws + 3 * align256(4LL * n));
  int* total = reinterpret_cast<int*>(ws + 3 * align256(4LL * n) + align256(4LL * 256 * nb));
  int bits = 1;
  while ((1LL << bits) < k) ++bits;
  const int passes = (bits + 7) / 8;
  // ping-pong so that the final values land in `order`
  int* vin = vals_a;
  int* kin = keys_a;
  int* vout = (passes % 2 == 1) ? order : vals_a;
  e = cudaMemcpyAsync(keys_a, assign, 4LL * n, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "cluster_sort copy");
  // values start as the identity permutation
  int* v0 = (passes % 2 == 1) ? vals_a : order;
  { skm::iota_kernel<<<grid_for(n, 256), 256, 0, st>>>(v0, n); SKM_COUNT_LAUNCH(); }
  vin = v0;
  int* kbuf[2] = {keys_a, keys_b};
  int* vbuf[2] = {v0, (v0 == order) ? vals_a : order};
  for (int p = 0; p < passes; ++p) {
    kin = kbuf[p & 1];
    int* kout = kbuf[(p + 1) & 1];
    vin = vbuf[p & 1];
    vout = vbuf[(p + 1) & 1];
    { skm::radix_hist_kernel<<<nb, skm::RADIX_THREADS, 0, st>>>(kin, n, 8 * p, hist, nb); SKM_COUNT_LAUNCH(); }
    { skm::exclusive_scan_kernel<<<1, 1024, 0, st>>>(hist, 256 * nb, total); SKM_COUNT_LAUNCH(); }
    { skm::radix_scatter_kernel<<<nb, skm::RADIX_THREADS, 0, st>>>(kin, vin, kout, vout, n, 8 * p, hist, nb); SKM_COUNT_LAUNCH(); }
  }
  SKM_LAUNCH_CHECK("cluster_sort radix");
  if (vout != order) return fail(SKM_E_ARG, "cluster_sort: internal ping-pong error");
  { skm::count_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(assign, n, counts); SKM_COUNT_LAUNCH(); }
  e = cudaMemcpyAsync(offsets, counts, sizeof(int) * k, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "cluster_sort copy");
  { skm::exclusive_scan_kernel<<<1, 1024, 0, st>>>(offsets, k, total); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("cluster_sort counts");
  return SKM_OK;
}

int skm_cluster_sums(const float* x, long long ldx, const int* order, const int* offsets, const int* counts, int k,
                     int d, double* sums, int accumulate, float* centroids, long long ldc, int mode, void* stream) {
  if (k <= 0 || d <= 0) return SKM_OK;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && ldx % 4 == 0) {
    const int groups = (d + 3) / 4;
    const int threads = std::min(768, (groups + 31) / 32 * 32);  // ring <= 768 x 16 x 16 B = 192 KB
    static unsigned long long set_mask = 0;
    if (first_use_on_device(set_mask)) {
      cudaError_t e = cudaFuncSetAttribute(skm::ordered_cluster_sums_vec_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, skm::SUMV_RING * 768 * 16);
      if (e != cudaSuccess) return cuda_fail(e, "cluster_sums smem attribute");
    }
    { skm::ordered_cluster_sums_vec_kernel<<<k, threads, skm::SUMV_RING * threads * 16, as_stream(stream)>>>(
        x, ldx, order, offsets, counts, d, sums, accumulate, centroids, ldc, mode); SKM_COUNT_LAUNCH(); }
  } else {
    dim3 grid(k, (d + skm::SUM_THREADS - 1) / skm::SUM_THREADS);
    { skm::ordered_cluster_sums_kernel<<<grid, skm::SUM_THREADS, 0, as_stream(stream)>>>(
        x, ldx, order, offsets, counts, d, sums, accumulate, centroids, ldc, mode); SKM_COUNT_LAUNCH(); }
  }
  SKM_LAUNCH_CHECK("cluster_sums");
  return SKM_OK;
}

int skm_finalize_centroids(const double* sums, const long long* counts, int k, int d, float* centroids,
                           long long ldc, void* stream) {
  if ((long long)k * d <= 0) return SKM_OK;
  { skm::finalize_centroids_kernel<<<grid_for((long long)k * d, 256), 256, 0, as_stream(stream)>>>(sums, counts, k, d,
                                                                                               centroids, ldc); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("finalize_centroids");
  return SKM_OK;
}

int skm_counts_to_i64(const int* c32, long long* c64, int k, int accumulate, void* stream) {
  if (k <= 0) return SKM_OK;
  { skm::counts_to_i64_kernel<<<grid_for(k, 256), 256, 0, as_stream(stream)>>>(c32, c64, k, accumulate); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("counts_to_i64");
  return SKM_OK;
}

int skm_accumulate_centroid_sums(const float* x, long long ldx, const int* assign, int n, int d, int k,
                                 double* sums, long long* counts, void* workspace, long long workspace_bytes,
                                 void* stream) {
  // workspace layout: [sort workspace][order n][counts k][offsets k]
  const long long sort_ws = skm_update_workspace_bytes(n, k);
  const long long need = sort_ws + align256(4LL * std::max(n, 1)) + 2 * align256(4LL * k);
  if (workspace_bytes < need) return fail(SKM_E_WORKSPACE, "accumulate_centroid_sums: workspace too small");
  char* ws = static_cast<char*>(workspace);
  int* order = reinterpret_cast<int*>(ws + sort_ws);
  int* c32 = reinterpret_cast<int*>(ws + sort_ws + align256(4LL * std::max(n, 1)));
  int* off = reinterpret_cast<int*>(ws + sort_ws + align256(4LL * std::max(n, 1)) + align256(4LL * k));
  int rc = skm_cluster_sort(assign, n, k, order, c32, off, ws, sort_ws, stream);
  if (rc) return rc;
  rc = skm_cluster_sums(x, ldx, order, off, c32, k, d, sums, 1, nullptr, 0, 1, stream);
  if (rc) return rc;
  return skm_counts_to_i64(c32, counts, k, 1, stream);
}

int skm_apply_splits(float* centroids, long long ldc, int d, const int* empties, const int* donors, int n_splits,
                     float eps, void* stream) {
  if (n_splits <= 0) return SKM_OK;
  { skm::apply_splits_kernel<<<1, 256, 0, as_stream(stream)>>>(centroids, ldc, d, empties, donors, n_splits, eps); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("apply_splits");
  return SKM_OK;
}

long long skm_stats_workspace_bytes(int n) {
  const long long chunks = (std::max(n, 1) + skm::NP_SUM_BUF - 1) / skm::NP_SUM_BUF;
  return 2 * align256(16LL * 1024) + align256(8 * chunks);
}

int skm_tau_chunk_sums(const float* tau, long long n, double* out, void* stream) {
  if (n <= 0) return SKM_OK;
  const long long chunks = (n + skm::NP_SUM_BUF - 1) / skm::NP_SUM_BUF;
  { skm::np_sum_chunks_kernel<<<static_cast<unsigned>(chunks), 64, 0, as_stream(stream)>>>(tau, n, out); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("tau_chunk_sums");
  return SKM_OK;
}

int skm_assign_stats(const float* tau, const int* assign, const int* prev, int n, double* out_sum,
                     unsigned long long* out_changed, void* workspace, long long workspace_bytes, void* stream) {
  if (workspace_bytes < skm_stats_workspace_bytes(n)) return fail(SKM_E_WORKSPACE, "assign_stats: workspace too small");
  const int parts = std::max(1, std::min(1024, (n + 4095) / 4096));
  const int chunks = (n + skm::NP_SUM_BUF - 1) / skm::NP_SUM_BUF;
  char* ws = static_cast<char*>(workspace);
  double* ps = reinterpret_cast<double*>(ws);
  unsigned long long* pc = reinterpret_cast<unsigned long long*>(ws + align256(16LL * 1024));
  double* cs = reinterpret_cast<double*>(ws + 2 * align256(16LL * 1024));
  cudaStream_t st = as_stream(stream);
  { skm::assign_stats_partial_kernel<<<parts, skm::STAT_THREADS, 0, st>>>(tau, assign, prev, n, ps, pc); SKM_COUNT_LAUNCH(); }
  if (chunks > 0) { skm::np_sum_chunks_kernel<<<chunks, 64, 0, st>>>(tau, n, cs); SKM_COUNT_LAUNCH(); }
  { skm::assign_stats_final_kernel<<<1, 32, 0, st>>>(cs, chunks, pc, parts, out_sum, out_changed); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("assign_stats");
  return SKM_OK;
}

// ---------------------------------------------------------------- GEMM
int skm_gemm_tf32x3(const skm_gemm_params* p, void* stream) {
  if (!p) return fail(SKM_E_ARG, "gemm: null params");
  if (p->M <= 0 || p->N <= 0) return SKM_OK;
  if (p->K <= 0) return fail(SKM_E_ARG, "gemm: K must be > 0");
  cudaStream_t st = as_stream(stream);
  switch (p->mode) {
    case SKM_GEMM_STORE: return launch_gemm<2, skm::GEMM_STORE, skm::GEMM_BN>(p, st);
    case SKM_GEMM_DIST: return launch_gemm<2, skm::GEMM_DIST, skm::GEMM_BN>(p, st);
    case SKM_GEMM_ARGMIN: return launch_gemm<2, skm::GEMM_ARGMIN, skm::GEMM_BN>(p, st);
    case SKM_GEMM_GATE: return launch_gemm<SKM_GATE_STAGES, skm::GEMM_GATE, skm::GEMM_BN_GATE>(p, st);
    default: return fail(SKM_E_ARG, "gemm: unknown mode");
  }
}

int skm_argmin_merge(const int* top, int n_split, int n, const float* xsq, const float* ysq_max, float kap,
                     int* assign, float* tau, int* amb_rows, unsigned int* amb_count, void* stream) {
  if (n <= 0) return SKM_OK;
  { skm::argmin_merge_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(
      reinterpret_cast<const int4*>(top), n_split, n, xsq, ysq_max, kap, assign, tau, amb_rows, amb_count); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("argmin_merge");
  return SKM_OK;
}

int skm_dense_argmin(const float* dist, long long ld, int rows, int cols, const int* row_ids, int* assign,
                     float* tau, void* stream) {
  if (rows <= 0) return SKM_OK;
  { skm::dense_argmin_kernel<<<grid_for((long long)rows * 32, 256), 256, 0, as_stream(stream)>>>(dist, ld, rows, cols,
                                                                                             row_ids, assign, tau); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("dense_argmin");
  return SKM_OK;
}

int skm_argmin_candidates(const int* rows, int n_rows, const float* tau, const float* xsq, const float* ysq_max,
                          float kap, float* thr, float* xs_out, void* stream) {
  if (n_rows <= 0) return SKM_OK;
  { skm::argmin_cand_threshold_kernel<<<(n_rows + 255) / 256, 256, 0, as_stream(stream)>>>(rows, n_rows, tau, xsq,
                                                                                      ysq_max, kap, thr, xs_out); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("argmin_candidates");
  return SKM_OK;
}

int skm_cand_exact_argmin(const int* rows, int n_rows, const int* cand, const int* cand_cnt, int cap, const float* x,
                          long long ldx, const float* centroids, long long ldc, int d, const float* xsq,
                          const float* ysq, int flavour, int q, int* assign, float* tau, void* stream) {
  if (n_rows <= 0) return SKM_OK;
  { skm::cand_exact_argmin_kernel<<<grid_for((long long)n_rows * 32, 256), 256, 0, as_stream(stream)>>>(
      rows, n_rows, reinterpret_cast<const int2*>(cand), cand_cnt, cap, x, ldx, centroids, ldc, d, xsq, ysq, flavour,
      q, assign, tau); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("cand_exact_argmin");
  return SKM_OK;
}

int skm_max_f32(const float* v, int n, float* out, void* stream) {
  { skm::max_f32_kernel<<<1, 1024, 0, as_stream(stream)>>>(v, n, out); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("max_f32");
  return SKM_OK;
}

int skm_exact_pair_dist(const float* x, long long ldx, const float* centroids, long long ldc, const int* assign,
                        int n, int d, const float* xsq, const float* ysq, int flavour, int q, float* out,
                        void* stream) {
  if (n <= 0) return SKM_OK;
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(centroids)) & 15) == 0 &&
                       ldx % 4 == 0 && ldc % 4 == 0;
  if (!aligned) return fail(SKM_E_ARG, "exact_pair_dist: needs 16-byte aligned rows");
  auto k1 = skm::seed_thresholds_async_kernel<1>;
  auto k2 = skm::seed_thresholds_async_kernel<2>;
  static unsigned long long set_dev_mask = 0;
  if (first_use_on_device(set_dev_mask)) {
    cudaError_t e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, skm::SEEDA_SMEM);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, skm::SEEDA_SMEM);
    if (e != cudaSuccess) return cuda_fail(e, "exact_pair_dist smem attribute");
  }
  const int grid = (n + skm::SEED_ROWS - 1) / skm::SEED_ROWS;
  if (flavour == 0)
    { k1<<<grid, skm::SEED_ROWS, skm::SEEDA_SMEM, as_stream(stream)>>>(x, ldx, centroids, ldc, assign, n, d, out, xsq,
                                                                     ysq, q); SKM_COUNT_LAUNCH(); }
  else
    { k2<<<grid, skm::SEED_ROWS, skm::SEEDA_SMEM, as_stream(stream)>>>(x, ldx, centroids, ldc, assign, n, d, out, xsq,
                                                                     ysq, 0); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("exact_pair_dist");
  return SKM_OK;
}


// ---------------------------------------------------------------- pruning scan
int skm_build_tails(const float* centroids, long long ldc, int k, int d, int d_prime, float* tails, void* stream) {
  const int nb = (d - d_prime + 63) / 64;
  if (k <= 0 || nb <= 0) return SKM_OK;
  { skm::build_tails_kernel<<<grid_for((long long)k * 64 * nb, 256), 256, 0, as_stream(stream)>>>(centroids, ldc, k, d,
                                                                                              d_prime, nb, tails); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("build_tails");
  return SKM_OK;
}

int skm_gate_threshold(const float* tau, int n, float f0, int sentinel, float* thr, const float* xsq,
                       const float* ysq_max, float kap, void* stream) {
  if (n <= 0) return SKM_OK;
  if (kap > 0.0f && (!xsq || !ysq_max)) return fail(SKM_E_ARG, "gate_threshold: kap needs xsq and ysq_max");
  { skm::gate_threshold_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(tau, n, f0, sentinel, thr, xsq, ysq_max,
                                                                             kap); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("gate_threshold");
  return SKM_OK;
}

int skm_defer_cert_flags(const int* cand, const int* cand_cnt, int cap, int n_rows, int* skip, void* stream) {
  if (n_rows <= 0) return SKM_OK;
  if (!cand || !cand_cnt || !skip || cap <= 0) return fail(SKM_E_ARG, "defer_cert_flags: null argument");
  { skm::defer_cert_flags_kernel<<<(n_rows + 7) / 8, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const int2*>(cand), cand_cnt, cap, n_rows, skip); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("defer_cert_flags");
  return SKM_OK;
}

int skm_deferred_cert_count(const skm_scan_params* p, const float* tau_seed, void* stream) {
  if (!p || !tau_seed) return fail(SKM_E_ARG, "deferred_cert_count: null argument");
  if (p->n_rows <= 0) return SKM_OK;
  if (!p->skip_cert || !p->imp || !p->imp_cnt || !p->cand || !p->cand_cnt || p->kap <= 0.0f || !p->xsq ||
      !p->ysq || !p->ysq_max || !p->cent || !p->theta || !p->block_dims)
    return fail(SKM_E_ARG, "deferred_cert_count: needs the scan's list, skip/imp records and exact-chain inputs");
  if ((p->row_group != nullptr) != (p->group_counters != nullptr) || (!p->group_counters && !p->counters))
    return fail(SKM_E_ARG, "deferred_cert_count: counters or row_group + group_counters");
  skm::ScanArgs a{};
  a.cand = reinterpret_cast<decltype(a.cand)>(p->cand);
  a.cand_cnt = p->cand_cnt;
  a.cap = p->cap;
  a.n_rows = p->n_rows;
  a.row0 = p->row0;
  a.row_map = p->row_map;
  a.x = p->x;
  a.ldx = p->ldx;
  a.d_prime = p->d_prime;
  a.theta = p->theta;
  a.block_dims = p->block_dims;
  a.counters = p->counters;
  a.kap = p->kap;
  a.xsq = p->xsq;
  a.ysq = p->ysq;
  a.ysq_max = p->ysq_max;
  a.cent = p->cent;
  a.ldc = p->ldc;
  a.chain_flavour = p->chain_flavour;
  a.chain_q = p->chain_q;
  a.row_group = p->row_group;
  a.group_counters = p->group_counters;
  a.skip_cert = p->skip_cert;
  a.imp = reinterpret_cast<int2*>(p->imp);
  a.imp_cnt = p->imp_cnt;
  { skm::deferred_cert_count_kernel<<<(p->n_rows + 7) / 8, 256, 0, as_stream(stream)>>>(a, tau_seed);
    SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("deferred_cert_count");
  return SKM_OK;
}

// One warp per CTA: the scan for tails of SCAN_NB_MAX < nb <= SCAN_NB_MAX_WIDE blocks (d - d' up
// to 27648).  Same per-row algorithm and results as the 4-warp kernel; exact re-evaluations read
// the fronts from global memory when they do not fit beside the tail staging.
static int launch_pruned_scan_wide(skm::ScanArgs a, const skm_scan_params* p, void* stream) {
  static int dyn_wide = -1;
  if (dyn_wide < 0) {
    int dv = 0, optin = 0;
    cudaGetDevice(&dv);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dv);
    cudaFuncAttributes fa{}, fb{};
    cudaFuncGetAttributes(&fa, skm::pruned_scan_kernel<false, 1>);
    cudaFuncGetAttributes(&fb, skm::pruned_scan_kernel<true, 1>);
    dyn_wide = optin - static_cast<int>(std::max(fa.sharedSizeBytes, fb.sharedSizeBytes));
  }
  if (skm::scan_dyn_smem(p->nb, 0, false, 1) > static_cast<size_t>(dyn_wide))
    return fail(SKM_E_ARG, "pruned_scan: tail too long for the shared-memory staging");
  a.ex_stage = (a.kap > 0.0f && skm::scan_dyn_smem(p->nb, p->d_prime, true, 1) <= static_cast<size_t>(dyn_wide)) ? 1 : 0;
  const size_t smem = skm::scan_dyn_smem(p->nb, p->d_prime, a.ex_stage != 0, 1);
  cudaStream_t st = as_stream(stream);
  static unsigned long long set_mask_d = 0, set_mask_l = 0;
  if (first_use_on_device(set_mask_d))
    cudaFuncSetAttribute(skm::pruned_scan_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_wide);
  if (first_use_on_device(set_mask_l))
    cudaFuncSetAttribute(skm::pruned_scan_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_wide);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (p->dense_mode)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skm::pruned_scan_kernel<true, 1>, 32, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skm::pruned_scan_kernel<false, 1>, 32, smem);
  const int blocks = std::max(1, std::min(p->n_rows, sms * std::max(per_sm, 1)));
  if (p->dense_mode)
    { skm::pruned_scan_kernel<true, 1><<<blocks, 32, smem, st>>>(a); SKM_COUNT_LAUNCH(); }
  else
    { skm::pruned_scan_kernel<false, 1><<<blocks, 32, smem, st>>>(a); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("pruned_scan_wide");
  return SKM_OK;
}

int skm_pruned_scan(const skm_scan_params* p, void* stream) {
  if (!p) return fail(SKM_E_ARG, "pruned_scan: null params");
  if (p->n_rows <= 0) return SKM_OK;
  if (p->nb <= 0 || p->nb > skm::SCAN_NB_MAX_WIDE)
    return fail(SKM_E_ARG, "pruned_scan: tail block count out of range (d - d' > 27648)");
  skm::ScanArgs a{};
  a.cand = reinterpret_cast<decltype(a.cand)>(p->cand);
  a.cand_cnt = p->cand_cnt;
  a.cap = p->cap;
  a.dense = p->dense;
  a.ld_dense = p->ld_dense;
  a.dense_row = p->dense_row;
  a.k = p->k;
  a.rows = p->rows;
  a.n_rows = p->n_rows;
  a.row0 = p->row0;
  a.row_map = p->row_map;
  a.work = reinterpret_cast<unsigned int*>(p->work);
  if (!a.work) return fail(SKM_E_ARG, "pruned_scan: work counter required");
  {
    // one global row queue: concurrently running warps then scan neighbouring cluster-sorted
    // rows (per-SM queues over contiguous ranges measured 3x slower)
    cudaError_t e = cudaMemsetAsync(p->work, 0, sizeof(unsigned int), as_stream(stream));
    if (e != cudaSuccess) return cuda_fail(e, "pruned_scan work reset");
  }
  a.x = p->x;
  a.ldx = p->ldx;
  a.tails = reinterpret_cast<const float4*>(p->tails);
  a.nb = p->nb;
  a.d_prime = p->d_prime;
  a.theta = p->theta;
  a.block_dims = p->block_dims;
  a.tau = p->tau;
  a.assign = p->assign;
  a.counters = p->counters;
  a.counters_ext = p->counters_ext;
  a.prune_hist = p->prune_hist;
  a.kap = p->kap;
  a.xsq = p->xsq;
  a.ysq = p->ysq;
  a.ysq_max = p->ysq_max;
  a.cent = p->cent;
  a.ldc = p->ldc;
  a.chain_flavour = p->chain_flavour;
  a.chain_q = p->chain_q;
  a.row_group = p->row_group;
  a.group_counters = p->group_counters;
  a.skip_cert = p->skip_cert;
  a.imp = reinterpret_cast<int2*>(p->imp);
  a.imp_cnt = p->imp_cnt;
  if (a.skip_cert && (!a.imp || !a.imp_cnt || p->flat || p->dense_mode || a.kap <= 0.0f))
    return fail(SKM_E_ARG, "pruned_scan: skip_cert needs imp/imp_cnt, list mode, flat = 0 and kap > 0");
  if ((a.row_group != nullptr) != (a.group_counters != nullptr))
    return fail(SKM_E_ARG, "pruned_scan: row_group and group_counters go together");
  if (a.kap > 0.0f && (!a.xsq || !a.ysq || !a.ysq_max || !a.cent))
    return fail(SKM_E_ARG, "pruned_scan: kap > 0 needs xsq, ysq, ysq_max and cent");
  // dynamic shared memory available to the scan kernel: the opt-in limit minus its static part
  static int dyn_limit = -1;
  if (dyn_limit < 0) {
    int dv = 0, optin = 0;
    cudaGetDevice(&dv);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dv);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, skm::pruned_scan_kernel<false>);
    cudaFuncAttributes fb{};
    cudaFuncGetAttributes(&fb, skm::pruned_scan_kernel<true>);
    dyn_limit = optin - static_cast<int>(std::max(fa.sharedSizeBytes, fb.sharedSizeBytes));
  }
  // tails longer than the 4-warp CTA's staging: the one-warp instantiation (no flat pass)
  // (SKM_SCAN_FORCE_WIDE=1: every tail, for cross-checking the two instantiations)
  static const bool force_wide = getenv("SKM_SCAN_FORCE_WIDE") && atoi(getenv("SKM_SCAN_FORCE_WIDE")) != 0;
  const bool wide = force_wide || p->nb > skm::SCAN_NB_MAX || skm::scan_dyn_smem(p->nb) > static_cast<size_t>(dyn_limit);
  if (wide) return launch_pruned_scan_wide(a, p, stream);
  // exact re-evaluations from shared memory when the row's front + SCAN_EXS centroid fronts fit
  a.ex_stage = (a.kap > 0.0f && skm::scan_dyn_smem(p->nb, p->d_prime, true) <= static_cast<size_t>(dyn_limit)) ? 1 : 0;
  if (getenv("SKM_SCAN_EXSTAGE") && atoi(getenv("SKM_SCAN_EXSTAGE")) == 0) a.ex_stage = 0;
  const size_t smem = skm::scan_dyn_smem(p->nb, p->d_prime, a.ex_stage != 0);
  cudaStream_t st = as_stream(stream);
  {
    static unsigned long long set_mask_d = 0, set_mask_l = 0;
    if (first_use_on_device(set_mask_d))
      cudaFuncSetAttribute(skm::pruned_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit);
    if (first_use_on_device(set_mask_l)) {
      cudaFuncSetAttribute(skm::pruned_scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit);
      const char* cv = getenv("SKM_SCAN_CARVEOUT");
      if (cv) cudaFuncSetAttribute(skm::pruned_scan_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
    }
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (p->dense_mode)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skm::pruned_scan_kernel<true>, skm::SCAN_WARPS * 32, smem);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, skm::pruned_scan_kernel<false>, skm::SCAN_WARPS * 32, smem);
  const int blocks = std::max(1, std::min((p->n_rows + skm::SCAN_WARPS - 1) / skm::SCAN_WARPS, sms * std::max(per_sm, 1)));
  const bool flat = p->flat && !p->dense_mode && a.ex_stage && a.kap > 0.0f && !a.rows &&
                    skm::flat_dyn_smem(p->nb, p->d_prime) <= static_cast<size_t>(dyn_limit);
  if (p->flat && flat && (!p->fb_rows || !p->fb_count)) return fail(SKM_E_ARG, "pruned_scan: flat needs fb_rows/fb_count");
  if (flat) {
    static unsigned long long set_mask_f = 0;
    if (first_use_on_device(set_mask_f))
      cudaFuncSetAttribute(skm::flat_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_limit);
    const size_t fsm = skm::flat_dyn_smem(p->nb, p->d_prime);
    int per_sm_f = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_f, skm::flat_scan_kernel, skm::SCAN_WARPS * 32, fsm);
    const int fblocks =
        std::max(1, std::min((p->n_rows + skm::SCAN_WARPS - 1) / skm::SCAN_WARPS, sms * std::max(per_sm_f, 1)));
    cudaError_t e = cudaMemsetAsync(p->fb_count, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return cuda_fail(e, "pruned_scan fallback reset");
    { skm::flat_scan_kernel<<<fblocks, skm::SCAN_WARPS * 32, fsm, st>>>(a, p->fb_rows, p->fb_count); SKM_COUNT_LAUNCH(); }
    SKM_LAUNCH_CHECK("flat_scan");
    // the fallback rows through the exact kernel (row count read on the device)
    e = cudaMemsetAsync(p->work, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return cuda_fail(e, "pruned_scan work reset");
    a.rows = p->fb_rows;
    a.n_rows_dev = p->fb_count;
  }
  if (p->dense_mode)
    { skm::pruned_scan_kernel<true><<<blocks, skm::SCAN_WARPS * 32, smem, st>>>(a); SKM_COUNT_LAUNCH(); }
  else
    { skm::pruned_scan_kernel<false><<<blocks, skm::SCAN_WARPS * 32, smem, st>>>(a); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("pruned_scan");
  return SKM_OK;
}


// ---------------------------------------------------------------- top-k / ETR
int skm_topk_rows(const float* d, long long ld, int rows, int cols, int k, int* out_idx, float* out_val,
                  long long out_ld, int col_offset, void* stream) {
  if (rows <= 0 || k <= 0) return SKM_OK;
  if (k > skm::TOPK_MAX) return fail(SKM_E_ARG, "topk_rows: k too large (max 2048)");
  { skm::topk_rows_kernel<<<rows, skm::TOPK_THREADS, 0, as_stream(stream)>>>(d, ld, cols, k, out_idx, out_val, out_ld,
                                                                           col_offset); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("topk_rows");
  return SKM_OK;
}

int skm_topk_merge(const int* in_idx, const float* in_val, int shards, int k, int rows, int* out_idx, float* out_val,
                   void* stream) {
  if (rows <= 0) return SKM_OK;
  if (shards > 8) return fail(SKM_E_ARG, "topk_merge: at most 8 shards");
  { skm::topk_merge_kernel<<<(rows + 127) / 128, 128, 0, as_stream(stream)>>>(in_idx, in_val, shards, k, rows, out_idx,
                                                                            out_val); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("topk_merge");
  return SKM_OK;
}

int skm_etr_hits(const int* gt, int gt_ld, int top_k, const int* probe, int probe_ld, int nprobe, const int* assign,
                 long long row_lo, long long row_hi, int k, int nq, int* hits, void* stream) {
  if (nq <= 0) return SKM_OK;
  const size_t smem = sizeof(unsigned) * ((k + 31) / 32);
  if (smem > 200 * 1024) return fail(SKM_E_ARG, "etr_hits: k too large for the shared bitmap");
  static unsigned long long set_mask = 0;
  if (first_use_on_device(set_mask)) {
    cudaFuncSetAttribute(skm::etr_hits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  { skm::etr_hits_kernel<<<nq, 256, smem, as_stream(stream)>>>(gt, gt_ld, top_k, probe, probe_ld, nprobe, assign, row_lo,
                                                             row_hi, k, hits); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("etr_hits");
  return SKM_OK;
}

// probe_eval tally (evaluation.py:173-203): hits[q] = #{g in gt[q][:top_k] : assign[g] in
// probe[q][:nprobe]} and explored[q] += sum of sizes[c] over the probed clusters.
int skm_probe_tally(const int* gt, int gt_ld, int top_k, const int* probe, int probe_ld, int nprobe, const int* assign,
                    long long n, int k, int nq, const int* sizes, int* hits, long long* explored, void* stream) {
  if (nq <= 0) return SKM_OK;
  const size_t smem = sizeof(unsigned) * ((k + 31) / 32);
  if (smem > 200 * 1024) return fail(SKM_E_ARG, "probe_tally: k too large for the shared bitmap");
  static unsigned long long set_mask = 0;
  if (first_use_on_device(set_mask)) {
    cudaFuncSetAttribute(skm::etr_hits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  { skm::etr_hits_kernel<<<nq, 256, smem, as_stream(stream)>>>(gt, gt_ld, top_k, probe, probe_ld, nprobe, assign, 0, n,
                                                             k, hits, sizes, explored); SKM_COUNT_LAUNCH(); }
  SKM_LAUNCH_CHECK("probe_tally");
  return SKM_OK;
}

}  // extern "C"
