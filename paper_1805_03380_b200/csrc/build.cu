// build.cu -- COO->CSC construction, insertion-log flush and CSC transpose.
//
// All three are "bucket by major index, sort each bucket by (minor index,
// input order), reduce runs, compact":
//   construction  csc.canonicalize (csc.py:148-193): bucket = col, minor = row,
//                 reduce = np.add.reduceat order (Sum) or last (LastWins)
//   flush         rbt.to_csc over RbtStore semantics (rbt.py:371-458):
//                 base CSC ++ write log, reduce = last, prune zeros (= erase)
//   transpose     _kernels.transpose (_kernels.py:130-150): bucket = row,
//                 minor = col (unique per bucket), no reduce, no prune
// Each call is two memsets and ONE cooperative launch of
// persist_bucket_kernel (persist.cuh); no host synchronisation.
#include "capi_util.cuh"
#include "persist.cuh"

#include <stdlib.h>

namespace as {

constexpr long long kMaxDim = 0x7fffffffll;
constexpr long long kMaxGrid = 148 * 8;  // upper bound of the co-resident grid

struct PersistWs {
  unsigned* zero;  // [0] ticket, [16] barrier arrive, [32] barrier generation, then cb_cnt
  unsigned* cb_cnt;
  size_t zero_bytes;
  long long* cb_start;
  unsigned long long* keys;
  unsigned long long* keys_alt;
  unsigned* colb;
  unsigned* colb_alt;
  void* vals_b;
  int* tmp_rows;
  void* tmp_vals;
  unsigned* col_kept;
  long long* cta_sums;
  long long* own_info;
  int wbits;
  long long n_cb;
};

// Coarse buckets of W = 2^wbits output columns: ~0.8 * kCap elements per
// bucket on average, at most kMaxCoarse buckets.  Returns -1 when the column
// count exceeds kMaxCoarse * kMaxW.
static inline int choose_wbits(long long n, long long n_cols) {
  const double avg = n_cols > 0 ? (double)n / (double)n_cols : 0.0;
  int wb = 0;
  while ((1 << (wb + 1)) <= kMaxW && (double)(1 << (wb + 1)) * avg <= 0.8 * kCap) wb++;
  while (wb <= 10 && ((n_cols + (1ll << wb) - 1) >> wb) > kMaxCoarse) wb++;
  return ((n_cols + (1ll << wb) - 1) >> wb) > kMaxCoarse || (1 << wb) > kMaxW ? -1 : wb;
}

static size_t carve_persist(Carve& c, PersistWs* w, long long n, long long n_cols, size_t val_bytes) {
  w->wbits = choose_wbits(n, n_cols);
  const int wb = w->wbits < 0 ? 10 : w->wbits;
  w->n_cb = (n_cols + (1ll << wb) - 1) >> wb;
  w->zero = c.take<unsigned>(64);
  w->cb_cnt = c.take<unsigned>(std::max(1ll, w->n_cb));
  w->zero_bytes = c.off;
  w->cb_start = c.take<long long>(w->n_cb + 1);
  const long long n1 = std::max(1ll, n);
  w->keys = c.take<unsigned long long>(n1);
  w->keys_alt = c.take<unsigned long long>(n1);
  w->colb = c.take<unsigned>(n1);
  w->colb_alt = c.take<unsigned>(n1);
  w->vals_b = (void*)c.take<char>(n1 * val_bytes);
  w->tmp_rows = c.take<int>(n1);
  w->tmp_vals = (void*)c.take<char>(n1 * val_bytes);
  w->col_kept = c.take<unsigned>(std::max(1ll, n_cols));
  w->cta_sums = c.take<long long>(kMaxGrid);
  w->own_info = c.take<long long>(2);
  return c.off;
}

template <class T, class S1, class S2>
static int launch_persist(PersistArgs<T, S1, S2>& a, cudaStream_t st) {
  static int grid = 0;
  const size_t smem = sizeof(PersistSmem<T>);
  auto kern = persist_bucket_kernel<T, S1, S2>;
  if (grid == 0) {
    AS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, dev = 0, sms = 0;
    AS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSegThreads, smem));
    AS_CUDA_TRY(cudaGetDevice(&dev));
    AS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    AS_REQUIRE(per_sm > 0, AS_ERR_CUDA, "persistent kernel does not fit on an SM");
    grid = (int)std::min<long long>((long long)per_sm * sms, kMaxGrid);
  }
  void* args[] = {(void*)&a};
  AS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSegThreads), args, smem, st));
  return AS_OK;
}

template <class T, class S1, class S2>
static int run_persist(const S1& s1, const S2& s2, long long n_cols, int row_bits, int mode, int prune, ValSrc<T> vs,
                       int* col_ptr, int* row_idx, T* out_vals, long long* info, bool init_info, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  const long long n = s1.size() + s2.size();
  Carve c(ws, ws_bytes);
  PersistWs w;
  carve_persist(c, &w, n, n_cols, sizeof(T));
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  AS_REQUIRE(w.wbits >= 0, AS_ERR_ARG, "%lld output columns exceed the %lld supported by the bucket kernel",
             n_cols, (long long)kMaxCoarse * kMaxW);
  if (info == nullptr) info = w.own_info;
  AS_CUDA_TRY(cudaMemsetAsync(w.zero, 0, w.zero_bytes, st));
  if (init_info) AS_CUDA_TRY(cudaMemsetAsync(info, 0x7f, 2 * sizeof(long long), st));
  PersistArgs<T, S1, S2> a;
  a.s1 = s1;
  a.s2 = s2;
  a.n_cols = n_cols;
  a.n_upper = n;
  a.wbits = w.wbits;
  a.n_cb = w.n_cb;
  a.cb_cnt = w.cb_cnt;
  a.cb_start = w.cb_start;
  a.keys = w.keys;
  a.keys_alt = w.keys_alt;
  a.colb = w.colb;
  a.colb_alt = w.colb_alt;
  a.vals_b = (T*)w.vals_b;
  a.tmp_rows = w.tmp_rows;
  a.tmp_vals = (T*)w.tmp_vals;
  a.col_kept = w.col_kept;
  a.cta_sums = w.cta_sums;
  a.row_bits = row_bits;
  a.idx_bits = bits_for(n > 0 ? n - 1 : 0);
  a.mode = mode;
  a.prune = prune;
  a.vs = vs;
  a.col_ptr = col_ptr;
  a.row_idx = row_idx;
  a.out_vals = out_vals;
  a.info = info;
  a.ticket = w.zero;
  a.gb = GridBar{w.zero + 16, w.zero + 32};
  a.phase_ts = nullptr;
  static unsigned long long* dbg_ts = nullptr;
  const bool phase_dbg = getenv("AS_PHASE_TIMES") != nullptr;
  if (phase_dbg) {
    if (!dbg_ts) AS_CUDA_TRY(cudaMalloc(&dbg_ts, 16 * sizeof(unsigned long long)));
    AS_CUDA_TRY(cudaMemsetAsync(dbg_ts, 0, 16 * sizeof(unsigned long long), st));
    a.phase_ts = dbg_ts;
  }
  const int rc = launch_persist<T, S1, S2>(a, st);
  if (phase_dbg && rc == AS_OK) {
    unsigned long long h[16];
    AS_CUDA_TRY(cudaMemcpyAsync(h, dbg_ts, sizeof(h), cudaMemcpyDeviceToHost, st));
    AS_CUDA_TRY(cudaStreamSynchronize(st));
    fprintf(stderr, "[phases n=%lld n_cols=%lld W=%d n_cb=%lld]", n, n_cols, 1 << w.wbits, w.n_cb);
    for (int i = 1; i < 16 && h[i]; i++) fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, " us\n");
  }
  return rc;
}

size_t persist_ws_bytes(long long n, long long n_cols, size_t val_bytes) {
  Carve c(nullptr, 0);
  PersistWs w;
  carve_persist(c, &w, n, n_cols, val_bytes);
  return c.off;
}

template <class T, class IdxT>
static int coo_to_csc(long long n_rows, long long n_cols, long long n, const IdxT* rows, const IdxT* cols,
                      const T* vals, int dup, int* col_ptr, int* row_idx, T* out_vals, long long* info, void* ws,
                      size_t ws_bytes, cudaStream_t st) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", n_rows, n_cols);
  AS_REQUIRE(n >= 0 && n <= kMaxDim, AS_ERR_ARG, "triplet count %lld outside the int32 range", n);
  AS_REQUIRE(dup == AS_DUP_SUM || dup == AS_DUP_LAST, AS_ERR_ARG, "unknown duplicate policy %d", dup);
  CooSrc<IdxT, T> s1{rows, cols, vals, n, n_rows, n_cols, 0ull, info + 1};
  ValSrc<T> vs{vals, nullptr, (unsigned long long)n};
  return run_persist<T>(s1, NoSrc<T>{}, n_cols, bits_for(n_rows > 0 ? n_rows - 1 : 0),
                        dup == AS_DUP_SUM ? kSumPairwise : kLast, 1, vs, col_ptr, row_idx, out_vals, info, true, ws,
                        ws_bytes, st);
}

template <class T>
static int csc_transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
                         const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", n_rows, n_cols);
  AS_REQUIRE(nnz >= 0 && nnz <= kMaxDim, AS_ERR_ARG, "nnz %lld outside the int32 range", nnz);
  CscSrc<T> s1{col_ptr, row_idx, vals, n_cols, nnz, true, 0ull};
  ValSrc<T> vs{vals, nullptr, (unsigned long long)nnz};
  return run_persist<T>(s1, NoSrc<T>{}, n_rows, bits_for(n_cols > 0 ? n_cols - 1 : 0), kLast, 0, vs, t_col_ptr,
                        t_row_idx, t_vals, nullptr, false, ws, ws_bytes, st);
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_build_workspace_bytes(int64_t n, int64_t n_cols) { return persist_ws_bytes(n, n_cols, 8); }
size_t as_flush_workspace_bytes(int64_t nnz_base, int64_t n_log, int64_t n_cols) {
  return persist_ws_bytes(nnz_base + n_log, n_cols, 8);
}
size_t as_transpose_workspace_bytes(int64_t nnz, int64_t n_rows) { return persist_ws_bytes(nnz, n_rows, 8); }

#define AS_BUILD_DISPATCH(T)                                                                                    \
  if (idx_bytes == 4)                                                                                            \
    return coo_to_csc<T, int>(n_rows, n_cols, n, (const int*)rows, (const int*)cols, vals, dup, col_ptr, row_idx, \
                              out_vals, (long long*)info, ws, ws_bytes, S(stream));                              \
  if (idx_bytes == 8)                                                                                            \
    return coo_to_csc<T, long long>(n_rows, n_cols, n, (const long long*)rows, (const long long*)cols, vals, dup, \
                                    col_ptr, row_idx, out_vals, (long long*)info, ws, ws_bytes, S(stream));       \
  set_error("idx_bytes must be 4 or 8, got %d", idx_bytes);                                                      \
  return AS_ERR_ARG;

int as_coo_to_csc_f64(int64_t n_rows, int64_t n_cols, int64_t n, const void* rows, const void* cols, int idx_bytes,
                      const double* vals, int dup, int32_t* col_ptr, int32_t* row_idx, double* out_vals,
                      int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  AS_BUILD_DISPATCH(double)
}

int as_coo_to_csc_f32(int64_t n_rows, int64_t n_cols, int64_t n, const void* rows, const void* cols, int idx_bytes,
                      const float* vals, int dup, int32_t* col_ptr, int32_t* row_idx, float* out_vals,
                      int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  AS_BUILD_DISPATCH(float)
}

int as_flush_log_f64(int64_t n_rows, int64_t n_cols, int64_t nnz_base, const int32_t* base_col_ptr,
                     const int32_t* base_row_idx, const double* base_vals, int64_t n_log, const int32_t* log_rows,
                     const int32_t* log_cols, const double* log_vals, int32_t* col_ptr, int32_t* row_idx,
                     double* out_vals, int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", (long long)n_rows, (long long)n_cols);
  AS_REQUIRE(nnz_base >= 0 && n_log >= 0 && nnz_base + n_log <= kMaxDim, AS_ERR_ARG,
             "element count outside the int32 range");
  CscSrc<double> s1{base_col_ptr, base_row_idx, base_vals, n_cols, nnz_base, false, 0ull};
  CooSrc<int, double> s2{log_rows, log_cols, log_vals, n_log, n_rows, n_cols, (unsigned long long)nnz_base,
                         (long long*)info + 1};
  ValSrc<double> vs{base_vals, log_vals, (unsigned long long)nnz_base};
  return run_persist<double>(s1, s2, n_cols, bits_for(n_rows > 0 ? n_rows - 1 : 0), kLast, 1, vs, col_ptr, row_idx,
                             out_vals, (long long*)info, true, ws, ws_bytes, S(stream));
}

int as_csc_transpose_f64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* col_ptr, const int32_t* row_idx,
                         const double* vals, int32_t* t_col_ptr, int32_t* t_row_idx, double* t_vals, void* ws,
                         size_t ws_bytes, void* stream) {
  return csc_transpose<double>(n_rows, n_cols, nnz, col_ptr, row_idx, vals, t_col_ptr, t_row_idx, t_vals, ws,
                               ws_bytes, S(stream));
}

int as_csc_transpose_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* col_ptr, const int32_t* row_idx,
                         const float* vals, int32_t* t_col_ptr, int32_t* t_row_idx, float* t_vals, void* ws,
                         size_t ws_bytes, void* stream) {
  return csc_transpose<float>(n_rows, n_cols, nnz, col_ptr, row_idx, vals, t_col_ptr, t_row_idx, t_vals, ws,
                              ws_bytes, S(stream));
}

}  // extern "C"
