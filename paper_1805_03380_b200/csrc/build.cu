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
// Kernel sequence per call (one stream, no host sync):
//   memset -> count (warp-aggregated atomics) -> chained-scan of counts ->
//   scatter (u64 keys) -> seg_tile_kernel (sort + reduce + chained compaction)
#include "capi_util.cuh"
#include "segsort.cuh"

namespace as {

struct BuildWs {
  unsigned* tickets;               // [0] scan, [1] seg engine
  unsigned long long* scan_states;
  unsigned long long* seg_states;
  unsigned* counts;
  long long* seg_ptr;
  unsigned long long* keys;
  unsigned long long* keys_alt;
  char* zero_begin;
  size_t zero_bytes;
};

static inline long long seg_tiles(long long n) { return seg_engine_tiles(n); }
static inline long long scan_tiles(long long n) {
  const long long per = (long long)kScanThreads * kScanItems;
  return n > 0 ? (n + per - 1) / per : 1;
}

static size_t carve_build(Carve& c, BuildWs* w, long long n, long long n_seg) {
  w->tickets = c.take<unsigned>(64);
  w->scan_states = c.take<unsigned long long>(scan_tiles(n_seg));
  w->seg_states = c.take<unsigned long long>(seg_tiles(n));
  w->counts = c.take<unsigned>(n_seg > 0 ? n_seg : 1);
  w->zero_begin = (char*)w->tickets;
  w->zero_bytes = c.off;
  w->seg_ptr = c.take<long long>(n_seg + 1);
  w->keys = c.take<unsigned long long>(n > 0 ? n : 1);
  w->keys_alt = c.take<unsigned long long>(n > 0 ? n : 1);
  return c.off;
}

template <class T>
static int run_seg_engine(const BuildWs& w, long long n_seg, long long n_upper, int row_bits, int idx_bits,
                          int presorted, ValSrc<T> vs, int mode, int prune, int* col_ptr, int* row_idx,
                          T* vals, long long* info, cudaStream_t st) {
  return launch_seg_engine<T>(w.seg_ptr, n_seg, n_upper, w.keys, w.keys_alt, row_bits, idx_bits, presorted, vs, mode,
                              prune, col_ptr, row_idx, vals, info, w.seg_states, w.tickets + 1, st);
}

static int run_scan(const BuildWs& w, long long n_seg, cudaStream_t st) {
  count_scan_kernel<<<(unsigned)scan_tiles(n_seg), kScanThreads, 0, st>>>(w.counts, n_seg, w.seg_ptr,
                                                                          w.scan_states, w.tickets);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

#define AS_TRY(expr)             \
  do {                           \
    int _rc = (expr);            \
    if (_rc != AS_OK) return _rc; \
  } while (0)

constexpr long long kMaxDim = 0x7fffffffll;

template <class T, class IdxT>
static int coo_to_csc(long long n_rows, long long n_cols, long long n, const IdxT* rows, const IdxT* cols,
                      const T* vals, int dup, int* col_ptr, int* row_idx, T* out_vals, long long* info,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", n_rows, n_cols);
  AS_REQUIRE(n >= 0 && n <= kMaxDim, AS_ERR_ARG, "triplet count %lld outside the int32 range", n);
  AS_REQUIRE(dup == AS_DUP_SUM || dup == AS_DUP_LAST, AS_ERR_ARG, "unknown duplicate policy %d", dup);
  Carve c(ws, ws_bytes);
  BuildWs w;
  carve_build(c, &w, n, n_cols);
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  AS_CUDA_TRY(cudaMemsetAsync(w.zero_begin, 0, w.zero_bytes, st));
  AS_CUDA_TRY(cudaMemsetAsync(info, 0x7f, 2 * sizeof(long long), st));
  const int B = 256;
  if (n > 0) {
    coo_count_kernel<IdxT><<<grid_for(n, B), B, 0, st>>>(n, rows, cols, n_rows, n_cols, w.counts, info + 1);
    AS_LAUNCH_CHECK();
  }
  AS_TRY(run_scan(w, n_cols, st));
  if (n > 0) {
    coo_scatter_kernel<IdxT><<<grid_for(n, B), B, 0, st>>>(n, rows, cols, n_rows, n_cols, w.seg_ptr, w.counts,
                                                           w.keys, 0ull);
    AS_LAUNCH_CHECK();
  }
  ValSrc<T> vs{vals, nullptr, (unsigned long long)n};
  return run_seg_engine<T>(w, n_cols, n, bits_for(n_rows > 0 ? n_rows - 1 : 0), bits_for(n > 0 ? n - 1 : 0), 0,
                           vs, dup == AS_DUP_SUM ? kSumPairwise : kLast, 1, col_ptr, row_idx, out_vals, info, st);
}

template <class T>
static int csc_transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr,
                         const int* row_idx, const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals,
                         void* ws, size_t ws_bytes, cudaStream_t st) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", n_rows, n_cols);
  AS_REQUIRE(nnz >= 0 && nnz <= kMaxDim, AS_ERR_ARG, "nnz %lld outside the int32 range", nnz);
  Carve c(ws, ws_bytes);
  BuildWs w;
  carve_build(c, &w, nnz, n_rows);
  long long* info = c.take<long long>(2);
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  AS_CUDA_TRY(cudaMemsetAsync(w.zero_begin, 0, w.zero_bytes, st));
  const int B = 256;
  if (nnz > 0) {
    row_count_kernel<<<grid_for(nnz, B), B, 0, st>>>(nnz, row_idx, w.counts);
    AS_LAUNCH_CHECK();
  }
  AS_TRY(run_scan(w, n_rows, st));
  if (nnz > 0) {
    csc_scatter_kernel<true><<<grid_for(nnz, B), B, 0, st>>>(n_cols, nnz, col_ptr, row_idx, w.seg_ptr, w.counts,
                                                             w.keys);
    AS_LAUNCH_CHECK();
  }
  ValSrc<T> vs{vals, nullptr, (unsigned long long)nnz};
  return run_seg_engine<T>(w, n_rows, nnz, bits_for(n_cols > 0 ? n_cols - 1 : 0), bits_for(nnz > 0 ? nnz - 1 : 0),
                           0, vs, kLast, 0, t_col_ptr, t_row_idx, t_vals, info, st);
}

size_t build_ws_bytes(long long n, long long n_seg) {
  Carve c(nullptr, 0);
  BuildWs w;
  carve_build(c, &w, n, n_seg);
  c.take<long long>(2);
  return c.off;
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_build_workspace_bytes(int64_t n, int64_t n_cols) { return build_ws_bytes(n, n_cols); }
size_t as_flush_workspace_bytes(int64_t nnz_base, int64_t n_log, int64_t n_cols) {
  return build_ws_bytes(nnz_base + n_log, n_cols);
}
size_t as_transpose_workspace_bytes(int64_t nnz, int64_t n_rows) { return build_ws_bytes(nnz, n_rows); }

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
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", (long long)n_rows, (long long)n_cols);
  const long long n = nnz_base + n_log;
  AS_REQUIRE(nnz_base >= 0 && n_log >= 0 && n <= kMaxDim, AS_ERR_ARG, "element count outside the int32 range");
  Carve c(ws, ws_bytes);
  BuildWs w;
  carve_build(c, &w, n, n_cols);
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  AS_CUDA_TRY(cudaMemsetAsync(w.zero_begin, 0, w.zero_bytes, st));
  AS_CUDA_TRY(cudaMemsetAsync(info, 0x7f, 2 * sizeof(long long), st));
  const int B = 256;
  if (nnz_base > 0) {
    csc_count_kernel<<<grid_for(n_cols, B), B, 0, st>>>(n_cols, base_col_ptr, w.counts);
    AS_LAUNCH_CHECK();
  }
  if (n_log > 0) {
    coo_count_kernel<int><<<grid_for(n_log, B), B, 0, st>>>(n_log, log_rows, log_cols, n_rows, n_cols, w.counts,
                                                             (long long*)info + 1);
    AS_LAUNCH_CHECK();
  }
  AS_TRY(run_scan(w, n_cols, st));
  if (nnz_base > 0) {
    csc_scatter_kernel<false><<<grid_for(nnz_base, B), B, 0, st>>>(n_cols, nnz_base, base_col_ptr, base_row_idx,
                                                                   w.seg_ptr, w.counts, w.keys);
    AS_LAUNCH_CHECK();
  }
  if (n_log > 0) {
    coo_scatter_kernel<int><<<grid_for(n_log, B), B, 0, st>>>(n_log, log_rows, log_cols, n_rows, n_cols, w.seg_ptr,
                                                              w.counts, w.keys, (unsigned long long)nnz_base);
    AS_LAUNCH_CHECK();
  }
  ValSrc<double> vs{base_vals, log_vals, (unsigned long long)nnz_base};
  return run_seg_engine<double>(w, n_cols, n, bits_for(n_rows > 0 ? n_rows - 1 : 0), bits_for(n > 0 ? n - 1 : 0), 0,
                                vs, kLast, 1, col_ptr, row_idx, out_vals, (long long*)info, st);
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
