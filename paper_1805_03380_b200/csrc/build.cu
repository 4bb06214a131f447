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
#include "persist_host.cuh"
#include "sortreduce_api.h"
#include "largen_api.h"


namespace as {

// pinned (or mapped) host memory: device-accessible through UVA
static bool is_host_pointer(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

inline size_t staging_bytes(long long n, size_t val_bytes) {
  Carve c(nullptr, 0);
  c.take<int>(n);
  c.take<int>(n);
  c.take<char>(n * (long long)val_bytes);
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
  const int mode = dup == AS_DUP_SUM ? kSumPairwise : kLast;
  const int row_bits = bits_for(n_rows > 0 ? n_rows - 1 : 0);
  if (g_engine == 0) {  // the lean single-level kernel when the input fits its envelope (device or pinned host triplets)
    const int rc = sr::coo_to_csc<T, IdxT>(n_rows, n_cols, n, rows, cols, vals, mode, col_ptr, row_idx, out_vals, info,
                                           ws, ws_bytes, st);
    if (rc != -1) return rc;
  }
  if (n > 0 && is_host_pointer(rows)) {
    // pinned host triplets: read once over PCIe inside the kernel (CooHostSrc),
    // staged in the tail of the workspace; outputs may be pinned host memory too
    AS_REQUIRE(is_host_pointer(cols) && is_host_pointer(vals), AS_ERR_ARG,
               "rows, cols and vals must all be device or all pinned host memory");
    const size_t pb = persist_ws_bytes(n, n_cols, sizeof(T));
    AS_REQUIRE(ws_bytes >= pb + staging_bytes(n, sizeof(T)), AS_ERR_ARG, "workspace too small for host input");
    Carve c((char*)ws + pb, ws_bytes - pb);
    CooHostSrc<IdxT, T> hs{s1, c.take<int>(n), c.take<int>(n), c.take<T>(n)};
    AS_CUDA_TRY(cudaMemsetAsync(hs.st_rows, 0xff, (size_t)n * sizeof(int), st));  // skipped bad triplets stay -1
    ValSrc<T> vs{hs.st_vals, nullptr, (unsigned long long)n};
    return run_persist<T>(hs, NoSrc<T>{}, n_cols, row_bits, mode, 1, vs, col_ptr, row_idx, out_vals, info, true, ws,
                          pb, st);
  }
  if (g_engine != 2) {  // large inputs: LSD bucket passes + the same tiles (largen.cuh)
    const int rc = ln::coo_to_csc<T, IdxT>(n_rows, n_cols, n, rows, cols, vals, mode, col_ptr, row_idx, out_vals, info,
                                           ws, ws_bytes, st);
    if (rc != -1) return rc;
  }
  ValSrc<T> vs{vals, nullptr, (unsigned long long)n};
  return run_persist<T>(s1, NoSrc<T>{}, n_cols, row_bits, mode, 1, vs, col_ptr, row_idx, out_vals, info, true, ws,
                        ws_bytes, st);
}

template <class T>
static int csc_transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
                         const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && n_rows <= kMaxDim && n_cols <= kMaxDim, AS_ERR_SHAPE,
             "dimensions %lldx%lld outside the int32 device index range", n_rows, n_cols);
  AS_REQUIRE(nnz >= 0 && nnz <= kMaxDim, AS_ERR_ARG, "nnz %lld outside the int32 range", nnz);
  if (g_engine == 0) {
    const int rc = sr::transpose<T>(n_rows, n_cols, nnz, col_ptr, row_idx, vals, t_col_ptr, t_row_idx, t_vals, ws,
                                    ws_bytes, st);
    if (rc != -1) return rc;
  }
  if (g_engine != 2) {
    const int rc = ln::transpose<T>(n_rows, n_cols, nnz, col_ptr, row_idx, vals, t_col_ptr, t_row_idx, t_vals, ws,
                                    ws_bytes, st);
    if (rc != -1) return rc;
  }
  CscSrc<T> s1{col_ptr, row_idx, vals, n_cols, nnz, true, 0ull};
  ValSrc<T> vs{vals, nullptr, (unsigned long long)nnz};
  return run_persist<T>(s1, NoSrc<T>{}, n_rows, bits_for(n_cols > 0 ? n_cols - 1 : 0), kLast, 0, vs, t_col_ptr,
                        t_row_idx, t_vals, nullptr, false, ws, ws_bytes, st);
}

}  // namespace as

using namespace as;

extern "C" {

// (includes the staging of pinned-host triplets; a device-input build uses only the first part)
size_t as_build_workspace_bytes(int64_t n, int64_t n_cols) {
  return std::max({persist_ws_bytes(n, n_cols, 8) + staging_bytes(n, 8), sr::ws_bytes_api(n, 8),
                   ln::ws_bytes(n, n_cols, 8)});
}
size_t as_flush_workspace_bytes(int64_t nnz_base, int64_t n_log, int64_t n_cols) {
  return std::max(persist_ws_bytes(nnz_base + n_log, n_cols, 8), sr::ws_bytes_api(nnz_base + n_log, 8));
}
size_t as_transpose_workspace_bytes(int64_t nnz, int64_t n_rows) {
  return std::max({persist_ws_bytes(nnz, n_rows, 8), sr::ws_bytes_api(nnz, 8), ln::ws_bytes(nnz, n_rows, 8)});
}

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
  if (g_engine == 0) {
    const int rc = sr::flush_f64(n_rows, n_cols, nnz_base, base_col_ptr, base_row_idx, base_vals, n_log, log_rows,
                                 log_cols, log_vals, col_ptr, row_idx, out_vals, (long long*)info, ws, ws_bytes,
                                 S(stream));
    if (rc != -1) return rc;
  }
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
