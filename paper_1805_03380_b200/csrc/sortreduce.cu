// sortreduce.cu -- instantiations of the lean sort-reduce kernel for
// construction, flush and transpose (its own translation unit: compiled in
// parallel with build.cu).
#include "sortreduce_host.cuh"
#include "sortreduce_api.h"

namespace as {
namespace sr {

size_t ws_bytes_api(long long n, size_t val_bytes) { return ws_bytes(n, val_bytes); }

template <class T, class IdxT>
int coo_to_csc(long long n_rows, long long n_cols, long long n, const IdxT* rows, const IdxT* cols, const T* vals,
               int mode, int* col_ptr, int* row_idx, T* out_vals, long long* info, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  return run<T>(Coo<IdxT, T>{rows, cols, vals, n, n_rows, n_cols}, None{}, n, n, n_cols,
                bits_for(n_rows > 0 ? n_rows - 1 : 0), n_rows, mode, 1, col_ptr, row_idx, out_vals, info, ws, ws_bytes, st);
}

template <class T>
int transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
              const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals, void* ws, size_t ws_bytes, cudaStream_t st) {
  return run<T>(Csc<T>{col_ptr, row_idx, vals, n_cols, nnz, true}, None{}, nnz, nnz, n_rows,
                bits_for(n_cols > 0 ? n_cols - 1 : 0), n_cols, kLast, 0, t_col_ptr, t_row_idx, t_vals, nullptr, ws, ws_bytes,
                st);
}

int flush_f64(long long n_rows, long long n_cols, long long nnz_base, const int* base_col_ptr, const int* base_row_idx,
              const double* base_vals, long long n_log, const int* log_rows, const int* log_cols,
              const double* log_vals, int* col_ptr, int* row_idx, double* out_vals, long long* info, void* ws,
              size_t ws_bytes, cudaStream_t st) {
  return run<double>(Csc<double>{base_col_ptr, base_row_idx, base_vals, n_cols, nnz_base, false},
                     Coo<int, double>{log_rows, log_cols, log_vals, n_log, n_rows, n_cols}, nnz_base, nnz_base + n_log,
                     n_cols, bits_for(n_rows > 0 ? n_rows - 1 : 0), n_rows, kLast, 1, col_ptr, row_idx, out_vals, info, ws,
                     ws_bytes, st);
}

template int coo_to_csc<double, int>(long long, long long, long long, const int*, const int*, const double*, int, int*,
                                     int*, double*, long long*, void*, size_t, cudaStream_t);
template int coo_to_csc<double, long long>(long long, long long, long long, const long long*, const long long*,
                                           const double*, int, int*, int*, double*, long long*, void*, size_t,
                                           cudaStream_t);
template int coo_to_csc<float, int>(long long, long long, long long, const int*, const int*, const float*, int, int*,
                                    int*, float*, long long*, void*, size_t, cudaStream_t);
template int coo_to_csc<float, long long>(long long, long long, long long, const long long*, const long long*,
                                          const float*, int, int*, int*, float*, long long*, void*, size_t,
                                          cudaStream_t);
template int transpose<double>(long long, long long, long long, const int*, const int*, const double*, int*, int*,
                               double*, void*, size_t, cudaStream_t);
template int transpose<float>(long long, long long, long long, const int*, const int*, const float*, int*, int*,
                              float*, void*, size_t, cudaStream_t);

}  // namespace sr
}  // namespace as
