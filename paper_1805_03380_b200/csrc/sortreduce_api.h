// sortreduce_api.h -- entry points of the lean sort-reduce kernel
// (sortreduce.cu), called by build.cu's C-ABI functions before they fall back
// to the general bucket kernel.  Each returns AS_OK / an error status after
// launching, or -1 when the input is outside the kernel's envelope.
#pragma once

namespace as {
namespace sr {

size_t ws_bytes_api(long long n, size_t val_bytes);

template <class T, class IdxT>
int coo_to_csc(long long n_rows, long long n_cols, long long n, const IdxT* rows, const IdxT* cols, const T* vals,
               int mode, int* col_ptr, int* row_idx, T* out_vals, long long* info, void* ws, size_t ws_bytes,
               cudaStream_t st);

template <class T>
int transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
              const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals, void* ws, size_t ws_bytes, cudaStream_t st);

int flush_f64(long long n_rows, long long n_cols, long long nnz_base, const int* base_col_ptr, const int* base_row_idx,
              const double* base_vals, long long n_log, const int* log_rows, const int* log_cols,
              const double* log_vals, int* col_ptr, int* row_idx, double* out_vals, long long* info, void* ws,
              size_t ws_bytes, cudaStream_t st);

}  // namespace sr
}  // namespace as
