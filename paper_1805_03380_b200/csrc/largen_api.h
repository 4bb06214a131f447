// largen_api.h -- entry points of the large-input pipeline (largen.cu),
// called by build.cu's C-ABI functions after the single-launch kernel
// declines.  Each returns AS_OK / an error status after launching, or -1 when
// the input is outside the pipeline's envelope (the caller falls back to the
// general bucket kernel).  Device pointers only.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace as {
namespace ln {

size_t ws_bytes(long long n, long long n_out_cols, size_t val_bytes);

template <class T, class IdxT>
int coo_to_csc(long long n_rows, long long n_cols, long long n, const IdxT* rows, const IdxT* cols, const T* vals,
               int mode, int* col_ptr, int* row_idx, T* out_vals, long long* info, void* ws, size_t ws_bytes,
               cudaStream_t st);

template <class T>
int transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
              const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace ln
}  // namespace as
