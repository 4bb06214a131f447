// spgemm.cu -- Gustavson SpGEMM C = A @ B over CSC operands.
//
// Replaces _kernels.spgemm (_kernels.py:51-103) via ops.matmul
// (ops.py:110-120).  The reference accumulates, per output column j, the
// products a(i,k)*b(k,j) in B-column order then A-column order into a dense
// accumulator (first product assigns, later ones add), sorts the touched
// rows, and prunes exact zeros.
//
// B200 design (expand - sort - fold, bit-exact):
//  1. as_spgemm_products: per column of B, the number of products
//     (sum of |A[:,k]| over its entries) -> chained scan -> prod_ptr.
//  2. expand: one warp per B column flattens its products in reference order
//     (kk ascending, ii ascending) with a load-balanced warp scan, writing
//     key = (row << 32) | product_index and the separately rounded product.
//  3. the segmented tile engine (segsort.cuh) sorts each column's products by
//     (row, product_index) -- the product index *is* the reference's
//     accumulation order -- folds runs sequentially (kSumSeq), prunes zeros
//     and compacts into CSC with one chained scan.  Columns whose products
//     overflow shared memory are radix-sorted by row bits only, since they
//     arrive already in index order.
#include "capi_util.cuh"
#include "persist_host.cuh"

namespace as {

constexpr int kGThreads = 256;

// products per column of B, one warp per column
__global__ void __launch_bounds__(kGThreads)
spgemm_count_kernel(long long n_cols_b, const int* __restrict__ a_ptr, const int* __restrict__ b_ptr,
                    const int* __restrict__ b_rows, unsigned* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long j = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n_cols_b; j += warps) {
    unsigned long long s = 0;
    for (int kk = b_ptr[j] + lane; kk < b_ptr[j + 1]; kk += 32) {
      int k = b_rows[kk];
      s += (unsigned)(a_ptr[k + 1] - a_ptr[k]);
    }
    s = warp_reduce_sum(s);
    if (lane == 0) counts[j] = (unsigned)s;
  }
}

// flatten the products of each B column in reference order
__global__ void __launch_bounds__(kGThreads)
spgemm_expand_kernel(long long n_cols_b, const int* __restrict__ a_ptr, const int* __restrict__ a_rows,
                     const double* __restrict__ a_vals, const int* __restrict__ b_ptr, const int* __restrict__ b_rows,
                     const double* __restrict__ b_vals, const long long* __restrict__ prod_ptr,
                     unsigned long long* __restrict__ keys, unsigned* __restrict__ colb, double* __restrict__ pvals) {
  __shared__ int s_off[kGThreads / 32][33];
  __shared__ int s_k[kGThreads / 32][32];
  __shared__ double s_b[kGThreads / 32][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long j = (long long)blockIdx.x * (blockDim.x >> 5) + wib; j < n_cols_b; j += warps) {
    long long out = prod_ptr[j];
    const int kb = b_ptr[j], ke = b_ptr[j + 1];
    for (int base = kb; base < ke; base += 32) {
      const int kk = base + lane;
      int len = 0, k = 0;
      double bv = 0.0;
      if (kk < ke) {
        k = b_rows[kk];
        bv = b_vals[kk];
        len = a_ptr[k + 1] - a_ptr[k];
      }
      int inc = warp_inclusive_scan(len);
      s_off[wib][lane + 1] = inc;
      if (lane == 0) s_off[wib][0] = 0;
      s_k[wib][lane] = a_ptr[k];
      s_b[wib][lane] = bv;
      const int total = __shfl_sync(0xffffffffu, inc, 31);
      __syncwarp();
      const int nent = min(32, ke - base);
      for (int q = lane; q < total; q += 32) {
        // entry e with s_off[e] <= q < s_off[e+1]
        int lo = 0, hi = nent - 1;
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (s_off[wib][mid] <= q) lo = mid;
          else hi = mid - 1;
        }
        const int ii = s_k[wib][lo] + (q - s_off[wib][lo]);
        const long long pos = out + q;
        keys[pos] = ((unsigned long long)(unsigned)a_rows[ii] << 32) | (unsigned long long)pos;
        colb[pos] = (unsigned)j;
        pvals[pos] = __dmul_rn(a_vals[ii], s_b[wib][lo]);
      }
      out += total;
      __syncwarp();
    }
  }
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_spgemm_products_workspace_bytes(int64_t n_cols_b) {
  const long long per = (long long)kScanThreads * kScanItems;
  long long tiles = n_cols_b > 0 ? (n_cols_b + per - 1) / per : 1;
  Carve c(nullptr, 0);
  c.take<unsigned>(64);
  c.take<unsigned long long>(tiles);
  c.take<unsigned>(n_cols_b > 0 ? n_cols_b : 1);
  return c.off;
}

int as_spgemm_products(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t* a_col_ptr,
                       const int32_t* b_col_ptr, const int32_t* b_row_idx, int64_t* prod_ptr, int64_t* info, void* ws,
                       size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows_a >= 0 && n_inner >= 0 && n_cols_b >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(ws_bytes >= as_spgemm_products_workspace_bytes(n_cols_b), AS_ERR_ARG, "workspace too small");
  const long long per = (long long)kScanThreads * kScanItems;
  long long tiles = n_cols_b > 0 ? (n_cols_b + per - 1) / per : 1;
  Carve c(ws, ws_bytes);
  unsigned* ticket = c.take<unsigned>(64);
  unsigned long long* states = c.take<unsigned long long>(tiles);
  unsigned* counts = c.take<unsigned>(n_cols_b > 0 ? n_cols_b : 1);
  AS_CUDA_TRY(cudaMemsetAsync(ws, 0, c.off, st));
  if (n_cols_b > 0) {
    spgemm_count_kernel<<<grid_for(n_cols_b * 32, kGThreads), kGThreads, 0, st>>>(n_cols_b, a_col_ptr, b_col_ptr,
                                                                                   b_row_idx, counts);
    AS_LAUNCH_CHECK();
  }
  count_scan_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(counts, n_cols_b, (long long*)prod_ptr, states, ticket,
                                                              nullptr, 0);
  AS_LAUNCH_CHECK();
  AS_CUDA_TRY(cudaMemcpyAsync(info, prod_ptr + n_cols_b, sizeof(long long), cudaMemcpyDeviceToDevice, st));
  return AS_OK;
}

size_t as_spgemm_workspace_bytes(int64_t n_cols_b, int64_t total_products) {
  return persist_ws_bytes(total_products, n_cols_b, sizeof(double));
}

int as_spgemm_f64(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t* a_col_ptr,
                  const int32_t* a_row_idx, const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx,
                  const double* b_vals, const int64_t* prod_ptr, int64_t total_products, int32_t* col_ptr,
                  int32_t* row_idx, double* out_vals, int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows_a >= 0 && n_inner >= 0 && n_cols_b >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(n_rows_a <= 0x7fffffffll && n_cols_b <= 0x7fffffffll, AS_ERR_SHAPE, "dimension outside int32 range");
  AS_REQUIRE(total_products >= 0 && total_products <= 0x7fffffffll, AS_ERR_ARG,
             "%lld products exceed the 31-bit product index", (long long)total_products);
  Carve c(ws, ws_bytes);
  PersistWs w;
  carve_persist(c, &w, total_products, n_cols_b, sizeof(double));
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  if (n_cols_b > 0 && total_products > 0) {
    spgemm_expand_kernel<<<grid_for(n_cols_b * 32, kGThreads, 16), kGThreads, 0, st>>>(
        n_cols_b, a_col_ptr, a_row_idx, a_vals, b_col_ptr, b_row_idx, b_vals, (const long long*)prod_ptr, w.keys,
        w.colb, (double*)w.vals_b);
    AS_LAUNCH_CHECK();
  }
  ValSrc<double> vs{(const double*)w.vals_b, nullptr, (unsigned long long)total_products};
  return run_persist_ws<double>(w, NoSrc<double>{}, NoSrc<double>{}, total_products, n_cols_b,
                                bits_for(n_rows_a > 0 ? n_rows_a - 1 : 0), kSumSeq, 1, vs, col_ptr, row_idx, out_vals,
                                (long long*)info, false, (const long long*)prod_ptr, st);
}

}  // extern "C"
