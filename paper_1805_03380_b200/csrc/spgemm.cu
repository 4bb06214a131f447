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
//  2. as_spgemm_f64 first scans the per-entry product counts of B
//     (|A[:,b_rows[kk]]|) into ent_ptr, then expands with CTAs over equal
//     ranges of products -- not over columns, so a 90k-product column costs
//     what any 90k products cost.  Each CTA stages the B entries its range
//     touches (start, A column start, b value, column) in shared memory and
//     every thread locates its product with a shared-memory search; writes
//     key = (row << 32) | product_index, the column and the separately
//     rounded product, all coalesced.
//  3. the persistent bucket kernel (persist.cuh, pre-bucketed mode) sorts
//     each column's products by (row, product_index) -- the product index
//     *is* the reference's accumulation order -- folds runs sequentially
//     (kSumSeq), prunes zeros and compacts into CSC.
#include "capi_util.cuh"
#include "persist_host.cuh"

namespace as {

constexpr int kGThreads = 256;

// products per column of B, three tiers: a lane sums a column of up to
// kCountShort entries itself (entries and A column lengths 4 at a time), the
// warp sums a column of up to kCountLong entries together, and a longer one
// is listed for spgemm_count_long_kernel, where a whole CTA sums it (a warp
// walking a 4096-entry Zipf column alone was the critical path: 64
// dependent round trips).
constexpr int kCountShort = 64, kCountLong = 256;

__global__ void __launch_bounds__(kGThreads)
spgemm_count_kernel(long long n_cols_b, const int* __restrict__ a_ptr, const int* __restrict__ b_ptr,
                    const int* __restrict__ b_rows, unsigned* __restrict__ counts, unsigned* __restrict__ longs,
                    unsigned* __restrict__ n_longs) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long j0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; j0 < n_cols_b;
       j0 += nw * 32) {  // warp-uniform trip count
    const long long j = j0 + lane;
    const bool valid = j < n_cols_b;
    const int b0 = valid ? __ldg(&b_ptr[j]) : 0, b1 = valid ? __ldg(&b_ptr[j + 1]) : 0;
    const int len = b1 - b0;
    if (valid && len <= kCountShort) {
      unsigned long long s = 0;
      for (int kk = b0; kk < b1; kk += 4) {
        int k[4];
#pragma unroll
        for (int u = 0; u < 4; u++) k[u] = kk + u < b1 ? __ldg(&b_rows[kk + u]) : -1;
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (k[u] >= 0) s += (unsigned)(__ldg(&a_ptr[k[u] + 1]) - __ldg(&a_ptr[k[u]]));
      }
      counts[j] = (unsigned)s;
    }
    if (valid && len > kCountLong) longs[atomicAdd(n_longs, 1u)] = (unsigned)j;
    unsigned mm = __ballot_sync(0xffffffffu, valid && len > kCountShort && len <= kCountLong);
    while (mm) {
      const int src = __ffs(mm) - 1;
      mm &= mm - 1;
      const int c0 = __shfl_sync(0xffffffffu, b0, src), c1 = __shfl_sync(0xffffffffu, b1, src);
      unsigned long long t = 0;
      for (int kk = c0 + lane; kk < c1; kk += 32 * 4) {
        int k[4];
#pragma unroll
        for (int u = 0; u < 4; u++) k[u] = kk + 32 * u < c1 ? __ldg(&b_rows[kk + 32 * u]) : -1;
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (k[u] >= 0) t += (unsigned)(__ldg(&a_ptr[k[u] + 1]) - __ldg(&a_ptr[k[u]]));
      }
      t = warp_reduce_sum(t);
      if (lane == src) counts[j] = (unsigned)t;
    }
  }
}

__global__ void __launch_bounds__(kGThreads)
spgemm_count_long_kernel(const int* __restrict__ a_ptr, const int* __restrict__ b_ptr,
                         const int* __restrict__ b_rows, unsigned* __restrict__ counts,
                         const unsigned* __restrict__ longs, const unsigned* __restrict__ n_longs) {
  __shared__ long long red[kGThreads / 32 + 1];
  const unsigned nl = *n_longs;
  for (unsigned i = blockIdx.x; i < nl; i += gridDim.x) {
    const unsigned j = longs[i];
    const int b0 = __ldg(&b_ptr[j]), b1 = __ldg(&b_ptr[j + 1]);
    long long s = 0;
    for (int kk = b0 + threadIdx.x; kk < b1; kk += 4 * kGThreads) {
      int k[4];
#pragma unroll
      for (int u = 0; u < 4; u++) k[u] = kk + u * kGThreads < b1 ? __ldg(&b_rows[kk + u * kGThreads]) : -1;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (k[u] >= 0) s += (long long)(__ldg(&a_ptr[k[u] + 1]) - __ldg(&a_ptr[k[u]]));
    }
    s = block_reduce_sum<long long>(s, red);
    if (threadIdx.x == 0) counts[j] = (unsigned)s;
  }
}

// |A[:, b_rows[kk]]| for every entry of B
__global__ void __launch_bounds__(kGThreads)
spgemm_entry_len_kernel(long long nnz_b, const int* __restrict__ a_ptr, const int* __restrict__ b_rows,
                        unsigned* __restrict__ lens) {
  for (long long kk = (long long)blockIdx.x * blockDim.x + threadIdx.x; kk < nnz_b; kk += (long long)gridDim.x * blockDim.x) {
    const int k = __ldg(&b_rows[kk]);
    lens[kk] = (unsigned)(__ldg(&a_ptr[k + 1]) - __ldg(&a_ptr[k]));
  }
}

constexpr int kExThreads = 256;
constexpr int kExItems = 8;
constexpr int kExRange = kExThreads * kExItems;  // products per CTA
constexpr int kExWin = kExRange + 1;             // staged B entries (longer windows search globally)

// For every product range t: the first / last B entry it touches and their
// columns (one thread per range; the expand CTAs then start without a
// dependent chain of global binary searches).
__global__ void __launch_bounds__(kExThreads)
spgemm_range_bounds_kernel(long long n_ranges, long long nnz_b, long long n_cols_b, long long total,
                           const int* __restrict__ b_ptr, const long long* __restrict__ ent_ptr,
                           long long* __restrict__ bounds) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n_ranges;
       t += (long long)gridDim.x * blockDim.x) {
    const long long P0 = t * kExRange, P1 = min(total, P0 + kExRange);
    auto last_le = [&](long long q) {  // last entry with ent_ptr <= q
      long long lo = 0, hi = nnz_b - 1;
      while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (__ldg(&ent_ptr[mid]) <= q) lo = mid;
        else hi = mid - 1;
      }
      return lo;
    };
    auto col_of = [&](long long kk) {  // last j with b_ptr[j] <= kk
      long long lo = 0, hi = n_cols_b - 1;
      while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (__ldg(&b_ptr[mid]) <= kk) lo = mid;
        else hi = mid - 1;
      }
      return lo;
    };
    const long long kk0 = last_le(P0), kk1 = last_le(P1 - 1);
    bounds[4 * t] = kk0;
    bounds[4 * t + 1] = kk1;
    bounds[4 * t + 2] = col_of(kk0);
    bounds[4 * t + 3] = col_of(kk1);
  }
}

// Flatten products [t*kExRange, (t+1)*kExRange) in reference order (entry kk
// ascending, A position ascending): product q belongs to the last entry with
// ent_ptr[kk] <= q.
__global__ void __launch_bounds__(kExThreads)
spgemm_expand_kernel(long long nnz_b, long long n_cols_b, long long total, const int* __restrict__ a_ptr,
                     const int* __restrict__ a_rows, const double* __restrict__ a_vals,
                     const int* __restrict__ b_ptr, const int* __restrict__ b_rows,
                     const double* __restrict__ b_vals, const long long* __restrict__ ent_ptr,
                     const long long* __restrict__ bounds, const long long* __restrict__ prod_ptr,
                     long long dense_min, unsigned long long* __restrict__ keys, unsigned* __restrict__ colb,
                     double* __restrict__ pvals) {
  // products of a column with more than dense_min products go to the dense
  // column path of the bucket kernel, which needs only their row (in colb)
  // and value: no key, no column
  __shared__ unsigned s_ent[kExWin];  // range position -> its entry (marks at entry starts, then a max-scan)
  __shared__ int s_ast[kExWin];       // A position of the entry's product q is s_ast[e] + q
  __shared__ int s_col[kExWin];
  __shared__ double s_bv[kExWin];
  __shared__ unsigned s_scan[kExThreads / 32 + 1];
  const int tid = threadIdx.x;
  for (long long t = blockIdx.x; t * kExRange < total; t += gridDim.x) {
    const long long P0 = t * kExRange, P1 = min(total, P0 + kExRange);
    __syncthreads();
    const long long kk0 = __ldg(&bounds[4 * t]), kk1 = __ldg(&bounds[4 * t + 1]);
    const long long j0 = __ldg(&bounds[4 * t + 2]), j1 = __ldg(&bounds[4 * t + 3]);
    const int nw = (int)(kk1 - kk0 + 1);
    const bool staged = nw <= kExWin;
    auto dense_col = [&](long long c) { return __ldg(&prod_ptr[c + 1]) - __ldg(&prod_ptr[c]) > dense_min; };
    const int cnt = (int)(P1 - P0);
    if (staged) {
      for (int q = tid; q < cnt; q += kExThreads) s_ent[q] = 0u;
      __syncthreads();
      for (int e = tid; e < nw; e += kExThreads) {
        const long long kk = kk0 + e;
        const long long off = __ldg(&ent_ptr[kk]) - P0;
        const long long end = (kk + 1 < nnz_b ? __ldg(&ent_ptr[kk + 1]) : total) - P0;
        const int k = __ldg(&b_rows[kk]);
        // entry kk's product at range position q sits at A position a_ptr[k] + (q - off)
        s_ast[e] = (int)(__ldg(&a_ptr[k]) - off);
        s_bv[e] = __ldg(&b_vals[kk]);
        const long long st0 = max(off, 0ll);
        if (min(end, (long long)cnt) > st0) s_ent[st0] = (unsigned)e;  // the one non-empty entry starting here
        long long lo = j0, hi = j1;
        while (lo < hi) {
          const long long mid = (lo + hi + 1) >> 1;
          if (__ldg(&b_ptr[mid]) <= kk) lo = mid;
          else hi = mid - 1;
        }
        s_col[e] = dense_col(lo) ? -1 - (int)lo : (int)lo;  // negative: dense column
      }
      __syncthreads();
      {  // every position's entry: inclusive max-scan of the marks
        const int q0 = tid * kExItems;
        unsigned m[kExItems], run = 0u;
#pragma unroll
        for (int u = 0; u < kExItems; u++) {
          m[u] = q0 + u < cnt ? s_ent[q0 + u] : 0u;
          run = max(run, m[u]);
        }
        unsigned ex = block_exclusive_max(run, s_scan);
#pragma unroll
        for (int u = 0; u < kExItems; u++) {
          ex = max(ex, m[u]);
          if (q0 + u < cnt) s_ent[q0 + u] = ex;
        }
      }
      __syncthreads();
    }
    auto emit = [&](long long pos, int col, unsigned row, double v) {
      if (col >= 0) {
        keys[pos] = ((unsigned long long)row << 32) | (unsigned long long)pos;
        colb[pos] = (unsigned)col;
      } else {
        colb[pos] = row;
      }
      pvals[pos] = v;
    };
    if (staged) {
      // kExItems products per thread: all shared-memory searches, then all
      // gathers of A (in flight together), then the stores
      int ii[kExItems], cl[kExItems];
      double bv[kExItems];
#pragma unroll
      for (int u = 0; u < kExItems; u++) {
        const int q = tid + u * kExThreads;
        const int e = q < cnt ? (int)s_ent[q] : 0;
        ii[u] = s_ast[e] + q;
        cl[u] = s_col[e];
        bv[u] = s_bv[e];
      }
      unsigned rw[kExItems];
      double av[kExItems];
#pragma unroll
      for (int u = 0; u < kExItems; u++) {
        const bool in = tid + u * kExThreads < cnt;
        rw[u] = in ? (unsigned)__ldg(&a_rows[ii[u]]) : 0u;
        av[u] = in ? __ldg(&a_vals[ii[u]]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kExItems; u++) {
        const int q = tid + u * kExThreads;
        if (q < cnt) emit(P0 + q, cl[u], rw[u], __dmul_rn(av[u], bv[u]));
      }
    } else {  // many empty A columns in the window: search globally
      for (int q = tid; q < cnt; q += kExThreads) {
        long long lo = kk0, hi = kk1;
        while (lo < hi) {
          const long long mid = (lo + hi + 1) >> 1;
          if (__ldg(&ent_ptr[mid]) <= P0 + q) lo = mid;
          else hi = mid - 1;
        }
        const int k = __ldg(&b_rows[lo]);
        const int ii = (int)(__ldg(&a_ptr[k]) + (P0 + q - __ldg(&ent_ptr[lo])));
        const double bv = __ldg(&b_vals[lo]);
        long long cl = j0, ch = j1;
        while (cl < ch) {
          const long long mid = (cl + ch + 1) >> 1;
          if (__ldg(&b_ptr[mid]) <= lo) cl = mid;
          else ch = mid - 1;
        }
        int col = (int)cl;
        if (dense_col(col)) col = -1 - col;
        emit(P0 + q, col, (unsigned)__ldg(&a_rows[ii]), __dmul_rn(__ldg(&a_vals[ii]), bv));
      }
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
  c.take<unsigned>(n_cols_b > 0 ? n_cols_b : 1);  // long-column list
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
  unsigned* longs = c.take<unsigned>(n_cols_b > 0 ? n_cols_b : 1);  // columns above kCountLong entries
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small");
  if (n_cols_b > 0) {
    spgemm_count_kernel<<<grid_for((n_cols_b + 31) / 32 * 32, kGThreads), kGThreads, 0, st>>>(n_cols_b, a_col_ptr, b_col_ptr,
                                                                             b_row_idx, counts, longs, ticket + 32);
    AS_LAUNCH_CHECK();
    spgemm_count_long_kernel<<<num_sms() * 4, kGThreads, 0, st>>>(a_col_ptr, b_col_ptr, b_row_idx, counts, longs,
                                                               ticket + 32);
    AS_LAUNCH_CHECK();
  }
  count_scan_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(counts, n_cols_b, (long long*)prod_ptr, states, ticket);
  AS_LAUNCH_CHECK();
  AS_CUDA_TRY(cudaMemcpyAsync(info, prod_ptr + n_cols_b, sizeof(long long), cudaMemcpyDeviceToDevice, st));
  return AS_OK;
}

static void carve_spgemm(Carve& c, PersistWs* w, long long n_cols_b, long long nnz_b, long long total,
                         unsigned** scan_zero, size_t* scan_zero_bytes, unsigned long long** states, unsigned** lens,
                         long long** ent_ptr, long long** bounds) {
  carve_persist(c, w, total, n_cols_b, sizeof(double), true);
  const long long per = (long long)kScanThreads * kScanItems;
  const long long tiles = nnz_b > 0 ? (nnz_b + per - 1) / per : 1;
  const size_t z0 = c.off;
  *scan_zero = c.take<unsigned>(64);
  *states = c.take<unsigned long long>(tiles);
  *scan_zero_bytes = c.off - z0;
  *lens = c.take<unsigned>(std::max(1ll, nnz_b));
  *ent_ptr = c.take<long long>(nnz_b + 1);
  *bounds = c.take<long long>(4 * std::max(1ll, (total + kExRange - 1) / kExRange));
}

size_t as_spgemm_workspace_bytes(int64_t n_cols_b, int64_t nnz_b, int64_t total_products) {
  Carve c(nullptr, 0);
  PersistWs w;
  unsigned *z, *lens;
  size_t zb;
  unsigned long long* states;
  long long *ent, *bounds;
  carve_spgemm(c, &w, n_cols_b, nnz_b, total_products, &z, &zb, &states, &lens, &ent, &bounds);
  return c.off;
}

int as_spgemm_f64(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t* a_col_ptr,
                  const int32_t* a_row_idx, const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx,
                  const double* b_vals, int64_t nnz_b, const int64_t* prod_ptr, int64_t total_products,
                  int32_t* col_ptr, int32_t* row_idx, double* out_vals, int64_t* info, void* ws, size_t ws_bytes,
                  void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows_a >= 0 && n_inner >= 0 && n_cols_b >= 0 && nnz_b >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(n_rows_a <= 0x7fffffffll && n_cols_b <= 0x7fffffffll, AS_ERR_SHAPE, "dimension outside int32 range");
  AS_REQUIRE(total_products >= 0 && total_products <= 0x7fffffffll, AS_ERR_ARG,
             "%lld products exceed the 31-bit product index", (long long)total_products);
  Carve c(ws, ws_bytes);
  PersistWs w;
  unsigned *scan_zero, *lens;
  size_t zb;
  unsigned long long* states;
  long long *ent_ptr, *bounds;
  carve_spgemm(c, &w, n_cols_b, nnz_b, total_products, &scan_zero, &zb, &states, &lens, &ent_ptr, &bounds);
  w.dense_rows = n_rows_a;
  // the dense column path (and the expand's row-only products) when the
  // output rows fit its shared-memory bitmaps
  const bool dense = dense_column_bytes(n_rows_a) <= (long long)kPersistSmemBytes;
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  if (n_cols_b > 0 && nnz_b > 0 && total_products > 0) {
    const long long per = (long long)kScanThreads * kScanItems;
    const long long tiles = (nnz_b + per - 1) / per;
    AS_CUDA_TRY(cudaMemsetAsync(scan_zero, 0, zb, st));
    spgemm_entry_len_kernel<<<grid_for(nnz_b, kGThreads), kGThreads, 0, st>>>(nnz_b, a_col_ptr, b_row_idx, lens);
    AS_LAUNCH_CHECK();
    count_scan_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(lens, nnz_b, ent_ptr, states, scan_zero);
    AS_LAUNCH_CHECK();
    const long long ranges = (total_products + kExRange - 1) / kExRange;
    spgemm_range_bounds_kernel<<<grid_for(ranges, kExThreads), kExThreads, 0, st>>>(
        ranges, nnz_b, n_cols_b, total_products, b_col_ptr, ent_ptr, bounds);
    AS_LAUNCH_CHECK();
    spgemm_expand_kernel<<<(unsigned)std::min<long long>(ranges, (long long)num_sms() * 32), kExThreads, 0, st>>>(
        nnz_b, n_cols_b, total_products, a_col_ptr, a_row_idx, a_vals, b_col_ptr, b_row_idx, b_vals, ent_ptr, bounds,
        (const long long*)prod_ptr, dense ? (long long)kCap : LLONG_MAX, w.keys, w.colb, (double*)w.vals_b);
    AS_LAUNCH_CHECK();
  }
  ValSrc<double> vs{(const double*)w.vals_b, nullptr, (unsigned long long)total_products};
  return run_persist_ws<double>(w, NoSrc<double>{}, NoSrc<double>{}, total_products, n_cols_b,
                                bits_for(n_rows_a > 0 ? n_rows_a - 1 : 0), kSumSeq, 1, vs, col_ptr, row_idx, out_vals,
                                (long long*)info, false, (const long long*)prod_ptr, st);
}

}  // extern "C"
