// add.cu -- alpha*A + beta*B of two canonical CSC matrices.
//
// Replaces _kernels.linear_combine (_kernels.py:12-48) via ops._combine /
// add / subtract / scaled_sum (ops.py:50-73).  Per column a two-pointer row
// merge; coincident rows give alpha*a + beta*b (product and sum separately
// rounded, as numba evaluates it: no FMA), others alpha*a or beta*b; exact
// zeros are pruned.
//
// B200 design: the (A,B) column pairs form one merged sequence; tile t owns
// the columns whose merged start lies in [t*kAddTile, (t+1)*kAddTile).  Each
// thread merges kAddItems consecutive positions (merge path, so long and
// short columns balance), a count pass feeds a single-pass chained scan
// (decoupled look-back) for the tile's output offset, and the write pass
// stages the compacted chunk in shared memory so the row/value stores are
// coalesced.  One kernel, no separate sizing pass over HBM.
#include "capi_util.cuh"
#include "common.cuh"

namespace as {

constexpr int kAddThreads = 256;
constexpr int kAddItems = 8;
constexpr int kAddChunk = kAddThreads * kAddItems;
constexpr int kAddTile = 2048;

AS_DEVICE_INLINE long long mstart2(const int* ap, const int* bp, long long c) {
  return (long long)ap[c] + (long long)bp[c];
}

// first c in [lo, hi) with mstart(c) >= x
AS_DEVICE_INLINE long long ms_lower_bound(const int* ap, const int* bp, long long lo, long long hi, long long x) {
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (mstart2(ap, bp, mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Merge kAddItems diagonal positions [d0, d1) of the tile's merged sequence.
// emit(row, value) for kept outputs in order; on_col(c, produced) when the
// thread owns the start of column c.
template <class Emit, class OnCol>
__device__ void merge_range(long long c_lo, long long c_hi, long long d0, long long d1, const int* __restrict__ ap,
                            const int* __restrict__ ar, const double* __restrict__ av, const int* __restrict__ bp,
                            const int* __restrict__ br, const double* __restrict__ bv, double alpha, double beta,
                            Emit emit, OnCol on_col) {
  // last c in [c_lo, c_hi) with mstart(c) <= d0
  long long lo = c_lo, hi = c_hi - 1;
  while (lo < hi) {
    long long mid = (lo + hi + 1) >> 1;
    if (mstart2(ap, bp, mid) <= d0) lo = mid;
    else hi = mid - 1;
  }
  long long c = lo;
  long long a0 = ap[c], b0 = bp[c];
  long long la = ap[c + 1] - a0, lb = bp[c + 1] - b0;
  long long dl = d0 - (a0 + b0);
  if (dl == 0) {  // we own the starts of c and of the empty columns sharing it
    for (long long cc = c; cc >= c_lo && mstart2(ap, bp, cc) == d0; cc--) on_col(cc, 0);
  }
  long long i_lo = max(0ll, dl - lb), i_hi = min(dl, la);
  while (i_lo < i_hi) {
    long long mid = (i_lo + i_hi) >> 1;
    if (ar[a0 + mid] <= br[b0 + dl - mid - 1]) i_lo = mid + 1;
    else i_hi = mid;
  }
  long long i = i_lo, j = dl - i_lo;
  if (i > 0 && j < lb && br[b0 + j] == ar[a0 + i - 1]) j++;
  long long pos = a0 + b0 + i + j;
  int produced = 0;
  while (pos < d1) {
    if (i == la && j == lb) {
      c++;
      a0 = ap[c];
      b0 = bp[c];
      la = ap[c + 1] - a0;
      lb = bp[c + 1] - b0;
      i = j = 0;
      on_col(c, produced);
      continue;
    }
    int r;
    double v;
    if (j == lb || (i < la && ar[a0 + i] < br[b0 + j])) {
      r = ar[a0 + i];
      v = __dmul_rn(alpha, av[a0 + i]);
      i++;
    } else if (i == la || br[b0 + j] < ar[a0 + i]) {
      r = br[b0 + j];
      v = __dmul_rn(beta, bv[b0 + j]);
      j++;
    } else {
      r = ar[a0 + i];
      v = __dadd_rn(__dmul_rn(alpha, av[a0 + i]), __dmul_rn(beta, bv[b0 + j]));
      i++;
      j++;
    }
    if (v != 0.0) {
      emit(r, v);
      produced++;
    }
    pos = a0 + b0 + i + j;
  }
}

struct AddSmem {
  int rows[kAddChunk];
  double vals[kAddChunk];
  long long scan_tmp[kAddThreads / 32 + 1];
  long long tile, c0, c1, m0, m;
  unsigned long long prefix;
};

__global__ void __launch_bounds__(kAddThreads)
csc_add_kernel(long long n_cols, double alpha, double beta, const int* __restrict__ ap, const int* __restrict__ ar,
               const double* __restrict__ av, const int* __restrict__ bp, const int* __restrict__ br,
               const double* __restrict__ bv, int* __restrict__ out_ptr, int* __restrict__ out_rows,
               double* __restrict__ out_vals, long long* info, unsigned long long* states, unsigned* ticket) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AddSmem& S = *reinterpret_cast<AddSmem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long n_tiles = gridDim.x;
  if (tid == 0) {
    long long t = atomicAdd(ticket, 1u);
    long long c0 = ms_lower_bound(ap, bp, 0, n_cols, t * kAddTile);
    long long c1 = (t == n_tiles - 1) ? n_cols : ms_lower_bound(ap, bp, c0, n_cols, (t + 1) * kAddTile);
    S.tile = t;
    S.c0 = c0;
    S.c1 = c1;
    S.m0 = mstart2(ap, bp, c0);
    S.m = mstart2(ap, bp, c1) - S.m0;
  }
  __syncthreads();
  const long long t = S.tile, c0 = S.c0, c1 = S.c1, m0 = S.m0, m = S.m;

  // pass 1: count
  long long total = 0;
  for (long long b = 0; b < m; b += kAddChunk) {
    const long long d0 = m0 + b + (long long)tid * kAddItems;
    const long long d1 = min(d0 + kAddItems, m0 + m);
    int cnt = 0;
    if (d0 < d1)
      merge_range(c0, c1, d0, d1, ap, ar, av, bp, br, bv, alpha, beta, [&](int, double) { cnt++; },
                  [&](long long, int) {});
    total += block_reduce_sum<long long>((long long)cnt, S.scan_tmp);
  }
  if (warp == 0) {
    unsigned long long pre = tile_lookback_warp(states, t, (unsigned long long)total);
    if (lane == 0) S.prefix = pre;
  }
  __syncthreads();
  const long long P = (long long)S.prefix;

  // pass 2: write, staged through shared memory
  long long run = 0;
  for (long long b = 0; b < m; b += kAddChunk) {
    const long long d0 = m0 + b + (long long)tid * kAddItems;
    const long long d1 = min(d0 + kAddItems, m0 + m);
    int cnt = 0;
    if (d0 < d1)
      merge_range(c0, c1, d0, d1, ap, ar, av, bp, br, bv, alpha, beta, [&](int, double) { cnt++; },
                  [&](long long, int) {});
    long long ctot;
    long long off = block_exclusive_scan<long long>((long long)cnt, S.scan_tmp, &ctot);
    int w = (int)off;
    if (d0 < d1)
      merge_range(
          c0, c1, d0, d1, ap, ar, av, bp, br, bv, alpha, beta,
          [&](int r, double v) {
            S.rows[w] = r;
            S.vals[w] = v;
            w++;
          },
          [&](long long c, int produced) {
            if (c < c1) out_ptr[c] = (int)(P + run + off + produced);
          });
    __syncthreads();
    for (long long q = tid; q < ctot; q += kAddThreads) {
      out_rows[P + run + q] = S.rows[q];
      out_vals[P + run + q] = S.vals[q];
    }
    run += ctot;
    __syncthreads();
  }
  // empty columns at the end of the tile
  for (long long c = c0 + tid; c < c1; c += kAddThreads)
    if (mstart2(ap, bp, c) >= m0 + m) out_ptr[c] = (int)(P + total);
  if (t == n_tiles - 1 && tid == 0) {
    out_ptr[n_cols] = (int)(P + total);
    info[0] = P + total;
  }
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_add_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b) {
  (void)n_cols;
  long long M = nnz_a + nnz_b;
  long long tiles = M > 0 ? (M + kAddTile - 1) / kAddTile : 1;
  return 256 + (size_t)tiles * 8;
}

int as_csc_add_f64(int64_t n_rows, int64_t n_cols, double alpha, double beta, const int32_t* a_col_ptr,
                   const int32_t* a_row_idx, const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx,
                   const double* b_vals, int64_t nnz_a, int64_t nnz_b, int32_t* col_ptr, int32_t* row_idx,
                   double* out_vals, int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(nnz_a + nnz_b <= 0x7fffffffll, AS_ERR_ARG, "nnz outside the int32 range");
  AS_REQUIRE(ws_bytes >= as_add_workspace_bytes(n_cols, nnz_a, nnz_b), AS_ERR_ARG, "workspace too small");
  long long M = nnz_a + nnz_b;
  long long tiles = M > 0 ? (M + kAddTile - 1) / kAddTile : 1;
  unsigned* ticket = (unsigned*)ws;
  unsigned long long* states = (unsigned long long*)((char*)ws + 256);
  AS_CUDA_TRY(cudaMemsetAsync(ws, 0, as_add_workspace_bytes(n_cols, nnz_a, nnz_b), st));
  static bool attr = false;
  if (!attr) {
    AS_CUDA_TRY(cudaFuncSetAttribute(csc_add_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(AddSmem)));
    attr = true;
  }
  csc_add_kernel<<<(unsigned)tiles, kAddThreads, sizeof(AddSmem), st>>>(n_cols, alpha, beta, a_col_ptr, a_row_idx,
                                                                         a_vals, b_col_ptr, b_row_idx, b_vals, col_ptr,
                                                                         row_idx, out_vals, (long long*)info, states,
                                                                         ticket);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

}  // extern "C"
