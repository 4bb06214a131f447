// funnel.cu -- SURVEY 8f-2: the construction-funnelled operations and the
// segmented reductions of the reference's ops module, on the device.
//
//   kron / repmat (ops.py:131-163)   triplet generators; the caller funnels
//                                    them through as_coo_to_csc (the
//                                    reference funnels them through
//                                    csc.canonicalize, pruning underflows)
//   sum/min/max_dim (ops.py:166-206) sequential fold per column (CSC) or per
//                                    row (the CSR): np.add.at / minimum.at /
//                                    maximum.at visit a label's elements in
//                                    storage order; the implicit-zero rule
//                                    for min/max of a non-dense slice
//   trace, norms (ops.py:209-248)    numpy pairwise summation (np.sum) in
//                                    its exact association order
//   submat (ops.py:277-298)          window of a CSC (binary search per
//                                    column, count, scan, copy)
//   diag (ops.py:345-355)            one diagonal as a dense vector
//   normalise (ops.py:251-274)       value / norm[label] (then the caller
//                                    re-canonicalises, like the reference)
#include "capi_util.cuh"
#include "common.cuh"
#include "tile_common.cuh"

#include <cmath>

namespace as {

constexpr int kFThreads = 256;

// column of every element of a CSC (warp per column)
__global__ void __launch_bounds__(kFThreads)
expand_cols_kernel(long long n_cols, const int* __restrict__ col_ptr, int* __restrict__ cols) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n_cols; c += warps)
    for (int e = __ldg(&col_ptr[c]) + lane; e < __ldg(&col_ptr[c + 1]); e += 32) cols[e] = (int)c;
}

// kron: element e = ia * nnz_b + ib (the reference's ravel order) ->
// (ra * br + rb, ca * bc + cb, va * vb)
__global__ void __launch_bounds__(kFThreads)
kron_triplets_kernel(long long nnz_a, long long nnz_b, const int* __restrict__ a_rows, const int* __restrict__ a_cols,
                     const double* __restrict__ a_vals, const int* __restrict__ b_rows,
                     const int* __restrict__ b_cols, const double* __restrict__ b_vals, long long br, long long bc,
                     int* __restrict__ rows, int* __restrict__ cols, double* __restrict__ vals) {
  const long long total = nnz_a * nnz_b;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long ia = e / nnz_b, ib = e - ia * nnz_b;
    rows[e] = (int)(__ldg(&a_rows[ia]) * br + __ldg(&b_rows[ib]));
    cols[e] = (int)(__ldg(&a_cols[ia]) * bc + __ldg(&b_cols[ib]));
    vals[e] = __dmul_rn(__ldg(&a_vals[ia]), __ldg(&b_vals[ib]));
  }
}

// repmat: the reference concatenates row blocks i (rows + i*r) then column
// blocks j (cols + j*c): element e = (j * reps_r + i) * nnz + q
__global__ void __launch_bounds__(kFThreads)
repmat_triplets_kernel(long long nnz, const int* __restrict__ a_rows, const int* __restrict__ a_cols,
                       const double* __restrict__ a_vals, long long r, long long c, long long reps_r,
                       long long reps_c, int* __restrict__ rows, int* __restrict__ cols, double* __restrict__ vals) {
  const long long total = nnz * reps_r * reps_c;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long q = e % nnz, blk = e / nnz;
    const long long i = blk % reps_r, j = blk / reps_r;
    rows[e] = (int)(__ldg(&a_rows[q]) + i * r);
    cols[e] = (int)(__ldg(&a_cols[q]) + j * c);
    vals[e] = __ldg(&a_vals[q]);
  }
}

// elementwise transforms of the norms: 0 identity, 1 |x|, 2 x*x (numpy's
// square fast path for ** 2), 3 |x| ** p
AS_DEVICE_INLINE double xform(double x, int t, double p) {
  switch (t) {
    case 1: return fabs(x);
    case 2: return __dmul_rn(x, x);
    case 3: return pow(fabs(x), p);
    default: return x;
  }
}

// one segment per thread: sequential fold in storage order (np.add.at),
// or min / max with the implicit-zero rule (count < full)
__global__ void __launch_bounds__(kFThreads)
segment_reduce_kernel(long long n_seg, const int* __restrict__ seg_ptr, const double* __restrict__ vals, int kind,
                      int xf, double p, long long full, double* __restrict__ out) {
  for (long long sgi = (long long)blockIdx.x * blockDim.x + threadIdx.x; sgi < n_seg;
       sgi += (long long)gridDim.x * blockDim.x) {
    const int b = __ldg(&seg_ptr[sgi]), e = __ldg(&seg_ptr[sgi + 1]);
    double acc;
    if (kind == 0) {
      acc = 0.0;
      for (int i = b; i < e; i++) acc = __dadd_rn(acc, xform(__ldg(&vals[i]), xf, p));
    } else if (kind == 1) {
      acc = INFINITY;
      for (int i = b; i < e; i++) acc = fmin(acc, xform(__ldg(&vals[i]), xf, p));
      if (e - b < full) acc = fmin(acc, 0.0);
    } else {
      acc = -INFINITY;
      for (int i = b; i < e; i++) acc = fmax(acc, xform(__ldg(&vals[i]), xf, p));
      if (kind == 2 && e - b < full) acc = fmax(acc, 0.0);
      if (kind == 3 && e == b) acc = 0.0;  // max of |x| over an empty slice (norm inf / normalise inf)
    }
    out[sgi] = acc;
  }
}

// numpy's pairwise summation (np.sum of a contiguous float64 array) in its
// exact association order, in parallel: the recursion splits a range of n >
// 128 elements at n/2 rounded down to a multiple of 8.  Block b of 2^top
// follows the bits of b down the first `top` levels of that tree, then
// thread t of its 1024 follows the bits of t down kPwDepth more (a range <=
// 128 stops splitting: the leftmost thread below it owns it), sums its node
// sequentially with the same rule (pw_sum), and the nodes are combined
// bottom-up exactly as the recursion adds its two halves -- inside the block,
// then across the blocks in a one-block pass.
constexpr int kPwThreads = 1024, kPwDepth = 10, kPwTopMax = 6;

struct PwNode {
  long long lo, len;
  unsigned split;  // bit L: the node on the path at level L was split
  bool owner;
};

// descend `levels` levels from (lo, len) following the bits of `path` (MSB first)
AS_DEVICE_INLINE PwNode pw_descend(long long lo, long long len, unsigned path, int levels) {
  PwNode nd{lo, len, 0u, true};
  for (int L = 0; L < levels; L++) {
    const unsigned bit = (path >> (levels - 1 - L)) & 1u;
    if (nd.len > 128) {
      nd.split |= 1u << L;
      long long n2 = nd.len / 2;
      n2 -= n2 % 8;
      if (bit) {
        nd.lo += n2;
        nd.len -= n2;
      } else {
        nd.len = n2;
      }
    } else if (bit) {
      nd.owner = false;
    }
  }
  return nd;
}

__global__ void __launch_bounds__(kPwThreads)
pairwise_sum_kernel(long long n, const double* __restrict__ x, int xf, double p, int top, double* __restrict__ part) {
  __shared__ double s[kPwThreads];
  const int t = threadIdx.x;
  const PwNode blk = pw_descend(0, n, blockIdx.x, top);
  const PwNode nd = pw_descend(blk.lo, blk.len, (unsigned)t, kPwDepth);
  double v = 0.0;
  if (blk.owner && nd.owner && nd.len > 0)
    v = pw_sum<double>([&](long long i) { return xform(__ldg(&x[nd.lo + i]), xf, p); }, 0, nd.len);
  s[t] = v;
  __syncthreads();
  for (int L = kPwDepth - 1; L >= 0; L--) {
    const int span = 1 << (kPwDepth - L);  // threads under a level-L node
    if ((t & (span - 1)) == 0 && ((nd.split >> L) & 1u)) s[t] = __dadd_rn(s[t], s[t + span / 2]);
    __syncthreads();
  }
  if (t == 0) part[blockIdx.x] = s[0];
}

__global__ void pairwise_combine_kernel(long long n, int top, double* __restrict__ part, double* __restrict__ out) {
  const int t = threadIdx.x;  // blockDim = 2^top
  const PwNode nd = pw_descend(0, n, (unsigned)t, top);
  for (int L = top - 1; L >= 0; L--) {
    const int span = 1 << (top - L);
    __syncthreads();
    if ((t & (span - 1)) == 0 && ((nd.split >> L) & 1u)) part[t] = __dadd_rn(part[t], part[t + span / 2]);
  }
  __syncthreads();
  if (t == 0) out[0] = part[0];
}

// submat: rows [r0, r1] of columns [c0, c1]; counts via binary search
__global__ void __launch_bounds__(kFThreads)
window_count_kernel(long long c0, long long n_out_cols, const int* __restrict__ col_ptr, const int* __restrict__ rows,
                    int r0, int r1, unsigned* __restrict__ counts, int* __restrict__ starts) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n_out_cols;
       j += (long long)gridDim.x * blockDim.x) {
    const int b = __ldg(&col_ptr[c0 + j]), e = __ldg(&col_ptr[c0 + j + 1]);
    const int lo = b + (int)lower_bound_dev(rows + b, (long long)(e - b), r0);
    const int hi = b + (int)upper_bound_dev(rows + b, (long long)(e - b), r1);
    counts[j] = (unsigned)(hi - lo);
    starts[j] = lo;
  }
}

__global__ void __launch_bounds__(kFThreads)
window_fill_kernel(long long n_out_cols, const long long* __restrict__ out_ptr64, const int* __restrict__ starts,
                   const int* __restrict__ rows, const double* __restrict__ vals, int r0, int* __restrict__ out_ptr,
                   int* __restrict__ out_rows, double* __restrict__ out_vals) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long j = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j <= n_out_cols; j += warps) {
    const long long o = out_ptr64[j];
    if (lane == 0) out_ptr[j] = (int)o;
    if (j == n_out_cols) continue;
    const long long len = out_ptr64[j + 1] - o;
    const int s0 = starts[j];
    for (long long q = lane; q < len; q += 32) {
      out_rows[o + q] = __ldg(&rows[s0 + q]) - r0;
      out_vals[o + q] = __ldg(&vals[s0 + q]);
    }
  }
}

// diag k: out[t] = A(row0 + t, col0 + t) (0 where absent)
__global__ void __launch_bounds__(kFThreads)
diag_kernel(long long length, long long row0, long long col0, const int* __restrict__ col_ptr,
            const int* __restrict__ rows, const double* __restrict__ vals, double* __restrict__ out) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < length;
       t += (long long)gridDim.x * blockDim.x) {
    const int b = __ldg(&col_ptr[col0 + t]), e = __ldg(&col_ptr[col0 + t + 1]);
    const int r = (int)(row0 + t);
    const long long q = b + lower_bound_dev(rows + b, (long long)(e - b), r);
    out[t] = (q < e && __ldg(&rows[q]) == r) ? __ldg(&vals[q]) : 0.0;
  }
}

// normalise: v / norm[label] (label = column, or the row index itself)
__global__ void __launch_bounds__(kFThreads)
scale_by_label_kernel(long long nnz, const int* __restrict__ labels, const double* __restrict__ vals,
                      const double* __restrict__ norms, double* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    double nv = __ldg(&norms[__ldg(&labels[e])]);
    if (nv == 0.0) nv = 1.0;  // all-zero slices untouched (ops.py:271)
    out[e] = __ddiv_rn(__ldg(&vals[e]), nv);
  }
}

}  // namespace as

using namespace as;

extern "C" {

int as_expand_cols(int64_t n_cols, const int32_t* col_ptr, int32_t* cols, void* stream) {
  AS_REQUIRE(n_cols >= 0, AS_ERR_SHAPE, "negative dimension");
  if (n_cols > 0) {
    expand_cols_kernel<<<grid_for(n_cols * 32, kFThreads), kFThreads, 0, S(stream)>>>(n_cols, col_ptr, cols);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

int as_kron_triplets_f64(int64_t nnz_a, const int32_t* a_rows, const int32_t* a_cols, const double* a_vals,
                         int64_t nnz_b, const int32_t* b_rows, const int32_t* b_cols, const double* b_vals,
                         int64_t b_n_rows, int64_t b_n_cols, int32_t* rows, int32_t* cols, double* vals,
                         void* stream) {
  AS_REQUIRE(nnz_a >= 0 && nnz_b >= 0 && b_n_rows >= 0 && b_n_cols >= 0, AS_ERR_SHAPE, "negative size");
  AS_REQUIRE(nnz_a * nnz_b <= 0x7fffffffll, AS_ERR_ARG, "Kronecker product of %lld x %lld entries exceeds int32",
             (long long)nnz_a, (long long)nnz_b);
  const long long total = nnz_a * nnz_b;
  if (total > 0) {
    kron_triplets_kernel<<<grid_for(total, kFThreads), kFThreads, 0, S(stream)>>>(
        nnz_a, nnz_b, a_rows, a_cols, a_vals, b_rows, b_cols, b_vals, b_n_rows, b_n_cols, rows, cols, vals);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

int as_repmat_triplets_f64(int64_t nnz, const int32_t* a_rows, const int32_t* a_cols, const double* a_vals,
                           int64_t n_rows, int64_t n_cols, int64_t reps_r, int64_t reps_c, int32_t* rows,
                           int32_t* cols, double* vals, void* stream) {
  AS_REQUIRE(nnz >= 0 && reps_r >= 1 && reps_c >= 1, AS_ERR_SHAPE, "invalid replication");
  AS_REQUIRE(nnz * reps_r * reps_c <= 0x7fffffffll, AS_ERR_ARG, "replicated entry count exceeds int32");
  const long long total = nnz * reps_r * reps_c;
  if (total > 0) {
    repmat_triplets_kernel<<<grid_for(total, kFThreads), kFThreads, 0, S(stream)>>>(
        nnz, a_rows, a_cols, a_vals, n_rows, n_cols, reps_r, reps_c, rows, cols, vals);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

int as_segment_reduce_f64(int64_t n_seg, const int32_t* seg_ptr, const double* vals, int kind, int xf, double p,
                          int64_t full, double* out, void* stream) {
  AS_REQUIRE(n_seg >= 0, AS_ERR_SHAPE, "negative segment count");
  AS_REQUIRE(kind >= 0 && kind <= 3 && xf >= 0 && xf <= 3, AS_ERR_ARG, "unknown reduction %d / transform %d",
             kind, xf);
  if (n_seg > 0) {
    segment_reduce_kernel<<<grid_for(n_seg, kFThreads), kFThreads, 0, S(stream)>>>(n_seg, seg_ptr, vals, kind, xf,
                                                                                   p, full, out);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

size_t as_pairwise_workspace_bytes(void) { return sizeof(double) << kPwTopMax; }

int as_pairwise_sum_f64(int64_t n, const double* x, int xf, double p, double* out, void* ws, size_t ws_bytes,
                        void* stream) {
  AS_REQUIRE(n >= 0, AS_ERR_SHAPE, "negative length");
  AS_REQUIRE(xf >= 0 && xf <= 3, AS_ERR_ARG, "unknown transform %d", xf);
  AS_REQUIRE(ws_bytes >= as_pairwise_workspace_bytes(), AS_ERR_ARG, "workspace too small");
  int top = 0;  // 2^top blocks of 1024 threads, >= ~64 elements per thread
  while (top < kPwTopMax && (n >> (kPwDepth + top + 1)) >= 64) top++;
  double* part = (double*)ws;
  pairwise_sum_kernel<<<1u << top, kPwThreads, 0, S(stream)>>>(n, x, xf, p, top, part);
  AS_LAUNCH_CHECK();
  pairwise_combine_kernel<<<1, 1u << top, 0, S(stream)>>>(n, top, part, out);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

size_t as_window_workspace_bytes(int64_t n_out_cols) {
  const long long per = (long long)kScanThreads * kScanItems;
  const long long tiles = n_out_cols > 0 ? (n_out_cols + per - 1) / per : 1;
  Carve c(nullptr, 0);
  c.take<unsigned>(64);
  c.take<unsigned long long>(tiles);
  c.take<unsigned>(n_out_cols + 1);
  c.take<int>(n_out_cols + 1);
  c.take<long long>(n_out_cols + 1);
  return c.off;
}

int as_csc_window_f64(int64_t n_rows, int64_t n_cols, const int32_t* col_ptr, const int32_t* row_idx,
                      const double* vals, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int32_t* out_col_ptr,
                      int32_t* out_rows, double* out_vals, int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(0 <= r0 && r0 <= r1 && r1 < n_rows && 0 <= c0 && c0 <= c1 && c1 < n_cols, AS_ERR_SHAPE,
             "window [%lld,%lld]x[%lld,%lld] outside %lldx%lld", (long long)r0, (long long)r1, (long long)c0,
             (long long)c1, (long long)n_rows, (long long)n_cols);
  const long long nc = c1 - c0 + 1;
  AS_REQUIRE(ws_bytes >= as_window_workspace_bytes(nc), AS_ERR_ARG, "workspace too small");
  const long long per = (long long)kScanThreads * kScanItems;
  const long long tiles = (nc + per - 1) / per;
  Carve c(ws, ws_bytes);
  unsigned* ticket = c.take<unsigned>(64);
  unsigned long long* states = c.take<unsigned long long>(tiles);
  const size_t zb = c.off;
  unsigned* counts = c.take<unsigned>(nc + 1);
  int* starts = c.take<int>(nc + 1);
  long long* ptr64 = c.take<long long>(nc + 1);
  AS_CUDA_TRY(cudaMemsetAsync(ws, 0, zb, st));
  window_count_kernel<<<grid_for(nc, kFThreads), kFThreads, 0, st>>>(c0, nc, col_ptr, row_idx, (int)r0, (int)r1,
                                                                      counts, starts);
  AS_LAUNCH_CHECK();
  count_scan_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(counts, nc, ptr64, states, ticket);
  AS_LAUNCH_CHECK();
  window_fill_kernel<<<grid_for((nc + 1) * 32, kFThreads), kFThreads, 0, st>>>(nc, ptr64, starts, row_idx, vals,
                                                                                (int)r0, out_col_ptr, out_rows,
                                                                                out_vals);
  AS_LAUNCH_CHECK();
  AS_CUDA_TRY(cudaMemcpyAsync(info, ptr64 + nc, sizeof(long long), cudaMemcpyDeviceToDevice, st));
  return AS_OK;
}

int as_csc_diag_f64(int64_t n_rows, int64_t n_cols, const int32_t* col_ptr, const int32_t* row_idx,
                    const double* vals, int64_t k, int64_t length, double* out, void* stream) {
  (void)n_cols;
  AS_REQUIRE(length >= 0, AS_ERR_SHAPE, "negative diagonal length");
  const long long row0 = k < 0 ? -k : 0, col0 = k >= 0 ? k : 0;
  AS_REQUIRE(row0 + length <= n_rows && col0 + length <= n_cols, AS_ERR_SHAPE, "diagonal %lld outside matrix",
             (long long)k);
  if (length > 0) {
    diag_kernel<<<grid_for(length, kFThreads), kFThreads, 0, S(stream)>>>(length, row0, col0, col_ptr, row_idx, vals,
                                                                          out);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

int as_scale_by_label_f64(int64_t nnz, const int32_t* labels, const double* vals, const double* norms, double* out,
                          void* stream) {
  AS_REQUIRE(nnz >= 0, AS_ERR_SHAPE, "negative length");
  if (nnz > 0) {
    scale_by_label_kernel<<<grid_for(nnz, kFThreads), kFThreads, 0, S(stream)>>>(nnz, labels, vals, norms, out);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

}  // extern "C"
