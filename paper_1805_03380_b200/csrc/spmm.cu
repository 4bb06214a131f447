// spmm.cu -- sparse x dense products over the CSR (= cached transpose) of A.
//
//   C = A @ B, B column-major (n_cols x k), C column-major (n_rows x k).
// Reference: _kernels.mat_times_vec (_kernels.py:118-127) is the k = 1 case;
// SURVEY 3.3 defines k > 1 as k independent calls.  _kernels.vec_times_mat
// (_kernels.py:106-115) is the row-vector product over the CSC itself.
//
// B200 design (row split, dense operand chunked to stay L2-resident):
//  * the k dense columns are processed in chunks of KC (16 f32 / 8 f64 = 64 B
//    per row); each chunk of B is first transposed into a row-major scratch
//    Bt[n_cols][KC] (coalesced column reads, 64-byte row writes) that stays
//    resident in the 126 MB L2 while A streams past it;
//  * one thread per output row walks its CSR row in column order and gathers
//    whole 64-byte Bt rows with 128-bit loads, so every L2 sector fetched is
//    fully used;
//  * the C chunk is written column by column, 32 consecutive rows per warp
//    store (128-byte coalesced).
// Exact mode mirrors the reference's arithmetic: float64 accumulator, product
// and sum separately rounded, columns with B[j,c] == 0 skipped, contributions
// in ascending column order -- bit-identical to mat_times_vec for float64.
#include "capi_util.cuh"
#include "common.cuh"

namespace as {

constexpr int kMmThreads = 256;
#ifndef AS_SPMM_KC
#define AS_SPMM_KC 16
#endif

// L2 eviction-priority policy for the dense chunk: written by the transpose
// and gathered ~nnz/n_cols times by the row kernel, it must outlive the
// streams of A and C passing through L2 (evict_first / streaming hints).
AS_DEVICE_INLINE unsigned long long l2_keep_policy() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
AS_DEVICE_INLINE void st_keep(float* p, float4 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
AS_DEVICE_INLINE void st_keep(double* p, double2 v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
AS_DEVICE_INLINE float4 ld_keep(const float* p, unsigned long long pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
AS_DEVICE_INLINE double2 ld_keep(const double* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

template <class T, int KC>
__global__ void __launch_bounds__(kMmThreads)
dense_chunk_transpose_kernel(long long n, const T* __restrict__ B, long long ldb, int kc, T* __restrict__ Bt) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  T v[KC];
#pragma unroll
  for (int c = 0; c < KC; c++) v[c] = c < kc ? __ldcs(&B[j + (long long)c * ldb]) : T(0);
  T* dst = Bt + j * KC;
  constexpr int kVec = 16 / sizeof(T);
  const unsigned long long pol = l2_keep_policy();
#pragma unroll
  for (int c = 0; c < KC; c += kVec) {
    if constexpr (sizeof(T) == 4) st_keep(dst + c, make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]), pol);
    else st_keep(dst + c, make_double2(v[c], v[c + 1]), pol);
  }
}

AS_DEVICE_INLINE float fma_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }
AS_DEVICE_INLINE double fma_t(double a, double b, double c) { return __fma_rn(a, b, c); }

template <class T>
AS_DEVICE_INLINE void load_row16B(const T* p, T* out);

template <>
AS_DEVICE_INLINE void load_row16B<float>(const float* p, float* out) {
  float4 q = __ldg(reinterpret_cast<const float4*>(p));
  out[0] = q.x;
  out[1] = q.y;
  out[2] = q.z;
  out[3] = q.w;
}
template <>
AS_DEVICE_INLINE void load_row16B<double>(const double* p, double* out) {
  double2 q = __ldg(reinterpret_cast<const double2*>(p));
  out[0] = q.x;
  out[1] = q.y;
}

// one thread per output row; KC dense columns from the row-major chunk Bt
template <class T, int KC, bool kExact>
__global__ void __launch_bounds__(kMmThreads)
spmm_rows_kernel(long long n_rows, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                 const T* __restrict__ vals, const T* __restrict__ Bt, int kc, T* __restrict__ C, long long ldc) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  using Acc = typename std::conditional<kExact, double, T>::type;
  Acc acc[KC];
#pragma unroll
  for (int c = 0; c < KC; c++) acc[c] = Acc(0);
  const int beg = row_ptr[r], end = row_ptr[r + 1];
  constexpr int kVec = 16 / sizeof(T);
  int k = beg;
  for (; k + 1 < end; k += 2) {  // two entries in flight
    const int j0 = __ldcs(&col_idx[k]), j1 = __ldcs(&col_idx[k + 1]);
    const T v0 = __ldcs(&vals[k]), v1 = __ldcs(&vals[k + 1]);
    T b0[KC], b1[KC];
#pragma unroll
    for (int c = 0; c < KC; c += kVec) {
      load_row16B<T>(Bt + (long long)j0 * KC + c, b0 + c);
      load_row16B<T>(Bt + (long long)j1 * KC + c, b1 + c);
    }
#pragma unroll
    for (int c = 0; c < KC; c++) {
      if (kExact) {
        if (b0[c] != T(0)) acc[c] = __dadd_rn(acc[c], __dmul_rn((double)v0, (double)b0[c]));
        if (b1[c] != T(0)) acc[c] = __dadd_rn(acc[c], __dmul_rn((double)v1, (double)b1[c]));
      } else {
        acc[c] = fma_t(v0, b0[c], acc[c]);
        acc[c] = fma_t(v1, b1[c], acc[c]);
      }
    }
  }
  if (k < end) {
    const int j0 = __ldcs(&col_idx[k]);
    const T v0 = __ldcs(&vals[k]);
    T b0[KC];
#pragma unroll
    for (int c = 0; c < KC; c += kVec) load_row16B<T>(Bt + (long long)j0 * KC + c, b0 + c);
#pragma unroll
    for (int c = 0; c < KC; c++) {
      if (kExact) {
        if (b0[c] != T(0)) acc[c] = __dadd_rn(acc[c], __dmul_rn((double)v0, (double)b0[c]));
      } else {
        acc[c] = fma_t(v0, b0[c], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < KC; c++)
    if (c < kc) __stcs(&C[r + (long long)c * ldc], (T)acc[c]);
}

// kL = 4 lanes per output row, each owning 16 bytes (4 f32 / 2 f64) of the
// KC-wide chunk: one 128-bit gather per lane and entry, a whole 64-byte Bt
// row per lane group; 8 rows per warp.  Few registers -> full occupancy and
// many independent gathers in flight.  Entries are folded in CSR (column)
// order, so exact mode keeps the reference's per-element order.
template <class T, int KC, bool kExact>
__global__ void __launch_bounds__(kMmThreads)
spmm_rows_lanes_kernel(long long n_rows, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                       const T* __restrict__ vals, const T* __restrict__ Bt, int kc, T* __restrict__ C, long long ldc) {
  constexpr int kVec = 16 / sizeof(T);
  constexpr int kL = KC / kVec;
  static_assert(32 % kL == 0, "lane groups must tile a warp");
  using Acc = typename std::conditional<kExact, double, T>::type;
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long r = gt / kL;
  const int sub = (int)(gt % kL);
  if (r >= n_rows) return;
  const unsigned long long pol = l2_keep_policy();
  Acc acc[kVec];
#pragma unroll
  for (int c = 0; c < kVec; c++) acc[c] = Acc(0);
  const T* bt = Bt + sub * kVec;
  auto fold = [&](T v, const V& b) {
    const T* bb = reinterpret_cast<const T*>(&b);
#pragma unroll
    for (int c = 0; c < kVec; c++) {
      if (kExact) {
        if (bb[c] != T(0)) acc[c] = __dadd_rn(acc[c], __dmul_rn((double)v, (double)bb[c]));
      } else {
        acc[c] = fma_t(v, bb[c], acc[c]);
      }
    }
  };
  const int beg = __ldg(&row_ptr[r]), end = __ldg(&row_ptr[r + 1]);
  // batches of kB entries: all indices, then all gathers (predicated), then
  // the folds in entry order -- two dependent round trips per batch
#ifndef AS_SPMM_KB
#define AS_SPMM_KB 8
#endif
  constexpr int kB = AS_SPMM_KB;
  for (int k = beg; k < end; k += kB) {
    int j[kB];
    T v[kB];
#pragma unroll
    for (int u = 0; u < kB; u++) {
      j[u] = k + u < end ? __ldcs(&col_idx[k + u]) : -1;
      v[u] = k + u < end ? __ldcs(&vals[k + u]) : T(0);
    }
    V b[kB];
#pragma unroll
    for (int u = 0; u < kB; u++)
      if (j[u] >= 0) b[u] = ld_keep(bt + (long long)j[u] * KC, pol);
#pragma unroll
    for (int u = 0; u < kB; u++)
      if (j[u] >= 0) fold(v[u], b[u]);
  }
#pragma unroll
  for (int c = 0; c < kVec; c++) {
    const int col = sub * kVec + c;
    if (col < kc) __stcs(&C[r + (long long)col * ldc], (T)acc[c]);
  }
}

// k == 1 exact: y = A x as a per-row left fold (mat_times_vec, bit-exact)
template <class T>
__global__ void __launch_bounds__(kMmThreads)
spmv_rows_exact_kernel(long long n_rows, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
                       const T* __restrict__ vals, const T* __restrict__ x, T* __restrict__ y) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  double acc = 0.0;
  const int beg = row_ptr[r], end = row_ptr[r + 1];
  for (int k = beg; k < end; k++) {
    const double xj = (double)__ldg(&x[col_idx[k]]);
    if (xj != 0.0) acc = __dadd_rn(acc, __dmul_rn((double)vals[k], xj));
  }
  y[r] = (T)acc;
}

// w = v^T A over the CSC: w[j] = left fold of v[row] * val in column order
// (_kernels.vec_times_mat, _kernels.py:106-115); one warp per 32 columns,
// one thread per column.
__global__ void __launch_bounds__(kMmThreads)
vecmat_csc_kernel(long long n_cols, const int* __restrict__ col_ptr, const int* __restrict__ row_idx,
                  const double* __restrict__ vals, const double* __restrict__ v, double* __restrict__ w) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_cols) return;
  double s = 0.0;
  for (int k = col_ptr[j]; k < col_ptr[j + 1]; k++) s = __dadd_rn(s, __dmul_rn(__ldg(&v[row_idx[k]]), vals[k]));
  w[j] = s;
}

template <class T, int KC, bool kExact>
static int spmm_impl(long long n_rows, long long n_cols, long long k, const int* row_ptr, const int* col_idx,
                     const T* vals, const T* B, long long ldb, T* C, long long ldc, T* Bt, cudaStream_t st) {
  constexpr int kL = KC / (16 / sizeof(T));
  const long long blocks_r = (n_rows * kL + kMmThreads - 1) / kMmThreads;
  const int blocks_c = (int)((n_cols + kMmThreads - 1) / kMmThreads);
  for (long long k0 = 0; k0 < k; k0 += KC) {
    const int kc = (int)min((long long)KC, k - k0);
    if (n_cols > 0) {
      dense_chunk_transpose_kernel<T, KC><<<blocks_c, kMmThreads, 0, st>>>(n_cols, B + k0 * ldb, ldb, kc, Bt);
      AS_LAUNCH_CHECK();
    }
    if (n_rows > 0) {
      spmm_rows_lanes_kernel<T, KC, kExact><<<(unsigned)blocks_r, kMmThreads, 0, st>>>(n_rows, row_ptr, col_idx,
                                                                                      vals, Bt, kc, C + k0 * ldc, ldc);
      AS_LAUNCH_CHECK();
    }
  }
  return AS_OK;
}

// ---------------------------------------------------------------------------
// Column-merge SpMM straight over the CSC (no CSR, no transpose): the
// reference's own loop order (_kernels.mat_times_vec, _kernels.py:118-127:
// for each column c, y[row] += val * x[c]) done for KC = 16 dense columns at
// a time.  The nonzeros are cut into fixed tiles of kCmE consecutive entries
// (a merge of col_ptr and the entry range: a heavy column spans several
// tiles, light columns share one).  Per tile, one elected thread moves the
// tile's B rows -- B[cb .. ce, j0 .. j0 + 15], 16 contiguous runs of the
// column-major B -- and its row indices / values into shared memory with bulk
// copies (the TMA engine, completion on one mbarrier); every entry's column
// comes from expanding the tile's column pointers.  Each entry's
// contribution val * B[c, j0 .. j0 + 15] is added into a row-major scratch
// Ct[n_rows][16] (64 MB at 1e6 rows: L2-resident) by 4 lanes with one
// red.global.add.v4.f32 each; a second kernel moves Ct into C's columns and
// re-zeroes it for the next chunk.  Float32 only, additions in arrival order
// (the tolerance of the float32 path, 1e-5); exact mode and float64 use the
// CSR route.  Measured (tools/micro/l2_red.cu, B200): random 64-byte row
// red.v4 8.6e10 rows/s into a 64 MB footprint vs 1.9e11 rows/s for plain
// 64-byte gathers -- slower per row than the row split's gathers, but it
// needs no CSR, so it is the first product on a fresh CSC.
constexpr int kCmE = 2048;    // entries per tile
constexpr int kCmT = 256;     // threads: 64 lane groups of 4
constexpr int kCmSpan = 512;  // columns a tile may span with its B rows staged
constexpr int kCmSP = 548;    // largest staged row stride: round_up(kCmSpan + 6, 32) + 4

struct CmSmem {
  alignas(16) float b[16 * kCmSP];  // B[cbA + x, j0 + j] at b[j * SP + x]
  alignas(16) int rows[kCmE];
  alignas(16) float vals[kCmE];
  alignas(16) unsigned short col[kCmE];  // column of each entry - cb
  int ps[kCmSpan + 2];                    // ptr[cb .. ce + 1]
  unsigned scan[32];
  unsigned long long bar;
};

// tile_col[t] = column holding entry t * kCmE (t < T); tile_col[T] = column
// holding the last entry
static __global__ void cm_tile_col_kernel(const int* __restrict__ ptr, long long n_cols, long long nnz, long long T,
                                          unsigned* __restrict__ tile_col) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const long long b = __ldg(&ptr[c]), e = __ldg(&ptr[c + 1]);
  for (long long t = (b + kCmE - 1) / kCmE; t * kCmE < e; t++) tile_col[t] = (unsigned)c;
  if (b <= nnz - 1 && nnz - 1 < e) tile_col[T] = (unsigned)c;
}

AS_DEVICE_INLINE void red_add_v4(float* p, float a, float b, float c, float d, unsigned long long pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(pol)
               : "memory");
}
AS_DEVICE_INLINE void bulk_g2s_hint(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar,
                                    unsigned long long pol) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          d),
      "l"(gsrc), "r"(bytes), "r"(b), "l"(pol)
      : "memory");
}
// L2 policies of the column merge: the accumulator Ct (64 MB) must outlive
// the streams of A and B passing through L2 (round 2 without hints: 69 MB
// of Ct re-fetched and 104 MB written back per 16-column chunk)
AS_DEVICE_INLINE unsigned long long l2_policy(int kind) {
  unsigned long long p;
  if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Lane s of a group owns dense columns j = s, s + 4, s + 8, s + 12 (its four
// staged reads fall in distinct banks: the row stride is 4 mod 32) and adds
// them into Ct slots 4 s .. 4 s + 3 of the entry's row.
template <bool kBulk>
__global__ void __launch_bounds__(kCmT)
spmm_csc_merge_kernel(long long n_cols, long long nnz, long long T, const int* __restrict__ ptr,
                      const int* __restrict__ rows, const float* __restrict__ vals, const float* __restrict__ B,
                      long long ldb, int kc, const unsigned* __restrict__ tile_col, float* __restrict__ Ct,
                      int hints) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CmSmem& S = *reinterpret_cast<CmSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int g = tid >> 2, s = tid & 3;
  const long long t = blockIdx.x;
  const long long e0 = t * kCmE, e1 = min(nnz, e0 + kCmE);
  const int ne = (int)(e1 - e0);
  const long long cb = __ldg(&tile_col[t]);
  const long long ce = __ldg(&tile_col[t + 1 < T ? t + 1 : T]);
  float* ct = Ct + 4 * s;
  const unsigned long long keep = l2_policy(hints ? 2 : 0), stream = l2_policy(hints ? 1 : 0);
  if (ce - cb + 1 > kCmSpan) {  // hypersparse range: columns by search, B from global memory
    for (int i = g; i < ne; i += kCmT / 4) {
      const long long e = e0 + i;
      long long lo = cb, hi = ce;  // last c in [cb, ce] with ptr[c] <= e
      while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (__ldg(&ptr[mid]) <= e) lo = mid;
        else hi = mid - 1;
      }
      const int r = __ldg(&rows[e]);
      const float a = __ldg(&vals[e]);
      float b[4];
#pragma unroll
      for (int u = 0; u < 4; u++) b[u] = s + 4 * u < kc ? __ldg(&B[lo + (long long)(s + 4 * u) * ldb]) : 0.f;
      red_add_v4(ct + (long long)r * 16, a * b[0], a * b[1], a * b[2], a * b[3], keep);
    }
    return;
  }
  const long long cbA = cb & ~3ll;
  const int width = (int)((ce + 1 - cbA + 3) & ~3ll);
  const int SP = ((width + 31) & ~31) + 4;
  if (kBulk) {
    if (tid == 0) {
      mbar_init(&S.bar, 1);
      const unsigned eb = (unsigned)(ne * 4) & ~15u;
      mbar_expect_tx(&S.bar, (unsigned)(kc * width * 4) + 2u * eb);
      for (int j = 0; j < kc; j++) bulk_g2s_hint(S.b + j * SP, B + (long long)j * ldb + cbA, width * 4, &S.bar, stream);
      if (eb) {
        bulk_g2s_hint(S.rows, rows + e0, eb, &S.bar, stream);
        bulk_g2s_hint(S.vals, vals + e0, eb, &S.bar, stream);
      }
    }
    for (int i = (ne & ~3) + tid; i < ne; i += kCmT) {
      S.rows[i] = __ldg(&rows[e0 + i]);
      S.vals[i] = __ldg(&vals[e0 + i]);
    }
  } else {
    for (int q = tid; q < kc * width; q += kCmT) {
      const int j = q / width, x = q - j * width;
      S.b[j * SP + x] = cbA + x < n_cols ? __ldg(&B[(long long)j * ldb + cbA + x]) : 0.f;
    }
    for (int i = tid; i < ne; i += kCmT) {
      S.rows[i] = __ldg(&rows[e0 + i]);
      S.vals[i] = __ldg(&vals[e0 + i]);
    }
  }
  // every entry's column: the tile's column pointers, a mark at the start of
  // every non-empty column (relative to cb; distinct starts, no atomics),
  // then a block max-scan over the tile's positions
  const int span = (int)(ce - cb) + 1;
  for (int c = tid; c <= span; c += kCmT) S.ps[c] = __ldg(&ptr[cb + c]);
  reinterpret_cast<uint4*>(S.col)[tid] = make_uint4(0u, 0u, 0u, 0u);  // kCmE / 8 = kCmT
  __syncthreads();
  for (int c = 1 + tid; c < span; c += kCmT) {
    const long long p = (long long)S.ps[c] - e0;
    if (p < ne && S.ps[c + 1] > S.ps[c]) S.col[p] = (unsigned short)c;
  }
  __syncthreads();
  {
    uint4 q = reinterpret_cast<const uint4*>(S.col)[tid];
    unsigned w[4] = {q.x, q.y, q.z, q.w}, m = 0;
#pragma unroll
    for (int u = 0; u < 4; u++) m = max(m, max(w[u] & 0xffffu, w[u] >> 16));
    unsigned run = block_exclusive_max(m, S.scan);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const unsigned lo = max(run, w[u] & 0xffffu);
      run = max(lo, w[u] >> 16);
      w[u] = lo | (run << 16);
    }
    reinterpret_cast<uint4*>(S.col)[tid] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  __syncthreads();
  if (kBulk) mbar_wait(&S.bar, 0);
  const float* bs = S.b + s * SP;
  const int cb_off = (int)(cb - cbA);
#pragma unroll 4
  for (int i = g; i < ne; i += kCmT / 4) {
    const int r = S.rows[i];
    const float a = S.vals[i];
    const int x = S.col[i] + cb_off;
    red_add_v4(ct + (long long)r * 16, a * bs[x], a * bs[x + 4 * SP], a * bs[x + 8 * SP], a * bs[x + 12 * SP],
               keep);
  }
}

// C[r, j0 + j] = Ct[r][4 (j % 4) + j / 4] for j < kc (4 lanes per row, one
// 16-byte load each), then the row is re-zeroed for the next chunk
__global__ void __launch_bounds__(kMmThreads)
cm_ct_to_c_kernel(long long n_rows, float* __restrict__ Ct, int kc, bool rezero, float* __restrict__ C, long long ldc,
                  int hints) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long r = gt >> 2;
  const int s = (int)(gt & 3);
  if (r >= n_rows) return;
  float4* p = reinterpret_cast<float4*>(Ct + r * 16 + 4 * s);
  const float4 q = __ldcg(p);
  const float v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int j = s + 4 * u;
    if (j < kc) __stcs(&C[r + (long long)j * ldc], v[u]);
  }
  if (rezero) {
    const unsigned long long keep = l2_policy(hints ? 2 : 0);
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(p), "f"(0.f), "l"(keep) : "memory");
  }
}

static size_t cm_ws_bytes(long long n_rows, long long nnz) {
  const long long T = (nnz + kCmE - 1) / kCmE;
  return (size_t)std::max(1ll, n_rows) * 64 + (size_t)(T + 2) * 4 + 256;
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_spmm_workspace_bytes(int64_t n_cols, int64_t k, int dtype_bytes) {
  // one row-major chunk of B: n_cols x 64 bytes
  (void)k;
  (void)dtype_bytes;
  return (size_t)(n_cols > 0 ? n_cols : 1) * (AS_SPMM_KC * 4 > 64 ? AS_SPMM_KC * 4 : 64) + 256;
}

int as_spmm_csr_f32(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t* row_ptr, const int32_t* col_idx,
                    const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc, int exact, void* ws,
                    size_t ws_bytes, void* stream) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && k >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(ldb >= n_cols && ldc >= n_rows, AS_ERR_ARG, "leading dimension too small");
  AS_REQUIRE(ws_bytes >= as_spmm_workspace_bytes(n_cols, k, 4), AS_ERR_ARG, "workspace too small");
  cudaStream_t st = S(stream);
  if (k == 1 && exact) {
    if (n_rows > 0)
      spmv_rows_exact_kernel<float><<<(unsigned)((n_rows + kMmThreads - 1) / kMmThreads), kMmThreads, 0, st>>>(
          n_rows, row_ptr, col_idx, vals, B, C);
    AS_LAUNCH_CHECK();
    return AS_OK;
  }
  if (exact) return spmm_impl<float, AS_SPMM_KC, true>(n_rows, n_cols, k, row_ptr, col_idx, vals, B, ldb, C, ldc, (float*)ws, st);
  return spmm_impl<float, AS_SPMM_KC, false>(n_rows, n_cols, k, row_ptr, col_idx, vals, B, ldb, C, ldc, (float*)ws, st);
}

int as_spmm_csr_f64(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t* row_ptr, const int32_t* col_idx,
                    const double* vals, const double* B, int64_t ldb, double* C, int64_t ldc, void* ws,
                    size_t ws_bytes, void* stream) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && k >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(ldb >= n_cols && ldc >= n_rows, AS_ERR_ARG, "leading dimension too small");
  AS_REQUIRE(ws_bytes >= as_spmm_workspace_bytes(n_cols, k, 8), AS_ERR_ARG, "workspace too small");
  cudaStream_t st = S(stream);
  if (k == 1) {
    if (n_rows > 0)
      spmv_rows_exact_kernel<double><<<(unsigned)((n_rows + kMmThreads - 1) / kMmThreads), kMmThreads, 0, st>>>(
          n_rows, row_ptr, col_idx, vals, B, C);
    AS_LAUNCH_CHECK();
    return AS_OK;
  }
  return spmm_impl<double, 8, true>(n_rows, n_cols, k, row_ptr, col_idx, vals, B, ldb, C, ldc, (double*)ws, st);
}

size_t as_spmm_csc_workspace_bytes(int64_t n_rows, int64_t nnz) { return cm_ws_bytes(n_rows, nnz); }

int as_spmm_csc_f32(int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t k, const int32_t* col_ptr,
                    const int32_t* row_idx, const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc,
                    void* ws, size_t ws_bytes, void* stream) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && k >= 0 && nnz >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(ldb >= n_cols && ldc >= n_rows, AS_ERR_ARG, "leading dimension too small");
  AS_REQUIRE(ws_bytes >= cm_ws_bytes(n_rows, nnz), AS_ERR_ARG, "workspace too small");
  AS_REQUIRE(n_rows <= (1ll << 40) && nnz < (1ll << 31), AS_ERR_ARG, "matrix too large");
  cudaStream_t st = S(stream);
  if (n_rows == 0 || k == 0) return AS_OK;
  if (nnz == 0 || n_cols == 0) {
    AS_CUDA_TRY(cudaMemset2DAsync(C, (size_t)ldc * 4, 0, (size_t)n_rows * 4, (size_t)k, st));
    return AS_OK;
  }
  float* Ct = (float*)ws;
  const long long T = (nnz + kCmE - 1) / kCmE;
  unsigned* tile_col = (unsigned*)((char*)ws + (size_t)n_rows * 64);
  cm_tile_col_kernel<<<(unsigned)((n_cols + kMmThreads - 1) / kMmThreads), kMmThreads, 0, st>>>(col_ptr, n_cols, nnz,
                                                                                                 T, tile_col);
  AS_LAUNCH_CHECK();
  AS_CUDA_TRY(cudaMemsetAsync(Ct, 0, (size_t)n_rows * 64, st));
  // bulk copies need 16-byte aligned runs of B: aligned base, ldb % 4 == 0
  // (then a run rounded out to 4 columns stays inside its column of B)
  const bool bulk = ((uintptr_t)B % 16 == 0) && (ldb % 4 == 0) && ((uintptr_t)row_idx % 16 == 0) &&
                    ((uintptr_t)vals % 16 == 0) && !getenv("AS_CM_NO_BULK");
  static std::atomic<bool> attr[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < kMaxDevices && !attr[dev]) {
    AS_CUDA_TRY(cudaFuncSetAttribute(spmm_csc_merge_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(CmSmem)));
    AS_CUDA_TRY(cudaFuncSetAttribute(spmm_csc_merge_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(CmSmem)));
    attr[dev] = true;
  }
  const unsigned blocks_b = (unsigned)((n_rows * 4 + kMmThreads - 1) / kMmThreads);
  static const int hints = getenv("AS_CM_NO_HINTS") ? 0 : 1;
  for (long long k0 = 0; k0 < k; k0 += 16) {
    const int kc = (int)std::min(16ll, k - k0);
    if (bulk)
      spmm_csc_merge_kernel<true><<<(unsigned)T, kCmT, sizeof(CmSmem), st>>>(n_cols, nnz, T, col_ptr, row_idx, vals,
                                                                             B + k0 * ldb, ldb, kc, tile_col, Ct, hints);
    else
      spmm_csc_merge_kernel<false><<<(unsigned)T, kCmT, sizeof(CmSmem), st>>>(n_cols, nnz, T, col_ptr, row_idx, vals,
                                                                              B + k0 * ldb, ldb, kc, tile_col, Ct, hints);
    AS_LAUNCH_CHECK();
    cm_ct_to_c_kernel<<<blocks_b, kMmThreads, 0, st>>>(n_rows, Ct, kc, k0 + 16 < k, C + k0 * ldc, ldc, hints);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

int as_vecmat_csc_f64(int64_t n_rows, int64_t n_cols, const int32_t* col_ptr, const int32_t* row_idx,
                      const double* vals, const double* v, double* w, void* stream) {
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0, AS_ERR_SHAPE, "negative dimension");
  if (n_cols > 0) {
    vecmat_csc_kernel<<<(unsigned)((n_cols + kMmThreads - 1) / kMmThreads), kMmThreads, 0, S(stream)>>>(
        n_cols, col_ptr, row_idx, vals, v, w);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}

}  // extern "C"
