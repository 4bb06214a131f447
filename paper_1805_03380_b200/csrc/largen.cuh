// largen.cuh -- the large-input pipeline behind COO->CSC construction
// (csc.canonicalize, csc.py:148-193) and the CSC transpose
// (_kernels.transpose, _kernels.py:130-150) for inputs beyond the
// single-launch kernel's envelope (sortreduce.cuh: n <= grid x 4096).
//
// Throughput-oriented: the elements are first put in bucket order by a
// stable LSD counting sort on the bucket id (a bucket = a range of
// consecutive output columns holding <= ~0.85 tile), one or two passes of
// 8-bit digits (fanout 256, so every (tile, digit) run is long and the
// scatter is coalesced), then every bucket is sorted and reduced in shared
// memory by the same tile phase as the single-launch kernel
// (sortreduce.cuh: tile_phase) with a chained decoupled look-back for the
// output offsets.
//
//   count   (per pass) tile t of 4096 elements: digit histogram -> H[d][t]
//   scan    exclusive scan of H (digit-major) -> every (digit, tile) run's
//           global offset; a second scan gives the bucket starts
//   scatter (per pass) the tile again: stable rank of each element among the
//           tile's elements of its digit (warp match_any + per-warp digit
//           counters, element order = input order), staged in shared memory
//           in digit order, written out run by run
//   tiles   bucket t = the contiguous slots [bstart[t], bstart[t+1]); the
//           slot order is the input order (both passes are stable), so the
//           slot breaks key ties exactly as the reference's stable lexsort.
//
// Pass A (two-pass case) writes (major, minor, value) records keyed by the
// low digit of the bucket id; pass B (or the only pass) writes the
// bucket-local 32-bit key (local column << minor_bits | minor) and the value.
#pragma once

#include "sortreduce.cuh"

namespace as {
namespace ln {

constexpr int kT = 256;          // threads of the count / scatter / finish CTAs
constexpr int kI = 8;            // elements per thread
constexpr int kE = kT * kI;      // elements per pipeline tile
constexpr int kR = 256;          // digit radix
constexpr int kW = kT / 32;      // warps
constexpr int kScanN = 4096;     // entries per scan tile (256 threads x 16)
constexpr int kJoinSpan = 2;     // low digits a pass-B tile may span for its bucket histogram (more: global atomics)

// element sources: major (output column), minor (output row), value
template <class IdxT, class T>
struct CooIn {
  const IdxT* rows;
  const IdxT* cols;
  const T* vals;
  long long n, n_rows, n_cols;
};

template <class T>
struct CscIn {  // the elements of a CSC visited by row: major = row, minor = column
  const int* ptr;
  const int* idx;
  const T* vals;
  long long n_cols, nnz;
  const unsigned* tile_col;  // [T + 1] column of each tile's first element (ln_tile_col_kernel)
};

// tile_col[t] = the column holding element t * kE (the last column with
// ptr[c] <= t * kE): every column writes the tiles whose first element it holds
static __global__ void ln_tile_col_kernel(const int* __restrict__ ptr, long long n_cols, long long nnz,
                                          unsigned* __restrict__ tile_col) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const long long b = __ldg(&ptr[c]), e = __ldg(&ptr[c + 1]);
  for (long long t = (b + kE - 1) / kE; t * kE < e; t++) tile_col[t] = (unsigned)c;
}

template <class T>
struct RecIn {  // pass A records
  const unsigned* maj;
  const unsigned* mn;
  const T* vals;
};

template <class T>
struct Args {
  long long n;                 // elements
  long long T_;                // pipeline tiles
  long long n_out_cols;
  int mb;                      // minor bits
  int lob;                     // low-digit bits (0: single pass)
  long long nb;                // buckets
  unsigned long long cb_mul;   // bucket(c) = (c * cb_mul) >> 32
  unsigned* H;                 // [kR x T] digit counts -> run offsets
  unsigned* bcnt;              // [nb + 1] bucket counts -> bucket starts
  const unsigned* cbcol;       // [nb + 1] first column of each bucket
  unsigned long long* bad;     // first invalid COO element (min), or ~0
  unsigned* aM;                // pass A records
  unsigned* aN;
  T* aV;
  unsigned* bK;                // pass B records (bucket order)
  T* bV;
  double inv_cb;               // 1.0 / cb_mul (local_col)
};

AS_DEVICE_INLINE unsigned bucket_of(unsigned maj, unsigned long long cb_mul) {
  return (unsigned)(((unsigned long long)maj * cb_mul) >> 32);
}

// column of maj inside its bucket: maj - cbcol[bucket_of(maj)] = floor(f / cb_mul)
// with f = maj * cb_mul mod 2^32 (moving d columns down stays in the bucket
// while d * cb_mul <= f).  The quotient comes from a double reciprocal
// (relative error ~2^-52, so it is off by at most one) and one exact integer
// correction -- no 32-bit division (which was a sixth of the scatter's
// instructions).
AS_DEVICE_INLINE unsigned local_col(unsigned maj, unsigned long long cb_mul, double inv_cb) {
  if (cb_mul >> 32) return 0u;  // one column per bucket
  const unsigned f = (unsigned)((unsigned long long)maj * cb_mul);
  unsigned q = (unsigned)((double)f * inv_cb);
  const unsigned long long d = cb_mul;
  if ((unsigned long long)q * d > f) q--;
  else if ((unsigned long long)(q + 1) * d <= f) q++;
  return q;
}

// ---- items: every element of a thread is loaded first (all loads in
// flight together), then decoded.  Item k of a thread is element
// t * kE + warp * 32 kI + 32 k + lane: warp-blocked and lane-consecutive, so
// (warp, item, lane) order is the input order and every load is coalesced.
AS_DEVICE_INLINE long long elem_of(long long t, int k) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  return t * kE + (long long)warp * (32 * kI) + k * 32 + lane;
}

// upper_bound(ptr[0..N), x) by the whole block (any block size): one sample
// per thread per round, __syncthreads_count of the samples <= x
__device__ inline long long blk_upper_bound(const int* ptr, long long N, long long x) {
  const long long nt = blockDim.x;
  long long base = 0, len = N;
  while (len > nt) {
    const long long step = (len + nt - 1) / nt;
    const long long j = (long long)threadIdx.x * step;
    const int c = __syncthreads_count(j < len && __ldg(&ptr[base + j]) <= x);
    if (c == 0) return base;
    base += (long long)(c - 1) * step + 1;
    len = min(step - 1, N - base);
    if (len <= 0) return base;
  }
  const int c = __syncthreads_count((long long)threadIdx.x < len && __ldg(&ptr[base + threadIdx.x]) <= x);
  return base + c;
}

// CSC visited by row: the tile's column pointers cached in shared memory
// (colc[0..nc] = ptr[cb..cb+nc]) when they fit, else global searches
struct ColCache {
  long long cb;
  int nc;  // cached entries - 1, or -1 when not cached
};

template <class T, class In>
struct Items;

template <class T, class IdxT>
struct Items<T, CooIn<IdxT, T>> {
  IdxT r[kI], c[kI];
  T v[kI];
  __device__ void prep(const CooIn<IdxT, T>&, long long, long long, int*, ColCache*) {}
  template <bool kVal>
  AS_DEVICE_INLINE void fetch(const CooIn<IdxT, T>& s, int k, long long e) {
    r[k] = __ldcs(&s.rows[e]);
    c[k] = __ldcs(&s.cols[e]);
    if (kVal) v[k] = __ldcs(&s.vals[e]);
  }
  // false: an out-of-range triplet (skipped; its index goes to *bad).  int32
  // indices compare unsigned (a negative index wraps above any dimension)
  AS_DEVICE_INLINE bool major(const CooIn<IdxT, T>& s, int k, long long e, unsigned& maj, unsigned long long* bad) {
    bool ok;
    if constexpr (sizeof(IdxT) == 4) {
      ok = (unsigned)r[k] < (unsigned)s.n_rows && (unsigned)c[k] < (unsigned)s.n_cols;
    } else {
      ok = (unsigned long long)r[k] < (unsigned long long)s.n_rows &&
           (unsigned long long)c[k] < (unsigned long long)s.n_cols;
    }
    if (!ok) {
      if (bad) atomicMin(bad, (unsigned long long)e);
      return false;
    }
    maj = (unsigned)c[k];
    return true;
  }
  AS_DEVICE_INLINE unsigned maj_raw(int k) const { return (unsigned)c[k]; }  // (already validated)
  AS_DEVICE_INLINE unsigned minor(const CooIn<IdxT, T>&, int k, long long, const ColCache&, const int*) {
    return (unsigned)r[k];
  }
};

template <class T>
struct Items<T, CscIn<T>> {
  int i[kI];
  T v[kI];
  long long cur = -1;  // column of this thread's previous element (its elements come in increasing order)
  __device__ void prep(const CscIn<T>& s, long long lo, long long hi, int* colc, ColCache* cc) {
    // the columns holding the tile's first / last element (tile_col: one
    // search per tile boundary, done once for all tiles by ln_tile_col_kernel)
    const long long t = lo / kE;
    const long long cb = __ldg(&s.tile_col[t]);
    const long long ce = hi < s.nnz ? __ldg(&s.tile_col[t + 1]) : s.n_cols - 1;
    const bool cached = ce - cb + 1 <= sr::kColCache;
    if (cached)
      for (long long c = cb + threadIdx.x; c <= ce + 1 && c <= s.n_cols; c += blockDim.x) colc[c - cb] = __ldg(&s.ptr[c]);
    if (threadIdx.x == 0) *cc = ColCache{cb, cached ? (int)(ce - cb) : -1};
    __syncthreads();
  }
  template <bool kVal>
  AS_DEVICE_INLINE void fetch(const CscIn<T>& s, int k, long long e) {
    i[k] = __ldcs(&s.idx[e]);
    if (kVal) v[k] = __ldcs(&s.vals[e]);
  }
  AS_DEVICE_INLINE bool major(const CscIn<T>&, int k, long long, unsigned& maj, unsigned long long*) {
    maj = (unsigned)i[k];
    return true;
  }
  AS_DEVICE_INLINE unsigned maj_raw(int k) const { return (unsigned)i[k]; }
  AS_DEVICE_INLINE unsigned minor(const CscIn<T>& s, int, long long e, const ColCache& cc, const int* colc) {
    if (cur < 0) {  // first element: binary search
      if (cc.nc >= 0) {
        int l = 0, h = cc.nc;  // last l with colc[l] <= e
        while (l < h) {
          const int mid = (l + h + 1) >> 1;
          if (colc[mid] <= e) l = mid;
          else h = mid - 1;
        }
        cur = cc.cb + l;
      } else {
        cur = upper_bound_dev(s.ptr, s.n_cols + 1, (int)e) - 1;
      }
    } else if (cc.nc >= 0) {  // advance (32 elements on: a few columns at most)
      while (colc[cur + 1 - cc.cb] <= e) cur++;
    } else {
      while (__ldg(&s.ptr[cur + 1]) <= e) cur++;
    }
    return (unsigned)cur;
  }
};

template <class T>
struct Items<T, RecIn<T>> {
  unsigned m[kI], n[kI];
  T v[kI];
  __device__ void prep(const RecIn<T>&, long long, long long, int*, ColCache*) {}
  template <bool kVal>
  AS_DEVICE_INLINE void fetch(const RecIn<T>& s, int k, long long e) {
    m[k] = __ldcs(&s.maj[e]);
    if (kVal) {
      n[k] = __ldcs(&s.mn[e]);
      v[k] = __ldcs(&s.vals[e]);
    }
  }
  AS_DEVICE_INLINE bool major(const RecIn<T>&, int k, long long, unsigned& maj, unsigned long long*) {
    maj = m[k];
    return true;
  }
  AS_DEVICE_INLINE unsigned maj_raw(int k) const { return m[k]; }
  AS_DEVICE_INLINE unsigned minor(const RecIn<T>&, int k, long long, const ColCache&, const int*) { return n[k]; }
};

// kind of a pass: 0 = pass A (digit = low bits, writes records A),
// 1 = pass B from records A (digit = high bits), 2 = single pass (digit = bucket)
template <int kPass>
AS_DEVICE_INLINE unsigned digit_of(unsigned b, int lob) {
  if (kPass == 0) return b & ((1u << lob) - 1u);
  if (kPass == 1) return b >> lob;
  return b;
}

// ------------------------------------------------------------------------
// count: digit histogram of tile t -> H[d * T + t]; pass 1 / 2 also add the
// tile's bucket counts into bcnt
template <class T, class In, int kPass>
__global__ void __launch_bounds__(kT) ln_count_kernel(Args<T> a, In src) {
  __shared__ unsigned h[kR];
  __shared__ unsigned jb[kPass == 1 ? kJoinSpan * kR : 1];
  __shared__ unsigned lo0s;
  const int tid = threadIdx.x;
  const long long t = blockIdx.x;
  const long long lo = t * kE, hi = min(a.n, lo + kE);
  for (int i = tid; i < kR; i += kT) h[i] = 0u;
  if constexpr (kPass == 1) {
    for (int i = tid; i < kJoinSpan * kR; i += kT) jb[i] = 0u;
    if (tid == 0) lo0s = bucket_of(__ldg(&src.maj[lo]), a.cb_mul) & ((1u << a.lob) - 1u);
  }
  Items<T, In> it;
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const long long e = elem_of(t, k);
    if (e < hi) it.template fetch<false>(src, k, e);
  }
  __syncthreads();
  const unsigned lo0 = kPass == 1 ? lo0s : 0u;
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const long long e = elem_of(t, k);
    unsigned maj;
    if (e >= hi || !it.major(src, k, e, maj, kPass != 1 ? a.bad : nullptr)) continue;
    const unsigned b = bucket_of(maj, a.cb_mul);
    atomicAdd(&h[digit_of<kPass>(b, a.lob)], 1u);
    if constexpr (kPass == 1) {
      const unsigned lw = (b & ((1u << a.lob) - 1u)) - lo0;
      if (lw < (unsigned)kJoinSpan) atomicAdd(&jb[lw * kR + (b >> a.lob)], 1u);
      else atomicAdd(&a.bcnt[b], 1u);
    }
  }
  __syncthreads();
  const int R = kPass == 0 ? (1 << a.lob) : kR;
  for (int d = tid; d < R; d += kT) {
    a.H[(long long)d * a.T_ + t] = h[d];
    if (kPass == 2 && h[d]) atomicAdd(&a.bcnt[d], h[d]);
  }
  if constexpr (kPass == 1) {
    for (int i = tid; i < kJoinSpan * kR; i += kT) {
      if (jb[i]) {
        const unsigned b = ((unsigned)(i % kR) << a.lob) | (lo0 + (unsigned)(i / kR));
        if (b < (unsigned)a.nb) atomicAdd(&a.bcnt[b], jb[i]);
      }
    }
  }
}

// ------------------------------------------------------------------------
// in-place exclusive scan of n u32 counts (chained; states / ticket zeroed);
// out_total (optional) receives the grand total
constexpr int kScanT = 256;
static __global__ void __launch_bounds__(kScanT)
ln_scan_kernel(unsigned* x, long long n, unsigned* out_total, unsigned long long* states, unsigned* ticket) {
  __shared__ long long tmp[kScanT / 32 + 1];
  __shared__ long long s_tile;
  __shared__ unsigned long long s_prefix;
  __shared__ unsigned sx[kScanN + kScanN / 32];  // the tile, moved through shared memory (coalesced I/O)
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long t = s_tile;
  constexpr int kPer = kScanN / kScanT;
  const long long t0 = t * kScanN;
  auto pad = [](int i) { return i + (i >> 5); };
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int q = k * kScanT + threadIdx.x;
    sx[pad(q)] = t0 + q < n ? x[t0 + q] : 0u;
  }
  __syncthreads();
  unsigned v[kPer];
  long long sum = 0;
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    v[k] = sx[pad(threadIdx.x * kPer + k)];
    sum += v[k];
  }
  long long total;
  const long long off = block_exclusive_scan<long long>(sum, tmp, &total);
  if ((threadIdx.x >> 5) == 0) {
    const unsigned long long pre = tile_lookback_warp(states, t, (unsigned long long)total);
    if ((threadIdx.x & 31) == 0) s_prefix = pre;
  }
  __syncthreads();
  long long run = (long long)s_prefix + off;
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    sx[pad(threadIdx.x * kPer + k)] = (unsigned)run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const int q = k * kScanT + threadIdx.x;
    if (t0 + q < n) x[t0 + q] = sx[pad(q)];
  }
  if (t == gridDim.x - 1 && threadIdx.x == 0 && out_total) *out_total = (unsigned)((long long)s_prefix + total);
}

// ------------------------------------------------------------------------
// scatter: stable counting sort of tile t by digit into the pass's records
template <class T, class In, int kPass>
struct ScatterSmem {
  alignas(16) unsigned wc[kW][kR];  // per-warp digit counters -> per-warp offsets
  unsigned tstart[kR];      // tile-local digit starts
  unsigned gbase[kR];       // global start of the tile's run of each digit
  unsigned k1[kE];          // major (pass A) or bucket-local key
  unsigned k2[kPass == 0 ? kE : 1];  // minor (pass A only)
  T v[kE];
  unsigned char d[kE];
  long long scan[kT / 32 + 1];
  int colc[sr::kColCache + 1];
  ColCache cc;
};

#ifndef AS_LN_SCATTER_MINB
#define AS_LN_SCATTER_MINB 4
#endif
template <class T, class In, int kPass>
__global__ void __launch_bounds__(kT, AS_LN_SCATTER_MINB) ln_scatter_kernel(Args<T> a, In src) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScatterSmem<T, In, kPass>& S = *reinterpret_cast<ScatterSmem<T, In, kPass>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t = blockIdx.x;
  const long long lo = t * kE, hi = min(a.n, lo + kE);
  const int R = kPass == 0 ? (1 << a.lob) : kR;
  const unsigned gb = tid < R ? __ldcg(&a.H[(long long)tid * a.T_ + t]) : 0u;  // the tile's run offsets, early
  Items<T, In> it;
#pragma unroll
  for (int k = 0; k < kI; k++) {  // every load of the tile in flight first
    const long long e = elem_of(t, k);
    if (e < hi) it.template fetch<true>(src, k, e);
  }
  reinterpret_cast<uint4*>(S.wc[warp])[lane] = make_uint4(0u, 0u, 0u, 0u);  // 256 counters: 2 x 16 B per lane
  reinterpret_cast<uint4*>(S.wc[warp])[lane + 32] = make_uint4(0u, 0u, 0u, 0u);
  it.prep(src, lo, hi, S.colc, &S.cc);  // (CSC source: the tile's column pointers; syncs)
  __syncthreads();
  const ColCache cc = S.cc;
  unsigned dg[kI], rk[kI];
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const long long e = elem_of(t, k);
    unsigned maj = 0;
    const bool ok = e < hi && it.major(src, k, e, maj, nullptr);
    dg[k] = ok ? digit_of<kPass>(bucket_of(maj, a.cb_mul), a.lob) : 0xffffu;
  }
  // stable ranks: item by item (input order); the lanes of one digit by match
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const unsigned peers = __match_any_sync(0xffffffffu, dg[k]);
    const bool ok = dg[k] != 0xffffu;
    unsigned base = 0;
    if (ok) base = S.wc[warp][dg[k]];
    rk[k] = base + __popc(peers & lanemask_lt());
    __syncwarp();
    if (ok && (peers & lanemask_lt()) == 0u) S.wc[warp][dg[k]] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: offsets of the warps (in warp order), tile count, tile start
  unsigned cnt = 0;
  if (tid < kR) {
#pragma unroll
    for (int w = 0; w < kW; w++) {
      const unsigned c = S.wc[w][tid];
      S.wc[w][tid] = cnt;
      cnt += c;
    }
  }
  long long tot;
  const long long st = block_exclusive_scan<long long>(tid < kR ? (long long)cnt : 0ll, S.scan, &tot);
  if (tid < kR) {
    S.tstart[tid] = (unsigned)st;
    S.gbase[tid] = gb;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kI; k++) {
    if (dg[k] == 0xffffu) continue;
    const long long e = elem_of(t, k);
    const unsigned p = S.tstart[dg[k]] + S.wc[warp][dg[k]] + rk[k];
    const unsigned maj = it.maj_raw(k);
    const unsigned mn = it.minor(src, k, e, cc, S.colc);
    if (kPass == 0) {
      S.k1[p] = maj;
      S.k2[p] = mn;
    } else {
      S.k1[p] = (local_col(maj, a.cb_mul, a.inv_cb) << a.mb) | mn;
    }
    S.v[p] = it.v[k];
    S.d[p] = (unsigned char)dg[k];
  }
  __syncthreads();
  const unsigned m = (unsigned)tot;
  for (unsigned q = tid; q < m; q += kT) {
    const unsigned d = S.d[q];
    const unsigned gp = S.gbase[d] + (q - S.tstart[d]);
    if (kPass == 0) {
      a.aM[gp] = S.k1[q];
      a.aN[gp] = S.k2[q];
      a.aV[gp] = S.v[q];
    } else {
      a.bK[gp] = S.k1[q];
      a.bV[gp] = S.v[q];
    }
  }
}

// ------------------------------------------------------------------------
// tiles: bucket t = slots [bstart[t], bstart[t+1]) of the pass B records,
// split evenly over the CTA's threads; slot = input order; chained look-back
template <class T>
struct SegLN {
  static constexpr bool kContig = true;  // bucket t = slots [bstart[t], bstart[t+1])
  const unsigned* bstart;
  const unsigned* bK;
  const T* bV;
  const unsigned* cbcol;
  unsigned long long* tstate;
  __device__ __forceinline__ void seg(long long t, int tid, unsigned& len, unsigned& src) const {
    const unsigned s0 = __ldg(&bstart[t]), L = __ldg(&bstart[t + 1]) - s0;
    const unsigned per = (L + sr::kThreads - 1) / sr::kThreads;
    const unsigned o = (unsigned)tid * per;
    len = o < L ? min(per, L - o) : 0u;
    src = s0 + o;
  }
  __device__ __forceinline__ unsigned base(long long t) const { return __ldg(&bstart[t]); }
  __device__ __forceinline__ unsigned key(unsigned s) const { return __ldcs(&bK[s]); }
  __device__ __forceinline__ unsigned idx(unsigned s) const { return s; }
  __device__ __forceinline__ const T* val(unsigned s) const { return bV + s; }
  __device__ __forceinline__ unsigned col0(long long t) const { return __ldg(&cbcol[t]); }
  __device__ __forceinline__ unsigned long long prefix(long long t, unsigned long long kept) const {
    return tile_lookback_warp(tstate, t, kept);
  }
};

template <class T>
__global__ void __launch_bounds__(sr::kThreads, sr::kMinBlocks)
ln_tiles_kernel(SegLN<T> sg_, sr::TileOut<T> o_, long long nb, const unsigned long long* bad, long long n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SegLN<T> sg;
  __shared__ sr::TileOut<T> o;
  if (threadIdx.x == 0) {
    sg = sg_;
    o = o_;
  }
  __syncthreads();
  sr::TileSmem<T>& S = *reinterpret_cast<sr::TileSmem<T>*>(smem_raw);
  if (blockIdx.x == 0 && threadIdx.x == 0 && o.info) {
    const unsigned long long b = bad ? *bad : ~0ull;
    o.info[1] = b < (unsigned long long)n ? (long long)b : 0x7f7f7f7f7f7f7f7fll;
  }
  sr::tile_phase<T>(sg, o, S, blockIdx.x, gridDim.x, nb);
}

// Transpose finish, one CTA per bucket (no look-back): a transpose keeps
// every element, so bucket t's output is exactly the slots [bstart[t],
// bstart[t+1]); its rows' pointers are bstart[t] + a scan of the bucket's
// per-row counts, and each element's place in its row is its stable rank --
// the bucket's slots are in input (column-major) order, so the rank by arrival
// IS the column order the output needs.  No sort, no reduce, any bucket size
// (chunks of kE elements in order, running row cursors); a bucket that fits
// one chunk is staged in shared memory and written out coalesced.
template <class T>
struct FinishSmem {
  unsigned wc[kW][sr::kMaxW];  // per-warp row counters -> offsets within the chunk
  unsigned run[sr::kMaxW];     // row cursors (bucket-local output position)
  unsigned ctot[sr::kMaxW];    // the chunk's count of each row
  unsigned rk[kE];             // staged output rows
  T v[kE];                     // staged output values
  unsigned long long scan[kT / 32 + 1];
};

template <class T>
__global__ void __launch_bounds__(kT, 3)
ln_transpose_finish_kernel(long long nb, const unsigned* __restrict__ bstart, const unsigned* __restrict__ bK,
                           const T* __restrict__ bV, const unsigned* __restrict__ cbcol, int mb, long long n_out_cols,
                           int* __restrict__ col_ptr, int* __restrict__ row_idx, T* __restrict__ out_vals,
                           long long* info) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FinishSmem<T>& S = *reinterpret_cast<FinishSmem<T>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned mmask = mb >= 32 ? 0xffffffffu : ((1u << mb) - 1u);
  if (blockIdx.x == 0 && tid == 0) {
    const unsigned n = __ldg(&bstart[nb]);
    col_ptr[n_out_cols] = (int)n;
    if (info) info[0] = n;
  }
  for (long long t = blockIdx.x; t < nb; t += gridDim.x) {
    const unsigned s0 = __ldg(&bstart[t]), L = __ldg(&bstart[t + 1]) - s0;
    const unsigned c0 = __ldg(&cbcol[t]);
    const int W = (int)(__ldg(&cbcol[t + 1]) - c0);
    const bool one = L <= (unsigned)kE;
    // the first chunk's loads go out before anything waits
    unsigned key[kI];
    T v[kI];
#pragma unroll
    for (int k = 0; k < kI; k++) {
      const unsigned i = warp * (32 * kI) + k * 32 + lane;
      if (i < L) {
        key[k] = __ldcs(&bK[s0 + i]);
        v[k] = __ldcs(&bV[s0 + i]);
      }
    }
    __syncthreads();  // the previous bucket's shared memory is free
    if (one) {
      // one chunk (the common case): the per-warp ranks come first, and the
      // rows' totals from them -- no separate counting pass
      for (int l = lane; l < W; l += 32) S.wc[warp][l] = 0u;
      __syncwarp();
      unsigned rk[kI], lr[kI];
#pragma unroll
      for (int k = 0; k < kI; k++) {
        const bool in = warp * (32 * kI) + k * 32 + lane < L;
        lr[k] = in ? key[k] >> mb : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, lr[k]);
        unsigned b0 = 0;
        if (in) b0 = S.wc[warp][lr[k]];
        rk[k] = b0 + __popc(peers & lanemask_lt());
        __syncwarp();
        if (in && (peers & lanemask_lt()) == 0u) S.wc[warp][lr[k]] = b0 + __popc(peers);
        __syncwarp();
      }
      __syncthreads();
      for (int l = tid; l < W; l += kT) {  // per row: warp offsets (warp order), total
        unsigned run = 0;
#pragma unroll
        for (int w = 0; w < kW; w++) {
          const unsigned c = S.wc[w][l];
          S.wc[w][l] = run;
          run += c;
        }
        S.run[l] = run;
      }
      __syncthreads();
      {
        constexpr int kPerT = (sr::kMaxW + kT - 1) / kT;
        unsigned c[kPerT], sum = 0;
#pragma unroll
        for (int q = 0; q < kPerT; q++) {
          const int l = tid * kPerT + q;
          c[q] = l < W ? S.run[l] : 0u;
          sum += c[q];
        }
        unsigned long long tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(sum, S.scan, &tot);
#pragma unroll
        for (int q = 0; q < kPerT; q++) {
          const int l = tid * kPerT + q;
          if (l < W) {
            S.run[l] = (unsigned)ex;
            col_ptr[c0 + l] = (int)(s0 + ex);
          }
          ex += c[q];
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kI; k++) {
        if (lr[k] == 0xffffffffu) continue;
        const unsigned p = S.run[lr[k]] + S.wc[warp][lr[k]] + rk[k];
        S.rk[p] = key[k] & mmask;
        S.v[p] = v[k];
      }
      __syncthreads();
      for (unsigned q = tid; q < L; q += kT) {
        __stcs(&row_idx[s0 + q], (int)S.rk[q]);
        __stcs(&out_vals[s0 + q], S.v[q]);
      }
      continue;
    }
    for (int l = tid; l < W; l += kT) S.run[l] = 0u;
    __syncthreads();
    // row counts of the whole bucket -> row starts (run) and col_ptr
    if (one) {
#pragma unroll
      for (int k = 0; k < kI; k++)
        if (warp * (32 * kI) + k * 32 + lane < L) atomicAdd(&S.run[key[k] >> mb], 1u);
    } else {
      for (unsigned i = tid; i < L; i += kT) atomicAdd(&S.run[__ldcs(&bK[s0 + i]) >> mb], 1u);
    }
    __syncthreads();
    {
      constexpr int kPerT = (sr::kMaxW + kT - 1) / kT;
      unsigned c[kPerT], sum = 0;
#pragma unroll
      for (int q = 0; q < kPerT; q++) {
        const int l = tid * kPerT + q;
        c[q] = l < W ? S.run[l] : 0u;
        sum += c[q];
      }
      unsigned long long tot;
      unsigned long long ex = block_exclusive_scan<unsigned long long>(sum, S.scan, &tot);
#pragma unroll
      for (int q = 0; q < kPerT; q++) {
        const int l = tid * kPerT + q;
        if (l < W) {
          S.run[l] = (unsigned)ex;
          col_ptr[c0 + l] = (int)(s0 + ex);
        }
        ex += c[q];
      }
    }
    for (unsigned base = 0; base < L; base += kE) {  // chunks in input order
      if (base > 0) {
#pragma unroll
        for (int k = 0; k < kI; k++) {
          const unsigned i = base + warp * (32 * kI) + k * 32 + lane;
          if (i < L) {
            key[k] = __ldcs(&bK[s0 + i]);
            v[k] = __ldcs(&bV[s0 + i]);
          }
        }
      }
      for (int l = lane; l < W; l += 32) S.wc[warp][l] = 0u;
      __syncwarp();
      unsigned rk[kI], lr[kI];
#pragma unroll
      for (int k = 0; k < kI; k++) {
        const bool in = base + warp * (32 * kI) + k * 32 + lane < L;
        lr[k] = in ? key[k] >> mb : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, lr[k]);
        unsigned b0 = 0;
        if (in) b0 = S.wc[warp][lr[k]];
        rk[k] = b0 + __popc(peers & lanemask_lt());
        __syncwarp();
        if (in && (peers & lanemask_lt()) == 0u) S.wc[warp][lr[k]] = b0 + __popc(peers);
        __syncwarp();
      }
      __syncthreads();
      for (int l = tid; l < W; l += kT) {  // per row: warp offsets (warp order), chunk count
        unsigned run = 0;
#pragma unroll
        for (int w = 0; w < kW; w++) {
          const unsigned c = S.wc[w][l];
          S.wc[w][l] = run;
          run += c;
        }
        S.ctot[l] = run;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kI; k++) {
        if (lr[k] == 0xffffffffu) continue;
        const unsigned p = S.run[lr[k]] + S.wc[warp][lr[k]] + rk[k];  // bucket-local output position
        if (one) {
          S.rk[p] = key[k] & mmask;
          S.v[p] = v[k];
        } else {
          __stcs(&row_idx[s0 + p], (int)(key[k] & mmask));
          __stcs(&out_vals[s0 + p], v[k]);
        }
      }
      __syncthreads();
      if (one) {
        for (unsigned q = tid; q < L; q += kT) {
          __stcs(&row_idx[s0 + q], (int)S.rk[q]);
          __stcs(&out_vals[s0 + q], S.v[q]);
        }
      } else {
        for (int l = tid; l < W; l += kT) S.run[l] += S.ctot[l];
        __syncthreads();
      }
    }
  }
}

// first column of every bucket: cbcol[b] = ceil(b * 2^32 / cb_mul) (capped)
static __global__ void ln_cbcol_kernel(unsigned* cbcol, long long nb, unsigned long long cb_mul, long long n_out_cols) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  const unsigned long long c0 = cb_mul ? (((unsigned long long)b << 32) + cb_mul - 1) / cb_mul : 0ull;
  cbcol[b] = (unsigned)(b == nb ? n_out_cols : min((long long)c0, n_out_cols));
}

}  // namespace ln
}  // namespace as
