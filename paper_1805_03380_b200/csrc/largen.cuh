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

constexpr int kT = 512;          // threads of the count / scatter CTAs
constexpr int kI = 8;            // elements per thread
constexpr int kE = kT * kI;      // elements per pipeline tile
constexpr int kR = 256;          // digit radix
constexpr int kW = kT / 32;      // warps
constexpr int kScanN = 4096;     // entries per scan tile (256 threads x 16)
constexpr int kJoinSpan = 16;    // low digits a pass-B tile may span for its bucket histogram

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
};

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
};

AS_DEVICE_INLINE unsigned bucket_of(unsigned maj, unsigned long long cb_mul) {
  return (unsigned)(((unsigned long long)maj * cb_mul) >> 32);
}

// ---- element loads of one item: e = global element index; returns valid
template <class IdxT, class T>
AS_DEVICE_INLINE bool load_el(const CooIn<IdxT, T>& s, long long e, unsigned& maj, unsigned& mn, T& v,
                              unsigned long long* bad, bool need_minor, bool need_val) {
  const long long r = (long long)__ldcs(&s.rows[e]), c = (long long)__ldcs(&s.cols[e]);
  if (r < 0 || r >= s.n_rows || c < 0 || c >= s.n_cols) {
    if (bad) atomicMin(bad, (unsigned long long)e);
    return false;
  }
  maj = (unsigned)c;
  mn = (unsigned)r;
  if (need_val) v = __ldcs(&s.vals[e]);
  (void)need_minor;
  return true;
}

// CSC visited by row: the column of element e from the tile's cached column
// pointers (colc[0..nc] = ptr[cb..cb+nc]) or a global binary search
struct ColCache {
  long long cb;
  int nc;          // cached entries - 1, or -1 when not cached
};

template <class T>
AS_DEVICE_INLINE bool load_el_csc(const CscIn<T>& s, long long e, const ColCache& cc, const int* colc, unsigned& maj,
                                  unsigned& mn, T& v, bool need_minor, bool need_val) {
  maj = (unsigned)__ldcs(&s.idx[e]);
  if (need_minor) {
    long long c;
    if (cc.nc >= 0) {
      int l = 0, h = cc.nc;  // last l with colc[l] <= e
      while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (colc[mid] <= e) l = mid;
        else h = mid - 1;
      }
      c = cc.cb + l;
    } else {
      c = upper_bound_dev(s.ptr, s.n_cols + 1, (int)e) - 1;
    }
    mn = (unsigned)c;
  }
  if (need_val) v = __ldcs(&s.vals[e]);
  return true;
}

template <class T>
AS_DEVICE_INLINE bool load_el_rec(const RecIn<T>& s, long long e, unsigned& maj, unsigned& mn, T& v, bool need_minor,
                                  bool need_val) {
  maj = __ldcs(&s.maj[e]);
  if (need_minor) mn = __ldcs(&s.mn[e]);
  if (need_val) v = __ldcs(&s.vals[e]);
  return true;
}

// the tile's column range of a CSC source, cached in shared memory when it fits
template <class T>
__device__ void csc_cache(const CscIn<T>& s, long long lo, long long hi, int* colc, ColCache* cc) {
  const long long cb = sr::block_upper_bound(s.ptr, s.n_cols + 1, lo) - 1;
  const long long ce = sr::block_upper_bound(s.ptr, s.n_cols + 1, hi - 1) - 1;
  const bool cached = ce - cb + 1 <= sr::kColCache;
  if (cached)
    for (long long c = cb + threadIdx.x; c <= ce + 1 && c <= s.n_cols; c += blockDim.x) colc[c - cb] = __ldg(&s.ptr[c]);
  cc->cb = cb;
  cc->nc = cached ? (int)(ce - cb) : -1;
  __syncthreads();
}

// kind of a pass: 0 = pass A (digit = low bits, writes records A),
// 1 = pass B from records A (digit = high bits), 2 = single pass (digit = bucket)
template <int kPass>
AS_DEVICE_INLINE unsigned digit_of(unsigned b, int lob) {
  if (kPass == 0) return b & ((1u << lob) - 1u);
  if (kPass == 1) return b >> lob;
  return b;
}

// generic item loader for the three sources
template <class T, class In>
struct Loader;

template <class T, class IdxT>
struct Loader<T, CooIn<IdxT, T>> {
  const CooIn<IdxT, T>& s;
  unsigned long long* bad;
  __device__ void prep(long long, long long, int*, ColCache*) {}
  AS_DEVICE_INLINE bool operator()(long long e, unsigned& maj, unsigned& mn, T& v, bool need_minor, bool need_val,
                                   const ColCache&, const int*) {
    return load_el(s, e, maj, mn, v, bad, need_minor, need_val);
  }
};

template <class T>
struct Loader<T, CscIn<T>> {
  const CscIn<T>& s;
  unsigned long long* bad;
  __device__ void prep(long long lo, long long hi, int* colc, ColCache* cc) { csc_cache(s, lo, hi, colc, cc); }
  AS_DEVICE_INLINE bool operator()(long long e, unsigned& maj, unsigned& mn, T& v, bool need_minor, bool need_val,
                                   const ColCache& cc, const int* colc) {
    return load_el_csc(s, e, cc, colc, maj, mn, v, need_minor, need_val);
  }
};

template <class T>
struct Loader<T, RecIn<T>> {
  const RecIn<T>& s;
  unsigned long long* bad;
  __device__ void prep(long long, long long, int*, ColCache*) {}
  AS_DEVICE_INLINE bool operator()(long long e, unsigned& maj, unsigned& mn, T& v, bool need_minor, bool need_val,
                                   const ColCache&, const int*) {
    return load_el_rec(s, e, maj, mn, v, need_minor, need_val);
  }
};

// element e of item k of this thread: warp-blocked, lane-consecutive, so the
// (warp, item, lane) order is the input order
AS_DEVICE_INLINE long long elem_of(long long t, int k) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  return t * kE + (long long)warp * (32 * kI) + k * 32 + lane;
}

// ------------------------------------------------------------------------
// count: digit histogram of tile t -> H[d * T + t]; pass 1 / 2 also add the
// tile's bucket counts into bcnt
template <class T, class In, int kPass>
__global__ void __launch_bounds__(kT) ln_count_kernel(Args<T> a, In src) {
  __shared__ unsigned h[kR];
  __shared__ unsigned jb[kJoinSpan * kR];
  __shared__ int colc[sr::kColCache + 1];
  __shared__ ColCache cc;
  __shared__ unsigned lo0s;
  const int tid = threadIdx.x;
  const long long t = blockIdx.x;
  const long long lo = t * kE, hi = min(a.n, lo + kE);
  for (int i = tid; i < kR; i += kT) h[i] = 0u;
  if (kPass == 1)
    for (int i = tid; i < kJoinSpan * kR; i += kT) jb[i] = 0u;
  Loader<T, In> ld{src, kPass != 1 ? a.bad : nullptr};
  if (tid == 0) cc = ColCache{0, -1};
  if constexpr (kPass == 1) {
    if (tid == 0) lo0s = bucket_of(__ldg(&src.maj[lo]), a.cb_mul) & ((1u << a.lob) - 1u);
  }
  __syncthreads();
  const unsigned lo0 = kPass == 1 ? lo0s : 0u;
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const long long e = elem_of(t, k);
    if (e >= hi) continue;
    unsigned maj = 0, mn = 0;
    T v;
    if (!ld(e, maj, mn, v, false, false, cc, colc)) continue;
    const unsigned b = bucket_of(maj, a.cb_mul);
    atomicAdd(&h[digit_of<kPass>(b, a.lob)], 1u);
    if (kPass == 1) {
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
  if (kPass == 1) {
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
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long t = s_tile;
  constexpr int kPer = kScanN / kScanT;
  const long long base = t * kScanN + (long long)threadIdx.x * kPer;
  unsigned v[kPer];
  long long sum = 0;
#pragma unroll
  for (int k = 0; k < kPer; k++) {
    const long long i = base + k;
    v[k] = i < n ? x[i] : 0u;
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
    const long long i = base + k;
    if (i < n) x[i] = (unsigned)run;
    run += v[k];
  }
  if (t == gridDim.x - 1 && threadIdx.x == 0 && out_total) *out_total = (unsigned)((long long)s_prefix + total);
}

// ------------------------------------------------------------------------
// scatter: stable counting sort of tile t by digit into the pass's records
template <class T, int kPass>
struct ScatterSmem {
  unsigned wc[kW][kR];      // per-warp digit counters -> per-warp offsets
  unsigned tstart[kR];      // tile-local digit starts
  unsigned gbase[kR];       // global start of the tile's run of each digit
  unsigned k1[kE];          // major (pass A) or bucket-local key
  unsigned k2[kE];          // minor (pass A only)
  T v[kE];
  unsigned short d[kE];
  long long scan[kT / 32 + 1];
  int colc[sr::kColCache + 1];
  ColCache cc;
};

template <class T, class In, int kPass>
__global__ void __launch_bounds__(kT, 2) ln_scatter_kernel(Args<T> a, In src) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ScatterSmem<T, kPass>& S = *reinterpret_cast<ScatterSmem<T, kPass>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t = blockIdx.x;
  const long long lo = t * kE, hi = min(a.n, lo + kE);
  Loader<T, In> ld{src, nullptr};
  if (tid == 0) S.cc = ColCache{0, -1};
  for (int i = lane; i < kR; i += 32) S.wc[warp][i] = 0u;
  __syncthreads();
  ld.prep(lo, hi, S.colc, &S.cc);  // (CSC source: block-wide; others no-op)
  const ColCache cc = S.cc;
  unsigned maj[kI], mn[kI], dg[kI], rk[kI];
  T v[kI];
  bool ok[kI];
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const long long e = elem_of(t, k);
    ok[k] = e < hi && ld(e, maj[k], mn[k], v[k], true, true, cc, S.colc);
    dg[k] = ok[k] ? digit_of<kPass>(bucket_of(maj[k], a.cb_mul), a.lob) : 0xffffu;
  }
  // stable ranks: item by item (input order), lanes of one digit by match
#pragma unroll
  for (int k = 0; k < kI; k++) {
    const unsigned peers = __match_any_sync(0xffffffffu, dg[k]);
    unsigned base = 0;
    if (ok[k]) base = S.wc[warp][dg[k]];
    rk[k] = base + __popc(peers & lanemask_lt());
    __syncwarp();
    if (ok[k] && (peers & lanemask_lt()) == 0u) S.wc[warp][dg[k]] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: offsets of the warps (in warp order), tile count, tile start
  unsigned cnt = 0;
  if (tid < kR) {
    for (int w = 0; w < kW; w++) {
      const unsigned c = S.wc[w][tid];
      S.wc[w][tid] = cnt;
      cnt += c;
    }
  }
  long long tot;
  const long long st = block_exclusive_scan<long long>(tid < kR ? (long long)cnt : 0ll, S.scan, &tot);
  const int R = kPass == 0 ? (1 << a.lob) : kR;
  if (tid < kR) {
    S.tstart[tid] = (unsigned)st;
    S.gbase[tid] = tid < R ? __ldcg(&a.H[(long long)tid * a.T_ + t]) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kI; k++) {
    if (!ok[k]) continue;
    const unsigned p = S.tstart[dg[k]] + S.wc[warp][dg[k]] + rk[k];
    if (kPass == 0) {
      S.k1[p] = maj[k];
      S.k2[p] = mn[k];
    } else {
      const unsigned b = bucket_of(maj[k], a.cb_mul);
      S.k1[p] = ((maj[k] - __ldg(&a.cbcol[b])) << a.mb) | mn[k];
    }
    S.v[p] = v[k];
    S.d[p] = (unsigned short)dg[k];
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
  __device__ __forceinline__ unsigned key(unsigned s) const { return __ldcs(&bK[s]); }
  __device__ __forceinline__ unsigned idx(unsigned s) const { return s; }
  __device__ __forceinline__ const T* val(unsigned s) const { return bV + s; }
  __device__ __forceinline__ unsigned col0(long long t) const { return __ldg(&cbcol[t]); }
  __device__ __forceinline__ unsigned long long prefix(long long t, unsigned long long kept) const {
    return tile_lookback_warp(tstate, t, kept);
  }
};

template <class T>
__global__ void __launch_bounds__(sr::kThreads, 2)
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

// first column of every bucket: cbcol[b] = ceil(b * 2^32 / cb_mul) (capped)
static __global__ void ln_cbcol_kernel(unsigned* cbcol, long long nb, unsigned long long cb_mul, long long n_out_cols) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  const unsigned long long c0 = cb_mul ? (((unsigned long long)b << 32) + cb_mul - 1) / cb_mul : 0ull;
  cbcol[b] = (unsigned)(b == nb ? n_out_cols : min((long long)c0, n_out_cols));
}

}  // namespace ln
}  // namespace as
