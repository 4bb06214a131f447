// segsort.cuh -- the segmented sort / run-reduce / compact engine.
//
// Shared by COO->CSC construction (csc.canonicalize, csc.py:148-193), the
// insertion-cache flush (rbt.to_csc, rbt.py:444-458), CSC transpose
// (_kernels.transpose, _kernels.py:130-150) and Gustavson SpGEMM
// (_kernels.spgemm, _kernels.py:51-103).
//
// Input: N 64-bit keys already bucketed into n_seg contiguous segments
// (seg_ptr, int64[n_seg+1]); key = (out_row << 32) | idx where idx indexes the
// value source and encodes the reference's input order.  Each segment is
// sorted by key -- i.e. by (row, input order) -- runs of equal row are
// reduced in input order (pairwise / sequential / last), exact zeros are
// optionally pruned, and the survivors are compacted into CSC with one
// chained-scan pass (no second kernel for the output offsets).
//
// Tiling: tile t owns the segments whose start lies in [t*kTileNom,
// (t+1)*kTileNom).  A tile whose elements fit kCap is sorted in shared memory
// (warp-level bitonic per segment, block-level for long ones); a larger tile
// sorts its segments in place in global memory (block LSD radix for segments
// above kCap) and streams the reduce.
#pragma once

#include "capi_util.cuh"
#include "common.cuh"

namespace as {

constexpr int kSegThreads = 256;
constexpr int kTileNom = 2048;
constexpr int kCap = 4096;
constexpr int kItems = kCap / kSegThreads;  // 16 positions per thread
constexpr int kWarpSortMax = 512;

template <class T>
struct ValSrc {
  const T* a;
  const T* b;
  unsigned long long na;
  AS_DEVICE_INLINE T operator()(unsigned long long i) const { return i < na ? a[i] : b[i - na]; }
};

struct SegIn {
  const long long* seg_ptr;    // [n_seg + 1]
  long long n_seg;
  long long N;
  unsigned long long* keys;     // [N], sorted in place by oversized tiles
  unsigned long long* keys_alt; // [N] scratch for the block radix sort
  int row_bits;                 // significant bits of the row field
  int idx_bits;                 // significant bits of the idx field
  int presorted_idx;            // segments arrive in idx order (skip idx passes)
};

template <class T>
struct SegOut {
  int* col_ptr;    // [n_seg + 1]
  int* row_idx;    // [capacity]
  T* vals;         // [capacity]
  long long* info; // info[0] = nnz
  unsigned long long* tile_states;
  unsigned int* ticket;
};

AS_DEVICE_INLINE unsigned key_row(unsigned long long k) { return (unsigned)(k >> 32); }
AS_DEVICE_INLINE unsigned key_idx(unsigned long long k) { return (unsigned)(k & 0xffffffffull); }

AS_DEVICE_INLINE void cmpswap(unsigned long long* a, int i, int j) {
  unsigned long long x = a[i], y = a[j];
  if (y < x) {
    a[i] = y;
    a[j] = x;
  }
}

AS_DEVICE_INLINE int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Ascending bitonic sort of a[0..L) in place with virtual +inf padding to the
// next power of two.  Every compare-exchange is ascending with i < j, so pairs
// that reach past L are no-ops.  `sync` is __syncwarp or __syncthreads.
template <bool kBlock>
__device__ void bitonic_sort(unsigned long long* a, int L, int tid, int nthr) {
  const int P = next_pow2(L);
  const int npairs = P >> 1;
  for (int k = 2; k <= P; k <<= 1) {
    const int half = k >> 1;
    const int lh = __ffs(half) - 1;
    for (int p = tid; p < npairs; p += nthr) {
      int blk = p >> lh, t = p & (half - 1);
      int i = blk * k + t, j = blk * k + k - 1 - t;
      if (j < L) cmpswap(a, i, j);
    }
    if (kBlock) __syncthreads(); else __syncwarp();
    for (int h = half >> 1; h > 0; h >>= 1) {
      const int lh2 = __ffs(h) - 1;
      for (int p = tid; p < npairs; p += nthr) {
        int blk = p >> lh2, t = p & (h - 1);
        int i = (blk << (lh2 + 1)) + t, j = i + h;
        if (j < L) cmpswap(a, i, j);
      }
      if (kBlock) __syncthreads(); else __syncwarp();
    }
  }
}

// Block-level stable LSD radix sort of a global segment src[0..L) over the
// digit passes given by (shift, bits); ping-pongs with alt and leaves the
// result in src.  Scratch: smem_hist[256], smem_wcnt[256 * nwarps].
static __device__ void block_radix_sort_global(unsigned long long* src, unsigned long long* alt, long long L,
                                        const int* shifts, const int* nbits, int npass,
                                        unsigned* hist, unsigned* wcnt) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  unsigned long long* s = src;
  unsigned long long* d = alt;
  for (int ps = 0; ps < npass; ps++) {
    const int sh = shifts[ps];
    const unsigned mask = (1u << nbits[ps]) - 1u;
    for (int i = tid; i < 256; i += nthr) hist[i] = 0;
    for (int i = tid; i < 256 * nwarps; i += nthr) wcnt[i] = 0;
    __syncthreads();
    for (long long i = tid; i < L; i += nthr) atomicAdd(&hist[(unsigned)(s[i] >> sh) & mask], 1u);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of 256 bins -> running cursor
      unsigned carry = 0;
      for (int b = 0; b < 256; b += 32) {
        unsigned v = hist[b + lane];
        unsigned inc = warp_inclusive_scan(v);
        hist[b + lane] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    for (long long base = 0; base < L; base += nthr) {
      long long i = base + tid;
      bool in = i < L;
      unsigned long long k = in ? s[i] : 0ull;
      unsigned dg = in ? ((unsigned)(k >> sh) & mask) : 0xffffffffu;
      unsigned act = __ballot_sync(0xffffffffu, in);
      unsigned peers = 0, rank = 0;
      if (in) {
        peers = __match_any_sync(act, dg);
        rank = __popc(peers & lanemask_lt());
        if (rank == 0) wcnt[warp * 256 + dg] = __popc(peers);
      }
      __syncthreads();
      for (int b = tid; b < 256; b += nthr) {
        unsigned run = hist[b];
        for (int w = 0; w < nwarps; w++) {
          unsigned c = wcnt[w * 256 + b];
          wcnt[w * 256 + b] = run;
          run += c;
        }
        hist[b] = run;
      }
      __syncthreads();
      if (in) d[wcnt[warp * 256 + dg] + rank] = k;
      __syncthreads();
      for (int b = tid; b < 256 * nwarps; b += nthr) wcnt[b] = 0;
      __syncthreads();
    }
    unsigned long long* t = s;
    s = d;
    d = t;
  }
  if (s != src) {
    for (long long i = tid; i < L; i += nthr) src[i] = s[i];
    __syncthreads();
  }
}

template <class T>
struct SegSmem {
  unsigned long long sk[kCap];
  union {
    T rv[kCap];  // reduced run values (reduce phase)
    struct {     // block radix sort scratch (sort phase of oversized tiles)
      unsigned hist[256];
      unsigned wcnt[256 * (kSegThreads / 32)];
    } rs;
  } u;
  unsigned short excl[kCap + 1];
  long long scan_tmp[kSegThreads / 32 + 1];
  long long tile, c0, c1, e0, m;
  unsigned long long prefix;
};

// Locate the segment containing tile-local position p (first non-empty one).
AS_DEVICE_INLINE long long seg_of(const long long* seg_ptr, long long c0, long long c1, long long pos) {
  // last c in [c0, c1) with seg_ptr[c] <= pos
  long long lo = c0, hi = c1;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (seg_ptr[mid] <= pos) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
}

// Decide head / reduced value for tile-local positions [p_begin, p_end) of a
// sorted tile whose keys are at `kb` (tile-local indexing, smem or global).
// Calls emit(p, value) for each run head.  Returns nothing; counting is done
// by the caller through emit.
template <class T, class VS, class Emit>
__device__ void reduce_range(const unsigned long long* kb, long long m, long long e0, const long long* seg_ptr,
                             long long c0, long long c1, long long p_begin, long long p_end, VS vs, int mode,
                             Emit emit) {
  if (p_begin >= p_end) return;
  long long c = seg_of(seg_ptr, c0, c1, e0 + p_begin);
  long long s_beg = seg_ptr[c] - e0, s_end = seg_ptr[c + 1] - e0;
  for (long long p = p_begin; p < p_end; p++) {
    while (p >= s_end) {  // advance to the segment holding p
      c++;
      s_beg = seg_ptr[c] - e0;
      s_end = seg_ptr[c + 1] - e0;
    }
    unsigned long long k = kb[p];
    unsigned row = key_row(k);
    bool head = (p == s_beg) || key_row(kb[p - 1]) != row;
    if (!head) continue;
    long long q = p + 1;
    while (q < s_end && key_row(kb[q]) == row) q++;
    const unsigned long long* run = kb + p;
    auto get = [&](long long i) -> T { return vs((unsigned long long)key_idx(run[i])); };
    T v = reduce_run<T>(get, q - p, mode);
    emit(p, row, v);
  }
}

template <class T, class VS>
__global__ void __launch_bounds__(kSegThreads)
seg_tile_kernel(SegIn in, VS vs, int mode, int prune, SegOut<T> out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SegSmem<T>& S = *reinterpret_cast<SegSmem<T>*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, nwarps = nthr >> 5, lane = tid & 31;
  const long long n_tiles = gridDim.x;

  if (tid == 0) {
    long long t = atomicAdd(out.ticket, 1u);
    long long lo = t * kTileNom;
    long long c0 = lower_bound_dev(in.seg_ptr, in.n_seg, lo);
    long long c1 = (t == n_tiles - 1) ? in.n_seg : lower_bound_dev(in.seg_ptr, in.n_seg, lo + kTileNom);
    S.tile = t;
    S.c0 = c0;
    S.c1 = c1;
    S.e0 = in.seg_ptr[c0];
    S.m = in.seg_ptr[c1] - S.e0;
  }
  __syncthreads();
  const long long t = S.tile, c0 = S.c0, c1 = S.c1, e0 = S.e0, m = S.m;
  const long long* seg_ptr = in.seg_ptr;

  if (m <= kCap) {
    // ---------------- shared-memory path ----------------
    for (long long i = tid; i < m; i += nthr) S.sk[i] = in.keys[e0 + i];
    __syncthreads();
    for (long long c = c0 + warp; c < c1; c += nwarps) {
      int L = (int)(seg_ptr[c + 1] - seg_ptr[c]);
      if (L > 1 && L <= kWarpSortMax) bitonic_sort<false>(S.sk + (seg_ptr[c] - e0), L, lane, 32);
    }
    __syncthreads();
    for (long long c = c0; c < c1; c++) {  // block-uniform loop
      int L = (int)(seg_ptr[c + 1] - seg_ptr[c]);
      if (L > kWarpSortMax) bitonic_sort<true>(S.sk + (seg_ptr[c] - e0), L, tid, nthr);
    }
    __syncthreads();
    // reduce: thread owns positions [tid*kItems, tid*kItems + kItems)
    const long long pb = (long long)tid * kItems, pe = min(pb + kItems, m);
    for (long long p = pb; p < pe; p++) S.excl[p] = 0;
    int cnt = 0;
    reduce_range<T>(S.sk, m, e0, seg_ptr, c0, c1, pb, pe, vs, mode,
                    [&](long long p, unsigned row, T v) {
                      bool keep = !prune || v != T(0);
                      S.u.rv[p] = v;
                      S.excl[p] = keep ? 1 : 0;
                      cnt += keep;
                    });
    long long total;
    long long off = block_exclusive_scan<long long>((long long)cnt, S.scan_tmp, &total);
    {
      unsigned run = (unsigned)off;
      for (long long p = pb; p < pe; p++) {
        unsigned f = S.excl[p];
        S.excl[p] = (unsigned short)run;
        run += f;
      }
      if (tid == 0) S.excl[m] = (unsigned short)total;
    }
    if (warp == 0) {
      unsigned long long pre = tile_lookback_warp(out.tile_states, t, (unsigned long long)total);
      if (lane == 0) S.prefix = pre;
    }
    __syncthreads();
    const long long P = (long long)S.prefix;
    for (long long p = tid; p < m; p += nthr) {
      unsigned a = S.excl[p], b = S.excl[p + 1];
      if (b != a) {
        long long o = P + a;
        out.row_idx[o] = (int)key_row(S.sk[p]);
        out.vals[o] = S.u.rv[p];
      }
    }
    for (long long c = c0 + tid; c < c1; c += nthr) out.col_ptr[c] = (int)(P + S.excl[seg_ptr[c] - e0]);
    if (t == n_tiles - 1 && tid == 0) {
      out.col_ptr[in.n_seg] = (int)(P + total);
      out.info[0] = P + total;
    }
    return;
  }

  // ---------------- oversized tile: global path ----------------
  unsigned long long* gk = in.keys + e0;
  for (long long c = c0; c < c1; c++) {  // block-uniform
    long long L = seg_ptr[c + 1] - seg_ptr[c];
    if (L <= 1) continue;
    unsigned long long* seg = in.keys + seg_ptr[c];
    if (L <= kCap) {
      for (long long i = tid; i < L; i += nthr) S.sk[i] = seg[i];
      __syncthreads();
      bitonic_sort<true>(S.sk, (int)L, tid, nthr);
      for (long long i = tid; i < L; i += nthr) seg[i] = S.sk[i];
      __syncthreads();
    } else {
      int shifts[16], nbits[16], np = 0;
      if (!in.presorted_idx)
        for (int b = 0; b < in.idx_bits; b += 8) { shifts[np] = b; nbits[np] = min(8, in.idx_bits - b); np++; }
      for (int b = 0; b < in.row_bits; b += 8) { shifts[np] = 32 + b; nbits[np] = min(8, in.row_bits - b); np++; }
      block_radix_sort_global(seg, in.keys_alt + seg_ptr[c], L, shifts, nbits, np, S.u.rs.hist, S.u.rs.wcnt);
    }
  }
  __syncthreads();
  // count pass
  long long total = 0;
  for (long long b = 0; b < m; b += kCap) {
    const long long pb = b + (long long)tid * kItems, pe = min(pb + kItems, m);
    int cnt = 0;
    reduce_range<T>(gk, m, e0, seg_ptr, c0, c1, pb, pe, vs, mode,
                    [&](long long p, unsigned row, T v) { cnt += (!prune || v != T(0)); });
    total += block_reduce_sum<long long>((long long)cnt, S.scan_tmp);
  }
  if (warp == 0) {
    unsigned long long pre = tile_lookback_warp(out.tile_states, t, (unsigned long long)total);
    if (lane == 0) S.prefix = pre;
  }
  __syncthreads();
  const long long P = (long long)S.prefix;
  // write pass
  long long run_base = 0;
  for (long long b = 0; b < m; b += kCap) {
    const long long cm = min((long long)kCap, m - b);
    const long long pb = b + (long long)tid * kItems, pe = min(pb + kItems, m);
    for (long long p = pb; p < pe; p++) S.excl[p - b] = 0;
    int cnt = 0;
    reduce_range<T>(gk, m, e0, seg_ptr, c0, c1, pb, pe, vs, mode,
                    [&](long long p, unsigned row, T v) {
                      bool keep = !prune || v != T(0);
                      S.u.rv[p - b] = v;
                      S.excl[p - b] = keep ? 1 : 0;
                      cnt += keep;
                    });
    long long ctot;
    long long off = block_exclusive_scan<long long>((long long)cnt, S.scan_tmp, &ctot);
    {
      unsigned run = (unsigned)off;
      for (long long p = pb; p < pe; p++) {
        unsigned f = S.excl[p - b];
        S.excl[p - b] = (unsigned short)run;
        run += f;
      }
      if (tid == 0) S.excl[cm] = (unsigned short)ctot;
    }
    __syncthreads();
    for (long long p = tid; p < cm; p += nthr) {
      unsigned a = S.excl[p], c = S.excl[p + 1];
      if (c != a) {
        long long o = P + run_base + a;
        out.row_idx[o] = (int)key_row(gk[b + p]);
        out.vals[o] = S.u.rv[p];
      }
    }
    for (long long c = c0 + tid; c < c1; c += nthr) {
      long long s = seg_ptr[c] - e0;
      if (s >= b && s < b + cm) out.col_ptr[c] = (int)(P + run_base + S.excl[s - b]);
    }
    run_base += ctot;
    __syncthreads();
  }
  for (long long c = c0 + tid; c < c1; c += nthr)
    if (seg_ptr[c] - e0 >= m) out.col_ptr[c] = (int)(P + total);
  if (t == n_tiles - 1 && tid == 0) {
    out.col_ptr[in.n_seg] = (int)(P + total);
    out.info[0] = P + total;
  }
}

// ------------------------------------------------------------------------
// bucket counting / scan / scatter

// count column occupancy of COO triplets; validate coordinates and record the
// first invalid triplet index (csc.py:215-221 / coo.py:54-61 report it).
template <class IdxT>
__global__ void coo_count_kernel(long long n, const IdxT* rows, const IdxT* cols, long long n_rows,
                                 long long n_cols, unsigned* counts, long long* bad) {
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += stride) {
    long long i = base + lane;
    bool in = i < n;
    long long r = in ? (long long)rows[i] : 0, c = in ? (long long)cols[i] : 0;
    bool ok = in && r >= 0 && r < n_rows && c >= 0 && c < n_cols;
    if (in && !ok) atomicMin((unsigned long long*)bad, (unsigned long long)i);
    unsigned act = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      unsigned peers = __match_any_sync(act, (unsigned)c);
      if ((peers & lanemask_lt()) == 0) atomicAdd(&counts[c], (unsigned)__popc(peers));
    }
  }
}

// add the per-column lengths of a CSC (the base of a flush)
static __global__ void csc_count_kernel(long long n_cols, const int* col_ptr, unsigned* counts) {
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n_cols;
       c += (long long)gridDim.x * blockDim.x)
    counts[c] += (unsigned)(col_ptr[c + 1] - col_ptr[c]);
}

// count rows of a CSC (buckets of the transpose)
static __global__ void row_count_kernel(long long nnz, const int* row_idx, unsigned* counts) {
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nnz;
       base += stride) {
    long long i = base + lane;
    bool in = i < nnz;
    unsigned r = in ? (unsigned)row_idx[i] : 0u;
    unsigned act = __ballot_sync(0xffffffffu, in);
    if (in) {
      unsigned peers = __match_any_sync(act, r);
      if ((peers & lanemask_lt()) == 0) atomicAdd(&counts[r], (unsigned)__popc(peers));
    }
  }
}

// exclusive scan counts[0..n) -> seg_ptr[0..n] (int64) and zero counts (so
// they can serve as fill cursors).  Chained scan, 4096 counts per tile.
constexpr int kScanThreads = 256, kScanItems = 16;
static __global__ void __launch_bounds__(kScanThreads)
count_scan_kernel(unsigned* counts, long long n, long long* seg_ptr, unsigned long long* states,
                  unsigned* ticket) {
  __shared__ long long tmp[kScanThreads / 32 + 1];
  __shared__ long long s_tile;
  __shared__ unsigned long long s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long t = s_tile;
  const long long base = t * (kScanThreads * kScanItems) + (long long)threadIdx.x * kScanItems;
  unsigned v[kScanItems];
  long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    long long i = base + k;
    v[k] = i < n ? counts[i] : 0u;
    sum += v[k];
  }
  long long total;
  long long off = block_exclusive_scan<long long>(sum, tmp, &total);
  if ((threadIdx.x >> 5) == 0) {
    unsigned long long pre = tile_lookback_warp(states, t, (unsigned long long)total);
    if ((threadIdx.x & 31) == 0) s_prefix = pre;
  }
  __syncthreads();
  long long run = (long long)s_prefix + off;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    long long i = base + k;
    if (i < n) {
      seg_ptr[i] = run;
      counts[i] = 0u;
    }
    run += v[k];
  }
  if (t == gridDim.x - 1 && threadIdx.x == 0) seg_ptr[n] = (long long)s_prefix + total;
}

// scatter valid COO triplets into their column buckets: key = (row << 32) | (i + idx_off)
template <class IdxT>
__global__ void coo_scatter_kernel(long long n, const IdxT* rows, const IdxT* cols, long long n_rows,
                                   long long n_cols, const long long* seg_ptr, unsigned* fill,
                                   unsigned long long* keys, unsigned long long idx_off) {
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n;
       base += stride) {
    long long i = base + lane;
    bool in = i < n;
    long long r = in ? (long long)rows[i] : 0, c = in ? (long long)cols[i] : 0;
    bool ok = in && r >= 0 && r < n_rows && c >= 0 && c < n_cols;
    unsigned act = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      unsigned peers = __match_any_sync(act, (unsigned)c);
      int leader = __ffs(peers) - 1;
      unsigned rank = __popc(peers & lanemask_lt());
      unsigned b = 0;
      if (rank == 0) b = atomicAdd(&fill[c], (unsigned)__popc(peers));
      b = __shfl_sync(peers, b, leader);
      keys[seg_ptr[c] + b + rank] = ((unsigned long long)r << 32) | (unsigned long long)(i + idx_off);
    }
  }
}

// scatter the elements of a CSC.  kByRow: bucket = row, key = (col << 32) | k
// (transpose); else bucket = col, key = (row << 32) | k  (flush base).
template <bool kByRow>
__global__ void csc_scatter_kernel(long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
                                   const long long* seg_ptr, unsigned* fill, unsigned long long* keys) {
  const int lane = threadIdx.x & 31;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nnz;
       base += stride) {
    long long k = base + lane;
    bool in = k < nnz;
    unsigned r = 0, c = 0;
    if (in) {
      r = (unsigned)row_idx[k];
      c = (unsigned)(upper_bound_dev(col_ptr, n_cols + 1, (int)k) - 1);
    }
    unsigned bucket = kByRow ? r : c;
    unsigned other = kByRow ? c : r;
    unsigned act = __ballot_sync(0xffffffffu, in);
    if (in) {
      unsigned peers = __match_any_sync(act, bucket);
      int leader = __ffs(peers) - 1;
      unsigned rank = __popc(peers & lanemask_lt());
      unsigned b = 0;
      if (rank == 0) b = atomicAdd(&fill[bucket], (unsigned)__popc(peers));
      b = __shfl_sync(peers, b, leader);
      keys[seg_ptr[bucket] + b + rank] = ((unsigned long long)other << 32) | (unsigned long long)k;
    }
  }
}

// ------------------------------------------------------------------------
// host-side launcher of the tile engine (one kernel, chained-scan compaction)
inline long long seg_engine_tiles(long long n_upper) {
  return n_upper > 0 ? (n_upper + kTileNom - 1) / kTileNom : 1;
}

template <class T>
inline int launch_seg_engine(const long long* seg_ptr, long long n_seg, long long n_upper, unsigned long long* keys,
                             unsigned long long* keys_alt, int row_bits, int idx_bits, int presorted, ValSrc<T> vs,
                             int mode, int prune, int* col_ptr, int* row_idx, T* vals, long long* info,
                             unsigned long long* states, unsigned* ticket, cudaStream_t st) {
  const size_t smem = sizeof(SegSmem<T>);
  static bool attr_set = false;
  if (!attr_set) {
    AS_CUDA_TRY(cudaFuncSetAttribute(seg_tile_kernel<T, ValSrc<T>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attr_set = true;
  }
  SegIn in{seg_ptr, n_seg, n_upper, keys, keys_alt, row_bits, idx_bits, presorted};
  SegOut<T> out{col_ptr, row_idx, vals, info, states, ticket};
  seg_tile_kernel<T, ValSrc<T>><<<(unsigned)seg_engine_tiles(n_upper), kSegThreads, smem, st>>>(in, vs, mode, prune,
                                                                                               out);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

}  // namespace as
