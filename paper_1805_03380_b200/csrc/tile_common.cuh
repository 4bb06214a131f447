// tile_common.cuh -- shared-memory tile primitives and the chained count
// scan used by the bucket-sort-reduce kernel (persist.cuh) and SpGEMM.
//
// Keys are u64 = (row << 32) | idx: the high word is the row (or the minor
// index), the low word indexes the value source and encodes the reference's
// input order, so ascending keys are (row, input order) -- the order every
// duplicate reduction of the reference folds in.
#pragma once

#include "capi_util.cuh"
#include "common.cuh"

namespace as {

#ifndef AS_SEG_THREADS
#define AS_SEG_THREADS 512
#endif
constexpr int kSegThreads = AS_SEG_THREADS;  // threads of a tile CTA
#ifndef AS_KCAP
#define AS_KCAP 2048
#endif
constexpr int kCap = AS_KCAP;               // elements of a shared-memory tile
constexpr int kItems = kCap / kSegThreads;  // 8 positions per thread
constexpr int kWarpSortMax = 512;           // bins up to this sort in one warp
constexpr int kRankMax = 32;                // bins up to this rank keys directly

// values by input index: a[0..na) then b (base CSC ++ write log for a flush)
template <class T>
struct ValSrc {
  const T* a;
  const T* b;
  unsigned long long na;
  AS_DEVICE_INLINE T operator()(unsigned long long i) const { return i < na ? a[i] : b[i - na]; }
};

AS_DEVICE_INLINE unsigned key_row(unsigned long long k) { return (unsigned)(k >> 32); }
AS_DEVICE_INLINE unsigned key_idx(unsigned long long k) { return (unsigned)(k & 0xffffffffull); }

AS_DEVICE_INLINE void cmpswap(unsigned long long* a, unsigned short* pm, int i, int j) {
  unsigned long long x = a[i], y = a[j];
  if (y < x) {
    a[i] = y;
    a[j] = x;
    if (pm) {
      const unsigned short t = pm[i];
      pm[i] = pm[j];
      pm[j] = t;
    }
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
__device__ void bitonic_sort(unsigned long long* a, int L, int tid, int nthr, unsigned short* pm = nullptr) {
  const int P = next_pow2(L);
  const int npairs = P >> 1;
  for (int k = 2; k <= P; k <<= 1) {
    const int half = k >> 1;
    const int lh = __ffs(half) - 1;
    for (int p = tid; p < npairs; p += nthr) {
      int blk = p >> lh, t = p & (half - 1);
      int i = blk * k + t, j = blk * k + k - 1 - t;
      if (j < L) cmpswap(a, pm, i, j);
    }
    if (kBlock) __syncthreads(); else __syncwarp();
    for (int h = half >> 1; h > 0; h >>= 1) {
      const int lh2 = __ffs(h) - 1;
      for (int p = tid; p < npairs; p += nthr) {
        int blk = p >> lh2, t = p & (h - 1);
        int i = (blk << (lh2 + 1)) + t, j = i + h;
        if (j < L) cmpswap(a, pm, i, j);
      }
      if (kBlock) __syncthreads(); else __syncwarp();
    }
  }
}

AS_DEVICE_INLINE bool bit_at(const unsigned* bits, int p) { return (bits[p >> 5] >> (p & 31)) & 1u; }

// first set bit at position >= p (positions < lim), or lim
AS_DEVICE_INLINE int next_bit(const unsigned* bits, int p, int lim) {
  if (p >= lim) return lim;
  int w = p >> 5;
  unsigned word = bits[w] & (~0u << (p & 31));
  const int wl = (lim + 31) >> 5;
  while (true) {
    if (word) {
      int q = (w << 5) + __ffs(word) - 1;
      return q < lim ? q : lim;
    }
    if (++w >= wl) return lim;
    word = bits[w];
  }
}

// exclusive scan counts[0..n) -> seg_ptr[0..n] (int64) and zero counts (so
// they can serve as fill cursors).  Chained scan, 4096 counts per tile; the
// tile moves through shared memory so every global access is coalesced (each
// thread scans 16 consecutive counts: reading them straight from global memory
// made every warp access touch 32 sectors).
constexpr int kScanThreads = 256, kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
AS_DEVICE_INLINE int scan_pad(int i) { return i + (i >> 5); }
static __global__ void __launch_bounds__(kScanThreads)
count_scan_kernel(unsigned* counts, long long n, long long* seg_ptr, unsigned long long* states, unsigned* ticket) {
  __shared__ long long tmp[kScanThreads / 32 + 1];
  __shared__ long long s_tile;
  __shared__ unsigned long long s_prefix;
  __shared__ long long sx[kScanTile + kScanTile / 32];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const long long t = s_tile;
  const long long t0 = t * kScanTile;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    const int q = k * kScanThreads + threadIdx.x;
    sx[scan_pad(q)] = t0 + q < n ? (long long)counts[t0 + q] : 0ll;
  }
  __syncthreads();
  unsigned v[kScanItems];
  long long sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    v[k] = (unsigned)sx[scan_pad(threadIdx.x * kScanItems + k)];
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
    sx[scan_pad(threadIdx.x * kScanItems + k)] = run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    const int q = k * kScanThreads + threadIdx.x;
    if (t0 + q < n) {
      seg_ptr[t0 + q] = sx[scan_pad(q)];
      counts[t0 + q] = 0u;
    }
  }
  if (t == gridDim.x - 1 && threadIdx.x == 0) {
    seg_ptr[n] = (long long)s_prefix + total;
  }
}

}  // namespace as
