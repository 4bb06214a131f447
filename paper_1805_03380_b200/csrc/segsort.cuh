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
constexpr int kTileNom = 1024;
constexpr int kCap = 2048;
constexpr int kItems = kCap / kSegThreads;  // 8 positions per thread
constexpr int kMaxBins = 512;               // second-level buckets per tile
constexpr int kWarpSortMax = 512;

template <class T>
struct ValSrc {
  const T* a;
  const T* b;
  unsigned long long na;
  AS_DEVICE_INLINE T operator()(unsigned long long i) const { return i < na ? a[i] : b[i - na]; }
  AS_DEVICE_INLINE void prefetch(unsigned long long i) const {
    const T* p = i < na ? a + i : b + (i - na);
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
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
  const long long* tile_c0;     // [n_tiles + 1] first segment of each tile
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

constexpr int kSegBatch = 256;

template <class T>
struct SegSmem {
  unsigned long long sk[kCap];
  union {
    T rv[kCap];                       // gathered values, then reduced run values at heads
    unsigned long long sk2[kCap];     // second-level bucketing target
    struct {                          // block radix sort scratch (oversized tiles)
      unsigned hist[256];
      unsigned wcnt[256 * (kSegThreads / 32)];
    } rs;
  } u;
  union {
    unsigned short excl[kCap + 8];    // exclusive kept counts (reduce phase)
    struct {
      unsigned cursor[kMaxBins];
      unsigned short bstart[kMaxBins + 8];
    } bk;                             // second-level bucket counters (sort phase)
  } v;
  unsigned sbits[kCap / 32];  // segment starts within the chunk
  unsigned hbits[kCap / 32];  // run heads within the chunk
  unsigned wpre[kCap / 32];   // exclusive popcount of sbits per word
  unsigned short sbin[kCap];  // second-level bin of each bucketed key
  unsigned short perm[kCap];  // tile-local bucket slot of each key in sk
  unsigned short perm2[kCap]; // same for sk2
  int sseg[kSegBatch + 1];
  short med[kMaxBins], big[kMaxBins];
  int n_med, n_big, nseg;
  long long scan_tmp[kSegThreads / 32 + 1];
  long long scan_tmp2[kSegThreads];
  long long tile, c0, c1, e0, m;
  unsigned long long prefix;
};

// Last c in [c0, c1) with seg_ptr[c] <= pos: the (non-empty) segment holding pos.
AS_DEVICE_INLINE long long seg_of(const long long* seg_ptr, long long c0, long long c1, long long pos) {
  long long lo = c0, hi = c1;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (seg_ptr[mid] <= pos) lo = mid + 1;
    else hi = mid;
  }
  return lo - 1;
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

// Sort every segment of the tile whose keys sit in S.sk (tile-local
// positions).  Segment bounds are staged through shared memory in batches
// (coalesced) and classified by length: up to kThreadSortMax one thread does
// an insertion sort, up to kWarpSortMax one warp a bitonic sort, longer ones
// the whole block.
constexpr int kThreadSortMax = 16;
constexpr int kRankMax = 32;

AS_DEVICE_INLINE void insertion_sort(unsigned long long* a, unsigned short* pm, int L) {
  for (int i = 1; i < L; i++) {
    const unsigned long long x = a[i];
    const unsigned short px = pm[i];
    int j = i - 1;
    while (j >= 0 && a[j] > x) {
      a[j + 1] = a[j];
      pm[j + 1] = pm[j];
      j--;
    }
    a[j + 1] = x;
    pm[j + 1] = px;
  }
}

template <class T>
__device__ void sort_segments_smem(SegSmem<T>& S, const long long* seg_ptr, long long c0, long long c1,
                                   long long e0) {
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, nwarps = nthr >> 5, lane = tid & 31;
  for (long long cb = c0; cb < c1; cb += kSegBatch) {
    const int nb = (int)min((long long)kSegBatch, c1 - cb);
    if (tid == 0) {
      S.n_med = 0;
      S.n_big = 0;
    }
    for (int i = tid; i <= nb; i += nthr) S.sseg[i] = (int)(seg_ptr[cb + i] - e0);
    __syncthreads();
    for (int i = tid; i < nb; i += nthr) {
      const int s0 = S.sseg[i], L = S.sseg[i + 1] - s0;
      if (L > 1 && L <= kThreadSortMax) insertion_sort(S.sk + s0, S.perm + s0, L);
      else if (L > kThreadSortMax && L <= kWarpSortMax) S.med[atomicAdd(&S.n_med, 1)] = (short)i;
      else if (L > kWarpSortMax) S.big[atomicAdd(&S.n_big, 1)] = (short)i;
    }
    __syncthreads();
    const int n_med = S.n_med, n_big = S.n_big;
    for (int q = warp; q < n_med; q += nwarps) {
      const int i = S.med[q];
      bitonic_sort<false>(S.sk + S.sseg[i], S.sseg[i + 1] - S.sseg[i], lane, 32, S.perm + S.sseg[i]);
    }
    for (int q = 0; q < n_big; q++) {  // block-uniform
      const int i = S.big[q];
      bitonic_sort<true>(S.sk + S.sseg[i], S.sseg[i + 1] - S.sseg[i], tid, nthr, S.perm + S.sseg[i]);
    }
    __syncthreads();
  }
}

// Sort the segments of a tile held in S.sk by a second-level bucketing in
// shared memory: bin = (segment, high bits of the row), R = 2^lr bins per
// segment chosen so a bin holds ~4 keys; counting pass, exclusive scan,
// scatter into S.u.sk2, then each bin is sorted by its full key (row, input
// order) by one thread (insertion sort), a warp or the block depending on
// its size.  Bins are (segment, row-prefix) ordered, so the concatenation is
// the segmented sort.  Falls back to per-segment sorting when a tile has more
// than kMaxBins non-empty segments.
template <class T>
__device__ void sort_tile_smem(SegSmem<T>& S, const long long* seg_ptr, long long c0, long long c1, long long e0,
                               int m, int row_bits) {
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  const int nw = (m + 31) >> 5;
  for (int i = tid; i < nw; i += nthr) S.sbits[i] = 0u;
  __syncthreads();
  for (long long c = c0 + tid; c < c1; c += nthr) {
    const long long s0 = seg_ptr[c] - e0;
    if (seg_ptr[c + 1] > seg_ptr[c]) atomicOr(&S.sbits[s0 >> 5], 1u << (s0 & 31));
  }
  __syncthreads();
  if (warp == 0) {
    unsigned carry = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
      const int w = w0 + lane;
      const unsigned c = w < nw ? (unsigned)__popc(S.sbits[w]) : 0u;
      const unsigned inc = warp_inclusive_scan(c);
      if (w < nw) S.wpre[w] = carry + inc - c;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) S.nseg = (int)carry;
  }
  __syncthreads();
  const int nseg = S.nseg;
  if (nseg > kMaxBins) {
    sort_segments_smem(S, seg_ptr, c0, c1, e0);
    return;
  }
  int lr = 0;
  while (lr < row_bits && nseg * (2 << lr) <= kMaxBins && nseg * (2 << lr) * 4 <= m) lr++;
  const int R = 1 << lr, sh = row_bits - lr, nbins = nseg * R;
  auto bin_of = [&](int p, unsigned long long k) -> int {
    const int w = p >> 5;
    const int seg = (int)S.wpre[w] + __popc(S.sbits[w] & (0xffffffffu >> (31 - (p & 31)))) - 1;
    return seg * R + (int)(key_row(k) >> sh);
  };
  for (int b = tid; b < nbins; b += nthr) S.v.bk.cursor[b] = 0u;
  __syncthreads();
  for (int p = tid; p < m; p += nthr) atomicAdd(&S.v.bk.cursor[bin_of(p, S.sk[p])], 1u);
  __syncthreads();
  {  // exclusive scan of the bin counts (kMaxBins / kSegThreads = 4 bins per thread)
    constexpr int kPer = kMaxBins / kSegThreads;
    const int b0 = tid * kPer;
    unsigned loc[kPer];
    long long sum = 0;
#pragma unroll
    for (int q = 0; q < kPer; q++) {
      loc[q] = (b0 + q < nbins) ? S.v.bk.cursor[b0 + q] : 0u;
      sum += loc[q];
    }
    long long tot;
    long long run = block_exclusive_scan<long long>(sum, S.scan_tmp, &tot);
#pragma unroll
    for (int q = 0; q < kPer; q++) {
      if (b0 + q < nbins) {
        S.v.bk.bstart[b0 + q] = (unsigned short)run;
        S.v.bk.cursor[b0 + q] = (unsigned)run;
      }
      run += loc[q];
    }
    if (tid == 0) S.v.bk.bstart[nbins] = (unsigned short)m;
  }
  __syncthreads();
  for (int p = tid; p < m; p += nthr) {
    const unsigned long long k = S.sk[p];
    const int b = bin_of(p, k);
    const unsigned slot = atomicAdd(&S.v.bk.cursor[b], 1u);
    S.u.sk2[slot] = k;
    S.perm2[slot] = S.perm[p];
    S.sbin[slot] = (unsigned short)b;
  }
  if (tid == 0) {
    S.n_med = 0;
    S.n_big = 0;
  }
  __syncthreads();
  // bins up to kRankMax keys: every key computes its rank inside its bin and
  // lands directly at its sorted position in S.sk (keys are distinct: the
  // low word is the input index); longer bins are sorted in place by a warp
  // or the block and copied back.
  for (int b = tid; b < nbins; b += nthr) {
    const int L = S.v.bk.bstart[b + 1] - S.v.bk.bstart[b];
    if (L > kRankMax && L <= kWarpSortMax) S.med[atomicAdd(&S.n_med, 1)] = (short)b;
    else if (L > kWarpSortMax) S.big[atomicAdd(&S.n_big, 1)] = (short)b;
  }
  for (int q = tid; q < m; q += nthr) {
    const int b = S.sbin[q];
    const int s0 = S.v.bk.bstart[b], e0b = S.v.bk.bstart[b + 1];
    if (e0b - s0 <= kRankMax) {
      const unsigned long long k = S.u.sk2[q];
      int r = 0;
      for (int j = s0; j < e0b; j++) r += (S.u.sk2[j] < k);
      S.sk[s0 + r] = k;
      S.perm[s0 + r] = S.perm2[q];
    }
  }
  __syncthreads();
  const int n_med = S.n_med, n_big = S.n_big;
  for (int q = warp; q < n_med; q += nwarps) {
    const int b = S.med[q];
    const int s0 = S.v.bk.bstart[b], L = S.v.bk.bstart[b + 1] - s0;
    bitonic_sort<false>(S.u.sk2 + s0, L, lane, 32, S.perm2 + s0);
    for (int i = lane; i < L; i += 32) {
      S.sk[s0 + i] = S.u.sk2[s0 + i];
      S.perm[s0 + i] = S.perm2[s0 + i];
    }
  }
  for (int q = 0; q < n_big; q++) {
    const int b = S.big[q];
    const int s0 = S.v.bk.bstart[b], L = S.v.bk.bstart[b + 1] - s0;
    bitonic_sort<true>(S.u.sk2 + s0, L, tid, nthr, S.perm2 + s0);
    for (int i = tid; i < L; i += nthr) {
      S.sk[s0 + i] = S.u.sk2[s0 + i];
      S.perm[s0 + i] = S.perm2[s0 + i];
    }
    __syncthreads();
  }
  __syncthreads();
}

// Reduce the runs of one chunk [b, b+cm) of a sorted tile whose keys are in
// S.sk[0..cm).  gk: the tile's keys in global memory (runs that cross the
// chunk end continue there; nullptr when the chunk is the whole tile).
// Leaves S.u.rv[p] = run value at kept heads, S.v.excl[0..cm] = exclusive kept
// counts (S.v.excl[cm] = chunk total) and returns the chunk total.
template <class T, class VS>
__device__ long long chunk_reduce(SegSmem<T>& S, long long b, int cm, long long m, const unsigned long long* gk,
                                  const long long* seg_ptr, long long c0, long long c1, long long e0, VS vs,
                                  int mode, int prune, const T* vslot = nullptr) {
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nw = (cm + 31) >> 5;
  for (int i = tid; i < nw; i += nthr) S.sbits[i] = 0u;
  __syncthreads();
  for (long long c = c0 + tid; c < c1; c += nthr) {
    const long long s0 = seg_ptr[c] - e0 - b;
    if (s0 >= 0 && s0 < cm && seg_ptr[c + 1] > seg_ptr[c]) atomicOr(&S.sbits[s0 >> 5], 1u << (s0 & 31));
  }
  __syncthreads();
  // pass A (strided, independent gathers): head bits and raw values
  for (int base = 0; base < cm; base += nthr) {
    const int p = base + tid;
    bool head = false;
    if (p < cm) {
      const unsigned long long k = S.sk[p];
      const unsigned row = key_row(k);
      unsigned prev;
      if (p > 0) prev = key_row(S.sk[p - 1]);
      else prev = (b > 0) ? key_row(gk[b - 1]) : ~row;
      head = bit_at(S.sbits, p) || row != prev;
      S.u.rv[p] = vslot ? vslot[S.perm[p]] : vs((unsigned long long)key_idx(k));
    }
    const unsigned hb = __ballot_sync(0xffffffffu, head);
    if (lane == 0 && base + warp * 32 < cm) S.hbits[(base >> 5) + warp] = hb;
  }
  __syncthreads();
  // pass B (blocked): run reduction at heads
  const int pb = tid * kItems, pe = min(pb + kItems, cm);
  int cnt = 0;
  for (int p = pb; p < pe; p++) {
    unsigned short f = 0;
    if (bit_at(S.hbits, p)) {
      const int q = next_bit(S.hbits, p + 1, cm);
      T v;
      if (q < cm || gk == nullptr || b + cm >= m) {
        if (q == p + 1) {
          v = S.u.rv[p];
        } else {
          const T* rvp = S.u.rv + p;
          v = reduce_run<T>([&](long long i) -> T { return rvp[i]; }, q - p, mode);
        }
      } else {  // the run may continue past the chunk, in global memory
        const unsigned row = key_row(S.sk[p]);
        const long long c = seg_of(seg_ptr, c0, c1, e0 + b + p);
        const long long s_end = seg_ptr[c + 1] - e0;
        long long qg = b + cm;
        while (qg < s_end && key_row(gk[qg]) == row) qg++;
        const T* rvp = S.u.rv + p;
        const long long in_chunk = cm - p;
        const unsigned long long* gkp = gk + b + p;
        v = reduce_run<T>(
            [&](long long i) -> T { return i < in_chunk ? rvp[i] : vs((unsigned long long)key_idx(gkp[i])); },
            qg - (b + p), mode);
      }
      if (!prune || v != T(0)) {
        f = 1;
        S.u.rv[p] = v;
      }
    }
    S.v.excl[p] = f;
    cnt += f;
  }
  long long total;
  const long long off = block_exclusive_scan<long long>((long long)cnt, S.scan_tmp, &total);
  unsigned run = (unsigned)off;
  for (int p = pb; p < pe; p++) {
    const unsigned f = S.v.excl[p];
    S.v.excl[p] = (unsigned short)run;
    run += f;
  }
  if (tid == 0) S.v.excl[cm] = (unsigned short)total;
  __syncthreads();
  return total;
}

// write the kept entries of a chunk and the col_ptr of segments starting in it
template <class T>
__device__ void chunk_write(SegSmem<T>& S, long long b, int cm, bool last_chunk, long long base_out,
                            const long long* seg_ptr, long long c0, long long c1, long long e0, SegOut<T>& out,
                            long long ptr_bias = 0) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int p = tid; p < cm; p += nthr) {
    const unsigned a = S.v.excl[p], n = S.v.excl[p + 1];
    if (n != a) {
      const long long o = base_out + a;
      out.row_idx[o] = (int)key_row(S.sk[p]);
      out.vals[o] = S.u.rv[p];
    }
  }
  for (long long c = c0 + tid; c < c1; c += nthr) {
    const long long s0 = seg_ptr[c] - e0 - b;
    if (s0 >= 0 && (s0 < cm || (last_chunk && s0 == cm))) out.col_ptr[c] = (int)(base_out - ptr_bias + S.v.excl[s0]);
  }
}

// Process tile t of the engine (all threads of the block call it).
// kTmp = false: chained-scan output straight to the final CSC.
// kTmp = true : no look-back; the tile's compacted entries go to the
//               temporaries at the tile's own input offset e0, col_ptr gets
//               tile-local offsets and tile_total[t] the count -- a later
//               grid-wide pass adds the tile prefixes (persistent kernels).
// vslot: bucketed values addressed by bucket slot (nullptr: gather by index).
template <bool kTmp, class T, class VS>
__device__ void process_tile(SegSmem<T>& S, const SegIn& in, VS vs, int mode, int prune, SegOut<T>& out,
                             long long t, long long n_tiles, const T* vslot, long long* tile_total) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    const long long c0 = in.tile_c0[t], c1 = in.tile_c0[t + 1];
    S.c0 = c0;
    S.c1 = c1;
    S.e0 = in.seg_ptr[c0];
    S.m = in.seg_ptr[c1] - S.e0;
  }
  __syncthreads();
  const long long c0 = S.c0, c1 = S.c1, e0 = S.e0, m = S.m;
  const long long* seg_ptr = in.seg_ptr;

  if (m <= kCap) {
    // ---------------- shared-memory path: the whole tile in one chunk ----------------
    for (long long i = tid; i < m; i += nthr) {
      const unsigned long long k = in.keys[e0 + i];
      S.sk[i] = k;
      S.perm[i] = (unsigned short)i;
      if (vslot == nullptr) vs.prefetch((unsigned long long)key_idx(k));
    }
    __syncthreads();
    sort_tile_smem(S, seg_ptr, c0, c1, e0, (int)m, in.row_bits);
    const long long total =
        chunk_reduce<T>(S, 0, (int)m, m, nullptr, seg_ptr, c0, c1, e0, vs, mode, prune, vslot ? vslot + e0 : nullptr);
    long long P;
    if (kTmp) {
      P = e0;
      if (tid == 0) tile_total[t] = total;
    } else {
      if (warp == 0) {
        const unsigned long long pre = tile_lookback_warp(out.tile_states, t, (unsigned long long)total);
        if (lane == 0) S.prefix = pre;
      }
      __syncthreads();
      P = (long long)S.prefix;
    }
    chunk_write<T>(S, 0, (int)m, true, P, seg_ptr, c0, c1, e0, out, kTmp ? e0 : 0);
    if (!kTmp && t == n_tiles - 1 && tid == 0) {
      out.col_ptr[in.n_seg] = (int)(P + total);
      out.info[0] = P + total;
    }
    __syncthreads();
    return;
  }

  // ---------------- oversized tile: sort in global, then stream chunks ----------------
  unsigned long long* gk = in.keys + e0;
  for (long long c = c0; c < c1; c++) {  // block-uniform
    const long long L = seg_ptr[c + 1] - seg_ptr[c];
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
        for (int bb = 0; bb < in.idx_bits; bb += 8) { shifts[np] = bb; nbits[np] = min(8, in.idx_bits - bb); np++; }
      for (int bb = 0; bb < in.row_bits; bb += 8) { shifts[np] = 32 + bb; nbits[np] = min(8, in.row_bits - bb); np++; }
      block_radix_sort_global(seg, in.keys_alt + seg_ptr[c], L, shifts, nbits, np, S.u.rs.hist, S.u.rs.wcnt);
    }
  }
  __syncthreads();
  long long total = 0;
  long long P = e0;
  if (!kTmp) {
    for (long long b = 0; b < m; b += kCap) {
      const int cm = (int)min((long long)kCap, m - b);
      for (int i = tid; i < cm; i += nthr) S.sk[i] = gk[b + i];
      __syncthreads();
      total += chunk_reduce<T>(S, b, cm, m, gk, seg_ptr, c0, c1, e0, vs, mode, prune);
    }
    if (warp == 0) {
      const unsigned long long pre = tile_lookback_warp(out.tile_states, t, (unsigned long long)total);
      if (lane == 0) S.prefix = pre;
    }
    __syncthreads();
    P = (long long)S.prefix;
  }
  long long run_base = 0;
  for (long long b = 0; b < m; b += kCap) {
    const int cm = (int)min((long long)kCap, m - b);
    for (int i = tid; i < cm; i += nthr) S.sk[i] = gk[b + i];
    __syncthreads();
    const long long ctot = chunk_reduce<T>(S, b, cm, m, gk, seg_ptr, c0, c1, e0, vs, mode, prune);
    chunk_write<T>(S, b, cm, b + cm >= m, P + run_base, seg_ptr, c0, c1, e0, out, kTmp ? e0 : 0);
    run_base += ctot;
    __syncthreads();
  }
  if (kTmp) {
    if (tid == 0) tile_total[t] = run_base;
  } else if (t == n_tiles - 1 && tid == 0) {
    out.col_ptr[in.n_seg] = (int)(P + total);
    out.info[0] = P + total;
  }
  __syncthreads();
}

// Claim tiles in ticket order until none are left (persistent use), or one
// tile per block (grid == n_tiles).  Ticket order keeps the chained scan
// deadlock-free: every predecessor of a claimed tile is already claimed.
template <class T, class VS>
__device__ void run_tiles(SegSmem<T>& S, const SegIn& in, VS vs, int mode, int prune, SegOut<T>& out,
                          long long n_tiles) {
  while (true) {
    if (threadIdx.x == 0) S.tile = (long long)atomicAdd(out.ticket, 1u);
    __syncthreads();
    const long long t = S.tile;
    __syncthreads();
    if (t >= n_tiles) break;
    process_tile<false, T>(S, in, vs, mode, prune, out, t, n_tiles, nullptr, nullptr);
  }
}

template <class T, class VS>
__global__ void __launch_bounds__(kSegThreads, 3)
seg_tile_kernel(SegIn in, VS vs, int mode, int prune, SegOut<T> out, long long n_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SegSmem<T>& S = *reinterpret_cast<SegSmem<T>*>(smem_raw);
  run_tiles<T>(S, in, vs, mode, prune, out, n_tiles);
}

// ------------------------------------------------------------------------
// bucket counting / scan / scatter

// count column occupancy of COO triplets; validate coordinates and record the
// first invalid triplet index (csc.py:215-221 / coo.py:54-61 report it).
constexpr int kCntItems = 4;  // consecutive elements per thread (ILP)

// Warp-aggregated bucket increment: lanes with the same bucket share one
// atomic; returns this lane's slot when kWantSlot.
template <bool kWantSlot>
AS_DEVICE_INLINE unsigned bucket_inc(unsigned act, unsigned bucket, unsigned* counts) {
  const unsigned peers = __match_any_sync(act, bucket);
  const unsigned rank = __popc(peers & lanemask_lt());
  unsigned b = 0;
  if (kWantSlot) {
    if (rank == 0) b = atomicAdd(&counts[bucket], (unsigned)__popc(peers));
    b = __shfl_sync(peers, b, __ffs(peers) - 1);
    return b + rank;
  }
  if (rank == 0) atomicAdd(&counts[bucket], (unsigned)__popc(peers));
  return 0;
}

// Count column occupancy of COO triplets (kScatter = false) or scatter them
// into their column buckets (kScatter = true): key = (row << 32) | (i + idx_off).
// Out-of-range triplets are skipped; the first one is recorded in *bad
// (csc.py:215-221 / coo.py:54-61 report it).  Each thread handles kCntItems
// consecutive triplets so a warp streams 32*kCntItems contiguous elements.
template <class IdxT, bool kScatter>
__global__ void __launch_bounds__(256)
coo_bucket_kernel(long long n, const IdxT* __restrict__ rows, const IdxT* __restrict__ cols, long long n_rows,
                  long long n_cols, unsigned* counts, long long* bad, const long long* __restrict__ seg_ptr,
                  unsigned long long* __restrict__ keys, unsigned long long idx_off) {
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * blockDim.x * kCntItems;
  for (long long wbase = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * kCntItems; wbase < n;
       wbase += wstride) {
    const long long i0 = wbase + (long long)lane * kCntItems;
    long long r[kCntItems], c[kCntItems];
#pragma unroll
    for (int k = 0; k < kCntItems; k++) {
      const long long i = i0 + k;
      r[k] = i < n ? (long long)__ldg(&rows[i]) : 0;
      c[k] = i < n ? (long long)__ldg(&cols[i]) : 0;
    }
#pragma unroll
    for (int k = 0; k < kCntItems; k++) {
      const long long i = i0 + k;
      const bool in = i < n;
      const bool ok = in && r[k] >= 0 && r[k] < n_rows && c[k] >= 0 && c[k] < n_cols;
      if (!kScatter && in && !ok) atomicMin((unsigned long long*)bad, (unsigned long long)i);
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const unsigned slot = bucket_inc<kScatter>(act, (unsigned)c[k], counts);
        if (kScatter)
          keys[seg_ptr[c[k]] + slot] = ((unsigned long long)r[k] << 32) | (unsigned long long)(i + idx_off);
      }
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
static __global__ void __launch_bounds__(256) row_count_kernel(long long nnz, const int* __restrict__ row_idx,
                                                               unsigned* counts) {
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * blockDim.x * kCntItems;
  for (long long wbase = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * kCntItems; wbase < nnz;
       wbase += wstride) {
    const long long i0 = wbase + (long long)lane * kCntItems;
    unsigned r[kCntItems];
#pragma unroll
    for (int k = 0; k < kCntItems; k++) r[k] = i0 + k < nnz ? (unsigned)__ldg(&row_idx[i0 + k]) : 0u;
#pragma unroll
    for (int k = 0; k < kCntItems; k++) {
      const bool in = i0 + k < nnz;
      const unsigned act = __ballot_sync(0xffffffffu, in);
      if (in) bucket_inc<false>(act, r[k], counts);
    }
  }
}

// Tile t of the engine owns the segments whose start lies in
// [t*kTileNom, (t+1)*kTileNom): tile_c0[t] = first segment with start >=
// t*kTileNom.  Segment i (start s, end e) owns the boundaries in (s, e].
AS_DEVICE_INLINE void emit_tile_bounds(long long i, long long s, long long e, long long n_tiles, long long* tile_c0) {
  for (long long t = s / kTileNom + 1; t * kTileNom <= e && t < n_tiles; t++) tile_c0[t] = i + 1;
}

AS_DEVICE_INLINE void finish_tile_bounds(long long n_seg, long long N, long long n_tiles, long long* tile_c0) {
  tile_c0[0] = 0;
  for (long long t = N / kTileNom + 1; t < n_tiles; t++) tile_c0[t] = n_seg;
  tile_c0[n_tiles] = n_seg;
}

// tile_c0 from an existing seg_ptr (used when the scan did not produce it)
static __global__ void tile_bounds_kernel(const long long* seg_ptr, long long n_seg, long long n_tiles,
                                          long long* tile_c0) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_seg; i += stride)
    emit_tile_bounds(i, seg_ptr[i], seg_ptr[i + 1], n_tiles, tile_c0);
  if (blockIdx.x == 0 && threadIdx.x == 0) finish_tile_bounds(n_seg, seg_ptr[n_seg], n_tiles, tile_c0);
}

// exclusive scan counts[0..n) -> seg_ptr[0..n] (int64) and zero counts (so
// they can serve as fill cursors).  Chained scan, 4096 counts per tile.
// With tile_c0 != nullptr it also emits the engine's tile -> segment map.
constexpr int kScanThreads = 256, kScanItems = 16;
static __global__ void __launch_bounds__(kScanThreads)
count_scan_kernel(unsigned* counts, long long n, long long* seg_ptr, unsigned long long* states, unsigned* ticket,
                  long long* tile_c0, long long n_tiles) {
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
      if (tile_c0 != nullptr) emit_tile_bounds(i, run, run + v[k], n_tiles, tile_c0);
    }
    run += v[k];
  }
  if (t == gridDim.x - 1 && threadIdx.x == 0) {
    seg_ptr[n] = (long long)s_prefix + total;
    if (tile_c0 != nullptr) finish_tile_bounds(n, (long long)s_prefix + total, n_tiles, tile_c0);
  }
}

// scatter the elements of a CSC.  kByRow: bucket = row, key = (col << 32) | k
// (transpose); else bucket = col, key = (row << 32) | k  (flush base).
// Each thread takes kCntItems consecutive elements: one binary search on
// col_ptr, then a forward walk.
template <bool kByRow>
__global__ void __launch_bounds__(256)
csc_scatter_kernel(long long n_cols, long long nnz, const int* __restrict__ col_ptr, const int* __restrict__ row_idx,
                   const long long* __restrict__ seg_ptr, unsigned* fill, unsigned long long* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * blockDim.x * kCntItems;
  for (long long wbase = ((long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) * kCntItems; wbase < nnz;
       wbase += wstride) {
    const long long k0 = wbase + (long long)lane * kCntItems;
    unsigned r[kCntItems], c[kCntItems];
    if (k0 < nnz) {
      long long cc = upper_bound_dev(col_ptr, n_cols + 1, (int)k0) - 1;
#pragma unroll
      for (int q = 0; q < kCntItems; q++) {
        const long long k = k0 + q;
        if (k < nnz) {
          while (col_ptr[cc + 1] <= k) cc++;
          r[q] = (unsigned)__ldg(&row_idx[k]);
          c[q] = (unsigned)cc;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kCntItems; q++) {
      const long long k = k0 + q;
      const bool in = k < nnz;
      const unsigned act = __ballot_sync(0xffffffffu, in);
      if (in) {
        const unsigned bucket = kByRow ? r[q] : c[q];
        const unsigned other = kByRow ? c[q] : r[q];
        const unsigned slot = bucket_inc<true>(act, bucket, fill);
        keys[seg_ptr[bucket] + slot] = ((unsigned long long)other << 32) | (unsigned long long)k;
      }
    }
  }
}

// ------------------------------------------------------------------------
// host-side launcher of the tile engine (one kernel, chained-scan compaction)
inline long long seg_engine_tiles(long long n_upper) {
  return n_upper > 0 ? (n_upper + kTileNom - 1) / kTileNom : 1;
}

template <class T>
inline int launch_seg_engine(const long long* seg_ptr, const long long* tile_c0, long long n_seg, long long n_upper,
                             unsigned long long* keys,
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
  SegIn in{seg_ptr, n_seg, n_upper, keys, keys_alt, row_bits, idx_bits, presorted, tile_c0};
  SegOut<T> out{col_ptr, row_idx, vals, info, states, ticket};
  const long long n_tiles = seg_engine_tiles(n_upper);
  seg_tile_kernel<T, ValSrc<T>><<<(unsigned)n_tiles, kSegThreads, smem, st>>>(in, vs, mode, prune, out, n_tiles);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

}  // namespace as
