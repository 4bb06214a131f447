// sortreduce.cuh -- the lean single-level sort-reduce kernel behind
// COO->CSC construction (csc.canonicalize, csc.py:148-193), the insertion-log
// flush (rbt.to_csc over RbtStore semantics, rbt.py:371-458) and the CSC
// transpose (_kernels.transpose, _kernels.py:130-150), for inputs whose
// per-CTA chunk fits in registers (n <= grid x 4096 elements).
//
// One cooperative launch of exactly the co-resident grid, three phases:
//
//   P1  every CTA loads its chunk ONCE (vectorised, 8 elements per thread in
//       registers), validates it, computes the coarse bucket (a range of
//       consecutive output columns) and the bucket-local 32-bit key
//       (local column << minor_bits | minor), counts the chunk per bucket in
//       shared memory (the atomic's return value is the element's rank in
//       its (CTA, bucket) run), reserves the CTA's range inside every
//       non-empty bucket with one global atomic and stages the chunk in
//       bucket order in shared memory.                          [grid barrier]
//   P2  every CTA scans the bucket totals (the bucket starts stay in shared
//       memory for P3) and writes its staged chunk out run by run: key, input
//       index and value of consecutive elements of a bucket go to
//       consecutive slots.                                      [grid barrier]
//   P3  CTA g takes buckets g, g + G, ... (static: the buckets are sized to
//       ~0.85 of a tile and rounded to whole waves).  A bucket of m <= 2048
//       elements is loaded into registers / shared memory, counting-sorted
//       over <= 1024 bins of its key range (bins never straddle a column),
//       every element ranks itself inside its bin by (key, input index)
//       (large bins: warp / block bitonic), runs of equal keys reduce in the
//       reference's order (np.add.reduceat pairwise, or last wins), exact
//       zeros are pruned, the kept count is published to the group
//       look-back, and rows / values / col_ptr go straight to their final
//       CSC positions.  A bucket above the tile (a heavy column) is sorted
//       by a block radix sort in global memory and streamed (rare path).
//
// Compared with the general bucket kernel (persist.cuh, which also serves
// SpGEMM's pre-bucketed mode and the two-level scatter of large inputs) the
// chunk is read once, keys are 32-bit, no per-element 64-bit arithmetic on
// the hot path and no stack frame: runs of several values are summed by their
// lane one at a time with the pairwise recursion's stack in shared memory.
#pragma once

#include <cooperative_groups.h>

#include "tile_common.cuh"

namespace as {
namespace sr {

// CTA shape (experiments: AS_SR_THREADS / AS_SR_TILE / AS_SR_MINB; measured
// best: 512 threads, 2048-element tiles, 2 CTAs per SM)
#ifndef AS_SR_THREADS
#define AS_SR_THREADS 512
#endif
#ifndef AS_SR_TILE
#define AS_SR_TILE 2048
#endif
#ifndef AS_SR_MINB
#define AS_SR_MINB 2
#endif
constexpr int kThreads = AS_SR_THREADS;
constexpr int kMinBlocks = AS_SR_MINB;         // co-resident CTAs per SM
constexpr int kPer = 8;                        // P1: elements per thread (two groups of 4)
// P1 values by bulk copies (cp.async.bulk on an mbarrier, UBLKCP / SYNCS in
// the SASS) instead of per-thread cp.async: measured no faster (ncu build
// 47.0 vs 47.2 us, transpose 46.8 vs 45.6 us; event time +1-2 us with 1, 4, 8
// or 16 copies per CTA), so off by default -- a build knob
#ifndef AS_SR_BULK
#define AS_SR_BULK 0
#endif
constexpr bool kBulkVals = AS_SR_BULK != 0;
#ifndef AS_SR_BULK_PARTS
#define AS_SR_BULK_PARTS 4
#endif
constexpr int kBulkParts = AS_SR_BULK_PARTS;
constexpr int kChunkMax = kThreads * kPer;     // elements per CTA chunk
constexpr int kTile = AS_SR_TILE;              // elements of a shared-memory tile
constexpr int kTP = kTile / kThreads;          // tile elements per thread
#ifndef AS_SR_NB
#define AS_SR_NB (AS_SR_TILE / 2)
#endif
constexpr int kNB = AS_SR_NB;                  // bins per tile
constexpr int kMaxW = 1024;                    // columns per bucket
constexpr int kRankMax = 32;                   // bins up to this rank by counting
#ifndef AS_SR_RANK_UNROLL
#define AS_SR_RANK_UNROLL 1
#endif
constexpr int kRankUnroll = AS_SR_RANK_UNROLL;  // unroll of the in-bin rank loop
constexpr int kColCache = 1024;                // CSC source: cached column pointers of a chunk
constexpr int kMaxCb = 4096;                   // buckets (shared-memory tables)
constexpr int kRankBits = 12;                  // P1 rank in (CTA, bucket): < kChunkMax
#ifdef AS_SR_DEBUG
constexpr bool kDbg = true;  // phase timestamps / step clocks / early exits (tools/sr_time.py)
#else
constexpr bool kDbg = false;
#endif

// ------------------------------------------------------------------------
// element sources (major = output column, minor = output row)

template <class IdxT, class T>
struct Coo {  // COO triplets: major = col, minor = row (construction, the flush's write log)
  const IdxT* rows;
  const IdxT* cols;
  const T* vals;
  long long n, n_rows, n_cols;
};

template <class T>
struct Csc {  // elements of a CSC; by_row: major = row, minor = col (transpose)
  const int* ptr;
  const int* idx;
  const T* vals;
  long long n_cols, nnz;
  bool by_row;
};

struct None {};

template <class T, class S1, class S2>
struct Args {
  S1 s1;
  S2 s2;
  long long n1, n;                 // elements of s1; of s1 ++ s2
  long long n_out_cols;            // output columns (major range)
  int minor_bits;
  long long n_minor;               // minor index range [0, n_minor)
  long long ncb;
  unsigned long long cb_mul;       // bucket(c) = (c * cb_mul) >> 32
  int mode, prune;
  // workspace
  // Workspace (nothing needs zeroing before the launch -- a memset costs ~4.7 us
  // of event time on B200 -- P1 zeroes what P3 accumulates into)
  unsigned* loffT;                 // [(ncb + 1) x G]: offset of bucket b inside chunk g's staged run
  unsigned long long* ctr;         // [0] finished CTAs, [1] oversized-bucket scratch allocator (zeroed in P1)
  unsigned long long* tstate;      // [ncb + ncb / 32 + 1] group look-back words
  unsigned* gK;                    // [G x chunk] each chunk's elements in bucket order: keys
  unsigned* gX;                    //   input indices
  T* gV;                           //   values
  long long ch;                    // chunk capacity (elements per CTA)
  long long* cta_bad;              // [grid] first invalid element of each chunk (or n)
  // oversized buckets (rare): radix sort in global memory, run values
  unsigned long long* oK;
  unsigned long long* oK2;
  unsigned* oP;
  unsigned* oP2;
  int* oR;
  T* oV;
  int idx_bits;
  // outputs
  int* col_ptr;
  int* row_idx;
  T* out_vals;
  long long* info;                 // [0] nnz, [1] first invalid triplet of the COO source (or >= n)
  int stop;                        // diagnostics (AS_SR_STOP): end after phase `stop` (results invalid)
  unsigned long long* phase_ts;    // optional (AS_PHASE_TIMES): [0] first CTA start, [1] last CTA start,
                                   // [2] barrier 1 passed (CTA 0), [3] barrier 2 passed (CTA 0), [4] last CTA end
};

// ------------------------------------------------------------------------
// numpy pairwise summation (pairwise_sum_@TYPE@, loops_utils.h.src) over a
// contiguous shared-memory run; np.add.reduceat applies v[0] + pairwise(v[1:]).
template <class T>
__device__ __forceinline__ T pw_leaf_a(const T* a, int n) {
  if (n < 8) {
    T r = T(-0.0);
    for (int i = 0; i < n; i++) r = r + a[i];
    return r;
  }
  T r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int i;
  for (i = 8; i < n - (n % 8); i += 8) {
    r0 = r0 + a[i];
    r1 = r1 + a[i + 1];
    r2 = r2 + a[i + 2];
    r3 = r3 + a[i + 3];
    r4 = r4 + a[i + 4];
    r5 = r5 + a[i + 5];
    r6 = r6 + a[i + 6];
    r7 = r7 + a[i + 7];
  }
  T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; i++) res = res + a[i];
  return res;
}

// Runs longer than 128 values (n > 128 splits at n2 = n/2 rounded down to a
// multiple of 8, sum(left) + sum(right)), evaluated post-order with an
// explicit stack in the warp's shared-memory slot; the warp serialises its
// lanes' long runs (a thread holds at most one: its other positions lie
// inside the run).  Depth <= 27 for n < 2^31.
struct WarpStack {
  int off[32];
  int n[32];
  double left[32];
  unsigned char stage[32];
};

template <class T, class Get>
__device__ T pw_stack(Get get, int n, WarpStack& S) {
  auto leaf = [&](int o, int len) -> T {
    if (len < 8) {
      T r = T(-0.0);
#pragma unroll 1
      for (int i = 0; i < len; i++) r = r + get(o + i);
      return r;
    }
    T r0 = get(o), r1 = get(o + 1), r2 = get(o + 2), r3 = get(o + 3), r4 = get(o + 4), r5 = get(o + 5),
      r6 = get(o + 6), r7 = get(o + 7);
    int i;
#pragma unroll 1
    for (i = 8; i < len - (len % 8); i += 8) {
      r0 = r0 + get(o + i);
      r1 = r1 + get(o + i + 1);
      r2 = r2 + get(o + i + 2);
      r3 = r3 + get(o + i + 3);
      r4 = r4 + get(o + i + 4);
      r5 = r5 + get(o + i + 5);
      r6 = r6 + get(o + i + 6);
      r7 = r7 + get(o + i + 7);
    }
    T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
#pragma unroll 1
    for (; i < len; i++) res = res + get(o + i);
    return res;
  };
  if (n <= 128) return leaf(0, n);
  int sp = 1;
  S.off[0] = 0;
  S.n[0] = n;
  S.stage[0] = 0;
  T ret = T(0);
  bool have = false;
  while (true) {
    if (!have) {
      const int top = sp - 1;
      if (S.n[top] <= 128) {
        ret = leaf(S.off[top], S.n[top]);
        have = true;
        sp--;
      } else {
        int n2 = S.n[top] / 2;
        n2 -= n2 % 8;
        S.off[sp] = S.off[top];
        S.n[sp] = n2;
        S.stage[sp] = 0;
        sp++;
      }
    } else {
      if (sp == 0) return ret;
      const int top = sp - 1;
      int n2 = S.n[top] / 2;
      n2 -= n2 % 8;
      if (S.stage[top] == 0) {
        S.left[top] = (double)ret;
        S.stage[top] = 1;
        have = false;
        S.off[sp] = S.off[top] + n2;
        S.n[sp] = S.n[top] - n2;
        S.stage[sp] = 0;
        sp++;
      } else {
        ret = (T)S.left[top] + ret;
        sp--;
      }
    }
  }
}

// Block-wide exclusive scan of 32-bit counts (totals < 2^32); `smem` holds
// kThreads / 32 + 1 words.  Every thread calls.
__device__ __forceinline__ unsigned block_scan_u32(unsigned v, unsigned* smem, unsigned* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned w = lane < kThreads / 32 ? smem[lane] : 0u;
    unsigned wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    if (lane < kThreads / 32) smem[lane] = wi - w;
    if (lane == kThreads / 32 - 1) smem[kThreads / 32] = wi;
  }
  __syncthreads();
  const unsigned res = smem[warp] + inc - v;
  *total = smem[kThreads / 32];
  __syncthreads();
  return res;
}

// ------------------------------------------------------------------------
// shared memory

template <class T>
struct TileSmem {  // P3
  union {
    struct {
      T V[kTile];                        // tile values (tile order)
      unsigned TK[kTile];                // keys, bin order
      unsigned TX[kTile];                // input indices, bin order
      union {
        unsigned long long BK[kTile];    // bins above kRankMax: (key << 32 | index) for the bitonic sort
        T RV[kTile];                     // then: run values by sorted position (heads only)
      };
    } a;
    struct {                             // oversized path
      unsigned hist[256];
      unsigned wcnt[256 * (kThreads / 32)];
      unsigned ckept[kMaxW];
    } r;
  } u;
  unsigned SK[kTile];                    // sorted keys
  unsigned short SI[kTile];              // tile index of each sorted position
  unsigned short BI[kTile];              // bitonic payload (tile index)
  unsigned cnt[kNB];                     // bin counts (zero between tiles)
  unsigned bs[kNB + 1];                  // bin starts
  unsigned kw[kTile / 32];               // kept bits of sorted positions [32 w, 32 w + 32)
  unsigned kwp[kTile / 32 + 1];          // kept outputs before word w
  unsigned short cstart[kMaxW + 1];      // first sorted position of each local column
  unsigned short big[kNB];               // bins above kRankMax
  WarpStack wst[kThreads / 32];          // long pairwise runs
  long long scan[kThreads / 32 + 1];
  unsigned scan32[kThreads / 32 + 1];
  int n_big;
  long long prefix;
};

// Shared-memory layout: the first column of every bucket ([ncb + 1], kept
// for P3), then P1's tables -- colc [kColCache + 1], hist [ncb], loff
// [ncb + 1] -- and the chunk's staging (values in input order, keys and
// local indices in bucket order); P3's tile reuses everything after the
// first table.
struct Layout {
  long long persist;  // bytes of the bucket column table
  long long hist, loff, colc, st_key, st_idx, st_val, p12_end;
  long long tile_off, total;
};

template <class T>
__host__ __device__ inline Layout layout(long long ncb, long long chunk) {
  Layout L;
  auto al = [](long long x) { return (x + 15) & ~15ll; };
  L.persist = al(4 * (ncb + 1));
  long long o = L.persist;
  L.hist = o;
  o = al(o + 4 * ncb);
  L.loff = o;
  o = al(o + 4 * (ncb + 1));
  L.colc = o;
  o = al(o + 4 * (kColCache + 1));
  L.st_val = o;
  o = al(o + (long long)sizeof(T) * chunk);
  L.st_key = o;
  o = al(o + 4 * chunk);
  L.st_idx = o;
  o = al(o + 2 * chunk);
  L.p12_end = o;
  L.tile_off = L.persist;
  L.total = o > L.persist + (long long)sizeof(TileSmem<T>) ? o : L.persist + (long long)sizeof(TileSmem<T>);
  return L;
}

// ------------------------------------------------------------------------
// P1 element loading: group of 4 consecutive elements [e0, e0 + 4) of the
// concatenated source space; out[k] = (major, minor, value), ok bit k.

template <class IdxT>
AS_DEVICE_INLINE void ld4_idx(const IdxT* p, long long i, long long hi, long long* out) {
  const bool al = ((reinterpret_cast<unsigned long long>(p + i) & 15ull) == 0);
  if (i + 3 < hi && sizeof(IdxT) == 4 && al) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(p + i));
    out[0] = q.x;
    out[1] = q.y;
    out[2] = q.z;
    out[3] = q.w;
  } else if (i + 3 < hi && sizeof(IdxT) == 8 && al) {
    const longlong2 a = __ldg(reinterpret_cast<const longlong2*>(p + i));
    const longlong2 b = __ldg(reinterpret_cast<const longlong2*>(p + i + 2));
    out[0] = a.x;
    out[1] = a.y;
    out[2] = b.x;
    out[3] = b.y;
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++) out[k] = (i + k < hi) ? (long long)__ldg(&p[i + k]) : 0;
  }
}

template <class T>
AS_DEVICE_INLINE void ld4_val(const T* p, long long i, long long hi, T* out) {
  const bool al = ((reinterpret_cast<unsigned long long>(p + i) & 15ull) == 0);
  if (i + 3 < hi && sizeof(T) == 8 && al) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p + i));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p + i + 2));
    out[0] = (T)a.x;
    out[1] = (T)a.y;
    out[2] = (T)b.x;
    out[3] = (T)b.y;
  } else if (i + 3 < hi && sizeof(T) == 4 && al) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p + i));
    out[0] = (T)a.x;
    out[1] = (T)a.y;
    out[2] = (T)a.z;
    out[3] = (T)a.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++) out[k] = (i + k < hi) ? __ldg(&p[i + k]) : T(0);
  }
}

// Chunk context of a CSC source: its column pointers over the chunk, cached
// in shared memory when they fit.
struct CscCtx {
  long long cb, ce;  // columns holding the first / last element of the chunk's part of this source
  bool cached;
};

// upper_bound(ptr[0..N), x) by the whole block: a sample of 512 entries per
// round, __syncthreads_count of the entries <= x (ptr is non-decreasing), so
// a search over N entries takes ceil(log512 N) round trips instead of log2 N.
__device__ inline long long block_upper_bound(const int* ptr, long long N, long long x) {
  long long base = 0, len = N;  // answer = base + #{j < len : ptr[base + j] <= x}
  while (len > kThreads) {
    const long long step = (len + kThreads - 1) / kThreads;
    const long long j = (long long)threadIdx.x * step;
    const int c = __syncthreads_count(j < len && __ldg(&ptr[base + j]) <= x);
    if (c == 0) return base;
    // samples 0..c-1 are <= x: the answer lies in (base + (c-1)*step, base + c*step]
    base += (long long)(c - 1) * step + 1;
    len = min(step - 1, N - base);
    if (len <= 0) return base;
  }
  const int c = __syncthreads_count((long long)threadIdx.x < len && __ldg(&ptr[base + threadIdx.x]) <= x);
  return base + c;
}

// lo / hi: the chunk's element range inside this source (every thread calls)
template <class T>
__device__ void csc_ctx(const Csc<T>& s, long long lo, long long hi, int* colc, CscCtx* ctx) {
  if (lo >= hi) {  // (uniform)
    ctx->cb = ctx->ce = 0;
    ctx->cached = false;
    return;
  }
  ctx->cb = block_upper_bound(s.ptr, s.n_cols + 1, lo) - 1;
  ctx->ce = block_upper_bound(s.ptr, s.n_cols + 1, hi - 1);
  ctx->cached = (ctx->ce - ctx->cb) <= kColCache;
  if (ctx->cached)
    for (long long c = ctx->cb + threadIdx.x; c <= ctx->ce; c += blockDim.x) colc[c - ctx->cb] = __ldg(&s.ptr[c]);
  __syncthreads();
}

// asynchronous copy of one value into shared memory (cp.async: no register)
template <class T>
AS_DEVICE_INLINE void cp_async_val(T* sdst, const T* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  if constexpr (sizeof(T) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}

// values of a group of 4: two 16-byte copies when both sides are aligned
template <class T>
AS_DEVICE_INLINE void cp_async_vals4(T* sdst, const T* gsrc, long long i, long long hi) {
  if (i + 3 < hi && ((reinterpret_cast<unsigned long long>(gsrc + i) & 15ull) == 0)) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    if constexpr (sizeof(T) == 8) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc + i) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16), "l"(gsrc + i + 2) : "memory");
    } else {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc + i) : "memory");
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (i + k < hi) cp_async_val(sdst + k, gsrc + i + k);
  }
}

template <class IdxT, class T>
__device__ __forceinline__ unsigned ld_group(const Coo<IdxT, T>& s, const CscCtx&, const int*, long long e0,
                                             long long hi, unsigned* mj, unsigned* mn, T* vdst, long long* bad,
                                             bool vbulk = false) {
  long long r[4], c[4];
  ld4_idx(s.rows, e0, hi, r);
  ld4_idx(s.cols, e0, hi, c);
  if (!vbulk) cp_async_vals4(vdst, s.vals + e0, 0, hi - e0);
  unsigned ok = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    if (e0 + k >= hi) continue;
    if (r[k] < 0 || r[k] >= s.n_rows || c[k] < 0 || c[k] >= s.n_cols) {
      *bad = min(*bad, e0 + k);
      continue;
    }
    mj[k] = (unsigned)c[k];
    mn[k] = (unsigned)r[k];
    ok |= 1u << k;
  }
  return ok;
}

template <class T>
__device__ __forceinline__ unsigned ld_group(const Csc<T>& s, const CscCtx& cx, const int* colc, long long e0,
                                             long long hi, unsigned* mj, unsigned* mn, T* vdst, long long*,
                                             bool vbulk = false) {
  long long r[4];
  ld4_idx(s.idx, e0, hi, r);
  if (!vbulk) cp_async_vals4(vdst, s.vals + e0, 0, hi - e0);
  long long c;
  if (cx.cached) {
    int l = 0, h = (int)(cx.ce - cx.cb);
    while (l < h) {
      const int mid = (l + h + 1) >> 1;
      if (colc[mid] <= e0) l = mid;
      else h = mid - 1;
    }
    c = cx.cb + l;
  } else {
    c = upper_bound_dev(s.ptr + cx.cb, cx.ce - cx.cb + 1, (int)e0) - 1 + cx.cb;
  }
  unsigned ok = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const long long e = e0 + k;
    if (e >= hi) continue;
    while ((cx.cached ? colc[c + 1 - cx.cb] : __ldg(&s.ptr[c + 1])) <= e) c++;
    if (s.by_row) {
      mj[k] = (unsigned)r[k];
      mn[k] = (unsigned)c;
    } else {
      mj[k] = (unsigned)c;
      mn[k] = (unsigned)r[k];
    }
    ok |= 1u << k;
  }
  return ok;
}


AS_DEVICE_INLINE int bits_for_dev(long long maxval) {
  int b = 0;
  while (b < 63 && (1ll << b) <= maxval) b++;
  return b;
}

// Block-level stable LSD radix sort (8-bit digits) of (u64 key, u32 payload)
// pairs in global memory, by the low idx_bits of the key, then key bits
// [32, 32 + key_bits): (key32, input index) order.  Result in (k, p).
__device__ inline void block_radix_sort_sr(unsigned long long* k, unsigned* p, unsigned long long* k_alt, unsigned* p_alt,
                                    long long L, int idx_bits, int key_bits, unsigned* hist, unsigned* wcnt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kThreads / 32;
  unsigned long long *sk = k, *dk = k_alt;
  unsigned *sp = p, *dp = p_alt;
  const int nip = (idx_bits + 7) / 8, npass = nip + (key_bits + 7) / 8;
  for (int ps = 0; ps < npass; ps++) {
    const int sh = ps < nip ? 8 * ps : 32 + 8 * (ps - nip);
    const int nb = ps < nip ? min(8, idx_bits - 8 * ps) : min(8, key_bits - 8 * (ps - nip));
    const unsigned mask = (1u << nb) - 1u;
    for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
    for (int i = tid; i < 256 * nwarps; i += kThreads) wcnt[i] = 0;
    __syncthreads();
    for (long long i = tid; i < L; i += kThreads) atomicAdd(&hist[(unsigned)(sk[i] >> sh) & mask], 1u);
    __syncthreads();
    if (warp == 0) {
      unsigned carry = 0;
      for (int b = 0; b < 256; b += 32) {
        const unsigned v = hist[b + lane];
        const unsigned inc = warp_inclusive_scan(v);
        hist[b + lane] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    for (long long base = 0; base < L; base += kThreads) {
      const long long i = base + tid;
      const bool in = i < L;
      const unsigned dg = in ? ((unsigned)(sk[i] >> sh) & mask) : 0xffffffffu;
      unsigned rank = 0;
      const unsigned act = __ballot_sync(0xffffffffu, in);
      if (in) {
        const unsigned peers = __match_any_sync(act, dg);
        rank = __popc(peers & lanemask_lt());
        if (rank == 0) wcnt[warp * 256 + dg] = __popc(peers);
      }
      __syncthreads();
      for (int b = tid; b < 256; b += kThreads) {
        unsigned run = hist[b];
        for (int w = 0; w < nwarps; w++) {
          const unsigned c = wcnt[w * 256 + b];
          wcnt[w * 256 + b] = run;
          run += c;
        }
        hist[b] = run;
      }
      __syncthreads();
      if (in) {
        const unsigned o = wcnt[warp * 256 + dg] + rank;
        dk[o] = sk[i];
        dp[o] = sp[i];
      }
      __syncthreads();
      for (int b = tid; b < 256 * nwarps; b += kThreads) wcnt[b] = 0;
      __syncthreads();
    }
    unsigned long long* t1 = sk;
    sk = dk;
    dk = t1;
    unsigned* t2 = sp;
    sp = dp;
    dp = t2;
  }
  if (sk != k) {
    for (long long i = tid; i < L; i += kThreads) {
      k[i] = sk[i];
      p[i] = sp[i];
    }
  }
  __syncthreads();
}

// diagnostic step clocks (AS_PHASE_TIMES): CTA 0 records clock64 at step k
#define SR_CLK(k, cond)                                                                                  \
  do {                                                                                                   \
    if (kDbg && sr_dbg_ && tid == 0 && (cond)) {                                                           \
      const unsigned long long now_ = clock64();                                                         \
      if (g == 0) sr_dbg_[8 + 3 * kMaxCb + (k)] = now_;                                                    \
      if ((k) <= 9) {                                                                                    \
        if ((k) > 0) {                                                                                   \
          atomicAdd(&sr_dbg_[8 + 3 * kMaxCb + 32 + 2 * (k)], now_ - clk_prev_);                            \
          atomicMax(&sr_dbg_[8 + 3 * kMaxCb + 33 + 2 * (k)], now_ - clk_prev_);                            \
        }                                                                                                \
        clk_prev_ = now_;                                                                                \
      }                                                                                                  \
    }                                                                                                    \
  } while (0)

// bucket t of the single-launch kernel = one run per chunk: run j at
// gK[j * ch + loffT[t][j] ...]; prefix by the group look-back
template <class T>
struct SegSR {
  static constexpr bool kContig = false;
  const unsigned* loffT;
  long long G, ch, ncb;
  const unsigned* gK;
  const unsigned* gX;
  const T* gV;
  unsigned long long* tstate;
  const unsigned* cbcol;  // shared memory
  __device__ __forceinline__ void seg(long long t, int tid, unsigned& len, unsigned& src) const {
    if (tid < G) {
      const unsigned s0 = __ldcg(&loffT[t * G + tid]), s1 = __ldcg(&loffT[(t + 1) * G + tid]);
      len = s1 - s0;
      src = (unsigned)(tid * ch) + s0;
    }
  }
  __device__ __forceinline__ unsigned key(unsigned s) const { return __ldcg(&gK[s]); }
  __device__ __forceinline__ unsigned idx(unsigned s) const { return __ldcg(&gX[s]); }
  __device__ __forceinline__ const T* val(unsigned s) const { return gV + s; }
  __device__ __forceinline__ unsigned col0(long long t) const { return cbcol[t]; }
  __device__ __forceinline__ unsigned long long prefix(long long t, unsigned long long kept) const {
    return group_lookback_warp(tstate, tstate + ncb, t, kept);
  }
};

// ------------------------------------------------------------------------
// The tile phase (P3 of the kernel below; also the last phase of the
// large-input pipeline, largen.cuh): CTA-strided buckets t = t0, t0 + tstep,
// ... < ncb.  A bucket of m <= kTile elements is loaded into registers /
// shared memory, counting-sorted over <= kNB bins of its key range (bins never
// straddle a column), every element ranks itself inside its bin by (key,
// input index) (large bins: warp / block bitonic), runs of equal keys reduce
// in the reference's order (np.add.reduceat pairwise, or last wins), exact
// zeros are pruned, the kept count goes to the look-back, and rows / values /
// col_ptr go straight to their final CSC positions.  A bucket above the tile
// (a heavy column) is sorted by a block radix sort in global memory and
// streamed (rare path).  `sg` names the bucket's elements: sg.seg (the runs
// making up the bucket), sg.key / sg.idx / sg.val (bucket-local key, input
// order, value address of a staging slot), sg.col0 (first column of a
// bucket), sg.prefix (the look-back).  Both structs live in shared memory.
template <class T>
struct TileOut {
  int mode, prune, mb, idx_bits, stop;
  long long n_minor;  // minor values in use: [0, n_minor)
  long long n_out_cols;
  int* col_ptr;
  int* row_idx;
  T* out_vals;
  long long* info;
  unsigned long long* ctr1;  // oversized-bucket scratch allocator (zeroed before the phase)
  unsigned long long* oK;
  unsigned long long* oK2;
  unsigned* oP;
  unsigned* oP2;
  int* oR;
  T* oV;
  unsigned long long* phase_ts;
};

template <class T, class Seg>
__device__ __forceinline__ void tile_phase(const Seg& sg, const TileOut<T>& o, TileSmem<T>& S, long long t0,
                                           long long tstep, long long ncb) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long g = blockIdx.x;
  const int mb = o.mb;
  unsigned long long clk_prev_ = 0;
  unsigned long long* const sr_dbg_ = o.phase_ts;
  (void)clk_prev_;
  (void)g;
  (void)sr_dbg_;
  for (int b = tid; b < kNB; b += kThreads) S.cnt[b] = 0u;
  const unsigned mmask = mb >= 32 ? 0xffffffffu : ((1u << mb) - 1u);
  for (long long t = t0; t < ncb; t += tstep) {
    const unsigned col_base = sg.col0(t);
    const int Wt = (int)(sg.col0(t + 1) - col_base);
    // bucket t = one run per chunk: run j at gK[j * ch + loffT[t][j] ...]
    unsigned seglen = 0, segsrc = 0;
    sg.seg(t, tid, seglen, segsrc);
    __syncthreads();  // the previous tile's shared memory is free; cnt zeroed
    unsigned m_u;
    const unsigned segoff = block_scan_u32(seglen, S.scan32, &m_u);
    const int m = (int)m_u;
    auto lookback = [&](long long kept) -> long long {
      if (kDbg && o.phase_ts && tid == 0) o.phase_ts[8 + 3 * t] = global_ns();
      if (tid < 32) {
        const unsigned long long pre = sg.prefix(t, (unsigned long long)kept);
        if (tid == 0) S.prefix = (long long)pre;
      }
      __syncthreads();
      if (kDbg && o.phase_ts && tid == 0) o.phase_ts[8 + 3 * t + 1] = global_ns();
      const long long base = S.prefix;
      if (t == ncb - 1 && tid == 0) {
        o.col_ptr[o.n_out_cols] = (int)(base + kept);
        o.info[0] = base + kept;
      }
      return base;
    };
    if (m == 0) {
      const long long base = lookback(0);
      for (int l = tid; l < Wt; l += kThreads) o.col_ptr[col_base + l] = (int)base;
      continue;
    }
    if (__builtin_expect(m > kTile, 0)) {
      // ---------- oversized bucket (rare): global-memory radix sort ----------
      if (tid == 0) S.prefix = (long long)atomicAdd(o.ctr1, (unsigned long long)m);  // scratch range
      __syncthreads();
      const long long s = S.prefix;
      unsigned long long* K1 = o.oK + s;
      unsigned long long* K2 = o.oK2 + s;
      unsigned* P1 = o.oP + s;
      unsigned* P2 = o.oP2 + s;
      for (unsigned e = 0; e < seglen; e++) {  // gather the runs (payload: staging slot of the value)
        K1[segoff + e] = ((unsigned long long)sg.key(segsrc + e) << 32) | sg.idx(segsrc + e);
        P1[segoff + e] = segsrc + e;
      }
      for (int l = tid; l < Wt; l += kThreads) S.u.r.ckept[l] = 0u;
      __syncthreads();
      block_radix_sort_sr(K1, P1, K2, P2, m, o.idx_bits, mb + bits_for_dev(Wt > 0 ? Wt - 1 : 0), S.u.r.hist,
                          S.u.r.wcnt);
      auto gv = [&](unsigned s) -> T { return *sg.val(s); };
      long long running = 0;
      for (int base0 = 0; base0 < m; base0 += kThreads) {
        const int p = base0 + tid;
        bool kept = false, longrun = false;
        T v = T(0);
        unsigned k = 0;
        long long rl = 0;
        if (p < m) {
          k = (unsigned)(K1[p] >> 32);
          const bool head = p == 0 || (unsigned)(K1[p - 1] >> 32) != k;
          if (head) {
            int q = p + 1;
            while (q < m && (unsigned)(K1[q] >> 32) == k) q++;
            rl = q - p;
            if (o.mode == kLast) {
              v = gv(P1[q - 1]);
            } else if (rl == 1) {
              v = gv(P1[p]);
            } else {
              longrun = true;
            }
            kept = !longrun && (!o.prune || v != T(0));
          }
        }
        for (unsigned lm = __ballot_sync(0xffffffffu, longrun); lm; lm &= lm - 1) {
          if (lane == __ffs(lm) - 1) {
            const unsigned* pp = P1 + p + 1;
            v = gv(P1[p]) + pw_stack<T>([&](int i) -> T { return gv(pp[i]); }, (int)(rl - 1), S.wst[warp]);
            kept = !o.prune || v != T(0);
          }
          __syncwarp();
        }
        long long tot;
        const long long off = block_exclusive_scan<long long>(kept ? 1ll : 0ll, S.scan, &tot);
        if (kept) {
          o.oR[s + running + off] = (int)(k & mmask);
          o.oV[s + running + off] = v;
          atomicAdd(&S.u.r.ckept[k >> mb], 1u);
        }
        running += tot;
      }
      __syncthreads();
      const long long base = lookback(running);
      for (long long i = tid; i < running; i += kThreads) {
        o.row_idx[base + i] = __ldcg(&o.oR[s + i]);
        o.out_vals[base + i] = __ldcg(&o.oV[s + i]);
      }
      long long run = base;
      for (int l0 = 0; l0 < Wt; l0 += kThreads) {
        const int l = l0 + tid;
        long long tot;
        const long long ex = block_exclusive_scan<long long>(l < Wt ? (long long)S.u.r.ckept[l] : 0ll, S.scan, &tot);
        if (l < Wt) o.col_ptr[col_base + l] = (int)(run + ex);
        run += tot;
      }
      continue;
    }

    // ---------- tile ----------
    // element i = tid + u * kThreads (striped: a warp's shared-memory accesses
    // are consecutive wherever the layout allows); bins: aligned ranges of the
    // key between 0 and Wt << mb, at most kNB, never wider than one column
    SR_CLK(0, t == g);
    // bins: bpc per column over the minor range actually used ([0, n_minor),
    // not the 2^mb the key reserves), each 2^sh minor values wide
    const unsigned nmin = o.n_minor > 0 ? (unsigned)o.n_minor : 1u;
    // smallest sh with Wt * ceil(nmin / 2^sh) <= kNB: 2^sh >= ceil(nmin / (kNB / Wt))
    const unsigned bpc_max = (unsigned)kNB / (unsigned)max(Wt, 1);
    const unsigned xq = (nmin + bpc_max - 1) / bpc_max;
    const int sh = xq <= 1u ? 0 : 32 - __clz(xq - 1u);
    const unsigned bpc = ((nmin - 1) >> sh) + 1;
    const int nbins = (int)((unsigned)Wt * bpc);
    // staging slot of every element of the tile (the map aliases TK, written
    // later); a contiguous bucket (large-input pipeline) needs no map
    unsigned cbase = 0;
    if constexpr (Seg::kContig) {
      cbase = sg.base(t);
    } else {
      for (unsigned e = 0; e < seglen; e++) S.u.a.TK[segoff + e] = segsrc + e;
      __syncthreads();
    }
    unsigned k4[kTP], x4[kTP], br[kTP];
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      const int i = tid + u * kThreads;
      if (i < m) {
        const unsigned src = Seg::kContig ? cbase + (unsigned)i : S.u.a.TK[i];
        k4[u] = sg.key(src);
        x4[u] = sg.idx(src);
        const unsigned d = (unsigned)__cvta_generic_to_shared(&S.u.a.V[i]);
        if constexpr (sizeof(T) == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(sg.val(src)) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(sg.val(src)) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    SR_CLK(1, t == g);
    if (kDbg && o.phase_ts && tid == 0) o.phase_ts[8 + 3 * t + 2] = global_ns();
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      if (tid + u * kThreads < m) {
        const unsigned b = (k4[u] >> mb) * bpc + ((k4[u] & mmask) >> sh);
        br[u] = (b << 16) | atomicAdd(&S.cnt[b], 1u);
      }
    }
    if (tid == 0) S.n_big = 0;
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's values landed
    __syncthreads();
    SR_CLK(2, t == g);
    if (kDbg && o.stop == 3) return;
    {  // bin starts (kNB / kThreads consecutive bins per thread); counts re-zeroed
      constexpr int kB = kNB / kThreads;
      const int b0 = tid * kB;
      unsigned c[kB], sum = 0;
#pragma unroll
      for (int q = 0; q < kB; q++) {
        c[q] = b0 + q < nbins ? S.cnt[b0 + q] : 0u;
        sum += c[q];
      }
      unsigned tot;
      unsigned run = block_scan_u32(sum, S.scan32, &tot);
#pragma unroll
      for (int q = 0; q < kB; q++) {
        if (b0 + q < nbins) {
          S.bs[b0 + q] = run;
          S.cnt[b0 + q] = 0u;
          if (c[q] > kRankMax) S.big[atomicAdd(&S.n_big, 1)] = (unsigned short)(b0 + q);
        }
        run += c[q];
      }
      if (tid == 0) S.bs[nbins] = (unsigned)m;
    }
    __syncthreads();
    SR_CLK(3, t == g);
    if (kDbg && o.stop == 7) return;
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      if (tid + u * kThreads < m) {
        const unsigned pos = S.bs[br[u] >> 16] + (br[u] & 0xffffu);
        S.u.a.TK[pos] = k4[u];
        S.u.a.TX[pos] = x4[u];
      }
    }
    for (int l = tid; l <= Wt; l += kThreads) {
      const unsigned bl = (unsigned)l * bpc;
      S.cstart[l] = (unsigned short)S.bs[bl < (unsigned)nbins ? bl : (unsigned)nbins];
    }
    __syncthreads();
    SR_CLK(4, t == g);
    if (kDbg && o.stop == 8) return;
    // each element ranks itself inside its bin by (key, input index): final position
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      const int i = tid + u * kThreads;
      if (i < m) {
        const unsigned b = br[u] >> 16;
        const unsigned b0 = S.bs[b], b1 = S.bs[b + 1];
        if (b1 - b0 <= kRankMax) {
          // branch-free count of the bin's (key, index) pairs below this one
          unsigned r = 0;
          const unsigned k = k4[u], x = x4[u];
#pragma unroll kRankUnroll
          for (unsigned j = b0; j < b1; j++) {
            const unsigned kj = S.u.a.TK[j], xj = S.u.a.TX[j];
            r += (unsigned)(kj < k) | ((unsigned)(kj == k) & (unsigned)(xj < x));
          }
          S.SK[b0 + r] = k;
          S.SI[b0 + r] = (unsigned short)i;
        }
      }
    }
    const int n_big = S.n_big;
    if (kDbg && o.phase_ts && tid == 0 && n_big) atomicAdd(&o.phase_ts[5], (unsigned long long)n_big);
    if (__builtin_expect(n_big != 0, 0)) {  // bins above kRankMax (rare): warp bitonic (<= 512), block bitonic beyond
      for (int q = warp; q < n_big; q += kThreads / 32) {
        const int b = S.big[q];
        const int b0 = S.bs[b], L = S.bs[b + 1] - b0;
        if (L > 512) continue;
        for (int j = lane; j < L; j += 32) S.u.a.BK[b0 + j] = ((unsigned long long)S.u.a.TK[b0 + j] << 32) | S.u.a.TX[b0 + j];
        __syncwarp();
        bitonic_sort<false>(S.u.a.BK + b0, L, lane, 32);
        for (int j = lane; j < L; j += 32) S.SK[b0 + j] = (unsigned)(S.u.a.BK[b0 + j] >> 32);
      }
      __syncthreads();
      for (int q = 0; q < n_big; q++) {
        const int b = S.big[q];
        const int b0 = S.bs[b], L = S.bs[b + 1] - b0;
        if (L <= 512) continue;
        for (int j = tid; j < L; j += kThreads) S.u.a.BK[b0 + j] = ((unsigned long long)S.u.a.TK[b0 + j] << 32) | S.u.a.TX[b0 + j];
        __syncthreads();
        bitonic_sort<true>(S.u.a.BK + b0, L, tid, kThreads);
        for (int j = tid; j < L; j += kThreads) S.SK[b0 + j] = (unsigned)(S.u.a.BK[b0 + j] >> 32);
        __syncthreads();
      }
    }
    __syncthreads();
    if (__builtin_expect(n_big != 0, 0)) {  // the sorted (key, index) pairs of big bins name their elements by input index
#pragma unroll
      for (int u = 0; u < kTP; u++) {
        const int i = tid + u * kThreads;
        if (i < m) {
          const unsigned b = br[u] >> 16;
          const unsigned b0 = S.bs[b], b1 = S.bs[b + 1];
          if (b1 - b0 > kRankMax) {  // find this element's (key, index) in the sorted bin
            const unsigned long long kx = ((unsigned long long)k4[u] << 32) | x4[u];
            unsigned lo2 = b0, hi2 = b1;
            while (lo2 < hi2) {
              const unsigned mid = (lo2 + hi2) >> 1;
              if (S.u.a.BK[mid] < kx) lo2 = mid + 1;
              else hi2 = mid;
            }
            S.SI[lo2] = (unsigned short)i;
          }
        }
      }
      __syncthreads();
    }
    SR_CLK(5, t == g);
    if (kDbg && o.stop == 4) return;
    // runs (striped positions p = tid + u * kThreads): a run belongs to its
    // head, whose value goes to RV[head]; runs of several values are summed
    // in one non-unrolled loop (a single copy of the pairwise code), the
    // ones above one pairwise leaf with the warp's stack one lane at a time
    unsigned hmask = 0, multi = 0;
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      const int p = tid + u * kThreads;
      if (p < m) {
        const unsigned k = S.SK[p];
        if (p == 0 || S.SK[p - 1] != k) {
          hmask |= 1u << u;
          if (p + 1 < m && S.SK[p + 1] == k) {
            multi |= 1u << u;
          } else {
            S.u.a.RV[p] = S.u.a.V[S.SI[p]];
          }
        }
      }
    }
    if (o.mode == kLast) {
#pragma unroll 1
      for (int u = 0; u < kTP; u++) {
        if (!(multi >> u & 1u)) continue;
        const int p = tid + u * kThreads;
        const unsigned k = S.SK[p];
        int q = p + 2;
        while (q < m && S.SK[q] == k) q++;
        S.u.a.RV[p] = S.u.a.V[S.SI[q - 1]];
      }
      multi = 0;
    }
    // Sum runs of several values (pairwise order, np.add.reduceat): the
    // warp's lanes one at a time, sharing the warp's stack (rare: duplicates)
    for (unsigned lm = __ballot_sync(0xffffffffu, multi != 0); __builtin_expect(lm != 0, 0); lm &= lm - 1) {
      if (lane == __ffs(lm) - 1) {
#pragma unroll 1
        for (int u = 0; u < kTP; u++) {
          if (!(multi >> u & 1u)) continue;
          const int p = tid + u * kThreads;
          const unsigned k = S.SK[p];
          int q = p + 2;
          while (q < m && S.SK[q] == k) q++;
          const unsigned short* si = S.SI + p + 1;
          S.u.a.RV[p] = S.u.a.V[S.SI[p]] + pw_stack<T>([&](int j) -> T { return S.u.a.V[si[j]]; }, q - p - 1,
                                                        S.wst[warp]);
        }
      }
      __syncwarp();
    }
    bool kp[kTP];
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      const int p = tid + u * kThreads;
      kp[u] = (hmask >> u & 1u) && (!o.prune || S.u.a.RV[p] != T(0));
      const unsigned w = __ballot_sync(0xffffffffu, kp[u]);
      if (lane == 0) S.kw[u * (kThreads / 32) + warp] = w;
    }
    SR_CLK(6, t == g);
    __syncthreads();
    long long total = 0;
    if (warp == 0) {  // prefix over the kTile / 32 words
      constexpr int kW = kTile / 32;
      unsigned c[kW / 32], sum = 0;
#pragma unroll
      for (int q = 0; q < kW / 32; q++) {
        c[q] = __popc(S.kw[lane * (kW / 32) + q]);
        sum += c[q];
      }
      const unsigned inc = warp_inclusive_scan(sum);
      unsigned run = inc - sum;
#pragma unroll
      for (int q = 0; q < kW / 32; q++) {
        S.kwp[lane * (kW / 32) + q] = run;
        run += c[q];
      }
      if (lane == 31) S.kwp[kW] = inc;
    }
    __syncthreads();
    total = S.kwp[kTile / 32];
    SR_CLK(7, t == g);
    if (kDbg && o.stop == 5) return;
    const long long base = lookback(total);
    SR_CLK(8, t == g);
    if (kDbg && o.stop == 6) return;
#pragma unroll
    for (int u = 0; u < kTP; u++) {
      if (kp[u]) {
        const int p = tid + u * kThreads;
        const int w = p >> 5;
        const long long e = base + S.kwp[w] + __popc(S.kw[w] & lanemask_lt());
        __stcs(&o.row_idx[e], (int)(S.SK[p] & mmask));
        __stcs(&o.out_vals[e], S.u.a.RV[p]);
      }
    }
    for (int l = tid; l < Wt; l += kThreads) {
      const int p = S.cstart[l];
      const int w = p >> 5;
      const unsigned e = p >= m ? (unsigned)total : S.kwp[w] + __popc(S.kw[w] & ((1u << (p & 31)) - 1u));
      o.col_ptr[col_base + l] = (int)(base + e);
    }
    SR_CLK(9, t == g);
  }
}


// ------------------------------------------------------------------------
template <class T, class S1, class S2>
__global__ void __launch_bounds__(kThreads, kMinBlocks) sortreduce_kernel(Args<T, S1, S2> a_) {
  extern __shared__ __align__(16) unsigned char smem[];
  // the arguments live in shared memory: kernel-parameter loads go through
  // the constant cache, which shares the SM's L1.5 with instructions and
  // missed to L2 on every phase of this long kernel (ncu: the top stall)
  __shared__ Args<T, S1, S2> a;
  if (threadIdx.x == 0) a = a_;
  __syncthreads();
  __shared__ unsigned xs32[kThreads / 32 + 1];
  __shared__ long long s_bad;
  constexpr bool kTwoSrc = !std::is_same<S2, None>::value;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long G = gridDim.x, g = blockIdx.x;
  const long long ncb = a.ncb;
  const Layout LY = layout<T>(ncb, kChunkMax);  // only the offsets up to colc are used with the real chunk below
  unsigned* cbcol = reinterpret_cast<unsigned*>(smem);  // [ncb + 1] first column of each bucket
  unsigned* hist = reinterpret_cast<unsigned*>(smem + LY.hist);
  unsigned* loff = reinterpret_cast<unsigned*>(smem + LY.loff);
  int* colc = reinterpret_cast<int*>(smem + LY.colc);
  const unsigned long long cb_mul = a.cb_mul;
  const int mb = a.minor_bits;
  unsigned long long clk_prev_ = 0;
  unsigned long long* const sr_dbg_ = a.phase_ts;
  if (kDbg && a.phase_ts && tid == 0) {
    const unsigned long long t0 = global_ns();
    atomicMin(&a.phase_ts[0], t0);
    atomicMax(&a.phase_ts[1], t0);
  }

  // ---------------- P1 ----------------
  const long long ch = (((a.n + G - 1) / G) + 3) & ~3ll;
  const long long lo = min(a.n, g * ch), hi = min(a.n, lo + ch);
  const Layout LC = layout<T>(ncb, ch);
  T* st_val = reinterpret_cast<T*>(smem + LC.st_val);
  // one source: the chunk's values travel to shared memory by bulk copies
  // (TMA engine, kBulkParts pieces, completed on one mbarrier) issued before
  // anything else; two sources (the flush) keep per-thread cp.async
  __shared__ __align__(8) unsigned long long vbar;
  const bool vbulk = !kTwoSrc && kBulkVals && hi > lo && ((reinterpret_cast<unsigned long long>(a.s1.vals) & 15ull) == 0);
  if (vbulk && warp == 0) {
    const long long body = ((hi - lo) * (long long)sizeof(T)) & ~15ll;  // bytes
    const long long part = (((body + kBulkParts - 1) / kBulkParts) + 15) & ~15ll;
    if (lane == 0) {
      mbar_init(&vbar, kBulkParts);
      for (long long e = lo + body / (long long)sizeof(T); e < hi; e++) st_val[e - lo] = __ldg(&a.s1.vals[e]);
    }
    __syncwarp();
    if (lane < kBulkParts) {
      const long long b0 = min(body, lane * part), b1 = min(body, b0 + part);
      if (b1 > b0)
        bulk_g2s(reinterpret_cast<unsigned char*>(st_val) + b0,
                 reinterpret_cast<const unsigned char*>(a.s1.vals + lo) + b0, (unsigned)(b1 - b0), &vbar);
      else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&vbar))
                     : "memory");
    }
  }
  unsigned* st_key = reinterpret_cast<unsigned*>(smem + LC.st_key);
  unsigned short* st_idx = reinterpret_cast<unsigned short*>(smem + LC.st_idx);  // local input index
  for (long long t = tid; t <= ncb; t += kThreads) {
    // first column of bucket t = ceil(t 2^32 / cb_mul): a double quotient (off by
    // at most one) and exact integer corrections instead of a 64-bit division
    unsigned long long c0 = 0ull;
    if (cb_mul) {
      const unsigned long long num = (unsigned long long)t << 32;
      c0 = (unsigned long long)((double)num / (double)cb_mul);
      while (c0 * cb_mul < num) c0++;
      while (c0 > 0 && (c0 - 1) * cb_mul >= num) c0--;
    }
    cbcol[t] = (unsigned)(t == ncb ? a.n_out_cols : min((long long)c0, a.n_out_cols));
  }
  for (long long b = tid; b < ncb; b += kThreads) hist[b] = 0u;
  {
    const long long nts = ncb + ncb / 32 + 1;  // look-back words: zeroed here, first read after two barriers
    for (long long q = g * kThreads + tid; q < nts; q += G * kThreads) a.tstate[q] = 0ull;
  }
  if (g == 0 && tid < 2) a.ctr[tid] = 0ull;  // first used after the grid barrier
  SR_CLK(10, true);
  if (tid == 0) s_bad = a.n;
  // source contexts (CSC column caches) for the chunk's part of each source
  CscCtx cx1{0, 0, false}, cx2{0, 0, false};
  if constexpr (std::is_same<S1, Csc<T>>::value) csc_ctx(a.s1, min(lo, a.n1), min(hi, a.n1), colc, &cx1);
  __syncthreads();
  // all loads first (indices to registers, values straight to shared memory
  // in input order), then the bucket / key / rank of each element
  unsigned mj[kPer], mn[kPer], ok = 0;
  long long bad = a.n;
#pragma unroll
  for (int q = 0; q < kPer / 4; q++) {
    const long long e0 = lo + 4ll * (tid + (long long)q * kThreads);
    T* vd = st_val + (e0 - lo);
    unsigned o = 0;
    if (e0 < hi) {
      if (!kTwoSrc || e0 + 4 <= a.n1 || hi <= a.n1) {
        o = ld_group(a.s1, cx1, colc, e0, min(hi, a.n1), mj + 4 * q, mn + 4 * q, vd, &bad, vbulk);
      } else if constexpr (kTwoSrc) {
        if (e0 >= a.n1) {
          long long b2 = a.n;
          o = ld_group(a.s2, cx2, colc, e0 - a.n1, hi - a.n1, mj + 4 * q, mn + 4 * q, vd, &b2);
          bad = min(bad, b2);  // (an index of the second source)
        } else {  // a group straddling the two sources: element by element
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const long long e = e0 + k;
            if (e >= hi) continue;
            unsigned j1[4], n1_[4];
            unsigned o1;
            if (e < a.n1) {
              o1 = ld_group(a.s1, cx1, colc, e, e + 1, j1, n1_, vd + k, &bad);
            } else {
              long long b2 = a.n;
              o1 = ld_group(a.s2, cx2, colc, e - a.n1, e - a.n1 + 1, j1, n1_, vd + k, &b2);
              bad = min(bad, b2);
            }
            if (o1 & 1u) {
              mj[4 * q + k] = j1[0];
              mn[4 * q + k] = n1_[0];
              o |= 1u << k;
            }
          }
        }
      }
    }
    ok |= o << (4 * q);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  unsigned key[kPer], bk[kPer];
  SR_CLK(11, true);
  if (kDbg && a.stop == 11) return;
#pragma unroll
  for (int i = 0; i < kPer; i++) {
    bk[i] = 0xffffffffu;
    if (ok >> i & 1u) {
      const unsigned b = (unsigned)(((unsigned long long)mj[i] * cb_mul) >> 32);
      key[i] = ((mj[i] - cbcol[b]) << mb) | mn[i];
      const unsigned r = atomicAdd(&hist[b], 1u);
      bk[i] = (b << kRankBits) | r;
    }
  }
  SR_CLK(12, true);
  if (kDbg && a.stop == 12) {
    __syncthreads();
    return;
  }
  if (bad < a.n) atomicMin((unsigned long long*)&s_bad, (unsigned long long)bad);
  __syncthreads();
  {  // local bucket offsets of the chunk; published transposed for the tiles
    unsigned run = 0;
    for (long long c0 = 0; c0 < ncb; c0 += kThreads) {
      const long long b = c0 + tid;
      const unsigned h = b < ncb ? hist[b] : 0u;
      unsigned tot;
      const unsigned ex = block_scan_u32(h, xs32, &tot);
      if (b < ncb) {
        loff[b] = run + ex;
        a.loffT[b * G + g] = run + ex;
      }
      run += tot;
    }
    if (tid == 0) {
      loff[ncb] = run;
      a.loffT[ncb * G + g] = run;
      a.cta_bad[g] = s_bad;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kPer; i++) {
    if (bk[i] != 0xffffffffu) {
      const unsigned b = bk[i] >> kRankBits;
      const unsigned pos = loff[b] + (bk[i] & ((1u << kRankBits) - 1u));
      st_key[pos] = key[i];
      st_idx[pos] = (unsigned short)(4 * (tid + (i >> 2) * kThreads) + (i & 3));
    }
  }
  SR_CLK(13, true);
  if (kDbg && a.stop == 13) return;
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (vbulk) mbar_wait(&vbar, 0);
  __syncthreads();
  {  // the chunk in bucket order, contiguous (coalesced): its bucket runs are
     // what the tiles gather
    const unsigned total = loff[ncb];
    const long long cb0 = g * a.ch;
    for (unsigned q = tid; q < total; q += kThreads) {
      const unsigned li = st_idx[q];
      __stcg(&a.gK[cb0 + q], st_key[q]);
      __stcg(&a.gX[cb0 + q], (unsigned)lo + li);
      __stcg(&a.gV[cb0 + q], st_val[li]);
    }
  }
  SR_CLK(14, true);
  cooperative_groups::this_grid().sync();
  if (kDbg && a.stop == 1) return;
  if (kDbg && a.phase_ts && g == 0 && tid == 0) a.phase_ts[2] = a.phase_ts[3] = global_ns();

  // ---------------- P3 ----------------
  TileSmem<T>& S = *reinterpret_cast<TileSmem<T>*>(smem + LY.tile_off);
  __shared__ TileOut<T> to;
  __shared__ SegSR<T> sgs;
  if (tid == 0) {
    to.mode = a.mode;
    to.prune = a.prune;
    to.mb = a.minor_bits;
    to.n_minor = a.n_minor;
    to.idx_bits = a.idx_bits;
    to.stop = a.stop;
    to.n_out_cols = a.n_out_cols;
    to.col_ptr = a.col_ptr;
    to.row_idx = a.row_idx;
    to.out_vals = a.out_vals;
    to.info = a.info;
    to.ctr1 = a.ctr + 1;
    to.oK = a.oK;
    to.oK2 = a.oK2;
    to.oP = a.oP;
    to.oP2 = a.oP2;
    to.oR = a.oR;
    to.oV = a.oV;
    to.phase_ts = a.phase_ts;
    sgs.loffT = a.loffT;
    sgs.G = G;
    sgs.ch = a.ch;
    sgs.ncb = ncb;
    sgs.gK = a.gK;
    sgs.gX = a.gX;
    sgs.gV = a.gV;
    sgs.tstate = a.tstate;
    sgs.cbcol = cbcol;
  }
  __syncthreads();
  tile_phase<T>(sgs, to, S, g, G, ncb);
  // the last CTA to finish reduces the chunks' first invalid triplets
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_bad = atomicAdd(&a.ctr[0], 1ull) == (unsigned long long)G - 1 ? 1 : 0;
  }
  __syncthreads();
  if (s_bad) {
    long long bad = a.n;
    for (long long q = tid; q < G; q += kThreads) bad = min(bad, __ldcg(&a.cta_bad[q]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (lane == 0) atomicMin((unsigned long long*)&a.cta_bad[0], (unsigned long long)bad);
    __syncthreads();
    if (tid == 0) {
      const long long b0 = __ldcg(&a.cta_bad[0]);
      a.info[1] = b0 < a.n ? b0 : 0x7f7f7f7f7f7f7f7fll;
    }
  }
  if (tid == 0) {
    if (kDbg && a.phase_ts) atomicMax(&a.phase_ts[4], global_ns());
  }
}

}  // namespace sr
}  // namespace as
