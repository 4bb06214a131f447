// common.cuh -- shared device utilities for the sm_100a sparse hot path.
//
// Block/warp scans, the single-pass chained-scan (decoupled look-back) tile
// state used by every kernel whose output size is only known after it runs,
// the numpy pairwise-sum emulation that makes duplicate sums bit-exact with
// the reference's np.add.reduceat (csc.py:179), and small index helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef AS_DEVICE_INLINE
#define AS_DEVICE_INLINE __device__ __forceinline__
#endif

namespace as {

constexpr int kWarp = 32;

// ------------------------------------------------------------------------
// reduce modes for runs of equal (segment, row) keys
enum ReduceMode : int {
  kSumPairwise = 0,  // np.add.reduceat order: v0 + pairwise(v1..)  (csc.py:179)
  kLast = 1,         // LastWins: last in input order (csc.py:181-182, rbt.py:115-117)
  kSumSeq = 2,       // sequential left fold (Gustavson accumulator, _kernels.py:83-93)
};

// ------------------------------------------------------------------------
// warp / block scans (inclusive and exclusive) over 32- or 64-bit values
template <class T>
AS_DEVICE_INLINE T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <class T>
AS_DEVICE_INLINE T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan; every thread must call.  `smem` needs
// (blockDim.x/32 + 1) elements.  Returns the exclusive prefix of `v`, and the
// block total in *total.
template <class T>
__device__ T block_exclusive_scan(T v, T* smem, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nwarps ? smem[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < nwarps) smem[lane] = wi - w;
    if (lane == nwarps - 1) smem[nwarps] = wi;
  }
  __syncthreads();
  T res = smem[warp] + inc - v;
  *total = smem[nwarps];
  __syncthreads();
  return res;
}

template <class T>
__device__ T block_reduce_sum(T v, T* smem) {
  T total;
  (void)block_exclusive_scan(v, smem, &total);
  return total;
}

// block-wide exclusive max-scan of unsigned values (every thread calls)
__device__ inline unsigned block_exclusive_max(unsigned v, unsigned* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = max(inc, n);
  }
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned w = lane < nwarps ? smem[lane] : 0u;
    unsigned wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi = max(wi, n);
    }
    const unsigned ex = __shfl_up_sync(0xffffffffu, wi, 1);
    if (lane < nwarps) smem[lane] = lane ? ex : 0u;
  }
  __syncthreads();
  unsigned ex_in_warp = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex_in_warp = 0u;
  const unsigned res = max(smem[warp], ex_in_warp);
  __syncthreads();
  return res;
}

// ------------------------------------------------------------------------
// Chained scan (single-pass decoupled look-back).  One 64-bit word per tile:
// (value << 2) | flag, flag 1 = tile aggregate, 2 = inclusive prefix.
// The tile state array and the ticket counter must be zeroed before launch.
constexpr unsigned long long kFlagAgg = 1ull, kFlagInc = 2ull;

// No memory fence: every user publishes only the count carried by the state
// word itself (outputs are written after the prefix is known), and an atomic
// is performed at L2 where the polling loads see it.  (Fenced publishes cost
// the sparse add 11 us of 83.)
AS_DEVICE_INLINE void tile_publish(unsigned long long* st, unsigned long long value,
                                   unsigned long long flag) {
  atomicExch(st, (value << 2) | flag);
}

AS_DEVICE_INLINE unsigned long long tile_peek(const unsigned long long* st) {
  return *((volatile const unsigned long long*)st);
}

// Executed by one full warp of the tile.  Returns the exclusive prefix of
// tile `t` after publishing its aggregate and, then, its inclusive prefix.
__device__ inline unsigned long long tile_lookback_warp(unsigned long long* states, long long t,
                                                        unsigned long long aggregate) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) tile_publish(&states[0], aggregate, kFlagInc);
    return 0;
  }
  if (lane == 0) tile_publish(&states[t], aggregate, kFlagAgg);
  unsigned long long prefix = 0;
  long long base = t - 1;
  while (true) {
    long long i = base - lane;
    unsigned long long s = 0;
    if (i >= 0) {
      do {
        s = tile_peek(&states[i]);
      } while ((s & 3ull) == 0ull);
    } else {
      s = kFlagInc;  // virtual inclusive 0 before tile 0
    }
    unsigned inc_mask = __ballot_sync(0xffffffffu, (s & 3ull) == kFlagInc);
    // lanes up to and including the first inclusive one contribute
    int first = inc_mask ? (__ffs(inc_mask) - 1) : 32;
    unsigned long long v = (lane <= first) ? (s >> 2) : 0ull;
    prefix += warp_reduce_sum(v);
    if (inc_mask) break;
    base -= 32;
  }
  if (lane == 0) tile_publish(&states[t], prefix + aggregate, kFlagInc);
  return prefix;
}

// Executed by one full warp of the tile: the exclusive prefix of bucket t's
// kept count over buckets [0, t).  Each bucket publishes its count to st[t]
// and adds it to its group word grp[t / 32] (publishers << 56 | sum); the
// prefix is the completed words of the preceding groups plus the in-group
// predecessors -- two parallel polls.  (A chained look-back walked back up to
// n_cb / 32 serial rounds: the tiles of a wave reach this point together, so
// few inclusive prefixes were ever published in time.)  Tickets are handed
// out in bucket order by co-resident CTAs, so every predecessor is running.
__device__ __forceinline__ unsigned long long group_lookback_warp(unsigned long long* st, unsigned long long* grp,
                                                                  long long t, unsigned long long kept) {
  const int lane = threadIdx.x & 31;
  constexpr unsigned long long kOne = 1ull << 56, kSum = kOne - 1;
  if (lane == 0) {
    atomicExch(&st[t], (kept << 1) | 1ull);
    atomicAdd(&grp[t >> 5], kOne | kept);
  }
  unsigned long long pre = 0;
  const long long q = (t & ~31ll) + lane;  // in-group predecessor of this lane
  if (q < t) {
    unsigned long long s;
    do {
      s = tile_peek(&st[q]);
    } while (!(s & 1ull));
    pre = s >> 1;
  }
  const long long ng = t >> 5;  // complete groups before t's
  for (long long i0 = 0; i0 < ng; i0 += 32 * 4) {
    unsigned long long v[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const long long i = i0 + lane + 32 * u;
      v[u] = i < ng ? tile_peek(&grp[i]) : 32 * kOne;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const long long i = i0 + lane + 32 * u;
      while ((v[u] >> 56) < 32) v[u] = tile_peek(&grp[i]);
      pre += v[u] & kSum;
    }
  }
  return warp_reduce_sum(pre);
}

// ------------------------------------------------------------------------
// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum_@TYPE@), applied by np.add.reduceat to a segment as
// v[0] + pairwise(v[1:]).  `get(k)` returns the k-th value of the run.
// Leaves: n < 8 sequential from -0.0; n <= 128 eight accumulators, a fixed
// tree, then the tail.
template <class T, class Get>
__device__ T pw_leaf(Get get, long long off, long long n) {
  if (n < 8) {
    T r = T(-0.0);
    for (long long i = 0; i < n; i++) r = r + get(off + i);
    return r;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = get(off + j);
  long long i;
  for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = r[j] + get(off + i + j);
  }
  T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; i++) res = res + get(off + i);
  return res;
}

// n > 128 splits at n2 = n/2 rounded down to a multiple of 8 and returns
// sum(left) + sum(right).  Evaluated post-order with an explicit stack
// (depth <= 26 for n < 2^32) -- no device recursion.
template <class T, class Get>
__device__ T pw_sum(Get get, long long off, long long n) {
  if (n <= 128) return pw_leaf<T>(get, off, n);
  long long s_off[32], s_n[32];
  T s_left[32];
  unsigned char s_stage[32];
  int sp = 1;
  s_off[0] = off;
  s_n[0] = n;
  s_stage[0] = 0;
  T ret = T(0);
  bool have = false;
  while (true) {
    if (!have) {
      const int top = sp - 1;
      if (s_n[top] <= 128) {
        ret = pw_leaf<T>(get, s_off[top], s_n[top]);
        have = true;
        sp--;
      } else {
        long long n2 = s_n[top] / 2;
        n2 -= n2 % 8;
        s_stage[top] = 0;
        s_off[sp] = s_off[top];
        s_n[sp] = n2;
        s_stage[sp] = 0;
        sp++;
      }
    } else {
      if (sp == 0) return ret;
      const int top = sp - 1;
      long long n2 = s_n[top] / 2;
      n2 -= n2 % 8;
      if (s_stage[top] == 0) {
        s_left[top] = ret;
        s_stage[top] = 1;
        have = false;
        s_off[sp] = s_off[top] + n2;
        s_n[sp] = s_n[top] - n2;
        s_stage[sp] = 0;
        sp++;
      } else {
        ret = s_left[top] + ret;
        sp--;
      }
    }
  }
}

// kSeqOnly: an instantiation that only ever folds sequentially (SpGEMM's
// pre-bucketed mode) -- the pairwise summation and its explicit stack are not
// compiled in (they were most of that kernel's 1 KB stack frame)
template <class T, class Get, bool kSeqOnly = false>
__device__ T reduce_run(Get get, long long n, int mode) {
  if (mode == kLast) return get(n - 1);
  T v0 = get(0);
  if (n == 1) return v0;
  if (kSeqOnly || mode == kSumSeq) {
    T acc = v0;
    for (long long i = 1; i < n; i++) acc = acc + get(i);
    return acc;
  }
  return v0 + pw_sum<T>(get, 1, n - 1);
}

// ------------------------------------------------------------------------
template <class T>
AS_DEVICE_INLINE long long lower_bound_dev(const T* a, long long n, T x) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <class T>
AS_DEVICE_INLINE long long upper_bound_dev(const T* a, long long n, T x) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

AS_DEVICE_INLINE unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ------------------------------------------------------------------------
// grid barrier for cooperatively launched (co-resident) grids
struct GridBar {
  unsigned* arrive;
  unsigned* gen;
};

// Sense-free grid barrier for a cooperatively launched (co-resident) grid.
// ------------------------------------------------------------------------
// Bulk asynchronous copies (the TMA engine's 1-D mode) into shared memory,
// completed on a shared-memory mbarrier: one elected thread moves a whole
// contiguous range, no per-thread copy instructions.  Both addresses 16-byte
// aligned and the size a multiple of 16 (callers guarantee it).
AS_DEVICE_INLINE void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// the calling thread arrives and announces `bytes` of transfers, then issues
// the copy of `bytes` from gsrc to sdst
AS_DEVICE_INLINE void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(gsrc), "r"(bytes), "r"(b)
               : "memory");
}

// one arrival announcing `bytes` of transfers (then issue the copies with
// bulk_g2s_noarrive): lets one mbarrier of count 1 track several copies
AS_DEVICE_INLINE void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
AS_DEVICE_INLINE void bulk_g2s_noarrive(void* sdst, const void* gsrc, unsigned bytes, unsigned long long* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(gsrc), "r"(bytes), "r"(b)
               : "memory");
}

AS_DEVICE_INLINE void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  }
}

AS_DEVICE_INLINE unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

AS_DEVICE_INLINE void grid_sync(const GridBar& gb, unsigned& gen_local) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned a = atomicAdd(gb.arrive, 1u);
    if (a == gridDim.x - 1) {
      *((volatile unsigned*)gb.arrive) = 0u;
      __threadfence();
      atomicAdd(gb.gen, 1u);
    } else {
      while (*((volatile unsigned*)gb.gen) == gen_local) __nanosleep(64);
    }
    __threadfence();
  }
  gen_local++;
  __syncthreads();
}


}  // namespace as
