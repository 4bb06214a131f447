// persist.cuh -- one persistent, cooperatively launched kernel per
// bucket-sort-reduce operation (COO->CSC construction, insertion-log flush,
// CSC transpose).
//
// At the sizes of the BASELINE configs (1e5-1e7 elements) a pipeline of
// separate kernels is latency bound, and per-element global atomics on ~1e4
// buckets serialise in L2 (measured on B200: 1M RED.ADD over 10k bins take
// ~24 us, tools/micro/atomic_micro.cu).  Here the whole operation is one
// launch of exactly the co-resident grid, phases separated by grid barriers:
//
//   1 coarse histogram  buckets = W consecutive output columns (W chosen so a
//                       bucket holds ~1k elements and there are <= 8192 of
//                       them); each CTA counts its chunk in shared memory and
//                       reserves its range inside every non-empty bucket with
//                       ONE global atomic per bucket.           [grid barrier]
//   2 coarse scan       every CTA scans the bucket counts itself (no barrier)
//   3 scatter           each chunk re-read; slot = bucket start + CTA range +
//                       shared cursor; key (row << 32 | input index), column
//                       and value moved to the slot.            [grid barrier]
//   4 bucket tiles      a CTA per bucket (dynamic tickets) sorts it by
//                       (column, row, input order) in shared memory -- up to
//                       1024 bins over the tile's (column, row) range, every
//                       key ranking itself in its bin -- reduces runs in the
//                       reference order, prunes zeros, writes the compacted
//                       bucket to temporaries and the kept count of each
//                       column.  Buckets larger than the tile are split in
//                       global memory into per-column row-prefix bins and
//                       processed a tile-sized group of bins at a time.
//                                                               [grid barrier]
//   5 columns           grid-wide scan of the kept counts -> col_ptr; output
//                       ranges copied to their final offsets.   [2 barriers]
//
// Pre-bucketed mode (pre_ptr != nullptr, SpGEMM): the input already sits in
// column order, phases 1-3 are replaced by variable-width buckets computed
// from pre_ptr (kPreT) and queued largest size class first.
#pragma once

#include "tile_common.cuh"

namespace as {

#define AS_PHASE_MARK(a, gen)                                                                   \
  do {                                                                                          \
    if ((a).phase_ts && blockIdx.x == 0 && threadIdx.x == 0) (a).phase_ts[gen] = global_ns();   \
  } while (0)

// Tile-step timers (diagnostic build only, -DAS_TILE_TIMES): thread 0 of
// block 0 accumulates clock64 cycles per step of the tile loop in g_tt.
#ifdef AS_TILE_TIMES
__device__ unsigned long long g_tt[33];
AS_DEVICE_INLINE void tt_mark(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long n = clock64();
    if (i >= 0) g_tt[i] += n - g_tt[32];
    g_tt[32] = n;
  }
}
#else
AS_DEVICE_INLINE void tt_mark(int) {}
#endif

// ------------------------------------------------------------------------
// element sources: visit(p, P, report, f) calls f(col, row, idx, i) for every
// valid element of chunk p of P (the same partition every time it is called)

constexpr int kVisitVec = 4;  // consecutive elements per thread (ILP)

template <class IdxT>
AS_DEVICE_INLINE void load_vec4(const IdxT* p, long long i, long long hi, long long* out) {
  const bool al = ((reinterpret_cast<unsigned long long>(p + i) & 15ull) == 0);  // any base pointer
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

// four consecutive values (128-bit loads when aligned)
template <class T>
AS_DEVICE_INLINE void load_vals4(const T* p, long long i, long long hi, T* out) {
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

template <class IdxT, class T>
struct CooSrc {
  const IdxT* rows;
  const IdxT* cols;
  const T* vals;
  long long n;
  long long n_rows, n_cols;
  unsigned long long idx_off;
  long long* bad;  // first invalid triplet (reported in phase 1)

  // f(col, minor, idx, i, value); kVal: the values are loaded with the
  // indices (vectorised) so the scatter does not wait on a late scalar load
  template <bool kVal = false, class F>
  __device__ void visit(long long p, long long P, bool report, F f) const {
    const long long ch = (((n + P - 1) / P) + 3) & ~3ll;
    const long long lo = min(n, p * ch), hi = min(n, lo + ch);
    for (long long i = lo + (long long)threadIdx.x * kVisitVec; i < hi; i += (long long)blockDim.x * kVisitVec) {
      long long r[4], c[4];
      T v[4] = {T(0), T(0), T(0), T(0)};
      load_vec4(rows, i, hi, r);
      load_vec4(cols, i, hi, c);
      if (kVal) load_vals4(vals, i, hi, v);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const long long e = i + k;
        if (e >= hi) break;
        if (r[k] < 0 || r[k] >= n_rows || c[k] < 0 || c[k] >= n_cols) {
          if (report && bad) atomicMin((unsigned long long*)bad, (unsigned long long)e);
          continue;
        }
        f((unsigned)c[k], (unsigned)r[k], (unsigned long long)e + idx_off, e, v[k]);
      }
    }
  }
  AS_DEVICE_INLINE T value(long long i) const { return vals[i]; }
  __host__ __device__ long long size() const { return n; }
  AS_DEVICE_INLINE void set_cache(int*) {}
};

// COO triplets in pinned HOST memory (zero-copy over PCIe).  The first pass
// (phase 1, report = true) streams them once from the host -- coalesced, so
// the transfer runs at PCIe speed while the histogram is built -- and stages
// int32 rows / cols and the values in device memory; the second pass (phase
// 3) reads the staged copy.  The host->device copy thus happens inside the
// kernel, overlapped with its first phase (as_coo_to_csc_f64 on host pointers).
template <class IdxT, class T>
struct CooHostSrc {
  CooSrc<IdxT, T> host;  // the triplets as given (host pointers, valid on the device through UVA)
  int* st_rows;
  int* st_cols;
  T* st_vals;

  template <bool kVal = false, class F>
  __device__ void visit(long long p, long long P, bool report, F f) const {
    if (report) {
      host.template visit<true>(p, P, true, [&](unsigned c, unsigned r, unsigned long long idx, long long e, T v) {
        st_rows[e] = (int)r;
        st_cols[e] = (int)c;
        st_vals[e] = v;
        f(c, r, idx, e, v);
      });
    } else {
      CooSrc<int, T> dev{st_rows, st_cols, st_vals, host.n, host.n_rows, host.n_cols, host.idx_off, nullptr};
      dev.template visit<kVal>(p, P, false, f);
    }
  }
  AS_DEVICE_INLINE T value(long long i) const { return st_vals[i]; }
  __host__ __device__ long long size() const { return host.n; }
  AS_DEVICE_INLINE void set_cache(int*) {}
};

// The elements of a CSC: by_row = false -> output column = col, minor = row
// (flush base); by_row = true -> output column = row, minor = col (transpose).
// Chunk p is the element range [p*ch, (p+1)*ch); the column starts it spans
// are staged in shared memory (colc) when they fit.
constexpr int kColCache = 1024;

template <class T>
struct CscSrc {
  const int* col_ptr;
  const int* row_idx;
  const T* vals;
  long long n_cols;
  long long nnz;
  bool by_row;
  unsigned long long idx_off;
  int* colc;

  template <bool kVal = false, class F>
  __device__ void visit(long long p, long long P, bool report, F f) const {
    (void)report;
    __shared__ long long s_cb, s_ce;
    if (nnz == 0) return;
    const long long ch = (((nnz + P - 1) / P) + 3) & ~3ll;
    const long long lo = min(nnz, p * ch), hi = min(nnz, lo + ch);
    __syncthreads();
    if (threadIdx.x == 0 && lo < hi) {
      s_cb = upper_bound_dev(col_ptr, n_cols + 1, (int)lo) - 1;
      s_ce = upper_bound_dev(col_ptr, n_cols + 1, (int)(hi - 1));
    }
    __syncthreads();
    if (lo >= hi) return;
    const long long cb = s_cb, ce = s_ce;
    const bool cached = (ce - cb) <= kColCache;
    if (cached)
      for (long long c = cb + threadIdx.x; c <= ce; c += blockDim.x) colc[c - cb] = col_ptr[c];
    __syncthreads();
    for (long long i = lo + (long long)threadIdx.x * kVisitVec; i < hi; i += (long long)blockDim.x * kVisitVec) {
      long long c;
      if (cached) {
        int l = 0, h = (int)(ce - cb);
        while (l < h) {
          const int mid = (l + h + 1) >> 1;
          if (colc[mid] <= i) l = mid;
          else h = mid - 1;
        }
        c = cb + l;
      } else {
        c = upper_bound_dev(col_ptr + cb, ce - cb + 1, (int)i) - 1 + cb;
      }
      long long r[4];
      T v[4] = {T(0), T(0), T(0), T(0)};
      load_vec4(row_idx, i, hi, r);
      if (kVal) load_vals4(vals, i, hi, v);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const long long e = i + k;
        if (e >= hi) break;
        while ((cached ? colc[c + 1 - cb] : col_ptr[c + 1]) <= e) c++;
        if (by_row) f((unsigned)r[k], (unsigned)c, (unsigned long long)e + idx_off, e, v[k]);
        else f((unsigned)c, (unsigned)r[k], (unsigned long long)e + idx_off, e, v[k]);
      }
    }
    __syncthreads();
  }
  AS_DEVICE_INLINE T value(long long i) const { return vals[i]; }
  __host__ __device__ long long size() const { return nnz; }
  AS_DEVICE_INLINE void set_cache(int* p) { colc = p; }
};

template <class T>
struct NoSrc {
  template <bool kVal = false, class F>
  __device__ void visit(long long, long long, bool, F) const {}
  AS_DEVICE_INLINE T value(long long) const { return T(0); }
  __host__ __device__ long long size() const { return 0; }
  AS_DEVICE_INLINE void set_cache(int*) {}
};

// ------------------------------------------------------------------------
#ifndef AS_PERSIST_MINB
#define AS_PERSIST_MINB 2  // CTAs per SM the register allocation is sized for
#endif
constexpr int kMaxCoarse = 8192;  // coarse buckets (two u32 arrays in smem)
constexpr int kMaxW = 1024;       // columns per coarse bucket
#ifndef AS_TBINS
#define AS_TBINS 1024
#endif
constexpr int kTBins = AS_TBINS;  // second-level bins per bucket tile

// the pre-bucketed instantiation (SpGEMM's reduce, always kSumSeq)
template <class T, class S1, class S2>
constexpr bool kPreOnly = std::is_same<S1, NoSrc<T>>::value && std::is_same<S2, NoSrc<T>>::value;

template <class T, class S1, class S2>
struct PersistArgs {
  S1 s1;
  S2 s2;
  long long n_cols;   // output columns (fine buckets)
  long long n_upper;  // s1.size() + s2.size()
  unsigned long long cb_mul;  // coarse bucket = (column * cb_mul) >> 32 (phases 1-3)
  long long n_cb;
  unsigned* cb_cnt;       // [n_cb] zeroed
  long long* cb_start;    // [n_cb + 1]
  unsigned long long* keys;
  unsigned long long* keys_alt;
  unsigned* colb;         // output column of each bucketed element
  unsigned* colb_alt;
  T* vals_b;              // bucketed values (by slot)
  int* tmp_rows;
  T* tmp_vals;
  unsigned* col_kept;     // [n_cols]
  long long* cta_sums;    // [grid]
  int row_bits, idx_bits;
  int mode, prune;
  ValSrc<T> vs;           // values by input index (oversized buckets)
  int* col_ptr;
  int* row_idx;
  T* out_vals;
  long long* info;
  unsigned* ticket;
  GridBar gb;
  unsigned long long* phase_ts;  // optional: globaltimer after each phase (debug)
  int stage;                     // 1: phase 3 stages each CTA's chunk in shared memory (stage_layout)
  long long dense_rows;          // pre mode: > 0 = output rows; columns above the tile take the dense path
  const long long* pre_ptr;      // non-null: input already bucketed by column (SpGEMM products)
  // bucket t spans columns [cb_col[t], cb_col[t+1]); pre_ptr mode: tiles are
  // taken in `order` (largest size class first)
  unsigned* cb_col;              // [n_cb + 1]
  unsigned* order;               // [n_cb] (pre_ptr mode only)
  unsigned long long* tstate;    // zeroed: [n_cb] bucket kept counts, then [n_cb / 32 + 1] group words
  // two-level scatter (large inputs): super-buckets of sb_f consecutive buckets
  int sb_f;                      // buckets per super-bucket (<= 1: single level)
  long long n_sb;
  unsigned* sb_cnt;              // [n_sb] zeroed: per-super-bucket range reservation
  unsigned* sb_fill;             // [n_cb] zeroed: per-bucket fill of the second scatter
  T* vals_alt;                   // [n] staging of the first scatter
};

// Variable-width buckets of pre-bucketed input: column c weighs
// len(c) + kPreColCost, bucket t holds the columns whose cumulative weight
// starts in [t * kPreT, (t+1) * kPreT) -- at most kPreT / kPreColCost columns
// and kPreT elements plus the length of its last column.
constexpr long long kPreT = 1536;
constexpr long long kPreColCost = 2;
static_assert(kPreT / kPreColCost + 1 <= kMaxW, "variable bucket wider than a tile");

template <class T>
struct BTileSmem {
  unsigned long long sk[kCap];
  union {
    T rv[kCap];
    unsigned long long sk2[kCap];
    struct {
      unsigned hist[256];
      unsigned wcnt[256 * (kSegThreads / 32)];
    } rs;
  } u;
  union {
    unsigned short excl[kCap + 8];
    struct {  // the sort's bins and scatter (excl is written after it)
      unsigned cursor[kTBins];
      unsigned short bstart[kTBins + 8];
      unsigned short perm2[kCap];
      unsigned short sbin[kCap];
    } bk;
  } v;
  unsigned short scol[kCap];   // local column of each key (sk order)
  unsigned short perm[kCap];
  unsigned short cstart[kMaxW + 8];  // column boundaries (tile positions)
  unsigned hbits[kCap / 32];
  short med[kTBins], big[kTBins];
  int n_med, n_big;
  long long scan_tmp[kSegThreads / 32 + 1];
  unsigned ckept[kMaxW];  // kept per column (oversized path)
  unsigned obin[2 * kTBins + 1];  // bin starts of an oversized bucket's split
  unsigned long long cmin, cmax;  // (column, row) range of a tile
  long long tile, s, m, col_base, prefix;
  int wt;
};

// Dynamic shared memory of the persistent kernel: two CTAs per SM (the
// register file is the binding limit), so ~110 KB each is free to use.
#ifndef AS_PERSIST_SMEM_KB
#define AS_PERSIST_SMEM_KB (AS_PERSIST_MINB == 1 ? 224 : 110)
#endif
constexpr int kPersistSmemBytes = AS_PERSIST_SMEM_KB * 1024;

// Phases 1-3: colc, then three runtime-sized [n_cb] arrays (histogram /
// cursor, the CTA's range inside each bucket, the CTA-local bucket offsets),
// then the scatter staging (stage_layout).  Phase 4: the tile.
template <class T>
union PersistSmem {
  struct {
    int colc[kColCache + 1];
    unsigned ab[3 * kMaxCoarse];
  } h;
  BTileSmem<T> t;
  unsigned char raw[kPersistSmemBytes];
};
static_assert(sizeof(BTileSmem<double>) <= kPersistSmemBytes, "tile above the shared-memory budget");

// Scatter staging behind the [3 * n_cb] arrays: keys, values, columns of the
// CTA's chunk in local bucket order.  Returns the capacity in elements.
template <class T>
__host__ __device__ inline long long stage_layout(long long ncb, long long* off) {
  const long long o = ((long long)sizeof(int) * (kColCache + 1) + 12ll * ncb + 15) & ~15ll;
  *off = o;
  return o >= kPersistSmemBytes ? 0 : (kPersistSmemBytes - o) / (long long)(12 + sizeof(T));
}

AS_DEVICE_INLINE void cta_range(long long n, long long g, long long G, long long* lo, long long* hi) {
  const long long per = (n + G - 1) / G;
  *lo = min(n, g * per);
  *hi = min(n, *lo + per);
}

// Block-level stable LSD radix sort of (u64 key, u32 payload) pairs in global
// memory; pass i sorts by bits [shift, shift+nbits) of the key (from_payload
// = 0) or of the payload (1).  Leaves the result in (k, p).
static __device__ void block_radix_sort_kv(unsigned long long* k, unsigned* p, unsigned long long* k_alt, unsigned* p_alt,
                                    long long L, const int* shifts, const int* nbits, const int* from_payload,
                                    int npass, unsigned* hist, unsigned* wcnt) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  unsigned long long *sk = k, *dk = k_alt;
  unsigned *sp = p, *dp = p_alt;
  for (int ps = 0; ps < npass; ps++) {
    const int sh = shifts[ps];
    const unsigned mask = (1u << nbits[ps]) - 1u;
    const bool fp = from_payload[ps];
    auto digit = [&](long long i) -> unsigned {
      return fp ? ((sp[i] >> sh) & mask) : ((unsigned)(sk[i] >> sh) & mask);
    };
    for (int i = tid; i < 256; i += nthr) hist[i] = 0;
    for (int i = tid; i < 256 * nwarps; i += nthr) wcnt[i] = 0;
    __syncthreads();
    for (long long i = tid; i < L; i += nthr) atomicAdd(&hist[digit(i)], 1u);
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
    for (long long base = 0; base < L; base += nthr) {
      const long long i = base + tid;
      const bool in = i < L;
      const unsigned dg = in ? digit(i) : 0xffffffffu;
      const unsigned act = __ballot_sync(0xffffffffu, in);
      unsigned rank = 0;
      if (in) {
        const unsigned peers = __match_any_sync(act, dg);
        rank = __popc(peers & lanemask_lt());
        if (rank == 0) wcnt[warp * 256 + dg] = __popc(peers);
      }
      __syncthreads();
      for (int b = tid; b < 256; b += nthr) {
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
      for (int b = tid; b < 256 * nwarps; b += nthr) wcnt[b] = 0;
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
    for (long long i = tid; i < L; i += nthr) {
      k[i] = sk[i];
      p[i] = sp[i];
    }
    __syncthreads();
  }
}

// Reduce the runs of one chunk [b, b+cm) of a sorted bucket whose keys / local
// columns are in S.sk / S.scol.  Runs end at a column or row change; a run
// crossing the chunk end continues in global memory (gk, gcol; nullptr when
// the chunk is the whole bucket).  vslot: values by tile slot through S.perm
// (nullptr: values by input index).  Leaves S.u.rv[p] = run value at kept
// heads, S.v.excl[0..cm] exclusive kept counts; returns the chunk total.
template <class T, class VS, bool kSeqOnly = false>
__device__ long long bucket_chunk_reduce(BTileSmem<T>& S, long long b, int cm, long long m,
                                         const unsigned long long* gk, const unsigned* gcol, unsigned col_base,
                                         VS vs, int mode, int prune, const T* vslot) {
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
  for (int base = 0; base < cm; base += nthr) {
    const int p = base + tid;
    bool head = false;
    if (p < cm) {
      const unsigned long long k = S.sk[p];
      const unsigned row = key_row(k), col = S.scol[p];
      if (p > 0) head = row != key_row(S.sk[p - 1]) || col != S.scol[p - 1];
      else head = (b == 0) || row != key_row(gk[b - 1]) || col != gcol[b - 1] - col_base;
      if (vslot) {  // bucket-ordered values: an asynchronous copy, so the gathers of all
                    // iterations are in flight together (no registers held)
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&S.u.rv[p]);
        if constexpr (sizeof(T) == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(vslot + S.perm[p]) : "memory");
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(vslot + S.perm[p]) : "memory");
      } else {
        S.u.rv[p] = vs((unsigned long long)key_idx(k));
      }
    }
    const unsigned hb = __ballot_sync(0xffffffffu, head);
    if (lane == 0 && base + warp * 32 < cm) S.hbits[(base >> 5) + warp] = hb;
  }
  if (vslot) asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
  __syncthreads();
  tt_mark(8);
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
          auto get = [&](long long i) -> T { return rvp[i]; };
          v = reduce_run<T, decltype(get), kSeqOnly>(get, q - p, mode);
        }
      } else {
        const unsigned row = key_row(S.sk[p]), col = S.scol[p] + col_base;
        long long qg = b + cm;
        while (qg < m && key_row(gk[qg]) == row && gcol[qg] == col) qg++;
        const T* rvp = S.u.rv + p;
        const long long in_chunk = cm - p;
        const unsigned long long* gkp = gk + b + p;
        auto get = [&](long long i) -> T {
          return i < in_chunk ? rvp[i] : vs((unsigned long long)key_idx(gkp[i]));
        };
        v = reduce_run<T, decltype(get), kSeqOnly>(get, qg - (b + p), mode);
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
  tt_mark(9);
  return total;
}

// Sort a bucket held in S.sk / S.scol (tile positions, perm = identity) by
// (column, row, input order).  Bins are aligned ranges of the composite
// (column << row_bits | row) between the tile's min and max, at most kTBins
// of them and never wider than one column; counting pass, scan, scatter to
// S.u.sk2, then rank-in-bin placement back into S.sk (long bins: warp /
// block bitonic).  Leaves S.scol in sorted order and S.cstart[l] = first
// position of local column l (l = 0..Wt).  m >= 1.
template <class T>
__device__ void sort_bucket_smem(BTileSmem<T>& S, int m, int Wt, int row_bits) {
  const int tid = threadIdx.x, nthr = blockDim.x, warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  auto comp = [&](int p) -> unsigned long long {
    return ((unsigned long long)S.scol[p] << row_bits) | key_row(S.sk[p]);
  };
  if (tid == 0) {
    S.cmin = ~0ull;
    S.cmax = 0ull;
  }
  __syncthreads();
  {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int p = tid; p < m; p += nthr) {
      const unsigned long long c = comp(p);
      lo = min(lo, c);
      hi = max(hi, c);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      atomicMin(&S.cmin, lo);
      atomicMax(&S.cmax, hi);
    }
  }
  __syncthreads();
  tt_mark(2);
  const unsigned long long cmin = S.cmin, cmax = S.cmax;
  int sh = 0;
  while (sh < row_bits && (cmax >> sh) - (cmin >> sh) + 1 > (unsigned long long)kTBins) sh++;
  const unsigned long long cbase = cmin >> sh;
  const int nbins = (int)((cmax >> sh) - cbase + 1);  // <= kTBins: at sh = row_bits it counts columns
  auto bin_of = [&](int p) -> int { return (int)((comp(p) >> sh) - cbase); };
  auto col_of_bin = [&](int b) -> unsigned short {
    return (unsigned short)(((cbase + (unsigned long long)b) << sh) >> row_bits);
  };
  for (int b = tid; b < nbins; b += nthr) S.v.bk.cursor[b] = 0u;
  __syncthreads();
  for (int p = tid; p < m; p += nthr) atomicAdd(&S.v.bk.cursor[bin_of(p)], 1u);
  __syncthreads();
  tt_mark(3);
  {
    constexpr int kPer = kTBins / kSegThreads;
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
  tt_mark(4);
  for (int p = tid; p < m; p += nthr) {
    const int b = bin_of(p);
    const unsigned slot = atomicAdd(&S.v.bk.cursor[b], 1u);
    S.u.sk2[slot] = S.sk[p];
    S.v.bk.perm2[slot] = S.perm[p];
    S.v.bk.sbin[slot] = (unsigned short)b;
  }
  if (tid == 0) {
    S.n_med = 0;
    S.n_big = 0;
  }
  for (int l = tid; l <= Wt; l += nthr) {
    const long long bl = (long long)(((unsigned long long)l << row_bits) >> sh) - (long long)cbase;
    S.cstart[l] = S.v.bk.bstart[bl < 0 ? 0 : (bl > nbins ? nbins : bl)];
  }
  __syncthreads();
  tt_mark(5);
  for (int b = tid; b < nbins; b += nthr) {
    const int L = S.v.bk.bstart[b + 1] - S.v.bk.bstart[b];
    if (L > kRankMax && L <= kWarpSortMax) S.med[atomicAdd(&S.n_med, 1)] = (short)b;
    else if (L > kWarpSortMax) S.big[atomicAdd(&S.n_big, 1)] = (short)b;
  }
  for (int q = tid; q < m; q += nthr) {
    const int b = S.v.bk.sbin[q];
    const int s0 = S.v.bk.bstart[b], e0b = S.v.bk.bstart[b + 1];
    if (e0b - s0 <= kRankMax) {
      const unsigned long long k = S.u.sk2[q];
      int r = 0;
      for (int j = s0; j < e0b; j++) r += (S.u.sk2[j] < k);
      S.sk[s0 + r] = k;
      S.perm[s0 + r] = S.v.bk.perm2[q];
      S.scol[s0 + r] = col_of_bin(b);
    }
  }
  __syncthreads();
  tt_mark(6);
  const int n_med = S.n_med, n_big = S.n_big;
  for (int q = warp; q < n_med; q += nwarps) {
    const int b = S.med[q];
    const int s0 = S.v.bk.bstart[b], L = S.v.bk.bstart[b + 1] - s0;
    bitonic_sort<false>(S.u.sk2 + s0, L, lane, 32, S.v.bk.perm2 + s0);
    for (int i = lane; i < L; i += 32) {
      S.sk[s0 + i] = S.u.sk2[s0 + i];
      S.perm[s0 + i] = S.v.bk.perm2[s0 + i];
      S.scol[s0 + i] = col_of_bin(b);
    }
  }
  for (int q = 0; q < n_big; q++) {
    const int b = S.big[q];
    const int s0 = S.v.bk.bstart[b], L = S.v.bk.bstart[b + 1] - s0;
    bitonic_sort<true>(S.u.sk2 + s0, L, tid, nthr, S.v.bk.perm2 + s0);
    for (int i = tid; i < L; i += nthr) {
      S.sk[s0 + i] = S.u.sk2[s0 + i];
      S.perm[s0 + i] = S.v.bk.perm2[s0 + i];
      S.scol[s0 + i] = col_of_bin(b);
    }
    __syncthreads();
  }
  __syncthreads();
  tt_mark(7);
}

// A bucket larger than the tile: split it in global memory into bins of
// (column, high row bits) -- every (column, row) run stays inside one bin --
// then process consecutive bins in groups that fit the tile with the shared-
// memory sort; a single bin still larger than the tile is radix-sorted in
// global memory and streamed.  Values are read by input index.
template <class T, class S1, class S2>
__device__ long long process_oversized_bucket(BTileSmem<T>& S, PersistArgs<T, S1, S2>& a, long long s, long long m,
                                         unsigned col_base, int Wt) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int W = Wt;
  unsigned* bstart = S.obin;  // nbins + 1 u32 bin starts (bucket-relative)
  unsigned* cursor = reinterpret_cast<unsigned*>(&S.u) + kMaxW;  // [<= 2 * kTBins] (S.u is free here)
  unsigned long long* gk = a.keys + s;
  unsigned* gc = a.colb + s;
  unsigned long long* ak = a.keys_alt + s;
  unsigned* ac = a.colb_alt + s;
  // per-column row split sized from the column's count: column l gets
  // 2^lr[l] bins of ~`target` keys, so one heavy column does not overflow
  // the tile (bins of one (column, row prefix) still keep every run whole)
  unsigned* ccount = reinterpret_cast<unsigned*>(&S.u);  // [W] column counts
  unsigned short* bbase = S.scol;          // [W+1] first bin of each column
  unsigned short* clr = S.perm;            // [W]  row-prefix bits per column
  for (int l = tid; l < W; l += nthr) ccount[l] = 0u;
  for (int l = tid; l < Wt; l += nthr) S.ckept[l] = 0u;
  __syncthreads();
  for (long long i = tid; i < m; i += nthr) atomicAdd(&ccount[gc[i] - col_base], 1u);
  __syncthreads();
  // sum_l 2^lr[l] <= W + 2m/target <= 2*kTBins bins
  const unsigned target = (unsigned)max(1024ll, (2 * m + (2 * kTBins - W) - 1) / (2 * kTBins - W));
  if (tid < 32) {
    unsigned carry = 0;
    for (int l0 = 0; l0 < W; l0 += 32) {
      const int l = l0 + tid;
      int lr = 0;
      if (l < W)
        while (lr < a.row_bits && (ccount[l] >> lr) > target) lr++;
      const unsigned nb = l < W ? (1u << lr) : 0u;
      const unsigned inc = warp_inclusive_scan(nb);
      if (l < W) {
        bbase[l] = (unsigned short)(carry + inc - nb);
        clr[l] = (unsigned short)lr;
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (tid == 0) bbase[W] = (unsigned short)carry;
  }
  __syncthreads();
  const int nbins = bbase[W];
  auto bin_of = [&](unsigned long long k, unsigned c) -> int {
    const int l = (int)(c - col_base);
    return (int)bbase[l] + (int)(key_row(k) >> (a.row_bits - clr[l]));
  };
  for (int b = tid; b < nbins; b += nthr) cursor[b] = 0u;
  __syncthreads();
  for (long long i = tid; i < m; i += nthr) atomicAdd(&cursor[bin_of(gk[i], gc[i])], 1u);
  __syncthreads();
  if (tid < 32) {
    unsigned carry = 0;
    for (int b0 = 0; b0 < nbins; b0 += 32) {
      const unsigned v = (b0 + tid < nbins) ? cursor[b0 + tid] : 0u;
      const unsigned inc = warp_inclusive_scan(v);
      if (b0 + tid < nbins) {
        bstart[b0 + tid] = carry + inc - v;
        cursor[b0 + tid] = carry + inc - v;
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (tid == 0) bstart[nbins] = carry;
  }
  __syncthreads();
  for (long long i = tid; i < m; i += nthr) {
    const unsigned long long k = gk[i];
    const unsigned c = gc[i];
    const unsigned pos = atomicAdd(&cursor[bin_of(k, c)], 1u);
    ak[pos] = k;
    ac[pos] = c;
  }
  __syncthreads();
  long long run_base = 0;
  int b0 = 0;
  while (b0 < nbins) {  // block-uniform walk over groups of bins
    int b1 = b0 + 1;
    while (b1 < nbins && bstart[b1 + 1] - bstart[b0] <= (unsigned)kCap) b1++;
    const long long e0 = bstart[b0], L = (long long)bstart[b1] - e0;
    if (L > 0 && L <= kCap) {
      for (int i = tid; i < L; i += nthr) {
        S.sk[i] = ak[e0 + i];
        S.scol[i] = (unsigned short)(ac[e0 + i] - col_base);
        S.perm[i] = (unsigned short)i;
      }
      __syncthreads();
      sort_bucket_smem(S, (int)L, W, a.row_bits);
      const long long ctot = bucket_chunk_reduce<T, decltype(a.vs), kPreOnly<T, S1, S2>>(S, 0, (int)L, L, nullptr, nullptr, col_base, a.vs, a.mode,
                                                    a.prune, nullptr);
      for (int p = tid; p < L; p += nthr) {
        const unsigned x0 = S.v.excl[p], x1 = S.v.excl[p + 1];
        if (x1 != x0) {
          a.tmp_rows[s + run_base + x0] = (int)key_row(S.sk[p]);
          a.tmp_vals[s + run_base + x0] = S.u.rv[p];
          atomicAdd(&S.ckept[S.scol[p]], 1u);
        }
      }
      run_base += ctot;
      __syncthreads();
    } else if (L > kCap) {  // one bin (one column) above the tile: global radix sort by (row, idx), streamed reduce
      int shifts[16], nbits[16], fromp[16], np = 0;
      for (int bb = 0; bb < a.idx_bits; bb += 8) {
        shifts[np] = bb;
        nbits[np] = min(8, a.idx_bits - bb);
        fromp[np] = 0;
        np++;
      }
      for (int bb = 0; bb < a.row_bits; bb += 8) {
        shifts[np] = 32 + bb;
        nbits[np] = min(8, a.row_bits - bb);
        fromp[np] = 0;
        np++;
      }
      __syncthreads();
      block_radix_sort_kv(ak + e0, ac + e0, gk + e0, gc + e0, L, shifts, nbits, fromp, np, S.u.rs.hist,
                          S.u.rs.wcnt);
      unsigned long long* bk2 = ak + e0;
      unsigned* bc2 = ac + e0;
      for (long long b = 0; b < L; b += kCap) {
        const int cm = (int)min((long long)kCap, L - b);
        for (int i = tid; i < cm; i += nthr) {
          S.sk[i] = bk2[b + i];
          S.scol[i] = (unsigned short)(bc2[b + i] - col_base);
        }
        __syncthreads();
        const long long ctot = bucket_chunk_reduce<T, decltype(a.vs), kPreOnly<T, S1, S2>>(S, b, cm, L, bk2, bc2, col_base, a.vs, a.mode, a.prune,
                                                      nullptr);
        for (int p = tid; p < cm; p += nthr) {
          const unsigned x0 = S.v.excl[p], x1 = S.v.excl[p + 1];
          if (x1 != x0) {
            a.tmp_rows[s + run_base + x0] = (int)key_row(S.sk[p]);
            a.tmp_vals[s + run_base + x0] = S.u.rv[p];
            atomicAdd(&S.ckept[S.scol[p]], 1u);
          }
        }
        run_base += ctot;
        __syncthreads();
      }
    }
    b0 = b1;
  }
  for (int l = tid; l < Wt; l += nthr) a.col_kept[col_base + l] = S.ckept[l];
  __syncthreads();
  return run_base;
}

// Pre-bucketed mode (SpGEMM): a tile of m <= kCap products [s, s+m) over Wt
// columns sorted and folded in shared memory; kept entries to tmp[s + ...],
// kept counts per column to col_kept.  Returns the tile's kept total.
template <class T, class S1, class S2>
__device__ long long pre_tile_to_tmp(BTileSmem<T>& S, PersistArgs<T, S1, S2>& a, long long s, int m, unsigned col_base,
                                     int Wt) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < m; i += nthr) {
    S.sk[i] = __ldcg(&a.keys[s + i]);
    S.scol[i] = (unsigned short)(__ldcg(&a.colb[s + i]) - col_base);
    S.perm[i] = (unsigned short)i;
  }
  __syncthreads();
  sort_bucket_smem(S, m, Wt, a.row_bits);
  bucket_chunk_reduce<T, decltype(a.vs), kPreOnly<T, S1, S2>>(S, 0, m, m, nullptr, nullptr, col_base, a.vs, a.mode, a.prune, a.vals_b + s);
  for (int p = tid; p < m; p += nthr) {
    const unsigned e0 = S.v.excl[p], e1 = S.v.excl[p + 1];
    if (e1 != e0) {
      a.tmp_rows[s + e0] = (int)key_row(S.sk[p]);
      a.tmp_vals[s + e0] = S.u.rv[p];
    }
  }
  for (int l = tid; l < Wt; l += nthr) a.col_kept[col_base + l] = S.v.excl[S.cstart[l + 1]] - S.v.excl[S.cstart[l]];
  const long long kept = S.v.excl[m];
  __syncthreads();
  return kept;
}

// Multi-product rows whose counters / list cursors live in shared memory
// (more: global memory).
constexpr int kDenseSmemCnt = 4096;

// Shared memory of the dense column path for n_rows rows: two bitmaps of
// nw = ceil(n_rows / 32) words, their u16 prefixes inside groups of 32 words
// and the u32 group prefixes.
__host__ __device__ inline long long dense_column_bytes(long long n_rows) {
  const long long nw = (n_rows + 31) / 32;
  return nw <= 0 ? 0 : 12 * nw + 8 * (nw / 32 + 2) + 16 + 4 * kDenseSmemCnt;
}

// One output column of SpGEMM with L products at [g0, g0 + L) (product
// order = the reference's accumulation order: B entry, then A position),
// folded without sorting the products (Gustavson's dense accumulator,
// _kernels.py:83-93, made parallel):
//   1. every product sets its row's bit in `seen`; a row seen before also
//      sets `multi` (shared-memory bitmaps over all rows);
//   2. coarse popcount prefixes: rank(row) = the row's position in the
//      sorted output, mrank(row) = its index among the multi rows;
//   3. a product of a single-product row is the output itself: written to
//      tmp[out + rank]; a multi row counts its products;
//   4. the multi rows' products are listed per row (scan of the counts,
//      then placement) and each multi row folds its few products in product
//      order (first assigns, then +=: kSumSeq), written to tmp[out + rank];
//   5. exact zeros (underflowed products, cancellations) are compacted away.
// Scratch: keys_alt / colb_alt (and the keys of a row-only column) at
// [g0, g0 + L) (free in pre mode).  Returns the kept count.
template <class T, class S1, class S2>
__device__ long long pre_dense_column(BTileSmem<T>& S, PersistArgs<T, S1, S2>& a, long long g0, long long L,
                                      long long out) {
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  const int nw = (int)((a.dense_rows + 31) / 32);  // bitmap words
  const int ng = (nw + 31) >> 5;                  // groups of 32 words
  unsigned* seen = reinterpret_cast<unsigned*>(&S);
  unsigned* multi = seen + nw;
  unsigned* sgrp = multi + nw;   // [ng + 1] seen prefix per group
  unsigned* mgrp = sgrp + ng + 1;  // [ng + 1] multi prefix per group
  unsigned short* spre = reinterpret_cast<unsigned short*>(mgrp + ng + 1);  // [nw] seen prefix inside the group
  unsigned short* mpre = spre + nw;                                          // [nw] multi prefix inside the group
  unsigned* scnt = reinterpret_cast<unsigned*>(reinterpret_cast<unsigned char*>(seen) +
                                               ((dense_column_bytes(a.dense_rows) - 4 * kDenseSmemCnt) & ~15ll));
  __shared__ unsigned s_tot[2];
  __shared__ int s_zero;
  __shared__ long long s_scan[kSegThreads / 32 + 1];  // the tile's scan_tmp lies under the bitmaps
  for (int w = tid; w < 2 * nw; w += nthr) seen[w] = 0u;
  if (tid == 0) s_zero = 0;
  __syncthreads();
  tt_mark(12);
  // rows of the products: a column above kCap products was expanded without
  // keys, its rows in colb (spgemm_expand_kernel); a smaller one has keys
  const bool rows_in_colb = L > kCap;
  const unsigned* grow = a.colb + g0;
  const unsigned long long* gk = a.keys + g0;
  auto row_at = [&](long long i) -> unsigned { return rows_in_colb ? __ldcg(&grow[i]) : key_row(__ldcg(&gk[i])); };
  // 1. seen / multi
  constexpr int kU = 8;  // products in flight per thread (the keys stream from HBM)
  for (long long i0 = tid; i0 < L; i0 += (long long)kU * nthr) {
    unsigned r[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
      const long long i = i0 + (long long)u * nthr;
      r[u] = i < L ? row_at(i) : 0xffffffffu;
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
      if (r[u] == 0xffffffffu) continue;
      const unsigned bit = 1u << (r[u] & 31);
      if (atomicOr(&seen[r[u] >> 5], bit) & bit) atomicOr(&multi[r[u] >> 5], bit);
    }
  }
  __syncthreads();
  tt_mark(13);
  // 2. prefixes: per word inside its group of 32 (one warp per group), then
  //    over the groups (both counts in one scan: multi << 32 | seen)
  for (int g = warp; g < ng; g += nwarps) {
    const int w = g * 32 + lane;
    const unsigned cs = w < nw ? __popc(seen[w]) : 0u, cm = w < nw ? __popc(multi[w]) : 0u;
    const unsigned is = warp_inclusive_scan(cs), im = warp_inclusive_scan(cm);
    if (w < nw) {
      spre[w] = (unsigned short)(is - cs);
      mpre[w] = (unsigned short)(im - cm);
    }
    if (lane == 31) {
      sgrp[g] = is;
      mgrp[g] = im;
    }
  }
  __syncthreads();
  {
    unsigned long long run = 0;
    for (int g0g = 0; g0g < ng; g0g += nthr) {
      const int g = g0g + tid;
      const unsigned long long c = g < ng ? (((unsigned long long)mgrp[g] << 32) | sgrp[g]) : 0ull;
      long long tot;
      const long long ex = block_exclusive_scan<long long>((long long)c, s_scan, &tot);
      if (g < ng) {
        sgrp[g] = (unsigned)((run + ex) & 0xffffffffull);
        mgrp[g] = (unsigned)((run + ex) >> 32);
      }
      run += (unsigned long long)tot;
    }
    if (tid == 0) {
      s_tot[0] = (unsigned)(run & 0xffffffffull);
      s_tot[1] = (unsigned)(run >> 32);
    }
  }
  __syncthreads();
  tt_mark(14);
  const unsigned touched = s_tot[0], n_mr = s_tot[1];
  // the output rows in order straight from the bitmap (coalesced; the values
  // below land at the same ranks)
  for (int w = tid; w < nw; w += nthr) {
    unsigned bits = seen[w];
    unsigned rk = sgrp[w >> 5] + spre[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1u;
      a.tmp_rows[out + rk++] = w * 32 + b;
    }
  }
  auto rank_in = [&](const unsigned* bm, const unsigned* grp, const unsigned short* pre, unsigned r) -> unsigned {
    const int w = (int)(r >> 5);
    return grp[w >> 5] + pre[w] + __popc(bm[w] & ((1u << (r & 31)) - 1u));
  };
  unsigned long long* meta = a.keys_alt + g0;                              // [n_mr] (rank << 32) | row
  unsigned* cnt = n_mr <= (unsigned)kDenseSmemCnt
                      ? scnt
                      : reinterpret_cast<unsigned*>(a.keys_alt + g0 + (L + 1) / 2);  // [n_mr] counts, then cursors
  unsigned* list = a.colb_alt + g0;                                         // [multi products] local index
  // [multi products] local indices: in the unused keys of a row-only column,
  // else behind meta (n_mr <= kDenseSmemCnt then: the counts are in shared memory)
  unsigned* mlist = rows_in_colb ? reinterpret_cast<unsigned*>(a.keys + g0)
                                 : reinterpret_cast<unsigned*>(a.keys_alt + g0 + (L + 1) / 2);
  __shared__ unsigned s_nmp;
  for (unsigned q = tid; q < n_mr; q += nthr) cnt[q] = 0u;
  if (tid == 0) s_nmp = 0u;
  __syncthreads();
  // 3. single-product rows straight to their output slot; multi rows count
  const T* gv = reinterpret_cast<const T*>(a.vals_b) + g0;
  bool zero = false;
  constexpr int kU3 = 4;
  for (long long i0 = tid; i0 < L; i0 += (long long)kU3 * nthr) {  // warp-uniform trip count
    unsigned r[kU3];
    T v[kU3];
#pragma unroll
    for (int u = 0; u < kU3; u++) {
      const long long i = i0 + (long long)u * nthr;
      r[u] = 0xffffffffu;
      if (i < L) {
        r[u] = row_at(i);
        v[u] = __ldcg(&gv[i]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU3; u++) {
      bool is_multi = false;
      if (r[u] != 0xffffffffu) {
        const unsigned bit = 1u << (r[u] & 31);
        const unsigned rk = rank_in(seen, sgrp, spre, r[u]);
        if (!(multi[r[u] >> 5] & bit)) {
          a.tmp_vals[out + rk] = v[u];  // (the rows come from the bitmap, below)
          zero |= (v[u] == T(0));
        } else {
          const unsigned mr = rank_in(multi, mgrp, mpre, r[u]);
          atomicAdd(&cnt[mr], 1u);
          meta[mr] = ((unsigned long long)rk << 32) | r[u];
          is_multi = true;
        }
      }
      // warp-aggregated append of the multi products
      const unsigned ball = __ballot_sync(__activemask(), is_multi);
      unsigned base = 0;
      if ((tid & 31) == __ffs(ball | 0x80000000u) - 1 && ball) base = atomicAdd(&s_nmp, (unsigned)__popc(ball));
      base = __shfl_sync(__activemask(), base, __ffs(ball | 0x80000000u) - 1);
      if (is_multi) mlist[base + __popc(ball & lanemask_lt())] = (unsigned)(i0 + (long long)u * nthr);
    }
  }
  __syncthreads();
  tt_mark(15);
  // 4. per multi row: its segment of the list (exclusive scan of the counts)
  {
    long long run = 0;
    for (unsigned q0 = 0; q0 < n_mr; q0 += nthr) {
      const unsigned q = q0 + tid;
      const long long c = q < n_mr ? (long long)cnt[q] : 0ll;
      long long tot;
      const long long ex = block_exclusive_scan<long long>(c, s_scan, &tot);
      if (q < n_mr) cnt[q] = (unsigned)(run + ex);
      run += tot;
    }
  }
  __syncthreads();
  tt_mark(16);
  if (n_mr > 0) {
    const unsigned nmp = s_nmp;  // only the multi products, listed by the pass above
    for (unsigned j0 = tid; j0 < nmp; j0 += 4u * nthr) {
      unsigned ii[4], r[4];
#pragma unroll
      for (int u = 0; u < 4; u++) ii[u] = j0 + u * nthr < nmp ? __ldcg(&mlist[j0 + u * nthr]) : 0xffffffffu;
#pragma unroll
      for (int u = 0; u < 4; u++) r[u] = ii[u] != 0xffffffffu ? row_at(ii[u]) : 0u;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (ii[u] != 0xffffffffu) list[atomicAdd(&cnt[rank_in(multi, mgrp, mpre, r[u])], 1u)] = ii[u];
    }
    __syncthreads();
    tt_mark(19);
    for (unsigned q = tid; q < n_mr; q += nthr) {
      const unsigned st = q ? cnt[q - 1] : 0u, en = cnt[q];
      T acc;
      if (en - st <= 8) {  // the row's products in product order: sorted in registers
        unsigned li[8];
#pragma unroll
        for (int x = 0; x < 8; x++) li[x] = st + x < en ? list[st + x] : 0xffffffffu;
#pragma unroll
        for (int x = 1; x < 8; x++)
#pragma unroll
          for (int y = x; y > 0; y--)
            if (li[y] < li[y - 1]) {
              const unsigned t2 = li[y];
              li[y] = li[y - 1];
              li[y - 1] = t2;
            }
        T vv[8];
#pragma unroll
        for (int x = 0; x < 8; x++) vv[x] = li[x] != 0xffffffffu ? __ldcg(&gv[li[x]]) : T(0);
        acc = vv[0];
#pragma unroll
        for (int x = 1; x < 8; x++)
          if (li[x] != 0xffffffffu) acc = acc + vv[x];
      } else {  // long: insertion sort in place
        for (unsigned x = st + 1; x < en; x++) {
          const unsigned key = list[x];
          unsigned y = x;
          while (y > st && list[y - 1] > key) {
            list[y] = list[y - 1];
            y--;
          }
          list[y] = key;
        }
        acc = __ldcg(&gv[list[st]]);
        for (unsigned x = st + 1; x < en; x++) acc = acc + __ldcg(&gv[list[x]]);
      }
      const unsigned long long mt = meta[q];
      a.tmp_vals[out + (mt >> 32)] = acc;
      zero |= (acc == T(0));
    }
  }
  if (zero) s_zero = 1;
  __syncthreads();
  tt_mark(17);
  if (!s_zero || !a.prune) return touched;
  // 5. compact the exact zeros away (rare), chunk by chunk in place
  long long w = 0;
  for (long long b = 0; b < touched; b += nthr) {
    const long long i = b + tid;
    int r = 0;
    T v = T(0);
    if (i < touched) {
      r = __ldcg(&a.tmp_rows[out + i]);
      v = __ldcg(&a.tmp_vals[out + i]);
    }
    const bool keep = i < touched && v != T(0);
    long long tot;
    const long long ex = block_exclusive_scan<long long>(keep ? 1ll : 0ll, s_scan, &tot);
    if (keep) {
      a.tmp_rows[out + w + ex] = r;
      a.tmp_vals[out + w + ex] = v;
    }
    w += tot;
    __syncthreads();
  }
  return w;
}

// Pre mode, a bucket above the tile: all its columns but the last hold at
// most kPreT products (the bucket rule), so they are one shared-memory tile;
// the last column goes through the dense column path.
template <class T, class S1, class S2>
__device__ void pre_oversized_bucket(BTileSmem<T>& S, PersistArgs<T, S1, S2>& a, long long s, long long m,
                                     unsigned col_base, int Wt) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const unsigned c_last = col_base + (unsigned)Wt - 1u;
  const long long mp = __ldg(&a.pre_ptr[c_last]) - s;
  long long kept_p = 0;
  if (mp > 0) {
    kept_p = pre_tile_to_tmp<T>(S, a, s, (int)mp, col_base, Wt - 1);
  } else {
    for (int l = tid; l < Wt - 1; l += nthr) a.col_kept[col_base + l] = 0u;
  }
  tt_mark(18);
  const long long kh = pre_dense_column<T>(S, a, s + mp, m - mp, s + kept_p);
  if (tid == 0) a.col_kept[c_last] = (unsigned)kh;
  __syncthreads();
}


template <class T, class S1, class S2, bool kTwo = false>
__global__ void __launch_bounds__(kSegThreads, AS_PERSIST_MINB) persist_bucket_kernel(PersistArgs<T, S1, S2> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PersistSmem<T>& SM = *reinterpret_cast<PersistSmem<T>*>(smem_raw);
  BTileSmem<T>& S = SM.t;
  __shared__ long long xscan[kSegThreads / 32 + 1];  // scan scratch outside the phase union
  unsigned gen = 0;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const long long G = gridDim.x, g = blockIdx.x;
  const long long ncb = a.n_cb;
  const unsigned long long cb_mul = a.cb_mul;
  auto bucket_of = [&](unsigned c) -> unsigned { return (unsigned)(((unsigned long long)c * cb_mul) >> 32); };
  // pre-bucketed SpGEMM products (NoSrc, NoSrc) vs construction / flush /
  // transpose: separate instantiations, each without the other's code
  constexpr bool kPre = std::is_same<S1, NoSrc<T>>::value && std::is_same<S2, NoSrc<T>>::value;
  AS_PHASE_MARK(a, 0);
  unsigned* const ha = SM.h.ab;            // histogram, then cursor
  unsigned* const hb = SM.h.ab + ncb;      // CTA range inside each bucket, then slot base
  unsigned* const hl = SM.h.ab + 2 * ncb;  // CTA-local bucket offsets (staged scatter)
  a.s1.set_cache(SM.h.colc);
  a.s2.set_cache(SM.h.colc);

  long long n_work = ncb;  // pre mode: buckets with columns (the rest are skipped)
  if constexpr (kPre) {
    // pre-bucketed input (SpGEMM products): keys / colb / vals_b already sit
    // in output-column order; only the coarse bucket starts are needed
    // variable-width buckets (kPreT): bucket t starts at the first column whose
    // cumulative weight pre_ptr[c] + kPreColCost * c reaches t * kPreT;
    // oversized buckets are queued first so the long ones start early
    auto first_col = [&](long long target) -> long long {
      long long lo = 0, hi = a.n_cols;
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (__ldg(&a.pre_ptr[mid]) + kPreColCost * mid >= target) hi = mid;
        else lo = mid + 1;
      }
      return lo;
    };
    for (long long t = g * nthr + tid; t < ncb; t += G * nthr) {
      const long long c0 = first_col(t * kPreT);
      const long long c1 = t + 1 == ncb ? a.n_cols : first_col((t + 1) * kPreT);
      const long long s0 = __ldg(&a.pre_ptr[c0]);
      a.cb_col[t] = (unsigned)c0;
      a.cb_start[t] = s0;
      if (t + 1 == ncb) {
        a.cb_col[ncb] = (unsigned)a.n_cols;
        a.cb_start[ncb] = __ldg(&a.pre_ptr[a.n_cols]);
      }
      // size class (largest first: a rough longest-processing-time order);
      // class 4 = no columns at all (targets inside one long column): never
      // handed out
      const long long mt = __ldg(&a.pre_ptr[c1]) - s0;
      const unsigned cls = c1 == c0 ? 4u : mt > 32 * kCap ? 0u : mt > 4 * kCap ? 1u : mt > kCap ? 2u : 3u;
      const unsigned peers = __match_any_sync(__activemask(), cls);  // warp-aggregated slot
      const int leader = __ffs(peers) - 1;
      unsigned slot0 = 0;
      if ((tid & 31) == leader) slot0 = atomicAdd(a.ticket + 1 + cls, (unsigned)__popc(peers));
      slot0 = __shfl_sync(peers, slot0, leader);
      a.cb_cnt[t] = (cls << 28) | (slot0 + __popc(peers & lanemask_lt()));
    }
    grid_sync(a.gb, gen);
    {
      unsigned base[5];
      base[0] = 0;
      for (int q = 1; q < 5; q++) base[q] = base[q - 1] + __ldcg(a.ticket + q);
      n_work = base[4];
      for (long long t = g * nthr + tid; t < ncb; t += G * nthr) {
        const unsigned v = __ldcg(&a.cb_cnt[t]);
        if ((v >> 28) < 4u) a.order[base[v >> 28] + (v & 0x0fffffffu)] = (unsigned)t;
      }
    }
    grid_sync(a.gb, gen);
    AS_PHASE_MARK(a, gen);
  } else {
  // ---------------- phase 1: coarse histogram + range reservation ----------------
  // bucket(c) = (c * cb_mul) >> 32: monotone, ~n_cols / n_cb columns each;
  // bucket t starts at the first column with bucket(c) >= t
  for (long long t = g * nthr + tid; t <= ncb; t += G * nthr) {
    const unsigned long long c0 = cb_mul ? (((unsigned long long)t << 32) + cb_mul - 1) / cb_mul : 0ull;
    a.cb_col[t] = (unsigned)(t == ncb ? a.n_cols : min((long long)c0, a.n_cols));
  }
  for (long long b = tid; b < ncb; b += nthr) ha[b] = 0u;
  __syncthreads();
  {
    auto inc = [&](unsigned c, unsigned, unsigned long long, long long, T) { atomicAdd(&ha[bucket_of(c)], 1u); };
    a.s1.visit(g, G, true, inc);
    a.s2.visit(g, G, true, inc);
  }
  __syncthreads();
  const int F = a.sb_f;
  const long long nsb = a.n_sb;
  if constexpr (kTwo) {
    // two-level: this CTA reserves its range inside every super-bucket (runs of
    // >= ~32 elements per CTA, so the first scatter writes whole sectors) and
    // adds its per-bucket counts to the global bucket totals
    for (long long sb = tid; sb < nsb; sb += nthr) {
      unsigned sum = 0;
      for (long long b = sb * F; b < min(ncb, sb * F + F); b++) sum += ha[b];
      hb[sb] = sum ? atomicAdd(&a.sb_cnt[sb], sum) : 0u;
    }
    for (long long b = tid; b < ncb; b += nthr) {
      const unsigned h = ha[b];
      if (h) atomicAdd(&a.cb_cnt[b], h);
    }
    __syncthreads();
    for (long long b = tid; b < ncb; b += nthr) ha[b] = 0u;  // super-bucket cursors
  } else {
    // staged scatter: the counts stay in ha for phase 2's local scan
    const bool keep = a.stage != 0;
    for (long long b = tid; b < ncb; b += nthr) {
      const unsigned h = ha[b];
      hb[b] = h ? atomicAdd(&a.cb_cnt[b], h) : 0u;
      if (!keep) ha[b] = 0u;
    }
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);

  // ---------------- phase 2: every CTA scans the bucket counts ----------------
  {
    // one scan of (this CTA's count << 32 | global count): the global bucket
    // starts and, for the staged scatter, the CTA-local bucket offsets (the
    // global total is < 2^31, so the low half never carries)
    constexpr long long kLo = 0xffffffffll;
    const bool staged = !kTwo && a.stage;
    long long running = 0;
    for (long long cb = 0; cb < ncb; cb += nthr) {
      const long long b = cb + tid;
      long long cnt = b < ncb ? (long long)__ldcg(&a.cb_cnt[b]) : 0;
      if (staged && b < ncb) {
        cnt |= (long long)ha[b] << 32;
        ha[b] = 0u;  // cursor of the scatter
      }
      long long ctot;
      const long long ex = block_exclusive_scan<long long>(cnt, xscan, &ctot);
      if (b < ncb) {
        const long long start = (running + ex) & kLo;
        if constexpr (kTwo) {
          if (b % F == 0) hb[b / F] += (unsigned)start;  // super-bucket start
        } else {
          hb[b] += (unsigned)start;  // slot base of this CTA's range
          if (staged) hl[b] = (unsigned)((running + ex) >> 32);
        }
        if (g == 0) a.cb_start[b] = start;
      }
      running += ctot;
    }
    if (g == 0 && tid == 0) a.cb_start[ncb] = running & kLo;
  }
  __syncthreads();

  // ---------------- phase 3: scatter keys, columns and values ----------------
  if constexpr (kTwo) {
    // 3a: into super-bucket order (alt arrays)
    auto put = [&](unsigned c, unsigned minor, unsigned long long idx, long long, T v) {
      const unsigned sb = bucket_of(c) / (unsigned)F;
      const unsigned slot = hb[sb] + atomicAdd(&ha[sb], 1u);
      a.keys_alt[slot] = ((unsigned long long)minor << 32) | idx;
      a.colb_alt[slot] = c;
      a.vals_alt[slot] = v;
    };
    a.s1.template visit<true>(g, G, false, put);
    a.s2.template visit<true>(g, G, false, put);
    grid_sync(a.gb, gen);
    AS_PHASE_MARK(a, gen);
    // 3b: fixed slices of the super-bucket-ordered data, each spread over its
    // (<= 2F) buckets: count, reserve one range per bucket (global fill
    // counters), scatter -- runs of ~slice/F elements, whole sectors again
    constexpr long long kSlice = 8192;
    const long long n_all = __ldcg(&a.cb_start[ncb]);
    const long long n_slices = (n_all + kSlice - 1) / kSlice;
    for (long long t = g; t < n_slices; t += G) {
      const long long lo = t * kSlice, hi = min(n_all, lo + kSlice);
      __syncthreads();
      if (tid == 0) {  // first bucket of the super-bucket holding `lo`
        long long l = 0, h = nsb - 1;
        while (l < h) {
          const long long mid = (l + h + 1) >> 1;
          if (__ldcg(&a.cb_start[mid * F]) <= lo) l = mid;
          else h = mid - 1;
        }
        S.tile = l * F;
      }
      __syncthreads();
      const long long bb = S.tile;
      const long long nbk = min(ncb - bb, 2ll * F);
      for (long long f = tid; f < nbk; f += nthr) ha[f] = 0u;
      __syncthreads();
      constexpr int kU = 8;  // loads of kU elements in flight per thread
      for (long long i0 = lo + tid; i0 < hi; i0 += (long long)kU * nthr) {
        unsigned cc[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
          const long long i = i0 + (long long)u * nthr;
          cc[u] = i < hi ? __ldcg(&a.colb_alt[i]) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kU; u++)
          if (i0 + (long long)u * nthr < hi) atomicAdd(&ha[bucket_of(cc[u]) - bb], 1u);
      }
      __syncthreads();
      for (long long f = tid; f < nbk; f += nthr) {
        const unsigned h = ha[f];
        hb[f] = h ? (unsigned)__ldcg(&a.cb_start[bb + f]) + atomicAdd(&a.sb_fill[bb + f], h) : 0u;
        ha[f] = 0u;
      }
      __syncthreads();
      for (long long i0 = lo + tid; i0 < hi; i0 += (long long)kU * nthr) {
        unsigned cc[kU];
        unsigned long long kk[kU];
        T vv[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
          const long long i = i0 + (long long)u * nthr;
          if (i < hi) {
            cc[u] = __ldcg(&a.colb_alt[i]);
            kk[u] = __ldcg(&a.keys_alt[i]);
            vv[u] = __ldcg(&a.vals_alt[i]);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
          if (i0 + (long long)u * nthr >= hi) continue;
          const unsigned f = bucket_of(cc[u]) - (unsigned)bb;
          const unsigned slot = hb[f] + atomicAdd(&ha[f], 1u);
          a.keys[slot] = kk[u];
          a.colb[slot] = cc[u];
          a.vals_b[slot] = vv[u];
        }
      }
    }
  } else if (a.stage) {
    // staged: the chunk is counting-sorted by bucket in shared memory, then
    // written run by run -- consecutive threads store consecutive slots of a
    // bucket (the scatter is bound by L2 store transactions, one per
    // scattered element and array without this)
    long long off;
    const long long cap = stage_layout<T>(ncb, &off);
    unsigned long long* st_k = reinterpret_cast<unsigned long long*>(SM.raw + off);
    T* st_v = reinterpret_cast<T*>(SM.raw + off + 8 * cap);
    unsigned* st_c = reinterpret_cast<unsigned*>(SM.raw + off + (8 + sizeof(T)) * cap);
    auto put = [&](unsigned c, unsigned minor, unsigned long long idx, long long, T v) {
      const unsigned cb = bucket_of(c);
      const unsigned q = hl[cb] + atomicAdd(&ha[cb], 1u);
      st_k[q] = ((unsigned long long)minor << 32) | idx;
      st_c[q] = c;
      st_v[q] = v;
    };
    a.s1.template visit<true>(g, G, false, put);
    a.s2.template visit<true>(g, G, false, put);
    __syncthreads();
    const unsigned total = ncb > 0 ? hl[ncb - 1] + ha[ncb - 1] : 0u;
    for (unsigned q = tid; q < total; q += nthr) {
      const unsigned c = st_c[q];
      const unsigned cb = bucket_of(c);
      const unsigned slot = hb[cb] + (q - hl[cb]);
      a.keys[slot] = st_k[q];
      a.colb[slot] = c;
      a.vals_b[slot] = st_v[q];
    }
  } else {
    a.s1.template visit<true>(g, G, false, [&](unsigned c, unsigned minor, unsigned long long idx, long long, T v) {
      const unsigned cb = bucket_of(c);
      const unsigned slot = hb[cb] + atomicAdd(&ha[cb], 1u);
      a.keys[slot] = ((unsigned long long)minor << 32) | idx;
      a.colb[slot] = c;
      a.vals_b[slot] = v;
    });
    a.s2.template visit<true>(g, G, false, [&](unsigned c, unsigned minor, unsigned long long idx, long long, T v) {
      const unsigned cb = bucket_of(c);
      const unsigned slot = hb[cb] + atomicAdd(&ha[cb], 1u);
      a.keys[slot] = ((unsigned long long)minor << 32) | idx;
      a.colb[slot] = c;
      a.vals_b[slot] = v;
    });
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  }

  // ---------------- phase 4: bucket tiles ----------------
  tt_mark(-1);
  while (true) {
    if (tid == 0) {
      long long t = (long long)atomicAdd(a.ticket, 1u);
      if (a.order) t = t < n_work ? (long long)__ldcg(&a.order[t]) : ncb;
      S.tile = t;
      if (t < ncb) {
        S.s = __ldcg(&a.cb_start[t]);
        S.m = __ldcg(&a.cb_start[t + 1]) - S.s;
        S.col_base = __ldcg(&a.cb_col[t]);
        S.wt = (int)(__ldcg(&a.cb_col[t + 1]) - S.col_base);
      }
    }
    __syncthreads();
    tt_mark(0);
    const long long t = S.tile;
    if (t >= ncb) break;
    const long long s = S.s, m = S.m;
    const unsigned col_base = (unsigned)S.col_base;
    const int Wt = S.wt;  // columns of this bucket
    // direct placement (construction / flush / transpose): the tickets hand
    // the buckets out in order, so a chained look-back over their kept counts
    // gives each bucket its output offset as soon as its own count is known
    // -- no column-scan or placement phase, no temporaries (pre mode keeps
    // them: its largest-first tile order would break the look-back chain)
    auto lookback = [&](long long kept) -> long long {
      if (tid < 32) {
        const unsigned long long pre = group_lookback_warp(a.tstate, a.tstate + ncb, t, (unsigned long long)kept);
        if (tid == 0) S.prefix = (long long)pre;
      }
      __syncthreads();
      const long long base = S.prefix;
      if (t == ncb - 1 && tid == 0) {
        a.col_ptr[a.n_cols] = (int)(base + kept);
        a.info[0] = base + kept;
      }
      return base;
    };
    if (m == 0) {
      if constexpr (kPre) {
        for (int l = tid; l < Wt; l += nthr) a.col_kept[col_base + l] = 0u;
      } else {
        const long long base = lookback(0);
        for (int l = tid; l < Wt; l += nthr) a.col_ptr[col_base + l] = (int)base;
      }
    } else if (m <= kCap) {
      {  // all loads of this thread in flight before the first store
        unsigned long long kk[kItems];
        unsigned cc[kItems];
#pragma unroll
        for (int q = 0; q < kItems; q++) {
          const int i = q * kSegThreads + tid;
          if (i < m) {
            kk[q] = __ldcg(&a.keys[s + i]);
            cc[q] = __ldcg(&a.colb[s + i]);
          }
        }
#pragma unroll
        for (int q = 0; q < kItems; q++) {
          const int i = q * kSegThreads + tid;
          if (i < m) {
            S.sk[i] = kk[q];
            S.scol[i] = (unsigned short)(cc[q] - col_base);
            S.perm[i] = (unsigned short)i;
          }
        }
      }
      __syncthreads();
      tt_mark(1);
      sort_bucket_smem(S, (int)m, Wt, a.row_bits);
      bucket_chunk_reduce<T, decltype(a.vs), kPreOnly<T, S1, S2>>(S, 0, (int)m, m, nullptr, nullptr, col_base, a.vs, a.mode, a.prune, a.vals_b + s);
      if constexpr (kPre) {
        for (int p = tid; p < m; p += nthr) {
          const unsigned e0 = S.v.excl[p], e1 = S.v.excl[p + 1];
          if (e1 != e0) {
            a.tmp_rows[s + e0] = (int)key_row(S.sk[p]);
            a.tmp_vals[s + e0] = S.u.rv[p];
          }
        }
        for (int l = tid; l < Wt; l += nthr)
          a.col_kept[col_base + l] = S.v.excl[S.cstart[l + 1]] - S.v.excl[S.cstart[l]];
      } else {
        const long long base = lookback((long long)S.v.excl[m]);
        tt_mark(10);
        for (int p = tid; p < m; p += nthr) {
          const unsigned e0 = S.v.excl[p], e1 = S.v.excl[p + 1];
          if (e1 != e0) {
            a.row_idx[base + e0] = (int)key_row(S.sk[p]);
            a.out_vals[base + e0] = S.u.rv[p];
          }
        }
        for (int l = tid; l < Wt; l += nthr) a.col_ptr[col_base + l] = (int)(base + S.v.excl[S.cstart[l]]);
      }
    } else if (kPre && a.dense_rows > 0) {
      if constexpr (kPre) pre_oversized_bucket<T>(S, a, s, m, col_base, Wt);
    } else {
      const long long kept = process_oversized_bucket<T>(S, a, s, m, col_base, Wt);
      if constexpr (!kPre) {
        const long long base = lookback(kept);
        for (long long i = tid; i < kept; i += nthr) {
          a.row_idx[base + i] = __ldcg(&a.tmp_rows[s + i]);
          a.out_vals[base + i] = __ldcg(&a.tmp_vals[s + i]);
        }
        long long running = base;  // col_ptr of the bucket's columns: scan of the kept counts
        for (int l0 = 0; l0 < Wt; l0 += nthr) {
          const int l = l0 + tid;
          long long tot;
          const long long ex = block_exclusive_scan<long long>(l < Wt ? (long long)S.ckept[l] : 0ll, xscan, &tot);
          if (l < Wt) a.col_ptr[col_base + l] = (int)(running + ex);
          running += tot;
        }
      }
    }
    __syncthreads();
    tt_mark(11);
  }
  if constexpr (!kPre) {
    AS_PHASE_MARK(a, gen + 1);
    return;
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);

  // ---------------- phase 5: column scan and placement ----------------
  long long clo, chi;
  cta_range(a.n_cols, g, G, &clo, &chi);
  {
    long long sum = 0;
    for (long long c = clo + tid; c < chi; c += nthr) sum += __ldcg(&a.col_kept[c]);
    sum = block_reduce_sum<long long>(sum, xscan);
    if (tid == 0) a.cta_sums[g] = sum;
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  {
    long long pre = 0;
    for (long long q = tid; q < g; q += nthr) pre += __ldcg(&a.cta_sums[q]);
    pre = block_reduce_sum<long long>(pre, xscan);
    long long running = pre;
    for (long long cb = clo; cb < chi; cb += nthr) {
      const long long c = cb + tid;
      const long long k = c < chi ? (long long)__ldcg(&a.col_kept[c]) : 0;
      long long ctot;
      const long long ex = block_exclusive_scan<long long>(k, xscan, &ctot);
      if (c < chi) a.col_ptr[c] = (int)(running + ex);
      running += ctot;
    }
    if (g == G - 1 && tid == 0) {
      a.col_ptr[a.n_cols] = (int)running;
      a.info[0] = running;
    }
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  {
    // placement by equal output ranges (a heavy bucket is spread over many
    // CTAs): bucket t's kept entries sit at tmp[cb_start[t] ...] and go to
    // col_ptr[first column of t]; the bucket table of a range is staged in
    // shared memory nthr buckets at a time
    auto dst_of = [&](long long t) -> long long {
      const long long c = t >= ncb ? a.n_cols : (long long)__ldcg(&a.cb_col[t]);
      return __ldcg(&a.col_ptr[c]);
    };
    long long* sd = reinterpret_cast<long long*>(&S.u);  // [nthr + 1] bucket output starts
    long long* ss = sd + (kSegThreads + 1);              // [nthr] bucket tmp starts
    long long o0, o1;
    cta_range(__ldcg(&a.col_ptr[a.n_cols]), g, G, &o0, &o1);
    if (tid == 0) {
      long long lo = 0, hi = ncb - 1;  // last t with dst(t) <= o0
      while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (dst_of(mid) <= o0) lo = mid;
        else hi = mid - 1;
      }
      S.tile = lo;
    }
    __syncthreads();
    long long tb = S.tile;
    while (o0 < o1 && tb < ncb) {
      const int nb = (int)min((long long)nthr, ncb - tb);
      __syncthreads();
      for (int i = tid; i <= nb; i += nthr) {
        sd[i] = dst_of(tb + i);
        if (i < nb) ss[i] = __ldcg(&a.cb_start[tb + i]);
      }
      __syncthreads();
      const long long e = min(o1, sd[nb]);
      int k = 0;  // bucket of this thread's next position: one search, then a forward walk
      {
        const long long o = o0 + tid;
        int hi = nb - 1;
        while (k < hi) {
          const int mid = (k + hi + 1) >> 1;
          if (sd[mid] <= o) k = mid;
          else hi = mid - 1;
        }
      }
      constexpr int kU = 4;
      for (long long ob = o0 + tid; ob < e; ob += (long long)kU * nthr) {
        long long src[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
          const long long o = ob + (long long)u * nthr;
          src[u] = -1;
          if (o < e) {
            while (sd[k + 1] <= o) k++;
            src[u] = ss[k] + (o - sd[k]);
          }
        }
        int rr[kU];
        T vv[kU];
#pragma unroll
        for (int u = 0; u < kU; u++)
          if (src[u] >= 0) {
            rr[u] = __ldcg(&a.tmp_rows[src[u]]);
            vv[u] = __ldcg(&a.tmp_vals[src[u]]);
          }
#pragma unroll
        for (int u = 0; u < kU; u++)
          if (src[u] >= 0) {
            a.row_idx[ob + (long long)u * nthr] = rr[u];
            a.out_vals[ob + (long long)u * nthr] = vv[u];
          }
      }
      o0 = max(o0, e);
      tb += nb;
    }
  }
  __syncthreads();
  AS_PHASE_MARK(a, gen + 1);
}

}  // namespace as
