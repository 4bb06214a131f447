// persist.cuh -- one persistent, cooperatively launched kernel per
// bucket-sort-reduce operation (COO->CSC construction, insertion-log flush,
// CSC transpose).
//
// At the sizes of the BASELINE configs (1e5-1e7 elements) a pipeline of
// separate kernels is latency bound: every kernel boundary drains the GPU,
// and per-element global atomics on ~1e4 buckets serialise in L2 (measured
// on B200: 1M RED.ADD over 10k bins take ~24 us, tools/micro/atomic_micro.cu).
// Here the whole operation is one launch of exactly the co-resident grid
// (148 SMs x blocks/SM), phases separated by a grid barrier:
//
//   1 histogram   P1 chunks of the input, each counted in a shared-memory
//                 histogram, written as one row of partials[P1][n_bins]
//                 (no per-element global atomics); falls back to global
//                 atomics when n_bins exceeds the shared-memory histogram
//   2 scan        grid-wide exclusive scan of the bucket totals -> seg_ptr;
//                 partials rewritten in place as per-(chunk, bucket) bases;
//                 the tile -> segment map for phase 4
//   3 scatter     each chunk re-read; slot = shared-memory cursor; the key
//                 (minor << 32 | input index) and the VALUE move to the slot,
//                 so the tile phase reads values contiguously from L2
//   4 tiles       the segmented sort / run-reduce engine (segsort.cuh) on
//                 claimed tiles, compacted output into temporaries at the
//                 tile's own offset, tile totals recorded (no look-back chain)
//   5 place       grid-wide scan of tile totals; each tile copied to its final
//                 offset and its col_ptr entries shifted by the tile prefix
#pragma once

#include "segsort.cuh"

namespace as {

#define AS_PHASE_MARK(a, gen)                                                       \
  do {                                                                              \
    if ((a).phase_ts && blockIdx.x == 0 && threadIdx.x == 0) (a).phase_ts[gen] = global_ns(); \
  } while (0)

// ------------------------------------------------------------------------
// element sources: visit(p, P, f) calls f(bucket, minor, idx, i) for every
// valid element of chunk p of P (the same partition every time it is called)

constexpr int kVisitVec = 4;  // consecutive elements per thread (ILP)

template <class IdxT>
AS_DEVICE_INLINE void load_vec4(const IdxT* p, long long i, long long hi, long long* out) {
  if (i + 3 < hi && sizeof(IdxT) == 4 && ((i & 3) == 0)) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(p + i));
    out[0] = q.x;
    out[1] = q.y;
    out[2] = q.z;
    out[3] = q.w;
  } else if (i + 3 < hi && sizeof(IdxT) == 8 && ((i & 1) == 0)) {
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

template <class IdxT, class T>
struct CooSrc {
  const IdxT* rows;
  const IdxT* cols;
  const T* vals;
  long long n;
  long long n_rows, n_cols;
  unsigned long long idx_off;
  long long* bad;  // first invalid triplet (reported in phase 1)

  // chunk p of P: elements [p*ch, min(n, (p+1)*ch)), ch a multiple of 4;
  // each thread takes 4 consecutive elements per step (vector loads).
  template <class F>
  __device__ void visit(long long p, long long P, bool report, F f) const {
    const long long ch = (((n + P - 1) / P) + 3) & ~3ll;
    const long long lo = min(n, p * ch), hi = min(n, lo + ch);
    for (long long i = lo + (long long)threadIdx.x * kVisitVec; i < hi; i += (long long)blockDim.x * kVisitVec) {
      long long r[4], c[4];
      load_vec4(rows, i, hi, r);
      load_vec4(cols, i, hi, c);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const long long e = i + k;
        if (e >= hi) break;
        if (r[k] < 0 || r[k] >= n_rows || c[k] < 0 || c[k] >= n_cols) {
          if (report && bad) atomicMin((unsigned long long*)bad, (unsigned long long)e);
          continue;
        }
        f((unsigned)c[k], (unsigned)r[k], (unsigned long long)e + idx_off, e);
      }
    }
  }
  AS_DEVICE_INLINE T value(long long i) const { return vals[i]; }
  __host__ __device__ long long size() const { return n; }
  AS_DEVICE_INLINE void set_cache(int*) {}
};

// The elements of a CSC: by_row = false -> bucket col, minor row (flush
// base); by_row = true -> bucket row, minor col (transpose).  Chunk p is the
// element range [p*ch, (p+1)*ch); the columns it touches are staged in
// shared memory (colc) when they fit, and each thread finds the column of
// its 4 consecutive elements by binary search there (or in global memory).
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
  int* colc;  // shared-memory column-start cache (kColCache + 1 entries), set by the kernel

  template <class F>
  __device__ void visit(long long p, long long P, bool report, F f) const {
    (void)report;
    __shared__ long long s_cb, s_ce;
    if (nnz == 0) return;
    const long long ch = (((nnz + P - 1) / P) + 3) & ~3ll;
    const long long lo = min(nnz, p * ch), hi = min(nnz, lo + ch);
    __syncthreads();
    if (threadIdx.x == 0 && lo < hi) {
      s_cb = upper_bound_dev(col_ptr, n_cols + 1, (int)lo) - 1;      // column holding lo
      s_ce = upper_bound_dev(col_ptr, n_cols + 1, (int)(hi - 1));    // one past the column holding hi-1
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
        int l = 0, h = (int)(ce - cb);  // last q with colc[q] <= i
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
      load_vec4(row_idx, i, hi, r);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const long long e = i + k;
        if (e >= hi) break;
        while ((cached ? colc[c + 1 - cb] : col_ptr[c + 1]) <= e) c++;
        if (by_row) f((unsigned)r[k], (unsigned)c, (unsigned long long)e + idx_off, e);
        else f((unsigned)c, (unsigned)r[k], (unsigned long long)e + idx_off, e);
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
  template <class F>
  __device__ void visit(long long, long long, bool, F) const {}
  AS_DEVICE_INLINE T value(long long) const { return T(0); }
  __host__ __device__ long long size() const { return 0; }
  AS_DEVICE_INLINE void set_cache(int*) {}
};

constexpr int kHistMaxBins = 11264;  // shared-memory histogram capacity (44 KB)

template <class T, class S1, class S2>
struct PersistArgs {
  S1 s1;
  S2 s2;
  long long n_bins;
  long long n_upper;  // s1.size() + s2.size()
  long long P1;       // histogram chunks (smem path)
  int smem_hist;
  unsigned* partials;  // [P1][n_bins]
  unsigned* counts;    // [n_bins] (atomic path, zeroed)
  unsigned* range_sum; // [n_pr_max][n_bins] (smem path)
  long long n_pr_max;
  long long* cta_sums; // [2 * grid]
  long long* seg_ptr;  // [n_bins + 1]
  long long* tile_c0;  // [n_tiles + 1]
  long long n_tiles;
  long long* tile_total;  // [n_tiles]
  unsigned long long* keys;
  unsigned long long* keys_alt;
  T* vals_b;            // bucketed values (by slot)
  int* tmp_rows;
  T* tmp_vals;
  int row_bits, idx_bits;
  int mode, prune;
  ValSrc<T> vs;         // values by input index (oversized tiles)
  int* col_ptr;
  int* row_idx;
  T* out_vals;
  long long* info;
  unsigned* ticket;
  GridBar gb;
  unsigned long long* phase_ts;  // optional: globaltimer after each phase (debug)
};

template <class T>
union PersistSmem {
  struct {
    unsigned hist[kHistMaxBins];
    int colc[kColCache + 1];
  } h;
  SegSmem<T> seg;
};

// grid-wide exclusive scan helper: CTA g owns items [g*per, min(n, (g+1)*per))
AS_DEVICE_INLINE void cta_range(long long n, long long g, long long G, long long* lo, long long* hi) {
  const long long per = (n + G - 1) / G;
  *lo = min(n, g * per);
  *hi = min(n, *lo + per);
}

template <class T, class S1, class S2>
__global__ void __launch_bounds__(kSegThreads, 3) persist_bucket_kernel(PersistArgs<T, S1, S2> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PersistSmem<T>& SM = *reinterpret_cast<PersistSmem<T>*>(smem_raw);
  SegSmem<T>& S = SM.seg;
  unsigned gen = 0;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const long long G = gridDim.x, g = blockIdx.x;
  const long long nb = a.n_bins;
  AS_PHASE_MARK(a, 0);
  a.s1.set_cache(SM.h.colc);
  a.s2.set_cache(SM.h.colc);

  // ---------------- phase 1: histogram ----------------
  if (a.smem_hist) {
    for (long long p = g; p < a.P1; p += G) {
      for (long long b = tid; b < nb; b += nthr) SM.h.hist[b] = 0u;
      __syncthreads();
      auto inc = [&](unsigned b, unsigned, unsigned long long, long long) { atomicAdd(&SM.h.hist[b], 1u); };
      a.s1.visit(p, a.P1, true, inc);
      a.s2.visit(p, a.P1, true, inc);
      __syncthreads();
      unsigned* row = a.partials + p * nb;
      for (long long b = tid; b < nb; b += nthr) row[b] = SM.h.hist[b];
      __syncthreads();
    }
  } else {
    auto inc = [&](unsigned b, unsigned, unsigned long long, long long) { atomicAdd(&a.counts[b], 1u); };
    a.s1.visit(g, G, true, inc);
    a.s2.visit(g, G, true, inc);
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);

  // ---------------- phase 2: bucket scan ----------------
  // Smem-histogram path: the partials matrix [P1][nb] is walked in
  // (256-bucket block) x (range of chunks) work items so every access is
  // coalesced: 2a range sums, 2b bucket totals + grid-wide scan -> seg_ptr,
  // 2c per-(chunk, bucket) bases written back into partials.
  const long long n_bc = (nb + nthr - 1) / nthr;
  const long long n_pr = a.smem_hist ? max(1ll, min(a.n_pr_max, G / max(1ll, n_bc))) : 1;
  const long long pr_len = (a.P1 + n_pr - 1) / n_pr;
  if (a.smem_hist) {
    for (long long w = g; w < n_bc * n_pr; w += G) {
      const long long bc = w % n_bc, pr = w / n_bc;
      const long long b = bc * nthr + tid;
      if (b < nb) {
        const long long p0 = pr * pr_len, p1 = min(a.P1, p0 + pr_len);
        unsigned sacc = 0;
#pragma unroll 4
        for (long long p = p0; p < p1; p++) sacc += a.partials[p * nb + b];
        a.range_sum[pr * nb + b] = sacc;
      }
    }
    grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  }
  long long blo, bhi;
  cta_range(nb, g, G, &blo, &bhi);
  {
    long long running = 0;
    for (long long cb = blo; cb < bhi; cb += nthr) {
      const long long b = cb + tid;
      long long tot = 0;
      if (b < bhi) {
        if (a.smem_hist) {
          for (long long pr = 0; pr < n_pr; pr++) tot += a.range_sum[pr * nb + b];
        } else {
          tot = a.counts[b];
        }
      }
      long long ctot;
      const long long ex = block_exclusive_scan<long long>(tot, S.scan_tmp, &ctot);
      if (b < bhi) a.seg_ptr[b] = running + ex;  // CTA-local for now
      running += ctot;
    }
    if (tid == 0) a.cta_sums[g] = running;
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  {
    long long pre = 0;
    for (long long q = tid; q < g; q += nthr) pre += a.cta_sums[q];
    pre = block_reduce_sum<long long>(pre, S.scan_tmp);
    for (long long b = blo + tid; b < bhi; b += nthr) {
      const long long start = pre + a.seg_ptr[b];
      a.seg_ptr[b] = start;
      long long tot;
      if (a.smem_hist) {
        tot = 0;
        for (long long pr = 0; pr < n_pr; pr++) tot += a.range_sum[pr * nb + b];
      } else {
        tot = a.counts[b];
        a.counts[b] = 0u;
      }
      emit_tile_bounds(b, start, start + tot, a.n_tiles, a.tile_c0);
    }
    if (g == G - 1 && tid == 0) {
      long long total = pre + a.cta_sums[g];
      a.seg_ptr[nb] = total;
      finish_tile_bounds(nb, total, a.n_tiles, a.tile_c0);
    }
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  if (a.smem_hist) {
    for (long long w = g; w < n_bc * n_pr; w += G) {
      const long long bc = w % n_bc, pr = w / n_bc;
      const long long b = bc * nthr + tid;
      if (b < nb) {
        long long run = a.seg_ptr[b];
        for (long long q = 0; q < pr; q++) run += a.range_sum[q * nb + b];
        const long long p0 = pr * pr_len, p1 = min(a.P1, p0 + pr_len);
        for (long long p = p0; p < p1; p++) {
          const unsigned c = a.partials[p * nb + b];
          a.partials[p * nb + b] = (unsigned)run;
          run += c;
        }
      }
    }
    grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  }

  // ---------------- phase 3: scatter keys and values ----------------
  if (a.smem_hist) {
    for (long long p = g; p < a.P1; p += G) {
      const unsigned* row = a.partials + p * nb;
      for (long long b = tid; b < nb; b += nthr) SM.h.hist[b] = row[b];
      __syncthreads();
      a.s1.visit(p, a.P1, false, [&](unsigned b, unsigned minor, unsigned long long idx, long long i) {
        const unsigned slot = atomicAdd(&SM.h.hist[b], 1u);
        a.keys[slot] = ((unsigned long long)minor << 32) | idx;
        a.vals_b[slot] = a.s1.value(i);
      });
      a.s2.visit(p, a.P1, false, [&](unsigned b, unsigned minor, unsigned long long idx, long long i) {
        const unsigned slot = atomicAdd(&SM.h.hist[b], 1u);
        a.keys[slot] = ((unsigned long long)minor << 32) | idx;
        a.vals_b[slot] = a.s2.value(i);
      });
      __syncthreads();
    }
  } else {
    a.s1.visit(g, G, false, [&](unsigned b, unsigned minor, unsigned long long idx, long long i) {
      const long long slot = a.seg_ptr[b] + atomicAdd(&a.counts[b], 1u);
      a.keys[slot] = ((unsigned long long)minor << 32) | idx;
      a.vals_b[slot] = a.s1.value(i);
    });
    a.s2.visit(g, G, false, [&](unsigned b, unsigned minor, unsigned long long idx, long long i) {
      const long long slot = a.seg_ptr[b] + atomicAdd(&a.counts[b], 1u);
      a.keys[slot] = ((unsigned long long)minor << 32) | idx;
      a.vals_b[slot] = a.s2.value(i);
    });
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);

  // ---------------- phase 4: tiles -> temporaries ----------------
  SegIn in{a.seg_ptr, nb, a.n_upper, a.keys, a.keys_alt, a.row_bits, a.idx_bits, 0, a.tile_c0};
  SegOut<T> out{a.col_ptr, a.tmp_rows, a.tmp_vals, a.info, nullptr, a.ticket};
  while (true) {
    if (tid == 0) S.tile = (long long)atomicAdd(a.ticket, 1u);
    __syncthreads();
    const long long t = S.tile;
    __syncthreads();
    if (t >= a.n_tiles) break;
    process_tile<true, T>(S, in, a.vs, a.mode, a.prune, out, t, a.n_tiles, a.vals_b, a.tile_total);
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);

  // ---------------- phase 5: tile prefixes, placement ----------------
  long long tlo, thi;
  cta_range(a.n_tiles, g, G, &tlo, &thi);
  {
    long long s = 0;
    for (long long t = tlo + tid; t < thi; t += nthr) s += a.tile_total[t];
    s = block_reduce_sum<long long>(s, S.scan_tmp);
    if (tid == 0) a.cta_sums[G + g] = s;
  }
  grid_sync(a.gb, gen);
  AS_PHASE_MARK(a, gen);
  {
    long long pre = 0;
    for (long long q = tid; q < g; q += nthr) pre += a.cta_sums[G + q];
    pre = block_reduce_sum<long long>(pre, S.scan_tmp);
    for (long long t = tlo; t < thi; t++) {  // block-uniform
      const long long c0 = a.tile_c0[t], c1 = a.tile_c0[t + 1];
      const long long e0 = a.seg_ptr[c0];
      const long long cnt = a.tile_total[t];
      for (long long i = tid; i < cnt; i += nthr) {
        a.row_idx[pre + i] = a.tmp_rows[e0 + i];
        a.out_vals[pre + i] = a.tmp_vals[e0 + i];
      }
      for (long long c = c0 + tid; c < c1; c += nthr) a.col_ptr[c] += (int)pre;
      pre += cnt;
    }
    if (g == G - 1 && tid == 0) {
      a.col_ptr[nb] = (int)pre;
      a.info[0] = pre;
    }
  }
  __syncthreads();
  AS_PHASE_MARK(a, gen + 1);
}

}  // namespace as
