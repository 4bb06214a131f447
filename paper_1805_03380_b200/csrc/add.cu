// add.cu -- alpha*A + beta*B of two canonical CSC matrices.
//
// Replaces _kernels.linear_combine (_kernels.py:12-48) via ops._combine /
// add / subtract / scaled_sum (ops.py:50-73).  Per column a two-pointer row
// merge; coincident rows give alpha*a + beta*b (product and sum separately
// rounded, as numba evaluates it: no FMA), others alpha*a or beta*b; exact
// zeros are pruned.
//
// B200 design: a canonical CSC is sorted by the composite key (column, row),
// so the whole add is ONE merge of two sorted sequences (A wins ties; a
// coincident pair occupies two merged positions, the A one emits the sum and
// the B one emits nothing).  Merged positions are cut into tiles of kAddTile:
//  1. add_partition_kernel, one thread per column: every tile boundary that
//     falls inside the column gets its merge-path split (global A / B element
//     index; a warp-cooperative 32-probe search), the column holding it and a flag telling whether the tile's
//     first B element pairs with the A element just before the tile; the
//     column holding each tile's last position is recorded too;
//  2. add_tile_kernel, persistent CTAs taking tiles in ticket order: the tile's A and B
//     ranges are contiguous in the inputs, loaded coalesced into shared
//     memory; each element's column comes from a block max-scan of the
//     column starts, giving 64-bit composite keys; each thread merge-path
//     splits its kAddItems positions in shared memory and merges them; a
//     block scan of kept counts and a single-pass decoupled look-back give
//     the output offset; rows / values go out through shared memory
//     (coalesced) and the tile writes col_ptr of the columns whose merged
//     start lies in it.
// One pass over the data, no grid barrier, no re-merge.
#include "capi_util.cuh"
#include "common.cuh"

namespace as {

#ifndef AS_ADD_THREADS
#define AS_ADD_THREADS 256
#endif
#ifndef AS_ADD_ITEMS
#define AS_ADD_ITEMS 8
#endif
#ifndef AS_ADD_MINB
#define AS_ADD_MINB 4
#endif
constexpr int kAddThreads = AS_ADD_THREADS;
constexpr int kAddItems = AS_ADD_ITEMS;
constexpr int kAddTile = kAddThreads * kAddItems;
constexpr int kAddPartThreads = 256;

struct AddDesc {
  int ia;    // first A element of the tile
  int jb;    // first B element of the tile
  int skip;  // B[jb] coincides with A[ia - 1] (its sum was emitted by the previous tile)
  int col;   // column holding the tile's first merged position
};

// One thread per column: tile boundaries inside it.
__global__ void __launch_bounds__(kAddPartThreads)
add_partition_kernel(long long n_cols, long long nnz_a, long long nnz_b, long long n_tiles, const int* __restrict__ ap,
                     const int* __restrict__ ar, const int* __restrict__ bp, const int* __restrict__ br,
                     AddDesc* __restrict__ desc, int* __restrict__ cend, unsigned long long* __restrict__ states,
                     unsigned long long* __restrict__ ticket) {
  // the tile kernel may launch now (programmatic dependent launch); it waits
  // for this grid's writes at griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gsz = (long long)gridDim.x * blockDim.x;
  for (long long q = g; q < n_tiles; q += gsz) states[q] = 0ull;
  const long long M = nnz_a + nnz_b;
  if (g == 0) {
    *ticket = 0ull;
    desc[n_tiles] = AddDesc{(int)nnz_a, (int)nnz_b, 0, (int)n_cols};
  }
  const bool valid = g < n_cols;
  long long a0 = 0, a1 = 0, b0 = 0, b1 = 0;
  if (valid) {
    a0 = __ldg(&ap[g]);
    a1 = __ldg(&ap[g + 1]);
    b0 = __ldg(&bp[g]);
    b1 = __ldg(&bp[g + 1]);
  }
  const long long ms0 = a0 + b0, ms1 = a1 + b1;
  if (valid && ms0 < ms1)
    for (long long t = ms0 / kAddTile; t * kAddTile < ms1; t++) {
      const long long e = min((t + 1) * kAddTile, M) - 1;  // the tile's last merged position
      if (e >= ms0 && e < ms1) cend[t] = (int)g;
    }
  // Tile starts inside this thread's column, split warp-cooperatively: the
  // warp takes the pending boundaries one at a time and locates the first
  // i with A[i] > B[dl - i - 1] (A wins ties) with 32 probes per round trip
  // (a 4096-entry range resolves in 3 rounds).
  const int lane = threadIdx.x & 31;
  long long tb = (ms0 + kAddTile - 1) / kAddTile;
  bool pending = valid && ms0 < ms1 && tb * kAddTile < ms1;
  while (true) {
    const unsigned m = __ballot_sync(0xffffffffu, pending);
    if (!m) break;
    const int leader = __ffs(m) - 1;
    const long long ca0 = __shfl_sync(0xffffffffu, a0, leader), cb0 = __shfl_sync(0xffffffffu, b0, leader);
    const long long la = __shfl_sync(0xffffffffu, a1, leader) - ca0, lb = __shfl_sync(0xffffffffu, b1, leader) - cb0;
    const long long t = __shfl_sync(0xffffffffu, tb, leader);
    const long long dl = t * kAddTile - (ca0 + cb0);
    long long lo = max(0ll, dl - lb), hi = min(dl, la);
    while (lo < hi) {
      const long long w = hi - lo;
      const long long pq = w <= 32 ? lo + lane : lo + w * (lane + 1) / 33;
      const bool le = pq < hi && __ldg(&ar[ca0 + pq]) <= __ldg(&br[cb0 + dl - pq - 1]);
      const int cnt = __popc(__ballot_sync(0xffffffffu, le));  // a prefix of the probes
      if (w <= 32) {
        lo = lo + cnt;
        break;
      }
      const long long nlo = cnt ? lo + w * cnt / 33 + 1 : lo;
      hi = cnt < 32 ? lo + w * (cnt + 1) / 33 : hi;
      lo = nlo;
    }
    if (lane == leader) {
      const long long i = lo, j = dl - lo;
      AddDesc d;
      d.ia = (int)(ca0 + i);
      d.jb = (int)(cb0 + j);
      d.skip = (i > 0 && j < lb && __ldg(&ar[ca0 + i - 1]) == __ldg(&br[cb0 + j])) ? 1 : 0;
      d.col = (int)g;
      desc[t] = d;
      tb++;
      pending = tb * kAddTile < ms1;
    }
  }
}

// Per-thread blocks of kAddItems consecutive elements would put a warp's
// accesses kAddItems words apart (4- to 16-way bank conflicts); every array
// indexed by element / position is padded by one slot per 8: pad(e).
AS_DEVICE_INLINE int pad(int e) { return e + (e >> 3); }
constexpr int kAddPadded = kAddTile + kAddTile / 8 + 1;

struct AddSmem {
  union {
    unsigned long long key[kAddPadded];  // A range keys [0, na), B range keys [na, n)
    struct {                             // after the merge (the keys are dead):
      int orow[kAddPadded];              //   the tile's kept rows
      unsigned excl[kAddPadded];         //   kept outputs before each merged position
    };
  };
  union {
    double val[kAddPadded];
    double oval[kAddPadded];  // after the merge: the tile's kept values
  };
  // column starts (B: | 0x80000000).  Zero between tiles: written only below n
  // in step 1 and re-zeroed by the max-scan that reads them, so nothing else
  // may share this storage (a persistent CTA's next tile would read leftovers).
  unsigned mark[kAddPadded];
  int cms[kAddTile];  // merged start of column c_first + k, relative to the tile
  unsigned scan_u[kAddThreads / 32 + 1];
  int scan_i[kAddThreads / 32 + 1];
  long long prefix;
  long long tile;
};

struct AddArgs {
  long long n_cols, M, n_tiles;
  double alpha, beta;
  const int *ap, *ar, *bp, *br;
  const double *av, *bv;
  int* out_ptr;
  int* out_rows;
  double* out_vals;
  long long* info;
  const AddDesc* desc;
  const int* cend;
  unsigned long long* states;
  unsigned long long* ticket;
};

// Exclusive prefix of tile t whose aggregate is already published (the
// look-back half of tile_lookback_warp); one full warp; publishes t's
// inclusive prefix.
__device__ unsigned long long add_lookback_wait(unsigned long long* states, long long t, unsigned long long aggregate) {
  const int lane = threadIdx.x & 31;
  if (t == 0) return 0ull;
  unsigned long long prefix = 0;
  long long base = t - 1;
  while (true) {
    const long long i = base - lane;
    unsigned long long s = kFlagInc;  // virtual inclusive 0 before tile 0
    if (i >= 0) {
      do {
        s = tile_peek(&states[i]);
      } while ((s & 3ull) == 0ull);
    }
    const unsigned inc_mask = __ballot_sync(0xffffffffu, (s & 3ull) == kFlagInc);
    const int first = inc_mask ? (__ffs(inc_mask) - 1) : 32;
    prefix += warp_reduce_sum((lane <= first) ? (s >> 2) : 0ull);
    if (inc_mask) break;
    base -= 32;
  }
  // no fence: the state words carry only counts, nothing else is published
  if (lane == 0) atomicExch(&states[t], ((prefix + aggregate) << 2) | kFlagInc);
  return prefix;
}

// A tile's inputs, loaded into registers ahead of its turn: descriptors,
// kAddItems rows per thread (element tid + u * kAddThreads) and the column
// pointers of column c_first + tid.  (The values go straight to shared
// memory with cp.async when the tile starts: they are first needed by the
// merge, two barriers later.)
struct AddPrefetch {
  AddDesc d0, d1;
  int c_last, own_lo;
  unsigned rr[kAddItems];
  int as_, ae, bs, be;
};

__device__ __forceinline__ void add_prefetch(const AddArgs& a, long long t, AddPrefetch& P) {
  const int tid = threadIdx.x;
  P.d0 = a.desc[t];
  P.d1 = a.desc[t + 1];
  P.c_last = __ldg(&a.cend[t]);
  P.own_lo = t == 0 ? 0 : __ldg(&a.cend[t - 1]) + 1;
  const int ia0 = P.d0.ia, jb0 = P.d0.jb, na = P.d1.ia - ia0, n = na + P.d1.jb - jb0;
#pragma unroll
  for (int u = 0; u < kAddItems; u++) {
    const int e = tid + u * kAddThreads;
    const bool isa = e < na;
    const int* rp = isa ? a.ar + ia0 + e : a.br + jb0 + (e - na);
    P.rr[u] = e < n ? (unsigned)__ldg(rp) : 0u;
  }
  const long long c = (long long)P.d0.col + tid;
  if (c <= P.c_last) {
    P.as_ = __ldg(&a.ap[c]);
    P.ae = __ldg(&a.ap[c + 1]);
    P.bs = __ldg(&a.bp[c]);
    P.be = __ldg(&a.bp[c + 1]);
  }
}

// Persistent: each CTA takes tiles by ticket until none is left.  The next
// tile's ticket is taken when this tile starts, and its inputs are in flight
// while this tile looks back and writes.
__global__ void __launch_bounds__(kAddThreads, AS_ADD_MINB) add_tile_kernel(AddArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AddSmem& S = *reinterpret_cast<AddSmem*>(smem_raw);
  const int tid = threadIdx.x;
  for (int e = tid; e < kAddPadded; e += kAddThreads) S.mark[e] = 0u;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the partition kernel's writes
  if (tid == 0) S.tile = (long long)atomicAdd(a.ticket, 1ull);
  __syncthreads();
  long long t = S.tile;
  AddPrefetch P;
  if (t < a.n_tiles) add_prefetch(a, t, P);
  __syncthreads();  // S.tile is rewritten at the start of the first tile
  while (t < a.n_tiles) {
    const AddDesc d0 = P.d0, d1 = P.d1;
    const long long c_first = d0.col, c_last = P.c_last, own_lo = P.own_lo;
    const int ia0 = d0.ia, jb0 = d0.jb;
    const int na = d1.ia - ia0, nb = d1.jb - jb0, n = na + nb;
    const long long tpos = t * kAddTile;
    const long long span = c_last - c_first + 1;
    // the next ticket is claimed now (read behind this tile's first barrier), so its loads
    // can be issued as soon as the merge's registers are free -- no barrier in between
    if (tid == 0) S.tile = (long long)atomicAdd(a.ticket, 1ull);

    // 1. rows, values and the column starts of the tile's A and B ranges
#pragma unroll
    for (int u = 0; u < kAddItems; u++) {
      const int e = tid + u * kAddThreads;
      if (e < n) {
        S.key[pad(e)] = P.rr[u];
        const double* vp = e < na ? a.av + ia0 + e : a.bv + jb0 + (e - na);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&S.val[pad(e)]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(vp) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (long long k = tid; k < span; k += kAddThreads) {
      const long long c = c_first + k;
      int as_, ae, bs, be;
      if (k == tid) {
        as_ = P.as_;
        ae = P.ae;
        bs = P.bs;
        be = P.be;
      } else {  // tiles spanning more than kAddThreads columns
        as_ = __ldg(&a.ap[c]);
        ae = __ldg(&a.ap[c + 1]);
        bs = __ldg(&a.bp[c]);
        be = __ldg(&a.bp[c + 1]);
      }
      if (as_ < ae && ae > ia0 && as_ < ia0 + na) S.mark[pad(max(as_, ia0) - ia0)] = (unsigned)c;
      if (bs < be && be > jb0 && bs < jb0 + nb) S.mark[pad(na + max(bs, jb0) - jb0)] = (unsigned)c | 0x80000000u;
      if (span <= kAddTile) S.cms[k] = (int)((long long)as_ + bs - tpos);
    }
    __syncthreads();
    const long long tn = S.tile;
    {  // columns: inclusive max-scan of the marks (B's marks dominate A's); marks re-zeroed
      const int e0 = tid * kAddItems;
      unsigned m[kAddItems];
      unsigned run = 0u;
#pragma unroll
      for (int u = 0; u < kAddItems; u++) {
        m[u] = e0 + u < n ? S.mark[pad(e0 + u)] : 0u;
        if (e0 + u < n) S.mark[pad(e0 + u)] = 0u;
        run = max(run, m[u]);
      }
      unsigned ex = block_exclusive_max(run, S.scan_u);
#pragma unroll
      for (int u = 0; u < kAddItems; u++) {
        ex = max(ex, m[u]);
        if (e0 + u < n) S.key[pad(e0 + u)] |= (unsigned long long)(ex & 0x7fffffffu) << 32;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's values landed
    __syncthreads();

    // 2. merge kAddItems positions per thread
    auto kA = [&](int x) { return S.key[pad(x)]; };
    auto kB = [&](int x) { return S.key[pad(na + x)]; };
    auto vA = [&](int x) { return S.val[pad(x)]; };
    auto vB = [&](int x) { return S.val[pad(na + x)]; };
    const int p0 = tid * kAddItems;
    int i = 0, j = 0;
    if (p0 < n) {
      int lo = max(0, p0 - nb), hi = min(p0, na);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (kA(mid) <= kB(p0 - mid - 1)) lo = mid + 1;
        else hi = mid;
      }
      i = lo;
      j = p0 - lo;
    }
    // walk with the current A / B keys in registers (~0 = exhausted) and the
    // key of the A element consumed last (a B element equal to it was summed
    // into it and emits nothing)
    constexpr unsigned long long kNone = ~0ull;
    unsigned long long ka = i < na ? kA(i) : kNone, kb = j < nb ? kB(j) : kNone;
    unsigned long long last_a = i > 0 ? kA(i - 1) : (j == 0 && d0.skip ? kb : kNone);
    int orow[kAddItems];
    double oval[kAddItems];
    unsigned keep = 0u;
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < kAddItems; u++) {
      if (p0 + u < n) {
        bool emit = true;
        double v;
        if (ka <= kb) {
          const double av = vA(i);
          if (ka == kb || (kb == kNone && i == na - 1 && d1.skip)) {
            const double bv = kb != kNone ? vB(j) : __ldg(&a.bv[d1.jb]);
            v = __dadd_rn(__dmul_rn(a.alpha, av), __dmul_rn(a.beta, bv));
          } else {
            v = __dmul_rn(a.alpha, av);
          }
          orow[u] = (int)(unsigned)ka;
          last_a = ka;
          i++;
          ka = i < na ? kA(i) : kNone;
        } else {
          emit = kb != last_a;
          v = __dmul_rn(a.beta, vB(j));
          orow[u] = (int)(unsigned)kb;
          j++;
          kb = j < nb ? kB(j) : kNone;
        }
        oval[u] = v;
        if (emit && v != 0.0) {
          keep |= 1u << u;
          cnt++;
        }
      }
    }
    int total;
    const int off = block_exclusive_scan<int>(cnt, S.scan_i, &total);  // (its barriers end every merge)
    // 3a. the count is known: publish it and take the next ticket before staging the
    //     outputs, so the successors' look-backs find it that much earlier
    if (tid == 0)
      atomicExch(&a.states[t], ((unsigned long long)total << 2) | (t == 0 ? kFlagInc : kFlagAgg));  // (no fence needed)
    {
      int run = off;
#pragma unroll
      for (int u = 0; u < kAddItems; u++) {
        if (p0 + u < n) S.excl[pad(p0 + u)] = (unsigned)run;
        if (keep >> u & 1u) {
          S.orow[pad(run)] = orow[u];
          S.oval[pad(run)] = oval[u];
          run++;
        }
      }
      if (tid == 0) S.excl[pad(n)] = (unsigned)total;
    }

    // 3b. start the next tile's loads, then look back for the output offset and write
    if (tn < a.n_tiles) add_prefetch(a, tn, P);
    if (tid < 32) {
      const unsigned long long pre = add_lookback_wait(a.states, t, (unsigned long long)total);
      if (tid == 0) S.prefix = (long long)pre;
    }
    __syncthreads();
    const long long base = S.prefix;
    for (int q = tid; q < total; q += kAddThreads) {
      __stcs(&a.out_rows[base + q], S.orow[pad(q)]);
      __stcs(&a.out_vals[base + q], S.oval[pad(q)]);
    }
    // col_ptr of the columns whose merged start lies in this tile: (cend[t-1], c_last],
    // and for the last tile every column up to n_cols
    const bool last = t == a.n_tiles - 1;
    const long long own_hi = last ? a.n_cols : c_last;
    for (long long c = own_lo + tid; c <= own_hi; c += kAddThreads) {
      int rel;
      if (c < c_first) rel = 0;  // empty columns before the tile's first one
      else if (c > c_last) rel = n;
      else if (span <= kAddTile) rel = S.cms[c - c_first];
      else rel = (int)((long long)__ldg(&a.ap[c]) + __ldg(&a.bp[c]) - tpos);
      a.out_ptr[c] = (int)(base + S.excl[pad(rel)]);
    }
    if (last && tid == 0) a.info[0] = base + total;
    __syncthreads();  // the staging is free for the next tile
    t = tn;
  }
}

struct AddWs {
  unsigned long long* ticket;
  unsigned long long* states;
  AddDesc* desc;
  int* cend;
};

static AddWs carve_add(void* ws, size_t cap, long long n_tiles, size_t* need) {
  Carve cv(ws, cap);
  AddWs w;
  w.ticket = cv.take<unsigned long long>(1);
  w.states = cv.take<unsigned long long>((size_t)n_tiles + 1);
  w.desc = cv.take<AddDesc>((size_t)n_tiles + 1);
  w.cend = cv.take<int>((size_t)n_tiles + 1);
  if (need) *need = cv.off;
  return w;
}

// resident CTAs of the persistent tile kernel (per device; 0 = cannot configure)
static int add_resident() {
  static std::atomic<int> grid[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  if (grid[dev] == 0) {
    int per_sm = 0, sms = 0;
    if (cudaFuncSetAttribute(add_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(AddSmem)) !=
        cudaSuccess)
      return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, add_tile_kernel, kAddThreads, sizeof(AddSmem));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid[dev] = std::max(1, per_sm * sms);
  }
  return grid[dev];
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_add_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b) {
  (void)n_cols;
  const long long n_tiles = (nnz_a + nnz_b + kAddTile - 1) / kAddTile;
  size_t need = 0;
  carve_add(nullptr, 0, n_tiles, &need);
  return need;
}

int as_csc_add_f64(int64_t n_rows, int64_t n_cols, double alpha, double beta, const int32_t* a_col_ptr,
                   const int32_t* a_row_idx, const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx,
                   const double* b_vals, int64_t nnz_a, int64_t nnz_b, int32_t* col_ptr, int32_t* row_idx,
                   double* out_vals, int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0 && nnz_a >= 0 && nnz_b >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(nnz_a + nnz_b <= 0x7fffffffll, AS_ERR_ARG, "nnz outside the int32 range");
  AS_REQUIRE(ws_bytes >= as_add_workspace_bytes(n_cols, nnz_a, nnz_b), AS_ERR_ARG, "workspace too small");
  const int resident = add_resident();
  AS_REQUIRE(resident > 0, AS_ERR_CUDA, "cannot configure the add kernel");
  const long long M = nnz_a + nnz_b;
  const long long n_tiles = (M + kAddTile - 1) / kAddTile;
  if (n_tiles == 0) {
    AS_CUDA_TRY(cudaMemsetAsync(col_ptr, 0, (size_t)(n_cols + 1) * sizeof(int32_t), st));
    AS_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int64_t), st));
    return AS_OK;
  }
  const AddWs w = carve_add(ws, ws_bytes, n_tiles, nullptr);
  const long long part_threads = std::max((long long)n_cols, n_tiles);
  add_partition_kernel<<<(unsigned)((part_threads + kAddPartThreads - 1) / kAddPartThreads), kAddPartThreads, 0,
                         st>>>(n_cols, nnz_a, nnz_b, n_tiles, a_col_ptr, a_row_idx, b_col_ptr, b_row_idx, w.desc, w.cend,
                               w.states, w.ticket);
  AS_LAUNCH_CHECK();
  AddArgs a;
  a.n_cols = n_cols;
  a.M = M;
  a.n_tiles = n_tiles;
  a.alpha = alpha;
  a.beta = beta;
  a.ap = a_col_ptr;
  a.ar = a_row_idx;
  a.av = a_vals;
  a.bp = b_col_ptr;
  a.br = b_row_idx;
  a.bv = b_vals;
  a.out_ptr = col_ptr;
  a.out_rows = row_idx;
  a.out_vals = out_vals;
  a.info = (long long*)info;
  a.desc = w.desc;
  a.cend = w.cend;
  a.states = w.states;
  a.ticket = w.ticket;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min<long long>(n_tiles, resident));
  cfg.blockDim = dim3(kAddThreads);
  cfg.dynamicSmemBytes = sizeof(AddSmem);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AS_CUDA_TRY(cudaLaunchKernelEx(&cfg, add_tile_kernel, a));
  return AS_OK;
}

}  // extern "C"
