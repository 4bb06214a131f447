// trace.cu -- fused trace(A^T B) without forming the product.
//
// Replaces _kernels.fused_trace (_kernels.py:153-175): sum over columns j of
// the products of coincident nonzeros of A[:,j] and B[:,j].
//
// B200 design: two kernels, picked on the host from the mean column length.
// Up to 384 entries per column the warp-tile kernel runs (a warp's consecutive
// column pairs staged in shared memory by bulk copies -- TMA -- in a per-warp
// software pipeline, 2^LG lanes per pair merging list segments with two
// cursors); beyond, or when the row arrays are not 16-byte aligned, the
// warp-per-column kernel (register lists, a shared-memory row filter, deferred
// searches).  Every row index is read once, values are gathered only at
// matches.  Partial sums are double-double (TwoSum) and reduced in fixed
// trees, so the result is deterministic and within an ulp or two of the
// exactly rounded sum; the reference's sequential left fold
// (_kernels.py:158-168) differs from it only by its own rounding.
#include "capi_util.cuh"
#include "common.cuh"
#include "merge.cuh"

#include <climits>

namespace as {

constexpr int kTrThreads = 256;

struct DD {
  double s, e;
};

AS_DEVICE_INLINE void dd_add(DD& a, double p) {
  double t = __dadd_rn(a.s, p);
  double bp = __dsub_rn(t, a.s);
  double err = __dadd_rn(__dsub_rn(a.s, __dsub_rn(t, bp)), __dsub_rn(p, bp));
  a.s = t;
  a.e = __dadd_rn(a.e, err);
}

// the (rare) match path kept out of line so the pointer-advance loop is not
// if-converted into predicated double-double arithmetic on every step
__device__ __noinline__ void dd_add_match(DD& acc, const double* __restrict__ av, const double* __restrict__ bv,
                                          int ia, int ib) {
  dd_add(acc, __dmul_rn(__ldg(&av[ia]), __ldg(&bv[ib])));
}

AS_DEVICE_INLINE DD dd_merge(DD a, DD b) {
  DD r{a.s, __dadd_rn(a.e, b.e)};
  dd_add(r, b.s);
  return r;
}

AS_DEVICE_INLINE DD dd_shfl_xor(DD a, int o) {
  DD r;
  r.s = __shfl_xor_sync(0xffffffffu, a.s, o);
  r.e = __shfl_xor_sync(0xffffffffu, a.e, o);
  return r;
}

// One warp per column pair (grid-stride over columns), software-pipelined:
// while column c is processed, the row lists of the warp's next column are
// already loaded into registers (lists of <= kTrRegs * 32 entries) and the
// pointers of the one after that are in flight.  The longer list goes to the
// warp's shared buffer (sorted, for lower_bound) and to an 8192-bit filter on
// the low row bits; each shorter-list row tests its filter bit and only the
// hits (~1.2% false positives at 100 entries per list) are searched, one
// warp-wide round per pending hit.  Values are read only at true matches.
// Longer columns fall back to a shared-memory lower_bound over the whole
// shorter list (<= kTrWarpBuf) or a global-memory search.
// Measured on cfg 4 (B200, 100k columns x ~100 entries): per-thread merge
// path over the concatenated columns 90-96 us, lane-per-column merge 127 us,
// warp lower_bound 78 us, + register lists 70 us, + filter 59 us, + deferred
// search 53 us (instruction-issue bound: ~69% issue slots busy).
constexpr int kTrWarpBuf = 512;
#ifndef AS_TR_REGS
#define AS_TR_REGS 5
#endif
constexpr int kTrRegs = AS_TR_REGS;  // lists of up to kTrRegs * 32 entries are loaded straight into registers
constexpr int kTrBits = 8192;  // per-warp row filter (1 KB)

__global__ void __launch_bounds__(kTrThreads)
trace_partial_kernel(long long n_cols, const int* __restrict__ ap, const int* __restrict__ ar,
                     const double* __restrict__ av, const int* __restrict__ bp, const int* __restrict__ br,
                     const double* __restrict__ bv, DD* partials, unsigned* done, double* out) {
  __shared__ int sbuf[kTrThreads / 32][kTrWarpBuf];
  __shared__ unsigned sbm[kTrThreads / 32][kTrBits / 32];
  __shared__ DD s_warp[kTrThreads / 32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * (kTrThreads / 32);
  DD acc{0.0, 0.0};
  int* buf = sbuf[wib];
  unsigned* bm = sbm[wib];
  for (int q = lane; q < kTrBits / 32; q += 32) bm[q] = 0u;
  __syncwarp();
  long long c = (long long)blockIdx.x * (kTrThreads / 32) + wib;
  // software pipeline: while column c is searched, the row lists of column
  // c + nwarps (when short enough for registers) and the pointers of column
  // c + 2 * nwarps are already in flight
  auto load_ptrs = [&](long long cc, int* p4) {
    if (cc < n_cols) {
      p4[0] = __ldg(&ap[cc]);
      p4[1] = __ldg(&ap[cc + 1]);
      p4[2] = __ldg(&bp[cc]);
      p4[3] = __ldg(&bp[cc + 1]);
    } else {
      p4[0] = p4[1] = p4[2] = p4[3] = 0;
    }
  };
  auto fits = [&](const int* p4) { return max(p4[1] - p4[0], p4[3] - p4[2]) <= kTrRegs * 32; };
  auto load_lists = [&](const int* p4, int* ra, int* rb) {
#pragma unroll
    for (int u = 0; u < kTrRegs; u++) {
      const int q = lane + 32 * u;
      ra[u] = q < p4[1] - p4[0] ? __ldcs(&ar[p4[0] + q]) : -1;
      rb[u] = q < p4[3] - p4[2] ? __ldcs(&br[p4[2] + q]) : -1;
    }
  };
  int pc[4], pn[4], la_n[kTrRegs], lb_n[kTrRegs];
  load_ptrs(c, pc);
  if (fits(pc)) load_lists(pc, la_n, lb_n);
  load_ptrs(c + nwarps, pn);
  for (; c < n_cols; c += nwarps) {
    int p4[4], ra[kTrRegs], rb[kTrRegs];
#pragma unroll
    for (int q = 0; q < 4; q++) p4[q] = pc[q];
#pragma unroll
    for (int u = 0; u < kTrRegs; u++) {
      ra[u] = la_n[u];
      rb[u] = lb_n[u];
    }
#pragma unroll
    for (int q = 0; q < 4; q++) pc[q] = pn[q];
    if (c + nwarps < n_cols && fits(pc)) load_lists(pc, la_n, lb_n);
    load_ptrs(c + 2 * nwarps, pn);
    const int a0 = p4[0], a1 = p4[1], b0 = p4[2], b1 = p4[3];
    const int la = a1 - a0, lb = b1 - b0;
    if (la == 0 || lb == 0) continue;
    const bool a_long = la >= lb;
    const int* Lr = a_long ? ar : br;
    const int* Sr = a_long ? br : ar;
    const double* Lv = a_long ? av : bv;
    const double* Sv = a_long ? bv : av;
    const int l0 = a_long ? a0 : b0, ll = a_long ? la : lb;
    const int s0 = a_long ? b0 : a0, sl = a_long ? lb : la;
    if (ll <= kTrRegs * 32) {
      // the longer list goes to the warp's buffer and to a 4096-bit filter
      // on the low row bits; a shorter-list row is searched for only when its
      // filter bit is set (~2.5% of them at 100 entries per list)
#pragma unroll
      for (int u = 0; u < kTrRegs; u++) {
        const int lv = a_long ? ra[u] : rb[u];
        buf[lane + 32 * u] = lv < 0 ? INT_MAX : lv;
        if (lv >= 0) atomicOr(&bm[(lv >> 5) & (kTrBits / 32 - 1)], 1u << (lv & 31));
      }
      __syncwarp();
      // filter pass, then one warp-wide search round per pending hit (a lane
      // searches its hits one by one; the rounds are shared by all lanes)
      int sv[kTrRegs];
      unsigned pend = 0;
#pragma unroll
      for (int u = 0; u < kTrRegs; u++) {
        sv[u] = a_long ? rb[u] : ra[u];
        if (sv[u] >= 0 && ((bm[(sv[u] >> 5) & (kTrBits / 32 - 1)] >> (sv[u] & 31)) & 1u)) pend |= 1u << u;
      }
      while (__any_sync(0xffffffffu, pend != 0)) {
        if (pend) {
          const int u = __ffs(pend) - 1;
          pend &= pend - 1;
          int r = sv[0];
#pragma unroll
          for (int q = 1; q < kTrRegs; q++) r = (u == q) ? sv[q] : r;
          int pos = 0;
          for (int step = 128; step > 0; step >>= 1) {  // covers kTrRegs * 32 <= 255
            const int probe = pos + step;
            pos = (probe <= kTrRegs * 32 && buf[probe - 1] < r) ? probe : pos;
          }
          if (pos < ll && buf[pos] == r) dd_add_match(acc, Lv, Sv, l0 + pos, s0 + lane + 32 * u);
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kTrRegs; u++) {
        const int lv = a_long ? ra[u] : rb[u];
        if (lv >= 0) bm[(lv >> 5) & (kTrBits / 32 - 1)] = 0u;
      }
    } else if (ll <= kTrWarpBuf) {
      for (int q = lane; q < ll; q += 32) buf[q] = __ldg(&Lr[l0 + q]);
      __syncwarp();
      int span = 1;
      while (span < ll) span <<= 1;
      for (int q = lane; q < sl; q += 32) {
        const int r = __ldg(&Sr[s0 + q]);
        int pos = 0;
        for (int step = span >> 1; step > 0; step >>= 1) {
          const int probe = pos + step;
          pos = (probe <= ll && buf[probe - 1] < r) ? probe : pos;
        }
        if (pos < ll && buf[pos] == r) dd_add_match(acc, Lv, Sv, l0 + pos, s0 + q);
      }
    } else {
      const int* L = Lr + l0;
      for (int q = lane; q < sl; q += 32) {
        const int r = __ldg(&Sr[s0 + q]);
        int lo = 0, hi = ll;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(&L[mid]) < r) lo = mid + 1;
          else hi = mid;
        }
        if (lo < ll && __ldg(&L[lo]) == r) dd_add_match(acc, Lv, Sv, l0 + lo, s0 + q);
      }
    }
    __syncwarp();
  }
  // deterministic block reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = dd_merge(acc, dd_shfl_xor(acc, o));
  const int warp = wib;
  if (lane == 0) s_warp[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    DD v = lane < kTrThreads / 32 ? s_warp[lane] : DD{0.0, 0.0};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dd_merge(v, dd_shfl_xor(v, o));
    if (lane == 0) {
      partials[blockIdx.x] = v;
      __threadfence();
      unsigned prev = atomicAdd(done, 1u);
      s_last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (s_last && warp == 0) {
    __threadfence();
    DD v{0.0, 0.0};
    for (long long b = lane; b < gridDim.x; b += 32) {
      DD p{__ldcg(&partials[b].s), __ldcg(&partials[b].e)};
      v = dd_merge(v, p);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dd_merge(v, dd_shfl_xor(v, o));
    if (lane == 0) {
      double hi2 = __dadd_rn(v.s, v.e);
      double lo2 = __dsub_rn(v.e, __dsub_rn(hi2, v.s));
      out[0] = hi2;
      out[1] = lo2;
    }
  }
}

// ------------------------------------------------------------------------
// Warp-tile kernel (the default for mean column lengths up to kTwMaxMean): a
// warp takes 32 >> LG consecutive column pairs, 2^LG lanes per pair (LG picked
// on the host from the mean column length, <= 13 entries of each list per
// lane).  The pairs' row lists are contiguous in the CSC arrays, so a warp's
// tile -- A's run and B's run -- comes into the warp's shared-memory buffers
// with two bulk copies (the TMA engine's 1-D mode) completed on the warp's
// mbarrier; no thread issues a load for a row index.  Every warp runs its own
// three-stage software pipeline with no CTA barrier: the column pointers of
// tile k + 2 are in flight (registers) and the bulk copies of tile k + 1 land
// in the other buffer while tile k is merged.  A pair's lanes split the longer
// list into equal segments; each lane finds where its segment starts in the
// shorter list (one lower_bound in shared memory) and runs a branch-free
// two-pointer merge of its segment against it on shared-memory byte addresses
// (~17 instructions per list entry and lane; the warp-per-column kernel spends
// ~430 warp instructions per column pair at cfg 4, this one ~190).  Pairs
// far above the mean (more than kTwLongPerLane entries per lane) are searched
// by the whole warp afterwards (every lane a stride of the shorter list, a
// lower_bound in the longer one, both in shared memory); a tile whose runs
// exceed the buffers is searched pair by pair in global memory.  Tiles are
// assigned round-robin (static), every lane sums its matches in column order
// in double-double, and the block / grid reductions are fixed trees:
// deterministic.
// Measured on cfg 4: a CTA-wide variant (256 threads, 64 pairs per tile, one
// buffer, CTA barriers) ran 59 us -- every CTA of the grid loads, then every
// CTA merges, in lockstep, so the memory system and the issue slots idle in
// turn; the per-warp pipeline removes the lockstep.
#ifndef AS_TW_WARPS
#define AS_TW_WARPS 8      // 3 CTAs x 8 warps x 2 stages x 2 lists x 584 entries = 224 KB per SM
#define AS_TW_CAP 576
#define AS_TW_PER_LANE 13  // a warp tile holds <= 32 x 13 = 416 entries of each list at the mean: 72 % of a buffer
#endif
#ifndef AS_TW_ILP2
#define AS_TW_ILP2 0  // measured on cfg 4: 51 us with two chains per lane vs 43 us with one (more instructions, more searches)
#endif
constexpr bool kTwIlp2 = AS_TW_ILP2 != 0;  // two interleaved chains per lane
constexpr int kTwWarps = AS_TW_WARPS;  // warps per CTA
constexpr int kTwThreads = kTwWarps * 32;
constexpr int kTwCap = AS_TW_CAP;      // entries per list buffer of a warp
constexpr int kTwStride = kTwCap + 8; // + alignment slack (a run starts up to 3 entries into its first quad)
constexpr int kTwLongPerLane = 128;   // a pair with more entries per lane goes to the whole warp
constexpr int kTwPerLane = AS_TW_PER_LANE;        // target entries of each list per lane (picks LG)
constexpr int kTwMaxMean = 384;       // beyond: the warp-per-column kernel

struct TwSmem {
  alignas(16) int buf[kTwWarps][2][2][kTwStride];  // [warp][stage][A, B][entries]
  alignas(8) unsigned long long bar[kTwWarps][2];
  DD s_warp[kTwWarps];
  int s_last;
};

AS_DEVICE_INLINE int tt_lower_bound(const int* __restrict__ s, int n, int key) {
  int lo = 0;
  while (n > 0) {
    const int half = n >> 1;
    const bool right = s[lo + half] < key;
    lo = right ? lo + half + 1 : lo;
    n = right ? n - half - 1 : half;
  }
  return lo;
}

AS_DEVICE_INLINE int tt_lds(unsigned addr) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// one merge step for l != s: the cursor of the smaller entry moves on.  Each
// cursor keeps its next entry prefetched in a register (ln / sn), so the
// compare of the following step never waits for a shared-memory load issued
// in this one: the loop-carried chain is compare -> move, and the prefetch has
// a whole step (two when the cursors alternate) to arrive.
AS_DEVICE_INLINE void tt_step(unsigned& pl, unsigned& ps, int& l, int& s, int& ln, int& sn) {
  asm volatile(
      "{\n .reg .pred q1, q2;\n setp.lt.s32 q1, %2, %3;\n setp.lt.s32 q2, %3, %2;\n"
      " @q1 mov.b32 %2, %4;\n @q2 mov.b32 %3, %5;\n"
      " @q1 add.u32 %0, %0, 4;\n @q2 add.u32 %1, %1, 4;\n"
      " @q1 ld.shared.b32 %4, [%0+4];\n @q2 ld.shared.b32 %5, [%1+4];\n}"
      : "+r"(pl), "+r"(ps), "+r"(l), "+r"(s), "+r"(ln), "+r"(sn));
}

// the same step under an activity flag (two chains interleaved in one loop:
// a finished chain stands still)
AS_DEVICE_INLINE void tt_step_if(unsigned& pl, unsigned& ps, int& l, int& s, int& ln, int& sn, int act) {
  asm volatile(
      "{\n .reg .pred q0, q1, q2;\n setp.ne.s32 q0, %6, 0;\n"
      " setp.lt.and.s32 q1, %2, %3, q0;\n setp.lt.and.s32 q2, %3, %2, q0;\n"
      " @q1 mov.b32 %2, %4;\n @q2 mov.b32 %3, %5;\n"
      " @q1 add.u32 %0, %0, 4;\n @q2 add.u32 %1, %1, 4;\n"
      " @q1 ld.shared.b32 %4, [%0+4];\n @q2 ld.shared.b32 %5, [%1+4];\n}"
      : "+r"(pl), "+r"(ps), "+r"(l), "+r"(s), "+r"(ln), "+r"(sn)
      : "r"(act));
}

struct TtChain {  // one lane's merge of a segment of the longer list against the shorter one
  unsigned pl, ps, ple, pse;
  int l, s, ln, sn;
};

// chain over segment `seg` of `nseg` of L (ll entries) against Sh (sl entries); inert when empty
AS_DEVICE_INLINE void tt_chain_init(TtChain& c, const int* L, const int* Sh, unsigned Lb, unsigned Sb, int ll, int sl,
                                    int seg, int lg_nseg) {
  c.pl = c.ple = c.ps = c.pse = 0u;
  c.l = c.ln = 0;
  c.s = c.sn = 1;
  const int i0 = (ll * seg) >> lg_nseg, ie = (ll * (seg + 1)) >> lg_nseg;
  if (i0 < ie) {
    const int l = L[i0];
    const int j0 = seg == 0 ? 0 : tt_lower_bound(Sh, sl, l);
    if (j0 < sl) {
      c.pl = Lb + 4u * (unsigned)i0;
      c.ple = Lb + 4u * (unsigned)ie;
      c.ps = Sb + 4u * (unsigned)j0;
      c.pse = Sb + 4u * (unsigned)sl;
      c.l = l;
      c.s = tt_lds(c.ps);
      c.ln = tt_lds(c.pl + 4u);  // up to two entries past a list's end: inside the slack
      c.sn = tt_lds(c.ps + 4u);
    }
  }
}

// every entry of the shorter list (a stride per lane) searched in the longer one
template <bool kGlobal>
AS_DEVICE_INLINE void tw_search_pair(DD& acc, int lane, const int* La, const int* Lb, int a0, int a1, int b0, int b1,
                                     const double* __restrict__ av, const double* __restrict__ bv) {
  // La / Lb point at the pair's first A / B entry (shared or global memory)
  const int la = a1 - a0, lb = b1 - b0;
  if (la == 0 || lb == 0) return;
  const bool a_long = la >= lb;
  const int* L = a_long ? La : Lb;
  const int* Sh = a_long ? Lb : La;
  const int ll = a_long ? la : lb, sl = a_long ? lb : la;
  for (int q = lane; q < sl; q += 32) {
    const int r = kGlobal ? __ldg(&Sh[q]) : Sh[q];
    int lo = 0, n = ll;
    while (n > 0) {
      const int half = n >> 1;
      const int v = kGlobal ? __ldg(&L[lo + half]) : L[lo + half];
      const bool right = v < r;
      lo = right ? lo + half + 1 : lo;
      n = right ? n - half - 1 : half;
    }
    if (lo < ll && (kGlobal ? __ldg(&L[lo]) : L[lo]) == r)
      dd_add_match(acc, av, bv, a_long ? a0 + lo : a0 + q, a_long ? b0 + q : b0 + lo);
  }
}

template <int LG>
__global__ void __launch_bounds__(kTwThreads, 3)
trace_warp_tile_kernel(long long n_cols, const int* __restrict__ ap, const int* __restrict__ ar,
                       const double* __restrict__ av, const int* __restrict__ bp, const int* __restrict__ br,
                       const double* __restrict__ bv, int nnz_a, int nnz_b, DD* partials, unsigned* done,
                       double* out) {
  extern __shared__ __align__(16) unsigned char tw_raw[];
  TwSmem& S = *reinterpret_cast<TwSmem*>(tw_raw);
  constexpr int G = 1 << LG;   // lanes per column pair
  constexpr int WC = 32 >> LG; // column pairs per warp tile
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int lc = lane >> LG, sub = lane & (G - 1);
  const long long n_tiles = (n_cols + WC - 1) / WC;
  const long long nW = (long long)gridDim.x * kTwWarps;
  DD acc{0.0, 0.0};
  if (lane == 0) {
    mbar_init(&S.bar[wib][0], 1);
    mbar_init(&S.bar[wib][1], 1);
  }
  __syncwarp();
  // a tile's column pointers: lane q holds those of column c0 + q (clamped to
  // n_cols, so columns past the end read as empty), plus the tile's last one
  auto load_ptrs = [&](long long tile, int& pa, int& pb, int& pa_last, int& pb_last) {
    pa = pb = pa_last = pb_last = 0;
    if (tile < n_tiles) {
      const long long c0 = tile * WC;
      const long long c = c0 + lane < n_cols ? c0 + lane : n_cols;
      pa = __ldg(&ap[c]);
      pb = __ldg(&bp[c]);
      if (WC == 32) {
        const long long ce = c0 + WC < n_cols ? c0 + WC : n_cols;
        pa_last = __ldg(&ap[ce]);
        pb_last = __ldg(&bp[ce]);
      }
    }
  };
  // issue the tile's bulk copies into `stage`; false when its runs exceed the buffers
  auto issue = [&](int stage, int pa, int pb, int pa_last, int pb_last) -> bool {
    const int a_lo = __shfl_sync(0xffffffffu, pa, 0), b_lo = __shfl_sync(0xffffffffu, pb, 0);
    const int a_hi = WC == 32 ? pa_last : __shfl_sync(0xffffffffu, pa, WC & 31);
    const int b_hi = WC == 32 ? pb_last : __shfl_sync(0xffffffffu, pb, WC & 31);
    const int a_base = a_lo & ~3, b_base = b_lo & ~3;
    if (a_hi - a_base > kTwCap || b_hi - b_base > kTwCap) return false;
    // the copies end at the next 16-byte boundary, or at the last one inside
    // the array (then the array's last < 4 entries come by plain loads)
    const int a_end = min((a_hi + 3) & ~3, nnz_a & ~3), b_end = min((b_hi + 3) & ~3, nnz_b & ~3);
    int* sa = S.buf[wib][stage][0];
    int* sb = S.buf[wib][stage][1];
    if (lane == 0) {
      const unsigned na = a_end > a_base ? (unsigned)(a_end - a_base) * 4u : 0u;
      const unsigned nb = b_end > b_base ? (unsigned)(b_end - b_base) * 4u : 0u;
      mbar_expect_tx(&S.bar[wib][stage], na + nb);
      if (na) bulk_g2s_noarrive(sa, ar + a_base, na, &S.bar[wib][stage]);
      if (nb) bulk_g2s_noarrive(sb, br + b_base, nb, &S.bar[wib][stage]);
    }
    if (a_hi > a_end && lane < 4) {
      const int q = max(a_end, a_base) + lane;
      if (q < a_hi) sa[q - a_base] = __ldg(&ar[q]);
    }
    if (b_hi > b_end && lane >= 4 && lane < 8) {
      const int q = max(b_end, b_base) + lane - 4;
      if (q < b_hi) sb[q - b_base] = __ldg(&br[q]);
    }
    return true;
  };
  long long tile = (long long)blockIdx.x * kTwWarps + wib;
  int pa0, pb0, pal0, pbl0, pa1, pb1, pal1, pbl1;
  load_ptrs(tile, pa0, pb0, pal0, pbl0);
  load_ptrs(tile + nW, pa1, pb1, pal1, pbl1);
  bool fit0 = tile < n_tiles ? issue(0, pa0, pb0, pal0, pbl0) : false;
  unsigned phases = 0;  // bit s = the parity stage s's mbarrier completes next
  for (int k = 0; tile < n_tiles; tile += nW, k++) {
    const int stage = k & 1;
    int pan, pbn, paln, pbln;
    load_ptrs(tile + 2 * nW, pan, pbn, paln, pbln);
    const bool fit1 = tile + nW < n_tiles ? issue(stage ^ 1, pa1, pb1, pal1, pbl1) : false;
    const int a_base = __shfl_sync(0xffffffffu, pa0, 0) & ~3, b_base = __shfl_sync(0xffffffffu, pb0, 0) & ~3;
    // this lane's pair
    const int a0 = __shfl_sync(0xffffffffu, pa0, lc);
    const int b0 = __shfl_sync(0xffffffffu, pb0, lc);
    int a1 = __shfl_sync(0xffffffffu, pa0, (lc + 1) & 31);
    int b1 = __shfl_sync(0xffffffffu, pb0, (lc + 1) & 31);
    if (WC == 32 && lc == 31) {
      a1 = pal0;
      b1 = pbl0;
    }
    const int la = a1 - a0, lb = b1 - b0;
    if (fit0) {
      __syncwarp();  // the plain-loaded tail entries
      mbar_wait(&S.bar[wib][stage], (phases >> stage) & 1u);
      phases ^= 1u << stage;
      const int* sa = S.buf[wib][stage][0];
      const int* sb = S.buf[wib][stage][1];
      const bool is_long = la > 0 && lb > 0 && la + lb > G * kTwLongPerLane;
      if (la > 0 && lb > 0 && !is_long) {
        const bool a_long = la >= lb;
        const int* L = a_long ? sa + (a0 - a_base) : sb + (b0 - b_base);
        const int* Sh = a_long ? sb + (b0 - b_base) : sa + (a0 - a_base);
        const int ll = a_long ? la : lb, sl = a_long ? lb : la;
        const unsigned Lb = (unsigned)__cvta_generic_to_shared(L);
        const unsigned Sb = (unsigned)__cvta_generic_to_shared(Sh);
        auto match = [&](TtChain& c) {
          const int i = (int)((c.pl - Lb) >> 2), j = (int)((c.ps - Sb) >> 2);
          dd_add_match(acc, av, bv, a_long ? a0 + i : a0 + j, a_long ? b0 + j : b0 + i);
          c.pl += 4u;
          c.ps += 4u;
          c.l = c.ln;
          c.s = c.sn;
          c.ln = tt_lds(c.pl + 4u);
          c.sn = tt_lds(c.ps + 4u);
        };
        if (kTwIlp2 && LG >= 1) {
          // two chains per lane (2G segments per pair), interleaved in one loop: twice the
          // independent compare -> move chains per warp for the same shared memory
          TtChain c1, c2;
          tt_chain_init(c1, L, Sh, Lb, Sb, ll, sl, 2 * sub, LG + 1);
          tt_chain_init(c2, L, Sh, Lb, Sb, ll, sl, 2 * sub + 1, LG + 1);
          for (;;) {
            const bool act1 = c1.pl < c1.ple && c1.ps < c1.pse, act2 = c2.pl < c2.ple && c2.ps < c2.pse;
            if (!(act1 || act2)) break;
            const bool m1 = act1 && c1.l == c1.s, m2 = act2 && c2.l == c2.s;
            if (m1 || m2) {
              if (m1) match(c1);
              if (m2) match(c2);
              continue;
            }
            tt_step_if(c1.pl, c1.ps, c1.l, c1.s, c1.ln, c1.sn, act1);
            tt_step_if(c2.pl, c2.ps, c2.l, c2.s, c2.ln, c2.sn, act2);
          }
        } else {
          // two-pointer merge on shared-memory byte addresses; the inner loop runs to the
          // next match or the end of either range
          TtChain c;
          tt_chain_init(c, L, Sh, Lb, Sb, ll, sl, sub, LG);
          for (;;) {
            while (c.pl < c.ple && c.ps < c.pse && c.l != c.s) tt_step(c.pl, c.ps, c.l, c.s, c.ln, c.sn);
            if (c.pl >= c.ple || c.ps >= c.pse) break;
            match(c);
          }
        }
      }
      // pairs far above the mean length, in column order, by the whole warp
      unsigned m = __ballot_sync(0xffffffffu, is_long && sub == 0);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int xa0 = __shfl_sync(0xffffffffu, a0, src), xa1 = __shfl_sync(0xffffffffu, a1, src);
        const int xb0 = __shfl_sync(0xffffffffu, b0, src), xb1 = __shfl_sync(0xffffffffu, b1, src);
        tw_search_pair<false>(acc, lane, sa + (xa0 - a_base), sb + (xb0 - b_base), xa0, xa1, xb0, xb1, av, bv);
      }
    } else {
      // runs beyond the buffers: pair by pair in global memory
      for (int c = 0; c < WC; c++) {
        const int src = c << LG;
        const int xa0 = __shfl_sync(0xffffffffu, a0, src), xa1 = __shfl_sync(0xffffffffu, a1, src);
        const int xb0 = __shfl_sync(0xffffffffu, b0, src), xb1 = __shfl_sync(0xffffffffu, b1, src);
        tw_search_pair<true>(acc, lane, ar + xa0, br + xb0, xa0, xa1, xb0, xb1, av, bv);
      }
    }
    __syncwarp();  // the stage's buffers are free for the copies of tile k + 2
    pa0 = pa1, pb0 = pb1, pal0 = pal1, pbl0 = pbl1;
    pa1 = pan, pb1 = pbn, pal1 = paln, pbl1 = pbln;
    fit0 = fit1;
  }
  // deterministic block reduction, last block folds the partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = dd_merge(acc, dd_shfl_xor(acc, o));
  if (lane == 0) S.s_warp[wib] = acc;
  __syncthreads();
  if (wib == 0) {
    DD v = lane < kTwWarps ? S.s_warp[lane] : DD{0.0, 0.0};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dd_merge(v, dd_shfl_xor(v, o));
    if (lane == 0) {
      partials[blockIdx.x] = v;
      // launched with programmatic stream serialization behind the kernel that zeroes
      // `done`: everything above overlapped it, the counter is first touched here
      asm volatile("griddepcontrol.wait;" ::: "memory");
      __threadfence();
      const unsigned prev = atomicAdd(done, 1u);
      S.s_last = (prev == gridDim.x - 1);
    }
  }
  __syncthreads();
  if (S.s_last && wib == 0) {
    __threadfence();
    DD v{0.0, 0.0};
    for (long long b = lane; b < gridDim.x; b += 32) {
      DD p{__ldcg(&partials[b].s), __ldcg(&partials[b].e)};
      v = dd_merge(v, p);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dd_merge(v, dd_shfl_xor(v, o));
    if (lane == 0) {
      const double hi2 = __dadd_rn(v.s, v.e);
      const double lo2 = __dsub_rn(v.e, __dsub_rn(hi2, v.s));
      out[0] = hi2;
      out[1] = lo2;
    }
  }
}

// zeroes the last-block counter; the warp-tile kernel is launched behind it with
// programmatic stream serialization (no memset node in front of the trace)
__global__ void trace_zero_kernel(unsigned* done) {
  if (threadIdx.x == 0) *done = 0u;
}

template <int LG>
static int trace_tile_grid() {
  static std::atomic<int> grid[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
  if (grid[dev] == 0) {
    int per_sm = 0, sms = 0;
    if (cudaFuncSetAttribute(trace_warp_tile_kernel<LG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(TwSmem)) != cudaSuccess)
      return -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_warp_tile_kernel<LG>, kTwThreads, sizeof(TwSmem));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid[dev] = std::max(1, per_sm * sms);
  }
  return grid[dev];
}

int g_trace_engine = 0;  // as_set_trace_engine: 0 automatic (tile kernel), 1 warp-per-column kernel

static int trace_grid() {
  static std::atomic<int> grid[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  if (grid[dev] == 0) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_partial_kernel, kTrThreads, 0);
    per_sm = std::min(per_sm, 6);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid[dev] = std::max(1, per_sm * sms);
  }
  return grid[dev];
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_trace_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b) {
  (void)n_cols;
  (void)nnz_a;
  (void)nnz_b;
  return 256 + (size_t)148 * 32 * sizeof(DD);  // partials of the largest co-resident grid
}

int as_trace_atb_f64(int64_t n_rows, int64_t n_cols, const int32_t* a_col_ptr, const int32_t* a_row_idx,
                     const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx, const double* b_vals,
                     int64_t nnz_a, int64_t nnz_b, double* out, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_cols >= 0 && n_rows >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(ws_bytes >= as_trace_workspace_bytes(n_cols, nnz_a, nnz_b), AS_ERR_ARG, "workspace too small");
  unsigned* done = (unsigned*)ws;
  DD* partials = (DD*)((char*)ws + 256);
  // the warp-tile kernel's bulk copies need 16-byte aligned row arrays
  const bool aligned = (((uintptr_t)a_row_idx | (uintptr_t)b_row_idx) & 15u) == 0;
  const double mean = n_cols > 0 ? (double)(nnz_a + nnz_b) / (2.0 * (double)n_cols) : 0.0;
  if (g_trace_engine == 0 && aligned && n_cols > 0 && mean <= (double)kTwMaxMean && nnz_a < INT_MAX &&
      nnz_b < INT_MAX) {
    // lanes per column pair: <= kTwPerLane entries of each list per lane at the mean column length
    int lg = 0;
    while (lg < 5 && (double)(kTwPerLane << lg) < mean) lg++;
    int grid = -1;
#define AS_TT_LAUNCH(LG)                                                                                          \
  case LG:                                                                                                        \
    grid = trace_tile_grid<LG>();                                                                                 \
    if (grid > 0) {                                                                                               \
      const long long tiles = (n_cols + (32 >> LG) - 1) / (32 >> LG);                                             \
      const unsigned blocks =                                                                                     \
          (unsigned)std::min<long long>(std::min(grid, 148 * 32), (tiles + kTwWarps - 1) / kTwWarps);             \
      trace_zero_kernel<<<1, 32, 0, st>>>(done);                                                                  \
      cudaLaunchConfig_t cfg = {};                                                                                \
      cfg.gridDim = dim3(blocks);                                                                                 \
      cfg.blockDim = dim3(kTwThreads);                                                                            \
      cfg.dynamicSmemBytes = sizeof(TwSmem);                                                                      \
      cfg.stream = st;                                                                                            \
      cudaLaunchAttribute attr[1];                                                                                \
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                            \
      attr[0].val.programmaticStreamSerializationAllowed = 1;                                                     \
      cfg.attrs = attr;                                                                                           \
      cfg.numAttrs = 1;                                                                                           \
      AS_CUDA_TRY(cudaLaunchKernelEx(&cfg, trace_warp_tile_kernel<LG>, (long long)n_cols, a_col_ptr, a_row_idx,   \
                                     a_vals, b_col_ptr, b_row_idx, b_vals, (int)nnz_a, (int)nnz_b, partials,      \
                                     done, out));                                                                 \
    }                                                                                                             \
    break;
    switch (lg) {
      AS_TT_LAUNCH(0)
      AS_TT_LAUNCH(1)
      AS_TT_LAUNCH(2)
      AS_TT_LAUNCH(3)
      AS_TT_LAUNCH(4)
      AS_TT_LAUNCH(5)
    }
#undef AS_TT_LAUNCH
    if (grid > 0) {
      AS_LAUNCH_CHECK();
      return AS_OK;
    }
  }
  AS_CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(unsigned), st));
  const long long blocks = std::min(trace_grid(), 148 * 32);
  trace_partial_kernel<<<(unsigned)blocks, kTrThreads, 0, st>>>(n_cols, a_col_ptr, a_row_idx, a_vals, b_col_ptr,
                                                                b_row_idx, b_vals, partials, done, out);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

int as_set_trace_engine(int engine) {
  if (engine < 0 || engine > 1) {
    as::set_error("trace engine must be 0 or 1, got %d", engine);
    return AS_ERR_ARG;
  }
  as::g_trace_engine = engine;
  return AS_OK;
}

}  // extern "C"
