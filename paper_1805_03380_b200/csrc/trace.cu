// trace.cu -- fused trace(A^T B) without forming the product.
//
// Replaces _kernels.fused_trace (_kernels.py:153-175): sum over columns j of
// the products of coincident nonzeros of A[:,j] and B[:,j].
//
// B200 design: the (A,B) column pairs are laid end to end as one merged
// sequence of length nnzA + nnzB; every thread owns kItems consecutive
// positions of it (merge path), so the work is balanced whatever the column
// lengths, every row index is read exactly once (coalesced per warp), and
// values are gathered only at matches.  Partial sums are double-double
// (TwoSum) and reduced in a fixed tree, so the result is deterministic and
// within an ulp or two of the exactly rounded sum; the reference's sequential
// left fold (_kernels.py:158-168) differs from it only by its own rounding.
#include "capi_util.cuh"
#include "common.cuh"
#include "merge.cuh"

#include <climits>

namespace as {

constexpr int kTrThreads = 256;
constexpr int kTrItems = 32;
constexpr int kTrChunk = kTrThreads * kTrItems;

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
  const long long blocks = std::min(trace_grid(), 148 * 32);
  unsigned* done = (unsigned*)ws;
  DD* partials = (DD*)((char*)ws + 256);
  AS_CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(unsigned), st));
  trace_partial_kernel<<<(unsigned)blocks, kTrThreads, 0, st>>>(n_cols, a_col_ptr, a_row_idx, a_vals, b_col_ptr,
                                                                b_row_idx, b_vals, partials, done, out);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

}  // extern "C"
