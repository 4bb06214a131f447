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

// One warp per column pair (grid-stride over columns): the longer of the
// two row lists is staged in the warp's shared-memory buffer (coalesced),
// every lane takes elements of the shorter list (coalesced) and does a
// branch-free lower_bound there; values are read only at matches.  Columns
// whose longer list exceeds the buffer are searched in global memory.
// (Measured alternatives on cfg 4: per-thread merge path over the
// concatenated columns 90-96 us, lane-per-column sequential merge 127 us.)
constexpr int kTrWarpBuf = 1024;

__global__ void __launch_bounds__(kTrThreads)
trace_partial_kernel(long long n_cols, const int* __restrict__ ap, const int* __restrict__ ar,
                     const double* __restrict__ av, const int* __restrict__ bp, const int* __restrict__ br,
                     const double* __restrict__ bv, DD* partials, unsigned* done, double* out) {
  __shared__ int sbuf[kTrThreads / 32][kTrWarpBuf];
  __shared__ DD s_warp[kTrThreads / 32];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * (kTrThreads / 32);
  DD acc{0.0, 0.0};
  int* buf = sbuf[wib];
  for (long long c = (long long)blockIdx.x * (kTrThreads / 32) + wib; c < n_cols; c += nwarps) {
    const int a0 = __ldg(&ap[c]), a1 = __ldg(&ap[c + 1]), b0 = __ldg(&bp[c]), b1 = __ldg(&bp[c + 1]);
    const int la = a1 - a0, lb = b1 - b0;
    if (la == 0 || lb == 0) continue;
    const bool a_long = la >= lb;
    const int* Lr = a_long ? ar : br;
    const int* Sr = a_long ? br : ar;
    const double* Lv = a_long ? av : bv;
    const double* Sv = a_long ? bv : av;
    const int l0 = a_long ? a0 : b0, ll = a_long ? la : lb;
    const int s0 = a_long ? b0 : a0, sl = a_long ? lb : la;
    if (ll <= kTrWarpBuf) {
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
  static int grid = 0;
  if (grid == 0) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trace_partial_kernel, kTrThreads, 0);
    per_sm = std::min(per_sm, 6);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid = std::max(1, per_sm * sms);
  }
  return grid;
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
