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

namespace as {

constexpr int kTrThreads = 256;
constexpr int kTrItems = 16;
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

// merged start of column c
AS_DEVICE_INLINE long long mstart(const int* ap, const int* bp, long long c) {
  return (long long)ap[c] + (long long)bp[c];
}

__global__ void __launch_bounds__(kTrThreads)
trace_partial_kernel(long long n_cols, const int* __restrict__ ap, const int* __restrict__ ar,
                     const double* __restrict__ av, const int* __restrict__ bp, const int* __restrict__ br,
                     const double* __restrict__ bv, DD* partials, unsigned* done, double* out) {
  __shared__ long long s_clo, s_chi;
  __shared__ DD s_warp[kTrThreads / 32];
  __shared__ bool s_last;
  const long long M = mstart(ap, bp, n_cols);
  const long long cbase = (long long)blockIdx.x * kTrChunk;
  const long long cend = min(cbase + kTrChunk, M);
  if (threadIdx.x == 0) {
    // last column whose merged start <= cbase, and the one holding cend-1
    long long lo = 0, hi = n_cols;
    while (lo < hi) {
      long long mid = (lo + hi + 1) >> 1;
      if (mstart(ap, bp, mid) <= cbase) lo = mid;
      else hi = mid - 1;
    }
    s_clo = lo;
    long long lo2 = lo, hi2 = n_cols;
    while (lo2 < hi2) {
      long long mid = (lo2 + hi2 + 1) >> 1;
      if (mstart(ap, bp, mid) <= cend - 1) lo2 = mid;
      else hi2 = mid - 1;
    }
    s_chi = lo2;
  }
  __syncthreads();
  DD acc{0.0, 0.0};
  const long long d0 = cbase + (long long)threadIdx.x * kTrItems;
  const long long d1 = min(d0 + kTrItems, cend);
  if (d0 < d1) {
    // column holding d0: last c in [clo, chi] with mstart(c) <= d0
    long long lo = s_clo, hi = s_chi;
    while (lo < hi) {
      long long mid = (lo + hi + 1) >> 1;
      if (mstart(ap, bp, mid) <= d0) lo = mid;
      else hi = mid - 1;
    }
    long long c = lo;
    long long a0 = ap[c], b0 = bp[c];
    long long la = ap[c + 1] - a0, lb = bp[c + 1] - b0;
    long long dl = d0 - (a0 + b0);
    // merge-path split with A winning ties
    long long i_lo = max(0ll, dl - lb), i_hi = min(dl, la);
    while (i_lo < i_hi) {
      long long mid = (i_lo + i_hi) >> 1;
      if (ar[a0 + mid] <= br[b0 + dl - mid - 1]) i_lo = mid + 1;
      else i_hi = mid;
    }
    long long i = i_lo, j = dl - i_lo;
    // an equal pair split at our start was consumed by the previous thread
    if (i > 0 && j < lb && br[b0 + j] == ar[a0 + i - 1]) j++;
    long long pos = a0 + b0 + i + j;
    while (pos < d1) {
      if (i == la && j == lb) {
        c++;
        a0 = ap[c];
        b0 = bp[c];
        la = ap[c + 1] - a0;
        lb = bp[c + 1] - b0;
        i = j = 0;
        continue;
      }
      if (j == lb) {
        i++;
      } else if (i == la) {
        j++;
      } else {
        int ra = ar[a0 + i], rb = br[b0 + j];
        if (ra == rb) {
          dd_add(acc, __dmul_rn(av[a0 + i], bv[b0 + j]));
          i++;
          j++;
        } else if (ra < rb) {
          i++;
        } else {
          j++;
        }
      }
      pos = a0 + b0 + i + j;
    }
  }
  // deterministic block reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = dd_merge(acc, dd_shfl_xor(acc, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
      double hi = __dadd_rn(v.s, v.e);
      double lo = __dsub_rn(v.e, __dsub_rn(hi, v.s));
      out[0] = hi;
      out[1] = lo;
    }
  }
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_trace_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b) {
  long long M = nnz_a + nnz_b;
  long long blocks = M > 0 ? (M + kTrChunk - 1) / kTrChunk : 1;
  return 256 + ((size_t)blocks * sizeof(DD) + 255) / 256 * 256;
}

int as_trace_atb_f64(int64_t n_rows, int64_t n_cols, const int32_t* a_col_ptr, const int32_t* a_row_idx,
                     const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx, const double* b_vals,
                     int64_t nnz_a, int64_t nnz_b, double* out, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_cols >= 0 && n_rows >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(ws_bytes >= as_trace_workspace_bytes(n_cols, nnz_a, nnz_b), AS_ERR_ARG, "workspace too small");
  long long M = nnz_a + nnz_b;
  long long blocks = M > 0 ? (M + kTrChunk - 1) / kTrChunk : 1;
  unsigned* done = (unsigned*)ws;
  DD* partials = (DD*)((char*)ws + 256);
  AS_CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(unsigned), st));
  trace_partial_kernel<<<(unsigned)blocks, kTrThreads, 0, st>>>(n_cols, a_col_ptr, a_row_idx, a_vals, b_col_ptr,
                                                                b_row_idx, b_vals, partials, done, out);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

}  // extern "C"
