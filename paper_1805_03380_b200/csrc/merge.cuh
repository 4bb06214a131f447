// merge.cuh -- merge-path walking over the concatenated column pairs of two
// CSC matrices with the same shape (the decomposition shared by the fused
// trace and the sparse add).
//
// The merged sequence is A[:,0] (+) B[:,0], A[:,1] (+) B[:,1], ... of length
// nnzA + nnzB; merged column c starts at ms(c) = a_ptr[c] + b_ptr[c].  A CTA
// owns a contiguous range of it and walks it in chunks of kMThreads * items;
// for each chunk the merged starts of a window of kMWin columns are staged
// in shared memory (coalesced), so each thread finds its column with a
// shared-memory binary search, then splits the column with a merge-path
// search (A wins ties) and merges its positions.
#pragma once

#include "common.cuh"

namespace as {

constexpr int kMThreads = 256;
constexpr int kMWin = 512;

AS_DEVICE_INLINE long long mstart_of(const int* ap, const int* bp, long long c) {
  return (long long)__ldg(&ap[c]) + (long long)__ldg(&bp[c]);
}

// last c in [lo, hi] with ms(c) <= d (global memory)
AS_DEVICE_INLINE long long col_of_global(const int* ap, const int* bp, long long lo, long long hi, long long d) {
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (mstart_of(ap, bp, mid) <= d) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

struct MergeWindow {
  long long c_base;   // first column of the window
  int n;              // columns staged (window holds ms(c_base .. c_base + n))
  long long ms[kMWin + 1];
};

// Stage ms(c) for c in [c_base, c_base + kMWin] (clipped to n_cols).
AS_DEVICE_INLINE void stage_window(MergeWindow& W, const int* ap, const int* bp, long long n_cols, long long c_base) {
  const long long last = min(n_cols, c_base + kMWin);
  for (long long c = c_base + threadIdx.x; c <= last; c += blockDim.x) W.ms[c - c_base] = mstart_of(ap, bp, c);
  if (threadIdx.x == 0) {
    W.c_base = c_base;
    W.n = (int)(last - c_base);
  }
}

// Column holding merged position d (last c with ms(c) <= d, c < n_cols);
// uses the window when d lies inside it.
AS_DEVICE_INLINE long long col_of(const MergeWindow& W, const int* ap, const int* bp, long long n_cols, long long d) {
  if (d >= W.ms[0] && d < W.ms[W.n]) {
    int lo = 0, hi = W.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (W.ms[mid] <= d) lo = mid;
      else hi = mid - 1;
    }
    return W.c_base + lo;
  }
  return col_of_global(ap, bp, 0, n_cols - 1, d);
}

// Position a thread at merged position d inside column c: returns the merge
// path split (i, j) with A winning ties, after skipping a B element that the
// previous position's thread consumed together with an equal A element.
AS_DEVICE_INLINE void split_at(const int* __restrict__ ar, const int* __restrict__ br, long long a0, long long b0,
                               long long la, long long lb, long long dl, long long* pi, long long* pj) {
  long long lo = max(0ll, dl - lb), hi = min(dl, la);
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (__ldg(&ar[a0 + mid]) <= __ldg(&br[b0 + dl - mid - 1])) lo = mid + 1;
    else hi = mid;
  }
  long long i = lo, j = dl - lo;
  if (i > 0 && j < lb && __ldg(&br[b0 + j]) == __ldg(&ar[a0 + i - 1])) j++;
  *pi = i;
  *pj = j;
}

}  // namespace as
