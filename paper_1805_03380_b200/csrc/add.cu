// add.cu -- alpha*A + beta*B of two canonical CSC matrices.
//
// Replaces _kernels.linear_combine (_kernels.py:12-48) via ops._combine /
// add / subtract / scaled_sum (ops.py:50-73).  Per column a two-pointer row
// merge; coincident rows give alpha*a + beta*b (product and sum separately
// rounded, as numba evaluates it: no FMA), others alpha*a or beta*b; exact
// zeros are pruned.
//
// B200 design: one cooperative launch of the co-resident grid.  The (A,B)
// column pairs form one merged sequence (merge.cuh); each CTA owns a
// contiguous range and walks it in chunks, each thread merging kAddItems
// consecutive positions.  Pass 1 counts the surviving entries, a grid
// barrier and a grid-wide prefix over the CTA totals give every CTA its
// output offset, pass 2 re-merges, stages the compacted chunk in shared
// memory and writes it with coalesced stores; the thread owning a column's
// first merged position writes its col_ptr.  No per-tile look-back chain.
#include "capi_util.cuh"
#include "common.cuh"
#include "merge.cuh"

namespace as {

constexpr int kAddItems = 8;
constexpr int kAddChunk = kMThreads * kAddItems;

// Merge positions [d0, d1) starting in column c.  emit(row, value) for kept
// outputs in order; on_col(c, produced) for every column whose start this
// thread owns (including empty columns sharing the position).
template <class Emit, class OnCol>
__device__ void merge_range(long long n_cols, long long c, long long d0, long long d1, const int* __restrict__ ap,
                            const int* __restrict__ ar, const double* __restrict__ av, const int* __restrict__ bp,
                            const int* __restrict__ br, const double* __restrict__ bv, double alpha, double beta,
                            Emit emit, OnCol on_col) {
  long long a0 = __ldg(&ap[c]), b0 = __ldg(&bp[c]);
  long long la = __ldg(&ap[c + 1]) - a0, lb = __ldg(&bp[c + 1]) - b0;
  const long long dl = d0 - (a0 + b0);
  if (dl == 0)  // we own the starts of c and of the empty columns before it sharing the position
    for (long long cc = c; cc >= 0 && mstart_of(ap, bp, cc) == d0; cc--) on_col(cc, 0);
  long long i, j;
  split_at(ar, br, a0, b0, la, lb, dl, &i, &j);
  long long pos = a0 + b0 + i + j;
  int produced = 0;
  while (pos < d1) {
    if (i == la && j == lb) {
      c++;
      a0 = __ldg(&ap[c]);
      b0 = __ldg(&bp[c]);
      la = __ldg(&ap[c + 1]) - a0;
      lb = __ldg(&bp[c + 1]) - b0;
      i = j = 0;
      on_col(c, produced);
      continue;
    }
    int r;
    double v;
    if (j == lb || (i < la && __ldg(&ar[a0 + i]) < __ldg(&br[b0 + j]))) {
      r = __ldg(&ar[a0 + i]);
      v = __dmul_rn(alpha, __ldg(&av[a0 + i]));
      i++;
    } else if (i == la || __ldg(&br[b0 + j]) < __ldg(&ar[a0 + i])) {
      r = __ldg(&br[b0 + j]);
      v = __dmul_rn(beta, __ldg(&bv[b0 + j]));
      j++;
    } else {
      r = __ldg(&ar[a0 + i]);
      v = __dadd_rn(__dmul_rn(alpha, __ldg(&av[a0 + i])), __dmul_rn(beta, __ldg(&bv[b0 + j])));
      i++;
      j++;
    }
    if (v != 0.0) {
      emit(r, v);
      produced++;
    }
    pos = a0 + b0 + i + j;
  }
}

struct AddSmem {
  MergeWindow W;
  int rows[kAddChunk];
  double vals[kAddChunk];
  long long scan_tmp[kMThreads / 32 + 1];
  long long cb;
};

struct AddArgs {
  long long n_cols;
  double alpha, beta;
  const int *ap, *ar, *bp, *br;
  const double *av, *bv;
  int* out_ptr;
  int* out_rows;
  double* out_vals;
  long long* info;
  long long* cta_sums;
  unsigned char* tcount;  // [n_chunks * kMThreads] pass-1 output count of every thread's positions
  GridBar gb;
};

__device__ void ensure_window(AddSmem& S, const AddArgs& a, long long chunk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool inside = S.W.n > 0 && chunk >= S.W.ms[0] && chunk < S.W.ms[S.W.n];
    S.cb = inside ? -1 : col_of_global(a.ap, a.bp, S.W.n > 0 ? S.W.c_base : 0, a.n_cols - 1, chunk);
  }
  __syncthreads();
  if (S.cb >= 0) {
    stage_window(S.W, a.ap, a.bp, a.n_cols, S.cb);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kMThreads) csc_add_kernel(AddArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AddSmem& S = *reinterpret_cast<AddSmem*>(smem_raw);
  const int tid = threadIdx.x;
  unsigned gen = 0;
  const long long M = mstart_of(a.ap, a.bp, a.n_cols);
  const long long per = ((M + gridDim.x - 1) / gridDim.x + kAddChunk - 1) / kAddChunk * kAddChunk;
  const long long lo = min(M, (long long)blockIdx.x * per), hi = min(M, lo + per);
  if (tid == 0) {
    S.W.n = 0;
    S.W.c_base = 0;
  }
  auto no_col = [](long long, int) {};

  // pass 1: count
  long long total = 0;
  for (long long chunk = lo; chunk < hi; chunk += kAddChunk) {
    ensure_window(S, a, chunk);
    const long long d0 = chunk + (long long)tid * kAddItems;
    const long long d1 = min(d0 + kAddItems, min(hi, chunk + kAddChunk));
    int cnt = 0;
    if (d0 < d1)
      merge_range(a.n_cols, col_of(S.W, a.ap, a.bp, a.n_cols, d0), d0, d1, a.ap, a.ar, a.av, a.bp, a.br, a.bv, a.alpha,
                  a.beta, [&](int, double) { cnt++; }, no_col);
    a.tcount[(chunk / kAddChunk) * kMThreads + tid] = (unsigned char)cnt;  // reused by pass 2
    total += block_reduce_sum<long long>((long long)cnt, S.scan_tmp);
  }
  if (tid == 0) a.cta_sums[blockIdx.x] = total;
  grid_sync(a.gb, gen);
  long long pre = 0;
  for (long long q = tid; q < blockIdx.x; q += blockDim.x) pre += a.cta_sums[q];
  pre = block_reduce_sum<long long>(pre, S.scan_tmp);

  // pass 2: write, staged through shared memory
  long long run = pre;
  for (long long chunk = lo; chunk < hi; chunk += kAddChunk) {
    ensure_window(S, a, chunk);
    const long long d0 = chunk + (long long)tid * kAddItems;
    const long long d1 = min(d0 + kAddItems, min(hi, chunk + kAddChunk));
    const long long c0 = d0 < d1 ? col_of(S.W, a.ap, a.bp, a.n_cols, d0) : 0;
    const int cnt = __ldcg(&a.tcount[(chunk / kAddChunk) * kMThreads + tid]);
    long long ctot;
    const long long off = block_exclusive_scan<long long>((long long)cnt, S.scan_tmp, &ctot);
    int w = (int)off;
    if (d0 < d1)
      merge_range(
          a.n_cols, c0, d0, d1, a.ap, a.ar, a.av, a.bp, a.br, a.bv, a.alpha, a.beta,
          [&](int r, double v) {
            S.rows[w] = r;
            S.vals[w] = v;
            w++;
          },
          [&](long long c, int produced) { a.out_ptr[c] = (int)(run + off + produced); });
    __syncthreads();
    for (long long q = tid; q < ctot; q += blockDim.x) {
      a.out_rows[run + q] = S.rows[q];
      a.out_vals[run + q] = S.vals[q];
    }
    run += ctot;
  }
  // columns starting at M (empty trailing ones) and the final offset
  if (blockIdx.x == gridDim.x - 1) {
    __syncthreads();
    if (tid == 0) S.cb = M > 0 ? col_of_global(a.ap, a.bp, 0, a.n_cols - 1, M - 1) + 1 : 0;
    __syncthreads();
    const long long total_all = pre + total;
    for (long long c = S.cb + tid; c <= a.n_cols; c += blockDim.x) a.out_ptr[c] = (int)total_all;
    if (tid == 0) a.info[0] = total_all;
  }
}

static int add_grid() {
  static int grid[kMaxDevices] = {0};  // per device: the attribute and occupancy are per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  if (grid[dev] == 0) {
    int per_sm = 0, sms = 0;
    if (cudaFuncSetAttribute(csc_add_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(AddSmem)) !=
        cudaSuccess)
      return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csc_add_kernel, kMThreads, sizeof(AddSmem));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid[dev] = std::max(1, std::min(per_sm * sms, 148 * 8));
  }
  return grid[dev];
}

}  // namespace as

using namespace as;

extern "C" {

size_t as_add_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b) {
  (void)n_cols;
  const long long n_chunks = (nnz_a + nnz_b + kAddChunk - 1) / kAddChunk;
  return 256 + (size_t)148 * 8 * sizeof(long long) + (size_t)(n_chunks + 1) * kMThreads;
}

int as_csc_add_f64(int64_t n_rows, int64_t n_cols, double alpha, double beta, const int32_t* a_col_ptr,
                   const int32_t* a_row_idx, const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx,
                   const double* b_vals, int64_t nnz_a, int64_t nnz_b, int32_t* col_ptr, int32_t* row_idx,
                   double* out_vals, int64_t* info, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n_rows >= 0 && n_cols >= 0, AS_ERR_SHAPE, "negative dimension");
  AS_REQUIRE(nnz_a + nnz_b <= 0x7fffffffll, AS_ERR_ARG, "nnz outside the int32 range");
  AS_REQUIRE(ws_bytes >= as_add_workspace_bytes(n_cols, nnz_a, nnz_b), AS_ERR_ARG, "workspace too small");
  const int grid = add_grid();
  AS_REQUIRE(grid > 0, AS_ERR_CUDA, "cannot configure the add kernel");
  AS_CUDA_TRY(cudaMemsetAsync(ws, 0, 256, st));
  AddArgs a;
  a.n_cols = n_cols;
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
  a.cta_sums = (long long*)((char*)ws + 256);
  a.tcount = (unsigned char*)(a.cta_sums + 148 * 8);
  a.gb = GridBar{(unsigned*)ws, (unsigned*)ws + 32};
  void* args[] = {(void*)&a};
  AS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)csc_add_kernel, dim3(grid), dim3(kMThreads), args,
                                          sizeof(AddSmem), st));
  return AS_OK;
}

}  // extern "C"
