// mg.cu -- multi-GPU entry points of the C ABI: the
// column-sharded trace(A^T B), SpMM and SpGEMM as ONE call each -- the rank-local
// kernel followed by its NCCL collective on the caller's stream -- for a host
// that does not go through torch.distributed (paper_1805_03380_b200/dist.py
// is the Python twin and the reference for the combination order).
//
// One process per GPU.  The caller owns the communicator (ncclCommInitRank,
// or the one its framework created) and hands it to as_mg_init; the library
// resolves NCCL's entry points at run time from the libnccl the process has
// loaded (dlopen by soname, RTLD_NOLOAD first), so libbsparse.so carries no
// link-time dependency on a particular NCCL.  The reference has no multi-GPU
// path; the single-GPU results are the oracle (the sharded trace combines the
// ranks' double-double partials in rank order, so it does not depend on the
// reduction tree; the SpMM blocks are disjoint columns of C).
#include <dlfcn.h>

#include "capi_util.cuh"
#include "common.cuh"

namespace as {

namespace {

// the few NCCL entry points used (nccl.h: ncclResult_t is an int enum,
// ncclSuccess = 0; ncclInt64 = 4, ncclFloat32 = 7, ncclFloat64 = 8)
using nccl_all_gather_t = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
using nccl_error_string_t = const char* (*)(int);
constexpr int kNcclInt64 = 4, kNcclFloat32 = 7, kNcclFloat64 = 8;

struct MgState {
  void* lib = nullptr;
  nccl_all_gather_t all_gather = nullptr;
  nccl_error_string_t error_string = nullptr;
  void* comm = nullptr;
  int rank = -1, world = 0;
};
MgState g_mg;

bool resolve_nccl(const char* path) {
  if (g_mg.all_gather) return true;
  const char* names[] = {path, "libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    if (!n || !*n) continue;
    void* h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);  // the copy the process already runs on
    if (!h) h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    if (!h) continue;
    auto ag = (nccl_all_gather_t)dlsym(h, "ncclAllGather");
    if (!ag) {
      dlclose(h);
      continue;
    }
    g_mg.lib = h;
    g_mg.all_gather = ag;
    g_mg.error_string = (nccl_error_string_t)dlsym(h, "ncclGetErrorString");
    return true;
  }
  return false;
}

// gathered[r] = (hi, lo) of rank r: summed in rank order with TwoSum carries
// (dist.dd_combine), out[0] = the sum, out[1] = its residual
__global__ void mg_dd_combine_kernel(const double* __restrict__ gathered, int world, double* __restrict__ out) {
  double s = 0.0, e = 0.0;
  for (int r = 0; r < world; r++) {
    const double hi = gathered[2 * r], lo = gathered[2 * r + 1];
    e = __dadd_rn(e, lo);
    const double t = __dadd_rn(s, hi);
    const double bp = __dsub_rn(t, s);
    const double err = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(hi, bp));
    s = t;
    e = __dadd_rn(e, err);
  }
  const double total = __dadd_rn(s, e);
  out[0] = total;
  out[1] = __dsub_rn(e, __dsub_rn(total, s));
}

// this rank's first element in the concatenation of the ranks' slices
__global__ void mg_slice_offset_kernel(const long long* __restrict__ slice_nnz, int rank, long long* __restrict__ off) {
  long long s = 0;
  for (int r = 0; r < rank; r++) s += slice_nnz[r];
  off[0] = s;
}

constexpr size_t kMgSlots = 256;  // bytes reserved for one rank's partial in front of the gather buffer

}  // namespace

}  // namespace as

using namespace as;

#define AS_NCCL_TRY(expr)                                                                             \
  do {                                                                                                \
    const int _r = (expr);                                                                            \
    if (_r != 0) {                                                                                    \
      ::as::set_error("%s:%d %s: NCCL error %d (%s)", __FILE__, __LINE__, #expr, _r,                  \
                      g_mg.error_string ? g_mg.error_string(_r) : "?");                               \
      return AS_ERR_CUDA;                                                                             \
    }                                                                                                 \
  } while (0)

extern "C" {

int as_mg_init(void* nccl_comm, int rank, int world, const char* nccl_library) {
  AS_REQUIRE(nccl_comm != nullptr, AS_ERR_ARG, "null NCCL communicator");
  AS_REQUIRE(world >= 1 && rank >= 0 && rank < world, AS_ERR_ARG, "rank %d outside a world of %d", rank, world);
  if (!resolve_nccl(nccl_library)) {
    const char* why = dlerror();
    ::as::set_error("cannot resolve ncclAllGather: libnccl.so.2 is not loadable (%s)", why ? why : "no message");
    return AS_ERR_ARG;
  }
  g_mg.comm = nccl_comm;
  g_mg.rank = rank;
  g_mg.world = world;
  return AS_OK;
}

int as_mg_shutdown(void) {
  g_mg.comm = nullptr;  // the communicator stays the caller's
  g_mg.rank = -1;
  g_mg.world = 0;
  return AS_OK;
}

int as_mg_rank(void) { return g_mg.rank; }
int as_mg_world(void) { return g_mg.world; }

size_t as_mg_trace_workspace_bytes(int64_t n_cols, int64_t nnz_a, int64_t nnz_b, int world) {
  return ((as_trace_workspace_bytes(n_cols, nnz_a, nnz_b) + 255) & ~(size_t)255) + kMgSlots +
         (size_t)std::max(world, 1) * 2 * sizeof(double);
}

int as_mg_trace_atb_f64(int64_t n_rows, int64_t n_cols, const int32_t* a_col_ptr, const int32_t* a_row_idx,
                        const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx, const double* b_vals,
                        int64_t nnz_a, int64_t nnz_b, int64_t c0, int64_t c1, double* out, void* ws, size_t ws_bytes,
                        void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(g_mg.comm != nullptr, AS_ERR_ARG, "as_mg_init has not been called");
  AS_REQUIRE(0 <= c0 && c0 <= c1 && c1 <= n_cols, AS_ERR_SHAPE, "column range [%lld, %lld) outside %lld columns",
             (long long)c0, (long long)c1, (long long)n_cols);
  AS_REQUIRE(ws_bytes >= as_mg_trace_workspace_bytes(n_cols, nnz_a, nnz_b, g_mg.world), AS_ERR_ARG,
             "workspace too small");
  const size_t tw = (as_trace_workspace_bytes(n_cols, nnz_a, nnz_b) + 255) & ~(size_t)255;
  double* part = (double*)((char*)ws + tw);
  double* gathered = (double*)((char*)ws + tw + kMgSlots);
  // the rank's columns: the column pointers are absolute entry positions, so
  // the slice is the same arrays entered at column c0
  const int rc = as_trace_atb_f64(n_rows, c1 - c0, a_col_ptr + c0, a_row_idx, a_vals, b_col_ptr + c0, b_row_idx,
                                  b_vals, nnz_a, nnz_b, part, ws, tw, stream);
  if (rc != AS_OK) return rc;
  AS_NCCL_TRY(g_mg.all_gather(part, gathered, 2, kNcclFloat64, g_mg.comm, st));
  mg_dd_combine_kernel<<<1, 1, 0, st>>>(gathered, g_mg.world, out);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

int as_mg_spmm_csr_f32(int64_t n_rows, int64_t n_cols, int64_t k, const int32_t* row_ptr, const int32_t* col_idx,
                       const float* vals, const float* B, int64_t ldb, float* C, int64_t ldc, void* ws, size_t ws_bytes,
                       void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(g_mg.comm != nullptr, AS_ERR_ARG, "as_mg_init has not been called");
  AS_REQUIRE(k >= 0 && k % g_mg.world == 0, AS_ERR_SHAPE, "%lld dense columns do not split evenly over %d ranks",
             (long long)k, g_mg.world);
  AS_REQUIRE(ldc == n_rows, AS_ERR_SHAPE, "C must be packed (ldc == n_rows): a rank's block is one contiguous run");
  const int64_t kb = k / g_mg.world, k0 = kb * g_mg.rank;
  if (kb == 0) return AS_OK;
  // the rank's block of dense columns: A (its CSR) is replicated
  const int rc = as_spmm_csr_f32(n_rows, n_cols, kb, row_ptr, col_idx, vals, B + k0 * ldb, ldb, C + k0 * ldc, ldc, 0, ws,
                                 ws_bytes, stream);
  if (rc != AS_OK) return rc;
  // in place: every rank's block lands in the same columns of every C
  AS_NCCL_TRY(g_mg.all_gather(C + k0 * ldc, C, (size_t)(kb * ldc), kNcclFloat32, g_mg.comm, st));
  return AS_OK;
}

int as_mg_spgemm_f64(int64_t n_rows_a, int64_t n_inner, int64_t n_cols_b, const int32_t* a_col_ptr,
                     const int32_t* a_row_idx, const double* a_vals, const int32_t* b_col_ptr, const int32_t* b_row_idx,
                     const double* b_vals, int64_t nnz_b, const int64_t* prod_ptr, int64_t total_products,
                     int32_t* col_ptr, int32_t* row_idx, double* out_vals, int64_t* info, void* ws, size_t ws_bytes,
                     int64_t* slice_nnz, int64_t* slice_offset, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(g_mg.comm != nullptr, AS_ERR_ARG, "as_mg_init has not been called");
  AS_REQUIRE(slice_nnz != nullptr && slice_offset != nullptr, AS_ERR_ARG, "null slice_nnz / slice_offset");
  // the rank's column slice of B (a standalone CSC: dist.spgemm_shard cuts B into
  // ranges of equal Gustavson products); A is replicated
  const int rc = as_spgemm_f64(n_rows_a, n_inner, n_cols_b, a_col_ptr, a_row_idx, a_vals, b_col_ptr, b_row_idx, b_vals,
                               nnz_b, prod_ptr, total_products, col_ptr, row_idx, out_vals, info, ws, ws_bytes, stream);
  if (rc != AS_OK) return rc;
  // C stays distributed: one all-gather of the slices' nnz (info[0], still on the
  // device), each rank's global element offset by a scan in rank order
  AS_NCCL_TRY(g_mg.all_gather(info, slice_nnz, 1, kNcclInt64, g_mg.comm, st));
  mg_slice_offset_kernel<<<1, 1, 0, st>>>((const long long*)slice_nnz, g_mg.rank, (long long*)slice_offset);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

}  // extern "C"
