// largen.cu -- host side of the large-input pipeline (largen.cuh):
// applicability, bucket plan, workspace, launch sequence; instantiations for
// construction and transpose.
#include <stdlib.h>

#include <algorithm>

#include "capi_util.cuh"
#include "largen.cuh"
#include "largen_api.h"

namespace as {
namespace ln {

constexpr long long kMaxBuckets = (long long)kR * kR;
static const double kFill = getenv("AS_LN_FILL") ? atof(getenv("AS_LN_FILL")) : 0.85;  // mean bucket size / tile

struct Plan {
  bool ok = false;
  long long nb = 0, T_ = 0;
  int lob = 0;
  unsigned long long cb_mul = 0;
};

static Plan plan(long long n, long long n_out_cols, int mb) {
  Plan p;
  if (n <= 0 || n_out_cols <= 0 || mb > 31) return p;
  long long nb = (long long)((double)n / (kFill * sr::kTile)) + 1;
  nb = std::max(nb, (n_out_cols + (sr::kMaxW - 24) - 1) / (sr::kMaxW - 24));
  // the bucket-local key (column within the bucket << mb | minor) must fit 32 bits
  while (nb < n_out_cols && bits_for((n_out_cols + nb - 1) / nb) + mb > 32) nb *= 2;
  nb = std::min(nb, n_out_cols);
  if (nb > kMaxBuckets) return p;
  const long long max_w = (n_out_cols + nb - 1) / nb + 1;
  if (max_w > sr::kMaxW || bits_for(max_w - 1) + mb > 32) return p;
  p.ok = true;
  p.nb = nb;
  // two passes: the bucket id's bits split evenly between the low digit (pass A) and the
  // high digit (pass B), so both passes scatter runs of similar length (with a fixed 8-bit
  // low digit, 1e7 elements over 5,747 buckets gave pass A runs of 8 elements -- 9.4 store
  // sectors per request -- and pass B runs of 89; build 1e7 473 -> 461 us, transpose 5e7
  // 1.89 -> 1.83 ms)
  static const int kLobEnv = getenv("AS_LN_LOB") ? atoi(getenv("AS_LN_LOB")) : 0;
  const int bits = bits_for(nb - 1);
  int lob = kLobEnv > 0 ? kLobEnv : bits / 2;
  lob = std::min(8, std::max(lob, bits - 8));
  p.lob = nb <= kR ? 0 : lob;
  p.T_ = (n + kE - 1) / kE;
  p.cb_mul = (unsigned long long)((((unsigned __int128)nb) << 32) / (unsigned long long)n_out_cols);
  return p;
}

template <class T>
struct Ws {
  // zeroed region
  unsigned long long* st_a;
  unsigned long long* st_b;
  unsigned long long* st_c;
  unsigned* tickets;  // [3]
  unsigned* bcnt;
  unsigned long long* tstate;
  unsigned long long* ctr1;
  char* z_end;
  // 0xff
  unsigned long long* bad;
  // not initialised
  unsigned* H;
  unsigned* cbcol;
  unsigned* tile_col;
  long long* own_info;
  unsigned* aM;
  unsigned* aN;
  T* aV;
  unsigned* bK;
  T* bV;
  unsigned long long* oK;
  unsigned long long* oK2;
  unsigned* oP;
  unsigned* oP2;
  int* oR;
  T* oV;
};

template <class T>
static size_t carve(Carve& c, Ws<T>* w, long long n, long long nb, long long T_) {
  const long long n1 = std::max(1ll, n);
  const long long hs = (long long)kR * std::max(1ll, T_);
  const long long nsa = hs / kScanN + 2, nsc = (nb + 1) / kScanN + 2;
  w->st_a = c.take<unsigned long long>(nsa);
  w->st_b = c.take<unsigned long long>(nsa);
  w->st_c = c.take<unsigned long long>(nsc);
  w->tickets = c.take<unsigned>(4);
  w->bcnt = c.take<unsigned>(nb + 1);
  w->tstate = c.take<unsigned long long>(nb + 1);
  w->ctr1 = c.take<unsigned long long>(1);
  w->z_end = c.base ? c.base + c.off : nullptr;
  w->bad = c.take<unsigned long long>(1);
  w->H = c.take<unsigned>(hs);
  w->cbcol = c.take<unsigned>(nb + 1);
  w->tile_col = c.take<unsigned>(std::max(1ll, T_) + 1);
  w->own_info = c.take<long long>(2);
  w->aM = c.take<unsigned>(n1);
  w->aN = c.take<unsigned>(n1);
  w->aV = c.take<T>(n1);
  w->bK = c.take<unsigned>(n1);
  w->bV = c.take<T>(n1);
  w->oK = c.take<unsigned long long>(n1);
  w->oK2 = c.take<unsigned long long>(n1);
  w->oP = c.take<unsigned>(n1);
  w->oP2 = c.take<unsigned>(n1);
  w->oR = c.take<int>(n1);
  w->oV = c.take<T>(n1);
  return c.off;
}

size_t ws_bytes(long long n, long long n_out_cols, size_t val_bytes) {
  // bucket count bound: the plan's nb never exceeds kMaxBuckets
  const long long nb = kMaxBuckets;
  const long long T_ = (n + kE - 1) / kE;
  Carve c(nullptr, 0);
  if (val_bytes == 8) {
    Ws<double> w;
    return carve(c, &w, n, nb, T_);
  }
  Ws<float> w;
  return carve(c, &w, n, nb, T_);
}

bool disabled() {
  static const bool off = getenv("AS_NO_LN") != nullptr;
  return off;
}

// co-resident grid of the tile kernel (per device, cached)
template <class T>
static int tiles_grid() {
  static std::atomic<int> grid[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  if (grid[dev] == 0) {
    const int smem = (int)sizeof(sr::TileSmem<T>);
    if (cudaFuncSetAttribute(ln_tiles_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return 0;
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ln_tiles_kernel<T>, sr::kThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    grid[dev] = std::min(per_sm, sr::kMinBlocks) * sms;
  }
  return grid[dev];
}

template <class T, class In, int kPass>
static int scatter_launch(const Args<T>& a, const In& src, cudaStream_t st) {
  static std::atomic<bool> attr[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  const int smem = (int)sizeof(ScatterSmem<T, In, kPass>);
  if (dev >= 0 && dev < kMaxDevices && !attr[dev]) {
    AS_CUDA_TRY(cudaFuncSetAttribute(ln_scatter_kernel<T, In, kPass>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
    attr[dev] = true;
  }
  ln_scatter_kernel<T, In, kPass><<<(unsigned)a.T_, kT, smem, st>>>(a, src);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

static int scan_launch(unsigned* x, long long n, unsigned* total, unsigned long long* states, unsigned* ticket,
                       cudaStream_t st) {
  const long long tiles = std::max(1ll, (n + kScanN - 1) / kScanN);
  ln_scan_kernel<<<(unsigned)tiles, kScanT, 0, st>>>(x, n, total, states, ticket);
  AS_LAUNCH_CHECK();
  return AS_OK;
}

// The whole pipeline.  Returns AS_OK after launching, -1 when outside the
// envelope (the caller falls back to the general bucket kernel).
template <class T>
static int prepare(CscIn<T>& s, const Ws<T>& w, cudaStream_t st) {
  s.tile_col = w.tile_col;
  if (s.n_cols > 0) {
    ln_tile_col_kernel<<<(unsigned)((s.n_cols + 255) / 256), 256, 0, st>>>(s.ptr, s.n_cols, s.nnz, w.tile_col);
    AS_LAUNCH_CHECK();
  }
  return AS_OK;
}
template <class T, class IdxT>
static int prepare(CooIn<IdxT, T>&, const Ws<T>&, cudaStream_t) {
  return AS_OK;
}

template <class T, class In>
static int run(In src, long long n, long long n_out_cols, int mb, long long n_minor, int mode, int prune, int* col_ptr,
               int* row_idx, T* out_vals, long long* info, void* ws, size_t ws_bytes, cudaStream_t st,
               bool transpose_finish = false) {
  if (disabled()) return -1;
  const Plan p = plan(n, n_out_cols, mb);
  if (!p.ok) return -1;
  const int grid = tiles_grid<T>();
  if (grid <= 0) return -1;
  Carve c(ws, ws_bytes);
  Ws<T> w;
  carve(c, &w, n, p.nb, p.T_);
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  AS_CUDA_TRY(cudaMemsetAsync(w.st_a, 0, (size_t)(w.z_end - (char*)w.st_a), st));
  AS_CUDA_TRY(cudaMemsetAsync(w.bad, 0xff, sizeof(unsigned long long), st));
  ln_cbcol_kernel<<<(unsigned)((p.nb + 1 + 255) / 256), 256, 0, st>>>(w.cbcol, p.nb, p.cb_mul, n_out_cols);
  AS_LAUNCH_CHECK();
  if (int rc = prepare(src, w, st)) return rc;
  Args<T> a;
  a.n = n;
  a.T_ = p.T_;
  a.n_out_cols = n_out_cols;
  a.mb = mb;
  a.lob = p.lob;
  a.nb = p.nb;
  a.cb_mul = p.cb_mul;
  a.inv_cb = p.cb_mul ? 1.0 / (double)p.cb_mul : 0.0;
  a.H = w.H;
  a.bcnt = w.bcnt;
  a.cbcol = w.cbcol;
  a.bad = w.bad;
  a.aM = w.aM;
  a.aN = w.aN;
  a.aV = w.aV;
  a.bK = w.bK;
  a.bV = w.bV;
  const long long hs = (long long)kR * p.T_;
  if (p.lob > 0) {
    ln_count_kernel<T, In, 0><<<(unsigned)p.T_, kT, 0, st>>>(a, src);
    AS_LAUNCH_CHECK();
    if (int rc = scan_launch(w.H, hs, nullptr, w.st_a, w.tickets + 0, st)) return rc;
    if (int rc = scatter_launch<T, In, 0>(a, src, st)) return rc;
    RecIn<T> ra{w.aM, w.aN, w.aV};
    ln_count_kernel<T, RecIn<T>, 1><<<(unsigned)p.T_, kT, 0, st>>>(a, ra);
    AS_LAUNCH_CHECK();
    if (int rc = scan_launch(w.H, hs, nullptr, w.st_b, w.tickets + 1, st)) return rc;
    if (int rc = scan_launch(w.bcnt, p.nb, w.bcnt + p.nb, w.st_c, w.tickets + 2, st)) return rc;
    if (int rc = scatter_launch<T, RecIn<T>, 1>(a, ra, st)) return rc;
  } else {
    ln_count_kernel<T, In, 2><<<(unsigned)p.T_, kT, 0, st>>>(a, src);
    AS_LAUNCH_CHECK();
    if (int rc = scan_launch(w.H, hs, nullptr, w.st_a, w.tickets + 0, st)) return rc;
    if (int rc = scan_launch(w.bcnt, p.nb, w.bcnt + p.nb, w.st_c, w.tickets + 2, st)) return rc;
    if (int rc = scatter_launch<T, In, 2>(a, src, st)) return rc;
  }
  if (mode == kLast && !prune && transpose_finish) {  // every element kept, no duplicates: no sort
    static std::atomic<bool> attr[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    const int smem = (int)sizeof(FinishSmem<T>);
    if (dev >= 0 && dev < kMaxDevices && !attr[dev]) {
      AS_CUDA_TRY(cudaFuncSetAttribute(ln_transpose_finish_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem));
      attr[dev] = true;
    }
    const int blocks = (int)std::min<long long>(p.nb, 148ll * 3 * 4);
    ln_transpose_finish_kernel<T><<<blocks, kT, smem, st>>>(p.nb, w.bcnt, w.bK, w.bV, w.cbcol, mb, n_out_cols,
                                                           col_ptr, row_idx, out_vals, info);
    AS_LAUNCH_CHECK();
    return AS_OK;
  }
  SegLN<T> sg{w.bcnt, w.bK, w.bV, w.cbcol, w.tstate};
  sr::TileOut<T> o;
  o.mode = mode;
  o.prune = prune;
  o.mb = mb;
  o.n_minor = n_minor;
  o.idx_bits = bits_for(n > 0 ? n - 1 : 0);
  o.stop = 0;
  o.n_out_cols = n_out_cols;
  o.col_ptr = col_ptr;
  o.row_idx = row_idx;
  o.out_vals = out_vals;
  o.info = info ? info : w.own_info;
  o.ctr1 = w.ctr1;
  o.oK = w.oK;
  o.oK2 = w.oK2;
  o.oP = w.oP;
  o.oP2 = w.oP2;
  o.oR = w.oR;
  o.oV = w.oV;
  o.phase_ts = nullptr;
  const unsigned long long* bad = w.bad;
  long long nb = p.nb;
  void* args[] = {(void*)&sg, (void*)&o, (void*)&nb, (void*)&bad, (void*)&n};
  AS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)ln_tiles_kernel<T>, dim3(grid), dim3(sr::kThreads), args,
                                          sizeof(sr::TileSmem<T>), st));
  return AS_OK;
}

template <class T, class IdxT>
int coo_to_csc(long long n_rows, long long n_cols, long long n, const IdxT* rows, const IdxT* cols, const T* vals,
               int mode, int* col_ptr, int* row_idx, T* out_vals, long long* info, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  return run<T>(CooIn<IdxT, T>{rows, cols, vals, n, n_rows, n_cols}, n, n_cols,
                bits_for(n_rows > 0 ? n_rows - 1 : 0), n_rows, mode, 1, col_ptr, row_idx, out_vals, info, ws, ws_bytes,
                st);
}

template <class T>
int transpose(long long n_rows, long long n_cols, long long nnz, const int* col_ptr, const int* row_idx,
              const T* vals, int* t_col_ptr, int* t_row_idx, T* t_vals, void* ws, size_t ws_bytes, cudaStream_t st) {
  static const bool generic = getenv("AS_LN_GENERIC_TRANSPOSE") != nullptr;  // A/B: tile-phase finish
  return run<T>(CscIn<T>{col_ptr, row_idx, vals, n_cols, nnz, nullptr}, nnz, n_rows, bits_for(n_cols > 0 ? n_cols - 1 : 0),
                n_cols, kLast, 0, t_col_ptr, t_row_idx, t_vals, nullptr, ws, ws_bytes, st, !generic);
}

template int coo_to_csc<double, int>(long long, long long, long long, const int*, const int*, const double*, int, int*,
                                     int*, double*, long long*, void*, size_t, cudaStream_t);
template int coo_to_csc<double, long long>(long long, long long, long long, const long long*, const long long*,
                                           const double*, int, int*, int*, double*, long long*, void*, size_t,
                                           cudaStream_t);
template int coo_to_csc<float, int>(long long, long long, long long, const int*, const int*, const float*, int, int*,
                                    int*, float*, long long*, void*, size_t, cudaStream_t);
template int coo_to_csc<float, long long>(long long, long long, long long, const long long*, const long long*,
                                          const float*, int, int*, int*, float*, long long*, void*, size_t,
                                          cudaStream_t);
template int transpose<double>(long long, long long, long long, const int*, const int*, const double*, int*, int*,
                               double*, void*, size_t, cudaStream_t);
template int transpose<float>(long long, long long, long long, const int*, const int*, const float*, int*, int*,
                              float*, void*, size_t, cudaStream_t);

}  // namespace ln
}  // namespace as
