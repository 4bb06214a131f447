// persist_host.cuh -- host side of the persistent bucket-sort kernel:
// workspace carving, coarse-bucket sizing, cooperative launch.
#pragma once

#include <stdlib.h>

#include "capi_util.cuh"
#include "persist.cuh"

namespace as {

constexpr long long kMaxDim = 0x7fffffffll;
constexpr long long kMaxGrid = 148 * 8;  // upper bound of the co-resident grid

struct PersistWs {
  long long dense_rows = 0;  // pre mode: rows of the output (dense column path when they fit)
  unsigned* zero;  // [0] ticket, [16] barrier arrive, [32] barrier generation, then cb_cnt
  unsigned* cb_cnt;
  size_t zero_bytes;
  long long* cb_start;
  unsigned long long* keys;
  unsigned long long* keys_alt;
  unsigned* colb;
  unsigned* colb_alt;
  void* vals_b;
  int* tmp_rows;
  void* tmp_vals;
  unsigned* col_kept;
  long long* cta_sums;
  long long* own_info;
  unsigned* cb_col;  // [n_cb + 1] first column of each bucket
  unsigned* order;   // pre-bucketed input only
  unsigned long long* tstate;
  int sb_f;          // two-level scatter (sb_f > 1)
  long long n_sb;
  unsigned* sb_cnt;
  unsigned* sb_fill;
  void* vals_alt;
  unsigned long long cb_mul;
  bool ok;           // the column count is supported
  long long n_cb;
};

// Coarse buckets of ~n_cols / n_cb consecutive output columns (bucket(c) =
// (c * cb_mul) >> 32).  n_cb: ~0.9 * kCap elements per bucket on average,
// rounded up to whole waves of the co-resident grid (SMs x AS_PERSIST_MINB
// CTAs) when above one wave, so the tile phase has no half-empty last wave
// (AS_FILL / AS_WAVES override, for sweeps); at least n_cols / kMaxBucketCols
// (a bucket's columns index shared arrays), at most kMaxCoarse.  Returns 0
// when the column count exceeds kMaxCoarse * kMaxBucketCols.
constexpr long long kMaxBucketCols = kMaxW - 24;

static inline long long choose_ncb(long long n, long long n_cols) {
  static const double kFill = getenv("AS_FILL") ? atof(getenv("AS_FILL")) : 0.9;
  const long long wave = (long long)num_sms() * AS_PERSIST_MINB;
  long long nb = (long long)((double)n / (kFill * kCap)) + 1;
  static const int kWaves = getenv("AS_WAVES") ? atoi(getenv("AS_WAVES")) : 1;
  if (kWaves == 2 || (kWaves == 1 && nb > wave)) nb = (nb + wave - 1) / wave * wave;
  nb = std::max(nb, (n_cols + kMaxBucketCols - 1) / kMaxBucketCols);
  nb = std::min(nb, std::max(1ll, n_cols));
  nb = std::min(nb, (long long)kMaxCoarse);
  if (n_cols > 0 && (n_cols + nb - 1) / nb > kMaxBucketCols) return 0;
  return std::max(1ll, nb);
}

// pre = true: the input arrives bucketed by column (run_persist_ws pre_ptr);
// buckets are then variable-width (kPreT), with no column-count limit.
static size_t carve_persist(Carve& c, PersistWs* w, long long n, long long n_cols, size_t val_bytes,
                            bool pre = false) {
  w->cb_mul = 0;
  w->ok = true;
  if (pre) {
    w->n_cb = (n + kPreColCost * n_cols) / kPreT + 1;
  } else {
    w->n_cb = choose_ncb(n, n_cols);
    w->ok = w->n_cb > 0;
    if (!w->ok) w->n_cb = 1;
    // floor(2^32 * n_cb / n_cols): bucket(n_cols - 1) < n_cb
    w->cb_mul = n_cols > 0 ? (unsigned long long)((((unsigned __int128)w->n_cb) << 32) / (unsigned long long)n_cols) : 0;
  }
  w->zero = c.take<unsigned>(64);
  w->cb_cnt = c.take<unsigned>(std::max(1ll, w->n_cb));  // pre: size class and slot of each bucket
  // bucket states, then one word per group of 32 buckets (group_lookback_warp)
  w->tstate = c.take<unsigned long long>(std::max(1ll, w->n_cb) + (w->n_cb + 31) / 32 + 1);
  // two-level scatter when the scattered element data outgrows L2 and a
  // (CTA, bucket) run would be short: super-buckets of sb_f buckets so a
  // (CTA, super-bucket) run averages >= 32 elements
  w->sb_f = 1;
  if (!pre && w->ok && n * (long long)(12 + val_bytes) > (48ll << 20)) {
    // (CTA, super-bucket) runs of >= ~256 elements; <= 4096 buckets each
    const long long max_sb = std::max(1ll, n / (256ll * kMaxGrid / 2));
    const long long f = std::min(4096ll, (w->n_cb + max_sb - 1) / max_sb);
    if (f >= 2) w->sb_f = (int)f;
  }
  w->n_sb = (w->n_cb + w->sb_f - 1) / w->sb_f;
  w->sb_cnt = c.take<unsigned>(std::max(1ll, w->n_sb));
  w->sb_fill = c.take<unsigned>(w->sb_f > 1 ? w->n_cb : 1);
  w->zero_bytes = c.off;
  w->cb_start = c.take<long long>(w->n_cb + 1);
  w->cb_col = c.take<unsigned>(w->n_cb + 1);
  w->order = pre ? c.take<unsigned>(w->n_cb) : nullptr;
  const long long n1 = std::max(1ll, n);
  w->keys = c.take<unsigned long long>(n1);
  w->keys_alt = c.take<unsigned long long>(n1);
  w->colb = c.take<unsigned>(n1);
  w->colb_alt = c.take<unsigned>(n1);
  w->vals_b = (void*)c.take<char>(n1 * val_bytes);
  w->tmp_rows = c.take<int>(n1);
  w->tmp_vals = (void*)c.take<char>(n1 * val_bytes);
  w->col_kept = c.take<unsigned>(std::max(1ll, n_cols));
  w->cta_sums = c.take<long long>(kMaxGrid);
  w->own_info = c.take<long long>(2);
  w->vals_alt = w->sb_f > 1 ? (void*)c.take<char>(n1 * (long long)val_bytes) : nullptr;
  return c.off;
}

template <class T, class S1, class S2, bool kTwo>
static int launch_persist_k(PersistArgs<T, S1, S2>& a, cudaStream_t st) {
  static std::atomic<int> grid_of[kMaxDevices];  // per device: the attribute and occupancy are per device
  const size_t smem = sizeof(PersistSmem<T>);
  auto kern = persist_bucket_kernel<T, S1, S2, kTwo>;
  int dev = 0;
  AS_CUDA_TRY(cudaGetDevice(&dev));
  AS_REQUIRE(dev >= 0 && dev < kMaxDevices, AS_ERR_CUDA, "device ordinal %d beyond %d", dev, kMaxDevices);
  if (grid_of[dev] == 0) {
    AS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, sms = 0;
    AS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSegThreads, smem));
    AS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    AS_REQUIRE(per_sm > 0, AS_ERR_CUDA, "persistent kernel does not fit on an SM");
    grid_of[dev] = (int)std::min<long long>((long long)per_sm * sms, kMaxGrid);
  }
  const int grid = grid_of[dev];
  // staged scatter when the largest CTA chunk of the two sources fits
  auto chunk = [&](long long n) -> long long { return (((n + grid - 1) / grid) + 3) & ~3ll; };
  long long st_off;
  a.stage = (!kTwo && a.n_cb <= kMaxCoarse && a.s1.size() + a.s2.size() > 0 &&
             chunk(a.s1.size()) + chunk(a.s2.size()) <= stage_layout<T>(a.n_cb, &st_off))
                ? 1
                : 0;
  static const bool kNoStage = getenv("AS_NO_STAGE") != nullptr;
  if (kNoStage) a.stage = 0;
  // without the staging only the tile / the [3 * n_cb] arrays are needed: the
  // rest of the 256 KB goes back to L1 (the pre-bucketed SpGEMM tiles gather
  // through it)
  constexpr bool kPre = std::is_same<S1, NoSrc<T>>::value && std::is_same<S2, NoSrc<T>>::value;
  const size_t need = kPre ? std::max(sizeof(BTileSmem<T>), (size_t)(a.dense_rows ? dense_column_bytes(a.dense_rows) : 0))
                      : a.stage ? smem
                                : std::max(sizeof(BTileSmem<T>),
                                           (size_t)(((long long)sizeof(int) * (kColCache + 1) + 12ll * a.n_cb + 15) & ~15ll));
  void* args[] = {(void*)&a};
  AS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSegThreads), args, std::min(need, smem),
                                          st));
  return AS_OK;
}

template <class T, class S1, class S2>
static int launch_persist(PersistArgs<T, S1, S2>& a, cudaStream_t st) {
  constexpr bool kPre = std::is_same<S1, NoSrc<T>>::value && std::is_same<S2, NoSrc<T>>::value;
  if constexpr (!kPre) {
    if (a.sb_f > 1) return launch_persist_k<T, S1, S2, true>(a, st);
  }
  return launch_persist_k<T, S1, S2, false>(a, st);
}

// Launch the persistent kernel on an already carved workspace.  pre_ptr !=
// nullptr: w.keys / w.colb / w.vals_b already hold the input bucketed by
// output column (pre_ptr = its column pointer, n elements).
template <class T, class S1, class S2>
static int run_persist_ws(PersistWs& w, const S1& s1, const S2& s2, long long n, long long n_cols, int row_bits,
                          int mode, int prune, ValSrc<T> vs, int* col_ptr, int* row_idx, T* out_vals,
                          long long* info, bool init_info, const long long* pre_ptr, cudaStream_t st) {
  AS_REQUIRE(w.ok, AS_ERR_ARG, "%lld output columns exceed the %lld supported by the bucket kernel", n_cols,
             (long long)kMaxCoarse * kMaxBucketCols);
  if (info == nullptr) info = w.own_info;
  AS_CUDA_TRY(cudaMemsetAsync(w.zero, 0, w.zero_bytes, st));
  if (init_info) AS_CUDA_TRY(cudaMemsetAsync(info, 0x7f, 2 * sizeof(long long), st));
  PersistArgs<T, S1, S2> a;
  a.s1 = s1;
  a.s2 = s2;
  a.n_cols = n_cols;
  a.n_upper = n;
  a.cb_mul = w.cb_mul;
  a.n_cb = w.n_cb;
  a.cb_cnt = w.cb_cnt;
  a.cb_start = w.cb_start;
  a.keys = w.keys;
  a.keys_alt = w.keys_alt;
  a.colb = w.colb;
  a.colb_alt = w.colb_alt;
  a.vals_b = (T*)w.vals_b;
  a.tmp_rows = w.tmp_rows;
  a.tmp_vals = (T*)w.tmp_vals;
  a.col_kept = w.col_kept;
  a.cta_sums = w.cta_sums;
  a.row_bits = row_bits;
  a.idx_bits = bits_for(n > 0 ? n - 1 : 0);
  a.mode = mode;
  a.prune = prune;
  a.vs = vs;
  a.col_ptr = col_ptr;
  a.row_idx = row_idx;
  a.out_vals = out_vals;
  a.info = info;
  a.ticket = w.zero;
  a.gb = GridBar{w.zero + 16, w.zero + 32};
  a.phase_ts = nullptr;
  a.pre_ptr = pre_ptr;
  a.cb_col = w.cb_col;
  a.order = pre_ptr ? w.order : nullptr;
  a.tstate = w.tstate;
  a.sb_f = w.sb_f;
  a.n_sb = w.n_sb;
  a.sb_cnt = w.sb_cnt;
  a.sb_fill = w.sb_fill;
  a.vals_alt = (T*)w.vals_alt;
  a.dense_rows = (pre_ptr && dense_column_bytes(w.dense_rows) <= (long long)kPersistSmemBytes) ? w.dense_rows : 0;
  static unsigned long long* dbg_ts = nullptr;
  const bool phase_dbg = getenv("AS_PHASE_TIMES") != nullptr;
  if (phase_dbg) {
    if (!dbg_ts) AS_CUDA_TRY(cudaMalloc(&dbg_ts, 16 * sizeof(unsigned long long)));
    AS_CUDA_TRY(cudaMemsetAsync(dbg_ts, 0, 16 * sizeof(unsigned long long), st));
    a.phase_ts = dbg_ts;
#ifdef AS_TILE_TIMES
    unsigned long long z[33] = {0};
    AS_CUDA_TRY(cudaMemcpyToSymbolAsync(g_tt, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
#endif
  }
  const int rc = launch_persist<T, S1, S2>(a, st);
  if (phase_dbg && rc == AS_OK) {
    unsigned long long h[16];
    AS_CUDA_TRY(cudaMemcpyAsync(h, dbg_ts, sizeof(h), cudaMemcpyDeviceToHost, st));
    AS_CUDA_TRY(cudaStreamSynchronize(st));
    fprintf(stderr, "[phases n=%lld n_cols=%lld n_cb=%lld%s]", n, n_cols, w.n_cb, pre_ptr ? " pre" : "");
    for (int i = 1, last = 0; i < 16; i++)
      if (h[i]) {
        fprintf(stderr, " %.2f", (h[i] - h[last]) * 1e-3);
        last = i;
      }
    fprintf(stderr, " us\n");
#ifdef AS_TILE_TIMES
    unsigned long long tt[33];
    AS_CUDA_TRY(cudaMemcpyFromSymbolAsync(tt, g_tt, sizeof(tt), 0, cudaMemcpyDeviceToHost, st));
    AS_CUDA_TRY(cudaStreamSynchronize(st));
    fprintf(stderr, "[tile steps, block 0, kcycles]");
    for (int i = 0; i < 20; i++) fprintf(stderr, " %d:%.1f", i, tt[i] * 1e-3);
    fprintf(stderr, "\n");
#endif
  }
  return rc;
}

template <class T, class S1, class S2>
static int run_persist(const S1& s1, const S2& s2, long long n_cols, int row_bits, int mode, int prune, ValSrc<T> vs,
                       int* col_ptr, int* row_idx, T* out_vals, long long* info, bool init_info, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  const long long n = s1.size() + s2.size();
  Carve c(ws, ws_bytes);
  PersistWs w;
  carve_persist(c, &w, n, n_cols, sizeof(T));
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  return run_persist_ws<T>(w, s1, s2, n, n_cols, row_bits, mode, prune, vs, col_ptr, row_idx, out_vals, info,
                           init_info, nullptr, st);
}

inline size_t persist_ws_bytes(long long n, long long n_cols, size_t val_bytes, bool pre = false) {
  Carve c(nullptr, 0);
  PersistWs w;
  carve_persist(c, &w, n, n_cols, val_bytes, pre);
  return c.off;
}


}  // namespace as
