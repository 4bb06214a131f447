// sortreduce_host.cuh -- host side of the lean sort-reduce kernel
// (sortreduce.cuh): applicability, bucket sizing, workspace, launch.
#pragma once

#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "capi_util.cuh"
#include "sortreduce.cuh"

namespace as {
namespace sr {

constexpr size_t kSmemMax = (224 / kMinBlocks) * 1024;  // per CTA: kMinBlocks CTAs per SM
constexpr long long kGridMax = 148 * kMinBlocks;        // workspace bound (per-CTA scratch)

struct Ws {
  unsigned* loffT;
  unsigned long long* ctr;
  unsigned long long* tstate;
  unsigned* gK;
  unsigned* gX;
  void* gV;
  long long* cta_bad;
  unsigned long long* oK;
  unsigned long long* oK2;
  unsigned* oP;
  unsigned* oP2;
  int* oR;
  void* oV;
  long long* own_info;
};

// (sized for the largest grid and bucket count the kernel accepts)
static size_t carve(Carve& c, Ws* w, long long n, size_t vb) {
  const long long n1 = std::max(1ll, n);
  const long long nst = n1 + 4 * kGridMax;  // chunks rounded up to multiples of 4
  w->loffT = c.take<unsigned>((size_t)(kMaxCb + 1) * kGridMax);
  w->ctr = c.take<unsigned long long>(2);
  w->tstate = c.take<unsigned long long>(kMaxCb + kMaxCb / 32 + 1);
  w->gK = c.take<unsigned>(nst);
  w->gX = c.take<unsigned>(nst);
  w->gV = (void*)c.take<char>(nst * (long long)vb);
  w->cta_bad = c.take<long long>(kGridMax);
  w->oK = c.take<unsigned long long>(n1);
  w->oK2 = c.take<unsigned long long>(n1);
  w->oP = c.take<unsigned>(n1);
  w->oP2 = c.take<unsigned>(n1);
  w->oR = c.take<int>(n1);
  w->oV = (void*)c.take<char>(n1 * (long long)vb);
  w->own_info = c.take<long long>(2);
  return c.off;
}

inline size_t ws_bytes(long long n, size_t vb) {
  Carve c(nullptr, 0);
  Ws w;
  return carve(c, &w, n, vb);
}

struct Plan {
  bool ok = false;
  long long ncb = 0;
  unsigned long long cb_mul = 0;
  size_t smem = 0;
};

// Buckets of ~0.85 tile on average, rounded up to whole waves of the grid,
// each at most kMaxW - 24 columns; the bucket-local key (column bits + minor
// bits) must fit 32 bits and the chunk must fit the registers (n <= grid x
// kChunkMax).
template <class T>
static Plan plan(long long n, long long n_out_cols, int minor_bits, int grid) {
  Plan p;
  if (n > (long long)grid * kChunkMax || grid > kGridMax || n_out_cols <= 0) return p;
  static const double kFill = getenv("AS_SR_FILL") ? atof(getenv("AS_SR_FILL")) : 0.85;
  long long nb = (long long)((double)n / (kFill * kTile)) + 1;
  static const bool kWave = getenv("AS_SR_WAVE") == nullptr || atoi(getenv("AS_SR_WAVE")) != 0;
  if (nb > grid || kWave) nb = (nb + grid - 1) / grid * grid;  // whole waves: every CTA takes a tile
  nb = std::max(nb, (n_out_cols + (kMaxW - 24) - 1) / (kMaxW - 24));
  nb = std::min(nb, n_out_cols);
  nb = std::max(nb, 1ll);
  if (nb > kMaxCb) return p;
  const long long max_w = (n_out_cols + nb - 1) / nb + 1;
  if (max_w > kMaxW || minor_bits + bits_for(max_w - 1) > 32) return p;
  const long long chunk = (((n + grid - 1) / grid) + 3) & ~3ll;
  const Layout L = layout<T>(nb, chunk);
  if ((size_t)L.total > kSmemMax) return p;
  p.ok = true;
  p.ncb = nb;
  p.cb_mul = (unsigned long long)((((unsigned __int128)nb) << 32) / (unsigned long long)n_out_cols);
  p.smem = (size_t)L.total;
  return p;
}

// co-resident grid of the instantiation (per device, cached)
template <class T, class S1, class S2>
static int grid_of() {
  static std::atomic<int> grid[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  if (grid[dev] == 0) {
    auto kern = sortreduce_kernel<T, S1, S2>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax) != cudaSuccess)
      return 0;
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, kSmemMax);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int kCtas = getenv("AS_SR_CTAS") ? atoi(getenv("AS_SR_CTAS")) : kMinBlocks;
    grid[dev] = (int)std::min<long long>((long long)std::min(per_sm, kCtas) * sms, kGridMax);
  }
  return grid[dev];
}

inline bool disabled() {
  static const bool off = getenv("AS_NO_SR") != nullptr;
  return off;
}

// Returns AS_OK after launching, or -1 when the input is outside this
// kernel's envelope (the caller falls back to the general bucket kernel).
template <class T, class S1, class S2>
static int run(const S1& s1, const S2& s2, long long n1, long long n, long long n_out_cols, int minor_bits,
               long long n_minor, int mode,
               int prune, int* col_ptr, int* row_idx, T* out_vals, long long* info, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  if (disabled()) return -1;
  int grid = grid_of<T, S1, S2>();
  if (grid <= 0) return -1;
  // inputs that one tile per SM holds: one CTA per SM (half the participants of the grid
  // barrier and of the look-back; cfg 2's flush 26.3 -> 25.3 us under ncu)
  static const long long kSmallEnv = getenv("AS_SR_SMALL_N") ? atoll(getenv("AS_SR_SMALL_N")) : -1;
  const long long small_n = kSmallEnv >= 0 ? kSmallEnv : (long long)(0.85 * kTile) * num_sms();
  if (n <= small_n) grid = std::min(grid, num_sms());
  const Plan p = plan<T>(n, n_out_cols, minor_bits, grid);
  if (!p.ok) return -1;
  Carve c(ws, ws_bytes);
  Ws w;
  carve(c, &w, n, sizeof(T));
  AS_REQUIRE(c.ok, AS_ERR_ARG, "workspace too small: %zu < %zu", ws_bytes, c.off);
  Args<T, S1, S2> a;
  a.s1 = s1;
  a.s2 = s2;
  a.n1 = n1;
  a.n = n;
  a.n_out_cols = n_out_cols;
  a.minor_bits = minor_bits;
  a.n_minor = n_minor;
  a.ncb = p.ncb;
  a.cb_mul = p.cb_mul;
  a.mode = mode;
  a.prune = prune;
  a.loffT = w.loffT;
  a.ctr = w.ctr;
  a.tstate = w.tstate;
  a.ch = (((n + grid - 1) / grid) + 3) & ~3ll;
  a.gK = w.gK;
  a.gX = w.gX;
  a.gV = (T*)w.gV;
  a.cta_bad = w.cta_bad;
  a.oK = w.oK;
  a.oK2 = w.oK2;
  a.oP = w.oP;
  a.oP2 = w.oP2;
  a.oR = w.oR;
  a.oV = (T*)w.oV;
  a.idx_bits = bits_for(n > 0 ? n - 1 : 0);
  a.col_ptr = col_ptr;
  a.row_idx = row_idx;
  a.out_vals = out_vals;
  a.info = info ? info : w.own_info;
  a.phase_ts = nullptr;
  static const int kStop = getenv("AS_SR_STOP") ? atoi(getenv("AS_SR_STOP")) : 0;
  a.stop = kStop;
  static unsigned long long* dbg = nullptr;
  static const bool phase_dbg = getenv("AS_PHASE_TIMES") != nullptr;
  if (phase_dbg) {
    if (!dbg) AS_CUDA_TRY(cudaMalloc(&dbg, (8 + 3 * kMaxCb + 64) * sizeof(unsigned long long)));
    AS_CUDA_TRY(cudaMemsetAsync(dbg, 0, (8 + 3 * kMaxCb + 64) * sizeof(unsigned long long), st));
    unsigned long long init[1] = {~0ull};
    AS_CUDA_TRY(cudaMemcpyAsync(dbg, init, sizeof(init), cudaMemcpyHostToDevice, st));
    a.phase_ts = dbg;
  }
  void* args[] = {(void*)&a};
  AS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)sortreduce_kernel<T, S1, S2>, dim3(grid), dim3(kThreads), args,
                                          p.smem, st));
  if (phase_dbg) {
    static unsigned long long h[8 + 3 * kMaxCb + 64];
    AS_CUDA_TRY(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    AS_CUDA_TRY(cudaStreamSynchronize(st));
    // per tile (relative to barrier 2): loads done, count published, look-back done
    auto pct = [&](int k, double q) {
      std::vector<double> v;
      for (long long t = 0; t < p.ncb; t++)
        if (h[8 + 3 * t + k]) v.push_back((h[8 + 3 * t + k] - (double)h[3]) * 1e-3);
      if (v.empty()) return 0.0;
      std::sort(v.begin(), v.end());
      return v[(size_t)(q * (v.size() - 1))];
    };
    {
      const unsigned long long* c = h + 8 + 3 * kMaxCb;
      fprintf(stderr, "  CTA0 kcycles: P1 init %.1f loads %.1f rank %.1f resv+stage %.1f | barrier %.1f | P2 scan %.1f write %.1f |"
              " tile0: load %.1f wait+hist %.1f binscan %.1f place %.1f rank %.1f reduce %.1f scan %.1f lookback %.1f write %.1f\n",
              0.0, (c[11] - c[10]) * 1e-3, (c[12] - c[11]) * 1e-3, (c[13] - c[12]) * 1e-3, (c[14] - c[13]) * 1e-3,
              (c[15] - c[14]) * 1e-3, (c[16] - c[15]) * 1e-3, (c[1] - c[0]) * 1e-3, (c[2] - c[1]) * 1e-3,
              (c[3] - c[2]) * 1e-3, (c[4] - c[3]) * 1e-3, (c[5] - c[4]) * 1e-3, (c[6] - c[5]) * 1e-3,
              (c[7] - c[6]) * 1e-3, (c[8] - c[7]) * 1e-3, (c[9] - c[8]) * 1e-3);
    }
    {
      const unsigned long long* c = h + 8 + 3 * kMaxCb + 32;
      const int nt = (int)std::min<long long>(p.ncb, grid);
      fprintf(stderr, "  first tile per CTA, kcycles avg/max:");
      const char* nm[10] = {"", "load", "hist", "binscan", "place", "rank", "reduce", "prefix", "lookback", "write"};
      for (int k = 1; k <= 9; k++) fprintf(stderr, " %s %.1f/%.1f", nm[k], c[2 * k] * 1e-3 / nt, c[2 * k + 1] * 1e-3);
      fprintf(stderr, "\n");
    }
    fprintf(stderr, "  tiles: loaded p0/50/100 %.2f %.2f %.2f | published %.2f %.2f %.2f | placed %.2f %.2f %.2f us\n",
            pct(2, 0), pct(2, .5), pct(2, 1), pct(0, 0), pct(0, .5), pct(0, 1), pct(1, 0), pct(1, .5), pct(1, 1));
    fprintf(stderr, "[sr big bins %llu]", h[5]);
    fprintf(stderr, "[sr n=%lld ncb=%lld grid=%d smem=%zu] start skew %.2f, P1 %.2f, P2 %.2f, P3 %.2f us\n", n, p.ncb,
            grid, p.smem, (h[1] - h[0]) * 1e-3, (h[2] - h[0]) * 1e-3, (h[3] - h[2]) * 1e-3, (h[4] - h[3]) * 1e-3);
  }
  return AS_OK;
}

}  // namespace sr
}  // namespace as
