// upload.cu -- host side of the end-to-end construction path
// (SpMat.from_triplets / csc.canonicalize on host arrays, csc.py:148-222).
//
// The reference takes int64 row / column arrays (csc.py:63-67); the device
// path indexes in int32.  Instead of moving 24 bytes per triplet over PCIe
// and narrowing on the device, a pool of host threads narrows the indices
// into pinned int32 staging while the copy engine moves the values, then the
// narrowed chunks follow: 16 bytes per triplet on the wire, the narrowing
// hidden behind the value transfer.  An index outside [0, 2^31) becomes -1,
// so the build kernel still reports the first out-of-range triplet by its
// input position (csc.py:215-221 CoordinateError semantics).
#include <emmintrin.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "capi_util.cuh"

namespace as {
namespace {

// Persistent workers: a job is published by bumping `gen_`; workers spin for
// a while (back-to-back calls find them awake) and then block on a condition
// variable.  The caller runs share 0 itself.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool p;
    return p;
  }

  void run(int shares, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> call_lock(call_mu_);  // one job at a time
    ensure(shares - 1);
    const int helpers = shares - 1;
    if (helpers > 0) {
      {
        std::lock_guard<std::mutex> lk(mu_);
        job_ = &fn;
        helpers_ = helpers;
        done_.store(0, std::memory_order_relaxed);
        gen_.fetch_add(1, std::memory_order_release);
      }
      cv_.notify_all();
    }
    fn(0);
    while (done_.load(std::memory_order_acquire) < helpers) {
    }
  }

 private:
  HostPool() = default;
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

  void ensure(int n) {
    while ((int)workers_.size() < n) {
      const int id = (int)workers_.size() + 1;
      workers_.emplace_back([this, id] { loop(id); });
    }
  }

  void loop(int id) {
    unsigned long long seen = 0;
    while (true) {
      unsigned long long g = gen_.load(std::memory_order_acquire);
      for (long spin = 0; g == seen && spin < (1l << 21); spin++) g = gen_.load(std::memory_order_acquire);
      if (g == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        g = gen_.load(std::memory_order_acquire);
      }
      const std::function<void(int)>* job;
      int helpers;
      {  // the job and its generation together: a lagging worker runs the
         // current job once and never re-runs it
        std::lock_guard<std::mutex> lk(mu_);
        if (stop_) return;
        job = job_;
        helpers = helpers_;
        seen = gen_.load(std::memory_order_acquire);
      }
      if (id <= helpers) {
        (*job)(id);
        done_.fetch_add(1, std::memory_order_acq_rel);
      }
    }
  }

  std::mutex call_mu_, mu_;
  std::condition_variable cv_;
  std::vector<std::thread> workers_;
  const std::function<void(int)>* job_ = nullptr;
  int helpers_ = 0;
  bool stop_ = false;
  std::atomic<unsigned long long> gen_{0};
  std::atomic<int> done_{0};
};

inline int32_t narrow_index(int64_t v) { return (v >= 0 && v <= 0x7fffffffll) ? (int32_t)v : -1; }

// dst[a, b) = narrow(src[a, b)); the aligned middle with streaming 16-byte
// stores (the staging is only read by the copy engine: no read-for-ownership,
// no cache pollution)
void narrow_range(const int64_t* src, int32_t* dst, int64_t a, int64_t b) {
  int64_t i = a;
  for (; i < b && (reinterpret_cast<uintptr_t>(dst + i) & 15u); i++) dst[i] = narrow_index(src[i]);
  for (; i + 4 <= b; i += 4) {
    const __m128i q = _mm_set_epi32(narrow_index(src[i + 3]), narrow_index(src[i + 2]), narrow_index(src[i + 1]),
                                    narrow_index(src[i]));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), q);
  }
  for (; i < b; i++) dst[i] = narrow_index(src[i]);
}

// 32-bit keys (col << rbits | row) for coordinates inside the shape, ~0u
// outside; streaming stores as above
inline uint32_t pack_key(int64_t r, int64_t c, uint64_t nr, uint64_t nc, int rbits) {
  return ((uint64_t)r < nr && (uint64_t)c < nc) ? (uint32_t)(((uint64_t)c << rbits) | (uint64_t)r) : 0xffffffffu;
}

// returns the first index in [a, b) whose coordinate is outside the shape, or b
int64_t pack_range(const int64_t* rows, const int64_t* cols, uint32_t* dst, int64_t a, int64_t b, uint64_t nr,
                   uint64_t nc, int rbits) {
  int64_t i = a;
  int64_t bad = b;
  for (; i < b && (reinterpret_cast<uintptr_t>(dst + i) & 15u); i++) {
    dst[i] = pack_key(rows[i], cols[i], nr, nc, rbits);
    if (dst[i] == 0xffffffffu && bad == b) bad = i;
  }
  for (; i + 4 <= b; i += 4) {
    const uint32_t k0 = pack_key(rows[i], cols[i], nr, nc, rbits), k1 = pack_key(rows[i + 1], cols[i + 1], nr, nc, rbits),
                   k2 = pack_key(rows[i + 2], cols[i + 2], nr, nc, rbits),
                   k3 = pack_key(rows[i + 3], cols[i + 3], nr, nc, rbits);
    if (bad == b && (k0 == 0xffffffffu || k1 == 0xffffffffu || k2 == 0xffffffffu || k3 == 0xffffffffu))
      bad = i + (k0 == 0xffffffffu ? 0 : k1 == 0xffffffffu ? 1 : k2 == 0xffffffffu ? 2 : 3);
    const __m128i q = _mm_set_epi32((int)k3, (int)k2, (int)k1, (int)k0);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), q);
  }
  for (; i < b; i++) {
    dst[i] = pack_key(rows[i], cols[i], nr, nc, rbits);
    if (dst[i] == 0xffffffffu && bad == b) bad = i;
  }
  return bad;
}

}  // namespace

// keys[lo, hi) -> rows / cols (-1 for the out-of-shape marker)
__global__ void __launch_bounds__(256) unpack_keys_kernel(const uint32_t* __restrict__ keys, long long lo,
                                                          long long hi, int rbits, int32_t* __restrict__ rows,
                                                          int32_t* __restrict__ cols) {
  const long long i = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const uint32_t k = __ldcs(&keys[i]);
  const bool bad = k == 0xffffffffu;
  rows[i] = bad ? -1 : (int32_t)(k & ((1u << rbits) - 1u));
  cols[i] = bad ? -1 : (int32_t)(k >> rbits);
}

// row indices < 65536 -> uint16 (the CSC's rows travel back at half width)
__global__ void __launch_bounds__(256) narrow_u16_kernel(const int32_t* __restrict__ src, long long n,
                                                         uint16_t* __restrict__ dst) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (uint16_t)__ldcs(&src[i]);
}

}  // namespace as

using namespace as;

extern "C" {

int as_upload_coo_i64(const int64_t* rows, const int64_t* cols, const void* vals, int64_t n, int64_t val_bytes,
                      int32_t* stage_rows, int32_t* stage_cols, int32_t* d_rows, int32_t* d_cols, void* d_vals,
                      int n_threads, int n_chunks, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n >= 0 && (val_bytes == 4 || val_bytes == 8), AS_ERR_ARG, "bad upload arguments");
  if (n == 0) return AS_OK;
  const int T = std::max(1, std::min(n_threads, 256));
  const int K = (int)std::max<int64_t>(1, std::min<int64_t>(n_chunks, (n + 65535) / 65536));
  // the values first: the copy engine moves them while the indices are
  // narrowed (vals == nullptr: the caller moves them)
  if (vals) AS_CUDA_TRY(cudaMemcpyAsync(d_vals, vals, (size_t)(n * val_bytes), cudaMemcpyHostToDevice, st));
  const int64_t per = (n + K - 1) / K;
  for (int k = 0; k < K; k++) {
    const int64_t lo = (int64_t)k * per, hi = std::min(n, lo + per);
    if (lo >= hi) break;
    const int64_t span = hi - lo;
    HostPool::get().run(T, [&](int w) {
      const int64_t a = lo + span * w / T, b = lo + span * (w + 1) / T;
      narrow_range(rows, stage_rows, a, b);
      narrow_range(cols, stage_cols, a, b);
      _mm_sfence();  // streaming stores visible before the copy is enqueued
    });
    AS_CUDA_TRY(cudaMemcpyAsync(d_rows + lo, stage_rows + lo, (size_t)span * 4, cudaMemcpyHostToDevice, st));
    AS_CUDA_TRY(cudaMemcpyAsync(d_cols + lo, stage_cols + lo, (size_t)span * 4, cudaMemcpyHostToDevice, st));
  }
  return AS_OK;
}

int as_upload_coo_packed(const int64_t* rows, const int64_t* cols, const void* vals, int64_t n, int64_t val_bytes,
                         int64_t n_rows, int64_t n_cols, uint32_t* stage_keys, uint32_t* d_keys, int32_t* d_rows,
                         int32_t* d_cols, void* d_vals, int n_threads, int n_chunks, int64_t* first_bad,
                         void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n >= 0 && (val_bytes == 4 || val_bytes == 8), AS_ERR_ARG, "bad upload arguments");
  AS_REQUIRE(n_rows > 0 && n_cols > 0, AS_ERR_SHAPE, "packed upload needs a non-empty shape");
  const int rbits = bits_for(n_rows - 1), cbits = bits_for(n_cols - 1);
  AS_REQUIRE(rbits + cbits <= 31, AS_ERR_SHAPE, "%d + %d index bits do not fit a 32-bit key", rbits, cbits);
  if (first_bad) *first_bad = -1;
  if (n == 0) return AS_OK;
  const int T = std::max(1, std::min(n_threads, 256));
  const int K = (int)std::max<int64_t>(1, std::min<int64_t>(n_chunks, (n + 65535) / 65536));
  std::atomic<int64_t> bad_min{n};
  if (vals) AS_CUDA_TRY(cudaMemcpyAsync(d_vals, vals, (size_t)(n * val_bytes), cudaMemcpyHostToDevice, st));
  const int64_t per = (n + K - 1) / K;
  for (int k = 0; k < K; k++) {
    const int64_t lo = (int64_t)k * per, hi = std::min(n, lo + per);
    if (lo >= hi) break;
    const int64_t span = hi - lo;
    HostPool::get().run(T, [&](int w) {
      const int64_t a = lo + span * w / T, b = lo + span * (w + 1) / T;
      const int64_t bad = pack_range(rows, cols, stage_keys, a, b, (uint64_t)n_rows, (uint64_t)n_cols, rbits);
      if (bad < b) {
        int64_t cur = bad_min.load(std::memory_order_relaxed);
        while (bad < cur && !bad_min.compare_exchange_weak(cur, bad, std::memory_order_relaxed)) {
        }
      }
      _mm_sfence();
    });
    AS_CUDA_TRY(cudaMemcpyAsync(d_keys + lo, stage_keys + lo, (size_t)span * 4, cudaMemcpyHostToDevice, st));
    unpack_keys_kernel<<<(unsigned)((span + 255) / 256), 256, 0, st>>>(d_keys, lo, hi, rbits, d_rows, d_cols);
    AS_LAUNCH_CHECK();
  }
  if (first_bad) {
    const int64_t b = bad_min.load();
    *first_bad = b < n ? b : -1;
  }
  return AS_OK;
}

// D2H of row indices at half width: d_rows (all < 65536) -> uint16 on the
// device, copied into the pinned stage; the caller widens after the copy
// (as_widen_u16) while other copies are in flight.
int as_rows_to_host_u16(const int32_t* d_rows, int64_t n, uint16_t* d_scratch, uint16_t* h_stage, void* stream) {
  cudaStream_t st = S(stream);
  AS_REQUIRE(n >= 0, AS_ERR_ARG, "negative length");
  if (n == 0) return AS_OK;
  narrow_u16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_rows, n, d_scratch);
  AS_LAUNCH_CHECK();
  AS_CUDA_TRY(cudaMemcpyAsync(h_stage, d_scratch, (size_t)n * 2, cudaMemcpyDeviceToHost, st));
  return AS_OK;
}

// dst[i] = src[i] on host threads (the pinned uint16 stage -> int32 rows)
int as_widen_u16(const uint16_t* src, int32_t* dst, int64_t n, int n_threads) {
  AS_REQUIRE(n >= 0, AS_ERR_ARG, "negative length");
  if (n == 0) return AS_OK;
  const int T = std::max(1, std::min(n_threads, 256));
  HostPool::get().run(T, [&](int w) {
    const int64_t a = n * w / T, b = n * (w + 1) / T;
    for (int64_t i = a; i < b; i++) dst[i] = (int32_t)src[i];
  });
  return AS_OK;
}

}  // extern "C"
