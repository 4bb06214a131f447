// capi_util.cuh -- host-side helpers for the extern "C" entry points:
// status codes, thread-local error text, workspace carving, launch sizing.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/bsparse.h"

namespace as {

void set_error(const char* fmt, ...);
extern int g_engine;  // as_set_engine: 0 auto, 1 large-input pipeline, 2 general bucket kernel

#define AS_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::as::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return AS_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define AS_LAUNCH_CHECK() AS_CUDA_TRY(cudaGetLastError())

#define AS_REQUIRE(cond, code, ...) \
  do {                              \
    if (!(cond)) {                  \
      ::as::set_error(__VA_ARGS__); \
      return (code);                \
    }                               \
  } while (0)

// bump allocator over the caller's workspace; 256-byte aligned slices
struct Carve {
  char* base;
  size_t cap;
  size_t off = 0;
  bool ok = true;
  Carve(void* b, size_t c) : base((char*)b), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t bytes = ((count * sizeof(T)) + 255) & ~size_t(255);
    if (off + bytes > cap) ok = false;
    T* p = (T*)(base ? base + off : nullptr);
    off += bytes;
    return p;
  }
};

constexpr int kMaxDevices = 64;  // per-device launch-configuration caches

// SM count of the current device (queried once per device; B200: 148).  The
// per-device caches below and in the launchers are std::atomic: concurrent
// first calls from several host threads compute the same value.
inline int num_sms() {
  static std::atomic<int> sms[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  int v = sms[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

inline int grid_for(long long n, int block, int per_sm = 8) {
  long long g = (n + block - 1) / block;
  long long cap = (long long)num_sms() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

inline int bits_for(long long maxval) {  // bits needed to represent values in [0, maxval]
  int b = 0;
  while (b < 63 && (1ll << b) <= maxval) b++;
  return b;
}

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

}  // namespace as
