// Microbenchmark: random 64-byte row gathers from a footprint of F MB, with
// and without an L2 evict_last policy and with a concurrent streaming read
// (the SpMM row kernel's access mix).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ unsigned long long keep_pol() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_pol(const float* p, unsigned long long pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}

// 4 lanes per 64-byte row; each lane group gathers `per` random rows
template <int kMode>  // 0 plain ldg, 1 evict_last policy
__global__ void gather(const float* __restrict__ bt, unsigned rows, int per, const float* __restrict__ stream,
                       long long stream_n, float* out) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned grp = (unsigned)(gt >> 2), sub = gt & 3;
  const unsigned long long pol = keep_pol();
  float acc = 0.f;
  for (int i = 0; i < per; i += 4) {
    float4 b[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const unsigned r = hash32(grp * 977u + (unsigned)(i + u) * 0x9e3779b9u) % rows;
      const float* p = bt + (long long)r * 16 + sub * 4;
      b[u] = kMode ? ld_pol(p, pol) : __ldg(reinterpret_cast<const float4*>(p));
    }
#pragma unroll
    for (int u = 0; u < 4; u++) acc += b[u].x + b[u].y + b[u].z + b[u].w;
    if (stream_n) {
      const long long si = (gt * per + i) % stream_n;
      acc += __ldcs(stream + si);
    }
  }
  out[gt] = acc;
}

int main() {
  float *bt, *stream, *out;
  const long long n_groups = 1 << 20;  // 1M row groups x 4 lanes
  const int per = 8;
  cudaMalloc(&bt, 256ll << 20);
  cudaMalloc(&stream, 512ll << 20);
  cudaMalloc(&out, n_groups * 4 * 4);
  cudaMemset(bt, 0, 256ll << 20);
  cudaMemset(stream, 0, 512ll << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int mbs[] = {16, 32, 48, 64, 80, 96, 128};
  int maxp = 0, dev = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  int maxwin = 0;
  cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  printf("max persisting L2 %d MB, max window %d MB\n", maxp >> 20, maxwin >> 20);
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int withs = 0; withs < 2; withs++)
    for (int mode = 0; mode < 3; mode++)
      for (int mb : mbs) {
        cudaStreamAttrValue attr = {};
        if (mode == 2) {
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
          attr.accessPolicyWindow.base_ptr = bt;
          attr.accessPolicyWindow.num_bytes = std::min((size_t)maxwin, (size_t)mb << 20);
          attr.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxp / (float)((size_t)mb << 20));
          attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
          attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        }
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr);
        const unsigned rows = (unsigned)((long long)mb << 20) / 64;
        const long long sn = withs ? (128ll << 20) : 0;
        for (int rep = 0; rep < 3; rep++) {
          cudaEventRecord(a, st);
          if (mode == 1) gather<1><<<n_groups * 4 / 256, 256, 0, st>>>(bt, rows, per, stream, sn, out);
          else gather<0><<<n_groups * 4 / 256, 256, 0, st>>>(bt, rows, per, stream, sn, out);
          cudaEventRecord(b, st);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (rep == 2)
            printf("stream=%d policy=%d footprint=%3d MB: %.1f us, gather %.2f TB/s\n", withs, mode, mb, ms * 1e3,
                   n_groups * per * 64.0 / (ms * 1e-3) / 1e12);
        }
      }
  return 0;
}
