// Microbenchmark: random 64-byte row scatter-adds into an L2-resident f32
// buffer (the column-merge CSC SpMM's C update) -- 4 lanes per row, one
// red.global.add.v4.f32 each -- against the same number of random 64-byte
// row gathers (the row-split SpMM's B reads).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int kMode>  // 0 gather ld.v4, 1 red.v4.f32, 2 scalar red.f32 x4, 3 128-byte row gather (8 lanes)
__global__ void k(float* __restrict__ buf, unsigned rows, int per, float* out) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lpr = kMode == 3 ? 8 : 4, rw = kMode == 3 ? 32 : 16;
  const unsigned grp = (unsigned)(gt / lpr), sub = gt % lpr;
  float acc = 0.f;
  for (int i = 0; i < per; i += 4) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const unsigned r = hash32(grp * 977u + (unsigned)(i + u) * 0x9e3779b9u) % rows;
      float* p = buf + (long long)r * rw + sub * 4;
      const bool do_red = kMode == 1 || kMode == 2 || (kMode == 4 && ((threadIdx.x >> 5) & 1));
      if (kMode == 4) p = buf + (do_red ? (16ll << 20) : 0ll) + (long long)r * rw + sub * 4;  // two 64 MB regions
      if (kMode == 0 || kMode == 3 || (kMode == 4 && !do_red)) {
        float4 b = __ldg(reinterpret_cast<const float4*>(p));
        acc += b.x + b.y + b.z + b.w;
      } else if (kMode == 1 || kMode == 4) {
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f)
                     : "memory");
      } else {
        atomicAdd(p, 1.f); atomicAdd(p + 1, 2.f); atomicAdd(p + 2, 3.f); atomicAdd(p + 3, 4.f);
      }
    }
  }
  if (kMode == 0 || kMode == 3 || kMode == 4) out[gt] = acc;
}

int main() {
  float *buf, *out;
  const long long n_groups = 1 << 20;
  const int per = 8;  // 8M row operations per launch
  cudaMalloc(&buf, 256ll << 20);
  cudaMalloc(&out, n_groups * 4 * 4);
  cudaMemset(buf, 0, 256ll << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int mbs[] = {32, 64, 128};
  const char* names[] = {"gather ld.v4", "red.v4.f32", "red.f32 x4", "gather 128B", "half/half"};
  for (int mode = 0; mode < 5; mode++)
    for (int mb : mbs) {
      const unsigned rows = (unsigned)((long long)mb << 20) / (mode == 3 ? 128 : 64);
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<n_groups * 4 / 256, 256>>>(buf, rows, per, out);
        else if (mode == 1) k<1><<<n_groups * 4 / 256, 256>>>(buf, rows, per, out);
        else if (mode == 2) k<2><<<n_groups * 4 / 256, 256>>>(buf, rows, per, out);
        else if (mode == 3) k<3><<<n_groups * 8 / 256, 256>>>(buf, rows, per, out);
        else k<4><<<n_groups * 4 / 256, 256>>>(buf, rows, per, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2)
          printf("%-14s footprint=%3d MB: %7.1f us for %lld rows, %.2f TB/s, %.3e row-ops/s\n", names[mode], mb,
                 ms * 1e3, n_groups * per, n_groups * per * (mode == 3 ? 128.0 : 64.0) / (ms * 1e-3) / 1e12,
                 n_groups * per / (ms * 1e-3));
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
