// Microbenchmark: cost of the chained-scan building blocks on B200.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1805_03380_b200/csrc/common.cuh"
using namespace as;

__global__ void k_empty() {}
__global__ void k_ticket(unsigned* ticket, long long* out) {
  __shared__ long long t;
  if (threadIdx.x == 0) t = atomicAdd(ticket, 1u);
  __syncthreads();
  if (threadIdx.x == 0 && t < 0) out[0] = t;
}
__global__ void k_fence(unsigned* ticket, long long* out) {
  __shared__ long long t;
  if (threadIdx.x == 0) t = atomicAdd(ticket, 1u);
  __syncthreads();
  __threadfence();
  if (threadIdx.x == 0 && t < 0) out[0] = t;
}
__global__ void k_lookback(unsigned* ticket, unsigned long long* states, long long* out) {
  __shared__ long long t;
  __shared__ unsigned long long pre;
  if (threadIdx.x == 0) t = atomicAdd(ticket, 1u);
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long p = tile_lookback_warp(states, t, 5);
    if (threadIdx.x == 0) pre = p;
  }
  __syncthreads();
  if (threadIdx.x == 0 && t == gridDim.x - 1) out[0] = pre;
}

int main() {
  unsigned* ticket; unsigned long long* states; long long* out;
  cudaMalloc(&ticket, 4); cudaMalloc(&states, 8 * 100000); cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grids[] = {3, 13, 98, 489, 4883};
  for (int gi = 0; gi < 5; gi++) {
    int g = grids[gi];
    float t[4] = {0, 0, 0, 0};
    for (int rep = 0; rep < 20; rep++) {
      for (int v = 0; v < 4; v++) {
        cudaMemset(ticket, 0, 4); cudaMemset(states, 0, 8 * g);
        cudaEventRecord(a);
        if (v == 0) k_empty<<<g, 256>>>();
        if (v == 1) k_ticket<<<g, 256>>>(ticket, out);
        if (v == 2) k_fence<<<g, 256>>>(ticket, out);
        if (v == 3) k_lookback<<<g, 256>>>(ticket, states, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep >= 5) t[v] += ms * 1000 / 15;
      }
    }
    long long o; cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
    printf("grid %5d  empty %6.2f us  ticket %6.2f  fence %6.2f  lookback %6.2f (prefix %lld)\n", g, t[0], t[1], t[2], t[3], o);
  }
  return 0;
}
