// Microbenchmark: global / shared atomic throughput on B200 for bucket counting.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_rand(const unsigned* __restrict__ keys, long long n, unsigned* counts) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    atomicAdd(&counts[keys[i]], 1u);
}
__global__ void atom_rand(const unsigned* __restrict__ keys, long long n, unsigned* counts, unsigned* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = atomicAdd(&counts[keys[i]], 1u);
}
__global__ void smem_hist(const unsigned* __restrict__ keys, long long n, unsigned nb, unsigned* counts) {
  extern __shared__ unsigned h[];
  for (unsigned b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    atomicAdd(&h[keys[i]], 1u);
  __syncthreads();
  for (unsigned b = threadIdx.x; b < nb; b += blockDim.x) if (h[b]) atomicAdd(&counts[b], h[b]);
}
__global__ void copy_k(const unsigned* __restrict__ keys, long long n, unsigned* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = keys[i] + 1;
}

int main() {
  const long long n = 1 << 20;
  unsigned *keys, *counts, *out;
  cudaMalloc(&keys, n * 4); cudaMalloc(&counts, 4 << 20); cudaMalloc(&out, n * 4);
  unsigned* h = new unsigned[n];
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  unsigned nbs[] = {1, 32, 10000, 50000, 1000000};
  for (unsigned nb : nbs) {
    unsigned s = 12345;
    for (long long i = 0; i < n; i++) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % nb; }
    cudaMemcpy(keys, h, n * 4, cudaMemcpyHostToDevice);
    int grids[] = {148, 592, 2368};
    for (int g : grids) {
      float t[4] = {0, 0, 0, 0};
      for (int rep = 0; rep < 12; rep++) {
        for (int v = 0; v < 4; v++) {
          cudaMemset(counts, 0, 4 << 20);
          cudaEventRecord(a);
          if (v == 0) red_rand<<<g, 256>>>(keys, n, counts);
          if (v == 1) atom_rand<<<g, 256>>>(keys, n, counts, out);
          if (v == 2 && nb <= 50000) smem_hist<<<g, 256, nb * 4>>>(keys, n, nb, counts);
          if (v == 3) copy_k<<<g, 256>>>(keys, n, out);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (rep >= 2) t[v] += ms * 100;  // us averaged over 10
        }
      }
      printf("bins %7u grid %5d  RED %7.2f us  ATOM %7.2f us  smem-hist %7.2f us  copy %7.2f us  (%s)\n", nb, g, t[0], t[1], t[2], t[3], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
