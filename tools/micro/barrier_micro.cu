// Microbenchmark: cost of one grid-wide barrier in a cooperatively launched
// 296 x 512 grid (2 CTAs / SM), for the barrier of common.cuh (one arrival
// counter), cooperative groups' grid.sync(), and a two-level arrival (16
// counters, the last arriver of each goes on to the top counter).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1805_03380_b200/csrc barrier_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(512, 2) k_flat(unsigned* w, int iters) {
  as::GridBar gb{w + 16, w + 32};
  unsigned gen = 0;
  for (int i = 0; i < iters; i++) as::grid_sync(gb, gen);
}

__global__ void __launch_bounds__(512, 2) k_cg(unsigned* w, int iters) {
  for (int i = 0; i < iters; i++) cg::this_grid().sync();
}

// two-level: sub-counter per group of 16 CTAs (padded to separate lines), a
// top counter and a generation word; arrival / release by thread 0
__device__ __forceinline__ void grid_sync2(unsigned* w, unsigned& gen_local) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned G = gridDim.x, grp = blockIdx.x / 16, ngrp = (G + 15) / 16;
    const unsigned gsize = min(16u, G - grp * 16);
    unsigned* sub = w + 64 + grp * 32;
    unsigned* top = w + 16;
    volatile unsigned* gen = w + 32;
    __threadfence();
    const unsigned a = atomicAdd(sub, 1u);
    if (a == gsize - 1) {
      *sub = 0u;
      const unsigned t = atomicAdd(top, 1u);
      if (t == ngrp - 1) {
        *top = 0u;
        __threadfence();
        atomicAdd((unsigned*)gen, 1u);
      }
    }
    while (*gen == gen_local) {
    }
    __threadfence();
  }
  gen_local++;
  __syncthreads();
}

__global__ void __launch_bounds__(512, 2) k_two(unsigned* w, int iters) {
  unsigned gen = 0;
  for (int i = 0; i < iters; i++) grid_sync2(w, gen);
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaStream_t st;
  cudaStreamCreate(&st);
  const int grid = 296;
  auto run = [&](const char* name, void* kern) {
    float t[2];
    int its[2] = {1, 65};
    for (int k = 0; k < 2; k++) {
      float best = 1e9;
      for (int r = 0; r < 20; r++) {
        cudaMemsetAsync(d, 0, 1 << 20, st);
        int it = its[k];
        void* args[] = {&d, &it};
        cudaEventRecord(a, st);
        cudaLaunchCooperativeKernel(kern, grid, 512, args, 0, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      t[k] = best * 1e3f;
    }
    printf("%-28s 1 barrier %.2f us, 65 barriers %.2f us -> %.3f us per barrier (%s)\n", name, t[0], t[1],
           (t[1] - t[0]) / 64, cudaGetErrorString(cudaGetLastError()));
  };
  {  // launch overheads (event time, best of 50)
    auto best = [&](const char* name, auto fn) {
      for (int i = 0; i < 10; i++) fn();
      cudaStreamSynchronize(st);
      float bst = 1e9;
      for (int r = 0; r < 50; r++) {
        cudaEventRecord(a, st);
        fn();
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        bst = ms < bst ? ms : bst;
      }
      printf("%-40s %.2f us\n", name, bst * 1e3f);
    };
    int it0 = 0;
    best("normal launch 296x512 (empty)", [&] { k_flat<<<296, 512, 0, st>>>(d, 0); });
    best("cooperative launch 296x512 (empty)", [&] {
      void* args[] = {&d, &it0};
      cudaLaunchCooperativeKernel((void*)k_flat, 296, 512, args, 0, st);
    });
    best("memset 64KB + cooperative launch", [&] {
      void* args[] = {&d, &it0};
      cudaMemsetAsync(d, 0, 65536, st);
      cudaLaunchCooperativeKernel((void*)k_flat, 296, 512, args, 0, st);
    });
    best("memset 64KB alone", [&] { cudaMemsetAsync(d, 0, 65536, st); });
  }
  run("flat (common.cuh)", (void*)k_flat);
  run("cooperative groups", (void*)k_cg);
  run("two-level arrival", (void*)k_two);
  return 0;
}
