// Microbenchmark: event-timed cost of a normal vs a cooperative launch of the
// same tiny grid-wide kernel (444 x 256, one grid barrier), plus memsets.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void tiny(int* p) {
  if (threadIdx.x == 0) atomicAdd(p, 1);
}
__global__ void tiny_grid(int* p) {
  if (threadIdx.x == 0) atomicAdd(p, 1);
  cg::this_grid().sync();
}

int main() {
  int* d;
  cudaMalloc(&d, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaStream_t st;
  cudaStreamCreate(&st);
  const int grid = 444;
  auto bench = [&](const char* name, auto fn) {
    for (int i = 0; i < 20; i++) fn();
    cudaStreamSynchronize(st);
    float best = 1e9, sum = 0;
    for (int r = 0; r < 50; r++) {
      cudaEventRecord(a, st);
      fn();
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
      sum += ms;
    }
    printf("%-40s best %.2f us  mean %.2f us\n", name, best * 1e3, sum / 50 * 1e3);
  };
  bench("normal launch", [&] { tiny<<<grid, 256, 0, st>>>(d); });
  bench("cooperative launch (no grid sync)", [&] {
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((void*)tiny, grid, 256, args, 0, st);
  });
  bench("cooperative launch + grid sync", [&] {
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((void*)tiny_grid, grid, 256, args, 0, st);
  });
  bench("memset 256B + normal launch", [&] {
    cudaMemsetAsync(d, 0, 256, st);
    tiny<<<grid, 256, 0, st>>>(d);
  });
  bench("2 memsets + cooperative launch", [&] {
    cudaMemsetAsync(d, 0, 4096, st);
    cudaMemsetAsync(d + 2048, 0x7f, 16, st);
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((void*)tiny, grid, 256, args, 0, st);
  });
  bench("cooperative launch, 75KB dyn smem", [&] {
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((void*)tiny, 444, 256, args, 75 * 1024, st);
  });
  return 0;
}
