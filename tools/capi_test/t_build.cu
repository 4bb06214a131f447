// Standalone C-ABI smoke test (no torch): tiny COO->CSC build.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../include/bsparse.h"
int main() {
  int hr[3] = {0, 2, 1}, hc[3] = {0, 1, 1};
  double hv[3] = {1, 3, 2};
  int *r, *c, *cp, *ri; double *v, *ov; long long* info; void* ws;
  cudaMalloc(&r, 12); cudaMalloc(&c, 12); cudaMalloc(&v, 24); cudaMalloc(&cp, 12); cudaMalloc(&ri, 12); cudaMalloc(&ov, 24); cudaMalloc(&info, 16);
  cudaMemcpy(r, hr, 12, cudaMemcpyHostToDevice); cudaMemcpy(c, hc, 12, cudaMemcpyHostToDevice); cudaMemcpy(v, hv, 24, cudaMemcpyHostToDevice);
  size_t wb = as_build_workspace_bytes(3, 2);
  printf("ws %zu\n", wb); fflush(stdout);
  cudaMalloc(&ws, wb);
  int rc = as_coo_to_csc_f64(3, 2, 3, r, c, 4, v, 0, cp, ri, ov, (int64_t*)info, ws, wb, 0);
  printf("rc %d %s\n", rc, as_last_error()); fflush(stdout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("sync %s\n", cudaGetErrorString(e));
  int hcp[3]; cudaMemcpy(hcp, cp, 12, cudaMemcpyDeviceToHost);
  printf("col_ptr %d %d %d\n", hcp[0], hcp[1], hcp[2]);
  return 0;
}
