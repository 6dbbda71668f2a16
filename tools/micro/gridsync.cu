// grid.sync() cost on this GPU (cooperative launch), and a __syncthreads-only loop
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_sync(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  int x = 0;
  for (int i = 0; i < iters; ++i) { x += threadIdx.x; g.sync(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = x;
}
__global__ void k_bar(int iters, int* out) {
  int x = 0;
  for (int i = 0; i < iters; ++i) { x += threadIdx.x; __syncthreads(); }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = x;
}
int main() {
  int* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {2, 16, 148}) {
    int iters = 1000; void* args[] = {&iters, &d};
    cudaLaunchCooperativeKernel((void*)k_sync, grid, 512, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_sync, grid, 512, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %d: grid.sync %.3f us\n", grid, ms * 1e3 / iters);
  }
  cudaEventRecord(a);
  k_bar<<<16, 512>>>(100000, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("__syncthreads %.1f ns\n", ms * 1e6 / 100000);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
