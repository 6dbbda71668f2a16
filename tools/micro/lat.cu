// Latency microbenchmarks for FP64 ops on sm_100a (dependent chains, one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.000001;
  __shared__ double sh[64];
  sh[threadIdx.x & 63] = x;
  __syncthreads();
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // reciprocal chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // shfl chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // smem load chain
  int idx = threadIdx.x & 63;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = sh[idx] + x; idx = ((int)x) & 63; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
  // DFMA throughput: 8 independent chains
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = x + j;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], y, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
  for (int j = 0; j < 8; ++j) x += a[j];
  out[threadIdx.x] = x;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 64 * 8);
  const char* names[] = {"dfma", "dmul", "rcp(div)", "sqrt", "shfl", "lds", "syncthreads(128thr)", "dfma x8 indep (per iter)"};
  for (int threads : {32, 128}) {
    k<<<1, threads>>>(out, cyc, 1.5, 1000);
    cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
    printf("threads=%d\n", threads);
    for (int i = 0; i < 8; ++i) printf("  %-28s %.1f cycles/iter\n", names[i], h[i] / 1000.0);
  }
  // throughput across full GPU: 148 SMs x 1024 threads DFMA
  return 0;
}
