// DMMA issue rate per warp: NACC independent accumulators, operands in registers.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double2& d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d.x), "+d"(d.y) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double* out, long long* cyc, int iters) {
  double2 acc[NACC];
  for (int i = 0; i < NACC; ++i) acc[i] = make_double2(0, 0);
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NACC>
void run(int threads) {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int iters = 1000;
  k<NACC><<<1, threads>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("NACC %2d threads %4d: %.1f cycles per DMMA per warp (%.1f per SMSP)\n", NACC, threads,
         (double)c / (iters * NACC), (double)c / (iters * NACC) / (threads / 32 > 4 ? threads / 128.0 : 1.0));
}
int main() {
  run<4>(32); run<8>(32); run<16>(32); run<32>(32);
  run<8>(128); run<32>(128);
  run<8>(256); run<16>(256); run<32>(256);
  run<16>(512);
}
