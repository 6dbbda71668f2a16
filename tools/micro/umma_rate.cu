// Microbenchmark: tcgen05.mma kind::i8 issue rate vs N (M = 128, K = 32) with
// operands resident in shared memory (no TMA), one CTA per SM, all SMs busy.
// Prints cycles per MMA and chip-level int8 TOPS at the measured clock.
#include <cstdio>
#include <cstdint>
#include "../../paper_2505_21404_b200/csrc/tc05.cuh"

using namespace dngd;

template <int N, int COLL>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = smem_align(raw, 1024);
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 32 * 8 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&taddr, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = taddr;
  long long c0 = clock64();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_s8(128, N);
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 8 * 128 * 32;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t d = t + (j & 1) * 256;
        if (COLL == 0) umma_i8<0>(d, umma_desc_sw32(a0 + j * 4096), umma_desc_sw32(b0 + j * N * 32), idesc, 1);
        else if (j == 0) umma_i8<1>(d, umma_desc_sw32(a0), umma_desc_sw32(b0 + j * N * 32), idesc, 1);
        else if (j == 7) umma_i8<3>(d, umma_desc_sw32(a0), umma_desc_sw32(b0 + j * N * 32), idesc, 1);
        else umma_i8<2>(d, umma_desc_sw32(a0), umma_desc_sw32(b0 + j * N * 32), idesc, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = c1 - c0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

template <int N, int COLL>
void run(long long* d) {
  const int iters = 2000;
  const size_t smem = 1024 + (8 * 128 + 8 * 256) * 32;
  cudaFuncSetAttribute(k_rate<N, COLL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_rate<N, COLL><<<148, 128, smem>>>(iters, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_rate<N, COLL><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double n_mma = 8.0 * iters;
  const double ops = 2.0 * 128 * N * 32 * n_mma * 148;
  printf("N=%3d coll=%d: %.1f cycles/MMA, %.0f int8 TOPS (%.3f ms) err=%s\n", N, COLL, cyc / n_mma,
         ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<32, 0>(d); run<64, 0>(d); run<64, 1>(d); run<128, 0>(d); run<128, 1>(d); run<256, 0>(d); run<256, 1>(d);
  return 0;
}
