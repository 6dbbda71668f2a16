// Microbenchmark: TMA tensor-load throughput per SM vs box inner width, for the
// Ozaki operand shape (int8 digit planes, box {W bytes, 128 rows, 7 slices}), and
// for plain 1-D bulk copies of the same bytes.  One CTA per SM (148), a 3-stage
// ring; the consumer only waits on "full" and frees the stage.  Data ~96 MB
// (L2-resident share), every CTA streams different rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2505_21404_b200/csrc/common.cuh"

using namespace dngd;

constexpr int STAGES = 3, SL = 7, ROWS = 128;

template <int W, bool BULK>
__global__ void __launch_bounds__(64, 1) k_feed(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                               long long rows_total, long long kpad, int iters,
                                               long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = smem_align(raw, 1024);
  constexpr int STAGE = W * ROWS * SL;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  long long c0 = clock64();
  const long long row0 = (static_cast<long long>(blockIdx.x) * 1024) % (rows_total - ROWS);
  const int nk = static_cast<int>(kpad / W);
  if (threadIdx.x == 0) {
    for (int f = 0; f < iters; ++f) {
      const int st = f % STAGES;
      if (f >= STAGES) mbar_wait(&empty[st], ((f / STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[st], STAGE);
      const int kc = f % nk;
      const int r = static_cast<int>(row0 + (f / nk) * ROWS % 4096);
      if (BULK) {
        // contiguous block of STAGE bytes (pre-tiled layout)
        const uint8_t* g = src + ((static_cast<long long>(f) * 148 + blockIdx.x) % 2000) * STAGE;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(smem + st * STAGE)), "l"(g), "r"(STAGE), "r"(smem_u32(&full[st])) : "memory");
      } else {
        tma_load_3d(smem + st * STAGE, &map, &full[st], kc * W, r, 0);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int f = 0; f < iters; ++f) {
      const int st = f % STAGES;
      mbar_wait(&full[st], (f / STAGES) & 1);
      mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = clock64() - c0;
}

template <int W, bool BULK>
void run(PFN_cuTensorMapEncodeTiled_v12000 enc, uint8_t* buf, long long* d) {
  const long long kpad = 512, rows = 8192 * 3;
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)kpad, (cuuint64_t)rows, SL};
  cuuint64_t strides[2] = {(cuuint64_t)kpad, (cuuint64_t)(kpad * rows)};
  cuuint32_t box[3] = {W, ROWS, SL}, es[3] = {1, 1, 1};
  CUtensorMapSwizzle sw = W == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : W == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int iters = 4000;
  const size_t smem = 1024 + STAGES * (size_t)W * ROWS * SL + 64;
  cudaFuncSetAttribute(k_feed<W, BULK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_feed<W, BULK><<<148, 64, smem>>>(map, buf, rows, kpad, 50, d);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_feed<W, BULK><<<148, 64, smem>>>(map, buf, rows, kpad, iters, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)iters * W * ROWS * SL;
  printf("%s W=%3d: %.1f B/cycle/SM, %.2f TB/s chip (enc %d, %s)\n", BULK ? "bulk " : "tma3d", W,
         bytes / cyc, bytes * 148 / (ms * 1e-3) / 1e12, (int)r, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  uint8_t* buf; cudaMalloc(&buf, 512LL * 8192 * 3 * 7 + (64 << 20));
  cudaMemset(buf, 1, 512LL * 8192 * 3 * 7);
  long long* d; cudaMalloc(&d, 8);
  run<32, false>(enc, buf, d);
  run<64, false>(enc, buf, d);
  run<32, true>(enc, buf, d);
  return 0;
}
