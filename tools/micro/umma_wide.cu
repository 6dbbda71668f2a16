// Microbenchmark: cycles per Ozaki K-chunk (S = 7 digit slices, 28 digit products of
// a 128 x 64 tile) for the MMA issue patterns of k_gram_oz / k_oz_gemm, operands
// resident in shared memory (no TMA), one CTA per SM, all SMs busy:
//   0 wide   -- one MMA per A slice, N = 64 (S - t) split at 256 (oz_issue_chunk_wide)
//   1 narrow -- 28 N = 64 MMAs, A in the collector (oz_issue_chunk)
//   2 wide, A in 32-byte rows (SW32) instead of 64-byte rows
//   3 wide, N split at 128
//   4 wide, diagonals interleaved: MMAs ordered so consecutive ones never share
//     accumulator columns (t = 0, 4, 1, 5, 2, 6, 3 halves)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../../paper_2505_21404_b200/csrc/tc05.cuh"

using namespace dngd;
constexpr int S = 7;

template <int WA>
DNGD_DEV void wide_split(uint32_t tmem, uint32_t a0, int abytes, uint32_t b0, int bbytes, int t,
                         int blk0, int nblk, bool first) {
  const uint64_t ad = umma_desc_k<WA>(a0 + t * abytes);
  umma_i8<0>(tmem + (t + blk0) * 64, ad, umma_desc_k<32>(b0 + blk0 * bbytes),
             umma_idesc_s8(128, 64 * nblk), (first && t == 0) ? 0u : 1u);
}

__device__ int g_random;

template <int MODE>
__global__ void __launch_bounds__(128, 1) k_chunk(int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = smem_align(raw, 1024);
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[2];
  const int warp = threadIdx.x >> 5;
  constexpr int ABYTES = (MODE >= 7 ? 2 : 1) * S * 128 * 64, BBYTES = (MODE >= 7 ? 3 : 1) * S * 64 * 32;
  for (int i = threadIdx.x; i < (ABYTES + BBYTES) / 4; i += blockDim.x) {
    uint32_t x = static_cast<uint32_t>(i) * 2654435761u + blockIdx.x * 40503u;  // random digits
    x ^= x >> 15;
    x *= 2246822519u;
    x ^= x >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = g_random ? x : 0x01010101u * (i & 3);
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2[0], 1); mbar_init(&bar2[1], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&taddr, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = taddr;
  long long c0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = a0 + ABYTES;
    for (int it = 0; it < iters; ++it) {
      for (int h = 0; h < 2; ++h) {
        const uint32_t a = a0 + 32 * h;
        if constexpr (MODE == 0 || MODE == 5 || MODE == 6) {
          oz_issue_chunk_wide<S, 64, 32>(t, a, 128 * 64, b0, 64 * 32, false);
          if constexpr (MODE >= 5) umma_commit(&bar2[0]);
          if constexpr (MODE == 6) umma_commit(&bar2[1]);
        } else if constexpr (MODE == 7 || MODE == 8) {
          // k_gram_oz's rings: A slabs (2 x 64-byte rows), B chunks (3 x 32-byte rows)
          const int kc = 2 * it + h;
          const uint32_t ra = a0 + ((kc >> 1) % 2) * (128 * 64 * S) + 32 * (kc & 1);
          const uint32_t rb = b0 + (kc % 3) * (64 * 32 * S);
          oz_issue_chunk_wide<S, 64, 32>(t, ra, 128 * 64, rb, 64 * 32, MODE == 8 && (kc % 16) == 0);
          umma_commit(&bar2[0]);
        } else if constexpr (MODE == 1) {
          oz_issue_chunk<S, 64, 32>(t, 64, a, 128 * 64, b0, 64 * 32, umma_idesc_s8(128, 64), false);
        } else if constexpr (MODE == 2) {
          oz_issue_chunk_wide<S, 32, 32>(t, a0 + 4096 * h, 128 * 32, b0, 64 * 32, false);
        } else if constexpr (MODE == 3) {
#pragma unroll
          for (int tt = 0; tt < S; ++tt)
            for (int b = 0; b < S - tt; b += 2)
              wide_split<64>(t, a, 128 * 64, b0, 64 * 32, tt, b, (S - tt - b) < 2 ? 1 : 2, false);
        } else {
          // halves: t = 0 (blocks 0-3 | 4-6), 1 (0-3 | 4-5), 2 (0-3 | 4), 3..6 whole
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 0, 0, 4, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 3, 0, 4, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 0, 4, 3, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 1, 0, 4, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 4, 0, 3, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 1, 4, 2, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 2, 0, 4, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 5, 0, 2, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 2, 4, 1, false);
          wide_split<64>(t, a, 128 * 64, b0, 64 * 32, 6, 0, 1, false);
        }
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

static int g_iters = 500;
template <int MODE>
void run(long long* d, const char* name) {
  const int iters = g_iters;
  const size_t smem = 1024 + (MODE >= 7 ? 2 : 1) * S * 128 * 64 + (MODE >= 7 ? 3 : 1) * S * 64 * 32;
  cudaFuncSetAttribute(k_chunk<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_chunk<MODE><<<148, 128, smem>>>(iters, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_chunk<MODE><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double chunks = 2.0 * iters;
  const double ops = 28.0 * 2 * 128 * 64 * 32 * chunks * 148;
  printf("%-40s %.0f cycles/chunk (ideal 896 at 16384 ops/cycle), %.0f int8 TOPS, %.3f ms err=%s\n", name,
         cyc / chunks, ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  if (argc > 1) g_iters = atoi(argv[1]);  // long runs: the power-capped steady state
  const int rnd = argc > 2 ? atoi(argv[2]) : 0;  // 1: random operand bytes
  cudaMemcpyToSymbol(g_random, &rnd, sizeof rnd);
  long long* d;
  cudaMalloc(&d, 8);
  if (argc > 3) {  // sustained: mode 0 repeated argv[3] times (power-limited steady state)
    for (int r = 0; r < atoi(argv[3]); ++r) run<0>(d, "wide (N split at 256), A SW64");
    return 0;
  }
  run<0>(d, "wide (N split at 256), A SW64");
  run<1>(d, "narrow N=64 x 28, collector A");
  run<2>(d, "wide, A SW32");
  run<3>(d, "wide, N split at 128");
  run<4>(d, "wide, accumulators interleaved");
  run<5>(d, "wide + 1 commit per chunk");
  run<6>(d, "wide + 2 commits per chunk");
  run<7>(d, "wide, k_gram_oz ring addresses");
  run<8>(d, "wide, ring addresses + overwrite per 16");
  return 0;
}
