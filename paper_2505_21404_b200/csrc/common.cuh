// Shared device helpers for the D-NGD sm_100a kernels: mbarrier / TMA
// wrappers, FP64 DMMA (mma.sync m8n8k4 f64), warp reductions.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#define DNGD_DEV __device__ __forceinline__

namespace dngd {

constexpr int kNumSMs = 148;

DNGD_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Align a dynamic shared-memory base by pointer arithmetic on the __shared__
// array itself, so the compiler keeps the shared address space (LDS/STS).  An
// integer round trip (uintptr_t) makes every access a generic LD/ST.
DNGD_DEV uint8_t* smem_align(uint8_t* raw, uint32_t align) {
  return raw + ((align - (smem_u32(raw) & (align - 1))) & (align - 1));
}

// ---------------------------------------------------------------- mbarrier
DNGD_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
DNGD_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
DNGD_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
DNGD_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
DNGD_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
DNGD_DEV void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
DNGD_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
DNGD_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                          int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------- FP64 MMA
// D(8x8) += A(8x4, row) * B(4x8, col).  Lane l holds A[l/4][l%4], B[l%4][l/4],
// D[l/4][2(l%4)+{0,1}].  On sm_100a this is one DMMA.8x8x4 (the FP64 tensor op).
DNGD_DEV void dmma_8x8x4(double2& d, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d.x), "+d"(d.y)
      : "d"(a), "d"(b));
}

// lower-triangular tile index t -> (ti, tj), tj <= ti, row-major over the lower triangle
DNGD_DEV void decode_lower(int t, int& ti, int& tj) {
  int i = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  ti = i;
  tj = t - i * (i + 1) / 2;
}

// lower-triangular tile index t -> (ti, tj) on T tile rows, in G x G super-blocks
// (super-rows of G tile rows, row-major over the lower triangle of super-blocks,
// row-major inside a block): the ~2 waves of CTAs in flight cover about one
// super-block, so each operand tile they stream is reused ~G times from L2
// instead of once per tile row (row-major order re-reads every column tile).
DNGD_DEV void decode_lower_grouped(int t, int T, int G, int& ti, int& tj) {
  // tiles before super-row I (all full): G^2 I (I - 1) / 2 + I G (G + 1) / 2
  auto before = [&](long long I) { return G * G * I * (I - 1) / 2 + I * G * (G + 1) / 2; };
  long long I = static_cast<long long>(
      (-0.5 * G + sqrt(0.25 * G * G + 2.0 * G * G * static_cast<double>(t))) / (G * G) + 0.5);
  while (I > 0 && before(I) > t) --I;
  while (before(I + 1) <= t) ++I;
  const long long u = t - before(I);
  const long long h = min(static_cast<long long>(G), T - I * G);  // rows of super-row I
  if (u < I * h * G) {
    const long long jb = u / (h * G), v = u - jb * h * G;
    ti = static_cast<int>(I * G + v / G);
    tj = static_cast<int>(jb * G + v % G);
  } else {
    int r, c;
    decode_lower(static_cast<int>(u - I * h * G), r, c);
    ti = static_cast<int>(I * G + r);
    tj = static_cast<int>(I * G + c);
  }
}

// ---------------------------------------------------------------- reductions
DNGD_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction (fixed tree); result valid in thread 0.
template <int NT>
DNGD_DEV double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (l < NT / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

}  // namespace dngd
