// Emulated FP64 GEMM on the int8 tensor cores (Ozaki scheme, balanced base-256 digits).
//
// FP64 has no tcgen05 kind; the FP64 DMMA pipe peaks at ~35 TFLOP/s on B200
// while kind::i8 runs ~4.5 POPS.  Each row of A (and of B) is written as
//     x = 2^e sum_{t<S} d_t 2^{-8(t+1)},  d_t int8 (the whole range [-128, 127]),
// with 2^e > 2 max|row| (k_oz_slice).  Then
//     (A B^T)_ij = 2^{e_i + f_j} sum_D 2^{-8(D+2)} sum_{t+u=D} (A_t B_u^T)_ij
// and every A_t B_u^T is an exact int32 product on the tensor cores.  Products
// with t + u >= S sit below the slicing error and are skipped, so one K-chunk
// costs S(S+1)/2 MMAs accumulating into S diagonals in TMEM (S x 64 columns of
// a 128 x 64 tile).  Relative accuracy per entry is ~sqrt(K) 2^{-8S+4} max|a_i|
// max|b_j| (balanced digits: the dropped products average out): S = 6 (21 products,
// the default) is at the level of an FP64 dot product's own rounding for K ~ 512,
// S = 7 (28 products, 56 bits) is below it.  Round 2 started with base-128 digits
// (S = 7, 28 products for 50 bits); base 256 gives 48 bits in 21 products.
//
// This file holds the slicing kernel and a plain C = A B^T GEMM over sliced
// operands (dngd_oz_gemm_nt); the factored dual Gram uses the same machinery
// with its own epilogue (gram_oz.cuh).

#include <algorithm>
#include <cmath>

#include <math_constants.h>

#include "common.cuh"
#include "internal.h"
#include "oz_common.cuh"
#include "tc05.cuh"

namespace dngd {

// One warp per row: max |x| (non-finite flagged), scale 2^e with
// max 2^-e 256 <= 127, then S digits per entry (oz_digits4), written as
// 4-digit words per slice.
template <int S>
__global__ void __launch_bounds__(256) k_oz_slice(const double* __restrict__ X, long long rows,
                                                  long long K, long long ld, long long kpad,
                                                  size_t plane, int8_t* __restrict__ Q,
                                                  double* __restrict__ scale) {
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* x = X + row * ld;
  // 4 consecutive entries per lane and word (two 16-byte loads when aligned)
  const bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  auto load4 = [&](long long w, double (&v)[4]) {
    const long long k0 = 4 * w;
    if (vec && k0 + 3 < K) {
      const double2 a = *reinterpret_cast<const double2*>(x + k0);
      const double2 b = *reinterpret_cast<const double2*>(x + k0 + 2);
      v[0] = a.x;
      v[1] = a.y;
      v[2] = b.x;
      v[3] = b.y;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = k0 + b < K ? x[k0 + b] : 0.0;
    }
  };
  const long long words = kpad / 4;
  double mx = 0.0;
  bool bad = false;
  for (long long w = lane; w < words; w += 32) {
    double v[4];
    load4(w, v);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      bad |= !isfinite(v[b]);
      mx = fmax(mx, fabs(v[b]));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad ? 1 : 0, o) != 0;
  }
  const int e = bad ? 0 : oz_row_exponent(mx);
  if (lane == 0) scale[row] = bad ? CUDART_NAN : ldexp(1.0, e);
  const double sinv = ldexp(1.0, OZ_BITS * S - e);
  for (long long w = lane; w < words; w += 32) {
    double v[4];
    load4(w, v);
    uint32_t packed[S];
    oz_digits4<S>(v, sinv, bad, packed);
#pragma unroll
    for (int t = 0; t < S; ++t)
      reinterpret_cast<uint32_t*>(Q + t * plane + row * kpad)[w] = packed[t];
  }
}

int oz_slice_into(dngd_ctx* ctx, cudaStream_t s, const double* X, long long rows, long long K,
                  long long ld, long long kpad, size_t plane, int slices, int8_t* Q,
                  double* scale) {
  if (rows <= 0) return DNGD_OK;
  if (kpad < oz_kpad(K) || kpad % 32 != 0) return set_error(ctx, DNGD_ERR_DIMENSION, "oz_slice: bad kpad");
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  switch (slices) {
    case 6: k_oz_slice<6><<<grid, 256, 0, s>>>(X, rows, K, ld, kpad, plane, Q, scale); break;
    case 7: k_oz_slice<7><<<grid, 256, 0, s>>>(X, rows, K, ld, kpad, plane, Q, scale); break;
    default: return set_error(ctx, DNGD_ERR_DIMENSION, "oz_slice: slices must be 6 or 7");
  }
  return cuda_status(ctx, cudaGetLastError(), "oz_slice");
}

int oz_slice(dngd_ctx* ctx, cudaStream_t s, const double* X, long long rows, long long K,
             long long ld, int slices, int8_t* Q, double* scale) {
  const long long kp = oz_kpad(K);
  return oz_slice_into(ctx, s, X, rows, K, ld, kp, static_cast<size_t>(rows) * kp, slices, Q, scale);
}

// Split-K slicing of short, long rows (J^T w: 513 neuron rows x 25,000 activation
// rows): one 256-thread CTA per (row, split) -- the one-warp-per-row k_oz_slice left
// most SMs idle here.  Same scale rule and digits as k_oz_slice over the split's
// range [z kl, min(K, (z + 1) kl)); rows of split z land at z M + row.
template <int S>
__global__ void __launch_bounds__(256) k_oz_slice_split(const double* __restrict__ X, long long M,
                                                        long long K, long long ld, long long kl,
                                                        long long kpad, size_t plane,
                                                        int8_t* __restrict__ Q,
                                                        double* __restrict__ scale) {
  __shared__ double red[8];
  __shared__ int redbad[8];
  const long long row = blockIdx.x;
  const int z = blockIdx.y;
  const long long k0 = z * kl;
  const long long len = max(0LL, min(K, k0 + kl) - k0);
  const double* x = X + row * ld + k0;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  auto load4 = [&](long long w, double (&v)[4]) {
    const long long c0 = 4 * w;
    if (vec && c0 + 3 < len) {
      const double2 a = *reinterpret_cast<const double2*>(x + c0);
      const double2 b = *reinterpret_cast<const double2*>(x + c0 + 2);
      v[0] = a.x;
      v[1] = a.y;
      v[2] = b.x;
      v[3] = b.y;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = c0 + b < len ? x[c0 + b] : 0.0;
    }
  };
  const long long words = kpad / 4;
  double mx = 0.0;
  int bad = 0;
  for (long long w = tid; w < words; w += 256) {
    double v[4];
    load4(w, v);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      bad |= !isfinite(v[b]);
      mx = fmax(mx, fabs(v[b]));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    red[wp] = mx;
    redbad[wp] = bad;
  }
  __syncthreads();
  mx = 0.0;
  bad = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    mx = fmax(mx, red[k]);
    bad |= redbad[k];
  }
  const int e = bad ? 0 : oz_row_exponent(mx);
  const long long orow = z * M + row;
  if (tid == 0) scale[orow] = bad ? CUDART_NAN : ldexp(1.0, e);
  const double sinv = ldexp(1.0, OZ_BITS * S - e);
  for (long long w = tid; w < words; w += 256) {
    double v[4];
    load4(w, v);
    uint32_t packed[S];
    oz_digits4<S>(v, sinv, bad != 0, packed);
#pragma unroll
    for (int t = 0; t < S; ++t) reinterpret_cast<uint32_t*>(Q + t * plane + orow * kpad)[w] = packed[t];
  }
}

static int oz_slice_split(dngd_ctx* ctx, cudaStream_t s, const double* X, long long M, long long K,
                          long long ld, long long kl, long long kpad, int splits, int slices,
                          int8_t* Q, double* scale) {
  const dim3 grid(static_cast<unsigned>(M), static_cast<unsigned>(splits));
  const size_t plane = static_cast<size_t>(splits) * M * kpad;
  switch (slices) {
    case 6: k_oz_slice_split<6><<<grid, 256, 0, s>>>(X, M, K, ld, kl, kpad, plane, Q, scale); break;
    case 7: k_oz_slice_split<7><<<grid, 256, 0, s>>>(X, M, K, ld, kl, kpad, plane, Q, scale); break;
    default: return set_error(ctx, DNGD_ERR_DIMENSION, "oz_slice: slices must be 6 or 7");
  }
  return cuda_status(ctx, cudaGetLastError(), "oz_slice_split");
}

// C = alpha sum_z P_z (the split-K partials of oz_gemm_splitk), fixed order
__global__ void k_oz_splitk_sum(const double* __restrict__ part, int splits, long long M,
                                long long N, long long ldc, double alpha, double* __restrict__ C) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  double v = 0.0;
  for (int z = 0; z < splits; ++z) v += part[z * M * N + e];
  const long long r = e / N, c = e - (e / N) * N;
  C[r * ldc + c] = alpha * v;
}

size_t oz_splitk_bytes(long long M, long long N, long long K, int slices, int splits) {
  const long long kl = oz_kpad((K + splits - 1) / splits);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  return al(static_cast<size_t>(slices) * splits * M * kl) + al(static_cast<size_t>(slices) * splits * N * kl) +
         al(static_cast<size_t>(splits) * M * 8) + al(static_cast<size_t>(splits) * N * 8) +
         al(static_cast<size_t>(splits) * M * N * 8);
}

int oz_splitk_choose(dngd_ctx* ctx, long long M, long long N, long long K) {
  const long long tiles = ((M + OZ_BM - 1) / OZ_BM) * ((N + OZ_BN - 1) / OZ_BN);
  long long sp = (ctx->num_sms + tiles - 1) / tiles;            // about one wave
  sp = std::min(sp, std::max(1LL, K / 1024));                   // >= 1024 of K per split
  sp = std::min(sp, 32LL);
  // the int32 diagonal accumulators hold K <= 16384 (kOzMaxK) per split
  sp = std::max(sp, (K + (kOzMaxK - 32) - 1) / (kOzMaxK - 32));
  return static_cast<int>(std::max(1LL, sp));
}

// C (M x N, ldc) = alpha A B^T with A (M x K, lda) and B (N x K, ldb) K-major and K
// large (the J^T w contraction over activation rows): K cut into `splits` ranges,
// each sliced with its own row scales into one batch entry of the int8 engine, the
// partials summed in a fixed order.  work: oz_splitk_bytes.
OzSplitK oz_splitk_layout(void* work, long long M, long long N, long long K, int slices, int splits) {
  OzSplitK L;
  L.kl = (K + splits - 1) / splits;
  L.kp = oz_kpad(L.kl);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  char* w = static_cast<char*>(work);
  L.qa = reinterpret_cast<int8_t*>(w);
  w += al(static_cast<size_t>(slices) * splits * M * L.kp);
  L.qb = reinterpret_cast<int8_t*>(w);
  w += al(static_cast<size_t>(slices) * splits * N * L.kp);
  L.sa = reinterpret_cast<double*>(w);
  w += al(static_cast<size_t>(splits) * M * 8);
  L.sb = reinterpret_cast<double*>(w);
  w += al(static_cast<size_t>(splits) * N * 8);
  L.part = reinterpret_cast<double*>(w);
  return L;
}

// the batched GEMM over planes already in the oz_splitk_layout and the fixed-order sum
int oz_splitk_finish(dngd_ctx* ctx, cudaStream_t s, const OzSplitK& L, long long M, long long N,
                     int slices, int splits, double alpha, double* C, long long ldc) {
  int rc = oz_gemm_batched(ctx, s, L.qa, L.sa, splits * M, M, L.qb, L.sb, splits * N, N, L.kp, slices,
                           M, N, splits, L.part, N, M * N);
  if (rc) return rc;
  k_oz_splitk_sum<<<static_cast<unsigned>((M * N + 255) / 256), 256, 0, s>>>(L.part, splits, M, N, ldc,
                                                                          alpha, C);
  return cuda_status(ctx, cudaGetLastError(), "oz_splitk_sum");
}

int oz_gemm_splitk(dngd_ctx* ctx, cudaStream_t s, const double* A, long long lda, const double* B,
                   long long ldb, long long M, long long N, long long K, double alpha, double* C,
                   long long ldc, int slices, int splits, void* work, size_t work_bytes) {
  if (M <= 0 || N <= 0) return DNGD_OK;
  if (work_bytes < oz_splitk_bytes(M, N, K, slices, splits)) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm_splitk: workspace too small");
  }
  const OzSplitK L = oz_splitk_layout(work, M, N, K, slices, splits);
  if (L.kp > kOzMaxK) return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm_splitk: split longer than 16384");
  int rc = oz_slice_split(ctx, s, A, M, K, lda, L.kl, L.kp, splits, slices, L.qa, L.sa);
  if (rc) return rc;
  rc = oz_slice_split(ctx, s, B, N, K, ldb, L.kl, L.kp, splits, slices, L.qb, L.sb);
  if (rc) return rc;
  return oz_splitk_finish(ctx, s, L, M, N, slices, splits, alpha, C, ldc);
}

int oz_encode(dngd_ctx* ctx, CUtensorMap* map, const int8_t* Q, long long rows, long long kpad,
              int slices, int box_rows, int box_bytes) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kpad), static_cast<cuuint64_t>(std::max(rows, 1LL)),
                        static_cast<cuuint64_t>(slices)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(kpad),
                           static_cast<cuuint64_t>(kpad) * static_cast<cuuint64_t>(std::max(rows, 1LL))};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_bytes), static_cast<cuuint32_t>(box_rows),
                       static_cast<cuuint32_t>(slices)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(Q), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? DNGD_OK : set_error(ctx, DNGD_ERR_CUDA, "oz: tensor map encode failed");
}

// Persistent: one CTA per SM walks tiles (z, m-tile, n-tile), n fastest (the CTAs
// in flight share the 128-row A tile through L2).  Warp 0 streams K-chunks of
// consecutive tiles through the ring without waiting for epilogues; warp 1 issues
// a tile's MMAs once the epilogue has drained the previous tile's accumulators;
// warps 2-17 drain TMEM (fold -> FP64 in registers), release it, then scale and
// store while the next tile's MMAs run.
template <int S, int STAGES>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
              const double* __restrict__ scA, const double* __restrict__ scB,
              double* __restrict__ C, long long ldc, int M, int N, int nk, long long a_brows,
              long long b_brows, long long sC, int batch) {
  extern __shared__ uint8_t oz_smem_raw[];
  uint8_t* smem = smem_align(oz_smem_raw, 1024);
  // a stage is a 64-wide K-slab (two MMA K-steps) of every slice: 64-byte TMA rows
  constexpr int ABYTES = S * OZ_BM * 64, STAGE = S * (OZ_BM + OZ_BN) * 64;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* taddr_sh = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tn = (N + OZ_BN - 1) / OZ_BN, tm = (M + OZ_BM - 1) / OZ_BM;
  const int nslab = (nk + 1) / 2;
  const int ntiles = tn * tm * batch;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, OZ_EPI);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(taddr_sh, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *taddr_sh;
  auto decode = [&](int tile, int& z, int& m0, int& n0) {
    z = tile / (tn * tm);
    const int r = tile - z * tn * tm;
    m0 = (r / tn) * OZ_BM;
    n0 = (r - (r / tn) * tn) * OZ_BN;
  };
  if (warp == 0) {
    if (lane == 0) {
      int f = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int z, m0, n0;
        decode(tile, z, m0, n0);
        const int ar = static_cast<int>(z * a_brows + m0), br = static_cast<int>(z * b_brows + n0);
        for (int ks = 0; ks < nslab; ++ks, ++f) {
          const int st = f % STAGES;
          if (f >= STAGES) mbar_wait(&empty[st], ((f / STAGES) - 1) & 1);
          uint8_t* sa = smem + st * STAGE;
          mbar_arrive_expect_tx(&full[st], STAGE);
          tma_load_3d(sa, &mA, &full[st], ks * 64, ar, 0);
          tma_load_3d(sa + ABYTES, &mB, &full[st], ks * 64, br, 0);
        }
      }
    }
  } else if (warp == 1) {
    int f = 0, it = 0;
    if (lane == 0) {  // lane 0 alone waits and issues (no warp-wide mbarrier polling)
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        if (it > 0) mbar_wait(tempty, (it - 1) & 1);
        tc_fence_after();
        for (int ks = 0; ks < nslab; ++ks, ++f) {
          const int st = f % STAGES;
          mbar_wait(&full[st], (f / STAGES) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + st * STAGE);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (2 * ks + h >= nk) break;
            oz_issue_chunk_wide<S, 64, 64>(tbase, a0 + 32 * h, OZ_BM * 64, a0 + ABYTES + 32 * h,
                                           OZ_BN * 64, ks == 0 && h == 0);
          }
          umma_commit(&empty[st]);
          if (ks == nslab - 1) umma_commit(tfull);
        }
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3, h = (warp - 2) >> 2;  // lane quadrant, column group
    const int row = 32 * q + lane;
    const uint32_t tl = tbase + (static_cast<uint32_t>(32 * q) << 16);
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      int z, m0, n0;
      decode(tile, z, m0, n0);
      const double* sa_z = scA + z * a_brows;
      const double* sb_z = scB + z * b_brows;
      const double sa = m0 + row < M ? sa_z[m0 + row] : 0.0;
      const int c0 = h * OZ_COLS;
      const int cl = n0 + c0 + lane;
      const double scl = cl < N ? sb_z[cl] : 0.0;
      double v[OZ_COLS];
      if (threadIdx.x == 64) mbar_wait(tfull, it & 1);  // one poller (gram_oz.cuh)
      asm volatile("bar.sync 1, %0;" ::"n"(OZ_ETHREADS) : "memory");
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < OZ_COLS / OZ_LD; ++c) {
        int32_t acc[S][OZ_LD];
#pragma unroll
        for (int d = 0; d < S; ++d) tmem_ld<OZ_LD>(tl + d * OZ_BN + c0 + OZ_LD * c, acc[d]);
        tmem_ld_wait();
        if (c == OZ_COLS / OZ_LD - 1) {  // all diagonals in registers: release TMEM
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
        }
#pragma unroll
        for (int j = 0; j < OZ_LD; ++j) {
          int32_t a[S];
#pragma unroll
          for (int d = 0; d < S; ++d) a[d] = acc[d][j];
          v[OZ_LD * c + j] = oz_combine<S>(a) * (sa * __shfl_sync(0xffffffffu, scl, OZ_LD * c + j));
        }
      }
      if (m0 + row < M) {
        double* crow = C + z * sC + static_cast<long long>(m0 + row) * ldc + n0 + c0;
        const int nvalid = N - (n0 + c0);
        if (nvalid >= OZ_COLS && (reinterpret_cast<uintptr_t>(crow) & 15) == 0) {
#pragma unroll
          for (int j = 0; j < OZ_COLS; j += 2)
            *reinterpret_cast<double2*>(crow + j) = make_double2(v[j], v[j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < OZ_COLS; ++j)
            if (j < nvalid) crow[j] = v[j];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

template <int S, int STAGES = 2>
static int oz_gemm_launch(dngd_ctx* ctx, cudaStream_t s, const CUtensorMap& mA,
                          const CUtensorMap& mB, const double* scA, const double* scB, double* C,
                          long long ldc, long long M, long long N, int nk, int batch,
                          long long a_brows, long long b_brows, long long sC) {
  const size_t smem = oz_smem_bytes(S, 2 * STAGES);  // 64-wide slabs = 2 chunk-stages each
  auto kern = k_oz_gemm<S, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_status(ctx, e, "oz_gemm smem attribute");
  const long long tiles = ((N + OZ_BN - 1) / OZ_BN) * ((M + OZ_BM - 1) / OZ_BM) * batch;
  if (tiles >= (1LL << 31)) return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm: too many tiles");
  const unsigned grid = static_cast<unsigned>(std::min<long long>(tiles, ctx->num_sms));
  kern<<<grid, OZ_THREADS, smem, s>>>(mA, mB, scA, scB, C, ldc, static_cast<int>(M),
                                      static_cast<int>(N), nk, a_brows, b_brows, sC, batch);
  return cuda_status(ctx, cudaGetLastError(), "oz_gemm");
}

int oz_gemm_batched(dngd_ctx* ctx, cudaStream_t s, const int8_t* QA, const double* scA,
                    long long a_rows, long long a_brows, const int8_t* QB, const double* scB,
                    long long b_rows, long long b_brows, long long kpad, int slices, long long M,
                    long long N, int batch, double* C, long long ldc, long long sC) {
  if (M <= 0 || N <= 0 || batch <= 0) return DNGD_OK;
  CUtensorMap mA, mB;
  int rc = oz_encode(ctx, &mA, QA, a_rows, kpad, slices, OZ_BM, 64);
  if (rc) return rc;
  rc = oz_encode(ctx, &mB, QB, b_rows, kpad, slices, OZ_BN, 64);
  if (rc) return rc;
  const int nk = static_cast<int>(kpad / 32);
  switch (slices) {
    case 6: return oz_gemm_launch<6>(ctx, s, mA, mB, scA, scB, C, ldc, M, N, nk, batch, a_brows, b_brows, sC);
    case 7: return oz_gemm_launch<7>(ctx, s, mA, mB, scA, scB, C, ldc, M, N, nk, batch, a_brows, b_brows, sC);
    default: return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm: slices must be 6 or 7");
  }
}

}  // namespace dngd

using namespace dngd;

static size_t oz_al(size_t b) { return (b + 255) / 256 * 256; }

extern "C" int dngd_oz_gemm_workspace(dngd_ctx* ctx, int64_t M, int64_t N, int64_t K, int slices,
                                      size_t* bytes) {
  (void)ctx;
  const long long kp = oz_kpad(K);
  *bytes = oz_al(static_cast<size_t>(slices) * M * kp) + oz_al(static_cast<size_t>(slices) * N * kp) +
           oz_al(static_cast<size_t>(M) * 8) + oz_al(static_cast<size_t>(N) * 8);
  return DNGD_OK;
}

extern "C" int dngd_oz_gemm_nt(dngd_ctx* ctx, void* stream, int64_t M, int64_t N, int64_t K,
                               const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* C, int64_t ldc, int slices, void* work, size_t work_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (M <= 0 || N <= 0) return DNGD_OK;
  if (K <= 0 || K > kOzMaxK) return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm: K outside [1, 16384]");
  if (slices < OZ_SMIN || slices > OZ_SMAX) return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm: slices must be 6 or 7");
  size_t need = 0;
  dngd_oz_gemm_workspace(ctx, M, N, K, slices, &need);
  if (work_bytes < need) return set_error(ctx, DNGD_ERR_DIMENSION, "oz_gemm: workspace too small");
  const long long kp = oz_kpad(K);
  char* w = static_cast<char*>(work);
  int8_t* qa = reinterpret_cast<int8_t*>(w);
  w += oz_al(static_cast<size_t>(slices) * M * kp);
  int8_t* qb = reinterpret_cast<int8_t*>(w);
  w += oz_al(static_cast<size_t>(slices) * N * kp);
  double* sa = reinterpret_cast<double*>(w);
  w += oz_al(static_cast<size_t>(M) * 8);
  double* sb = reinterpret_cast<double*>(w);
  int rc = oz_slice(ctx, s, A, M, K, lda, slices, qa, sa);
  if (rc) return rc;
  rc = oz_slice(ctx, s, B, N, K, ldb, slices, qb, sb);
  if (rc) return rc;
  return oz_gemm_batched(ctx, s, qa, sa, M, 0, qb, sb, N, 0, kp, slices, M, N, 1, C, ldc, 0);
}
