// FP64 tensor-core GEMM / SYRK engine for sm_100a.
//
// C = alpha * A B^T + beta * C with A (M x K) and B (N x K) row-major, i.e.
// both operands K-contiguous -- the layout of J (rows = residuals, columns =
// parameters), of the activation channels and of the weight matrices.
//
//  * operands are staged global -> shared by TMA (cp.async.bulk.tensor, 16x128
//    FP64 boxes, SWIZZLE_128B) through a STAGES-deep full/empty mbarrier ring
//    refilled by thread 0 (a dedicated producer warp would cost the consumer
//    warps registers: 9 warps allocate as 12);
//  * WM x WN consumer warps run mma.sync.m8n8k4.f64 (DMMA.8x8x4, the FP64
//    tensor pipe -- tcgen05 has no f64 kind);
//  * fragments are read with conflict-free 128-bit LDS: lane l of a fragment
//    reads row l/4 and the swizzled 16-byte chunk 2(l%4)+h, whose two doubles
//    feed two consecutive MMAs.  A and B use the same lane->k permutation, so
//    the contraction is unchanged (sum over k is order-free per MMA);
//  * lower != 0 enumerates only lower-triangular tiles (SYRK, trailing
//    Cholesky updates);
//  * the SYRK uses split-K with per-split partial tiles and a fixed-order
//    reduction, so K is bitwise deterministic run to run (trajectory parity).
//
// Reference call sites replaced: solver.py:153 (J @ J.T), the trailing update
// inside LAPACK dpotrf (solver.py:166), solver.py:259-260 (K[:, I] sketch).

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace dngd {

struct GemmDev {
  long long M, N, K;
  int ntiles, tiles_n, kchunks, lower, vec_ok;
  double alpha, beta;
  double* C;
  long long ldc, sC;
  double* partial;
};


template <int BM, int BN, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int kConsumerWarps = WM * WN;
  static constexpr int kThreads = kConsumerWarps * 32;
  static constexpr int kStageA = BM * 128;
  static constexpr int kStageB = BN * 128;
  static constexpr int kStageBytes = kStageA + kStageB;
  static constexpr size_t kSmem = size_t(STAGES) * kStageBytes + 1024 + 2 * STAGES * 8;
};

template <int BM, int BN, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(WM * WN * 32, (WM * WN <= 4 ? 3 : 1))
    k_gemm_nt(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const GemmDev p) {
  using Cfg = GemmCfg<BM, BN, WM, WN, STAGES>;
  constexpr int NCW = Cfg::kConsumerWarps;
  constexpr int WTM = BM / WM, WTN = BN / WN, MI = WTM / 8, NJ = WTN / 8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align(smem_raw, 1024);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x;
  const int s = u / p.ntiles;
  const int t = u - s * p.ntiles;
  int tm, tn;
  if (p.lower) {
    decode_lower(t, tm, tn);
  } else {
    tm = t / p.tiles_n;
    tn = t - tm * p.tiles_n;
  }
  const int batch = blockIdx.y;
  const long long kc_total = (p.K + 15) / 16;
  const long long kc0 = static_cast<long long>(s) * p.kchunks;
  const long long kc1 = min(kc_total, kc0 + p.kchunks);
  const int nk = static_cast<int>(max(0LL, kc1 - kc0));

  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // Thread 0 doubles as the TMA producer: it fills the ring up front, then
  // refills the stage consumed in iteration kc-1 at the top of iteration kc
  // (by then the other warps have normally released it).
  auto issue = [&](int kc) {
    const int st = kc % STAGES;
    uint8_t* sa = smem + st * Cfg::kStageBytes;
    mbar_arrive_expect_tx(&full[st], Cfg::kStageBytes);
    const int kcoord = static_cast<int>((kc0 + kc) * 16);
    tma_load_3d(sa, &tmA, &full[st], kcoord, tm * BM, batch);
    tma_load_3d(sa + Cfg::kStageA, &tmB, &full[st], kcoord, tn * BN, batch);
  };
  if (threadIdx.x == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int kc = 0; kc < min(nk, STAGES); ++kc) issue(kc);
  }

  const int wm = warp / WN, wn = warp - (warp / WN) * WN;
  double2 acc[MI][NJ];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j] = make_double2(0.0, 0.0);

  const int lrow = lane >> 2;
  for (int kc = 0; kc < nk; ++kc) {
    const int st = kc % STAGES;
    const uint32_t ph = (kc / STAGES) & 1;
    if (threadIdx.x == 0 && kc >= 1 && kc - 1 + STAGES < nk) {
      const int pk = kc - 1;
      mbar_wait(&empty[pk % STAGES], (pk / STAGES) & 1);
      issue(pk + STAGES);
    }
    __syncwarp();
    mbar_wait(&full[st], ph);
    const uint8_t* sa = smem + st * Cfg::kStageBytes + (wm * WTM + lrow) * 128;
    const uint8_t* sb = smem + st * Cfg::kStageBytes + Cfg::kStageA + (wn * WTN + lrow) * 128;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sw = ((2 * (lane & 3) + h) ^ lrow) << 4;
      double2 a[MI], b[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = *reinterpret_cast<const double2*>(sa + i * 1024 + sw);
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[j] = *reinterpret_cast<const double2*>(sb + j * 1024 + sw);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j], a[i].x, b[j].x);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma_8x8x4(acc[i][j], a[i].y, b[j].y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // ------------------------------------------ epilogue
  if (p.partial != nullptr) {
    double* dst = p.partial + (static_cast<long long>(s) * p.ntiles + t) * (BM * BN);
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int lr = wm * WTM + i * 8 + lrow;
        const int lc = wn * WTN + j * 8 + 2 * (lane & 3);
        *reinterpret_cast<double2*>(dst + lr * BN + lc) = acc[i][j];
      }
    return;
  }
  double* C = p.C + static_cast<long long>(batch) * p.sC;
  // Epilogue in row groups of 8: the beta*C loads of a group are all issued before
  // any store (one L2 round trip per group instead of one per fragment).
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const long long r = static_cast<long long>(tm) * BM + wm * WTM + i * 8 + lrow;
    const bool rok = r < p.M;
    double2 cv[NJ];
    bool ok0[NJ], ok1[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const long long c = static_cast<long long>(tn) * BN + wn * WTN + j * 8 + 2 * (lane & 3);
      ok0[j] = rok && c < p.N && (!p.lower || c <= r);
      ok1[j] = rok && c + 1 < p.N && (!p.lower || c + 1 <= r);
      cv[j] = make_double2(0.0, 0.0);
      if (p.beta != 0.0) {
        const double* cp = C + r * p.ldc + c;
        if (ok0[j] && ok1[j] && p.vec_ok) {
          cv[j] = __ldcg(reinterpret_cast<const double2*>(cp));
        } else {
          if (ok0[j]) cv[j].x = __ldcg(cp);
          if (ok1[j]) cv[j].y = __ldcg(cp + 1);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const long long c = static_cast<long long>(tn) * BN + wn * WTN + j * 8 + 2 * (lane & 3);
      double* cp = C + r * p.ldc + c;
      const double v0 = fma(p.alpha, acc[i][j].x, p.beta * cv[j].x);
      const double v1 = fma(p.alpha, acc[i][j].y, p.beta * cv[j].y);
      if (ok0[j] && ok1[j] && p.vec_ok) {
        *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
      } else {
        if (ok0[j]) cp[0] = v0;
        if (ok1[j]) cp[1] = v1;
      }
    }
  }
}

// ------------------------------------------------------------------ host side

static int encode_map(dngd_ctx* ctx, CUtensorMap* map, const double* ptr, long long inner,
                      long long rows, int batch, long long ld, long long bstride, int box_rows) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (ld & 1) != 0 ||
      (batch > 1 && (bstride & 1) != 0)) {
    return set_error(ctx, DNGD_ERR_DIMENSION,
                     "TMA operand needs a 16-byte aligned base and even leading dimension");
  }
  if (batch <= 1) bstride = ((ld * rows + 1) / 2) * 2;
  if (bstride <= 0) bstride = 2;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(std::max(batch, 1))};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 8, static_cast<cuuint64_t>(bstride) * 8};
  cuuint32_t box[3] = {16, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr),
                           dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) inner=%lld rows=%lld ld=%lld",
             static_cast<int>(r), inner, rows, ld);
    return set_error(ctx, DNGD_ERR_CUDA, buf);
  }
  return DNGD_OK;
}

template <int BM, int BN, int WM, int WN, int STAGES>
static int launch_gemm(dngd_ctx* ctx, cudaStream_t s, const GemmCall& g) {
  using Cfg = GemmCfg<BM, BN, WM, WN, STAGES>;
  auto kern = k_gemm_nt<BM, BN, WM, WN, STAGES>;
  static std::atomic<bool> attr_set[64];  // per device (idempotent, race-free)
  if (!attr_set[ctx->device & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return cuda_status(ctx, e, "gemm smem attribute");
    attr_set[ctx->device & 63] = true;
  }
  CUtensorMap ta, tb;
  int rc = encode_map(ctx, &ta, g.A, g.K, g.M, g.batch, g.lda, g.sA, BM);
  if (rc) return rc;
  rc = encode_map(ctx, &tb, g.B, g.K, g.N, g.batch, g.ldb, g.sB, BN);
  if (rc) return rc;
  GemmDev p;
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  const long long tiles_m = (g.M + BM - 1) / BM, tiles_n = (g.N + BN - 1) / BN;
  if (g.lower) {
    p.ntiles = static_cast<int>(tiles_m * (tiles_m + 1) / 2);
  } else {
    p.ntiles = static_cast<int>(tiles_m * tiles_n);
  }
  p.tiles_n = static_cast<int>(tiles_n);
  const long long kc_total = (g.K + 15) / 16;
  p.kchunks = static_cast<int>((kc_total + g.splits - 1) / g.splits);
  p.lower = g.lower;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.C = g.C;
  p.ldc = g.ldc;
  p.sC = g.sC;
  p.partial = g.partial;
  p.vec_ok = ((g.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 &&
              (g.batch <= 1 || (g.sC & 1) == 0))
                 ? 1
                 : 0;
  dim3 grid(static_cast<unsigned>(static_cast<long long>(p.ntiles) * g.splits),
            static_cast<unsigned>(std::max(g.batch, 1)));
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, s>>>(ta, tb, p);
  return cuda_status(ctx, cudaGetLastError(), "gemm launch");
}

int gemm_nt(dngd_ctx* ctx, cudaStream_t s, const GemmCall& g) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return DNGD_OK;
  if (g.K <= 0) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gemm_nt: K must be positive");
  }
  if (g.lower && g.partial == nullptr && g.K <= 256) {
    // short-K lower updates (Cholesky trailing updates): small tiles, several
    // CTAs per SM so one CTA's read-modify-write epilogue hides behind another's
    // DMMA main loop
    return launch_gemm<64, 64, 2, 2, 4>(ctx, s, g);
  }
  if (g.lower || g.partial != nullptr || g.N > 64) {
    return launch_gemm<128, 128, 2, 4, 5>(ctx, s, g);
  }
  if (g.N > 32) return launch_gemm<128, 64, 4, 2, 4>(ctx, s, g);
  return launch_gemm<128, 32, 4, 1, 4>(ctx, s, g);
}

// ------------------------------------------------------------------ split-K GEMM
// For small outputs with a long reduction (J^T w over activation rows): S splits
// write raw 128x128 partial tiles, a fixed-order reduction applies alpha / beta.

// 256 threads = 64 output elements x 4 quarters of the splits; each quarter sums
// its contiguous split range in order, the quarters are added in order.
__global__ void __launch_bounds__(256) k_splitk_reduce(const double* __restrict__ partial,
                                                         int splits, int ntiles, int tiles_n,
                                                         long long M, long long N,
                                                         double* __restrict__ C, long long ldc,
                                                         double alpha, double beta) {
  __shared__ double sh[4][64];
  const int lane64 = threadIdx.x & 63, quarter = threadIdx.x >> 6;
  const long long e = static_cast<long long>(blockIdx.x) * 64 + lane64;
  const long long tile_elems = 128 * 128;
  const bool valid = e < static_cast<long long>(ntiles) * tile_elems;
  double v = 0.0;
  if (valid) {
    const int per = (splits + 3) / 4;
    const int s0 = quarter * per, s1 = min(splits, s0 + per);
    const double* src = partial + e;
    const long long sstride = static_cast<long long>(ntiles) * tile_elems;
    int s = s0;
    for (; s + 8 <= s1; s += 8) {  // loads issued ahead of the in-order sum
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldcs(src + (s + u) * sstride);
#pragma unroll
      for (int u = 0; u < 8; ++u) v += a[u];
    }
    for (; s < s1; ++s) v += __ldcs(src + s * sstride);
  }
  sh[quarter][lane64] = v;
  __syncthreads();
  if (quarter != 0 || !valid) return;
  v = ((sh[0][lane64] + sh[1][lane64]) + sh[2][lane64]) + sh[3][lane64];
  const int t = static_cast<int>(e / tile_elems);
  const int off = static_cast<int>(e - t * tile_elems);
  const int tm = t / tiles_n, tn = t - (t / tiles_n) * tiles_n;
  const long long r = static_cast<long long>(tm) * 128 + off / 128;
  const long long c = static_cast<long long>(tn) * 128 + off % 128;
  if (r >= M || c >= N) return;
  double* cp = C + r * ldc + c;
  *cp = alpha * v + (beta != 0.0 ? beta * *cp : 0.0);
}

size_t gemm_splitk_bytes(long long M, long long N, int splits) {
  const long long tiles = ((M + 127) / 128) * ((N + 127) / 128);
  return static_cast<size_t>(splits) * tiles * 128 * 128 * sizeof(double);
}

int gemm_splitk_choose(dngd_ctx* ctx, long long M, long long N, long long K) {
  const long long tiles = ((M + 127) / 128) * ((N + 127) / 128);
  long long s = (2LL * ctx->num_sms + tiles - 1) / tiles;
  s = std::min(s, std::max(1LL, ((K + 15) / 16) / 4));  // >= 64 columns of K per split
  return static_cast<int>(std::max(1LL, std::min(s, 64LL)));
}

int gemm_nt_splitk(dngd_ctx* ctx, cudaStream_t s, const GemmCall& g0, int splits,
                   double* partial, size_t partial_bytes) {
  if (g0.M <= 0 || g0.N <= 0) return DNGD_OK;
  if (partial == nullptr || partial_bytes < gemm_splitk_bytes(g0.M, g0.N, splits)) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gemm_nt_splitk: workspace too small");
  }
  GemmCall g = g0;
  g.lower = 0;
  g.batch = 1;
  g.splits = splits;
  g.partial = partial;
  int rc = launch_gemm<128, 128, 2, 4, 5>(ctx, s, g);
  if (rc) return rc;
  const int tiles_n = static_cast<int>((g.N + 127) / 128);
  const int ntiles = static_cast<int>(((g.M + 127) / 128) * tiles_n);
  const long long total = static_cast<long long>(ntiles) * 128 * 128;
  k_splitk_reduce<<<static_cast<unsigned>((total + 63) / 64), 256, 0, s>>>(
      partial, splits, ntiles, tiles_n, g.M, g.N, g.C, g.ldc, g.alpha, g.beta);
  return cuda_status(ctx, cudaGetLastError(), "splitk reduce");
}

// ------------------------------------------------------------------ SYRK

constexpr int kSyrkTile = 128;

// Sum split partials in fixed order and write the full symmetric K.
// Each CTA owns one 16x16 sub-block of a lower tile (64 per tile: a single-tile K,
// the STDE case, still spreads over the SMs); loads of consecutive splits are
// issued ahead of the in-order sum.  The transposed copy goes through shared
// memory so both writes are coalesced.
__global__ void __launch_bounds__(256) k_syrk_reduce(const double* __restrict__ partial,
                                                       int splits, int ntiles, long long m,
                                                       double* __restrict__ K, long long ldK,
                                                       int accumulate) {
  __shared__ double sh[16][17];
  const int t = blockIdx.x >> 6;
  const int sub = blockIdx.x & 63;
  int ti, tj;
  decode_lower(t, ti, tj);
  const int sr = sub >> 3, sc = sub & 7;
  if (ti == tj && sc > sr) return;  // above the diagonal of a diagonal tile
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long r0 = static_cast<long long>(ti) * kSyrkTile + sr * 16;
  const long long c0 = static_cast<long long>(tj) * kSyrkTile + sc * 16;
  if (r0 >= m || c0 >= m) return;
  const long long tile_elems = kSyrkTile * kSyrkTile;
  const double* src = partial + static_cast<long long>(t) * tile_elems +
                      (sr * 16 + ty) * kSyrkTile + sc * 16 + tx;
  const long long sstride = static_cast<long long>(ntiles) * tile_elems;
  double v = 0.0;
  int s = 0;
  for (; s + 8 <= splits; s += 8) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldcs(src + (s + u) * sstride);
#pragma unroll
    for (int u = 0; u < 8; ++u) v += a[u];
  }
  for (; s < splits; ++s) v += __ldcs(src + s * sstride);
  const long long r = r0 + ty, c = c0 + tx;
  if (r < m && c < m && c <= r) {
    if (accumulate) v += K[r * ldK + c];
    K[r * ldK + c] = v;
  }
  sh[ty][tx] = v;
  __syncthreads();
  // upper element K[c0+ty][r0+tx] mirrors lower element (r0+tx, c0+ty)
  const long long ru = c0 + ty, cu = r0 + tx;
  if (ru < m && cu < m && ru < cu) K[ru * ldK + cu] = sh[tx][ty];
}

int syrk_plan(dngd_ctx* ctx, long long m, long long ncols, int* splits, long long* ntiles,
              size_t* work_bytes) {
  const long long T = (m + kSyrkTile - 1) / kSyrkTile;
  const long long nt = T * (T + 1) / 2;
  const long long kc_total = std::max(1LL, (ncols + 15) / 16);
  const int conc = ctx->num_sms;  // 1 CTA / SM (160 KB of TMA stages)
  auto eff = [&](int S) {
    const long long units = nt * S;
    const long long waves = (units + conc - 1) / conc;
    return static_cast<double>(units) / static_cast<double>(waves * conc);
  };
  int best = 1;
  // up to two waves of splits: a tiny m (few tiles) over a huge K (the STDE case,
  // m = 100, n = 12.85M) needs every SM on the K reduction
  for (int S = 2; S <= 2 * conc; ++S) {
    if ((kc_total + S - 1) / S < 8) break;  // keep >= 128 columns of K per unit
    if (eff(S) > eff(best) + 0.03) best = S;
  }
  *splits = best;
  *ntiles = nt;
  *work_bytes = static_cast<size_t>(best) * nt * kSyrkTile * kSyrkTile * sizeof(double);
  return DNGD_OK;
}

int syrk(dngd_ctx* ctx, cudaStream_t s, const double* J, long long m, long long ncols,
         long long ldJ, double* K, long long ldK, int accumulate, void* work, size_t wb) {
  if (m <= 0) return DNGD_OK;
  int S;
  long long nt;
  size_t need;
  syrk_plan(ctx, m, ncols, &S, &nt, &need);
  if (work == nullptr || wb < need) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "syrk: workspace too small");
  }
  GemmCall g;
  g.M = m;
  g.N = m;
  g.K = std::max(1LL, ncols);
  g.A = J;
  g.lda = ldJ;
  g.B = J;
  g.ldb = ldJ;
  g.lower = 1;
  g.splits = S;
  g.partial = static_cast<double*>(work);
  if (ncols <= 0) {
    cudaError_t e = cudaMemsetAsync(work, 0, need, s);
    if (e != cudaSuccess) return cuda_status(ctx, e, "syrk memset");
  } else {
    int rc = launch_gemm<128, 128, 2, 4, 5>(ctx, s, g);
    if (rc) return rc;
  }
  k_syrk_reduce<<<static_cast<unsigned>(nt * 64), 256, 0, s>>>(
      static_cast<const double*>(work), S, static_cast<int>(nt), m, K, ldK, accumulate);
  return cuda_status(ctx, cudaGetLastError(), "syrk reduce");
}

}  // namespace dngd
