// HBM-streaming FP64 matvecs over the materialised Jacobian and small vector
// kernels for the PCG loop.
//
//   gemv_t : out = scale * (J^T y + g)  -- one pass over J (reference vjp,
//            residuals.py:220-227, used at solver.py:200,210,335,360) with the
//            dual-to-primal epilogue -(J^T y + g)/lam of solver.py:200 fused.
//   gemv_n : out = alpha * A x + beta * add -- J g (jvp, solver.py:198,315),
//            K f_vv (solver.py:208), J (J^T p) (solver.py:336).
// Both are deterministic (fixed reduction order): bitwise-reproducible steps.

#include <math_constants.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace dngd {

constexpr int kGT = 256;       // threads per CTA
constexpr int kGTV = 4;                // double2 per thread per row

static void gemv_t_plan(dngd_ctx* ctx, long long m, long long ncols, int* nchunks) {
  const long long cols = 2LL * kGT * kGTV;  // 2048: measured best of 1024 / 2048 / 4096
  const long long col_tiles = (ncols + cols - 1) / cols;
  const long long target = 4LL * ctx->num_sms;
  long long nc = (target + col_tiles - 1) / col_tiles;
  nc = std::min(nc, std::max(1LL, m / 16));
  *nchunks = static_cast<int>(std::max(1LL, nc));
}

// J row-major (m x ncols, ld even, 16B-aligned).  A CTA streams a strip of
// 512 V columns (V x 4 KB contiguous per row) over a chunk of rows; thread t
// owns the double2 column pairs t + 256 v, so every load instruction of a warp
// covers 512 contiguous bytes.  A pair at column c < ncols is always inside the
// row's ld (ld even), so odd ncols need no scalar tail.  grid.y = row chunks;
// partial sums go to a fixed-order reduction (deterministic).
template <int V>
__global__ void __launch_bounds__(kGT) k_gemv_t(const double* __restrict__ J, long long m,
                                                  long long ncols, long long ld,
                                                  const double* __restrict__ y, int nchunks,
                                                  const double* __restrict__ g, double scale,
                                                  double* __restrict__ out,
                                                  double* __restrict__ partial) {
  const long long c0 = static_cast<long long>(blockIdx.x) * (2 * kGT * V) + 2LL * threadIdx.x;
  const long long rows_per = (m + nchunks - 1) / nchunks;
  const long long i0 = blockIdx.y * rows_per;
  const long long i1 = min(m, i0 + rows_per);
  double2 acc[V];
  bool ok[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    acc[v] = make_double2(0.0, 0.0);
    ok[v] = c0 + 2LL * kGT * v < ncols;
  }
  const double* p = J + i0 * ld + c0;
  long long i = i0;
  for (; i + 1 < i1; i += 2) {
    double2 u[2][V];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int v = 0; v < V; ++v)
        u[k][v] = ok[v] ? __ldcs(reinterpret_cast<const double2*>(p + k * ld + 2 * kGT * v))
                        : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double yk = __ldg(y + i + k);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        acc[v].x = fma(u[k][v].x, yk, acc[v].x);
        acc[v].y = fma(u[k][v].y, yk, acc[v].y);
      }
    }
    p += 2 * ld;
  }
  if (i < i1) {
    const double yk = __ldg(y + i);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (ok[v]) {
        const double2 u = __ldcs(reinterpret_cast<const double2*>(p + 2 * kGT * v));
        acc[v].x = fma(u.x, yk, acc[v].x);
        acc[v].y = fma(u.y, yk, acc[v].y);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const long long c = c0 + 2LL * kGT * v;
    if (!ok[v]) continue;
    if (nchunks == 1) {
      out[c] = scale * (acc[v].x + (g ? g[c] : 0.0));
      if (c + 1 < ncols) out[c + 1] = scale * (acc[v].y + (g ? g[c + 1] : 0.0));
    } else {
      double* dst = partial + static_cast<long long>(blockIdx.y) * ncols + c;
      dst[0] = acc[v].x;
      if (c + 1 < ncols) dst[1] = acc[v].y;
    }
  }
}

__global__ void k_gemv_t_reduce(const double* __restrict__ partial, int nchunks, long long ncols,
                                const double* __restrict__ g, double scale,
                                double* __restrict__ out) {
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  double s = 0.0;
  int k = 0;
  // 8 loads in flight, added in the same (chunk) order as one at a time
  for (; k + 8 <= nchunks; k += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = partial[static_cast<long long>(k + j) * ncols + c];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; k < nchunks; ++k) s += partial[static_cast<long long>(k) * ncols + c];
  out[c] = scale * (s + (g ? g[c] : 0.0));
}

// out[i] = alpha * A[i,:] . x + beta * add[i]; one CTA (NT threads) per row.
template <int NT>
__global__ void __launch_bounds__(NT) k_gemv_n_row(const double* __restrict__ A, long long m,
                                                      long long ncols, long long ld,
                                                      const double* __restrict__ x, double alpha,
                                                      const double* __restrict__ add, double beta,
                                                      double* __restrict__ out, int vec) {
  __shared__ double sh[NT / 32];
  const long long i = blockIdx.x;
  const double* a = A + i * ld;
  double s0 = 0, s1 = 0;
  if (vec) {
    const long long n2 = ncols / 2;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (long long k = threadIdx.x; k < n2; k += NT) {
      const double2 u = __ldcs(a2 + k);
      const double2 v = __ldg(x2 + k);
      s0 = fma(u.x, v.x, s0);
      s1 = fma(u.y, v.y, s1);
    }
    if ((ncols & 1) && threadIdx.x == 0) s0 = fma(a[ncols - 1], x[ncols - 1], s0);
  } else {
    for (long long k = threadIdx.x; k < ncols; k += NT) s0 = fma(a[k], x[k], s0);
  }
  const double s = block_sum<NT>(s0 + s1, sh);
  if (threadIdx.x == 0) out[i] = alpha * s + (add ? beta * add[i] : 0.0);
}

// short rows: one warp per row
__global__ void __launch_bounds__(256) k_gemv_n_warp(const double* __restrict__ A, long long m,
                                                       long long ncols, long long ld,
                                                       const double* __restrict__ x,
                                                       double alpha,
                                                       const double* __restrict__ add,
                                                       double beta, double* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= m) return;
  const double* a = A + i * ld;
  double s = 0.0;
  for (long long k = lane; k < ncols; k += 32) s = fma(a[k], __ldg(x + k), s);
  s = warp_sum(s);
  if (lane == 0) out[i] = alpha * s + (add ? beta * add[i] : 0.0);
}

__global__ void __launch_bounds__(1024) k_dot(long long n, const double* __restrict__ x,
                                                const double* __restrict__ y,
                                                double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long k = threadIdx.x; k < n; k += 1024) s = fma(x[k], y[k], s);
  s = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

// large n: kDotBlocks contiguous chunks, one partial per CTA, the last CTA to
// arrive sums the partials in index order (deterministic, one launch)
__global__ void __launch_bounds__(512) k_dot_multi(long long n, const double* __restrict__ x,
                                                     const double* __restrict__ y,
                                                     double* __restrict__ part,
                                                     unsigned* __restrict__ counter,
                                                     double* __restrict__ out) {
  __shared__ double sh[32];
  __shared__ bool last;
  const long long chunk = (n + kDotBlocks - 1) / kDotBlocks;
  const long long k0 = blockIdx.x * chunk, k1 = min(n, k0 + chunk);
  double s = 0.0;
  for (long long k = k0 + threadIdx.x; k < k1; k += 512) s = fma(x[k], y[k], s);
  s = block_sum<512>(s, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = threadIdx.x < kDotBlocks ? __ldcg(part + threadIdx.x) : 0.0;
  t = block_sum<512>(t, sh);
  if (threadIdx.x == 0) {
    *out = t;
    *counter = 0u;
  }
}

__global__ void k_axpby(long long n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) out[k] = fma(a, x[k], y ? b * y[k] : 0.0);
}

// line-search selection + accept/reject bookkeeping on the device (one warp)
__global__ void k_ls_select(const double* __restrict__ losses, int ncand,
                            const double* __restrict__ etas, const double* __restrict__ rr,
                            const double* __restrict__ info, const double* __restrict__ anyd,
                            int reject_if_worse, double* __restrict__ mult,
                            double* __restrict__ sel) {
  const int lane = threadIdx.x;
  // first minimum over the finite losses: (value, index) min-reduction
  double best = CUDART_INF;
  int bi = 0x7fffffff;
  for (int k = lane; k < ncand; k += 32) {
    const double v = losses[k];
    if (isfinite(v) && (v < best || (v == best && k < bi))) {
      best = v;
      bi = k;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  if (lane != 0) return;
  const double loss = 0.5 * rr[0];
  double eta = 1.0, lsl = loss, status = 0.0, idx = 0.0;
  if (!isfinite(loss)) {
    status = 3.0;
  } else if (*info != 0.0) {
    status = 2.0;
  } else if (*anyd == 0.0) {
    // zero step: accepted with eta = 1 and the current loss (optimizer.py:222-223)
  } else if (bi == 0x7fffffff) {
    status = 1.0;
    lsl = CUDART_NAN;
  } else {
    eta = etas[bi];
    lsl = best;
    idx = bi;
    if (reject_if_worse && best > loss) status = 1.0;
  }
  if (status == 0.0) {
    *mult = 1.0;
  } else if (status == 1.0) {
    *mult = 10.0 * *mult;
  }
  sel[0] = eta;
  sel[1] = lsl;
  sel[2] = status;
  sel[3] = idx;
}

// grid-stride; the any-nonzero flag is one store per CTA at most (a store per
// warp from ~10^5 warps to one address serialises in L2)
__global__ void __launch_bounds__(256) k_ga_combine(long long n, const double* v,
                                                      const double* __restrict__ a,
                                                      const double* __restrict__ scal, double* out,
                                                      double* anyd) {
  bool take = false;
  if (a != nullptr) {
    const double vn = sqrt(scal[2]), an = sqrt(scal[3]);
    take = vn > 1e-12 && 2.0 * an <= 0.5 * vn;  // GA_NORM_GUARD, GA_RATIO_MAX
  }
  bool nz = false;
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double vk = v[k];
    const double d = take ? fma(0.5, a[k], vk) : vk;  // == v + 0.5 a (0.5 a is exact)
    out[k] = d;
    nz |= d != 0.0;
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0 &&
      *reinterpret_cast<volatile double*>(anyd) == 0.0) {
    *anyd = 1.0;  // order-free
  }
}

__global__ void k_theta_update(long long n, const double* __restrict__ theta,
                               const double* __restrict__ delta, const double* __restrict__ sel,
                               double* out) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const bool take = sel[2] == 0.0;
  const double t = theta[k];
  out[k] = take ? fma(sel[0], delta[k], t) : t;  // == dngd_axpby(eta, delta, 1, theta)
}

}  // namespace dngd

using namespace dngd;

extern "C" int dngd_gemv_t_workspace(dngd_ctx* ctx, int64_t m, int64_t ncols, size_t* bytes) {
  int nc;
  gemv_t_plan(ctx, m, ncols, &nc);
  *bytes = nc > 1 ? static_cast<size_t>(nc) * ncols * sizeof(double) : 0;
  return DNGD_OK;
}

extern "C" int dngd_gemv_t(dngd_ctx* ctx, void* stream, const double* J, int64_t m,
                           int64_t ncols, int64_t ldJ, const double* y, const double* g,
                           double scale, double* out, void* work, size_t work_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (ncols <= 0) return DNGD_OK;
  if ((ldJ & 1) || (reinterpret_cast<uintptr_t>(J) & 15)) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gemv_t: J needs an even leading dimension");
  }
  if (m <= 0) {
    k_axpby<<<static_cast<unsigned>((ncols + 255) / 256), 256, 0, s>>>(ncols, 0.0, g ? g : out,
                                                                       scale, g, out);
    return cuda_status(ctx, cudaGetLastError(), "gemv_t empty");
  }
  int nc;
  gemv_t_plan(ctx, m, ncols, &nc);
  if (nc > 1 && (work == nullptr || work_bytes < static_cast<size_t>(nc) * ncols * 8)) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gemv_t: workspace too small");
  }
  const long long cols = 2LL * kGT * kGTV;
  dim3 grid(static_cast<unsigned>((ncols + cols - 1) / cols), static_cast<unsigned>(nc));
  k_gemv_t<kGTV><<<grid, kGT, 0, s>>>(J, m, ncols, ldJ, y, nc, g, scale, out,
                                      static_cast<double*>(work));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(ctx, e, "gemv_t");
  if (nc > 1) {
    k_gemv_t_reduce<<<static_cast<unsigned>((ncols + 255) / 256), 256, 0, s>>>(
        static_cast<const double*>(work), nc, ncols, g, scale, out);
    e = cudaGetLastError();
  }
  return cuda_status(ctx, e, "gemv_t reduce");
}

extern "C" int dngd_gemv_n(dngd_ctx* ctx, void* stream, const double* A, int64_t m,
                           int64_t ncols, int64_t ldA, const double* x, double alpha,
                           const double* add, double beta, double* out) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (m <= 0) return DNGD_OK;
  if (ncols >= 2048) {
    const int vec = ((ldA & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(x) & 15) == 0)
                        ? 1
                        : 0;
    // short rows (K at m ~ 3000): 128 threads, more rows in flight per SM
    if (ncols < 8192) {
      k_gemv_n_row<128><<<static_cast<unsigned>(m), 128, 0, s>>>(A, m, ncols, ldA, x, alpha, add,
                                                                 beta, out, vec);
    } else {
      k_gemv_n_row<256><<<static_cast<unsigned>(m), 256, 0, s>>>(A, m, ncols, ldA, x, alpha, add,
                                                                 beta, out, vec);
    }
  } else {
    k_gemv_n_warp<<<static_cast<unsigned>((m + 7) / 8), 256, 0, s>>>(A, m, ncols, ldA, x, alpha,
                                                                      add, beta, out);
  }
  return cuda_status(ctx, cudaGetLastError(), "gemv_n");
}

extern "C" int dngd_dot(dngd_ctx* ctx, void* stream, int64_t n, const double* x, const double* y,
                        double* out_dev) {
  if (n >= (1LL << 18)) {
    k_dot_multi<<<kDotBlocks, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        n, x, y, ctx->dot_part, ctx->dot_counter, out_dev);
  } else {
    k_dot<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(n, x, y, out_dev);
  }
  return cuda_status(ctx, cudaGetLastError(), "dot");
}

extern "C" int dngd_ls_select(dngd_ctx* ctx, void* stream, const double* losses, int ncand,
                              const double* etas, const double* rr, const double* info,
                              const double* anyd, int reject_if_worse, double* mult,
                              double* sel) {
  if (ncand < 1) return set_error(ctx, DNGD_ERR_DIMENSION, "ls_select: no candidates");
  k_ls_select<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(losses, ncand, etas, rr, info, anyd,
                                                               reject_if_worse, mult, sel);
  return cuda_status(ctx, cudaGetLastError(), "ls_select");
}

extern "C" int dngd_ga_combine(dngd_ctx* ctx, void* stream, int64_t n, const double* v,
                               const double* a, const double* scal, double* out, double* anyd) {
  if (n <= 0) return DNGD_OK;
  const long long blocks = std::min<long long>((n + 255) / 256, 8LL * ctx->num_sms);
  k_ga_combine<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n, v, a, scal, out, anyd);
  return cuda_status(ctx, cudaGetLastError(), "ga_combine");
}

extern "C" int dngd_theta_update(dngd_ctx* ctx, void* stream, int64_t n, const double* theta,
                                 const double* delta, const double* sel, double* out) {
  if (n <= 0) return DNGD_OK;
  k_theta_update<<<static_cast<unsigned>((n + 255) / 256), 256, 0,
                   static_cast<cudaStream_t>(stream)>>>(n, theta, delta, sel, out);
  return cuda_status(ctx, cudaGetLastError(), "theta_update");
}

extern "C" int dngd_axpby(dngd_ctx* ctx, void* stream, int64_t n, double a, const double* x,
                          double b, const double* y, double* out) {
  if (n <= 0) return DNGD_OK;
  k_axpby<<<static_cast<unsigned>((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n, a, x, b, y, out);
  return cuda_status(ctx, cudaGetLastError(), "axpby");
}

// ---------------------------------------------------------------- non-finite report
namespace dngd {
__global__ void k_first_nonfinite(const double* __restrict__ x, long long n,
                                  unsigned long long* __restrict__ first) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && !isfinite(x[i])) atomicMin(first, static_cast<unsigned long long>(i));
}
}  // namespace dngd

extern "C" int dngd_nonfinite_report(dngd_ctx* ctx, void* stream, const double* x, int64_t n,
                                     const int64_t* class_ends, int nclass, int* class_out,
                                     int64_t* point_out) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (class_out) *class_out = -1;
  if (point_out) *point_out = -1;
  if (n <= 0) return DNGD_OK;
  cudaError_t e = cudaMemsetAsync(ctx->nf_word, 0xff, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_status(ctx, e, "nonfinite_report");
  dngd::k_first_nonfinite<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, n, ctx->nf_word);
  unsigned long long first = ~0ull;
  e = cudaMemcpyAsync(&first, ctx->nf_word, sizeof first, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(ctx, e, "nonfinite_report");
  if (first >= static_cast<unsigned long long>(n)) return DNGD_OK;
  long long row = static_cast<long long>(first), start = 0;
  int cls = -1;
  for (int c = 0; c < nclass; ++c) {
    if (row < class_ends[c]) {
      cls = c;
      break;
    }
    start = class_ends[c];
  }
  if (class_out) *class_out = cls;
  if (point_out) *point_out = cls >= 0 ? row - start : row;
  char buf[128];
  snprintf(buf, sizeof buf, "non-finite value in class %d at point %lld", cls,
           static_cast<long long>(cls >= 0 ? row - start : row));
  return dngd::set_error(ctx, DNGD_ERR_NONFINITE, buf);
}

