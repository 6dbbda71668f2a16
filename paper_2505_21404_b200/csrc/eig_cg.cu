// The small dense numerics of the Nystrom-PCG step (reference solver.py:237-366),
// hand-written so no library eigensolver and no host round trip sit on the path:
//
//  * dngd_syev_jacobi -- symmetric eigendecomposition of the l x l landmark block
//    K_II (solver.py:264, scipy eigh) by block one-sided (Hestenes) Jacobi: one
//    cooperative persistent kernel, one grid barrier per outer round of block
//    pairs (see below), threshold rotations until a sweep rotates nothing.
//    Eigenpairs come back unsorted (the preconditioner does not depend on order).
//
//  * dngd_nystrom_scale -- W[j] = V[:, j] / sqrt(lambda_j) for the kept
//    eigenpairs (lambda_j > 1e-10 lambda_max, else a zero column), the row scale
//    of U~ sqrt(Lambda) = K[:, I] Q Lambda^{-1/2} with U~[I] = Q (solver.py:269-274).
//
//  * dngd_cg_* -- the PCG control flow of solver.py:321-366 on the device: the
//    CG scalars (rho, alpha, |r|, best |r|, iteration, stop flag, warning) live
//    in a state block; the vector updates are gated by the stop flag; the last
//    kernel of an iteration sets the WHILE condition of a CUDA graph conditional
//    node (dngd_graph_*), so the whole CG loop runs as one graph launch with no
//    host synchronisation per iteration.

#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace dngd {

// ---------------------------------------------------------------- Jacobi eigensolver
//
// Block one-sided (Hestenes) Jacobi on the PSD matrix X: the columns of Y = X V are
// orthogonalised by plane rotations, V accumulating them; at convergence
// X V = V diag(lambda) with lambda_j = |Y_j| (X PSD).  Columns are cut into 2B
// blocks of bs; an outer round gives each of B CTAs one block pair (round-robin),
// the CTA holds the 2 bs rows of Y^T in shared memory, runs one inner cyclic
// sweep over all column pairs of the pair (one warp per rotation, shuffle
// reductions for the three dot products); one grid barrier per outer round (31
// per sweep at l = 512, bs = 16).  Rotations below eps sqrt(a.a b.b) are skipped;
// converged when a whole sweep rotates nothing.  Each pair's rotations are also
// accumulated (2bs x 2bs) and applied to its rows of V^T.

constexpr int kJT = 512;  // threads per CTA (16 warps)

struct JacobiArgs {
  double* Yt;  // N x ld: rows = columns of Y
  double* Vt;  // N x ld: rows = columns of V (the accumulated rotations)
  int N;       // padded order = 2 B bs
  int n;       // true order
  int bs;      // columns per block
  int nblk;    // 2 B
  long long ld;
  int max_sweeps;
  double eps;
  const double* fro2;  // |X|_F^2 (device): the absolute rotation floor (eps |X|_F)^2
  unsigned* rotated;  // [max_sweeps] flags
  int* sweeps_out;
  long long* trace;   // DNGD_JACOBI_TRACE builds only: clock64 marks of CTA 0
};

// pair k of round t of the round-robin tournament on M (even) indices: (p, q), p < q
DNGD_DEV void jac_pair(int k, int t, int M, int& p, int& q) {
  const int R = M - 1;
  int a, b;
  if (k == 0) {
    a = t;
    b = R;
  } else {
    a = (t + k) % R;
    b = (t - k + R) % R;
  }
  p = min(a, b);
  q = max(a, b);
}

// JR > 0: the pair's rows live in registers (N <= 32 JR); JR = 0: any N, shared only
template <int JR>
__global__ void __launch_bounds__(kJT) k_jacobi(JacobiArgs J) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double jsm[];
  const int N = J.N, bs = J.bs, rows = 2 * bs;
  const int sp = N + 1;  // smem row pitch
  double* S = jsm;       // rows x sp: this pair's rows of Y^T
  double* Rt = jsm + 2 * bs * sp;  // rows x rows: the pair's accumulated rotation (row form)
  __shared__ int s_rot;
  // rotations keep the relative criterion |a.b| > eps |a| |b| (full accuracy for
  // every column pair that matters) except between two columns both below
  // 1e-13 |X|: such pairs (far under the preconditioner's 1e-10 lambda_max floor,
  // down to pure rounding noise on the numerically rank-deficient Gram blocks of
  // a PINN) would otherwise keep rotating noise and never let the sweeps stop
  const double abs_tol = 1e-26 * (*J.fro2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int B = J.nblk / 2;
#ifdef DNGD_JACOBI_TRACE
  int nt = 0;
#define JTRACE() if (blockIdx.x == 0 && threadIdx.x == 0 && nt < 256 && J.trace) J.trace[nt++] = clock64();
#else
#define JTRACE()
#endif
  int sweep = 0;
  for (; sweep < J.max_sweeps; ++sweep) {
    for (int t = 0; t < J.nblk - 1; ++t) {
      JTRACE()
      if (static_cast<int>(blockIdx.x) < B) {
        int bi, bj;
        jac_pair(blockIdx.x, t, J.nblk, bi, bj);
        // rows of Y^T: local r < bs -> block bi, r >= bs -> block bj
        // all of a thread's row loads in flight before the shared stores (L2 latency
        // once per outer round, not once per element)
        for (int e0 = threadIdx.x; e0 < rows * N; e0 += 8 * blockDim.x) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            v[u] = 0.0;
            if (e < rows * N) {
              const int r = e / N, c = e - r * N;
              v[u] = J.Yt[static_cast<long long>(r < bs ? bi * bs + r : bj * bs + (r - bs)) * J.ld + c];
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * blockDim.x;
            if (e < rows * N) {
              const int r = e / N, c = e - r * N;
              S[r * sp + c] = v[u];
            }
          }
        }
        for (int e = threadIdx.x; e < rows * rows; e += blockDim.x)
          Rt[e] = (e / rows) == (e % rows) ? 1.0 : 0.0;
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        JTRACE()
        // one inner cyclic sweep over all column pairs of the 2 bs rows
        for (int ir = 0; ir < rows - 1; ++ir) {
          for (int k = warp; k < bs; k += nwarps) {
            int a, b;
            jac_pair(k, ir, rows, a, b);
            double* ra = S + a * sp;
            double* rb = S + b * sp;
            // the pair's rows in registers (N <= 32 JR) for the dots and the update
            constexpr int R = JR > 0 ? JR : 1;
            double xr[R], yr[R];
            double aa = 0.0, bb = 0.0, ab = 0.0;
            if constexpr (JR > 0) {
#pragma unroll
              for (int u = 0; u < JR; ++u) {
                const int c = lane + 32 * u;
                xr[u] = c < N ? ra[c] : 0.0;
                yr[u] = c < N ? rb[c] : 0.0;
              }
#pragma unroll
              for (int u = 0; u < JR; ++u) {
                aa = fma(xr[u], xr[u], aa);
                bb = fma(yr[u], yr[u], bb);
                ab = fma(xr[u], yr[u], ab);
              }
            } else {
              for (int c = lane; c < N; c += 32) {
                const double x = ra[c], y = rb[c];
                aa = fma(x, x, aa);
                bb = fma(y, y, bb);
                ab = fma(x, y, ab);
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              aa += __shfl_xor_sync(0xffffffffu, aa, o);
              bb += __shfl_xor_sync(0xffffffffu, bb, o);
              ab += __shfl_xor_sync(0xffffffffu, ab, o);
            }
            if (fabs(ab) > fmax(J.eps * sqrt(aa * bb), abs_tol)) {
              const double zeta = (bb - aa) / (2.0 * ab);
              const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
              const double c = 1.0 / sqrt(1.0 + tt * tt), s = tt * c;
              if constexpr (JR > 0) {
#pragma unroll
                for (int u = 0; u < JR; ++u) {
                  const int col = lane + 32 * u;
                  if (col < N) {
                    ra[col] = c * xr[u] - s * yr[u];
                    rb[col] = s * xr[u] + c * yr[u];
                  }
                }
              } else {
                for (int col = lane; col < N; col += 32) {
                  const double x = ra[col], y = rb[col];
                  ra[col] = c * x - s * y;
                  rb[col] = s * x + c * y;
                }
              }
              double* qa = Rt + a * rows;
              double* qb = Rt + b * rows;
              for (int col = lane; col < rows; col += 32) {
                const double x = qa[col], y = qb[col];
                qa[col] = c * x - s * y;
                qb[col] = s * x + c * y;
              }
              if (lane == 0) s_rot = 1;
            }
          }
          __syncthreads();
          JTRACE()
        }
        if (s_rot) {
          for (int r = 0; r < rows; ++r) {
            double* dst = J.Yt + static_cast<long long>(r < bs ? bi * bs + r : bj * bs + (r - bs)) * J.ld;
            for (int c = threadIdx.x; c < N; c += blockDim.x) dst[c] = S[r * sp + c];
          }
          // V^T rows <- Rt V^T rows: the eigenvectors as a product of rotations
          // (orthogonal to rounding: eigenvectors of tiny eigenvalues do not pick
          // up eps |X| / lambda_j of the large ones, as Y_j / |Y_j| would).  The
          // old rows are staged in S (free now), then every thread forms 4 rows of
          // one column from that column's 2 bs values held in registers.
          __syncthreads();
          for (int e0 = threadIdx.x; e0 < rows * N; e0 += 8 * blockDim.x) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int e = e0 + u * blockDim.x;
              v[u] = 0.0;
              if (e < rows * N) {
                const int r = e / N, c = e - r * N;
                v[u] = J.Vt[static_cast<long long>(r < bs ? bi * bs + r : bj * bs + (r - bs)) * J.ld + c];
              }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int e = e0 + u * blockDim.x;
              if (e < rows * N) {
                const int r = e / N, c = e - r * N;
                S[r * sp + c] = v[u];
              }
            }
          }
          __syncthreads();
          const int rgroups = rows / 4;  // rows is even; 4 | rows for bs >= 2
          for (int f = threadIdx.x; f < rgroups * N; f += blockDim.x) {
            const int g = f / N, c = f - g * N;
            double col[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) col[q] = q < rows ? S[q * sp + c] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int r = 4 * g + u;
              const double* rr = Rt + r * rows;
              double acc = 0.0;
#pragma unroll
              for (int q = 0; q < 32; ++q) {
                if (q < rows) acc = fma(rr[q], col[q], acc);
              }
              J.Vt[static_cast<long long>(r < bs ? bi * bs + r : bj * bs + (r - bs)) * J.ld + c] = acc;
            }
          }
          if (threadIdx.x == 0) J.rotated[sweep] = 1u;  // benign same-value race
        }
        JTRACE()
      }
      grid.sync();
    }
    const bool any = *(volatile unsigned*)&J.rotated[sweep] != 0u;
    grid.sync();
    if (!any) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *J.sweeps_out = sweep + 1;
}

// |X|_F^2 in a fixed order (one CTA): deterministic rotation decisions run to run
__global__ void k_fro2(const double* __restrict__ A, long long lda, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long e = threadIdx.x; e < static_cast<long long>(n) * n; e += blockDim.x) {
    const double a = A[(e / n) * lda + (e % n)];
    s = fma(a, a, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// X (n x n, lda) -> Yt = sym(X) padded to N x N (zero pad), Vt = I
__global__ void k_jacobi_init(const double* __restrict__ A, long long lda, int n, int N,
                              long long ld, double* __restrict__ Yt, double* __restrict__ Vt,
                              unsigned* __restrict__ rotated, int max_sweeps) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < max_sweeps) rotated[e] = 0u;
  if (e >= static_cast<long long>(N) * N) return;
  const int i = static_cast<int>(e / N), j = static_cast<int>(e - static_cast<long long>(i) * N);
  double a = 0.0;
  if (i < n && j < n) a = 0.5 * (A[static_cast<long long>(i) * lda + j] + A[static_cast<long long>(j) * lda + i]);
  Yt[i * ld + j] = a;
  Vt[i * ld + j] = i == j ? 1.0 : 0.0;
}

// w[j] = |Y_j| (row j of Y^T; X V = V diag(w) for PSD X), V[:, j] = row j of V^T
__global__ void k_jacobi_out(const double* __restrict__ Yt, const double* __restrict__ Vt,
                             long long ld, int n, double* __restrict__ w, double* __restrict__ V,
                             long long ldv) {
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double* y = Yt + static_cast<long long>(j) * ld;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) {
    s = fma(y[c], y[c], s);
    V[static_cast<long long>(c) * ldv + j] = Vt[static_cast<long long>(j) * ld + c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) w[j] = sqrt(s);
}

struct JacShape {
  int N, bs, nblk;
  long long ld;
  size_t smem;
};

static JacShape jac_shape(long long n) {
  JacShape sh;
  static const int bs_env = getenv("DNGD_JACOBI_BS") ? atoi(getenv("DNGD_JACOBI_BS")) : 8;
  int bs = std::max(2, std::min(16, bs_env));
  while (bs > 2 && static_cast<size_t>(2 * bs) * (n + 1) * 8 > 150 * 1024) bs /= 2;
  sh.bs = bs;
  const long long nb = (n + bs - 1) / bs;
  sh.nblk = static_cast<int>(std::max<long long>(2, (nb + 1) / 2 * 2));
  sh.N = sh.nblk * bs;
  sh.ld = sh.N + 2;
  sh.smem = (static_cast<size_t>(2 * bs) * (sh.N + 1) + static_cast<size_t>(4 * bs * bs)) * 8;
  return sh;
}

static size_t jacobi_bytes(long long n, int max_sweeps) {
  const JacShape sh = jac_shape(std::max<long long>(n, 1));
  const size_t mat = static_cast<size_t>(sh.N) * sh.ld * 8;
  return 2 * mat + 256 + static_cast<size_t>(max_sweeps) * 4 + 256;
}

// ---------------------------------------------------------------- pivoted Cholesky
//
// K_II ~ L L^T with diagonal pivoting, stopped once every remaining diagonal entry
// is <= tol * max diag (K_II - L L^T is PSD with trace <= l tol max diag, so every
// eigenvalue moves by at most that -- 1e-15 relative here, five orders under the
// preconditioner's 1e-10 lambda_max floor).  The Nystrom numerics then run on the
// k x k matrix L^T L (same nonzero eigenvalues) instead of l x l: k is the
// numerical rank of the landmark block, small for a PINN Gram (tens at config 5).
// One CTA; Lt (k x l) row j = column j of L.  Pivot ties go to the lower index.
constexpr int kPC = 1024;

__global__ void __launch_bounds__(kPC) k_pivchol(const double* __restrict__ K, long long ldk, int l,
                                                 double tol, int kmax, double* __restrict__ Lt,
                                                 long long ldl, double* __restrict__ d,
                                                 int* __restrict__ used, int* __restrict__ k_out) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  __shared__ double s_piv, s_dmax;
  __shared__ int s_p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < l; i += blockDim.x) {
    d[i] = K[static_cast<long long>(i) * ldk + i];
    used[i] = 0;
  }
  __syncthreads();
  int j = 0;
  for (; j < kmax; ++j) {
    // pivot: largest remaining diagonal (ties: lower index)
    double bv = -1.0;
    int bi = l;
    for (int i = tid; i < l; i += blockDim.x) {
      const double v = used[i] ? -1.0 : d[i];
      if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      s_v[warp] = bv;
      s_i[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = s_v[0];
      int p = s_i[0];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
        if (s_v[w] > v || (s_v[w] == v && s_i[w] < p)) {
          v = s_v[w];
          p = s_i[w];
        }
      }
      if (j == 0) s_dmax = v;
      s_p = p;
      s_piv = v;
    }
    __syncthreads();
    const int p = s_p;
    const double dp = s_piv;
    if (!(dp > tol * s_dmax) || p >= l) break;
    const double lpp = sqrt(dp);
    double* row = Lt + static_cast<long long>(j) * ldl;
    for (int i = tid; i < l; i += blockDim.x) {
      double v = 0.0;
      if (i == p) {
        v = lpp;
      } else if (!used[i]) {
        double acc = K[static_cast<long long>(i) * ldk + p];
        for (int t = 0; t < j; ++t) {
          const double* rt = Lt + static_cast<long long>(t) * ldl;
          acc = fma(-rt[i], rt[p], acc);
        }
        v = acc / lpp;
        d[i] -= v * v;
      }
      row[i] = v;
    }
    __syncthreads();
    if (tid == 0) used[p] = 1;
    __syncthreads();
  }
  if (tid == 0) *k_out = j;
}

// Qst[j, c] = sum_i W[i, j] Lt[i, c] (= sqrt(lam_j) V_j, V_j = L W_j / sqrt(lam_j)) and
// Wt[j, c] = Qst[j, c] / lam_j for the kept eigenpairs (lam_j > floor_rel max lam),
// zero rows otherwise; *rank = kept count.  W is the k x k eigenvector matrix of L^T L.
__global__ void k_nys_from_chol(const double* __restrict__ W, long long ldw, const double* __restrict__ lam,
                                int k, const double* __restrict__ Lt, long long ldl, int l,
                                double floor_rel, double* __restrict__ Wt, long long ldwt,
                                double* __restrict__ Qst, long long ldq, int* __restrict__ rank) {
  __shared__ double s_max;
  if (threadIdx.x == 0) {
    double mx = -CUDART_INF;
    for (int q = 0; q < k; ++q) mx = fmax(mx, lam[q]);
    s_max = mx;
    if (blockIdx.x == 0 && blockIdx.y == 0 && rank) {
      const double fl = floor_rel * fmax(mx, 0.0);
      int r = 0;
      for (int q = 0; q < k; ++q) r += lam[q] > fl ? 1 : 0;
      *rank = r;
    }
  }
  __syncthreads();
  const int j = blockIdx.y;
  const double lj = lam[j];
  const bool keep = lj > floor_rel * fmax(s_max, 0.0);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < l; c += gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (keep) {
      for (int i = 0; i < k; ++i) acc = fma(W[static_cast<long long>(i) * ldw + j], Lt[static_cast<long long>(i) * ldl + c], acc);
    }
    Qst[static_cast<long long>(j) * ldq + c] = acc;
    Wt[static_cast<long long>(j) * ldwt + c] = keep ? acc / lj : 0.0;
  }
}

// ---------------------------------------------------------------- Nystrom scale

// W^T[j][i] = V[i][j] / sqrt(lam_j) for kept j (lam_j > floor_rel * max lam), else 0.
// Also Qs^T[j][i] = V[i][j] sqrt(lam_j) (kept j): the landmark rows of M.
__global__ void k_nys_scale(const double* __restrict__ V, long long ldv, const double* __restrict__ lam,
                            int l, double floor_rel, double* __restrict__ Wt, long long ldw,
                            double* __restrict__ Qst, long long ldq, int* __restrict__ rank) {
  __shared__ double s_max;
  if (threadIdx.x == 0) {
    double mx = -CUDART_INF;
    for (int j = 0; j < l; ++j) mx = fmax(mx, lam[j]);
    s_max = mx;
    if (blockIdx.x == 0 && blockIdx.y == 0 && rank) {
      const double fl = floor_rel * fmax(mx, 0.0);
      int r = 0;
      for (int j = 0; j < l; ++j) r += lam[j] > fl ? 1 : 0;
      *rank = r;
    }
  }
  __syncthreads();
  const int j = blockIdx.y;
  const double lj = lam[j];
  const bool keep = lj > floor_rel * fmax(s_max, 0.0);
  const double inv = keep ? 1.0 / sqrt(lj) : 0.0;
  const double sq = keep ? sqrt(lj) : 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < l; i += gridDim.x * blockDim.x) {
    const double v = V[static_cast<long long>(i) * ldv + j];
    Wt[static_cast<long long>(j) * ldw + i] = v * inv;
    Qst[static_cast<long long>(j) * ldq + i] = v * sq;
  }
}

// Mt[:, landmarks[i]] = Qst[:, i]  (U~[I] = Q: the landmark rows of M exactly)
__global__ void k_nys_scatter(const double* __restrict__ Qst, long long ldq, int l,
                              const long long* __restrict__ idx, double* __restrict__ Mt,
                              long long ldm) {
  const int j = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < l; i += gridDim.x * blockDim.x)
    Mt[static_cast<long long>(j) * ldm + idx[i]] = Qst[static_cast<long long>(j) * ldq + i];
}

// ---------------------------------------------------------------- device-resident CG

// state block (doubles): see dngd_b200.h dngd_cg_* for the layout
enum {
  CG_RHO = 0, CG_PAP, CG_RR, CG_RZ, CG_ALPHA, CG_BEST, CG_TOLB, CG_FLOOR, CG_BNORM,
  CG_ITER, CG_DONE, CG_WARN, CG_MAXIT, CG_NSTATE
};

// after b.b is in st[CG_RR]: b_norm, the stop threshold, the breakdown floor;
// b_norm == 0 stops at once (the reference returns -g / lam, which is what the
// finish step computes from y = 0)
__global__ void k_cg_init(double* st, double tol, int max_iters) {
  const double bn = sqrt(st[CG_RR]);
  st[CG_BNORM] = bn;
  st[CG_TOLB] = tol * bn;
  st[CG_FLOOR] = 1e-300 * fmax(1.0, bn * bn);
  st[CG_BEST] = bn;
  st[CG_ITER] = 0.0;
  st[CG_DONE] = bn == 0.0 ? 1.0 : 0.0;
  st[CG_WARN] = 0.0;
  st[CG_MAXIT] = static_cast<double>(max_iters);
  st[CG_RHO] = st[CG_RZ];  // rho = r.z (computed before this kernel)
}

// p.Ap in st[CG_PAP]: breakdown test and alpha; then y += alpha p, r -= alpha Ap
__global__ void k_cg_update_yr(double* __restrict__ st, long long m, double* __restrict__ y,
                               double* __restrict__ r, const double* __restrict__ p,
                               const double* __restrict__ Ap) {
  __shared__ double s_alpha;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    int skip = st[CG_DONE] != 0.0;
    double alpha = 0.0;
    if (!skip) {
      const double pap = st[CG_PAP];
      if (fabs(pap) <= st[CG_FLOOR]) {
        skip = 1;
      } else {
        alpha = st[CG_RHO] / pap;
      }
    }
    s_alpha = alpha;
    s_skip = skip;
  }
  __syncthreads();
  if (s_skip) return;
  const double a = s_alpha;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    y[i] = fma(a, p[i], y[i]);
    r[i] = fma(-a, Ap[i], r[i]);
  }
}

// one thread: the iteration counter, the curvature breakdown (iterations -= 1)
__global__ void k_cg_after_pap(double* st) {
  if (st[CG_DONE] != 0.0) return;
  st[CG_ITER] += 1.0;
  if (fabs(st[CG_PAP]) <= st[CG_FLOOR]) {
    st[CG_WARN] = 1.0;  // cg_breakdown: search direction has near-zero curvature
    st[CG_ITER] -= 1.0;
    st[CG_DONE] = 1.0;
  }
}

// |r| in st[CG_RR] (= r.r): best iterate and the stop test
__global__ void k_cg_after_r(double* __restrict__ st, long long m, const double* __restrict__ y,
                             double* __restrict__ ybest, int* __restrict__ flag) {
  __shared__ int s_copy;
  if (threadIdx.x == 0) {
    int copy = 0;
    if (st[CG_DONE] == 0.0) {
      const double rn = sqrt(st[CG_RR]);
      if (rn < st[CG_BEST]) copy = 1;
    }
    s_copy = copy;
  }
  __syncthreads();
  if (s_copy) {
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
      ybest[i] = y[i];
  }
  // the scalar bookkeeping by the last CTA to finish (so every copy saw the old state)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(reinterpret_cast<unsigned*>(flag), 1u) + 1u;
    if (done == gridDim.x) {
      *reinterpret_cast<volatile unsigned*>(flag) = 0u;
      if (st[CG_DONE] == 0.0) {
        const double rn = sqrt(st[CG_RR]);
        if (rn < st[CG_BEST]) st[CG_BEST] = rn;
        if (rn <= st[CG_TOLB]) st[CG_DONE] = 1.0;
      }
    }
  }
}

// r.z in st[CG_RZ]: the collapse test on the OLD rho, then p = z + (rho_new / rho) p,
// the iteration cap; sets the loop condition (1 = run another iteration)
__global__ void k_cg_update_p(double* __restrict__ st, long long m, double* __restrict__ p,
                              const double* __restrict__ z, int* __restrict__ flag,
                              unsigned long long cond) {
  __shared__ double s_beta;
  __shared__ int s_skip;
  if (threadIdx.x == 0) {
    int skip = st[CG_DONE] != 0.0;
    double beta = 0.0;
    if (!skip) {
      if (fabs(st[CG_RHO]) <= st[CG_FLOOR]) {
        skip = 1;
      } else {
        beta = st[CG_RZ] / st[CG_RHO];
      }
    }
    s_beta = beta;
    s_skip = skip;
  }
  __syncthreads();
  if (!s_skip) {
    const double b = s_beta;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
      p[i] = fma(b, p[i], z[i]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(reinterpret_cast<unsigned*>(flag), 1u) + 1u;
    if (done == gridDim.x) {
      *reinterpret_cast<volatile unsigned*>(flag) = 0u;
      if (st[CG_DONE] == 0.0) {
        if (fabs(st[CG_RHO]) <= st[CG_FLOOR]) {
          st[CG_WARN] = 2.0;  // cg_breakdown: preconditioned residual collapsed
          st[CG_DONE] = 1.0;
        } else {
          st[CG_RHO] = st[CG_RZ];
          if (st[CG_ITER] >= st[CG_MAXIT]) st[CG_DONE] = 1.0;
        }
      }
      if (cond != 0ull) {
        cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(cond),
                                st[CG_DONE] == 0.0 ? 1u : 0u);
      }
    }
  }
}

// warning -> y = best iterate; then y += r_add (the +r of -(J^T (y + r))/lam)
__global__ void k_cg_finish(const double* __restrict__ st, long long m, double* __restrict__ y,
                            const double* __restrict__ ybest, const double* __restrict__ radd) {
  const bool best = st[CG_WARN] != 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double v = best ? ybest[i] : y[i];
    if (radd) v += radd[i];
    y[i] = v;
  }
}

// z = c (v - u) (the preconditioner's v / lam - M (...) / lam)
__global__ void k_axmy(long long m, double c, const double* __restrict__ v,
                       const double* __restrict__ u, double* __restrict__ z) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) z[i] = c * (v[i] - u[i]);
}

}  // namespace dngd

using namespace dngd;

static unsigned vec_blocks(dngd_ctx* ctx, long long m) {
  return static_cast<unsigned>(std::min<long long>((m + 255) / 256, 2LL * ctx->num_sms));
}

#ifdef DNGD_JACOBI_TRACE
long long* dngd_jacobi_trace_ptr = nullptr;
#endif

extern "C" int dngd_syev_workspace(dngd_ctx* ctx, int64_t n, size_t* bytes) {
  if (!ctx || !bytes || n < 0) return DNGD_ERR_DIMENSION;
  *bytes = jacobi_bytes(n, 60);
  return DNGD_OK;
}

extern "C" int dngd_syev_jacobi(dngd_ctx* ctx, void* stream, const double* A, int64_t n,
                                int64_t lda, double* w, double* V, int64_t ldv, int* sweeps,
                                void* work, size_t work_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 0 || lda < n || ldv < n) return set_error(ctx, DNGD_ERR_DIMENSION, "syev: bad sizes");
  if (n == 0) return DNGD_OK;
  const int max_sweeps = 60;
  if (work_bytes < jacobi_bytes(n, max_sweeps)) return set_error(ctx, DNGD_ERR_DIMENSION, "syev: workspace too small");
  if (n > 8192) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "syev: order above 8192");
  const JacShape sh = jac_shape(n);
  char* b = static_cast<char*>(work);
  const size_t mat = static_cast<size_t>(sh.N) * sh.ld * 8;
  JacobiArgs J;
  J.Yt = reinterpret_cast<double*>(b);
  J.Vt = reinterpret_cast<double*>(b + mat);
  J.rotated = reinterpret_cast<unsigned*>(b + 2 * mat + 256);
  J.fro2 = reinterpret_cast<const double*>(b + 2 * mat);
  J.N = sh.N;
  J.n = static_cast<int>(n);
  J.bs = sh.bs;
  J.nblk = sh.nblk;
  J.ld = sh.ld;
  J.max_sweeps = max_sweeps;
  J.eps = 2.220446049250313e-16;
  J.sweeps_out = sweeps;
  J.trace = nullptr;
#ifdef DNGD_JACOBI_TRACE
  static long long* tr = nullptr;
  if (!tr) cudaMalloc(&tr, 256 * 8);
  cudaMemsetAsync(tr, 0, 256 * 8, s);
  J.trace = tr;
  dngd_jacobi_trace_ptr = tr;
#endif
  const long long tot = std::max<long long>(static_cast<long long>(sh.N) * sh.N, max_sweeps);
  k_jacobi_init<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(A, lda, static_cast<int>(n), sh.N,
                                                                       sh.ld, J.Yt, J.Vt, J.rotated,
                                                                       max_sweeps);
  k_fro2<<<1, 1024, 0, s>>>(A, lda, static_cast<int>(n), reinterpret_cast<double*>(b + 2 * mat));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(ctx, e, "syev init");
  auto kern = sh.N <= 32 * 16 ? k_jacobi<16> : k_jacobi<0>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sh.smem));
  if (e != cudaSuccess) return cuda_status(ctx, e, "syev smem attribute");
  const unsigned grid = static_cast<unsigned>(std::min(sh.nblk / 2, ctx->num_sms));
  if (grid < static_cast<unsigned>(sh.nblk / 2)) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "syev: too many blocks");
  void* args[] = {&J};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(kJT), args,
                                  sh.smem, s);
  if (e != cudaSuccess) return cuda_status(ctx, e, "syev cooperative launch");
  k_jacobi_out<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(J.Yt, J.Vt, sh.ld, static_cast<int>(n), w,
                                                                 V, ldv);
  return cuda_status(ctx, cudaGetLastError(), "syev");
}

extern "C" int dngd_pivoted_cholesky(dngd_ctx* ctx, void* stream, const double* K, int64_t l,
                                     int64_t ldk, double tol, int kmax, double* Lt, int64_t ldl,
                                     void* work, size_t work_bytes, int* k_out) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (l <= 0 || kmax <= 0) return DNGD_OK;
  if (work_bytes < static_cast<size_t>(l) * 12 + 64) return set_error(ctx, DNGD_ERR_DIMENSION, "pivoted_cholesky: workspace too small");
  double* d = static_cast<double*>(work);
  int* used = reinterpret_cast<int*>(d + l);
  k_pivchol<<<1, kPC, 0, s>>>(K, ldk, static_cast<int>(l), tol, kmax, Lt, ldl, d, used, k_out);
  return cuda_status(ctx, cudaGetLastError(), "pivoted_cholesky");
}

extern "C" int dngd_nystrom_from_chol(dngd_ctx* ctx, void* stream, const double* W, int64_t ldw,
                                      const double* lam, int k, const double* Lt, int64_t ldl,
                                      int l, double floor_rel, double* Wt, int64_t ldwt,
                                      double* Qst, int64_t ldq, int* rank) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (k <= 0) return DNGD_OK;
  dim3 g(static_cast<unsigned>((l + 255) / 256), static_cast<unsigned>(k));
  k_nys_from_chol<<<g, 256, 0, s>>>(W, ldw, lam, k, Lt, ldl, l, floor_rel, Wt, ldwt, Qst, ldq, rank);
  return cuda_status(ctx, cudaGetLastError(), "nystrom_from_chol");
}

extern "C" int dngd_nystrom_scale(dngd_ctx* ctx, void* stream, const double* V, int64_t ldv,
                                  const double* lam, int l, double floor_rel, double* Wt,
                                  int64_t ldw, double* Qst, int64_t ldq, int* rank) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (l <= 0) return DNGD_OK;
  dim3 g(static_cast<unsigned>((l + 255) / 256), static_cast<unsigned>(l));
  k_nys_scale<<<g, 256, 0, s>>>(V, ldv, lam, l, floor_rel, Wt, ldw, Qst, ldq, rank);
  return cuda_status(ctx, cudaGetLastError(), "nystrom_scale");
}

extern "C" int dngd_nystrom_scatter(dngd_ctx* ctx, void* stream, const double* Qst, int64_t ldq,
                                    int rows, int l, const int64_t* landmarks_dev, double* Mt,
                                    int64_t ldm) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (l <= 0 || rows <= 0) return DNGD_OK;
  dim3 g(static_cast<unsigned>((l + 255) / 256), static_cast<unsigned>(rows));
  k_nys_scatter<<<g, 256, 0, s>>>(Qst, ldq, l, reinterpret_cast<const long long*>(landmarks_dev), Mt, ldm);
  return cuda_status(ctx, cudaGetLastError(), "nystrom_scatter");
}

extern "C" int dngd_cg_init(dngd_ctx* ctx, void* stream, double* state, double tol, int max_iters) {
  k_cg_init<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(state, tol, max_iters);
  return cuda_status(ctx, cudaGetLastError(), "cg_init");
}

extern "C" int dngd_cg_after_pap(dngd_ctx* ctx, void* stream, double* state, int64_t m, double* y,
                                 double* r, const double* p, const double* Ap) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_cg_after_pap<<<1, 1, 0, s>>>(state);
  // (k_cg_update_yr re-reads DONE: a breakdown set above skips the update)
  k_cg_update_yr<<<vec_blocks(ctx, m), 256, 0, s>>>(state, m, y, r, p, Ap);
  return cuda_status(ctx, cudaGetLastError(), "cg_after_pap");
}

extern "C" int dngd_cg_after_r(dngd_ctx* ctx, void* stream, double* state, int64_t m,
                               const double* y, double* ybest, int* flag) {
  k_cg_after_r<<<vec_blocks(ctx, m), 256, 0, static_cast<cudaStream_t>(stream)>>>(state, m, y, ybest,
                                                                                 flag);
  return cuda_status(ctx, cudaGetLastError(), "cg_after_r");
}

extern "C" int dngd_cg_update_p(dngd_ctx* ctx, void* stream, double* state, int64_t m, double* p,
                                const double* z, int* flag, uint64_t cond) {
  k_cg_update_p<<<vec_blocks(ctx, m), 256, 0, static_cast<cudaStream_t>(stream)>>>(state, m, p, z,
                                                                                  flag, cond);
  return cuda_status(ctx, cudaGetLastError(), "cg_update_p");
}

extern "C" int dngd_cg_finish(dngd_ctx* ctx, void* stream, const double* state, int64_t m,
                              double* y, const double* ybest, const double* radd) {
  k_cg_finish<<<vec_blocks(ctx, m), 256, 0, static_cast<cudaStream_t>(stream)>>>(state, m, y, ybest,
                                                                                radd);
  return cuda_status(ctx, cudaGetLastError(), "cg_finish");
}

extern "C" int dngd_axmy(dngd_ctx* ctx, void* stream, int64_t m, double c, const double* v,
                         const double* u, double* z) {
  k_axmy<<<static_cast<unsigned>((m + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(m, c, v, u,
                                                                                              z);
  return cuda_status(ctx, cudaGetLastError(), "axmy");
}

// ---------------------------------------------------------------- graph with a WHILE node

struct dngd_loop_graph {
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
};

extern "C" int dngd_loop_graph_create(dngd_ctx* ctx, void** out, uint64_t* handle) {
  auto* L = new dngd_loop_graph();
  cudaError_t e = cudaGraphCreate(&L->graph, 0);
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 1, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = L->handle;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, L->graph, nullptr, 0, &np);
    if (e == cudaSuccess) L->body = np.conditional.phGraph_out[0];
  }
  if (e != cudaSuccess) {
    if (L->graph) cudaGraphDestroy(L->graph);
    delete L;
    return cuda_status(ctx, e, "loop graph create");
  }
  *out = L;
  *handle = static_cast<uint64_t>(L->handle);
  return DNGD_OK;
}

// capture the loop body: the caller's launches on `stream` between begin and end
extern "C" int dngd_loop_graph_begin(dngd_ctx* ctx, void* lg, void* stream) {
  auto* L = static_cast<dngd_loop_graph*>(lg);
  cudaError_t e = cudaStreamBeginCaptureToGraph(static_cast<cudaStream_t>(stream), L->body, nullptr,
                                                nullptr, 0, cudaStreamCaptureModeThreadLocal);
  return cuda_status(ctx, e, "loop graph begin capture");
}

extern "C" int dngd_loop_graph_end(dngd_ctx* ctx, void* lg, void* stream) {
  auto* L = static_cast<dngd_loop_graph*>(lg);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g);
  if (e == cudaSuccess) e = cudaGraphInstantiate(&L->exec, L->graph, 0);
  return cuda_status(ctx, e, "loop graph end capture / instantiate");
}

extern "C" int dngd_loop_graph_launch(dngd_ctx* ctx, void* lg, void* stream) {
  auto* L = static_cast<dngd_loop_graph*>(lg);
  return cuda_status(ctx, cudaGraphLaunch(L->exec, static_cast<cudaStream_t>(stream)), "loop graph launch");
}

extern "C" int dngd_loop_graph_destroy(dngd_ctx* ctx, void* lg) {
  (void)ctx;
  auto* L = static_cast<dngd_loop_graph*>(lg);
  if (!L) return DNGD_OK;
  if (L->exec) cudaGraphExecDestroy(L->exec);
  if (L->graph) cudaGraphDestroy(L->graph);
  delete L;
  return DNGD_OK;
}
