// PINN residual map on device: forward-Laplacian MLP pass, per-point adjoints,
// Jacobian row writes, second directional derivative f_vv and batched
// line-search losses.
//
// Reference semantics (per collocation class, residuals.py:444-454):
//   r_i = w * (cu*u + sum_g cg[g] d_{dim g} u + cl * sum_{j in lap} d_jj u - f_i)
// where u is the tanh MLP of model.py:88-97.  The reference evaluates each
// d_jj u with its own Jet2 pass (model.py:251-256, jets.py:285-294); here one
// pass propagates "channels" per point: value, one first-derivative channel
// per needed input dimension, and one Laplacian channel
//     t = tanh z,  s = 1 - t^2,  d_j t = s d_j z,  Lap t = s Lap z - 2 t s sum_j (d_j z)^2.
// Channel rows of one point are contiguous, so every hidden-to-hidden layer is
// ONE FP64 tensor-core GEMM over all (point, channel) rows (gemm.cu) followed by
// an elementwise channel kernel.  The per-point adjoint of the channel map
// gives, for every layer, J[i, W_k|b_k] = sum_c Hext_k[i,c] (x) Zbar_k[i,c]:
// a rank-nch outer product written straight to HBM (the tape's per-sample
// einsum, tape.py:408-409).
//
// Row layout of the activation buffers: act0(class) + i * nch(class) + c.

#include <algorithm>
#include <cmath>
#include <vector>

#include <math_constants.h>

#include "common.cuh"
#include "internal.h"
#include "oz_common.cuh"
#include "tc05.cuh"

namespace dngd {

constexpr int MAXG = DNGD_MAX_GRAD;
constexpr int MAXC = DNGD_MAX_CLASSES;

struct ClassDev {
  long long row0, count, act0;
  int nch, ngrad, nlap;
  int grad_dims[MAXG];
  int lap_ch[MAXG];  // channel index (1-based grad channel) summed into the Laplacian
  double cg[MAXG];
  double cu, cl, weight;
  double c3;           // coefficient of u^3 (Allen-Cahn reaction; 0 = linear operator)
  const double* pts;
  const double* f;
  const double* inp;   // embedded input channels (N x nch x din) or nullptr = identity
  const int* pgi;      // per-point derivative dims (N x ngrad, STDE subsets) or nullptr
  const double* pco;   // per-point channel coefficients (N x nch) or nullptr
};

struct Classes {
  int n, din;
  long long m, R;
  ClassDev c[MAXC];
  double* u0;  // per-point network value (written by k_head; cubic-term adjoint seeds)
};

DNGD_DEV int find_class(const Classes& T, long long p) {
  int c = 0;
#pragma unroll
  for (int k = 0; k < MAXC - 1; ++k)
    if (k + 1 < T.n && p >= T.c[k + 1].row0) c = k + 1;
  return c;
}

DNGD_DEV double coef(const ClassDev& C, int ch) {
  if (ch == 0) return C.cu;
  if (ch <= C.ngrad) return C.cg[ch - 1];
  return C.cl;
}

// coefficient of channel ch at local point i (per-point coefficients when given)
DNGD_DEV double coefp(const ClassDev& C, int ch, long long i) {
  return C.pco ? C.pco[i * C.nch + ch] : coef(C, ch);
}

// input dimension of grad channel g (0-based) at local point i
DNGD_DEV int gdim(const ClassDev& C, int g, long long i) {
  return C.pgi ? C.pgi[i * C.ngrad + g] : C.grad_dims[g];
}

// adjoint seed of output channel ch at point p: d r_p / d u_ch (the value channel
// picks up 3 c3 u^2 from the cubic term)
DNGD_DEV double seedc(const Classes& T, const ClassDev& C, int ch, long long p) {
  double cf = coefp(C, ch, p - C.row0);
  if (ch == 0 && C.c3 != 0.0) {
    const double u = T.u0[p];
    cf = fma(3.0 * C.c3 * u, u, cf);
  }
  return C.weight * cf;
}

static inline long long ldw(long long w) { return (w + 3) / 4 * 4; }

// ------------------------------------------------------------------ forward

// input layer (K = din is tiny): z = x W0 + b0, d_j z = W0[j,:], Lap z = 0; then tanh channels.
// grid.y = candidate (theta stride th_s, activation stride act_s).
// Zx (optional, large din): precomputed x W0 rows (ld ldx); with Dx the candidate's
// value is Zx + eta_c Dx (x (W0 + eta V0) by linearity) -- see input_gemm.
__global__ void k_input_fwd(Classes T, const double* __restrict__ theta, long long th_s, int w1,
                            long long ld, double* __restrict__ Z, double* __restrict__ H,
                            long long act_s, const double* __restrict__ Zx,
                            const double* __restrict__ Dx, const double* __restrict__ etas,
                            long long ldx, const double* __restrict__ W0b,
                            const double* __restrict__ V0b) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.m * w1) return;
  const long long p = idx / w1;
  const int q = static_cast<int>(idx - p * w1);
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const double* th = theta + blockIdx.y * th_s;
  const double* W0 = th;
  const double* b0 = th + static_cast<long long>(T.din) * w1;
  const long long base = (C.act0 + i * C.nch) * ld + q + blockIdx.y * act_s;
  if (C.inp) {
    // embedded inputs: every channel is inputs_ch . W0 (value channel + b0)
    const double* xr = C.inp + i * C.nch * T.din;
    auto zch = [&](int ch) {
      double z = ch == 0 ? b0[q] : 0.0;
      for (int j = 0; j < T.din; ++j) z = fma(xr[ch * T.din + j], W0[j * w1 + q], z);
      return z;
    };
    const double z = zch(0);
    const double t = tanh(z), s = 1.0 - t * t;
    if (Z) Z[base] = z;
    H[base] = t;
    for (int g = 0; g < C.ngrad; ++g) {
      const double dz = zch(1 + g);
      if (Z) Z[base + (1 + g) * ld] = dz;
      H[base + (1 + g) * ld] = s * dz;
    }
    if (C.nlap) {
      double G = 0.0;
      for (int l = 0; l < C.nlap; ++l) {
        const double dz = zch(C.lap_ch[l]);
        G = fma(dz, dz, G);
      }
      const double zl = zch(C.nch - 1);
      if (Z) Z[base + (C.nch - 1) * ld] = zl;
      H[base + (C.nch - 1) * ld] = s * zl - 2.0 * t * s * G;
    }
    return;
  }
  double z;
  if (Zx) {
    z = Zx[p * ldx + q];
    if (Dx) z = fma(etas[blockIdx.y], Dx[p * ldx + q], z);
    z += b0[q];
  } else {
    const double* x = C.pts + i * T.din;
    z = b0[q];
    for (int j = 0; j < T.din; ++j) z = fma(x[j], W0[j * w1 + q], z);
  }
  const double t = tanh(z), s = 1.0 - t * t;
  if (Z) Z[base] = z;
  H[base] = t;
  // with Dx the candidates' W0 rows were not materialised: W0 + eta V0 on the fly
  // (the same fma as k_candidates)
  auto w0 = [&](int d) {
    const long long e = static_cast<long long>(d) * w1 + q;
    return Dx ? fma(etas[blockIdx.y], V0b[e], W0b[e]) : W0[e];
  };
  double G = 0.0;
  for (int g = 0; g < C.ngrad; ++g) {
    const double dz = w0(gdim(C, g, i));
    if (Z) Z[base + (1 + g) * ld] = dz;
    H[base + (1 + g) * ld] = s * dz;
  }
  if (C.nlap) {
    for (int l = 0; l < C.nlap; ++l) {
      const double dz = w0(gdim(C, C.lap_ch[l] - 1, i));
      G = fma(dz, dz, G);
    }
    if (Z) Z[base + (C.nch - 1) * ld] = 0.0;
    H[base + (C.nch - 1) * ld] = -2.0 * t * s * G;
  }
}

// hidden layer: Z already holds H_k W_k (GEMM); add bias to the value channel
// (written back so the adjoint sees the pre-activation) and apply tanh channels.
__global__ void k_tanh_fwd(Classes T, double* __restrict__ Z, double* __restrict__ H, int w,
                           long long ld, const double* __restrict__ bias, long long bias_s,
                           long long act_s) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.m * w) return;
  const long long p = idx / w;
  const int q = static_cast<int>(idx - p * w);
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long base = (C.act0 + i * C.nch) * ld + q + blockIdx.y * act_s;
  const double z = Z[base] + bias[q + blockIdx.y * bias_s];
  Z[base] = z;
  const double t = tanh(z), s = 1.0 - t * t;
  H[base] = t;
  for (int g = 0; g < C.ngrad; ++g) H[base + (1 + g) * ld] = s * Z[base + (1 + g) * ld];
  if (C.nlap) {
    double G = 0.0;
    for (int l = 0; l < C.nlap; ++l) {
      const double dz = Z[base + C.lap_ch[l] * ld];
      G = fma(dz, dz, G);
    }
    H[base + (C.nch - 1) * ld] = s * Z[base + (C.nch - 1) * ld] - 2.0 * t * s * G;
  }
}

// Channel map of one layer fused with the Ozaki slicing of its output (line-search
// forward): the rows never reach HBM in FP64, only the next GEMM's digit planes
// (rows cand R + act row) and row scales.  MODE 0: hidden layer, Z + bias -> tanh
// channels (k_tanh_fwd's map); MODE 1: input layer from the points and W0 (plain
// inputs; k_input_fwd's map).  Same operation order as those kernels, and the
// scale rule and digits of k_oz_slice, so the planes equal slicing their output.
// One warp per (point, candidate): lane l owns neurons 4 (l + 32 k) .. + 3 of every
// channel row; pass 1 computes the channel values and the per-row max |v| (warp
// shuffles only, no block barrier), pass 2 recomputes them (operands from L1/L2)
// and writes the digits -- a short dependent chain per warp and many warps per SM
// (the CTA-per-point version was latency-bound at ~1 TB/s).
constexpr int kTsMaxCh = 8;
constexpr int kCsWarps = 8;  // points per 256-thread CTA

// per-class constants of the channel map held in registers (the kernels index the
// Classes parameter block by a run-time class, which would otherwise be re-read
// from a local-memory copy inside the neuron loop)
template <int NCH>
struct ChanRegs {
  int ngrad;
  unsigned lapmask;  // bit ch: channel ch is summed into the Laplacian (C.lap_ch)
  int gd[NCH > 1 ? NCH - 1 : 1];  // derivative dims (class-wide; pgi overrides per point)
};

// channel values of neuron q of one (point, candidate) (0 past w); the Laplacian's
// sum runs over the channels in ascending order -- k_tanh_fwd / k_input_fwd's
// order when C.lap_ch is ascending, which the launcher requires
// TC: 1 = store tanh into the warp's shared cache tc (when given), 2 = read it back
// instead of evaluating tanh again (k_chan_slice's second pass; same value, same lane)
template <int NCH, int MODE, int TC = 0>
DNGD_DEV void chan_val1(const Classes& T, const ChanRegs<NCH>& cr, const int* pgi, const double* z0,
                        long long ld, const double* bs, const double* W0, const double* b0,
                        const double* x, int w, int q, double (&v)[NCH], double* tc = nullptr) {
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) v[ch] = 0.0;
  if (q >= w) return;
  if constexpr (MODE == 0) {
    double zz[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) zz[ch] = z0[ch * ld + q];
    double t;
    if (TC == 2 && tc) {
      t = tc[q];
    } else {
      t = tanh(zz[0] + bs[q]);
      if (TC == 1 && tc) tc[q] = t;
    }
    const double sd = 1.0 - t * t;
    v[0] = t;
#pragma unroll
    for (int gi = 0; gi < NCH - 1; ++gi)
      if (gi < cr.ngrad) v[1 + gi] = sd * zz[1 + gi];
    if (NCH > 1 && cr.lapmask) {
      double G = 0.0;
#pragma unroll
      for (int ch = 1; ch < NCH; ++ch)
        if ((cr.lapmask >> ch) & 1u) G = fma(zz[ch], zz[ch], G);
      v[NCH - 1] = sd * zz[NCH - 1] - 2.0 * t * sd * G;
    }
  } else {
    double t;
    if (TC == 2 && tc) {
      t = tc[q];
    } else {
      double z = b0[q];
      for (int d = 0; d < T.din; ++d) z = fma(x[d], W0[d * w + q], z);
      t = tanh(z);
      if (TC == 1 && tc) tc[q] = t;
    }
    const double sd = 1.0 - t * t;
    v[0] = t;
    double G = 0.0;
#pragma unroll
    for (int gi = 0; gi < NCH - 1; ++gi) {
      if (gi < cr.ngrad) {
        const double dz = W0[cr.gd[gi] + q];  // gd: first-layer row offsets (k_chan_slice)
        v[1 + gi] = sd * dz;
        if ((cr.lapmask >> (1 + gi)) & 1u) G = fma(dz, dz, G);
      }
    }
    if (NCH > 1 && cr.lapmask) v[NCH - 1] = -2.0 * t * sd * G;
  }
}

template <int S, int NCH, int MODE>
__global__ void __launch_bounds__(32 * kCsWarps, MODE == 1 ? 3 : 0) k_chan_slice(
    Classes T, int cls, const double* __restrict__ Z, int w, long long ld,
    const double* __restrict__ par, long long par_s, long long act_s, long long R, long long kpad,
    int8_t* __restrict__ Q, double* __restrict__ scale, int cache) {
  extern __shared__ double cs_tanh[];  // cache: kCsWarps x w tanh values (pass 1 -> pass 2)
  const ClassDev& C = T.c[cls];
  const long long i = static_cast<long long>(blockIdx.x) * kCsWarps + (threadIdx.x >> 5);
  if (i >= C.count) return;
  const int lane = threadIdx.x & 31;
  double* tc = cache ? cs_tanh + static_cast<size_t>(threadIdx.x >> 5) * w : nullptr;
  const int cand = blockIdx.y;
  // MODE 0: par = bias of every candidate; MODE 1: par = the candidates' thetas
  const double* z0 = MODE == 0 ? Z + cand * act_s + (C.act0 + i * NCH) * ld : nullptr;
  const double* bs = par + cand * par_s;
  const double* W0 = par + cand * par_s;
  const double* b0 = W0 + static_cast<long long>(T.din) * w;
  const double* x = MODE == 1 ? C.pts + i * T.din : nullptr;
  const long long row0 = cand * R + C.act0 + i * NCH;
  ChanRegs<NCH> cr;
  cr.ngrad = C.ngrad;
  cr.lapmask = 0;
  for (int l = 0; l < C.nlap; ++l) cr.lapmask |= 1u << C.lap_ch[l];
#pragma unroll
  // input-layer mode: gd = offset of the derivative dim's row of W0 (class-wide dims,
  // or this point's own: pgi), resolved once per warp instead of per neuron
  const int* pgi = C.pgi ? C.pgi + i * C.ngrad : nullptr;
  for (int g = 0; g < (NCH > 1 ? NCH - 1 : 1); ++g)
    cr.gd[g] = g < C.ngrad ? (MODE == 1 ? (pgi ? pgi[g] : C.grad_dims[g]) * w : C.grad_dims[g]) : 0;
  double mx[NCH];
  int bad[NCH];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    mx[ch] = 0.0;
    bad[ch] = 0;
  }
  // lane owns neurons lane, lane + 32, ...: coalesced operand rows, one digit byte
  // per (slice, row) and neuron -- 32 consecutive bytes per warp store
  for (int q = lane; q < w; q += 32) {
    double v[NCH];
    chan_val1<NCH, MODE, MODE == 1 ? 1 : 0>(T, cr, pgi, z0, ld, bs, W0, b0, x, w, q, v, tc);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      bad[ch] |= !isfinite(v[ch]);
      mx[ch] = fmax(mx[ch], fabs(v[ch]));
    }
  }
  double sinv[NCH];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx[ch] = fmax(mx[ch], __shfl_xor_sync(0xffffffffu, mx[ch], o));
      bad[ch] |= __shfl_xor_sync(0xffffffffu, bad[ch], o);
    }
    const int e = bad[ch] ? 0 : oz_row_exponent(mx[ch]);
    if (lane == ch) scale[row0 + ch] = bad[ch] ? CUDART_NAN : ldexp(1.0, e);
    sinv[ch] = ldexp(1.0, OZ_BITS * S - e);
  }
  const size_t plane = static_cast<size_t>(gridDim.y) * R * kpad;
  __syncwarp();
  // store addresses by pointer increments (row pitch kpad, plane pitch `plane`): the
  // 64-bit multiplies per (channel, digit) were a third of the loop's instructions
  int8_t* prow = Q + row0 * kpad + lane;
  for (int q = lane; q < kpad; q += 32, prow += 32) {
    double v[NCH];
    chan_val1<NCH, MODE, MODE == 1 ? 2 : 0>(T, cr, pgi, z0, ld, bs, W0, b0, x, w, q, v, tc);
    int8_t* pch = prow;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch, pch += kpad) {
      // oz_digits4's digits: byte S-1-t of (X + offset) ^ offset is digit t
      const long long y = oz_digit_bytes<S>(v[ch], sinv[ch], bad[ch] != 0);
      const uint32_t ylo = static_cast<uint32_t>(y);
      const uint32_t yhi = static_cast<uint32_t>(static_cast<unsigned long long>(y) >> 32);
      int8_t* dst = pch;
#pragma unroll
      for (int t = 0; t < S; ++t, dst += plane) {
        const int byte = S - 1 - t;
        *dst = static_cast<int8_t>((byte < 4 ? ylo : yhi) >> (8 * (byte & 3)));
      }
    }
  }
}

// Last hidden layer of the line-search forward fused with the output layer:
// k_tanh_fwd's channel map of one (point, candidate) straight into k_head's
// channel dot products and residual (same per-lane order over neurons, same warp
// tree, same residual arithmetic), so H_{L-1} never reaches HBM.  One warp per
// point of class cls, grid.y = candidates.
template <int NCH>
__global__ void __launch_bounds__(256) k_tanh_head(Classes T, int cls, const double* __restrict__ Z,
                                                   int w, long long ld,
                                                   const double* __restrict__ thetas,
                                                   long long th_s, long long bias_off,
                                                   long long wl_off, long long act_s,
                                                   double* __restrict__ r, long long r_s) {
  const ClassDev& C = T.c[cls];
  const long long i = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (i >= C.count) return;
  const int lane = threadIdx.x & 31;
  const int cand = blockIdx.y;
  const double* th = thetas + cand * th_s;
  const double* bs = th + bias_off;
  const double* WL = th + wl_off;
  const double* z0 = Z + cand * act_s + (C.act0 + i * NCH) * ld;
  ChanRegs<NCH> cr;
  cr.ngrad = C.ngrad;
  cr.lapmask = 0;
  for (int l = 0; l < C.nlap; ++l) cr.lapmask |= 1u << C.lap_ch[l];
  double u[NCH];
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) u[ch] = 0.0;
  for (int q = lane; q < w; q += 32) {
    double v[NCH];
    chan_val1<NCH, 0>(T, cr, nullptr, z0, ld, bs, nullptr, nullptr, nullptr, w, q, v);
    const double wq = WL[q];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) u[ch] = fma(v[ch], wq, u[ch]);
  }
  double res = 0.0, uv = 0.0;
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    double uc = warp_sum(u[ch]);
    if (ch == 0) {
      uc += WL[w];
      uv = uc;
    }
    res = fma(coefp(C, ch, i), uc, res);
  }
  if (C.c3 != 0.0) res = fma(C.c3 * uv * uv, uv, res);
  const long long p = C.row0 + i;
  if (lane == 0) {
    r[p + cand * r_s] = C.weight * (res - C.f[i]);
    if (T.u0 != nullptr && cand == 0) T.u0[p] = uv;
  }
}

static void launch_tanh_head(cudaStream_t s, const Classes& T, const double* Z, int w, long long ld,
                             const double* thetas, long long th_s, long long bias_off,
                             long long wl_off, long long act_s, int nb, double* r, long long r_s) {
  for (int c = 0; c < T.n; ++c) {
    if (T.c[c].count == 0) continue;
    const dim3 grid(static_cast<unsigned>((T.c[c].count + 7) / 8), nb);
#define DNGD_TH(N)                                                                                \
  case N:                                                                                         \
    k_tanh_head<N><<<grid, 256, 0, s>>>(T, c, Z, w, ld, thetas, th_s, bias_off, wl_off, act_s, r, \
                                         r_s);                                                    \
    break;
    switch (T.c[c].nch) {
      DNGD_TH(1) DNGD_TH(2) DNGD_TH(3) DNGD_TH(4) DNGD_TH(5) DNGD_TH(6) DNGD_TH(7) DNGD_TH(8)
      default: break;
    }
#undef DNGD_TH
  }
}

// k_chan_slice sums the Laplacian's channels in ascending order
static bool lap_ascending(const Classes& T) {
  for (int c = 0; c < T.n; ++c)
    for (int l = 1; l < T.c[c].nlap; ++l)
      if (T.c[c].lap_ch[l] <= T.c[c].lap_ch[l - 1]) return false;
  return true;
}

template <int S, int MODE>
static void launch_chan_slice(cudaStream_t s, const Classes& T, const double* Z, int w, long long ld,
                              const double* par, long long par_s, long long act_s, long long R,
                              long long kpad, int nb, int8_t* Q, double* scale) {
  for (int c = 0; c < T.n; ++c) {
    if (T.c[c].count == 0) continue;
    const dim3 grid(static_cast<unsigned>((T.c[c].count + kCsWarps - 1) / kCsWarps), nb);
    // tanh cache between the two passes while it fits the default 48 KB of shared memory
    const size_t cbytes = static_cast<size_t>(kCsWarps) * w * sizeof(double);
    // (input-layer mode only: the hidden-layer mode is bound by its Z reads and digit
    // writes, and the cache costs it a resident CTA -- measured 0.81 -> 0.94 ms)
    const int cache = (MODE == 1 && cbytes <= 48 * 1024) ? 1 : 0;
#define DNGD_CS(N)                                                                                 \
  case N:                                                                                          \
    k_chan_slice<S, N, MODE><<<grid, 32 * kCsWarps, cache ? cbytes : 0, s>>>(                      \
        T, c, Z, w, ld, par, par_s, act_s, R, kpad, Q, scale, cache);                              \
    break;
    switch (T.c[c].nch) {
      DNGD_CS(1) DNGD_CS(2) DNGD_CS(3) DNGD_CS(4) DNGD_CS(5) DNGD_CS(6) DNGD_CS(7) DNGD_CS(8)
      default: break;
    }
#undef DNGD_CS
  }
}

template <int S>
static void launch_tanh_slice(cudaStream_t s, const Classes& T, const double* Z, int w,
                              long long ld, const double* bias, long long bias_s, long long act_s,
                              long long R, long long kpad, int nb, int8_t* Q, double* scale) {
  launch_chan_slice<S, 0>(s, T, Z, w, ld, bias, bias_s, act_s, R, kpad, nb, Q, scale);
}

template <int S>
static void launch_input_slice(cudaStream_t s, const Classes& T, const double* thetas,
                               long long th_s, int w1, long long R, long long kpad, int nb,
                               int8_t* Q, double* scale) {
  launch_chan_slice<S, 1>(s, T, nullptr, w1, 0, thetas, th_s, 0, R, kpad, nb, Q, scale);
}

// output layer (width 1): one warp per point; channel dot products, residual.
__global__ void k_head(Classes T, const double* __restrict__ H, int w, long long ld,
                       const double* __restrict__ theta, long long th_s, long long wl_off,
                       long long act_s, double* __restrict__ r, long long r_s) {
  const long long p = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= T.m) return;
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const double* th = theta + blockIdx.y * th_s;
  const double* WL = th + wl_off;
  const double bL = WL[w];
  const double* h = H + (C.act0 + i * C.nch) * ld + blockIdx.y * act_s;
  double res = 0.0, u0 = 0.0;
  for (int c = 0; c < C.nch; ++c) {
    double u = 0.0;
    for (int q = lane; q < w; q += 32) u = fma(h[c * ld + q], WL[q], u);
    u = warp_sum(u);
    if (c == 0) {
      u += bL;
      u0 = u;
    }
    res = fma(coefp(C, c, i), u, res);
  }
  if (C.c3 != 0.0) res = fma(C.c3 * u0 * u0, u0, res);
  if (lane == 0) {
    r[p + blockIdx.y * r_s] = C.weight * (res - C.f[i]);
    if (T.u0 != nullptr && blockIdx.y == 0) T.u0[p] = u0;
  }
}

// ------------------------------------------------------------------ adjoint

// Hbar_{L-1}[c][q] = w * coef_c * W_L[q]
__global__ void k_seed_hbar(Classes T, double* __restrict__ Hb, int w, long long ld,
                            const double* __restrict__ WL) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.m * w) return;
  const long long p = idx / w;
  const int q = static_cast<int>(idx - p * w);
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long base = (C.act0 + i * C.nch) * ld + q;
  for (int c = 0; c < C.nch; ++c) Hb[base + c * ld] = seedc(T, C, c, p) * WL[q];
}

// Zbar = adjoint of (z channels -> tanh channels) applied to Hbar.
__global__ void k_tanh_bwd(Classes T, const double* __restrict__ Z, const double* __restrict__ H,
                           const double* __restrict__ Hb, double* __restrict__ Zb, int w,
                           long long ld) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.m * w) return;
  const long long p = idx / w;
  const int q = static_cast<int>(idx - p * w);
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long base = (C.act0 + i * C.nch) * ld + q;
  const double t = H[base], s = 1.0 - t * t;
  const double dsdz = -2.0 * t * s;
  double z0 = s * Hb[base];
  double cross = 0.0;
  for (int g = 0; g < C.ngrad; ++g) {
    const double hb = Hb[base + (1 + g) * ld];
    cross = fma(hb, Z[base + (1 + g) * ld], cross);
    Zb[base + (1 + g) * ld] = s * hb;
  }
  z0 = fma(dsdz, cross, z0);
  if (C.nlap) {
    const long long lb = base + (C.nch - 1) * ld;
    const double Lb = Hb[lb];
    double G = 0.0;
    for (int l = 0; l < C.nlap; ++l) {
      const long long o = base + C.lap_ch[l] * ld;
      const double dz = Z[o];
      G = fma(dz, dz, G);
      Zb[o] = fma(-4.0 * t * s * Lb, dz, Zb[o]);
    }
    Zb[lb] = s * Lb;
    z0 = fma(Lb, dsdz * Z[lb] - 2.0 * G * (s * s - 2.0 * t * t * s), z0);
  }
  Zb[base] = z0;
}

// ------------------------------------------------------------------ J rows

DNGD_DEV double hext(const ClassDev& C, int din, const double* __restrict__ xrow,
                     const double* __restrict__ hrow, long long ld, int win, int c, int p,
                     long long i) {
  if (p == win) return c == 0 ? 1.0 : 0.0;  // bias row
  if (hrow != nullptr) return hrow[c * ld + p];
  // input layer: embedded input channels, or x / e_j / 0 (identity)
  if (C.inp) return xrow[c * din + p];
  if (c == 0) return xrow[p];
  if (c <= C.ngrad) return gdim(C, c - 1, i) == p ? 1.0 : 0.0;
  return 0.0;
}

// Block of layer k in row i: (win+1) x wout row-major at flat column layer_off.
// VEC: wout even, (layer_off - col_begin) even, ldJ even -> double2 streaming stores.
template <bool VEC>
__global__ void __launch_bounds__(256) k_jwrite(Classes T, const double* __restrict__ Hk,
                                                  long long ldh, int win,
                                                  const double* __restrict__ Zb, long long ldz,
                                                  int wout, long long layer_off,
                                                  long long col_begin, long long col_end,
                                                  double* __restrict__ J, long long ldJ) {
  const long long p = blockIdx.y;
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long arow = C.act0 + i * C.nch;
  const double* hrow = Hk ? Hk + arow * ldh : nullptr;
  const double* xrow = C.inp ? C.inp + i * C.nch * T.din : C.pts + i * T.din;
  const double* zrow = Zb ? Zb + arow * ldz : nullptr;
  double* Jrow = J + p * ldJ - col_begin;
  const long long E = static_cast<long long>(win + 1) * wout;
  const int nch = C.nch;
  if (VEC) {
    // 32-bit element index (E = (win+1) wout < 2^31 for every layer this path
    // takes; the wide input layer goes through k_jwrite_in): the 64-bit division
    // per element was most of this kernel's time
    const int E32 = static_cast<int>(E);
    for (int e = (blockIdx.x * 256 + threadIdx.x) * 2; e < E32; e += gridDim.x * 512) {
      const int pp = e / wout;
      const int q = e - pp * wout;
      const long long col = layer_off + e;
      if (col + 1 < col_begin || col >= col_end) continue;
      double a0 = 0.0, a1 = 0.0;
      for (int c = 0; c < nch; ++c) {
        const double h = hext(C, T.din, xrow, hrow, ldh, win, c, pp, i);
        const double2 z = *reinterpret_cast<const double2*>(zrow + c * ldz + q);
        a0 = fma(h, z.x, a0);
        a1 = fma(h, z.y, a1);
      }
      if (col >= col_begin && col + 1 < col_end) {
        __stcs(reinterpret_cast<double2*>(Jrow + col), make_double2(a0, a1));
      } else {
        if (col >= col_begin && col < col_end) Jrow[col] = a0;
        if (col + 1 >= col_begin && col + 1 < col_end) Jrow[col + 1] = a1;
      }
    }
  } else {
    const long long e0 = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
    for (long long e = e0; e < E; e += static_cast<long long>(gridDim.x) * 256) {
      const long long col = layer_off + e;
      if (col < col_begin || col >= col_end) continue;
      const int pp = static_cast<int>(e / wout);
      const int q = static_cast<int>(e - static_cast<long long>(pp) * wout);
      double a = 0.0;
      for (int c = 0; c < nch; ++c) {
        const double h = hext(C, T.din, xrow, hrow, ldh, win, c, pp, i);
        const double z = zrow ? zrow[c * ldz + q] : seedc(T, C, c, p);
        a = fma(h, z, a);
      }
      Jrow[col] = a;
    }
  }
}

// Element loop of k_jwrite_staged (block fully inside the column range).
// NCH = 0: runtime channel count.  NCH > 0 register-blocks RB rows: a thread keeps
// the NCH adjoint pairs of its column pair qp in registers and sweeps RB rows pp
// (each row's NCH activations are warp-wide broadcasts), so the shared-memory
// reads per stored double2 drop from 2 NCH to NCH (1/RB + 1); a warp still writes
// 32 consecutive double2 of one row per store.
template <int NCH>
DNGD_DEV void jw_rows(const double* __restrict__ sh, const double* __restrict__ sz, int W1,
                      int wout, int nch_rt, double2* __restrict__ dst) {
  const int WP = wout >> 1, NP = W1 * WP;
  const double2* sz2 = reinterpret_cast<const double2*>(sz);
  if (NCH > 0 && WP >= 32) {
    constexpr int RB = 4;
    const int nblk = (W1 + RB - 1) / RB;  // row blocks
    for (int f = threadIdx.x; f < nblk * WP; f += 256) {
      const int rb = f / WP, qp = f - rb * WP;
      double2 z[NCH > 0 ? NCH : 1];
#pragma unroll
      for (int c = 0; c < (NCH > 0 ? NCH : 1); ++c) z[c] = sz2[c * WP + qp];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int pp = rb * RB + r;
        if (pp >= W1) break;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int c = 0; c < (NCH > 0 ? NCH : 1); ++c) {
          const double h = sh[c * W1 + pp];
          a0 = fma(h, z[c].x, a0);
          a1 = fma(h, z[c].y, a1);
        }
        __stcs(dst + static_cast<long long>(pp) * WP + qp, make_double2(a0, a1));
      }
    }
    return;
  }
  const int nch = NCH > 0 ? NCH : nch_rt;
  const int dpp = 256 / WP, dq = 256 - dpp * WP;
  int f = threadIdx.x;
  int pp = f / WP, qp = f - pp * WP;
  for (; f < NP; f += 256) {
    double a0 = 0.0, a1 = 0.0;
    for (int c = 0; c < nch; ++c) {
      const double h = sh[c * W1 + pp];
      const double2 z = sz2[c * WP + qp];
      a0 = fma(h, z.x, a0);
      a1 = fma(h, z.y, a1);
    }
    __stcs(dst + f, make_double2(a0, a1));
    pp += dpp;
    qp += dq;
    if (qp >= WP) {
      qp -= WP;
      ++pp;
    }
  }
}

// Hidden-layer block of J for one row, with the row's channel activations
// (nch x (win+1), bias column appended) and adjoints (nch x wout) staged in
// shared memory by coalesced loads first: every global load of the row is in
// flight at once, and the element loop reads only shared memory and streams
// double2 stores.  Same arithmetic (channel order, fma chain) as k_jwrite<true>.
__global__ void __launch_bounds__(256) k_jwrite_staged(Classes T, const double* __restrict__ Hk,
                                                         long long ldh, int win,
                                                         const double* __restrict__ Zb,
                                                         long long ldz, int wout,
                                                         long long layer_off, long long col_begin,
                                                         long long col_end,
                                                         double* __restrict__ J, long long ldJ) {
  extern __shared__ __align__(16) double jw_smem[];
  const long long p = blockIdx.x;
  const ClassDev& C = T.c[find_class(T, p)];
  const long long arow = C.act0 + (p - C.row0) * C.nch;
  const int nch = C.nch, W1 = win + 1;
  double* sh = jw_smem;                              // [nch][win + 1]
  double* sz = jw_smem + ((nch * W1 + 1) & ~1);      // [nch][wout], 16-byte aligned
  for (int idx = threadIdx.x; idx < nch * W1; idx += 256) {
    const int c = idx / W1, pp = idx - c * W1;
    sh[idx] = pp == win ? (c == 0 ? 1.0 : 0.0) : Hk[(arow + c) * ldh + pp];
  }
  for (int idx = threadIdx.x; idx < nch * wout; idx += 256) {
    const int c = idx / wout, q = idx - c * wout;
    sz[idx] = Zb[(arow + c) * ldz + q];
  }
  __syncthreads();
  double* Jrow = J + p * ldJ - col_begin;
  const int E = W1 * wout;
  if (layer_off >= col_begin && layer_off + E <= col_end) {
    // whole block inside the column range: flat double2 index f = pp * (wout/2) + qp,
    // (pp, qp) stepped incrementally (no division in the loop), nch unrolled
    double2* dst = reinterpret_cast<double2*>(Jrow + layer_off);
    switch (nch) {
      case 1: jw_rows<1>(sh, sz, W1, wout, nch, dst); break;
      case 2: jw_rows<2>(sh, sz, W1, wout, nch, dst); break;
      case 3: jw_rows<3>(sh, sz, W1, wout, nch, dst); break;
      case 4: jw_rows<4>(sh, sz, W1, wout, nch, dst); break;
      case 5: jw_rows<5>(sh, sz, W1, wout, nch, dst); break;
      case 6: jw_rows<6>(sh, sz, W1, wout, nch, dst); break;
      case 7: jw_rows<7>(sh, sz, W1, wout, nch, dst); break;
      case 8: jw_rows<8>(sh, sz, W1, wout, nch, dst); break;
      default: jw_rows<0>(sh, sz, W1, wout, nch, dst); break;
    }
    return;
  }
  for (int e = 2 * threadIdx.x; e < E; e += 512) {
    const int pp = e / wout;
    const int q = e - pp * wout;
    const long long col = layer_off + e;
    if (col + 1 < col_begin || col >= col_end) continue;
    double a0 = 0.0, a1 = 0.0;
    for (int c = 0; c < nch; ++c) {
      const double h = sh[c * W1 + pp];
      const double2 z = *reinterpret_cast<const double2*>(sz + c * wout + q);
      a0 = fma(h, z.x, a0);
      a1 = fma(h, z.y, a1);
    }
    if (col >= col_begin && col + 1 < col_end) {
      __stcs(reinterpret_cast<double2*>(Jrow + col), make_double2(a0, a1));
    } else {
      if (col >= col_begin && col < col_end) Jrow[col] = a0;
      if (col + 1 >= col_begin && col + 1 < col_end) Jrow[col + 1] = a1;
    }
  }
}

// Input-layer block of J for identity inputs (hext = x_j, e_{gdim}, 0, bias 1):
// one product per element plus a fix-up on the <= ngrad rows j that are
// derivative dims, found through a sorted list walked alongside the thread's
// (monotone) j.  Same arithmetic as k_jwrite<true> for layer 0; it exists for the
// STDE case (din ~ 1e5, J's input block is ~all of J).
__global__ void __launch_bounds__(256) k_jwrite_in(Classes T, const double* __restrict__ Zb,
                                                     long long ldz, int wout, long long col_begin,
                                                     long long col_end, double* __restrict__ J,
                                                     long long ldJ) {
  __shared__ int sdim[MAXG], sch[MAXG];
  const long long p = blockIdx.y;
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const int din = T.din, ng = C.ngrad;
  if (threadIdx.x == 0) {  // stable insertion sort of (dim, channel) by dim
    for (int g = 0; g < ng; ++g) {
      const int d = gdim(C, g, i);
      int t = g;
      while (t > 0 && sdim[t - 1] > d) {
        sdim[t] = sdim[t - 1];
        sch[t] = sch[t - 1];
        --t;
      }
      sdim[t] = d;
      sch[t] = 1 + g;
    }
  }
  __syncthreads();
  const double* xrow = C.pts + i * din;
  const double* zrow = Zb + (C.act0 + i * C.nch) * ldz;
  double* Jrow = J + p * ldJ - col_begin;
  const int half = wout / 2;
  const long long pairs = (din + 1LL) * half;
  int idx = 0;
  for (long long e2 = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x; e2 < pairs;
       e2 += static_cast<long long>(gridDim.x) * 256) {
    const int j = static_cast<int>(e2 / half);
    const int q = 2 * static_cast<int>(e2 - static_cast<long long>(j) * half);
    const long long col = 2 * e2;
    if (col + 1 < col_begin || col >= col_end) continue;
    const double2 z0 = __ldg(reinterpret_cast<const double2*>(zrow + q));
    double a0, a1;
    if (j == din) {
      a0 = z0.x;
      a1 = z0.y;
    } else {
      const double xj = __ldg(xrow + j);
      a0 = xj * z0.x;
      a1 = xj * z0.y;
      while (idx < ng && sdim[idx] < j) ++idx;
      for (int t = idx; t < ng && sdim[t] == j; ++t) {
        const double2 zg = __ldg(reinterpret_cast<const double2*>(zrow + sch[t] * ldz + q));
        a0 += zg.x;
        a1 += zg.y;
      }
    }
    if (col >= col_begin && col + 1 < col_end) {
      __stcs(reinterpret_cast<double2*>(Jrow + col), make_double2(a0, a1));
    } else {
      if (col >= col_begin && col < col_end) Jrow[col] = a0;
      if (col + 1 >= col_begin && col + 1 < col_end) Jrow[col + 1] = a1;
    }
  }
}

// ------------------------------------------------------------------ wide input layer, J-free
// For identity inputs with din > MAXG (the STDE case) J's input block is
//   J[p,(j,q)] = x_pj a_pq + sum_g [gd_pg = j] b_pgq  (j < din),   J[p,(din,q)] = a_pq,
// a = Zbar_0 value channel, b_g = Zbar_0 grad channels (the Laplacian channel's
// Hext is 0).  Its Gram block and J^T w are formed from X and Zbar_0 directly:
//   K_in[p,p'] = sum_q a_pq a_p'q (x_p . x_p' + 1) + a_pq sum_g' x_p[gd_p'g'] b_p'g'q
//              + a_p'q sum_g x_p'[gd_pg] b_pgq + sum_{gd_pg = gd_p'g'} b_pgq b_p'g'q.

// XX[p,p'] = x_p . x_p' for p' <= p (odd din / unaligned points; else a split-K GEMM)
__global__ void __launch_bounds__(256) k_xx_dot(Classes T, double* __restrict__ XX, long long ldxx) {
  const long long p = blockIdx.x;
  const ClassDev& C = T.c[find_class(T, p)];
  const double* xp = C.pts + (p - C.row0) * T.din;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long p2 = warp; p2 <= p; p2 += 8) {
    const ClassDev& D = T.c[find_class(T, p2)];
    const double* xq = D.pts + (p2 - D.row0) * T.din;
    double acc = 0.0;
    for (int j = lane; j < T.din; j += 32) acc = fma(xp[j], xq[j], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) XX[p * ldxx + p2] = acc;
  }
}

// K[p,p'] += K_in[p,p'] and its mirror (p' <= p): CTA (p, 8-column group), a warp per p'
__global__ void __launch_bounds__(256) k_gram_input(Classes T, const double* __restrict__ Zb,
                                                      long long ldz, int w1,
                                                      const double* __restrict__ XX,
                                                      long long ldxx, double* __restrict__ K,
                                                      long long ldK) {
  __shared__ int gdp[MAXG];
  const long long p = blockIdx.x;
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const int ngp = C.ngrad;
  if (threadIdx.x < ngp) gdp[threadIdx.x] = gdim(C, threadIdx.x, i);
  __syncthreads();
  const double* xp = C.pts + i * T.din;
  const double* zp = Zb + (C.act0 + i * C.nch) * ldz;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  {
    const long long p2 = static_cast<long long>(blockIdx.y) * 8 + warp;
    if (p2 > p) return;
    const ClassDev& D = T.c[find_class(T, p2)];
    const long long i2 = p2 - D.row0;
    const int ngq = D.ngrad;
    const double* xq = D.pts + i2 * T.din;
    const double* zq = Zb + (D.act0 + i2 * D.nch) * ldz;
    const double s0 = XX[p * ldxx + p2] + 1.0;
    double cq[MAXG], cp[MAXG];
    int gq[MAXG];
    unsigned mm[MAXG];
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
      gq[g] = g < ngq ? gdim(D, g, i2) : -1;
      cq[g] = g < ngq ? xp[gq[g]] : 0.0;   // x_p at p2's derivative dims
      cp[g] = g < ngp ? xq[gdp[g]] : 0.0;  // x_p2 at p's derivative dims
    }
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
      unsigned b = 0;
#pragma unroll
      for (int h = 0; h < MAXG; ++h)
        if (g < ngp && h < ngq && gdp[g] == gq[h]) b |= 1u << h;
      mm[g] = b;
    }
    double acc = 0.0;
    for (int q = lane; q < w1; q += 32) {
      const double ap = zp[q], aq = zq[q];
      double u = aq * s0, v = 0.0;
#pragma unroll
      for (int g = 0; g < MAXG; ++g) {
        if (g < ngq) u = fma(cq[g], zq[(1 + g) * ldz + q], u);
        if (g < ngp) v = fma(cp[g], zp[(1 + g) * ldz + q], v);
      }
      acc = fma(ap, u, acc);
      acc = fma(aq, v, acc);
#pragma unroll
      for (int g = 0; g < MAXG; ++g) {
        if (mm[g]) {
          const double bp = zp[(1 + g) * ldz + q];
          for (int h = 0; h < MAXG; ++h)
            if ((mm[g] >> h) & 1u) acc = fma(bp, zq[(1 + h) * ldz + q], acc);
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      K[p * ldK + p2] += acc;
      if (p2 != p) K[p2 * ldK + p] += acc;
    }
  }
}

// (J^T w) over the input block: out[j,q] = scale (sum_p x_pj w_p a_pq + sum_{gd_pg = j}
// w_p b_pgq), bias row j = din with x = 1.  CTA = 32 rows j x 128 neurons q (256
// threads: 128 q x two halves of 16 rows).  Points stream through double-buffered
// shared memory JW_P at a time, the next chunk's global loads in flight (registers)
// while the current one is multiplied.  The one-hot rows of a chunk are compacted
// in (point, channel) order by one warp (ballot) and applied one chunk later, so
// the summation order is fixed.
constexpr int JW_J = 32, JW_P = 16, JW_XLD = JW_J + 2, JW_L = JW_P * MAXG;
struct JwSmem {
  double xs[2][JW_P][JW_XLD];
  double was[2][JW_P][128];
  long long lz[2][JW_L];  // Zbar offset of the one-hot channel row
  double lw[2][JW_L];
  int ld[2][JW_L];
  int lcnt[2];
  long long szrow[2][JW_P];
  double swt[2][JW_P];
  int sgd[2][JW_P][MAXG];
  int sng[2][JW_P];
};
constexpr size_t kJwSmem = sizeof(JwSmem) + 16;

__global__ void __launch_bounds__(256, 2) k_jt_input_wide(Classes T, const double* __restrict__ Zb,
                                                            long long ldz, int w1,
                                                            const double* __restrict__ wvec,
                                                            double scale,
                                                            double* __restrict__ out) {
  extern __shared__ uint8_t jw_raw[];
  JwSmem& S = *reinterpret_cast<JwSmem*>(smem_align(jw_raw, 16));
  const int tid = threadIdx.x;
  // staging: thread column sq of the 128-neuron block; products: thread (jg, tq2)
  // owns rows jb .. jb+7 and neurons q, q+1 (8 x 2 accumulators: one LDS.128 of
  // w a and four of x per 16 FMAs)
  const int sq = tid & 127;
  const int sqg = blockIdx.y * 128 + sq;
  const int tq2 = tid & 63, jg = tid >> 6;
  const int j0 = blockIdx.x * JW_J;
  const int q = blockIdx.y * 128 + 2 * tq2;
  const int din = T.din;
  const int jb = j0 + jg * 8;
  const int nchunks = static_cast<int>((T.m + JW_P - 1) / JW_P);
  double acc[8][2];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r][0] = acc[r][1] = 0.0;
  // register stage of one chunk
  double xr[2], ar[8];
  // chunk c: x and w a into registers; the point info straight into buffer c & 1
  // (its last reader, the compaction of chunk c - 2, precedes the last barrier)
  auto load = [&](int c) {
    const long long p0 = static_cast<long long>(c) * JW_P;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const long long p = p0 + (tid >> 5) + 8 * k;
      const int j = j0 + (tid & 31);
      double x = 0.0;
      if (p < T.m) {
        const ClassDev& C = T.c[find_class(T, p)];
        x = j < din ? __ldg(C.pts + (p - C.row0) * din + j) : (j == din ? 1.0 : 0.0);
      }
      xr[k] = x;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long p = p0 + (tid >> 7) + 2 * k;
      double a = 0.0;
      if (p < T.m && sqg < w1) {
        const ClassDev& C = T.c[find_class(T, p)];
        a = __ldg(wvec + p) * __ldg(Zb + (C.act0 + (p - C.row0) * C.nch) * ldz + sqg);
      }
      ar[k] = a;
    }
    if (tid < JW_P) {
      const int b = c & 1;
      const long long p = p0 + tid;
      int ng = 0;
      if (p < T.m) {
        const ClassDev& C = T.c[find_class(T, p)];
        const long long i = p - C.row0;
        S.swt[b][tid] = __ldg(wvec + p);
        S.szrow[b][tid] = (C.act0 + i * C.nch) * ldz;
        ng = C.ngrad;
        for (int g = 0; g < ng; ++g) S.sgd[b][tid][g] = gdim(C, g, i);
      }
      S.sng[b][tid] = ng;
    }
  };
  auto apply = [&](int b) {  // one-hot rows of the chunk compacted into list b
    if (q >= w1) return;
    const int n = S.lcnt[b];
    for (int t = 0; t < n; ++t) {
      const int d = S.ld[b][t];
      if (d < jb || d >= jb + 8) continue;
      const double* zr = Zb + S.lz[b][t] + q;
      const double v0 = S.lw[b][t] * __ldg(zr);
      const double v1 = q + 1 < w1 ? S.lw[b][t] * __ldg(zr + 1) : 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (d == jb + r) {
          acc[r][0] += v0;
          acc[r][1] += v1;
        }
    }
  };
  if (nchunks > 0) load(0);
  for (int c = 0; c < nchunks; ++c) {
    const int b = c & 1;
    // registers -> buffer b (its last readers finished before the previous barrier)
#pragma unroll
    for (int k = 0; k < 2; ++k) S.xs[b][(tid >> 5) + 8 * k][tid & 31] = xr[k];
#pragma unroll
    for (int k = 0; k < 8; ++k) S.was[b][(tid >> 7) + 2 * k][sq] = ar[k];
    __syncthreads();
    if (tid < 32) {  // compact this chunk's one-hot rows into list b
      int base = 0;
      for (int e0 = 0; e0 < JW_L; e0 += 32) {
        const int e = e0 + tid;
        const int pp = e / MAXG, g = e - (e / MAXG) * MAXG;
        const int d = (e < JW_L && g < S.sng[b][pp]) ? S.sgd[b][pp][g] : -1;
        const bool hit = d >= j0 && d < j0 + JW_J;
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int pos = base + __popc(bal & ((1u << tid) - 1u));
          S.lz[b][pos] = S.szrow[b][pp] + (1 + g) * ldz;
          S.lw[b][pos] = S.swt[b][pp];
          S.ld[b][pos] = d;
        }
        base += __popc(bal);
      }
      if (tid == 0) S.lcnt[b] = base;
    }
    if (c + 1 < nchunks) load(c + 1);  // in flight during the products below
    const int np = static_cast<int>(min(static_cast<long long>(JW_P),
                                        T.m - static_cast<long long>(c) * JW_P));
    for (int pp = 0; pp < np; ++pp) {
      const double2 a2 = *reinterpret_cast<const double2*>(&S.was[b][pp][2 * tq2]);
      const double2* xv2 = reinterpret_cast<const double2*>(&S.xs[b][pp][jg * 8]);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double2 xv = xv2[r];
        acc[2 * r][0] = fma(xv.x, a2.x, acc[2 * r][0]);
        acc[2 * r][1] = fma(xv.x, a2.y, acc[2 * r][1]);
        acc[2 * r + 1][0] = fma(xv.y, a2.x, acc[2 * r + 1][0]);
        acc[2 * r + 1][1] = fma(xv.y, a2.y, acc[2 * r + 1][1]);
      }
    }
    if (c >= 1) apply(b ^ 1);  // previous chunk's list (complete since this barrier)
  }
  __syncthreads();
  if (nchunks > 0) apply((nchunks - 1) & 1);
  if (q >= w1) return;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (jb + r > din) continue;
    double* o = out + static_cast<long long>(jb + r) * w1 + q;
    o[0] = scale * acc[r][0];
    if (q + 1 < w1) o[1] = scale * acc[r][1];
  }
}

// ---- the same input block on the FP64 tensor cores (din >= 64): out = Xt Bt^T
// with Xt[j][p] = x_pj (row din = 1: the bias), Bt[q][p] = w_p a_pq, then the
// one-hot rows added by k_jt_onehot in (point, channel) order.
__global__ void k_xt_build(Classes T, double* __restrict__ Xt, long long ldm) {
  __shared__ double tile[32][33];
  const int din = T.din;
  const long long p0 = static_cast<long long>(blockIdx.x) * 32;
  const int j0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const long long p = p0 + r;
    const int j = j0 + threadIdx.x;
    double v = 0.0;
    if (p < T.m) {
      const ClassDev& C = T.c[find_class(T, p)];
      v = j < din ? C.pts[(p - C.row0) * din + j] : (j == din ? 1.0 : 0.0);
    }
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int j = j0 + r;
    const long long p = p0 + threadIdx.x;
    if (j <= din && p < ldm) Xt[static_cast<long long>(j) * ldm + p] = tile[threadIdx.x][r];
  }
}

__global__ void k_bt_build(Classes T, const double* __restrict__ Zb, long long ld, int w1,
                           const double* __restrict__ wvec, double* __restrict__ Bt,
                           long long ldm) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= w1 * ldm) return;
  const int q = static_cast<int>(idx / ldm);
  const long long p = idx - q * ldm;
  double v = 0.0;
  if (p < T.m) {
    const ClassDev& C = T.c[find_class(T, p)];
    v = wvec[p] * Zb[(C.act0 + (p - C.row0) * C.nch) * ld + q];
  }
  Bt[idx] = v;
}

// out[d][q] += scale w_p b_pgq for every derivative channel (p, g) with dim d in this
// CTA's row range, in (p, g) order (deterministic; one CTA owns each row).  The
// dims of 128 points at a time are staged in shared memory, so the scan over all
// (p, g) is a shared-memory loop instead of a chain of global loads.
constexpr int OH_ROWS = 512;
__global__ void __launch_bounds__(128) k_jt_onehot(Classes T, const double* __restrict__ Zb,
                                                     long long ld, int w1,
                                                     const double* __restrict__ wvec,
                                                     double scale, double* __restrict__ out) {
  __shared__ int sd[128][MAXG];
  __shared__ int sng[128];
  const int j0 = blockIdx.x * OH_ROWS, j1 = min(j0 + OH_ROWS, T.din);
  for (long long p0 = 0; p0 < T.m; p0 += 128) {
    const int np = static_cast<int>(min(128LL, T.m - p0));
    __syncthreads();
    if (threadIdx.x < np) {
      const long long p = p0 + threadIdx.x;
      const ClassDev& C = T.c[find_class(T, p)];
      const long long i = p - C.row0;
      sng[threadIdx.x] = C.ngrad;
      for (int g = 0; g < C.ngrad; ++g) sd[threadIdx.x][g] = gdim(C, g, i);
    }
    __syncthreads();
    for (int pp = 0; pp < np; ++pp) {
      const int ng = sng[pp];
      for (int g = 0; g < ng; ++g) {
        const int d = sd[pp][g];
        if (d < j0 || d >= j1) continue;
        const long long p = p0 + pp;
        const ClassDev& C = T.c[find_class(T, p)];
        const long long i = p - C.row0;
        const double wp = scale * wvec[p];
        const double* zr = Zb + (C.act0 + i * C.nch + 1 + g) * ld;
        double* o = out + static_cast<long long>(d) * w1;
        for (int q = threadIdx.x; q < w1; q += blockDim.x) o[q] = fma(wp, zr[q], o[q]);
      }
    }
  }
}

// ------------------------------------------------------------------ f_vv (t-jets)

struct T2 {
  double a, b, c;
};
DNGD_DEV T2 t2mul(T2 x, T2 y) {
  return {x.a * y.a, fma(x.b, y.a, x.a * y.b), fma(x.c, y.a, fma(x.a, y.c, 2.0 * x.b * y.b))};
}

// channels of one (point, neuron) given z triples -> tanh triples.
// zget(ch) returns the triple of channel ch; hput(ch, triple) stores it.
template <class ZGet, class HPut>
DNGD_DEV void tanh_tjet(const ClassDev& C, ZGet zget, HPut hput) {
  const T2 z0 = zget(0);
  const double t = tanh(z0.a), s = 1.0 - t * t;
  const T2 Tt = {t, s * z0.b, fma(s, z0.c, -2.0 * t * s * z0.b * z0.b)};
  const T2 S = {s, -2.0 * t * Tt.b, -2.0 * fma(Tt.b, Tt.b, t * Tt.c)};
  hput(0, Tt);
  for (int g = 0; g < C.ngrad; ++g) hput(1 + g, t2mul(S, zget(1 + g)));
  if (C.nlap) {
    T2 G = {0.0, 0.0, 0.0};
    for (int l = 0; l < C.nlap; ++l) {
      const T2 zg = zget(C.lap_ch[l]);
      const T2 sq = t2mul(zg, zg);
      G = {G.a + sq.a, G.b + sq.b, G.c + sq.c};
    }
    const T2 Q = t2mul(Tt, S);
    const T2 a = t2mul(S, zget(C.nch - 1));
    const T2 b = t2mul(Q, G);
    hput(C.nch - 1, {a.a - 2.0 * b.a, a.b - 2.0 * b.b, a.c - 2.0 * b.c});
  }
}

// input layer of the f_vv pass: H3 holds [a; b; c] blocks of R rows each.
template <int ORD>  // 2: f_vv (a, b, c jets); 1: J v (a, b only -- the c block is never read)
__global__ void k_fvv_input(Classes T, const double* __restrict__ theta,
                            const double* __restrict__ v, int w1, long long ld,
                            double* __restrict__ H3, const double* __restrict__ Zx,
                            const double* __restrict__ Dx, long long ldx) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.m * w1) return;
  const long long p = idx / w1;
  const int q = static_cast<int>(idx - p * w1);
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long boff = static_cast<long long>(T.din) * w1;
  const long long base = (C.act0 + i * C.nch) * ld + q;
  const long long blk = T.R * ld;
  auto hput = [&](int ch, T2 h) {
    const long long o = base + ch * ld;
    H3[o] = h.a;
    H3[o + blk] = h.b;
    if (ORD == 2) H3[o + 2 * blk] = h.c;
  };
  if (C.inp) {
    // embedded inputs: channel ch is inputs_ch . (W0 + t V0) (+ bias on the value channel)
    const double* xr = C.inp + i * C.nch * T.din;
    auto zget_e = [&](int ch) -> T2 {
      double a = ch == 0 ? theta[boff + q] : 0.0, b = ch == 0 ? v[boff + q] : 0.0;
      for (int j = 0; j < T.din; ++j) {
        a = fma(xr[ch * T.din + j], theta[j * w1 + q], a);
        b = fma(xr[ch * T.din + j], v[j * w1 + q], b);
      }
      return {a, b, 0.0};
    };
    tanh_tjet(C, zget_e, hput);
    return;
  }
  double za = theta[boff + q], zb = v[boff + q];
  if (Zx) {
    za += Zx[p * ldx + q];
    zb += Dx[p * ldx + q];
  } else {
    const double* x = C.pts + i * T.din;
    for (int j = 0; j < T.din; ++j) {
      za = fma(x[j], theta[j * w1 + q], za);
      zb = fma(x[j], v[j * w1 + q], zb);
    }
  }
  auto zget = [&](int ch) -> T2 {
    if (ch == 0) return {za, zb, 0.0};
    if (ch <= C.ngrad) {
      const int d = gdim(C, ch - 1, i);
      return {theta[d * w1 + q], v[d * w1 + q], 0.0};
    }
    return {0.0, 0.0, 0.0};
  };
  tanh_tjet(C, zget, hput);
}

// hidden layer: P = [Ha;Hb;Hc] W (3R rows), Q = [Ha;Hb] V (2R rows)
template <int ORD>  // 2: f_vv; 1: J v (first-order jets: P holds 2R rows, Q R rows)
__global__ void k_fvv_hidden(Classes T, const double* __restrict__ P, const double* __restrict__ Q,
                             const double* __restrict__ b, const double* __restrict__ vb, int w,
                             long long ld, double* __restrict__ H3) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.m * w) return;
  const long long p = idx / w;
  const int q = static_cast<int>(idx - p * w);
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long base = (C.act0 + i * C.nch) * ld + q;
  const long long blk = T.R * ld;
  auto zget = [&](int ch) -> T2 {
    const long long o = base + ch * ld;
    T2 z = {P[o], P[o + blk] + Q[o], ORD == 2 ? P[o + 2 * blk] + 2.0 * Q[o + blk] : 0.0};
    if (ch == 0) {
      z.a += b[q];
      z.b += vb[q];
    }
    return z;
  };
  auto hput = [&](int ch, T2 h) {
    const long long o = base + ch * ld;
    H3[o] = h.a;
    H3[o + blk] = h.b;
    if (ORD == 2) H3[o + 2 * blk] = h.c;
  };
  tanh_tjet(C, zget, hput);
}

// output, order 2: fvv_i = w * sum_c coef_c (Hc_c . W_L + 2 Hb_c . V_L)
//         order 1: (J v)_i = w * sum_c coef_c (Hb_c . W_L + Ha_c . V_L [+ vb_L on c = 0])
__global__ void k_fvv_head(Classes T, const double* __restrict__ H3, int w, long long ld,
                           const double* __restrict__ WL, const double* __restrict__ VL,
                           double* __restrict__ out, int order) {
  const long long p = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= T.m) return;
  const ClassDev& C = T.c[find_class(T, p)];
  const long long i = p - C.row0;
  const long long blk = T.R * ld;
  const double* h = H3 + (C.act0 + i * C.nch) * ld;
  double res = 0.0;
  if (order == 1) {
    for (int c = 0; c < C.nch; ++c) {
      double u = 0.0;
      for (int q = lane; q < w; q += 32)
        u = fma(h[blk + c * ld + q], WL[q], fma(h[c * ld + q], VL[q], u));
      u = warp_sum(u);
      if (c == 0) u += VL[w];
      res = fma(coefp(C, c, i), u, res);
    }
    if (C.c3 != 0.0) {  // d(c3 u^3) = 3 c3 u^2 u'
      double ua = 0.0, ub = 0.0;
      for (int q = lane; q < w; q += 32) {
        ua = fma(h[q], WL[q], ua);
        ub = fma(h[blk + q], WL[q], fma(h[q], VL[q], ub));
      }
      ua = warp_sum(ua) + WL[w];
      ub = warp_sum(ub) + VL[w];
      res = fma(3.0 * C.c3 * ua * ua, ub, res);
    }
    if (lane == 0) out[p] = C.weight * res;
    return;
  }
  for (int c = 0; c < C.nch; ++c) {
    double u = 0.0;
    for (int q = lane; q < w; q += 32)
      u = fma(h[2 * blk + c * ld + q], WL[q], fma(2.0 * h[blk + c * ld + q], VL[q], u));
    u = warp_sum(u);
    res = fma(coefp(C, c, i), u, res);
  }
  if (C.c3 != 0.0) {
    // (u^3)'' = 6 u u'^2 + 3 u^2 u'' on the value channel
    double ua = 0.0, ub = 0.0, uc = 0.0;
    for (int q = lane; q < w; q += 32) {
      ua = fma(h[q], WL[q], ua);
      ub = fma(h[blk + q], WL[q], fma(h[q], VL[q], ub));
      uc = fma(h[2 * blk + q], WL[q], fma(2.0 * h[blk + q], VL[q], uc));
    }
    ua = warp_sum(ua) + WL[w];
    ub = warp_sum(ub) + VL[w];
    uc = warp_sum(uc);
    res = fma(C.c3, 6.0 * ua * ub * ub + 3.0 * ua * ua * uc, res);
  }
  if (lane == 0) out[p] = C.weight * res;
}

// ------------------------------------------------------------------ helpers

// dst[b][j][i] = src[b][i][j] for an (rows x cols) block at src + b*src_s (ld = cols)
__global__ void k_transpose(const double* __restrict__ src, long long src_s, int rows, int cols,
                            double* __restrict__ dst, long long ldd, long long dst_s) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  const double* S = src + blockIdx.z * src_s;
  double* D = dst + blockIdx.z * dst_s;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int r = by + k, c = bx + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? S[static_cast<long long>(r) * cols + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int c = bx + k, r = by + threadIdx.x;  // dst row c, col r
    if (c < cols && r < rows) D[static_cast<long long>(c) * ldd + r] = tile[threadIdx.x][k];
  }
}

// dst (rows x ldd) = src (rows x cols, ld = cols)
__global__ void k_copy2d(const double* __restrict__ src, int rows, int cols,
                         double* __restrict__ dst, long long ldd) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long long>(rows) * cols) return;
  const long long r = idx / cols, c = idx - r * cols;
  dst[r * ldd + c] = src[idx];
}

// entries [k0, n) of every candidate (k0 > 0: the wide input layer's W0 block is
// never materialised per candidate, see input_gemm)
__global__ void k_candidates(const double* __restrict__ theta, const double* __restrict__ delta,
                             const double* __restrict__ etas, long long n,
                             double* __restrict__ out, long long k0 = 0) {
  const long long k = k0 + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (delta == nullptr) {  // explicit candidate stack (loss_many of residuals.py:188-201)
    out[blockIdx.y * n + k] = theta[blockIdx.y * n + k];
  } else {
    out[blockIdx.y * n + k] = fma(etas[blockIdx.y], delta[k], theta[k]);
  }
}

__global__ void __launch_bounds__(256) k_half_sumsq(const double* __restrict__ r, long long m,
                                                      double* __restrict__ out) {
  __shared__ double sh[8];
  const double* x = r + blockIdx.x * m;
  double s = 0.0;
  for (long long k = threadIdx.x; k < m; k += 256) s = fma(x[k], x[k], s);
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = 0.5 * s;
}

// ------------------------------------------------------------------ host

struct Plan {
  int L;
  std::vector<long long> w, off, ld;  // widths, layer offsets in theta, padded widths
  long long n, m, R, wmax, ldmax;
  Classes T;
  // large-din input layer as a split-K GEMM (input_gemm)
  bool bigin = false;
  int big_splits = 1;
  long long big_mmax = 0;
  // wide identity input layer (din > MAXG): J-free Gram through gram_wide_input
  bool wide_in = false;
  long long wi_ncols = 0, wi_ldh = 0, wi_ldxx = 0;
  size_t wi_syrk_bytes = 0, wi_xx_part = 0;
  int wi_xx_splits = 1;
};

// split count for a small M x N output over a long K (>= 256 columns per split,
// one wave of 128x128 tiles -- one CTA per SM -- and no empty split)
static int wide_k_splits(int nsm, long long M, long long N, long long K) {
  const long long tiles = ((M + 127) / 128) * ((N + 127) / 128);
  const long long kc = (K + 15) / 16;
  long long S = std::max(1LL, nsm / tiles);
  S = std::max(1LL, std::min(S, kc / 16));
  const long long per = (kc + S - 1) / S;
  return static_cast<int>((kc + per - 1) / per);
}

// din at which x W0 leaves the per-(point, neuron) loop for the tensor cores
constexpr int kBigInputDin = 64;

static int make_plan(dngd_ctx* ctx, const dngd_mlp_desc* mlp, const dngd_class_desc* cls,
                     int nclass, Plan& P) {
  if (!mlp || mlp->nlayers < 2 || mlp->nlayers > DNGD_MAX_LAYERS) {
    return set_error(ctx, DNGD_ERR_UNSUPPORTED, "pinn: need 2..8 affine layers");
  }
  if (nclass < 1 || nclass > MAXC) {
    return set_error(ctx, DNGD_ERR_UNSUPPORTED, "pinn: need 1..4 residual classes");
  }
  P.L = mlp->nlayers;
  P.w.assign(mlp->widths, mlp->widths + P.L + 1);
  if (P.w[P.L] != 1) return set_error(ctx, DNGD_ERR_DIMENSION, "pinn: scalar output required");
  P.off.resize(P.L);
  long long off = 0;
  P.wmax = 0;
  for (int k = 0; k < P.L; ++k) {
    P.off[k] = off;
    off += (P.w[k] + 1) * P.w[k + 1];
    if (k >= 1) P.wmax = std::max(P.wmax, P.w[k]);
  }
  P.n = off;
  P.ld.resize(P.L + 1);
  for (int k = 0; k <= P.L; ++k) P.ld[k] = ldw(P.w[k]);
  P.ldmax = ldw(P.wmax);
  Classes& T = P.T;
  T.n = nclass;
  T.din = static_cast<int>(P.w[0]);
  long long row = 0, act = 0;
  for (int k = 0; k < nclass; ++k) {
    const dngd_class_desc& d = cls[k];
    ClassDev& C = T.c[k];
    if (d.ngrad < 0 || d.ngrad > MAXG || d.nlap < 0 || d.nlap > d.ngrad) {
      return set_error(ctx, DNGD_ERR_UNSUPPORTED, "pinn: too many derivative channels");
    }
    C.row0 = row;
    C.count = d.count;
    C.act0 = act;
    C.ngrad = d.ngrad;
    C.nlap = d.nlap;
    C.nch = 1 + d.ngrad + (d.nlap ? 1 : 0);
    for (int g = 0; g < MAXG; ++g) {
      C.grad_dims[g] = g < d.ngrad ? d.grad_dims[g] : 0;
      C.cg[g] = g < d.ngrad ? d.cg[g] : 0.0;
      C.lap_ch[g] = g < d.nlap ? 1 + d.lap_grad[g] : 0;
      if (g < d.ngrad && (d.grad_dims[g] < 0 || d.grad_dims[g] >= T.din)) {
        return set_error(ctx, DNGD_ERR_DOMAIN, "pinn: derivative dimension out of range");
      }
    }
    C.cu = d.cu;
    C.cl = d.cl;
    C.weight = d.weight;
    C.c3 = d.c3;
    C.pts = d.points;
    C.f = d.f;
    C.inp = d.inputs;
    C.pgi = d.grad_idx;
    C.pco = d.coefs;
    if (C.inp == nullptr && C.pts == nullptr && d.count > 0) {
      return set_error(ctx, DNGD_ERR_DIMENSION, "pinn: class needs points or input channels");
    }
    row += d.count;
    act += d.count * C.nch;
  }
  T.m = row;
  T.R = act;
  T.u0 = nullptr;
  P.m = row;
  P.R = act;
  P.bigin = T.din >= kBigInputDin && (T.din % 2) == 0;
  P.big_mmax = 0;
  for (int k = 0; k < nclass; ++k) {
    const ClassDev& C = T.c[k];
    if (C.count == 0) continue;
    if (C.inp || (reinterpret_cast<uintptr_t>(C.pts) & 15)) P.bigin = false;
    P.big_mmax = std::max(P.big_mmax, C.count);
  }
  if (P.bigin && P.big_mmax > 0) {
    P.big_splits = wide_k_splits(ctx->num_sms, P.big_mmax, P.w[1], T.din);
  } else {
    P.bigin = false;
  }
  P.wide_in = T.din > MAXG;
  for (int k = 0; k < nclass; ++k)
    if (T.c[k].inp) P.wide_in = false;
  if (P.wide_in) {
    P.wi_ncols = P.n - P.off[1];
    P.wi_ldh = (P.wi_ncols + 3) / 4 * 4;
    P.wi_ldxx = (P.m + 3) / 4 * 4;
    int S;
    long long nt;
    int rc = syrk_plan(ctx, P.m, P.wi_ncols, &S, &nt, &P.wi_syrk_bytes);
    if (rc) return rc;
    if (P.bigin) {
      P.wi_xx_splits = wide_k_splits(ctx->num_sms, P.big_mmax, P.big_mmax, T.din);
      P.wi_xx_part = gemm_splitk_bytes(P.big_mmax, P.big_mmax, P.wi_xx_splits);
    }
  }
  return DNGD_OK;
}

// workspace carve-out (bytes, 256-aligned)
struct Arena {
  char* base;
  size_t off = 0;
  double* take(size_t elems) {
    double* p = reinterpret_cast<double*>(base ? base + off : nullptr);
    off += (elems * sizeof(double) + 255) / 256 * 256;
    return p;
  }
};

struct BigIn {
  double* Wt = nullptr;    // W0^T (w1 x din)
  double* part = nullptr;  // split-K partial tiles
  double* Zx = nullptr;    // x W0 rows (m x ld1)
  double* Dx = nullptr;    // x V0 rows: f_vv / line-search direction
};

static void carve_bigin(const Plan& P, Arena& A, BigIn& G, bool dir) {
  if (!P.bigin) return;
  G.Wt = A.take(static_cast<size_t>(P.w[1]) * P.w[0]);
  G.part = A.take(gemm_splitk_bytes(P.big_mmax, P.w[1], P.big_splits) / sizeof(double));
  G.Zx = A.take(static_cast<size_t>(P.m) * P.ld[1]);
  if (dir) G.Dx = A.take(static_cast<size_t>(P.m) * P.ld[1]);
}

// Ozaki digits of the hidden-layer GEMMs (activation pass, f_vv, line-search
// forward): DNGD_GEMM_SLICES (0, 6, 7) overrides; default 6 when a hidden layer is
// 128 wide or more (the int8 tensor cores beat the FP64 DMMA GEMM there), else the
// DMMA GEMM
static int oz_ls_slices(const Plan& P) {
  if (const char* e = getenv("DNGD_GEMM_SLICES")) {
    const int v = atoi(e);
    return (v == 6 || v == 7) ? v : 0;
  }
  if (P.L < 3) return 0;
  long long wmax = 0;
  for (int k = 1; k <= P.L - 2; ++k) wmax = std::max(wmax, std::max(P.w[k], P.w[k + 1]));
  return wmax >= 128 ? 6 : 0;
}

// digit planes for one emulated GEMM of up to rows_a x K by rows_b x K
struct OzScratch {
  int S = 0;
  long long cap_a = 0, cap_b = 0, kcap = 0;
  int8_t *QA = nullptr, *QB = nullptr;
  double *sA = nullptr, *sB = nullptr;
};

static void carve_oz(const Plan& P, Arena& A, OzScratch& O, long long rows_a, long long rows_b,
                     long long kmax) {
  O.S = oz_ls_slices(P);
  if (!O.S) return;
  O.cap_a = rows_a;
  O.cap_b = rows_b;
  O.kcap = oz_kpad(kmax);
  O.QA = reinterpret_cast<int8_t*>(A.take((static_cast<size_t>(O.S) * rows_a * O.kcap + 7) / 8));
  O.QB = reinterpret_cast<int8_t*>(A.take((static_cast<size_t>(O.S) * rows_b * O.kcap + 7) / 8));
  O.sA = A.take(static_cast<size_t>(rows_a));
  O.sB = A.take(static_cast<size_t>(rows_b));
}

static long long hidden_wmax(const Plan& P) {
  long long w = 1;
  for (int k = 1; k <= P.L - 1; ++k) w = std::max(w, P.w[k]);
  return w;
}

// C = A B^T (alpha 1, beta 0, one batch) on the int8 tensor cores when the
// scratch allows it, else the FP64 DMMA GEMM
static int gemm_nt_hidden(dngd_ctx* ctx, cudaStream_t s, const GemmCall& g, const OzScratch& O) {
  if (!O.S || g.batch != 1 || g.alpha != 1.0 || g.beta != 0.0 || g.lower || g.M > O.cap_a ||
      g.N > O.cap_b || oz_kpad(g.K) > O.kcap || g.K < 64) {
    return gemm_nt(ctx, s, g);
  }
  int rc = oz_slice(ctx, s, g.A, g.M, g.K, g.lda, O.S, O.QA, O.sA);
  if (rc == DNGD_OK) rc = oz_slice(ctx, s, g.B, g.N, g.K, g.ldb, O.S, O.QB, O.sB);
  if (rc == DNGD_OK) {
    rc = oz_gemm_batched(ctx, s, O.QA, O.sA, g.M, 0, O.QB, O.sB, g.N, 0, oz_kpad(g.K), O.S, g.M,
                         g.N, 1, g.C, g.ldc, 0);
  }
  return rc;
}

struct AsmBufs {
  std::vector<double*> Z, H, Zb, Wt, Wp;
  BigIn big;
  double* Hb;
  double* H0;  // materialised input channels (factored Gram), R x 16
  double* u0;  // per-point network value (cubic-term adjoint seeds), m
  // wide input layer: hidden/output columns of J, SYRK partials, X X^T (+ partials)
  double *Jh = nullptr, *syrk_work = nullptr, *XX = nullptr, *xx_part = nullptr;
  OzScratch oz;  // emulated hidden-layer GEMMs of the activation pass (carved last)
};

static void carve_assemble(const Plan& P, Arena& A, AsmBufs& B) {
  const int L = P.L;
  B.Z.assign(L, nullptr);
  B.H.assign(L, nullptr);
  B.Zb.assign(L, nullptr);
  B.Wt.assign(L, nullptr);
  B.Wp.assign(L, nullptr);
  for (int k = 0; k <= L - 2; ++k) B.Z[k] = A.take(P.R * P.ld[k + 1]);
  for (int k = 1; k <= L - 1; ++k) B.H[k] = A.take(P.R * P.ld[k]);
  for (int k = 0; k <= L - 2; ++k) B.Zb[k] = A.take(P.R * P.ld[k + 1]);
  B.Hb = A.take(P.R * P.ldmax);
  for (int k = 1; k <= L - 2; ++k) {
    B.Wt[k] = A.take(P.w[k + 1] * P.ld[k]);
    B.Wp[k] = A.take(P.w[k] * P.ld[k + 1]);
  }
  B.H0 = A.take(P.R * 16);
  B.u0 = A.take(P.m);
  carve_bigin(P, A, B.big, false);
  if (P.wide_in) {
    B.Jh = A.take(static_cast<size_t>(P.m) * P.wi_ldh);
    B.syrk_work = A.take(P.wi_syrk_bytes / sizeof(double) + 1);
    B.XX = A.take(static_cast<size_t>(P.m) * P.wi_ldxx);
    if (P.wi_xx_part) B.xx_part = A.take(P.wi_xx_part / sizeof(double));
  }
  carve_oz(P, A, B.oz, P.R, hidden_wmax(P), hidden_wmax(P));
}

struct FvvBufs {
  std::vector<double*> H3, Wt, Vt;
  double *P3, *Q2;
  BigIn big;
  OzScratch oz;
};

static void carve_fvv(const Plan& P, Arena& A, FvvBufs& B) {
  const int L = P.L;
  B.H3.assign(L, nullptr);
  B.Wt.assign(L, nullptr);
  B.Vt.assign(L, nullptr);
  B.H3[0] = A.take(3 * P.R * P.ldmax);  // ping
  B.H3[1] = A.take(3 * P.R * P.ldmax);  // pong
  B.P3 = A.take(3 * P.R * P.ldmax);
  B.Q2 = A.take(2 * P.R * P.ldmax);
  for (int k = 1; k <= L - 2; ++k) {
    B.Wt[k] = A.take(P.w[k + 1] * P.ld[k]);
    B.Vt[k] = A.take(P.w[k + 1] * P.ld[k]);
  }
  carve_bigin(P, A, B.big, true);
  carve_oz(P, A, B.oz, 3 * P.R, hidden_wmax(P), hidden_wmax(P));
}

struct LossBufs {
  double *thetas, *Hping, *Hpong, *Z, *r;
  std::vector<double*> Wt;
  BigIn big;
  // emulated-FP64 hidden-layer GEMMs (ozaki.cu): digit planes of cb candidates
  int oz_S = 0, oz_cb = 0;
  int8_t *ozQA = nullptr, *ozQB = nullptr;
  double *ozsA = nullptr, *ozsB = nullptr;
};

static void carve_loss(const Plan& P, Arena& A, LossBufs& B, int C) {
  B.thetas = A.take(static_cast<size_t>(C) * P.n);
  B.Hping = A.take(static_cast<size_t>(C) * P.R * P.ldmax);
  B.Hpong = A.take(static_cast<size_t>(C) * P.R * P.ldmax);
  B.Z = A.take(static_cast<size_t>(C) * P.R * P.ldmax);
  B.r = A.take(static_cast<size_t>(C) * P.m);
  B.Wt.assign(P.L, nullptr);
  for (int k = 1; k <= P.L - 2; ++k) B.Wt[k] = A.take(static_cast<size_t>(C) * P.w[k + 1] * P.ld[k]);
  carve_bigin(P, A, B.big, true);
  B.oz_S = P.L >= 3 ? oz_ls_slices(P) : 0;
  if (B.oz_S) {
    long long kp = 0, nmax = 0;
    for (int k = 1; k <= P.L - 2; ++k) {
      kp = std::max(kp, oz_kpad(P.w[k]));
      nmax = std::max(nmax, P.w[k + 1]);
    }
    // candidates per slicing pass: A digit planes within ~2 GiB
    const long long per = static_cast<long long>(B.oz_S) * P.R * kp;
    B.oz_cb = static_cast<int>(std::max(1LL, std::min<long long>(C, (2LL << 30) / std::max(per, 1LL))));
    const size_t qa = static_cast<size_t>(per) * B.oz_cb;
    const size_t qb = static_cast<size_t>(B.oz_S) * nmax * kp * B.oz_cb;
    B.ozQA = reinterpret_cast<int8_t*>(A.take((qa + 7) / 8));
    B.ozQB = reinterpret_cast<int8_t*>(A.take((qb + 7) / 8));
    B.ozsA = A.take(static_cast<size_t>(P.R) * B.oz_cb);
    B.ozsB = A.take(static_cast<size_t>(nmax) * B.oz_cb);
  }
}

static inline unsigned nblk(long long n, int t = 256) {
  return static_cast<unsigned>((n + t - 1) / t);
}

// transpose W_k (rows w_k x cols w_{k+1}, ld cols) of `batch` thetas into dst (cols x ldd)
static void launch_transpose(cudaStream_t s, const double* W, long long src_s, int rows, int cols,
                             double* dst, long long ldd, long long dst_s, int batch) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, batch);
  k_transpose<<<grid, dim3(32, 8), 0, s>>>(W, src_s, rows, cols, dst, ldd, dst_s);
}

// W_k -> W_k^T for every hidden layer k = 1..L-2 of one theta: one batched launch
// when the hidden layers share a shape (their theta blocks and the destination
// buffers are then equally spaced), else one launch per layer
static void transpose_hidden(cudaStream_t s, const Plan& P, const double* th,
                             const std::vector<double*>& Wt) {
  const int L = P.L;
  bool uniform = L - 2 >= 2;
  for (int k = 2; uniform && k <= L - 2; ++k) {
    uniform = P.w[k] == P.w[1] && P.w[k + 1] == P.w[2] && P.ld[k] == P.ld[1] &&
              Wt[k] - Wt[k - 1] == Wt[2] - Wt[1] && P.off[k] - P.off[k - 1] == P.off[2] - P.off[1];
  }
  if (uniform) {
    launch_transpose(s, th + P.off[1], P.off[2] - P.off[1], static_cast<int>(P.w[1]),
                     static_cast<int>(P.w[2]), Wt[1], P.ld[1], Wt[2] - Wt[1], L - 2);
    return;
  }
  for (int k = 1; k <= L - 2; ++k)
    launch_transpose(s, th + P.off[k], 0, static_cast<int>(P.w[k]), static_cast<int>(P.w[k + 1]),
                     Wt[k], P.ld[k], 0, 1);
}

// out = X W for the (din x w1) block W laid out like W0 (the STDE case, din ~ 1e5):
// per class one split-K FP64 tensor-core GEMM over the raw points instead of a
// din-long dot product per (point, neuron).  out rows are points (ld ld1).
static int input_gemm(dngd_ctx* ctx, cudaStream_t s, const Plan& P, const BigIn& G,
                      const double* W, double* out) {
  const int din = P.T.din, w1 = static_cast<int>(P.w[1]);
  launch_transpose(s, W, 0, din, w1, G.Wt, din, 0, 1);
  const size_t pb = gemm_splitk_bytes(P.big_mmax, w1, P.big_splits);
  for (int c = 0; c < P.T.n; ++c) {
    const ClassDev& C = P.T.c[c];
    if (C.count == 0) continue;
    GemmCall g;
    g.M = C.count;
    g.N = w1;
    g.K = din;
    g.A = C.pts;
    g.lda = din;
    g.B = G.Wt;
    g.ldb = din;
    g.C = out + C.row0 * P.ld[1];
    g.ldc = P.ld[1];
    const int rc = gemm_nt_splitk(ctx, s, g, P.big_splits, G.part, pb);
    if (rc) return rc;
  }
  return DNGD_OK;
}

// forward through all hidden layers; Hlast receives H_{L-1}.  Used by loss_many
// (batched over candidates) with Z scratch shared across layers.
static int forward_batched(dngd_ctx* ctx, cudaStream_t s, const Plan& P, const double* thetas,
                           int C, LossBufs& B, double** Hlast, const double* theta,
                           const double* delta, const double* etas,
                           const double* zx_act = nullptr, double* r_fused = nullptr) {
  const int L = P.L;
  const long long act_s = P.R * P.ldmax;
  // emulated GEMMs with plain inputs: the input layer is fused with the slicing of
  // H_1 (k_input_slice) inside the candidate-chunk loop below
  bool in_fused = B.oz_S != 0 && !P.bigin && oz_kpad(P.w[1]) <= 4LL * 1024 && lap_ascending(P.T);
  for (int c = 0; c < P.T.n; ++c) in_fused = in_fused && P.T.c[c].inp == nullptr && P.T.c[c].nch <= kTsMaxCh;
  if (!in_fused) {
    const double *Zx = nullptr, *Dx = nullptr;
    if (P.bigin && delta != nullptr) {  // x (W0 + eta V0) = x W0 + eta x V0
      int rc = DNGD_OK;
      if (zx_act != nullptr) {
        Zx = zx_act;
      } else {
        rc = input_gemm(ctx, s, P, B.big, theta, B.big.Zx);
        if (rc) return rc;
        Zx = B.big.Zx;
      }
      rc = input_gemm(ctx, s, P, B.big, delta, B.big.Dx);
      if (rc) return rc;
      Dx = B.big.Dx;
    }
    dim3 g(nblk(P.m * P.w[1]), C);
    k_input_fwd<<<g, 256, 0, s>>>(P.T, thetas, P.n, static_cast<int>(P.w[1]), P.ldmax, nullptr,
                                  B.Hping, act_s, Zx, Dx, etas, P.ld[1], theta, delta);
  }
  double* Hcur = B.Hping;
  double* Hnext = B.Hpong;
  if (B.oz_S) {
    // emulated FP64: candidate chunks of oz_cb, layer by layer inside a chunk; the
    // tanh channel map of every layer that feeds another GEMM writes that GEMM's
    // digit planes directly (k_tanh_slice), the last hidden layer writes H_{L-1}
    int maxch = 0;
    for (int c = 0; c < P.T.n; ++c) maxch = std::max(maxch, P.T.c[c].nch);
    const bool fuse = maxch <= kTsMaxCh && lap_ascending(P.T);
    for (int k = 1; k <= L - 2; ++k)
      launch_transpose(s, thetas + P.off[k], P.n, static_cast<int>(P.w[k]),
                       static_cast<int>(P.w[k + 1]), B.Wt[k], P.ld[k], P.w[k + 1] * P.ld[k], C);
    int rc = DNGD_OK;
    for (int b0 = 0; b0 < C && rc == DNGD_OK; b0 += B.oz_cb) {
      const int nb = std::min(B.oz_cb, C - b0);
      if (in_fused) {
        const long long kp1 = oz_kpad(P.w[1]);
        if (B.oz_S == 7) {
          launch_input_slice<7>(s, P.T, thetas + static_cast<long long>(b0) * P.n, P.n,
                                static_cast<int>(P.w[1]), P.R, kp1, nb, B.ozQA, B.ozsA);
        } else {
          launch_input_slice<6>(s, P.T, thetas + static_cast<long long>(b0) * P.n, P.n,
                                static_cast<int>(P.w[1]), P.R, kp1, nb, B.ozQA, B.ozsA);
        }
        rc = cuda_status(ctx, cudaGetLastError(), "input_slice");
      } else {
        rc = oz_slice(ctx, s, B.Hping + b0 * act_s, nb * P.R, P.w[1], P.ldmax, B.oz_S, B.ozQA, B.ozsA);
      }
      for (int k = 1; k <= L - 2 && rc == DNGD_OK; ++k) {
        const long long N = P.w[k + 1], Kd = P.w[k];
        const long long wst = P.w[k + 1] * P.ld[k];
        rc = oz_slice(ctx, s, B.Wt[k] + b0 * wst, nb * N, Kd, P.ld[k], B.oz_S, B.ozQB, B.ozsB);
        if (rc) break;
        rc = oz_gemm_batched(ctx, s, B.ozQA, B.ozsA, nb * P.R, P.R, B.ozQB, B.ozsB, nb * N, N,
                             oz_kpad(Kd), B.oz_S, P.R, N, nb, B.Z + b0 * act_s, P.ldmax, act_s);
        if (rc) break;
        const double* bias = thetas + static_cast<long long>(b0) * P.n + P.off[k] + P.w[k] * P.w[k + 1];
        if (k < L - 2 && fuse) {
          if (B.oz_S == 7) {
            launch_tanh_slice<7>(s, P.T, B.Z + b0 * act_s, static_cast<int>(N), P.ldmax, bias, P.n,
                                 act_s, P.R, oz_kpad(N), nb, B.ozQA, B.ozsA);
          } else {
            launch_tanh_slice<6>(s, P.T, B.Z + b0 * act_s, static_cast<int>(N), P.ldmax, bias, P.n,
                                 act_s, P.R, oz_kpad(N), nb, B.ozQA, B.ozsA);
          }
        } else if (k == L - 2 && r_fused != nullptr && fuse) {
          // last hidden layer + output layer: residuals of the chunk's candidates
          launch_tanh_head(s, P.T, B.Z + b0 * act_s, static_cast<int>(N), P.ldmax,
                           thetas + static_cast<long long>(b0) * P.n, P.n,
                           P.off[k] + P.w[k] * P.w[k + 1], P.off[L - 1], act_s, nb,
                           r_fused + static_cast<long long>(b0) * P.m, P.m);
        } else {
          k_tanh_fwd<<<dim3(nblk(P.m * N), nb), 256, 0, s>>>(P.T, B.Z + b0 * act_s,
                                                             B.Hpong + b0 * act_s, static_cast<int>(N),
                                                             P.ldmax, bias, P.n, act_s);
          if (k < L - 2) {
            rc = oz_slice(ctx, s, B.Hpong + b0 * act_s, nb * P.R, N, P.ldmax, B.oz_S, B.ozQA,
                          B.ozsA);
          }
        }
      }
    }
    if (rc) return rc;
    *Hlast = (r_fused != nullptr && fuse) ? nullptr : B.Hpong;  // nullptr: residuals written
    return cuda_status(ctx, cudaGetLastError(), "forward");
  }
  for (int k = 1; k <= L - 2; ++k) {
    launch_transpose(s, thetas + P.off[k], P.n, static_cast<int>(P.w[k]),
                     static_cast<int>(P.w[k + 1]), B.Wt[k], P.ld[k], P.w[k + 1] * P.ld[k], C);
    GemmCall g;
    g.M = P.R;
    g.N = P.w[k + 1];
    g.K = P.w[k];
    g.A = Hcur;
    g.lda = P.ldmax;
    g.sA = act_s;
    g.B = B.Wt[k];
    g.ldb = P.ld[k];
    g.sB = P.w[k + 1] * P.ld[k];
    g.C = B.Z;
    g.ldc = P.ldmax;
    g.sC = act_s;
    g.batch = C;
    const int rc = gemm_nt(ctx, s, g);
    if (rc) return rc;
    dim3 gr(nblk(P.m * P.w[k + 1]), C);
    k_tanh_fwd<<<gr, 256, 0, s>>>(P.T, B.Z, Hnext, static_cast<int>(P.w[k + 1]), P.ldmax,
                                  thetas + P.off[k] + P.w[k] * P.w[k + 1], P.n, act_s);
    std::swap(Hcur, Hnext);
  }
  *Hlast = Hcur;
  return cuda_status(ctx, cudaGetLastError(), "forward");
}

// ------------------------------------------------------------------ J^T w without J
// The vjp of residuals.py:220-227 from the activations of the last assembly:
//   (J^T w)[W_k|b_k] = sum_rho w_{i(rho)} Hext_k[rho] (x) Zbar_k[rho]
// = Hext_k^T diag(w) Zbar_k, a split-K FP64 tensor-core GEMM over activation
// rows for the hidden layers; the input layer (Hext = input channels) and the
// output layer (Zbar = seeds) are small deterministic reductions.

DNGD_DEV long long act_point(const Classes& T, long long rho, int& ch) {
  int c = 0;
#pragma unroll
  for (int k = 1; k < MAXC; ++k)
    if (k < T.n && rho >= T.c[k].act0) c = k;
  const ClassDev& C = T.c[c];
  const long long loc = rho - C.act0;
  const long long i = loc / C.nch;
  ch = static_cast<int>(loc - i * C.nch);
  return C.row0 + i;
}

// dst[q][rho] = w[point(rho)] * src[rho][q] for q < width; with bias_row the extra
// row dst[width][rho] = (channel(rho) == 0) * w[point(rho)] (Hext's bias entry)
__global__ void k_act_transpose(Classes T, const double* __restrict__ src, long long lds,
                                int width, const double* __restrict__ wvec, int bias_row,
                                double* __restrict__ dst, long long ldd) {
  __shared__ double tile[32][33];
  const long long rho0 = static_cast<long long>(blockIdx.x) * 32;
  const int q0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const long long rho = rho0 + k;
    const int q = q0 + threadIdx.x;
    double v = 0.0;
    if (rho < T.R) {
      int ch;
      const long long i = act_point(T, rho, ch);
      const double s = wvec ? wvec[i] : 1.0;
      if (q < width) {
        v = s * src[rho * lds + q];
      } else if (q == width && bias_row) {
        v = ch == 0 ? s : 0.0;
      }
    }
    tile[k][threadIdx.x] = v;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int q = q0 + k;
    const long long rho = rho0 + threadIdx.x;
    if (q < width + bias_row && rho < T.R) dst[q * ldd + rho] = tile[threadIdx.x][k];
  }
}

// input layer: part[chunk][p][q], p <= din (p == din: bias) over a chunk of points
__global__ void k_jt_input(Classes T, const double* __restrict__ Zb, long long ld, int w1,
                           const double* __restrict__ wvec, long long chunk,
                           double* __restrict__ part) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= w1) return;
  const long long i0 = blockIdx.y * chunk;
  const long long i1 = min(T.m, i0 + chunk);
  const int din = T.din;
  double acc[MAXG + 1];
#pragma unroll
  for (int p = 0; p <= MAXG; ++p) acc[p] = 0.0;
  for (long long i = i0; i < i1; ++i) {
    const ClassDev& C = T.c[find_class(T, i)];
    const long long base = C.act0 + (i - C.row0) * C.nch;
    const double wi = wvec[i];
    const double zv = wi * Zb[base * ld + q];
    acc[MAXG] += zv;
    if (C.inp) {  // embedded input channels: Hext_0[c] = inputs_c
      const double* xr = C.inp + (i - C.row0) * C.nch * din;
      for (int c = 0; c < C.nch; ++c) {
        const double zc = c == 0 ? zv : wi * Zb[(base + c) * ld + q];
#pragma unroll
        for (int p = 0; p < MAXG; ++p)
          if (p < din) acc[p] = fma(xr[c * din + p], zc, acc[p]);
      }
      continue;
    }
    const double* x = C.pts + (i - C.row0) * din;
#pragma unroll
    for (int p = 0; p < MAXG; ++p)
      if (p < din) acc[p] = fma(x[p], zv, acc[p]);
    for (int g = 0; g < C.ngrad; ++g) {
      const double zg = wi * Zb[(base + 1 + g) * ld + q];
#pragma unroll
      for (int p = 0; p < MAXG; ++p)
        if (p == gdim(C, g, i - C.row0)) acc[p] += zg;
    }
  }
  double* dst = part + static_cast<long long>(blockIdx.y) * (din + 1) * w1;
  for (int p = 0; p < din; ++p) dst[p * w1 + q] = acc[p];
  dst[din * w1 + q] = acc[MAXG];
}

// output layer: part[chunk][p], p <= w (p == w: bias)
__global__ void k_jt_output(Classes T, const double* __restrict__ H, long long ld, int w,
                            const double* __restrict__ wvec, long long chunk,
                            double* __restrict__ part) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > w) return;
  const long long i0 = blockIdx.y * chunk;
  const long long i1 = min(T.m, i0 + chunk);
  double acc = 0.0;
  for (long long i = i0; i < i1; ++i) {
    const ClassDev& C = T.c[find_class(T, i)];
    const long long base = C.act0 + (i - C.row0) * C.nch;
    double s = 0.0;
    for (int ch = 0; ch < C.nch; ++ch) {
      const double h = p < w ? H[(base + ch) * ld + p] : (ch == 0 ? 1.0 : 0.0);
      s = fma(seedc(T, C, ch, i), h, s);
    }
    acc = fma(wvec[i], s, acc);
  }
  part[static_cast<long long>(blockIdx.y) * (w + 1) + p] = acc;
}

__global__ void k_chunk_reduce(const double* __restrict__ part, int nchunks, long long count,
                               double scale, double* __restrict__ out) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= count) return;
  double s = 0.0;
  for (int k = 0; k < nchunks; ++k) s += part[static_cast<long long>(k) * count + e];
  out[e] = scale * s;
}

#include "gram_factored.cuh"
#include "gram_oz.cuh"

// ------------------------------------------------------------------ fused line search
// Line-search losses for narrow nets (every width <= 64) in one launch: a CTA
// takes one candidate theta + eta delta and one tile of 64 activation rows of
// one class (64/a points, channels padded to a = 1, 2, 4 or 8 per point), runs
// the whole forward-Laplacian MLP in shared memory -- input channels, per layer
// an FP64 tensor-core GEMM (16-byte fragment loads, pitch 72) and the tanh
// channel map, the head -- and writes the tile's sum of squared residuals.  The
// candidate weights are formed on the fly (fma(eta, delta, theta), bitwise the
// values k_candidates materialises).  No activation ever reaches HBM: the
// launch-per-layer path streamed ~2 GB per line search at config 2.
constexpr int LF_LD = 72;  // activation tiles: 16-byte A-fragment loads, conflict-free
constexpr int LF_WLD = 66;  // weights W[k][q]: the 8-byte B-fragment loads (k = 2(l%4)+h, q = l/4)
                            // and the row-wise staging stores are conflict-free per half warp
constexpr int LF_THREADS = 256;  // 8 warps: latency of the per-layer phases is hidden by 16 warps/SM
constexpr size_t kLossFusedSmem = 3 * 64 * LF_LD * sizeof(double) + (64 + 72) * sizeof(double);

struct LossFusedParams {
  Classes T;
  int L;
  int w[DNGD_MAX_LAYERS + 1];
  long long off[DNGD_MAX_LAYERS];
  const double* thetas;  // candidate stack [cand][n] (k_candidates)
  long long n;
  int lg[MAXC];
  int tile0[MAXC + 1];
  int ntiles;
  double* part;  // [cand][tile]
};

__global__ void __launch_bounds__(LF_THREADS, 2) k_loss_fused(const __grid_constant__ LossFusedParams p) {
  extern __shared__ __align__(16) double lf_smem[];
  double(*H)[LF_LD] = reinterpret_cast<double(*)[LF_LD]>(lf_smem);
  double(*Z)[LF_LD] = reinterpret_cast<double(*)[LF_LD]>(lf_smem + 64 * LF_LD);
  double(*Wk)[LF_WLD] = reinterpret_cast<double(*)[LF_WLD]>(lf_smem + 2 * 64 * LF_LD);
  double* bias = lf_smem + 3 * 64 * LF_LD;
  double* wl = bias + 64;
  __shared__ int s_gd[MAXG], s_lap[MAXG];
  __shared__ double s_coef[8], s_red[LF_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x, cand = blockIdx.y;
  int c = 0;
  while (c + 1 < p.T.n && tile >= p.tile0[c + 1]) ++c;
  const ClassDev& C = p.T.c[c];
  const int lg = p.lg[c], a = 1 << lg, PT = 64 >> lg;
  const long long P0 = static_cast<long long>(tile - p.tile0[c]) * PT;
  const int nch = C.nch, ngrad = C.ngrad, nlap = C.nlap, din = p.T.din;
  const long long count = C.count;
  const double* pts = C.pts;
  const double* inp = C.inp;
  const double c3 = C.c3;
  if (tid < MAXG) {
    s_gd[tid] = C.grad_dims[tid];
    s_lap[tid] = C.lap_ch[tid];
  }
  if (tid < 8) s_coef[tid] = tid < nch ? coef(C, tid) : 0.0;
  const double* th = p.thetas + static_cast<long long>(cand) * p.n;
  // weights -> shared memory with every load of a thread in flight at once
  // (<= 64 x 64 per layer = 16 per thread); dst(kk, q) picks the layout
  auto stage_weights = [&](long long off, int rows, int cols, int rpad, auto dst) {
    double v[4096 / LF_THREADS];
#pragma unroll
    for (int j = 0; j < 4096 / LF_THREADS; ++j) {
      const int e = tid + j * LF_THREADS;
      const int kk = e / cols;
      v[j] = (e < rpad * cols && kk < rows) ? __ldg(th + off + e) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4096 / LF_THREADS; ++j) {
      const int e = tid + j * LF_THREADS;
      if (e < rpad * cols) dst(e / cols, e - (e / cols) * cols) = v[j];
    }
  };
  for (int e = tid; e < 2 * 64 * LF_LD; e += LF_THREADS) lf_smem[e] = 0.0;  // H, Z pads stay 0
  // ---- layer 0: input channels -> tanh channels (thread per (point, unit))
  {
    const int w1 = p.w[1];
    const long long o0 = p.off[0];
    // W0 rows 0..din-1 and b0 (row din) as [row][unit]
    stage_weights(o0, din + 1, w1, din + 1, [&](int kk, int q) -> double& { return Wk[kk][q]; });
    __syncthreads();
    for (int e = tid; e < PT * w1; e += LF_THREADS) {
      const int pl = e / w1, q = e - (e / w1) * w1;
      const long long pi = P0 + pl;
      if (pi >= count) continue;
      double* hrow = &H[pl * a][q];
      if (inp) {  // embedded input channels (same arithmetic as k_input_fwd)
        const double* xr = inp + pi * nch * din;
        auto zch = [&](int ch) {
          double z = ch == 0 ? Wk[din][q] : 0.0;
          for (int d = 0; d < din; ++d) z = fma(xr[ch * din + d], Wk[d][q], z);
          return z;
        };
        const double z = zch(0);
        const double t = tanh(z), s = 1.0 - t * t;
        hrow[0] = t;
        for (int g = 0; g < ngrad; ++g) hrow[(1 + g) * LF_LD] = s * zch(1 + g);
        if (nlap) {
          double G = 0.0;
          for (int l = 0; l < nlap; ++l) {
            const double dz = zch(s_lap[l]);
            G = fma(dz, dz, G);
          }
          hrow[(nch - 1) * LF_LD] = s * zch(nch - 1) - 2.0 * t * s * G;
        }
        continue;
      }
      double z = Wk[din][q];
      for (int d = 0; d < din; ++d) z = fma(pts[pi * din + d], Wk[d][q], z);
      const double t = tanh(z), s = 1.0 - t * t;
      hrow[0] = t;
      for (int g = 0; g < ngrad; ++g) hrow[(1 + g) * LF_LD] = s * Wk[s_gd[g]][q];
      if (nlap) {
        double G = 0.0;
        for (int l = 0; l < nlap; ++l) {
          const double dz = Wk[s_gd[s_lap[l] - 1]][q];
          G = fma(dz, dz, G);
        }
        hrow[(nch - 1) * LF_LD] = -2.0 * t * s * G;
      }
    }
  }
  const int lrow = lane >> 2, kq = lane & 3, wm = warp >> 2, wn = warp & 3;  // warp tile 32 x 16
  // ---- hidden layers: Z = H W_k (tensor cores), H = tanh channels(Z + b_k)
  for (int k = 1; k <= p.L - 2; ++k) {
    const int wk = p.w[k], wk1 = p.w[k + 1];
    const int kpad = (wk + 7) & ~7;
    const long long ok = p.off[k];
    __syncthreads();  // H complete, Wk free
    stage_weights(ok, wk, wk1, kpad, [&](int kk, int q) -> double& { return Wk[kk][q]; });
    if (tid < wk1) bias[tid] = __ldg(th + ok + static_cast<long long>(wk) * wk1 + tid);
    __syncthreads();
    double2 acc[4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) acc[x][y] = make_double2(0.0, 0.0);
    for (int k8 = 0; k8 < kpad; k8 += 8) {
      double2 av[4], bv[2];
#pragma unroll
      for (int x = 0; x < 4; ++x)
        av[x] = *reinterpret_cast<const double2*>(&H[wm * 32 + x * 8 + lrow][k8 + 2 * kq]);
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        bv[y].x = Wk[k8 + 2 * kq][wn * 16 + y * 8 + lrow];
        bv[y].y = Wk[k8 + 2 * kq + 1][wn * 16 + y * 8 + lrow];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) dmma_8x8x4(acc[x][y], av[x].x, bv[y].x);
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) dmma_8x8x4(acc[x][y], av[x].y, bv[y].y);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
        *reinterpret_cast<double2*>(&Z[wm * 32 + x * 8 + lrow][wn * 16 + y * 8 + 2 * kq]) = acc[x][y];
    __syncthreads();
    for (int e = tid; e < PT * wk1; e += LF_THREADS) {
      const int pl = e / wk1, q = e - (e / wk1) * wk1;
      const double* zrow = &Z[pl * a][q];
      double* hrow = &H[pl * a][q];
      const double z = zrow[0] + bias[q];
      const double t = tanh(z), s = 1.0 - t * t;
      hrow[0] = t;
      for (int g = 0; g < ngrad; ++g) hrow[(1 + g) * LF_LD] = s * zrow[(1 + g) * LF_LD];
      if (nlap) {
        double G = 0.0;
        for (int l = 0; l < nlap; ++l) {
          const double dz = zrow[s_lap[l] * LF_LD];
          G = fma(dz, dz, G);
        }
        hrow[(nch - 1) * LF_LD] = s * zrow[(nch - 1) * LF_LD] - 2.0 * t * s * G;
      }
    }
  }
  // ---- head (width 1): residual per point, squared, summed over the tile
  const int wL = p.w[p.L - 1];
  const long long oL = p.off[p.L - 1];
  __syncthreads();
  if (tid <= wL) wl[tid] = __ldg(th + oL + tid);  // W_{L-1} (w x 1) and b_{L-1}
  __syncthreads();
  // one warp per (point, channel) dot product: lanes walk q (conflict-free);
  // the Z tile is free by now and holds the 64 channel outputs
  double* s_u = &Z[0][0];
  for (int pc = warp; pc < PT * a; pc += LF_THREADS / 32) {
    const double* hrow = &H[pc][0];
    double u = 0.0;
    for (int q = lane; q < wL; q += 32) u = fma(hrow[q], wl[q], u);
    u = warp_sum(u);
    if (lane == 0) s_u[pc] = u;
  }
  __syncthreads();
  double r2 = 0.0;
  if (tid < PT && P0 + tid < count) {
    double res = 0.0, u0 = 0.0;
    for (int ch = 0; ch < nch; ++ch) {
      double u = s_u[tid * a + ch];
      if (ch == 0) {
        u += wl[wL];
        u0 = u;
      }
      res = fma(s_coef[ch], u, res);
    }
    if (c3 != 0.0) res = fma(c3 * u0 * u0, u0, res);
    const double r = C.weight * (res - C.f[P0 + tid]);
    r2 = r * r;
  }
  r2 = warp_sum(r2);
  if (lane == 0) s_red[warp] = r2;
  __syncthreads();
  if (tid == 0) {
    double sacc = 0.0;
    for (int w = 0; w < LF_THREADS / 32; ++w) sacc += s_red[w];
    p.part[static_cast<long long>(cand) * p.ntiles + tile] = sacc;
  }
}

__global__ void __launch_bounds__(256) k_loss_reduce(const double* __restrict__ part, int ntiles,
                                                       double* __restrict__ losses) {
  __shared__ double sh[8];
  double s = 0.0;
  for (int t = threadIdx.x; t < ntiles; t += 256) s += part[static_cast<long long>(blockIdx.x) * ntiles + t];
  s = block_sum<256>(s, sh);
  if (threadIdx.x == 0) losses[blockIdx.x] = 0.5 * s;
}

// J^T w for every layer in one launch: out[W_k|b_k][p][q] =
//   sum_rho w(point rho) Hext_k[rho][p] Zbar_k[rho][q]
// (Hext_k = [H_k, bias (channel 0)], H_0 = the materialised input channels,
// Zbar_{L-1} = the residual-operator seeds).  Grid (tile, split): each CTA owns
// a 64 x 64 block of one layer's (w_k + 1) x w_{k+1} output and a contiguous
// range of activation rows, stages 32 rows at a time in shared memory and
// accumulates on the FP64 tensor cores (A fragment = Hext^T, read transposed
// from the row-major stage).  Per-split partials are reduced in fixed order by
// k_jt_reduce, so the result is bitwise reproducible.
constexpr int JT_BM = 64, JT_BK = 32, JT_LD = 68;

struct JtLayer {
  const double* H;  // Hext without the bias column
  long long ldh;
  int wh;
  const double* Z;  // nullptr: output-layer seeds (wz == 1)
  long long ldz;
  int wz;
  long long off;  // theta offset of W_k
  int tq, tile0;  // tiles along q; first tile of the layer
};

struct JtParams {
  Classes T;
  int L;
  JtLayer lay[DNGD_MAX_LAYERS];
  const double* w;
  long long rows_per_split;
  long long n;
  double* part;  // [split][n]
};

__global__ void __launch_bounds__(128) k_jt_tiles(const __grid_constant__ JtParams p) {
  __shared__ double Hs[JT_BK][JT_LD], Zs[JT_BK][JT_LD];
  __shared__ double wv[JT_BK], sd[JT_BK];
  __shared__ int chs[JT_BK];
  const int tile = blockIdx.x, split = blockIdx.y;
  int k = 0;
  while (k + 1 < p.L && tile >= p.lay[k + 1].tile0) ++k;
  const JtLayer& Lk = p.lay[k];
  const int t = tile - Lk.tile0;
  const int tpi = t / Lk.tq, tqi = t - (t / Lk.tq) * Lk.tq;
  const int p0 = tpi * JT_BM, q0 = tqi * JT_BM;
  const long long r0 = split * p.rows_per_split;
  const long long r1 = min(p.T.R, r0 + p.rows_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 1, wn = warp & 1;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  const bool seeds = Lk.Z == nullptr;
  // w_k a multiple of 64: no row tile holds the bias row; the first row tile sums
  // it (sum of the value-channel rows of w Zbar) alongside the tensor-core tile
  const bool xbias = (Lk.wh % JT_BM) == 0 && tpi == 0;
  double bsum = 0.0;
  for (long long rb = r0; rb < r1; rb += JT_BK) {
    if (threadIdx.x < JT_BK) {
      const long long rho = rb + threadIdx.x;
      double wr = 0.0, sv = 0.0;
      int ch = 1;
      if (rho < r1) {
        const long long i = act_point(p.T, rho, ch);
        const ClassDev& C = p.T.c[find_class(p.T, i)];
        wr = p.w[i];
        sv = seeds ? seedc(p.T, C, ch, i) : 0.0;
      }
      wv[threadIdx.x] = wr;
      sd[threadIdx.x] = sv;
      chs[threadIdx.x] = ch;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < JT_BK * JT_BM; e += 128) {
      const int r = e / JT_BM, c = e - (e / JT_BM) * JT_BM;
      const long long rho = rb + r;
      const bool ok = rho < r1;
      const int pc = p0 + c, qc = q0 + c;
      double h = 0.0, z = 0.0;
      if (ok) {
        if (pc < Lk.wh) {
          h = Lk.H[rho * Lk.ldh + pc];
        } else if (pc == Lk.wh) {
          h = chs[r] == 0 ? 1.0 : 0.0;
        }
        if (qc < Lk.wz) z = wv[r] * (seeds ? sd[r] : Lk.Z[rho * Lk.ldz + qc]);
      }
      Hs[r][c] = h;
      Zs[r][c] = z;
    }
    __syncthreads();
    if (xbias && threadIdx.x < JT_BM) {
      for (int r = 0; r < JT_BK; ++r)
        if (chs[r] == 0) bsum += Zs[r][threadIdx.x];
    }
#pragma unroll
    for (int kk = 0; kk < JT_BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Hs[kk + (lane & 3)][wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Zs[kk + (lane & 3)][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  double* dst = p.part + split * p.n + Lk.off;
  if (xbias && threadIdx.x < JT_BM && q0 + static_cast<int>(threadIdx.x) < Lk.wz)
    dst[static_cast<long long>(Lk.wh) * Lk.wz + q0 + threadIdx.x] = bsum;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pr = p0 + wm * 32 + i * 8 + (lane >> 2);
    if (pr > Lk.wh) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int qc = q0 + wn * 32 + j * 8 + 2 * (lane & 3);
      if (qc < Lk.wz) dst[static_cast<long long>(pr) * Lk.wz + qc] = acc[i][j].x;
      if (qc + 1 < Lk.wz) dst[static_cast<long long>(pr) * Lk.wz + qc + 1] = acc[i][j].y;
    }
  }
}

__global__ void k_jt_reduce(const double* __restrict__ part, int splits, long long n, double scale,
                            double* __restrict__ out) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = 0.0;
  int k = 0;
  // 8 loads in flight, added in the same (split) order as one at a time
  for (; k + 8 <= splits; k += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = part[static_cast<long long>(k + j) * n + e];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; k < splits; ++k) s += part[static_cast<long long>(k) * n + e];
  out[e] = scale * s;
}

// k_jt_reduce over the columns [c0, c0 + len) only, into out[0 .. len)
__global__ void k_jt_reduce_range(const double* __restrict__ part, int splits, long long n,
                                  long long c0, long long len, double scale,
                                  double* __restrict__ out) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= len) return;
  const long long e = c0 + q;
  double s = 0.0;
  int k = 0;
  // 8 loads in flight, added in the same (split) order as one at a time
  for (; k + 8 <= splits; k += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = part[static_cast<long long>(k + j) * n + e];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; k < splits; ++k) s += part[static_cast<long long>(k) * n + e];
  out[q] = scale * s;
}

static size_t bytes_of(const Plan& P, int mode, int C) {
  Arena A{nullptr};
  if (mode == 0) {
    AsmBufs b;
    carve_assemble(P, A, b);
  } else if (mode == 1) {
    FvvBufs b;
    carve_fvv(P, A, b);
  } else {
    LossBufs b;
    carve_loss(P, A, b, C);
  }
  return A.off;
}

}  // namespace dngd

using namespace dngd;

extern "C" int dngd_pinn_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp,
                                   const dngd_class_desc* classes, int nclass, int ncand,
                                   size_t* bytes) {
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  size_t b = std::max(bytes_of(P, 0, 1), bytes_of(P, 1, 1));
  b = std::max(b, bytes_of(P, 2, std::max(ncand, 1)));
  *bytes = b;
  return DNGD_OK;
}

static int assemble_impl(dngd_ctx* ctx, cudaStream_t s, const Plan& P, AsmBufs& B,
                         const double* theta, long long col_begin, long long col_end, double* r,
                         double* J, long long ldJ, bool adjoint) {
  int rc = DNGD_OK;
  const int L = P.L;
  // ---- forward
  if (P.bigin) {
    rc = input_gemm(ctx, s, P, B.big, theta, B.big.Zx);
    if (rc) return rc;
  }
  k_input_fwd<<<nblk(P.m * P.w[1]), 256, 0, s>>>(P.T, theta, 0, static_cast<int>(P.w[1]),
                                                  P.ld[1], B.Z[0], B.H[1], 0, B.big.Zx, nullptr,
                                                  nullptr, P.ld[1], nullptr, nullptr);
  transpose_hidden(s, P, theta, B.Wt);
  for (int k = 1; k <= L - 2; ++k) {
    GemmCall g;
    g.M = P.R;
    g.N = P.w[k + 1];
    g.K = P.w[k];
    g.A = B.H[k];
    g.lda = P.ld[k];
    g.B = B.Wt[k];
    g.ldb = P.ld[k];
    g.C = B.Z[k];
    g.ldc = P.ld[k + 1];
    rc = gemm_nt_hidden(ctx, s, g, B.oz);
    if (rc) return rc;
    k_tanh_fwd<<<nblk(P.m * P.w[k + 1]), 256, 0, s>>>(P.T, B.Z[k], B.H[k + 1],
                                                      static_cast<int>(P.w[k + 1]), P.ld[k + 1],
                                                      theta + P.off[k] + P.w[k] * P.w[k + 1], 0,
                                                      0);
  }
  const long long wl_off = P.off[L - 1];
  k_head<<<nblk(P.m, 8), 256, 0, s>>>(P.T, B.H[L - 1], static_cast<int>(P.w[L - 1]),
                                       P.ld[L - 1], theta, 0, wl_off, 0, r, 0);
  rc = cuda_status(ctx, cudaGetLastError(), "assemble forward");
  if (rc || (J == nullptr && !adjoint)) return rc;
  if (J != nullptr && (col_begin < 0 || col_end > P.n || col_begin > col_end)) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "assemble: column range outside [0, n]");
  }
  const bool jvec_ok = ((ldJ & 1) == 0) && ((reinterpret_cast<uintptr_t>(J) & 15) == 0);
  bool identity_inputs = true;
  for (int c = 0; c < P.T.n; ++c)
    if (P.T.c[c].inp) identity_inputs = false;
  int max_nch = 1;
  for (int c = 0; c < P.T.n; ++c) max_nch = std::max(max_nch, P.T.c[c].nch);
  auto jw_staged_bytes = [&](const auto&, int win, int wout) -> size_t {
    return static_cast<size_t>(((max_nch * (win + 1) + 1) & ~1) + max_nch * wout) * sizeof(double);
  };
  auto jwrite = [&](int k, const double* Hk, long long ldh, const double* Zb, long long ldz) {
    if (J == nullptr) return;
    const int win = static_cast<int>(P.w[k]), wout = static_cast<int>(P.w[k + 1]);
    const long long lo = P.off[k], hi = lo + (win + 1LL) * wout;
    if (hi <= col_begin || lo >= col_end) return;
    const long long E = (win + 1LL) * wout;
    const bool vec = Zb != nullptr && jvec_ok && (wout % 2 == 0) && ((lo - col_begin) % 2 == 0);
    if (vec && k == 0 && identity_inputs) {
      const unsigned gx = static_cast<unsigned>(std::min<long long>((E / 2 + 255) / 256, 64));
      k_jwrite_in<<<dim3(gx, static_cast<unsigned>(P.m)), 256, 0, s>>>(
          P.T, Zb, ldz, wout, col_begin, col_end, J, ldJ);
    } else if (vec && Hk != nullptr && jw_staged_bytes(P, win, wout) <= 200 * 1024) {
      // (config 3: 7 channels x 512 units = 57 KB staged per row, above the 48 KB default)
      static std::atomic<bool> attr[64];  // per device (idempotent, race-free)
      if (!attr[ctx->device & 63]) {
        cudaFuncSetAttribute(k_jwrite_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr[ctx->device & 63] = true;
      }
      k_jwrite_staged<<<static_cast<unsigned>(P.m), 256, jw_staged_bytes(P, win, wout), s>>>(
          P.T, Hk, ldh, win, Zb, ldz, wout, lo, col_begin, col_end, J, ldJ);
    } else if (vec && E < (1LL << 31)) {
      // ~8 column pairs per thread: one tiny CTA per 512 elements made the
      // launch of ~10^4 CTAs, not the stores, the cost
      const unsigned gx = static_cast<unsigned>(std::min<long long>((E + 4095) / 4096, 64));
      k_jwrite<true><<<dim3(gx, static_cast<unsigned>(P.m)), 256, 0, s>>>(
          P.T, Hk, ldh, win, Zb, ldz, wout, lo, col_begin, col_end, J, ldJ);
    } else {
      const unsigned gx = static_cast<unsigned>(std::min<long long>((E + 255) / 256, 64));
      k_jwrite<false><<<dim3(gx, static_cast<unsigned>(P.m)), 256, 0, s>>>(
          P.T, Hk, ldh, win, Zb, ldz, wout, lo, col_begin, col_end, J, ldJ);
    }
  };
  // ---- adjoint, last layer first
  jwrite(L - 1, B.H[L - 1], P.ld[L - 1], nullptr, 0);
  k_seed_hbar<<<nblk(P.m * P.w[L - 1]), 256, 0, s>>>(P.T, B.Hb, static_cast<int>(P.w[L - 1]),
                                                      P.ld[L - 1], theta + wl_off);
  for (int k = L - 2; k >= 0; --k) {
    // Hb holds the adjoint of H_{k+1} (ld = ld[k+1]); produce Zb_k
    k_tanh_bwd<<<nblk(P.m * P.w[k + 1]), 256, 0, s>>>(P.T, B.Z[k], B.H[k + 1], B.Hb, B.Zb[k],
                                                      static_cast<int>(P.w[k + 1]), P.ld[k + 1]);
    jwrite(k, k >= 1 ? B.H[k] : nullptr, k >= 1 ? P.ld[k] : 0, B.Zb[k], P.ld[k + 1]);
    if (k >= 1) {
      k_copy2d<<<nblk(P.w[k] * P.w[k + 1]), 256, 0, s>>>(theta + P.off[k], static_cast<int>(P.w[k]),
                                                         static_cast<int>(P.w[k + 1]), B.Wp[k],
                                                         P.ld[k + 1]);
      GemmCall g;
      g.M = P.R;
      g.N = P.w[k];
      g.K = P.w[k + 1];
      g.A = B.Zb[k];
      g.lda = P.ld[k + 1];
      g.B = B.Wp[k];
      g.ldb = P.ld[k + 1];
      g.C = B.Hb;
      g.ldc = P.ld[k];
      rc = gemm_nt_hidden(ctx, s, g, B.oz);
      if (rc) return rc;
    }
  }
  if (P.T.din <= DNGD_MAX_GRAD) {
    // Hext_0 for the J-free kernels: an assembly that also wrote J leaves a
    // complete activation workspace too (the factored Gram / J^T w may reuse it)
    k_input_channels<<<nblk(P.R * GF_H0_LD), 256, 0, s>>>(P.T, B.H0);
  }
  return cuda_status(ctx, cudaGetLastError(), "assemble adjoint");
}

extern "C" int dngd_assemble(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                             const double* theta, const dngd_class_desc* classes, int nclass,
                             int64_t col_begin, int64_t col_end, double* r, double* J,
                             int64_t ldJ, void* work, size_t work_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > work_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "assemble: workspace too small");
  if (P.m == 0) return DNGD_OK;
  Arena A{static_cast<char*>(work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  return assemble_impl(ctx, s, P, B, theta, col_begin, col_end, r, J, ldJ, false);
}

extern "C" int dngd_activations(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                const double* theta, const dngd_class_desc* classes, int nclass,
                                double* r, void* work, size_t work_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > work_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "activations: workspace too small");
  if (P.m == 0) return DNGD_OK;
  Arena A{static_cast<char*>(work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  return assemble_impl(ctx, s, P, B, theta, 0, P.n, r, nullptr, 0, true);
}

// 2-D maps (columns, packed channel rows) over one class's rows of H_k / Zbar_k:
// N points x nch channels, row pitch ld; a box of 16 x 64 is one G-space operand
// tile (rows past the class end arrive as zeros)
static int gf_encode2(dngd_ctx* ctx, CUtensorMap* map, const double* base, long long inner,
                      int nch, long long N, long long ld) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner),
                        static_cast<cuuint64_t>(std::max<long long>(N * nch, 1))};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2] = {16, static_cast<cuuint32_t>(GF_BM)};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = ctx->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base),
                             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? DNGD_OK
                             : set_error(ctx, DNGD_ERR_CUDA, "gram_factored: tensor map encode failed");
}

// channels per point, whole points per tile, layer K-dims and the row-side
// tensor maps of the factored Gram
static int gram_setup(dngd_ctx* ctx, const Plan& P, const AsmBufs& B, GramParams& gp) {
  int rc = DNGD_OK;
  memset(&gp, 0, sizeof gp);
  gp.T = P.T;
  gp.L = P.L;
  for (int c = 0; c < P.T.n; ++c) {
    const int nch = P.T.c[c].nch;
    if (nch > GF_MAXCH) {
      return set_error(ctx, DNGD_ERR_UNSUPPORTED,
                       "gram_factored: more than 16 channels per point; use assemble + syrk");
    }
    gp.nch[c] = nch;
    gp.ppt[c] = GF_BM / nch;
  }
  for (int k = 0; k < P.L; ++k) {
    gp.lay[k].kh = static_cast<int>(P.w[k]);
    gp.lay[k].kz = k <= P.L - 2 ? static_cast<int>(P.w[k + 1]) : 0;
    for (int c = 0; c < P.T.n; ++c) {
      const ClassDev& Cc = P.T.c[c];
      if (k >= 1) {
        rc = gf_encode2(ctx, &gp.maps[k][0][c], B.H[k] + Cc.act0 * P.ld[k], P.w[k], Cc.nch,
                        Cc.count, P.ld[k]);
      } else {
        rc = gf_encode2(ctx, &gp.maps[0][0][c], B.H0 + Cc.act0 * GF_H0_LD, P.T.din, Cc.nch,
                        Cc.count, GF_H0_LD);
      }
      if (rc) return rc;
      if (k <= P.L - 2) {
        rc = gf_encode2(ctx, &gp.maps[k][1][c], B.Zb[k] + Cc.act0 * P.ld[k + 1], P.w[k + 1],
                        Cc.nch, Cc.count, P.ld[k + 1]);
        if (rc) return rc;
      }
    }
  }
  return DNGD_OK;
}

// K = J J^T without J's input block (wide identity input layer): the hidden and
// output columns are materialised and SYRKed, the input block is added by
// k_gram_input from X X^T and Zbar_0.
static int gram_wide_input(dngd_ctx* ctx, cudaStream_t s, const Plan& P, AsmBufs& B,
                           const double* theta, double* r, double* K, long long ldK) {
  int rc = assemble_impl(ctx, s, P, B, theta, P.off[1], P.n, r, B.Jh, P.wi_ldh, true);
  if (rc) return rc;
  rc = syrk(ctx, s, B.Jh, P.m, P.wi_ncols, P.wi_ldh, K, ldK, 0, B.syrk_work, P.wi_syrk_bytes);
  if (rc) return rc;
  if (P.bigin) {
    for (int c = 0; c < P.T.n; ++c) {
      for (int cp = 0; cp <= c; ++cp) {
        const ClassDev &C = P.T.c[c], &D = P.T.c[cp];
        if (C.count == 0 || D.count == 0) continue;
        GemmCall g;
        g.M = C.count;
        g.N = D.count;
        g.K = P.T.din;
        g.A = C.pts;
        g.lda = P.T.din;
        g.B = D.pts;
        g.ldb = P.T.din;
        g.C = B.XX + C.row0 * P.wi_ldxx + D.row0;
        g.ldc = P.wi_ldxx;
        rc = gemm_nt_splitk(ctx, s, g, P.wi_xx_splits, B.xx_part, P.wi_xx_part);
        if (rc) return rc;
      }
    }
  } else {
    k_xx_dot<<<static_cast<unsigned>(P.m), 256, 0, s>>>(P.T, B.XX, P.wi_ldxx);
  }
  k_gram_input<<<dim3(static_cast<unsigned>(P.m), static_cast<unsigned>((P.m + 7) / 8)), 256, 0,
                 s>>>(P.T, B.Zb[0], P.ld[1],
                                                          static_cast<int>(P.w[1]), B.XX,
                                                          P.wi_ldxx, K, ldK);
  return cuda_status(ctx, cudaGetLastError(), "gram_wide_input");
}

static int gram_from_act(dngd_ctx* ctx, cudaStream_t s, const Plan& P, const AsmBufs& B, double* K,
                         long long ldK, int part, int nparts);

extern "C" int dngd_gram_factored(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                  const double* theta, const dngd_class_desc* classes,
                                  int nclass, double* r, double* K, int64_t ldK, void* work,
                                  size_t work_bytes) {
  return dngd_gram_factored_part(ctx, stream, mlp, theta, classes, nclass, r, K, ldK, 0, 1, work,
                                 work_bytes);
}

extern "C" int dngd_gram_factored_part(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                       const double* theta, const dngd_class_desc* classes,
                                       int nclass, double* r, double* K, int64_t ldK, int part,
                                       int nparts, void* work, size_t work_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nparts < 1 || part < 0 || part >= nparts) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gram_factored: part outside [0, nparts)");
  }
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > work_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_factored: workspace too small");
  if (P.m == 0) return DNGD_OK;
  if (P.wide_in) {
    if (nparts != 1) {
      return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_factored: wide input layer is not tile-sharded");
    }
    Arena A{static_cast<char*>(work)};
    AsmBufs B;
    carve_assemble(P, A, B);
    P.T.u0 = B.u0;
    return gram_wide_input(ctx, s, P, B, theta, r, K, ldK);
  }
  if (P.T.din > DNGD_MAX_GRAD) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_factored: input dim > 12");
  Arena A{static_cast<char*>(work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  rc = assemble_impl(ctx, s, P, B, theta, 0, P.n, r, nullptr, 0, true);
  if (rc) return rc;
  return gram_from_act(ctx, s, P, B, K, ldK, part, nparts);
}

// the factored Gram kernel over activations already in the workspace (left there
// by dngd_activations / dngd_gram_factored at the same theta)
static int gram_from_act(dngd_ctx* ctx, cudaStream_t s, const Plan& P, const AsmBufs& B, double* K,
                         long long ldK, int part, int nparts) {
  thread_local GramParams gp;  // ~17 KB of tensor maps: off the host stack, reentrant
  int rc = gram_setup(ctx, P, B, gp);
  if (rc) return rc;
  int np = 0, tiles = 0;
  gp.tstart[0] = 0;
  for (int c = 0; c < P.T.n; ++c) {
    for (int cp = 0; cp <= c; ++cp) {
      const int ti = static_cast<int>((P.T.c[c].count + gp.ppt[c] - 1) / gp.ppt[c]);
      const int tj = static_cast<int>((P.T.c[cp].count + gp.ppt[cp] - 1) / gp.ppt[cp]);
      gp.pc[np] = c;
      gp.pcp[np] = cp;
      gp.tj_n[np] = tj;
      tiles += c == cp ? ti * (ti + 1) / 2 : ti * tj;
      gp.tstart[np + 1] = tiles;
      ++np;
    }
  }
  gp.npairs = np;
  gp.K = K;
  gp.ldK = ldK;
  cudaError_t e = cudaFuncSetAttribute(k_gram_factored, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(gram_factored_smem()));
  if (e != cudaSuccess) return cuda_status(ctx, e, "gram_factored smem attribute");
  static_assert(GF_H0_LD == 16, "carve_assemble reserves R x 16 for H0");
  // tile-sharded Gram: part p of nparts computes the contiguous tile range
  // [p T / nparts, (p+1) T / nparts) (every 64x64 G-tile costs the same)
  const long long t0 = static_cast<long long>(tiles) * part / nparts;
  const long long t1 = static_cast<long long>(tiles) * (part + 1) / nparts;
  gp.tile0 = static_cast<int>(t0);
  if (t1 > t0) {
    k_gram_factored<<<static_cast<unsigned>(t1 - t0), GF_THREADS, gram_factored_smem(), s>>>(gp);
  }
  return cuda_status(ctx, cudaGetLastError(), "gram_factored");
}

extern "C" int dngd_gram_factored_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                      const dngd_class_desc* classes, int nclass, double* K,
                                      int64_t ldK, int part, int nparts, void* act_work,
                                      size_t act_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nparts < 1 || part < 0 || part >= nparts) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gram_factored_act: part outside [0, nparts)");
  }
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > act_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_factored_act: workspace too small");
  if (P.m == 0) return DNGD_OK;
  if (P.wide_in) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_factored_act: wide input layer");
  if (P.T.din > DNGD_MAX_GRAD) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_factored_act: input dim > 12");
  Arena A{static_cast<char*>(act_work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  return gram_from_act(ctx, s, P, B, K, ldK, part, nparts);
}

// ------------------------------------------------------------------ emulated-FP64 Gram
// dngd_gram_oz_act: the factored Gram over the activations in act_work with every
// G-space GEMM on the int8 tensor cores (gram_oz.cuh).  oz_work holds, per layer
// and part (H_k, Zbar_k), the R x kpad x S digit planes and R row scales.

static size_t oz_al256(size_t b) { return (b + 255) / 256 * 256; }

static long long goz_kdim(const Plan& P, int k, int part) {
  if (part == 0) return k == 0 ? P.T.din : P.w[k];
  return k <= P.L - 2 ? P.w[k + 1] : 0;
}

static size_t gram_oz_bytes(const Plan& P, int S) {
  size_t b = 0;
  for (int k = 0; k < P.L; ++k)
    for (int part = 0; part < 2; ++part) {
      const long long kd = goz_kdim(P, k, part);
      if (kd == 0) continue;
      b += oz_al256(static_cast<size_t>(S) * P.R * oz_kpad(kd)) + oz_al256(static_cast<size_t>(P.R) * 8);
    }
  return b;
}

static int goz_check(dngd_ctx* ctx, const Plan& P, int slices) {
  if (slices != 6 && slices != 7) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_oz: 6 or 7 digit slices");
  if (P.wide_in) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_oz: wide input layer");
  if (P.T.din > DNGD_MAX_GRAD) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_oz: input dim > 12");
  if (P.R >= (1LL << 31)) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_oz: too many activation rows");
  for (int k = 0; k < P.L; ++k)
    if (goz_kdim(P, k, 0) > kOzMaxK || goz_kdim(P, k, 1) > kOzMaxK)
      return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_oz: layer wider than 16384");
  for (int c = 0; c < P.T.n; ++c)
    if (P.T.c[c].nch > OZ_BN) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_oz: more than 64 channels per point");
  return DNGD_OK;
}

extern "C" int dngd_gram_oz_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp,
                                      const dngd_class_desc* classes, int nclass, int slices,
                                      size_t* bytes) {
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  rc = goz_check(ctx, P, slices);
  if (rc) return rc;
  *bytes = gram_oz_bytes(P, slices);
  return DNGD_OK;
}

extern "C" int dngd_gram_oz_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                const dngd_class_desc* classes, int nclass, double* K,
                                int64_t ldK, int part, int nparts, int slices, void* act_work,
                                size_t act_bytes, void* oz_work, size_t oz_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (nparts < 1 || part < 0 || part >= nparts) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "gram_oz: part outside [0, nparts)");
  }
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > act_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_oz: activation workspace too small");
  if (P.m == 0) return DNGD_OK;
  rc = goz_check(ctx, P, slices);
  if (rc) return rc;
  if (gram_oz_bytes(P, slices) > oz_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_oz: workspace too small");
  Arena A{static_cast<char*>(act_work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  thread_local GozParams gp;
  memset(&gp, 0, sizeof gp);
  gp.T = P.T;
  gp.L = P.L;
  gp.R = P.R;
  char* w = static_cast<char*>(oz_work);
  for (int k = 0; k < P.L; ++k) {
    for (int pt = 0; pt < 2; ++pt) {
      const long long kd = goz_kdim(P, k, pt);
      gp.nk[k][pt] = static_cast<int>(oz_kpad(kd) / 32);
      if (kd == 0) continue;
      const double* src;
      long long ld;
      if (pt == 0) {
        src = k == 0 ? B.H0 : B.H[k];
        ld = k == 0 ? GF_H0_LD : P.ld[k];
      } else {
        src = B.Zb[k];
        ld = P.ld[k + 1];
      }
      int8_t* Q = reinterpret_cast<int8_t*>(w);
      w += oz_al256(static_cast<size_t>(slices) * P.R * oz_kpad(kd));
      double* sc = reinterpret_cast<double*>(w);
      w += oz_al256(static_cast<size_t>(P.R) * 8);
      rc = oz_slice(ctx, s, src, P.R, kd, ld, slices, Q, sc);
      if (rc) return rc;
      rc = oz_encode(ctx, &gp.mA[k][pt], Q, P.R, oz_kpad(kd), slices, OZ_BM, 64);
      if (rc) return rc;
      rc = oz_encode(ctx, &gp.mB[k][pt], Q, P.R, oz_kpad(kd), slices, OZ_BN);
      if (rc) return rc;
      gp.sc[k][pt] = sc;
    }
  }
  int np = 0, tiles = 0;
  gp.tstart[0] = 0;
  for (int c = 0; c < P.T.n; ++c) {
    gp.nch[c] = P.T.c[c].nch;
    gp.ppc[c] = OZ_BN / P.T.c[c].nch;
  }
  for (int c = 0; c < P.T.n; ++c) {
    for (int cp = 0; cp <= c; ++cp) {
      const int TI = static_cast<int>((P.T.c[c].count + 2 * gp.ppc[c] - 1) / (2 * gp.ppc[c]));
      const int TJ = static_cast<int>((P.T.c[cp].count + gp.ppc[cp] - 1) / gp.ppc[cp]);
      gp.pc[np] = c;
      gp.pcp[np] = cp;
      gp.ti_n[np] = TI;
      gp.tj_n[np] = TJ;
      tiles += c == cp ? TI * (TI + 1) : TI * TJ;
      gp.tstart[np + 1] = tiles;
      ++np;
    }
  }
  gp.npairs = np;
  gp.K = K;
  gp.ldK = ldK;
  const long long t0 = static_cast<long long>(tiles) * part / nparts;
  const long long t1 = static_cast<long long>(tiles) * (part + 1) / nparts;
  gp.tile0 = static_cast<int>(t0);
  gp.dbg = getenv("DNGD_GOZ_DBG") ? atoi(getenv("DNGD_GOZ_DBG")) : 0;
  if (t1 <= t0) return DNGD_OK;
  const size_t smem = gram_oz_smem(slices);
  auto kern = slices == 7 ? k_gram_oz<7> : k_gram_oz<6>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_status(ctx, e, "gram_oz smem attribute");
  const int ntiles = static_cast<int>(t1 - t0);
  kern<<<static_cast<unsigned>(std::min(ntiles, ctx->num_sms)), OZ_THREADS, smem, s>>>(gp, ntiles);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    return set_error(ctx, DNGD_ERR_CUDA,
                     std::string("gram_oz: ") + cudaGetErrorString(e) + " (regs " +
                         std::to_string(fa.numRegs) + ", max threads " +
                         std::to_string(fa.maxThreadsPerBlock) + ", static smem " +
                         std::to_string(fa.sharedSizeBytes) + ", dynamic " + std::to_string(smem) + ")");
  }
  return DNGD_OK;
}

// ------------------------------------------------------------------ K[:, I] without J
// Nystrom sketch columns (solver.py:259-261 K[:, I] = J J_I^T): the activations of
// the landmark points are gathered into compact per-class buffers and the factored
// Gram kernel runs rectangular tiles (all points) x (landmarks).

__global__ void k_gather_rows(const double* __restrict__ src, long long ld,
                              const long long* __restrict__ idx, long long nrows,
                              double* __restrict__ dst) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nrows * ld) return;
  const long long r = e / ld, c = e - (e / ld) * ld;
  dst[e] = src[idx[r] * ld + c];
}

struct ColsPlan {
  long long lc[MAXC], lrow0[MAXC];  // landmarks per class; first gathered activation row
  long long rows;                   // gathered activation rows
  std::vector<long long> src;       // source activation row of every gathered row
};

static int cols_plan(dngd_ctx* ctx, const Plan& P, const int64_t* landmarks, int ell, ColsPlan& Q) {
  Q.rows = 0;
  Q.src.clear();
  int pos = 0;
  for (int c = 0; c < P.T.n; ++c) {
    const ClassDev& C = P.T.c[c];
    Q.lc[c] = 0;
    Q.lrow0[c] = Q.rows;
    while (pos < ell && landmarks[pos] < C.row0 + C.count) {
      const long long p = landmarks[pos];
      if (p < C.row0 || (pos > 0 && p <= landmarks[pos - 1])) {
        return set_error(ctx, DNGD_ERR_DIMENSION, "gram_cols: landmarks must be sorted and distinct");
      }
      for (int ch = 0; ch < C.nch; ++ch) Q.src.push_back(C.act0 + (p - C.row0) * C.nch + ch);
      Q.rows += C.nch;
      ++Q.lc[c];
      ++pos;
    }
  }
  if (pos != ell) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_cols: landmark outside [0, m)");
  return DNGD_OK;
}

static size_t cols_scratch_bytes(const Plan& P, long long rows) {
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  size_t b = al(static_cast<size_t>(rows) * 8) + al(static_cast<size_t>(rows) * GF_H0_LD * 8);
  for (int k = 1; k <= P.L - 1; ++k) b += al(static_cast<size_t>(rows) * P.ld[k] * 8);
  for (int k = 0; k <= P.L - 2; ++k) b += al(static_cast<size_t>(rows) * P.ld[k + 1] * 8);
  return b;
}

// K[:, I] on the int8 engine (gram_oz.cuh rect mode) under the same rule as the
// factored Gram (kernels.gram_emulation_slices: hidden layers >= 64 wide,
// DNGD_GRAM_SLICES=0 keeps the DMMA kernel); 0 where the emulated kernel does not apply
static bool goz_cols_slices_ok(const Plan& P) {
  long long hmax = 0;
  for (int k = 1; k < P.L; ++k) hmax = std::max(hmax, P.w[k]);
  if (hmax < 64 || P.wide_in || P.T.din > DNGD_MAX_GRAD || P.R >= (1LL << 31)) return 0;
  for (int k = 0; k < P.L; ++k)
    if (goz_kdim(P, k, 0) > kOzMaxK || goz_kdim(P, k, 1) > kOzMaxK) return 0;
  for (int c = 0; c < P.T.n; ++c)
    if (P.T.c[c].nch > OZ_BN) return false;
  return true;
}
static int goz_cols_slices(const Plan& P) {
  if (const char* e = getenv("DNGD_GRAM_SLICES")) {
    if (atoi(e) == 0) return 0;
    if (atoi(e) == 7) return goz_cols_slices_ok(P) ? 7 : 0;
  }
  return goz_cols_slices_ok(P) ? 6 : 0;
}

// digit planes of the full activations (R rows) and of the gathered landmark rows
static size_t cols_oz_bytes(const Plan& P, long long rows, int S) {
  size_t b = gram_oz_bytes(P, S);
  for (int k = 0; k < P.L; ++k)
    for (int part = 0; part < 2; ++part) {
      const long long kd = goz_kdim(P, k, part);
      if (kd == 0) continue;
      b += oz_al256(static_cast<size_t>(S) * rows * oz_kpad(kd)) + oz_al256(static_cast<size_t>(rows) * 8);
    }
  return b + oz_al256(static_cast<size_t>(rows) * 8);  // + the landmarks' global points
}

extern "C" int dngd_gram_cols_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp,
                                        const dngd_class_desc* classes, int nclass, int ell,
                                        size_t* bytes) {
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  const long long rows = static_cast<long long>(std::max(ell, 1)) * 8;
  *bytes = cols_scratch_bytes(P, rows);
  if (const int S = goz_cols_slices(P)) *bytes = (*bytes + 255) / 256 * 256 + cols_oz_bytes(P, rows, S);
  return DNGD_OK;
}

extern "C" int dngd_gram_factored_cols(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                       const dngd_class_desc* classes, int nclass,
                                       const int64_t* landmarks, int ell, double* Kc,
                                       int64_t ldKc, void* act_work, size_t act_bytes,
                                       void* scratch, size_t scratch_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > act_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_cols: activation workspace too small");
  if (P.m == 0 || ell <= 0) return DNGD_OK;
  if (P.T.din > DNGD_MAX_GRAD) return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_cols: input dim > 12");
  for (int c = 0; c < P.T.n; ++c) {
    if (P.T.c[c].c3 != 0.0) {
      return set_error(ctx, DNGD_ERR_UNSUPPORTED, "gram_cols: cubic residual terms need the materialised path");
    }
  }
  ColsPlan Q;
  rc = cols_plan(ctx, P, landmarks, ell, Q);
  if (rc) return rc;
  if (cols_scratch_bytes(P, Q.rows) > scratch_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "gram_cols: scratch too small");
  Arena A{static_cast<char*>(act_work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  thread_local GramParams gp;
  rc = gram_setup(ctx, P, B, gp);
  if (rc) return rc;
  // gathered buffers: [idx][H0][H_1..H_{L-1}][Zb_0..Zb_{L-2}]
  Arena S{static_cast<char*>(scratch)};
  long long* idx = reinterpret_cast<long long*>(S.take(Q.rows));
  cudaError_t e = cudaMemcpyAsync(idx, Q.src.data(), Q.rows * sizeof(long long),
                                  cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(ctx, e, "gram_cols index upload");
  auto gather = [&](const double* src, long long ld) {
    double* dst = S.take(static_cast<size_t>(Q.rows) * ld);
    k_gather_rows<<<nblk(Q.rows * ld), 256, 0, s>>>(src, ld, idx, Q.rows, dst);
    return dst;
  };
  double* gH0 = gather(B.H0, GF_H0_LD);
  std::vector<double*> gH(P.L, nullptr), gZ(P.L, nullptr);
  for (int k = 1; k <= P.L - 1; ++k) gH[k] = gather(B.H[k], P.ld[k]);
  for (int k = 0; k <= P.L - 2; ++k) gZ[k] = gather(B.Zb[k], P.ld[k + 1]);
  if (const int S = goz_cols_slices(P)) {
    // emulated FP64: the full activations give the row tiles, the gathered landmark
    // activations the column tiles (gram_oz.cuh rect mode)
    const long long rows_cap = static_cast<long long>(std::max(ell, 1)) * 8;
    char* w = static_cast<char*>(scratch) + (cols_scratch_bytes(P, rows_cap) + 255) / 256 * 256;
    if (scratch_bytes < static_cast<size_t>(w - static_cast<char*>(scratch)) + cols_oz_bytes(P, rows_cap, S)) {
      return set_error(ctx, DNGD_ERR_DIMENSION, "gram_cols: scratch too small for the int8 planes");
    }
    thread_local GozParams gq;
    memset(&gq, 0, sizeof gq);
    gq.T = P.T;
    gq.L = P.L;
    gq.R = P.R;
    gq.Rb = Q.rows;
    gq.rect = 1;
    for (int k = 0; k < P.L; ++k) {
      for (int pt = 0; pt < 2; ++pt) {
        const long long kd = goz_kdim(P, k, pt);
        gq.nk[k][pt] = static_cast<int>(oz_kpad(kd) / 32);
        if (kd == 0) continue;
        const double *src, *gsrc;
        long long ld;
        if (pt == 0) {
          src = k == 0 ? B.H0 : B.H[k];
          gsrc = k == 0 ? gH0 : gH[k];
          ld = k == 0 ? GF_H0_LD : P.ld[k];
        } else {
          src = B.Zb[k];
          gsrc = gZ[k];
          ld = P.ld[k + 1];
        }
        int8_t* Qa = reinterpret_cast<int8_t*>(w);
        w += oz_al256(static_cast<size_t>(S) * P.R * oz_kpad(kd));
        double* sa = reinterpret_cast<double*>(w);
        w += oz_al256(static_cast<size_t>(P.R) * 8);
        int8_t* Qb = reinterpret_cast<int8_t*>(w);
        w += oz_al256(static_cast<size_t>(S) * rows_cap * oz_kpad(kd));
        double* sb = reinterpret_cast<double*>(w);
        w += oz_al256(static_cast<size_t>(rows_cap) * 8);
        rc = oz_slice(ctx, s, src, P.R, kd, ld, S, Qa, sa);
        if (rc == DNGD_OK) rc = oz_slice(ctx, s, gsrc, Q.rows, kd, ld, S, Qb, sb);
        if (rc == DNGD_OK) rc = oz_encode(ctx, &gq.mA[k][pt], Qa, P.R, oz_kpad(kd), S, OZ_BM, 64);
        if (rc == DNGD_OK) rc = oz_encode(ctx, &gq.mB[k][pt], Qb, Q.rows, oz_kpad(kd), S, OZ_BN);
        if (rc) return rc;
        gq.sc[k][pt] = sa;
        gq.scB[k][pt] = sb;
      }
    }
    // global point index of every landmark (column order = class order)
    std::vector<long long> lpt(static_cast<size_t>(ell));
    for (int j = 0; j < ell; ++j) lpt[j] = landmarks[j];
    long long* lpt_dev = reinterpret_cast<long long*>(w);
    e = cudaMemcpyAsync(lpt_dev, lpt.data(), static_cast<size_t>(ell) * sizeof(long long),
                        cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(ctx, e, "gram_cols landmark upload");
    gq.lpt = lpt_dev;
    long long lc0 = 0;
    for (int c = 0; c < P.T.n; ++c) {
      gq.nch[c] = P.T.c[c].nch;
      gq.ppc[c] = OZ_BN / P.T.c[c].nch;
      gq.lcol0[c] = lc0;
      gq.lcnt[c] = Q.lc[c];
      gq.lrow0[c] = Q.lrow0[c];
      lc0 += Q.lc[c];
    }
    int npairs = 0, ntile = 0;
    gq.tstart[0] = 0;
    for (int c = 0; c < P.T.n; ++c) {
      for (int cp = 0; cp < P.T.n; ++cp) {
        if (Q.lc[cp] == 0 || P.T.c[c].count == 0) continue;
        const int TI = static_cast<int>((P.T.c[c].count + 2 * gq.ppc[c] - 1) / (2 * gq.ppc[c]));
        const int TJ = static_cast<int>((Q.lc[cp] + gq.ppc[cp] - 1) / gq.ppc[cp]);
        gq.pc[npairs] = c;
        gq.pcp[npairs] = cp;
        gq.ti_n[npairs] = TI;
        gq.tj_n[npairs] = TJ;
        ntile += TI * TJ;
        gq.tstart[npairs + 1] = ntile;
        ++npairs;
      }
    }
    gq.npairs = npairs;
    gq.K = Kc;
    gq.ldK = ldKc;
    gq.tile0 = 0;
    if (ntile == 0) return DNGD_OK;
    const size_t smem = gram_oz_smem(S);
    auto kern = S == 7 ? k_gram_oz<7> : k_gram_oz<6>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return cuda_status(ctx, e, "gram_cols oz smem attribute");
    kern<<<static_cast<unsigned>(std::min(ntile, ctx->num_sms)), OZ_THREADS, smem, s>>>(gq, ntile);
    return cuda_status(ctx, cudaGetLastError(), "gram_cols oz");
  }
  long long col0 = 0;
  for (int c = 0; c < P.T.n; ++c) {
    const ClassDev& Cc = P.T.c[c];
    gp.ccount[c] = Q.lc[c];
    gp.ccol0[c] = col0;
    col0 += Q.lc[c];
    for (int k = 0; k < P.L; ++k) {
      if (k >= 1) {
        rc = gf_encode2(ctx, &gp.cmaps[k][0][c], gH[k] + Q.lrow0[c] * P.ld[k], P.w[k], Cc.nch,
                        Q.lc[c], P.ld[k]);
      } else {
        rc = gf_encode2(ctx, &gp.cmaps[0][0][c], gH0 + Q.lrow0[c] * GF_H0_LD, P.T.din, Cc.nch,
                        Q.lc[c], GF_H0_LD);
      }
      if (rc) return rc;
      if (k <= P.L - 2) {
        rc = gf_encode2(ctx, &gp.cmaps[k][1][c], gZ[k] + Q.lrow0[c] * P.ld[k + 1], P.w[k + 1],
                        Cc.nch, Q.lc[c], P.ld[k + 1]);
        if (rc) return rc;
      }
    }
  }
  int np = 0, tiles = 0;
  gp.tstart[0] = 0;
  for (int c = 0; c < P.T.n; ++c) {
    for (int cp = 0; cp < P.T.n; ++cp) {
      if (Q.lc[cp] == 0) continue;
      const int ti = static_cast<int>((P.T.c[c].count + gp.ppt[c] - 1) / gp.ppt[c]);
      const int tj = static_cast<int>((Q.lc[cp] + gp.ppt[cp] - 1) / gp.ppt[cp]);
      gp.pc[np] = c;
      gp.pcp[np] = cp;
      gp.tj_n[np] = tj;
      tiles += ti * tj;
      gp.tstart[np + 1] = tiles;
      ++np;
    }
  }
  gp.npairs = np;
  gp.rect = 1;
  gp.K = Kc;
  gp.ldK = ldKc;
  gp.tile0 = 0;
  e = cudaFuncSetAttribute(k_gram_factored, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(gram_factored_smem()));
  if (e != cudaSuccess) return cuda_status(ctx, e, "gram_cols smem attribute");
  if (tiles > 0) {
    k_gram_factored<<<static_cast<unsigned>(tiles), GF_THREADS, gram_factored_smem(), s>>>(gp);
  }
  return cuda_status(ctx, cudaGetLastError(), "gram_cols");
}

static int fvv_impl(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
                    const double* v, const dngd_class_desc* classes, int nclass, double* fvv,
                    void* work, size_t work_bytes, int order, const double* zx_act = nullptr);

// x W0(theta) left in an activation workspace by the last assembly / Gram at theta
// (large-din input layer only; nullptr otherwise)
static const double* act_input_products(const Plan& P, void* act_work, size_t act_bytes) {
  if (!P.bigin || act_work == nullptr || bytes_of(P, 0, 1) > act_bytes) return nullptr;
  Arena A{static_cast<char*>(act_work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  return B.big.Zx;
}

extern "C" int dngd_fvv_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                            const double* theta, const double* v, const dngd_class_desc* classes,
                            int nclass, double* fvv, void* work, size_t work_bytes,
                            void* act_work, size_t act_bytes) {
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  return fvv_impl(ctx, stream, mlp, theta, v, classes, nclass, fvv, work, work_bytes, 2,
                  act_input_products(P, act_work, act_bytes));
}

extern "C" int dngd_fvv(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                        const double* theta, const double* v, const dngd_class_desc* classes,
                        int nclass, double* fvv, void* work, size_t work_bytes) {
  return fvv_impl(ctx, stream, mlp, theta, v, classes, nclass, fvv, work, work_bytes, 2);
}

extern "C" int dngd_jvp_factored(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                 const double* theta, const double* v,
                                 const dngd_class_desc* classes, int nclass, double* out,
                                 void* work, size_t work_bytes) {
  return fvv_impl(ctx, stream, mlp, theta, v, classes, nclass, out, work, work_bytes, 1);
}

// forward t-jets of the channel map along theta + t v: order 2 -> f_vv, order 1 -> J v
// (first-order jets only: the GEMMs cover 2R and R rows instead of 3R and 2R)
static int fvv_impl(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp, const double* theta,
                    const double* v, const dngd_class_desc* classes, int nclass, double* fvv,
                    void* work, size_t work_bytes, int order, const double* zx_act) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 1, 1) > work_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "fvv: workspace too small");
  if (P.m == 0) return DNGD_OK;
  Arena A{static_cast<char*>(work)};
  FvvBufs B;
  carve_fvv(P, A, B);
  const int L = P.L;
  const long long ld = P.ldmax;
  double* Hcur = B.H3[0];
  double* Hnext = B.H3[1];
  const double* zx = B.big.Zx;
  if (P.bigin) {
    if (zx_act != nullptr) {
      zx = zx_act;  // x W0(theta) from the activation pass at theta
    } else {
      rc = input_gemm(ctx, s, P, B.big, theta, B.big.Zx);
      if (rc) return rc;
    }
    rc = input_gemm(ctx, s, P, B.big, v, B.big.Dx);
    if (rc) return rc;
  }
  if (order == 1) {
    k_fvv_input<1><<<nblk(P.m * P.w[1]), 256, 0, s>>>(P.T, theta, v, static_cast<int>(P.w[1]), ld,
                                                     Hcur, zx, B.big.Dx, P.ld[1]);
  } else {
    k_fvv_input<2><<<nblk(P.m * P.w[1]), 256, 0, s>>>(P.T, theta, v, static_cast<int>(P.w[1]), ld,
                                                     Hcur, zx, B.big.Dx, P.ld[1]);
  }
  transpose_hidden(s, P, theta, B.Wt);
  transpose_hidden(s, P, v, B.Vt);
  for (int k = 1; k <= L - 2; ++k) {
    GemmCall g;
    g.M = (order == 1 ? 2 : 3) * P.R;
    g.N = P.w[k + 1];
    g.K = P.w[k];
    g.A = Hcur;
    g.lda = ld;
    g.B = B.Wt[k];
    g.ldb = P.ld[k];
    g.C = B.P3;
    g.ldc = ld;
    rc = gemm_nt_hidden(ctx, s, g, B.oz);
    if (rc) return rc;
    g.M = (order == 1 ? 1 : 2) * P.R;
    g.B = B.Vt[k];
    g.C = B.Q2;
    rc = gemm_nt_hidden(ctx, s, g, B.oz);
    if (rc) return rc;
    const long long boff = P.off[k] + P.w[k] * P.w[k + 1];
    if (order == 1) {
      k_fvv_hidden<1><<<nblk(P.m * P.w[k + 1]), 256, 0, s>>>(P.T, B.P3, B.Q2, theta + boff, v + boff,
                                                             static_cast<int>(P.w[k + 1]), ld, Hnext);
    } else {
      k_fvv_hidden<2><<<nblk(P.m * P.w[k + 1]), 256, 0, s>>>(P.T, B.P3, B.Q2, theta + boff, v + boff,
                                                             static_cast<int>(P.w[k + 1]), ld, Hnext);
    }
    std::swap(Hcur, Hnext);
  }
  k_fvv_head<<<nblk(P.m, 8), 256, 0, s>>>(P.T, Hcur, static_cast<int>(P.w[L - 1]), ld,
                                           theta + P.off[L - 1], v + P.off[L - 1], fvv, order);
  return cuda_status(ctx, cudaGetLastError(), order == 1 ? "jvp_factored" : "fvv");
}

// the fused line search handles nets whose every layer width is <= 64 and whose
// classes have <= 8 channels per point (one 64-row tile holds whole points)
static bool loss_fused_ok(const Plan& P) {
  for (int k = 1; k < P.L; ++k)
    if (P.w[k] > 64) return false;
  for (int c = 0; c < P.T.n; ++c)
    if (P.T.c[c].nch > 8 || P.T.c[c].pgi || P.T.c[c].pco) return false;
  return P.T.din <= MAXG;
}

static int loss_many_impl(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                          const double* theta, const double* delta, const double* etas, int ncand,
                          const dngd_class_desc* classes, int nclass, double* losses, void* work,
                          size_t work_bytes, void* act_work, size_t act_bytes);

extern "C" int dngd_loss_many(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                              const double* theta, const double* delta, const double* etas,
                              int ncand, const dngd_class_desc* classes, int nclass,
                              double* losses, void* work, size_t work_bytes) {
  return loss_many_impl(ctx, stream, mlp, theta, delta, etas, ncand, classes, nclass, losses, work,
                        work_bytes, nullptr, 0);
}

extern "C" int dngd_loss_many_act(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                  const double* theta, const double* delta, const double* etas,
                                  int ncand, const dngd_class_desc* classes, int nclass,
                                  double* losses, void* work, size_t work_bytes, void* act_work,
                                  size_t act_bytes) {
  return loss_many_impl(ctx, stream, mlp, theta, delta, etas, ncand, classes, nclass, losses, work,
                        work_bytes, act_work, act_bytes);
}

static int loss_many_impl(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                          const double* theta, const double* delta, const double* etas, int ncand,
                          const dngd_class_desc* classes, int nclass, double* losses, void* work,
                          size_t work_bytes, void* act_work, size_t act_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (ncand < 1) return DNGD_OK;
  if (ncand > 65535) return set_error(ctx, DNGD_ERR_DIMENSION, "loss_many: too many candidates");
  if (bytes_of(P, 2, ncand) > work_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "loss_many: workspace too small");
  if (loss_fused_ok(P)) {
    thread_local LossFusedParams lp;
    lp.T = P.T;
    lp.L = P.L;
    for (int k = 0; k <= P.L; ++k) lp.w[k] = static_cast<int>(P.w[k]);
    for (int k = 0; k < P.L; ++k) lp.off[k] = P.off[k];
    lp.n = P.n;
    int tiles = 0;
    for (int c = 0; c < P.T.n; ++c) {
      int lg = 0;
      while ((1 << lg) < P.T.c[c].nch) ++lg;
      lp.lg[c] = lg;
      lp.tile0[c] = tiles;
      tiles += static_cast<int>((P.T.c[c].count + (64 >> lg) - 1) / (64 >> lg));
    }
    lp.tile0[P.T.n] = tiles;
    lp.ntiles = tiles;
    lp.part = static_cast<double*>(work);
    double* thetas = lp.part + ((static_cast<size_t>(ncand) * tiles + 31) / 32) * 32;
    lp.thetas = thetas;
    k_candidates<<<dim3(nblk(P.n), ncand), 256, 0, s>>>(theta, delta, etas, P.n, thetas);
    static std::atomic<bool> attr[64];  // per device (idempotent, race-free)
    if (!attr[ctx->device & 63]) {
      cudaError_t e = cudaFuncSetAttribute(k_loss_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kLossFusedSmem));
      if (e != cudaSuccess) return cuda_status(ctx, e, "loss_fused smem attribute");
      attr[ctx->device & 63] = true;
    }
    if (tiles > 0) {
      k_loss_fused<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(ncand)), LF_THREADS,
                     kLossFusedSmem, s>>>(lp);
    }
    k_loss_reduce<<<ncand, 256, 0, s>>>(lp.part, tiles, losses);
    return cuda_status(ctx, cudaGetLastError(), "loss_many fused");
  }
  Arena A{static_cast<char*>(work)};
  LossBufs B;
  carve_loss(P, A, B, ncand);
  const long long k0 = (P.bigin && delta != nullptr) ? P.T.din * P.w[1] : 0;
  k_candidates<<<dim3(nblk(P.n - k0), ncand), 256, 0, s>>>(theta, delta, etas, P.n, B.thetas, k0);
  double* Hlast;
  rc = forward_batched(ctx, s, P, B.thetas, ncand, B, &Hlast, theta, delta, etas,
                       act_input_products(P, act_work, act_bytes), B.r);
  if (rc) return rc;
  if (Hlast != nullptr) {  // (else the last hidden layer wrote the residuals: k_tanh_head)
    k_head<<<dim3(nblk(P.m, 8), ncand), 256, 0, s>>>(P.T, Hlast, static_cast<int>(P.w[P.L - 1]),
                                                      P.ldmax, B.thetas, P.n, P.off[P.L - 1],
                                                      P.R * P.ldmax, B.r, P.m);
  }
  k_half_sumsq<<<ncand, 256, 0, s>>>(B.r, P.m, losses);
  return cuda_status(ctx, cudaGetLastError(), "loss_many");
}

namespace {

struct JtScratch {
  long long ldm = 0;                   // wide input on the tensor cores: Xt / Bt pitch
  size_t off_xt = 0, off_bt = 0;
  long long ldR, chunk;
  int nchunks, splits;
  size_t bytes, off_zt, off_part, part_bytes;
  bool tiled;  // one k_jt_tiles launch (narrow nets)
  int tiles, tsplits;
  long long rows_per_split;
  size_t off_tmp = 0;  // column-range mode: the input / output layer block before slicing
  int oz = 0;           // hidden-layer GEMMs on the int8 engine (Ozaki digits; 0 = DMMA)
  size_t off_oz = 0, oz_bytes = 0;
};

// narrow nets: every layer in one tiled launch; wide ones: per-layer split-K GEMM
static constexpr long long kJtTiledMaxWidth = 128;

// row tiles of layer k's (w_k + 1) x w_{k+1} block in k_jt_tiles: when w_k is a
// multiple of 64 the bias row is summed by the first row tile on the side
// instead of costing a whole extra 64-row tile
static int jt_row_tiles(long long wk) {
  return static_cast<int>(wk % JT_BM == 0 ? wk / JT_BM : (wk + 1 + JT_BM - 1) / JT_BM);
}

JtScratch jt_plan(dngd_ctx* ctx, const Plan& P) {
  JtScratch S;
  S.tiled = P.wmax <= kJtTiledMaxWidth && P.w[0] <= MAXG;
  if (S.tiled) {
    S.tiles = 0;
    for (int k = 0; k < P.L; ++k)
      S.tiles += jt_row_tiles(P.w[k]) * static_cast<int>((P.w[k + 1] + JT_BM - 1) / JT_BM);
    const int target = 2 * 2 * ctx->num_sms;  // two waves of two CTAs per SM
    long long sp = std::max(1, (target + S.tiles - 1) / S.tiles);
    sp = std::min(sp, std::max(1LL, P.R / 64));
    S.rows_per_split = (P.R + sp - 1) / sp;
    S.rows_per_split = (S.rows_per_split + JT_BK - 1) / JT_BK * JT_BK;
    S.tsplits = static_cast<int>(std::max(1LL, (P.R + S.rows_per_split - 1) / S.rows_per_split));
    S.part_bytes = static_cast<size_t>(S.tsplits) * P.n * 8;
    S.bytes = S.part_bytes;
    S.ldR = S.chunk = 0;
    S.nchunks = S.splits = 0;
    S.off_zt = S.off_part = 0;
    return S;
  }
  S.ldR = (P.R + 15) / 16 * 16;
  S.nchunks = static_cast<int>(std::max(1LL, std::min<long long>(256, P.m / 8)));
  S.chunk = (P.m + S.nchunks - 1) / S.nchunks;
  S.splits = 1;
  size_t part = 0;
  for (int k = 1; k <= P.L - 2; ++k) {
    const int sp = gemm_splitk_choose(ctx, P.w[k] + 1, P.w[k + 1], P.R);
    S.splits = std::max(S.splits, sp);
    part = std::max(part, gemm_splitk_bytes(P.w[k] + 1, P.w[k + 1], sp));
  }
  if (!P.wide_in) {  // (the wide input layer writes out directly)
    part = std::max(part, static_cast<size_t>(S.nchunks) * static_cast<size_t>((P.w[0] + 1) * P.w[1]) * 8);
  }
  part = std::max(part, static_cast<size_t>(S.nchunks) * static_cast<size_t>(P.w[P.L - 1] + 1) * 8);
  const size_t ht = static_cast<size_t>(P.wmax + 1) * S.ldR * 8;
  S.off_zt = (ht + 255) / 256 * 256;
  S.off_part = S.off_zt + (static_cast<size_t>(P.wmax) * S.ldR * 8 + 255) / 256 * 256;
  S.part_bytes = part;
  S.bytes = S.off_part + part;
  if (P.wide_in && P.bigin) {
    S.ldm = (P.m + 1) / 2 * 2;
    S.off_xt = (S.bytes + 255) / 256 * 256;
    S.off_bt = S.off_xt + (static_cast<size_t>(P.w[0] + 1) * S.ldm * 8 + 255) / 256 * 256;
    S.bytes = S.off_bt + static_cast<size_t>(P.w[1]) * S.ldm * 8;
  }
  S.off_tmp = (S.bytes + 255) / 256 * 256;  // column-range mode: the small edge layers
  S.bytes = S.off_tmp + static_cast<size_t>(std::max((P.w[0] + 1) * P.w[1], P.w[P.L - 1] + 1)) * 8;
  // hidden layers >= 128 wide: split-K over activation rows on the int8 tensor cores
  S.oz = oz_ls_slices(P);
  if (S.oz) {
    for (int k = 1; k <= P.L - 2; ++k) {
      const int sp = oz_splitk_choose(ctx, P.w[k] + 1, P.w[k + 1], P.R);
      S.oz_bytes = std::max(S.oz_bytes, oz_splitk_bytes(P.w[k] + 1, P.w[k + 1], P.R, S.oz, sp));
    }
    S.off_oz = (S.bytes + 255) / 256 * 256;
    S.bytes = S.off_oz + S.oz_bytes;
  }
  return S;
}

}  // namespace

extern "C" int dngd_jt_workspace(dngd_ctx* ctx, const dngd_mlp_desc* mlp,
                                 const dngd_class_desc* classes, int nclass, size_t* bytes) {
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  *bytes = jt_plan(ctx, P).bytes;
  return DNGD_OK;
}

// out[j - c0] = scale (J^T w)[j] for j in [c0, c1) (the full vector: [0, n)).  In
// a partial range every boundary inside a hidden layer block must fall on a row of
// that block (a multiple of w_{k+1} from the block start): those GEMMs then run
// only the owned rows (M = a1 - a0, the column-sharded multi-GPU step); the small
// input / output blocks are formed whole and sliced.
static int jt_range(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                    const dngd_class_desc* classes, int nclass, const double* w, double scale,
                    double* out, long long c0, long long c1, void* act_work, size_t act_bytes,
                    void* scratch, size_t scratch_bytes) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  if (bytes_of(P, 0, 1) > act_bytes) return set_error(ctx, DNGD_ERR_DIMENSION, "jt_factored: activation workspace too small");
  const JtScratch S = jt_plan(ctx, P);
  if (scratch == nullptr || scratch_bytes < S.bytes) {
    return set_error(ctx, DNGD_ERR_DIMENSION, "jt_factored: scratch workspace too small");
  }
  if (c0 < 0 || c1 > P.n || c0 > c1) return set_error(ctx, DNGD_ERR_DIMENSION, "jt_factored: column range outside [0, n)");
  const bool full = c0 == 0 && c1 == P.n;
  if (P.m == 0 || c0 == c1) return DNGD_OK;
  if (!full) {  // partial ranges: hidden-layer boundaries on block rows
    for (int k = 1; k <= P.L - 2; ++k) {
      const long long lo = P.off[k], hi = P.off[k] + (P.w[k] + 1) * P.w[k + 1];
      for (long long b : {c0, c1}) {
        if (b > lo && b < hi && (b - lo) % P.w[k + 1] != 0) {
          return set_error(ctx, DNGD_ERR_DIMENSION, "jt_factored: range boundary inside a hidden-layer row");
        }
      }
    }
  }
  char* const sc0 = static_cast<char*>(scratch);
  double* const tmp = reinterpret_cast<double*>(sc0 + S.off_tmp);
  // a small block [lo, lo + len) formed whole at dst (tmp unless the range covers it)
  auto edge_dst = [&](long long lo, long long len) -> double* {
    return (lo >= c0 && lo + len <= c1) ? out + (lo - c0) : tmp;
  };
  auto edge_copy = [&](double* dst, long long lo, long long len) -> int {
    if (dst != tmp) return DNGD_OK;
    const long long a = std::max(lo, c0), b = std::min(lo + len, c1);
    if (b <= a) return DNGD_OK;
    cudaError_t e = cudaMemcpyAsync(out + (a - c0), tmp + (a - lo), (b - a) * 8,
                                    cudaMemcpyDeviceToDevice, s);
    return e == cudaSuccess ? DNGD_OK : cuda_status(ctx, e, "jt_factored slice");
  };
  if (P.T.din > MAXG && !P.wide_in) {
    return set_error(ctx, DNGD_ERR_UNSUPPORTED, "jt_factored: embedded inputs wider than 12");
  }
  Arena A{static_cast<char*>(act_work)};
  AsmBufs B;
  carve_assemble(P, A, B);
  P.T.u0 = B.u0;
  if (S.tiled) {
    thread_local JtParams jp;
    jp.T = P.T;
    jp.L = P.L;
    int tile0 = 0;
    for (int k = 0; k < P.L; ++k) {
      JtLayer& l = jp.lay[k];
      l.H = k == 0 ? B.H0 : B.H[k];
      l.ldh = k == 0 ? GF_H0_LD : P.ld[k];
      l.wh = static_cast<int>(P.w[k]);
      l.Z = k <= P.L - 2 ? B.Zb[k] : nullptr;
      l.ldz = k <= P.L - 2 ? P.ld[k + 1] : 0;
      l.wz = static_cast<int>(P.w[k + 1]);
      l.off = P.off[k];
      l.tq = static_cast<int>((P.w[k + 1] + JT_BM - 1) / JT_BM);
      l.tile0 = tile0;
      tile0 += jt_row_tiles(P.w[k]) * l.tq;
    }
    jp.w = w;
    jp.rows_per_split = S.rows_per_split;
    jp.n = P.n;
    jp.part = static_cast<double*>(scratch);
    k_jt_tiles<<<dim3(static_cast<unsigned>(S.tiles), static_cast<unsigned>(S.tsplits)), 128, 0, s>>>(jp);
    if (full) {
      k_jt_reduce<<<nblk(P.n), 256, 0, s>>>(jp.part, S.tsplits, P.n, scale, out);
    } else {  // narrow nets: the whole vector is cheap; reduce only the range
      k_jt_reduce_range<<<nblk(c1 - c0), 256, 0, s>>>(jp.part, S.tsplits, P.n, c0, c1 - c0, scale, out);
    }
    return cuda_status(ctx, cudaGetLastError(), "jt_factored");
  }
  char* sc = static_cast<char*>(scratch);
  double* Ht = reinterpret_cast<double*>(sc);
  double* Zt = reinterpret_cast<double*>(sc + S.off_zt);
  double* part = reinterpret_cast<double*>(sc + S.off_part);
  const int L = P.L;
  // input layer W0 | b0
  const long long len0 = (P.w[0] + 1) * P.w[1];
  const bool in0 = P.off[0] < c1 && P.off[0] + len0 > c0;
  double* const d0 = edge_dst(P.off[0], len0);
  if (!in0) {
  } else if (P.wide_in && P.bigin) {
    const int w1 = static_cast<int>(P.w[1]);
    const int din = P.T.din;
    double* Xt = reinterpret_cast<double*>(sc + S.off_xt);
    double* Bt = reinterpret_cast<double*>(sc + S.off_bt);
    k_xt_build<<<dim3(static_cast<unsigned>((S.ldm + 31) / 32), static_cast<unsigned>((din + 1 + 31) / 32)),
                 dim3(32, 8), 0, s>>>(P.T, Xt, S.ldm);
    k_bt_build<<<nblk(w1 * S.ldm), 256, 0, s>>>(P.T, B.Zb[0], P.ld[1], w1, w, Bt, S.ldm);
    GemmCall g;
    g.M = din + 1;
    g.N = w1;
    g.K = P.m;
    g.A = Xt;
    g.lda = S.ldm;
    g.B = Bt;
    g.ldb = S.ldm;
    g.C = d0;
    g.ldc = w1;
    g.alpha = scale;
    g.beta = 0.0;
    rc = gemm_nt(ctx, s, g);
    if (rc) return rc;
    k_jt_onehot<<<static_cast<unsigned>((din + OH_ROWS - 1) / OH_ROWS), 128, 0, s>>>(
        P.T, B.Zb[0], P.ld[1], w1, w, scale, d0);
  } else if (P.wide_in) {
    const int w1 = static_cast<int>(P.w[1]);
    dim3 g(static_cast<unsigned>((P.w[0] + 1 + JW_J - 1) / JW_J), (w1 + 127) / 128);
    static std::atomic<bool> attr[64];  // per device (idempotent, race-free)
    if (!attr[ctx->device & 63]) {
      cudaError_t e = cudaFuncSetAttribute(k_jt_input_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kJwSmem));
      if (e != cudaSuccess) return cuda_status(ctx, e, "jt_input_wide smem attribute");
      attr[ctx->device & 63] = true;
    }
    k_jt_input_wide<<<g, 256, kJwSmem, s>>>(P.T, B.Zb[0], P.ld[1], w1, w, scale, d0);
  } else {
    const int w1 = static_cast<int>(P.w[1]);
    dim3 g((w1 + 127) / 128, S.nchunks);
    k_jt_input<<<g, 128, 0, s>>>(P.T, B.Zb[0], P.ld[1], w1, w, S.chunk, part);
    const long long cnt = (P.w[0] + 1) * P.w[1];
    k_chunk_reduce<<<nblk(cnt), 256, 0, s>>>(part, S.nchunks, cnt, scale, d0);
  }
  if (in0) {
    rc = edge_copy(d0, P.off[0], len0);
    if (rc) return rc;
  }
  // hidden layers: Hext_k^T diag(w) Zbar_k on the tensor cores
  for (int k = 1; k <= L - 2; ++k) {
    const int wk = static_cast<int>(P.w[k]), wk1 = static_cast<int>(P.w[k + 1]);
    const long long lo = P.off[k], hi = P.off[k] + static_cast<long long>(wk + 1) * wk1;
    if (hi <= c0 || lo >= c1) continue;
    const long long a0 = (std::max(lo, c0) - lo) / wk1, a1 = (std::min(hi, c1) - lo) / wk1;
    dim3 tg(static_cast<unsigned>((P.R + 31) / 32), static_cast<unsigned>((wk + 1 + 31) / 32));
    k_act_transpose<<<tg, dim3(32, 8), 0, s>>>(P.T, B.H[k], P.ld[k], wk, nullptr, 1, Ht, S.ldR);
    dim3 zg(static_cast<unsigned>((P.R + 31) / 32), static_cast<unsigned>((wk1 + 31) / 32));
    k_act_transpose<<<zg, dim3(32, 8), 0, s>>>(P.T, B.Zb[k], P.ld[k + 1], wk1, w, 0, Zt, S.ldR);
    GemmCall g;
    g.M = a1 - a0;
    g.N = wk1;
    g.K = P.R;
    g.A = Ht + a0 * S.ldR;
    g.lda = S.ldR;
    g.B = Zt;
    g.ldb = S.ldR;
    g.C = out + (lo + a0 * wk1 - c0);
    g.ldc = wk1;
    g.alpha = scale;
    g.beta = 0.0;
    if (S.oz) {
      const int sp0 = oz_splitk_choose(ctx, g.M, g.N, g.K);
      const int spmin = static_cast<int>((g.K + (kOzMaxK - 32) - 1) / (kOzMaxK - 32));
      int sp = sp0;
      while (sp > spmin && oz_splitk_bytes(g.M, g.N, g.K, S.oz, sp) > S.oz_bytes) --sp;
      rc = oz_gemm_splitk(ctx, s, g.A, g.lda, g.B, g.ldb, g.M, g.N, g.K, g.alpha, g.C, g.ldc, S.oz,
                          sp, sc0 + S.off_oz, S.oz_bytes);
      if (rc) return rc;
      continue;
    }
    int sp = gemm_splitk_choose(ctx, g.M, g.N, g.K);
    while (sp > 1 && gemm_splitk_bytes(g.M, g.N, sp) > S.part_bytes) --sp;
    rc = gemm_nt_splitk(ctx, s, g, sp, part, S.part_bytes);
    if (rc) return rc;
  }
  // output layer W_{L-1} | b_{L-1}
  if (P.off[L - 1] < c1 && P.off[L - 1] + P.w[L - 1] + 1 > c0) {
    const int wl = static_cast<int>(P.w[L - 1]);
    double* dl = edge_dst(P.off[L - 1], wl + 1);
    dim3 g((wl + 1 + 127) / 128, S.nchunks);
    k_jt_output<<<g, 128, 0, s>>>(P.T, B.H[L - 1], P.ld[L - 1], wl, w, S.chunk, part);
    k_chunk_reduce<<<nblk(wl + 1), 256, 0, s>>>(part, S.nchunks, wl + 1, scale, dl);
    rc = edge_copy(dl, P.off[L - 1], wl + 1);
    if (rc) return rc;
  }
  return cuda_status(ctx, cudaGetLastError(), "jt_factored");
}

extern "C" int dngd_jt_factored(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                const dngd_class_desc* classes, int nclass, const double* w,
                                double scale, double* out, void* act_work, size_t act_bytes,
                                void* scratch, size_t scratch_bytes) {
  Plan P;
  int rc = make_plan(ctx, mlp, classes, nclass, P);
  if (rc) return rc;
  return jt_range(ctx, stream, mlp, classes, nclass, w, scale, out, 0, P.n, act_work, act_bytes,
                  scratch, scratch_bytes);
}

extern "C" int dngd_jt_factored_range(dngd_ctx* ctx, void* stream, const dngd_mlp_desc* mlp,
                                      const dngd_class_desc* classes, int nclass, const double* w,
                                      double scale, double* out, int64_t col_begin,
                                      int64_t col_end, void* act_work, size_t act_bytes,
                                      void* scratch, size_t scratch_bytes) {
  return jt_range(ctx, stream, mlp, classes, nclass, w, scale, out, col_begin, col_end, act_work,
                  act_bytes, scratch, scratch_bytes);
}
