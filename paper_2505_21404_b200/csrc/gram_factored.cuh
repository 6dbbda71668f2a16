// Factored dual Gram K = J J^T straight from the per-point activations.
//
// Row i of J restricted to layer k is a rank-nch outer product
//     J[i, W_k|b_k] = sum_c Hext_k[i,c] (x) Zbar_k[i,c]
// (pinn.cu), hence
//     K_ij = sum_k sum_{c,c'} (Hext_k[i,c] . Hext_k[j,c']) (Zbar_k[i,c] . Zbar_k[j,c'])
//          = sum_k  S (G^H_k o G^Z_k) S^T
// with G^H_k = Hext_k Hext_k^T and G^Z_k = Zbar_k Zbar_k^T over (point, channel)
// rows and S summing the channels of a point.
//
// "G-space": the channel rows of each class are padded to a = 1, 2, 4 or 8 per
// point, so every 8x8 DMMA fragment covers whole point pairs.  The padding is
// free: a 3-D TMA tensor map (columns, channels, points) per (layer, operand,
// class) returns a box of 64/a points x a channels x 16 columns, zero-filling
// the channels >= nch, i.e. exactly 64 G-rows in the 128-byte-swizzled layout
// the DMMA fragment loads of gemm.cu expect.  Per 64x64 G-tile and layer the
// kernel runs two FP64 tensor-core GEMMs (K-dims w_k and w_{k+1}) through one
// TMA/mbarrier ring, multiplies the accumulators elementwise, reduces each
// a x b channel block with warp shuffles and adds the point-pair sums into a
// K tile in shared memory.  Layer 0 (Hext = input channels) is evaluated
// analytically; the output layer's Zbar are the residual-operator seeds.
// Work: sum_k (a_c a_c') (w_k + w_{k+1}) per point pair instead of w_k w_{k+1}
// for J J^T -- ~2x fewer FLOPs at config 2, ~4x at config 3, ~14x at config 4,
// and J (823 GB at config 4) never has to exist.

constexpr int GF_BM = 64;  // G-rows per tile side
constexpr int GF_STAGES = 4;
constexpr int GF_THREADS = 128;  // 2 x 2 warps, 32 x 32 warp tiles
constexpr int GF_STAGE_BYTES = 2 * GF_BM * 128;

struct GramLayer {
  int kh;  // w_k (0 for layer 0: analytic input channels)
  int kz;  // w_{k+1} (0 for the output layer: seeds)
};

struct GramParams {
  CUtensorMap maps[DNGD_MAX_LAYERS][2][DNGD_MAX_CLASSES];  // [layer][H/Z][class]
  Classes T;
  int L;
  GramLayer lay[DNGD_MAX_LAYERS];
  int lg[DNGD_MAX_CLASSES];  // log2(padded channels per point)
  int npairs;
  int pc[10], pcp[10];       // class pair (c >= c')
  int tstart[11];            // tile prefix sums
  int tj_n[10];
  double* K;
  long long ldK;
};

struct ChunkId {
  int k, part, kc, n_h, n_z;  // part 0 = H, 1 = Z
};

DNGD_DEV ChunkId decode_chunk(const GramParams& p, int f) {
  ChunkId id;
  for (int k = 0;; ++k) {
    const int nh = (p.lay[k].kh + 15) >> 4, nz = (p.lay[k].kz + 15) >> 4;
    if (f < nh + nz || k == p.L - 1) {
      id.k = k;
      id.n_h = nh;
      id.n_z = nz;
      id.part = f < nh ? 0 : 1;
      id.kc = f < nh ? f : f - nh;
      return id;
    }
    f -= nh + nz;
  }
}

// analytic Hext_0 . Hext_0' for input channels (value: [x, 1], grad d: [e_d, 0], lap: 0)
DNGD_DEV double gh_input(const ClassDev& C, int ch, const double* xi, const ClassDev& Cp, int chp,
                         const double* xj, int din) {
  if (ch >= C.nch || chp >= Cp.nch) return 0.0;
  const bool lap_i = C.nlap && ch == C.nch - 1;
  const bool lap_j = Cp.nlap && chp == Cp.nch - 1;
  if (lap_i || lap_j) return 0.0;
  if (ch == 0 && chp == 0) {
    double s = 1.0;
    for (int d = 0; d < din; ++d) s = fma(xi[d], xj[d], s);
    return s;
  }
  if (ch == 0) return xi[Cp.grad_dims[chp - 1]];
  if (chp == 0) return xj[C.grad_dims[ch - 1]];
  return C.grad_dims[ch - 1] == Cp.grad_dims[chp - 1] ? 1.0 : 0.0;
}

DNGD_DEV double seed_of(const ClassDev& C, int ch) {
  return ch < C.nch ? C.weight * coef(C, ch) : 0.0;
}

__global__ void __launch_bounds__(GF_THREADS, 2)
    k_gram_factored(const __grid_constant__ GramParams p) {
  extern __shared__ uint8_t gf_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(gf_smem_raw) + 1023) & ~uintptr_t(1023));
  double* Ks = reinterpret_cast<double*>(smem + GF_STAGES * GF_STAGE_BYTES);  // 64 x 64 points max
  double* XA = Ks + GF_BM * GF_BM;
  double* XB = XA + GF_BM * DNGD_MAX_GRAD;
  uint64_t* full = reinterpret_cast<uint64_t*>(XB + GF_BM * DNGD_MAX_GRAD);
  uint64_t* empty = full + GF_STAGES;
  // ---- tile decode
  int pi = 0;
  while (pi + 1 < p.npairs && static_cast<int>(blockIdx.x) >= p.tstart[pi + 1]) ++pi;
  const int t = blockIdx.x - p.tstart[pi];
  const int c = p.pc[pi], cp = p.pcp[pi];
  int ti, tj;
  if (c == cp) {
    decode_lower(t, ti, tj);
  } else {
    ti = t / p.tj_n[pi];
    tj = t - ti * p.tj_n[pi];
  }
  const ClassDev& C = p.T.c[c];
  const ClassDev& Cp = p.T.c[cp];
  const int lga = p.lg[c], lgb = p.lg[cp];
  const int np_r = GF_BM >> lga, np_c = GF_BM >> lgb;
  const int P0 = ti * np_r, Q0 = tj * np_c;  // first point of the tile rows / cols
  const int din = p.T.din;
  int nchunks = 0;
  for (int k = 0; k < p.L; ++k) nchunks += ((p.lay[k].kh + 15) >> 4) + ((p.lay[k].kz + 15) >> 4);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < GF_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], GF_THREADS / 32);
    }
    fence_barrier_init();
  }
  for (int e = threadIdx.x; e < GF_BM * GF_BM; e += GF_THREADS) Ks[e] = 0.0;
  for (int e = threadIdx.x; e < GF_BM * din; e += GF_THREADS) {
    const int r = e / din, d = e - (e / din) * din;
    XA[r * DNGD_MAX_GRAD + d] = (r < np_r && P0 + r < C.count) ? C.pts[static_cast<long long>(P0 + r) * din + d] : 0.0;
    XB[r * DNGD_MAX_GRAD + d] = (r < np_c && Q0 + r < Cp.count) ? Cp.pts[static_cast<long long>(Q0 + r) * din + d] : 0.0;
  }
  __syncthreads();

  auto issue = [&](int f) {
    const ChunkId id = decode_chunk(p, f);
    const int st = f % GF_STAGES;
    uint8_t* sa = smem + st * GF_STAGE_BYTES;
    mbar_arrive_expect_tx(&full[st], GF_STAGE_BYTES);
    tma_load_3d(sa, &p.maps[id.k][id.part][c], &full[st], id.kc * 16, 0, P0);
    tma_load_3d(sa + GF_BM * 128, &p.maps[id.k][id.part][cp], &full[st], id.kc * 16, 0, Q0);
  };
  if (threadIdx.x == 0) {
    for (int f = 0; f < min(nchunks, GF_STAGES); ++f) issue(f);
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 1, wn = warp & 1;
  const int lrow = lane >> 2;
  double2 accH[4][4], accZ[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      accH[i][j] = make_double2(0.0, 0.0);
      accZ[i][j] = make_double2(0.0, 0.0);
    }
  int k_cur = 0, f_layer_end = ((p.lay[0].kh + 15) >> 4) + ((p.lay[0].kz + 15) >> 4);
  for (int f = 0; f < nchunks; ++f) {
    const int st = f % GF_STAGES;
    if (threadIdx.x == 0 && f >= 1 && f - 1 + GF_STAGES < nchunks) {
      const int pf = f - 1;
      mbar_wait(&empty[pf % GF_STAGES], (pf / GF_STAGES) & 1);
      issue(pf + GF_STAGES);
    }
    __syncwarp();
    mbar_wait(&full[st], (f / GF_STAGES) & 1);
    const int nh_cur = (p.lay[k_cur].kh + 15) >> 4;
    const int f_layer_start = f_layer_end - nh_cur - ((p.lay[k_cur].kz + 15) >> 4);
    const bool partH = (f - f_layer_start) < nh_cur;
    const uint8_t* sa = smem + st * GF_STAGE_BYTES + (wm * 32 + lrow) * 128;
    const uint8_t* sb = smem + st * GF_STAGE_BYTES + GF_BM * 128 + (wn * 32 + lrow) * 128;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sw = ((2 * (lane & 3) + h) ^ lrow) << 4;
      double2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = *reinterpret_cast<const double2*>(sa + i * 1024 + sw);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = *reinterpret_cast<const double2*>(sb + j * 1024 + sw);
      // the .x and .y halves go through separate passes so consecutive DMMAs on
      // one accumulator are 16 instructions apart (no back-to-back dependency)
      if (partH) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(accH[i][j], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(accH[i][j], a[i].y, b[j].y);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(accZ[i][j], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_8x8x4(accZ[i][j], a[i].y, b[j].y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (f + 1 != f_layer_end) continue;
    // ---- layer k_cur done: K += S (G_H o G_Z) S^T for this warp's 32x32 G-block
    const bool analyticH = p.lay[k_cur].kh == 0, seedZ = p.lay[k_cur].kz == 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gr = wm * 32 + i * 8 + lrow;  // G-row within the tile
      const int chr = gr & ((1 << lga) - 1);
      const int pr = gr >> lga;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int gc = wn * 32 + j * 8 + 2 * (lane & 3);
        double v0, v1;
        {
          const int chc0 = gc & ((1 << lgb) - 1), chc1 = (gc + 1) & ((1 << lgb) - 1);
          const int pc0 = gc >> lgb, pc1 = (gc + 1) >> lgb;
          double gh0, gh1, gz0, gz1;
          if (analyticH) {
            gh0 = gh_input(C, chr, XA + pr * DNGD_MAX_GRAD, Cp, chc0, XB + pc0 * DNGD_MAX_GRAD, din);
            gh1 = gh_input(C, chr, XA + pr * DNGD_MAX_GRAD, Cp, chc1, XB + pc1 * DNGD_MAX_GRAD, din);
          } else {
            gh0 = accH[i][j].x + ((chr == 0 && chc0 == 0) ? 1.0 : 0.0);
            gh1 = accH[i][j].y + ((chr == 0 && chc1 == 0) ? 1.0 : 0.0);
          }
          if (seedZ) {
            const double sr = seed_of(C, chr);
            gz0 = sr * seed_of(Cp, chc0);
            gz1 = sr * seed_of(Cp, chc1);
          } else {
            gz0 = accZ[i][j].x;
            gz1 = accZ[i][j].y;
          }
          v0 = gh0 * gz0;
          v1 = gh1 * gz1;
        }
        // reduce each a x b channel block: col bits = (h, lane bit 0, lane bit 1),
        // row bits = lane bits 2, 3, 4
        if (lgb >= 1) {
          v0 += v1;
          v1 = 0.0;
        }
        if (lgb >= 2) v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
        if (lgb >= 3) v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
        if (lga >= 1) {
          v0 += __shfl_xor_sync(0xffffffffu, v0, 4);
          if (lgb == 0) v1 += __shfl_xor_sync(0xffffffffu, v1, 4);
        }
        if (lga >= 2) {
          v0 += __shfl_xor_sync(0xffffffffu, v0, 8);
          if (lgb == 0) v1 += __shfl_xor_sync(0xffffffffu, v1, 8);
        }
        if (lga >= 3) {
          v0 += __shfl_xor_sync(0xffffffffu, v0, 16);
          if (lgb == 0) v1 += __shfl_xor_sync(0xffffffffu, v1, 16);
        }
        const bool own_r = (lrow & ((1 << lga) - 1)) == 0;
        const bool own_c = lgb <= 1 || (lane & ((1 << (lgb - 1)) - 1)) == 0;
        if (own_r && own_c) {
          const int pcl0 = gc >> lgb;
          Ks[pr * GF_BM + pcl0] += v0;
          if (lgb == 0) Ks[pr * GF_BM + pcl0 + 1] += v1;
        }
        accH[i][j] = make_double2(0.0, 0.0);
        accZ[i][j] = make_double2(0.0, 0.0);
      }
    }
    if (k_cur + 1 < p.L) {
      ++k_cur;
      f_layer_end += ((p.lay[k_cur].kh + 15) >> 4) + ((p.lay[k_cur].kz + 15) >> 4);
    }
  }
  __syncthreads();
  // ---- epilogue: K[row][col] and its mirror (one writer per entry)
  for (int e = threadIdx.x; e < np_r * np_c; e += GF_THREADS) {
    const int r = e / np_c, cc = e - (e / np_c) * np_c;
    const long long pr = P0 + r, pcl = Q0 + cc;
    if (pr >= C.count || pcl >= Cp.count) continue;
    const long long row = C.row0 + pr, col = Cp.row0 + pcl;
    if (c == cp && col > row) continue;
    const double v = Ks[r * GF_BM + cc];
    p.K[row * p.ldK + col] = v;
    p.K[col * p.ldK + row] = v;
  }
}

static size_t gram_factored_smem() {
  return 1024 + GF_STAGES * GF_STAGE_BYTES + GF_BM * GF_BM * sizeof(double) +
         2 * GF_BM * DNGD_MAX_GRAD * sizeof(double) + 2 * GF_STAGES * sizeof(uint64_t);
}
