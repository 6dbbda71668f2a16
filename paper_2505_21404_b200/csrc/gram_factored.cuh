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
// "G-space": the channel rows of a class are packed, nch per point, exactly as
// the activation buffers store them (row act0 + i nch + ch).  A 64-row operand
// tile holds ppt = floor(64 / nch) whole points (63 useful rows at nch = 7,
// 64 at nch = 1, 2, 4, 8); its last 64 - ppt nch rows belong to the next tile
// and are ignored.  A 2-D TMA map (columns, class rows) per (layer, operand,
// class) returns the box of 64 rows x 16 columns in the 128-byte-swizzled layout
// the DMMA fragment loads of gemm.cu expect.  (Round 1 padded every point to a
// power-of-two channel count: at nch = 7 that multiplied zeros in (8/7)^2 - 1 =
// 31 % of the work.)  Per 64x64 G-tile and layer the kernel runs two FP64
// tensor-core GEMMs (K-dims w_k and w_{k+1}) through one TMA/mbarrier ring and
// adds the elementwise product of the accumulators into a G-space tile in
// shared memory (each thread owns its fragment elements: no races, fixed
// order).  After the last layer every point pair sums its nch_a x nch_b channel
// block in a fixed order (deterministic K) and the tile is written with its
// mirror.
//
// Every layer takes the same epilogue: layer 0's Hext (the input channels:
// value [x], d_j [e_j], Laplacian 0) is materialised once by k_input_channels,
// the bias entry of Hext (1 on the value channel) is a per-row flag product, and
// the output layer's Zbar are the residual-operator seeds, whose outer product
// is a per-row x per-column product.
// Work: sum_k (nch_c nch_c') (w_k + w_{k+1}) per point pair instead of
// w_k w_{k+1} for J J^T -- ~2x fewer FLOPs at config 2, ~5x at config 3, ~18x at
// config 4, and J (823 GB at config 4) never has to exist.

constexpr int GF_BM = 64;  // G-rows per tile side
constexpr int GF_STAGES = 4;
constexpr int GF_WM = 2, GF_WN = 4;            // warps along G-rows / G-columns
constexpr int GF_THREADS = 32 * GF_WM * GF_WN;  // 8 warps, 32 x 16 warp tiles
constexpr int GF_MI = GF_BM / GF_WM / 8;        // 8x8 fragments per warp tile: rows
constexpr int GF_NJ = GF_BM / GF_WN / 8;        //                               columns
constexpr int GF_STAGE_BYTES = 2 * GF_BM * 128;
constexpr int GF_H0_LD = 16;  // row pitch of the materialised input channels
constexpr int GF_GLD = GF_BM + 2;  // G-space product tile pitch (double2 RMW, fewer conflicts)
constexpr int GF_MAXCH = 16;       // channels per point the packed tiles support
constexpr int GF_GROUP = 16;       // tile rows per L2 super-block (decode_lower_grouped)

struct GramLayer {
  int kh;  // w_k (din for layer 0: materialised input channels)
  int kz;  // w_{k+1} (0 for the output layer: seeds)
};

struct GramParams {
  CUtensorMap maps[DNGD_MAX_LAYERS][2][DNGD_MAX_CLASSES];  // [layer][H/Z][class]
  Classes T;
  int L;
  GramLayer lay[DNGD_MAX_LAYERS];
  int nch[DNGD_MAX_CLASSES];  // channels per point (packed rows)
  int ppt[DNGD_MAX_CLASSES];  // whole points per 64-row tile = 64 / nch
  int npairs;
  int pc[10], pcp[10];       // class pair (c >= c')
  int tstart[11];            // tile prefix sums
  int tj_n[10];
  double* K;
  long long ldK;
  int tile0;  // first tile of this launch (tile-sharded multi-GPU Gram)
  // rect = 1: columns are gathered landmark points (Nystrom sketch K[:, I]):
  // column class cp has ccount[cp] points at output columns ccol0[cp] + j, read
  // through cmaps; all class pairs are rectangular and there is no mirror
  int rect;
  long long ccount[DNGD_MAX_CLASSES], ccol0[DNGD_MAX_CLASSES];
  CUtensorMap cmaps[DNGD_MAX_LAYERS][2][DNGD_MAX_CLASSES];
};

// Hext_0 rows: value channel [x], derivative channel d_j [e_j], Laplacian 0
__global__ void k_input_channels(Classes T, double* __restrict__ H0) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T.R * GF_H0_LD) return;
  const long long rho = idx / GF_H0_LD;
  const int d = static_cast<int>(idx - rho * GF_H0_LD);
  int ch;
  const long long p = act_point(T, rho, ch);
  const ClassDev& C = T.c[find_class(T, p)];
  double v = 0.0;
  if (d < T.din) {
    if (C.inp) {
      v = C.inp[((p - C.row0) * C.nch + ch) * T.din + d];
    } else if (ch == 0) {
      v = C.pts[(p - C.row0) * T.din + d];
    } else if (ch <= C.ngrad) {
      v = gdim(C, ch - 1, p - C.row0) == d ? 1.0 : 0.0;
    }
  }
  H0[idx] = v;
}

DNGD_DEV int gf_layer_chunks(const GramLayer& l) { return ((l.kh + 15) >> 4) + ((l.kz + 15) >> 4); }

// G[g-row][g-col] += (G_H + bias) o G_Z for one warp's 32 x 16 G-block.
// Fragment (i, j): rows lane/4 (+8i), columns 2(lane%4)+{0,1} (+8j).
// bias(gr, gc) = zA[gr] zB[gc] (1 where both rows are a value channel).
template <bool SEEDZ>
DNGD_DEV void gf_epilogue(double2 (&accH)[GF_MI][GF_NJ], double2 (&accZ)[GF_MI][GF_NJ],
                          const double* sA, const double* sB, const double* zA, const double* zB,
                          double* Gs, int wm, int wn, int lane) {
  const int lrow = lane >> 2;
#pragma unroll
  for (int i = 0; i < GF_MI; ++i) {
    const int gr = wm * (GF_MI * 8) + i * 8 + lrow;
    const double za = zA[gr], sa = sA[gr];
#pragma unroll
    for (int j = 0; j < GF_NJ; ++j) {
      const int gc = wn * (GF_NJ * 8) + j * 8 + 2 * (lane & 3);
      const double2 zb = *reinterpret_cast<const double2*>(zB + gc);
      double v0, v1;
      if (SEEDZ) {  // output layer: Zbar = per-row seeds (G^Z = seed_row * seed_col)
        const double2 sb = *reinterpret_cast<const double2*>(sB + gc);
        v0 = fma(za, zb.x, accH[i][j].x) * (sa * sb.x);
        v1 = fma(za, zb.y, accH[i][j].y) * (sa * sb.y);
      } else {
        v0 = fma(za, zb.x, accH[i][j].x) * accZ[i][j].x;
        v1 = fma(za, zb.y, accH[i][j].y) * accZ[i][j].y;
      }
      accH[i][j] = make_double2(0.0, 0.0);
      accZ[i][j] = make_double2(0.0, 0.0);
      double2* g = reinterpret_cast<double2*>(Gs + gr * GF_GLD + gc);
      double2 cur = *g;
      cur.x += v0;
      cur.y += v1;
      *g = cur;
    }
  }
}

__global__ void __launch_bounds__(GF_THREADS, 2)
    k_gram_factored(const __grid_constant__ GramParams p) {
  extern __shared__ uint8_t gf_smem_raw[];
  uint8_t* smem = smem_align(gf_smem_raw, 1024);
  double* Gs = reinterpret_cast<double*>(smem + GF_STAGES * GF_STAGE_BYTES);  // 64 x GF_GLD
  uint64_t* full = reinterpret_cast<uint64_t*>(Gs + GF_BM * GF_GLD);
  uint64_t* empty = full + GF_STAGES;
  // ---- tile decode
  int pi = 0;
  const int tile = static_cast<int>(blockIdx.x) + p.tile0;
  while (pi + 1 < p.npairs && tile >= p.tstart[pi + 1]) ++pi;
  const int t = tile - p.tstart[pi];
  const int c = p.pc[pi], cp = p.pcp[pi];
  int ti, tj;
  if (c == cp && !p.rect) {
    decode_lower_grouped(t, p.tj_n[pi], GF_GROUP, ti, tj);
  } else {
    ti = t / p.tj_n[pi];
    tj = t - ti * p.tj_n[pi];
  }
  const int na = p.nch[c], nb = p.nch[cp];
  const int np_r = p.ppt[c], np_c = p.ppt[cp];
  const int P0 = ti * np_r, Q0 = tj * np_c;  // first point of the tile rows / cols
  int nchunks = 0;
  for (int k = 0; k < p.L; ++k) nchunks += gf_layer_chunks(p.lay[k]);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < GF_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], GF_THREADS / 32);
    }
    fence_barrier_init();
  }
  for (int e = threadIdx.x; e < GF_BM * GF_GLD / 2; e += GF_THREADS)
    reinterpret_cast<double2*>(Gs)[e] = make_double2(0.0, 0.0);
  // per G-row: output-layer seeds and the value-channel flag of the bias entry
  // (0 past the tile's whole points and past the class end)
  __shared__ __align__(16) double sA[GF_BM], sB[GF_BM], zA[GF_BM], zB[GF_BM];
  if (threadIdx.x < GF_BM) {
    const int g = threadIdx.x;
    const ClassDev& Ca = p.T.c[c];
    const ClassDev& Cb = p.T.c[cp];
    const int cha = g % na, pa = P0 + g / na;
    const int chb = g % nb, pb = Q0 + g / nb;
    const bool oka = g < np_r * na && pa < Ca.count;
    const long long cntb = p.rect ? p.ccount[cp] : Cb.count;  // rect: c3 == 0 (no u0 lookup)
    const bool okb = g < np_c * nb && pb < cntb;
    sA[g] = oka ? seedc(p.T, Ca, cha, Ca.row0 + pa) : 0.0;
    sB[g] = okb ? seedc(p.T, Cb, chb, Cb.row0 + pb) : 0.0;
    zA[g] = (oka && cha == 0) ? 1.0 : 0.0;
    zB[g] = (okb && chb == 0) ? 1.0 : 0.0;
  }
  __syncthreads();

  auto issue = [&](int f) {
    int k = 0, g = f;
    while (k < p.L - 1 && g >= gf_layer_chunks(p.lay[k])) g -= gf_layer_chunks(p.lay[k++]);
    const int nh = (p.lay[k].kh + 15) >> 4;
    const int part = g < nh ? 0 : 1, kc = g < nh ? g : g - nh;
    const int st = f % GF_STAGES;
    uint8_t* sa = smem + st * GF_STAGE_BYTES;
    mbar_arrive_expect_tx(&full[st], GF_STAGE_BYTES);
    tma_load_2d(sa, &p.maps[k][part][c], &full[st], kc * 16, P0 * na);
    tma_load_2d(sa + GF_BM * 128, p.rect ? &p.cmaps[k][part][cp] : &p.maps[k][part][cp],
                &full[st], kc * 16, Q0 * nb);
  };
  if (threadIdx.x == 0) {
    for (int f = 0; f < min(nchunks, GF_STAGES); ++f) issue(f);
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / GF_WN, wn = warp - (warp / GF_WN) * GF_WN;
  const int lrow = lane >> 2;

  double2 accH[GF_MI][GF_NJ], accZ[GF_MI][GF_NJ];
#pragma unroll
  for (int i = 0; i < GF_MI; ++i)
#pragma unroll
    for (int j = 0; j < GF_NJ; ++j) {
      accH[i][j] = make_double2(0.0, 0.0);
      accZ[i][j] = make_double2(0.0, 0.0);
    }
  int k_cur = 0, f_layer_start = 0, f_layer_end = gf_layer_chunks(p.lay[0]);
  int nh_cur = (p.lay[0].kh + 15) >> 4;
  for (int f = 0; f < nchunks; ++f) {
    const int st = f % GF_STAGES;
    if (threadIdx.x == 0 && f >= 1 && f - 1 + GF_STAGES < nchunks) {
      const int pf = f - 1;
      mbar_wait(&empty[pf % GF_STAGES], (pf / GF_STAGES) & 1);
      issue(pf + GF_STAGES);
    }
    __syncwarp();
    mbar_wait(&full[st], (f / GF_STAGES) & 1);
    const bool partH = (f - f_layer_start) < nh_cur;
    const uint8_t* sa = smem + st * GF_STAGE_BYTES + (wm * GF_MI * 8 + lrow) * 128;
    const uint8_t* sb = smem + st * GF_STAGE_BYTES + GF_BM * 128 + (wn * GF_NJ * 8 + lrow) * 128;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sw = ((2 * (lane & 3) + h) ^ lrow) << 4;
      double2 a[GF_MI], b[GF_NJ];
#pragma unroll
      for (int i = 0; i < GF_MI; ++i) a[i] = *reinterpret_cast<const double2*>(sa + i * 1024 + sw);
#pragma unroll
      for (int j = 0; j < GF_NJ; ++j) b[j] = *reinterpret_cast<const double2*>(sb + j * 1024 + sw);
      // the .x and .y halves go through separate passes so consecutive DMMAs on
      // one accumulator are MI*NJ instructions apart (no back-to-back dependency)
      if (partH) {
#pragma unroll
        for (int i = 0; i < GF_MI; ++i)
#pragma unroll
          for (int j = 0; j < GF_NJ; ++j) dmma_8x8x4(accH[i][j], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < GF_MI; ++i)
#pragma unroll
          for (int j = 0; j < GF_NJ; ++j) dmma_8x8x4(accH[i][j], a[i].y, b[j].y);
      } else {
#pragma unroll
        for (int i = 0; i < GF_MI; ++i)
#pragma unroll
          for (int j = 0; j < GF_NJ; ++j) dmma_8x8x4(accZ[i][j], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < GF_MI; ++i)
#pragma unroll
          for (int j = 0; j < GF_NJ; ++j) dmma_8x8x4(accZ[i][j], a[i].y, b[j].y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (f + 1 != f_layer_end) continue;
    // ---- layer k_cur done: output layer Zbar = per-row seeds, else the Z accumulator
    if (p.lay[k_cur].kz == 0) {
      gf_epilogue<true>(accH, accZ, sA, sB, zA, zB, Gs, wm, wn, lane);
    } else {
      gf_epilogue<false>(accH, accZ, sA, sB, zA, zB, Gs, wm, wn, lane);
    }
    if (k_cur + 1 < p.L) {
      ++k_cur;
      f_layer_start = f_layer_end;
      f_layer_end += gf_layer_chunks(p.lay[k_cur]);
      nh_cur = (p.lay[k_cur].kh + 15) >> 4;
    }
  }
  __syncthreads();
  // ---- channel reduction (fixed order) and K[row][col] with its mirror
  const long long cnt_r = p.T.c[c].count;
  const long long row0 = p.T.c[c].row0;
  const long long cnt_c = p.rect ? p.ccount[cp] : p.T.c[cp].count;
  const long long col0 = p.rect ? p.ccol0[cp] : p.T.c[cp].row0;
  for (int e = threadIdx.x; e < np_r * np_c; e += GF_THREADS) {
    const int r = e / np_c, cc = e - (e / np_c) * np_c;
    const long long pr = P0 + r, pcl = Q0 + cc;
    if (pr >= cnt_r || pcl >= cnt_c) continue;
    const long long row = row0 + pr, col = col0 + pcl;
    if (!p.rect && c == cp && col > row) continue;
    const double* g = Gs + (r * na) * GF_GLD + cc * nb;
    double v = 0.0;
    for (int a = 0; a < na; ++a)
      for (int b = 0; b < nb; ++b) v += g[a * GF_GLD + b];
    p.K[row * p.ldK + col] = v;
    if (!p.rect) p.K[col * p.ldK + row] = v;
  }
}

static size_t gram_factored_smem() {
  return 1024 + GF_STAGES * GF_STAGE_BYTES + GF_BM * GF_GLD * sizeof(double) +
         2 * GF_STAGES * sizeof(uint64_t);
}
