// Factored dual Gram on the int8 tensor cores: the products of gram_factored.cuh
//     K_ij = sum_k sum_{c,c'} (Hext_k[i,c] . Hext_k[j,c']) (Zbar_k[i,c] . Zbar_k[j,c'])
// with every G-space GEMM (G^H_k = H_k H_k^T, G^Z_k = Zbar_k Zbar_k^T) emulated
// in FP64 by Ozaki slices (ozaki.cu, tc05.cuh): each activation row is cut into
// S int8 digits below a per-row power-of-two scale, and the S(S+1)/2 digit
// products of a 32-wide K-chunk run as exact int32 tcgen05 MMAs into S diagonal
// accumulators in TMEM.
//
// Tile: 128 G-rows (2 ppc whole points of the row class) x 64 G-columns (ppc =
// floor(64 / nch) whole points of the column class).  Per layer two MMA phases
// (Z then H; the output layer's Z is the per-row residual seeds).  Warp roles:
// warp 0 streams {32 B x rows x S slices} TMA boxes of the sliced activations
// through a 3-stage mbarrier ring; warp 1 owns TMEM (512 columns = S diagonals
// x 64) and issues the MMAs (one elected lane, A tiles held in the collector
// across their S - t products); warps 2-9 drain TMEM after each phase: thread
// (q, h) owns G-row 32q + lane and G-columns 32h .. 32h + 31, folds the S int32
// diagonals exactly into FP64 (oz_combine), applies the row/column scales and
// the bias entry, parks G^Z in shared memory (column-major, conflict-free) and
// accumulates G^H o G^Z in registers.  After the last layer the G tile goes to
// shared memory and every point pair sums its nch x nch' block in a fixed
// order (deterministic K, as the DMMA kernel).
//
// Tile order: lower triangle of (row tile, column tile) with column tiles half
// as tall, in super-rows of GO_GROUP row tiles walked column by column, so the
// ~148 CTAs in flight share their operand tiles through L2.

constexpr int GO_GROUP = 8;

struct GozParams {
  CUtensorMap mA[DNGD_MAX_LAYERS][2];  // sliced H_k / Zbar_k, box 64 B x 128 rows x S
  CUtensorMap mB[DNGD_MAX_LAYERS][2];  // same buffers, box 32 B x 64 rows x S
  const double* sc[DNGD_MAX_LAYERS][2];  // per activation row: 2^e (NaN = non-finite row)
  long long R;                           // activation rows
  Classes T;
  int L;
  int nk[DNGD_MAX_LAYERS][2];  // 32-wide K-chunks per phase (Z of the output layer: 0)
  int nch[DNGD_MAX_CLASSES];
  int ppc[DNGD_MAX_CLASSES];  // whole points per 64-row column tile; row tiles hold 2 ppc
  int npairs;
  int pc[10], pcp[10];
  int tstart[11];
  int ti_n[10], tj_n[10];
  double* K;
  long long ldK;
  int tile0;
  // rect: K[:, I] of the Nystrom sketch (solver.py:259-261) -- column tiles over the
  // gathered landmark activations (mB / scB over Rb gathered rows; landmarks of class
  // c are columns lcol0[c] .. + lcnt[c] - 1 of K, global points lpt[.]), every class
  // pair a full rectangle, one write per entry
  int rect;
  const double* scB[DNGD_MAX_LAYERS][2];
  long long Rb;
  long long lcol0[DNGD_MAX_CLASSES], lcnt[DNGD_MAX_CLASSES], lrow0[DNGD_MAX_CLASSES];
  const long long* lpt;
  int dbg;  // timing experiments only (tools/goz_dbg.sh): 1 narrow MMAs, 2 no MMA, 3 no MMA no drain,
           // 4 no drain, 5 no TMA no drain, 6 = 5 with narrow MMAs, 7 = 5 without the TMEM hand-off wait,
           // 8 = 7 without operand waits (MMA issue alone)
};

// lower-triangle tile t of TI row tiles (row tile ti spans column tiles 2ti, 2ti+1)
// in super-rows of GO_GROUP row tiles, column-major inside a super-row
DNGD_DEV void goz_decode_tri(int t, int TI, int& ti, int& tj) {
  constexpr int G = GO_GROUP;
  int I = static_cast<int>((sqrt(1.0 + 4.0 * t) - 1.0) * 0.5) / G;
  while (I > 0 && static_cast<long long>(G) * I * (G * I + 1) > t) --I;
  while (G * (I + 1) < TI && static_cast<long long>(G) * (I + 1) * (G * (I + 1) + 1) <= t) ++I;
  const int r0 = G * I, h = min(G, TI - r0);
  int u = t - r0 * (r0 + 1);
  const int full = h * (2 * r0 + 2);
  if (u < full) {
    tj = u / h;
    ti = r0 + u % h;
    return;
  }
  u -= full;
  for (int s = 0; s < h - 1; ++s) {
    const int n = h - 1 - s;
    if (u < 2 * n) {
      tj = 2 * r0 + 2 + 2 * s + u / n;
      ti = r0 + s + 1 + u % n;
      return;
    }
    u -= 2 * n;
  }
  ti = tj = 0;
}

DNGD_DEV void goz_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(256);
  }
}

// Operand rings: A (the 128-row tile) in 64-wide K slabs of 64-byte TMA rows, GO_SA
// deep; B (64 rows) in 32-wide K chunks of 32-byte rows, GO_SB deep.  TMA serves one
// box row per cycle per SM (tools/micro/tma_rate.cu), so A's rows carry two MMA
// K-steps each; B keeps the narrow rows so the whole ring + G^H fits in 227 KB.
constexpr int GO_SA = 2, GO_SB = 3;


// tile t (relative to p.tile0) -> (class pair, row tile, column tile)
struct GozTile {
  int c, cp, ti, tj;
};
DNGD_DEV GozTile goz_tile(const GozParams& p, int tile) {
  GozTile r;
  int pi = 0;
  while (pi + 1 < p.npairs && tile >= p.tstart[pi + 1]) ++pi;
  const int t = tile - p.tstart[pi];
  r.c = p.pc[pi];
  r.cp = p.pcp[pi];
  if (r.c == r.cp && !p.rect) {
    goz_decode_tri(t, p.ti_n[pi], r.ti, r.tj);
  } else {  // rectangle, column-major: CTAs in flight share the column tiles
    r.tj = t / p.ti_n[pi];
    r.ti = t - r.tj * p.ti_n[pi];
  }
  return r;
}

// Phase order within a layer: Z first (parked in PH), then H (multiplied in);
// the output layer has only its H phase (G^Z = the residual seeds).  Z-first puts
// a long phase (Z_0, w_1 wide) at the start of every tile, so the previous tile's
// point-pair reduction (which reads PH) overlaps its MMAs.
DNGD_DEV int goz_nphase(const GozParams& p, int k) { return p.nk[k][1] > 0 ? 2 : 1; }
DNGD_DEV int goz_part(const GozParams& p, int k, int i) { return p.nk[k][1] > 0 ? 1 - i : 0; }

// Persistent: one CTA per SM walks tiles blockIdx.x, + gridDim.x, ...  The TMA
// producer runs ahead across tile boundaries; the MMA warp starts a tile's first
// phase as soon as the epilogue has drained the previous tile's last one, while
// the epilogue reduces that tile's point pairs and writes K.
template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1) k_gram_oz(const __grid_constant__ GozParams p, int ntiles) {
  extern __shared__ uint8_t go_smem_raw[];
  uint8_t* smem = smem_align(go_smem_raw, 1024);
  constexpr int ASLAB = S * OZ_BM * 64, BCHUNK = S * OZ_BN * 32;
  uint8_t* ringA = smem;
  uint8_t* ringB = smem + GO_SA * ASLAB;
  double* PH = reinterpret_cast<double*>(ringB + GO_SB * BCHUNK);  // [64 cols][128 rows]
  uint64_t* fullA = reinterpret_cast<uint64_t*>(PH + OZ_BM * OZ_BN);
  uint64_t* emptyA = fullA + GO_SA;
  uint64_t* fullB = emptyA + GO_SA;
  uint64_t* emptyB = fullB + GO_SB;
  uint64_t* tfull = emptyB + GO_SB;
  uint64_t* tempty = tfull + 1;
  uint32_t* taddr_sh = reinterpret_cast<uint32_t*>(tempty + 1);
  __shared__ double sA[OZ_BM], sB[OZ_BN], zA[OZ_BM], zB[OZ_BN];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < GO_SA; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&emptyA[i], 1);
    }
    for (int i = 0; i < GO_SB; ++i) {
      mbar_init(&fullB[i], 1);
      mbar_init(&emptyB[i], 1);
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

  if (warp == 0) {
    // ---- TMA producer: every phase's K-chunks of every tile; an A slab every second chunk
    if (lane == 0 && p.dbg != 8) {
      int fa = 0, fb = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const GozTile g = goz_tile(p, tile + p.tile0);
        const int arow0 = static_cast<int>(p.T.c[g.c].act0 + static_cast<long long>(g.ti) * 2 * p.ppc[g.c] * p.nch[g.c]);
        const int brow0 = static_cast<int>((p.rect ? p.lrow0[g.cp] : p.T.c[g.cp].act0) +
                                           static_cast<long long>(g.tj) * p.ppc[g.cp] * p.nch[g.cp]);
        for (int k = 0; k < p.L; ++k) {
          for (int i = 0; i < goz_nphase(p, k); ++i) {
            const int part = goz_part(p, k, i);
            const int nk = p.nk[k][part];
            for (int kc = 0; kc < nk; ++kc, ++fb) {
              if ((kc & 1) == 0) {
                const int sa = fa % GO_SA;
                if (fa >= GO_SA) mbar_wait(&emptyA[sa], ((fa / GO_SA) - 1) & 1);
                if (p.dbg >= 5) {
                  mbar_arrive(&fullA[sa]);
                } else {
                  mbar_arrive_expect_tx(&fullA[sa], ASLAB);
                  tma_load_3d(ringA + sa * ASLAB, &p.mA[k][part], &fullA[sa], kc * 32, arow0, 0);
                }
                ++fa;
              }
              const int sb = fb % GO_SB;
              if (fb >= GO_SB) mbar_wait(&emptyB[sb], ((fb / GO_SB) - 1) & 1);
              if (p.dbg >= 5) {
                mbar_arrive(&fullB[sb]);
              } else {
                mbar_arrive_expect_tx(&fullB[sb], BCHUNK);
                tma_load_3d(ringB + sb * BCHUNK, &p.mB[k][part], &fullB[sb], kc * 32, brow0, 0);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: lane 0 alone waits and issues (no warp-wide mbarrier polling)
    constexpr uint32_t idesc = umma_idesc_s8(OZ_BM, OZ_BN);
    int fa = 0, fb = 0, ph = 0;
    if (lane == 0) {
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int k = 0; k < p.L; ++k) {
          for (int i = 0; i < goz_nphase(p, k); ++i) {
            const int nk = p.nk[k][goz_part(p, k, i)];
            if (ph > 0 && p.dbg < 7) mbar_wait(tempty, (ph - 1) & 1);  // epilogue drained the last phase
            tc_fence_after();
            for (int kc = 0; kc < nk; ++kc, ++fb) {
              const int sa = fa % GO_SA, sb = fb % GO_SB;
              if (p.dbg != 8) {
                if ((kc & 1) == 0) mbar_wait(&fullA[sa], (fa / GO_SA) & 1);
                mbar_wait(&fullB[sb], (fb / GO_SB) & 1);
              }
              tc_fence_after();
              const bool last_of_slab = (kc & 1) == 1 || kc == nk - 1;
              const uint32_t a0 = smem_u32(ringA + sa * ASLAB) + 32 * (kc & 1);
              const uint32_t b0 = smem_u32(ringB + sb * BCHUNK);
              if (p.dbg == 1 || p.dbg == 6) {
                oz_issue_chunk<S, 64, 32>(tbase, OZ_BN, a0, OZ_BM * 64, b0, OZ_BN * 32, idesc, kc == 0);
              } else if (p.dbg == 2 || p.dbg == 3) {
              } else {
                oz_issue_chunk_wide<S, 64, 32>(tbase, a0, OZ_BM * 64, b0, OZ_BN * 32, kc == 0);
              }
              umma_commit(&emptyB[sb]);
              if (last_of_slab) umma_commit(&emptyA[sa]);
              if (kc == nk - 1) umma_commit(tfull);
              if (last_of_slab) ++fa;
            }
            ++ph;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: thread owns G-row `row`, G-columns col0 .. col0 + OZ_COLS - 1
    // (warp w reaches TMEM lanes 32 (w % 4) ..; four consecutive warps cover all four)
    const int q = warp & 3, hh = (warp - 2) >> 2;
    const int row = 32 * q + lane, col0 = OZ_COLS * hh;
    const uint32_t tl = tbase + (static_cast<uint32_t>(32 * q) << 16);
    int ph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const GozTile g = goz_tile(p, tile + p.tile0);
      const int c = g.c, cp = g.cp;
      const int na = p.nch[c], nb = p.nch[cp];
      const int np_r = 2 * p.ppc[c], np_c = p.ppc[cp];
      const int P0 = g.ti * np_r, Q0 = g.tj * np_c;
      const ClassDev& Ca = p.T.c[c];
      const ClassDev& Cb = p.T.c[cp];
      const long long arow0 = Ca.act0 + static_cast<long long>(P0) * na;
      const long long brow0 = (p.rect ? p.lrow0[cp] : Cb.act0) + static_cast<long long>(Q0) * nb;
      const long long ccount = p.rect ? p.lcnt[cp] : Cb.count;  // column points
      // row seeds / value flags of this tile (the previous tile's last use of them was
      // its final drain; the barrier also orders the previous reduction's PH reads
      // before this tile's first PH writes)
      if (threadIdx.x < 64 + OZ_BM) {
        const int gi = threadIdx.x - 64;
        const int cha = gi % na, pa = P0 + gi / na;
        const bool ok = gi < np_r * na && pa < Ca.count;
        sA[gi] = ok ? seedc(p.T, Ca, cha, Ca.row0 + pa) : 0.0;
        zA[gi] = (ok && cha == 0) ? 1.0 : 0.0;
      } else if (threadIdx.x < 64 + OZ_BM + OZ_BN) {
        const int gi = threadIdx.x - 64 - OZ_BM;
        const int chb = gi % nb, pb = Q0 + gi / nb;
        const bool ok = gi < np_c * nb && pb < ccount;
        sB[gi] = ok ? seedc(p.T, Cb, chb, p.rect ? p.lpt[p.lcol0[cp] + pb] : Cb.row0 + pb) : 0.0;
        zB[gi] = (ok && chb == 0) ? 1.0 : 0.0;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(OZ_ETHREADS) : "memory");
      const long long arow = arow0 + row;
      double G[OZ_COLS];
#pragma unroll
      for (int j = 0; j < OZ_COLS; ++j) G[j] = 0.0;
      for (int k = 0; k < p.L; ++k) {
        const bool seeds = p.nk[k][1] == 0;  // output layer: G^Z = seed_row seed_col
        for (int i = 0; i < goz_nphase(p, k); ++i) {
          const int part = goz_part(p, k, i);
          // one thread polls the mbarrier, the other epilogue warps sleep on a named
          // barrier: eight warps spinning on try_wait took shared-memory cycles from
          // the tensor core's operand reads (MMA issue alone ran ~35 % slower)
          if (threadIdx.x == 64) mbar_wait(tfull, ph & 1);
          asm volatile("bar.sync 2, %0;" ::"n"(OZ_ETHREADS) : "memory");
          tc_fence_after();
          if (p.dbg >= 3) {  // timing experiments: no drain
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            ++ph;
            continue;
          }
          const double* scv = p.sc[k][part];
          const double sr = arow < p.R ? scv[arow] : 0.0;
          // this warp's column scales: lane j < OZ_COLS holds column col0 + j (shuffled below)
          const long long bl = brow0 + col0 + lane;
          const double scl = p.rect ? (bl < p.Rb ? p.scB[k][part][bl] : 0.0) : (bl < p.R ? scv[bl] : 0.0);
          const double za = zA[row], sar = sA[row];
#pragma unroll
          for (int cc = 0; cc < OZ_COLS / OZ_LD; ++cc) {
            int32_t acc[S][OZ_LD];
#pragma unroll
            for (int d = 0; d < S; ++d) tmem_ld<OZ_LD>(tl + d * OZ_BN + col0 + OZ_LD * cc, acc[d]);
            tmem_ld_wait();
            if (cc == OZ_COLS / OZ_LD - 1) {  // every diagonal is in registers: hand TMEM to the next phase
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(tempty);
            }
#pragma unroll
            for (int j = 0; j < OZ_LD; ++j) {
              const int gc = col0 + OZ_LD * cc + j;
              const double scol = __shfl_sync(0xffffffffu, scl, OZ_LD * cc + j);
              int32_t a[S];
#pragma unroll
              for (int d = 0; d < S; ++d) a[d] = acc[d][j];
              const double v = oz_combine<S>(a) * (sr * scol);
              if (part == 1) {
                PH[gc * OZ_BM + row] = v;  // G^Z, parked for the H phase
              } else {
                const double vh = fma(za, zB[gc], v);  // + bias entry (value channels)
                G[OZ_LD * cc + j] = seeds ? fma(vh, sar * sB[gc], G[OZ_LD * cc + j])
                                          : fma(PH[gc * OZ_BM + row], vh, G[OZ_LD * cc + j]);
              }
            }
          }
          ++ph;
        }
      }
      // ---- G tile to shared memory (PH is free: the last phase was the output layer's H)
#pragma unroll
      for (int j = 0; j < OZ_COLS; ++j) PH[(col0 + j) * OZ_BM + row] = G[j];
      asm volatile("bar.sync 1, %0;" ::"n"(OZ_ETHREADS) : "memory");
      const long long cnt_r = Ca.count, cnt_c = ccount;
      for (int e = threadIdx.x - 64; e < np_r * np_c; e += OZ_ETHREADS) {
        const int r = e / np_c, cc = e - (e / np_c) * np_c;
        const long long pr = P0 + r, pcl = Q0 + cc;
        if (pr >= cnt_r || pcl >= cnt_c) continue;
        const long long grow = Ca.row0 + pr, gcol = (p.rect ? p.lcol0[cp] : Cb.row0) + pcl;
        if (!p.rect && c == cp && gcol > grow) continue;
        double v = 0.0;
        for (int a = 0; a < na; ++a)
          for (int b = 0; b < nb; ++b) v += PH[(cc * nb + b) * OZ_BM + r * na + a];
        p.K[grow * p.ldK + gcol] = v;
        if (!p.rect) p.K[gcol * p.ldK + grow] = v;
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

static size_t gram_oz_smem(int S) {
  return 1024 + static_cast<size_t>(GO_SA) * S * OZ_BM * 64 + static_cast<size_t>(GO_SB) * S * OZ_BN * 32 +
         static_cast<size_t>(OZ_BM) * OZ_BN * 8 + (2 * GO_SA + 2 * GO_SB + 2) * 8 + 64;
}
