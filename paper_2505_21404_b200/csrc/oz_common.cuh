// Tile constants of the emulated-FP64 (Ozaki, int8 tcgen05) kernels.
#pragma once

#include <stddef.h>

namespace dngd {

constexpr int OZ_BM = 128;  // tile rows = MMA M (TMEM lanes)
constexpr int OZ_BN = 64;   // tile columns = MMA N; S diagonals x 64 <= 512 TMEM columns
// Warp roles: warp 0 TMA, warp 1 TMEM + MMA, warps 2 .. 2 + OZ_EPI - 1 epilogue.
// OZ_EPI / 4 epilogue warps per TMEM lane quadrant (warp w reaches lanes 32 (w % 4)
// ..); each thread drains OZ_COLS columns of its row in groups of OZ_LD
// (tcgen05.ld 32x32b.x{OZ_LD}).  Sixteen warps halve the per-thread drain of eight
// and keep four warps per scheduler: the MMA warp waits on the drain whenever the
// S diagonals fill TMEM (S x 64 of 512 columns, no second accumulator set).
constexpr int OZ_EPI = 16, OZ_LD = 4;
constexpr int OZ_COLS = OZ_BN / (OZ_EPI / 4);
constexpr int OZ_ETHREADS = 32 * OZ_EPI;
constexpr int OZ_THREADS = 64 + OZ_ETHREADS;
// Digit base 2^OZ_BITS: balanced base-256 digits fill the int8 range [-128, 127]
// (round 2 start: base 128, 7 digits = 28 products per FP64 product; base 256 needs
// 6 digits = 21 products for the same ~48 bits below the row maximum).
constexpr int OZ_BITS = 8;
constexpr int OZ_SMIN = 6, OZ_SMAX = 7;  // 48 / 56 bits; 8 digits would overflow the int64 X
constexpr long long kOzMaxK = 16384;  // |acc_D| <= K (2 127 128 + 5 128^2) < 2^31 (tc05.cuh)

inline long long oz_kpad(long long K) { return (K + 31) / 32 * 32; }

// ring of STAGES K-chunks (32 int8 of every slice of a 128-row and a 64-row tile)
// + mbarriers + the TMEM address, after 1024-byte alignment of the base
inline size_t oz_smem_bytes(int S, int stages) {
  return 1024 + static_cast<size_t>(stages) * S * (OZ_BM + OZ_BN) * 32 + (2 * stages + 10) * 8 + 16;
}

}  // namespace dngd
