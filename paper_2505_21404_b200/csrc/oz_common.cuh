// Tile constants of the emulated-FP64 (Ozaki, int8 tcgen05) kernels.
#pragma once

#include <stddef.h>

namespace dngd {

constexpr int OZ_BM = 128;  // tile rows = MMA M (TMEM lanes)
constexpr int OZ_BN = 64;   // tile columns = MMA N; S diagonals x 64 <= 512 TMEM columns
constexpr int OZ_THREADS = 320;  // warp 0 TMA, warp 1 TMEM + MMA, warps 2-9 epilogue
constexpr long long kOzMaxK = 32768;  // |acc_D| <= K (2 127 64 + 6 64^2) < 2^31 (tc05.cuh)

inline long long oz_kpad(long long K) { return (K + 31) / 32 * 32; }

// ring of STAGES K-chunks (32 int8 of every slice of a 128-row and a 64-row tile)
// + mbarriers + the TMEM address, after 1024-byte alignment of the base
inline size_t oz_smem_bytes(int S, int stages) {
  return 1024 + static_cast<size_t>(stages) * S * (OZ_BM + OZ_BN) * 32 + (2 * stages + 10) * 8 + 16;
}

}  // namespace dngd
