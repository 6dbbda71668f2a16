// tcgen05 (5th-generation tensor core) wrappers for the emulated-FP64 path:
// TMEM allocation, the kind::i8 MMA with shared-memory descriptors, commits to
// mbarriers and TMEM -> register loads.  Everything is raw PTX for sm_100a.
//
// Operand layout used throughout: K-major int8 tiles of 32-byte rows staged by
// TMA with CU_TENSOR_MAP_SWIZZLE_32B, i.e. the canonical UMMA K-major SW32
// layout ((8,m),2):((2,SBO),1) in 16-byte units -- rows 32 B apart, 8-row
// groups SBO = 256 B apart.  One MMA consumes exactly K = 32 int8 = one row.
#pragma once

#include "common.cuh"
#include "oz_common.cuh"

namespace dngd {

// ---------------------------------------------------------------- descriptors
// shared-memory matrix descriptor (sm100 UMMA): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48), base offset 0, layout [61,64)
DNGD_DEV uint64_t umma_desc_sw32(uint32_t saddr) {
  constexpr uint64_t kLBO = 1;            // unused for swizzled K-major
  constexpr uint64_t kSBO = 256 >> 4;     // 8 rows x 32 B
  constexpr uint64_t kLayoutSW32 = 6;
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (kLBO << 16) | (kSBO << 32) |
         (1ull << 46) | (kLayoutSW32 << 61);
}

// K-major, 64-byte rows (two 32-byte MMA K-steps per row; the second step starts
// 32 bytes in), 128-byte swizzle... of 64-byte rows: SWIZZLE_64B, SBO = 8 rows x 64 B
DNGD_DEV uint64_t umma_desc_sw64(uint32_t saddr) {
  constexpr uint64_t kLBO = 1;
  constexpr uint64_t kSBO = 512 >> 4;
  constexpr uint64_t kLayoutSW64 = 4;
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (kLBO << 16) | (kSBO << 32) |
         (1ull << 46) | (kLayoutSW64 << 61);
}

template <int W>
DNGD_DEV uint64_t umma_desc_k(uint32_t saddr) {
  static_assert(W == 32 || W == 64, "32- or 64-byte operand rows");
  if constexpr (W == 32) {
    return umma_desc_sw32(saddr);
  } else {
    return umma_desc_sw64(saddr);
  }
}

// instruction descriptor, kind::i8: D s32 [4,6) = 2, A s8 [7,10) = 1, B s8
// [10,13) = 1, both K-major, N >> 3 [17,23), M >> 4 [24,29)
__host__ __device__ constexpr uint32_t umma_idesc_s8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// ---------------------------------------------------------------- TMEM
// one full warp: allocate ncols columns, the address lands in *dst (shared)
DNGD_DEV void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
DNGD_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
DNGD_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DNGD_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] B[smem]^T, int8 x int8 -> int32; accumulate == 0 overwrites.
// COLL selects the A collector buffer: 0 none, 1 fill (keep A), 2 use (reuse and
// keep), 3 lastuse (reuse) -- consecutive MMAs on one A tile read it from shared
// memory once (SASS: A_KEEP / A_REUSE).
#define DNGD_UMMA_I8(SUFFIX)                                                          \
  asm volatile(                                                                       \
      "{\n\t.reg .pred p;\n\t"                                                        \
      "setp.ne.b32 p, %4, 0;\n\t"                                                     \
      "tcgen05.mma.cta_group::1.kind::i8" SUFFIX " [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d), \
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)                             \
      : "memory")
template <int COLL = 0>
DNGD_DEV void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  if constexpr (COLL == 0) {
    DNGD_UMMA_I8("");
  } else if constexpr (COLL == 1) {
    DNGD_UMMA_I8(".collector::a::fill");
  } else if constexpr (COLL == 2) {
    DNGD_UMMA_I8(".collector::a::use");
  } else {
    DNGD_UMMA_I8(".collector::a::lastuse");
  }
}
#undef DNGD_UMMA_I8

// the S(S+1)/2 digit products of one K-chunk into the S diagonal accumulators
// (tmem + D * ncols): A_t stays in the collector across its S - t products.
// WA / WB: operand row width in bytes (32: one K-step per row; 64: a0 / b0 already
// point at the K-step's 32-byte half of the row)
template <int S, int WA = 32, int WB = 32>
DNGD_DEV void oz_issue_chunk(uint32_t tmem, int ncols, uint32_t a0, int abytes, uint32_t b0,
                             int bbytes, uint32_t idesc, bool first_chunk) {
#pragma unroll
  for (int t = 0; t < S; ++t) {
    const uint64_t ad = umma_desc_k<WA>(a0 + t * abytes);
    const uint32_t acc = (!first_chunk || t > 0) ? 1u : 0u;
#pragma unroll
    for (int u = 0; u < S - t; ++u) {
      const uint32_t d = tmem + (t + u) * ncols;
      const uint64_t bd = umma_desc_k<WB>(b0 + u * bbytes);
      if (S - t == 1) {
        umma_i8<0>(d, ad, bd, idesc, acc);
      } else if (u == 0) {
        umma_i8<1>(d, ad, bd, idesc, acc);
      } else if (u == S - t - 1) {
        umma_i8<3>(d, ad, bd, idesc, acc);
      } else {
        umma_i8<2>(d, ad, bd, idesc, acc);
      }
    }
  }
}

// The same S(S+1)/2 products as oz_issue_chunk, issued as ONE wide MMA per A
// slice: B's slices 0 .. S-1-t are consecutive 64-row blocks in shared memory (one
// operand of N = 64 (S - t) rows) and the S diagonal accumulators are consecutive
// 64-column blocks of TMEM, so A_t x [B_0 .. B_{S-1-t}]^T written at column 64 t
// lands block u on diagonal t + u.  N > 256 is split in two.  10 MMAs per chunk at
// S = 7 instead of 28 N = 64 ones (each of which cost ~45-70 cycles against the
// 32 of the tensor-core rate), A read once per t.
template <int S, int WA = 32, int WB = 32>
DNGD_DEV void oz_issue_chunk_wide(uint32_t tmem, uint32_t a0, int abytes, uint32_t b0, int bbytes,
                                  bool first_chunk) {
  static_assert(OZ_BN == 64, "diagonal blocks are 64 columns");
#pragma unroll
  for (int t = 0; t < S; ++t) {
    const uint64_t ad = umma_desc_k<WA>(a0 + t * abytes);
    const uint32_t acc = (!first_chunk || t > 0) ? 1u : 0u;
    constexpr int kMaxBlocks = 4;  // N <= 256
    const int nblk = S - t;
    const int n1 = nblk < kMaxBlocks ? nblk : kMaxBlocks;
    // compile-time N per t (the loop is unrolled)
    umma_i8<0>(tmem + t * OZ_BN, ad, umma_desc_k<WB>(b0), umma_idesc_s8(OZ_BM, OZ_BN * n1), acc);
    if (nblk > kMaxBlocks) {
      umma_i8<0>(tmem + (t + kMaxBlocks) * OZ_BN, ad, umma_desc_k<WB>(b0 + kMaxBlocks * bbytes),
                 umma_idesc_s8(OZ_BM, OZ_BN * (nblk - kMaxBlocks)), acc);
    }
  }
}

// arrive (once) on an mbarrier when every MMA issued so far by this thread completes
DNGD_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// warp loads 32 lanes x 8 consecutive 32-bit columns: lane i of the warp gets TMEM
// lane (addr.lane + i), columns addr.col .. +7
DNGD_DEV void tmem_ld8(uint32_t taddr, int32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
}
template <int W>
DNGD_DEV void tmem_ld(uint32_t taddr, int32_t (&r)[W]) {
  static_assert(W == 4 || W == 8, "x4 / x8");
  if constexpr (W == 8) {
    tmem_ld8(taddr, r);
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr)
                 : "memory");
  }
}
DNGD_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

DNGD_DEV bool elect_lane0() { return (threadIdx.x & 31) == 0; }

// ---------------------------------------------------------------- Ozaki digits
// x = scale * sum_{t<S} d_t 2^{-7(t+1)} + O(scale 2^{-7S-1}), |d_0| <= 127,
// |d_t| <= 64, scale a power of two >= max|row| (oz_digits4).  A product of two sliced values is
// sum_D acc_D 2^{-7(D+2)} with acc_D = sum_{t+u=D} d_t e_u; the diagonals
// D >= S are dropped (below the slicing error).  oz_combine folds the int32
// diagonals exactly into two int64 (|acc_D| < 2^31 for K <= 32768) and rounds
// once.
// Digits of 4 values of one row with scale 2^e: X = rint(v 2^(7S - e)) (exact
// power-of-two scaling, one rounding; |X| < 2^(7S) 127/128), then balanced
// base-128 digits from the bottom -- t = u + 64, d = (t & 127) - 64 in [-64, 63],
// u = t >> 7 -- and d_0 = the final u (|d_0| <= 127), so that
// v = 2^e sum_t d_t 2^{-7(t+1)} + O(2^(e - 7S - 1)).  Balanced digits matter: the
// products dropped below diagonal S then average out over K instead of adding up.
// One conversion per value, integer ops per digit (the FP64 rint/convert per digit
// was the slicing kernels' bottleneck).  Byte b of word t holds digit t of value b.
template <int S>
DNGD_DEV void oz_digits4(const double (&v)[4], double sinv, bool bad, uint32_t (&packed)[S]) {
#pragma unroll
  for (int t = 0; t < S; ++t) packed[t] = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    long long u = bad ? 0LL : __double2ll_rn(v[b] * sinv);
#pragma unroll
    for (int t = S - 1; t >= 1; --t) {
      const long long tt = u + 64;
      const int d = static_cast<int>(tt & 127) - 64;
      packed[t] |= (static_cast<uint32_t>(d) & 0xffu) << (8 * b);
      u = tt >> 7;
    }
    packed[0] |= (static_cast<uint32_t>(static_cast<int>(u)) & 0xffu) << (8 * b);
  }
}

// row scale exponent: 2^e >= max|row| with max 2^-e 128 < 127, so that the leading
// balanced digit (X - lower digits) / 2^(7(S-1)) < 127 + 0.504 stays inside int8
DNGD_DEV int oz_row_exponent(double mx) {
  int e = 0;
  if (mx > 0.0) {
    const double f = frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
    if (f * 128.0 >= 127.0) ++e;
  }
  return e;
}

template <int S>
DNGD_DEV double oz_combine(const int32_t (&acc)[S]) {
  // 32 x 32 -> 64-bit multiply-adds (IMAD.WIDE), exact
  long long hi = static_cast<long long>(acc[0]) * (1LL << 21);
  hi = static_cast<long long>(acc[1]) * (1LL << 14) + hi;
  hi = static_cast<long long>(acc[2]) * (1LL << 7) + hi;
  hi = static_cast<long long>(acc[3]) + hi;
  long long lo = static_cast<long long>(acc[4]) * (1LL << (7 * (S - 5)));
#pragma unroll
  for (int d = 5; d < S; ++d) lo = static_cast<long long>(acc[d]) * (1LL << (7 * (S - 1 - d))) + lo;
  // sum_{D<4} acc_D 2^{-7(D+2)} = hi 2^-35; sum_{4<=D<S} acc_D 2^{-7(D+2)} = lo 2^{-7(S+1)}
  static_assert(S >= 5 && S <= 8, "4 + 1..4 diagonals");
  constexpr double kLo = S == 8 ? 0x1p-63 : S == 7 ? 0x1p-56 : S == 6 ? 0x1p-49 : 0x1p-42;
  // int64 -> double without I2F: |hi|, |lo| < 2^51 (K <= 32768), so adding them to
  // the bit pattern of 1.5 2^52 ulp lands exactly on magic + hi ulp (one integer add,
  // no carry out of the mantissa).  ulp(M1) = 2^-35, ulp(M2) = kLo.
  constexpr double M1 = 0x1.8p17;
  constexpr double M2 = kLo * 0x1.8p52;
  const double a = __longlong_as_double(__double_as_longlong(M1) + hi) - (M1 + M2);  // hi 2^-35 - M2, exact
  const double b = __longlong_as_double(__double_as_longlong(M2) + lo);              // M2 + lo kLo, exact
  return a + b;  // = round(hi 2^-35 + lo kLo): the same single rounding as fma(lo, kLo, hi 2^-35)
}

}  // namespace dngd
