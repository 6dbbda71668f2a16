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
// x = scale * sum_{t<S} d_t 2^{-8(t+1)} + O(scale 2^{-8S-1}), |d_0| <= 127,
// d_t in [-128, 127] (balanced base-256 digits: the whole int8 range), scale = 2^e
// with max|row| 2^-e 256 <= 127 (oz_row_exponent).  A product of two sliced values
// is sum_D acc_D 2^{-8(D+2)} with acc_D = sum_{t+u=D} d_t e_u; the diagonals
// D >= S are dropped (below the slicing error).  oz_combine folds the int32
// diagonals exactly into two int64 (|acc_D| < 2^31 for K <= 16384) and rounds
// once.
// Digits of a value with row scale 2^e: X = rint(v 2^(8S - e)) (exact power-of-two
// scaling, one rounding; |X| <= 2^(8S) 127/256).  With the carry offsets added up
// front, Y = X + 128 (1 + 256 + ... + 256^(S-2)), the balanced digit t >= 1 is byte
// S-1-t of Y minus 128 -- i.e. that byte with its top bit flipped, read as int8 --
// and d_0 = Y >> 8(S-1) (arithmetic).  No per-digit arithmetic at all: one
// conversion, one 64-bit add, one XOR mask, byte extracts.  Balanced digits matter:
// the products dropped below diagonal S then average out over K instead of adding
// up.  Byte b of word t holds digit t of value b.
template <int S>
DNGD_DEV constexpr long long oz_offset() {
  long long o = 0;
  for (int t = 0; t < S - 1; ++t) o |= 0x80LL << (8 * t);
  return o;
}
// Y ^ mask: bytes 0 .. S-2 are the digits S-1 .. 1 (as int8), byte S-1 is d_0
template <int S>
DNGD_DEV long long oz_digit_bytes(double v, double sinv, bool bad) {
  const long long X = bad ? 0LL : __double2ll_rn(v * sinv);
  return (X + oz_offset<S>()) ^ oz_offset<S>();
}
template <int S>
DNGD_DEV void oz_digits4(const double (&v)[4], double sinv, bool bad, uint32_t (&packed)[S]) {
  static_assert(S >= 5 && S <= 7, "X must fit 2^55");
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const long long y = oz_digit_bytes<S>(v[b], sinv, bad);
    lo[b] = static_cast<uint32_t>(y);
    hi[b] = static_cast<uint32_t>(static_cast<unsigned long long>(y) >> 32);
  }
  // digit t = byte (S-1-t) of y: gather that byte of the four values into one word
#pragma unroll
  for (int t = 0; t < S; ++t) {
    const int byte = S - 1 - t;
    const uint32_t* w = byte < 4 ? lo : hi;
    const uint32_t sel = 0x4u * 0 + (byte & 3);  // byte index inside each word
    // __byte_perm(x, y, s): nibble k of s picks byte (0-3 from x, 4-7 from y)
    const uint32_t p01 = __byte_perm(w[0], w[1], sel | ((4u + sel) << 4));
    const uint32_t p23 = __byte_perm(w[2], w[3], sel | ((4u + sel) << 4));
    packed[t] = __byte_perm(p01, p23, 0x5410);
  }
}

// row scale exponent: 2^e with max|row| 2^-e 256 <= 127, so that the leading digit
// floor((X + offset) / 2^(8(S-1))) stays inside [-127, 127]
DNGD_DEV int oz_row_exponent(double mx) {
  int e = 0;
  if (mx > 0.0) {
    const double f = frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
    e += (f * 128.0 > 127.0) ? 2 : 1;
  }
  return e;
}

template <int S>
DNGD_DEV double oz_combine(const int32_t (&acc)[S]) {
  static_assert(S >= 5 && S <= 7, "two int64 halves");
  constexpr int B = OZ_BITS;
  constexpr int H = S / 2;  // diagonals 0 .. H-1 in hi, H .. S-1 in lo
  // 32 x 32 -> 64-bit multiply-adds (IMAD.WIDE), exact: |hi| < 2^31 2^(8(H-1)) 1.01
  // < 2^48, |lo| < 2^31 2^(8(S-H-1)) 1.01 < 2^56 (S = 7) -- the magic-constant
  // conversion below needs < 2^51, so S = 7 converts lo with I2F instead
  long long hi = static_cast<long long>(acc[0]);
#pragma unroll
  for (int d = 1; d < H; ++d) hi = hi * (1LL << B) + static_cast<long long>(acc[d]);
  long long lo = static_cast<long long>(acc[H]);
#pragma unroll
  for (int d = H + 1; d < S; ++d) lo = lo * (1LL << B) + static_cast<long long>(acc[d]);
  // sum_{D<H} acc_D 2^{-B(D+2)} = hi 2^{-B(H+1)}; sum_{H<=D<S} acc_D 2^{-B(D+2)} = lo 2^{-B(S+1)}
  constexpr double kHi = 1.0 / static_cast<double>(1ULL << (B * (H + 1)));
  constexpr double kLo = kHi / static_cast<double>(1ULL << (B * (S - H)));
  if constexpr (S - H - 1 <= 2) {
    // int64 -> double without I2F: |hi|, |lo| < 2^51, so adding them to the bit
    // pattern of 1.5 2^52 ulp lands exactly on magic + hi ulp (one integer add, no
    // carry out of the mantissa).  ulp(M1) = kHi, ulp(M2) = kLo.
    constexpr double M1 = kHi * 0x1.8p52;
    constexpr double M2 = kLo * 0x1.8p52;
    const double a = __longlong_as_double(__double_as_longlong(M1) + hi) - (M1 + M2);  // hi kHi - M2, exact
    const double b = __longlong_as_double(__double_as_longlong(M2) + lo);              // M2 + lo kLo, exact
    return a + b;  // = round(hi kHi + lo kLo): the same single rounding as an fma
  } else {
    return fma(static_cast<double>(lo), kLo, static_cast<double>(hi) * kHi);
  }
}

}  // namespace dngd
