// Slice layout and digit helpers of the INT8-emulated FP64 GEMM, shared by
// the GEMM/slicing kernels (ozgemm.cu) and the fused stage+slicing kernels
// (stages.cu).
#pragma once
#include <cstdint>

#include "cgl_internal.h"

namespace cgl {
namespace oz {

constexpr int NONFINITE = 0x7fffffff;  // exponent marker: the row/column holds NaN/Inf
                                       // -> its outputs are NaN (as an FP64 GEMM would give)
constexpr int KC = kOzKC;  // K bytes per pipeline chunk (UMMA k-steps of 32 int8)

// ---- operand slicing ---------------------------------------------------------
// Tiled slice layout: [row tile][k chunk][slice][RT rows x KC bytes], each tile
// as [row/8][kbyte/16][row%8][kbyte%16].  rows padded to RT, K to KC (zeros).
// Blocks are slice-major inside: [row tile][k chunk][slice][RT x KC], so the
// slices a pipeline stage needs are ONE contiguous range (one bulk copy).
__host__ __device__ inline int64_t tile_offset(int64_t R, int64_t kb, int RT, int nchunks, int S) {
  const int64_t rt = R / RT, r = R % RT, ch = kb / KC, kk = kb % KC;
  return ((rt * nchunks + ch) * S * (int64_t)(RT * KC)) + (((r >> 3) * (KC / 16) + (kk >> 4)) * 8 + (r & 7)) * 16 +
         (kk & 15);
}

// floor digits, packed: q = trunc(x 2^(56-e)) split into hi = q >> 28 (signed)
// and lo = q mod 2^28; the S = 8 base-128 digits of four values are packed
// into one 32-bit word per slice with byte permutes (same digits as
// digits8_floor: slice 0 = hi >> 21 two's complement, the others 7-bit).
__device__ __forceinline__ void q56_floor(double x, int e, int& hi, unsigned& lo) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int E = (int)((bits >> 52) & 0x7FF);
  long long q = 0;
  if (E != 0) {
    const unsigned long long M = (bits & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull;
    const int k = E - 1019 - e;
    const unsigned long long mag = k >= 0 ? (M << k) : (k > -64 ? (M >> (-k)) : 0ull);
    q = (bits >> 63) ? -(long long)mag : (long long)mag;
  }
  hi = (int)(q >> 28);
  lo = (unsigned)q & 0x0FFFFFFFu;
}
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ void words8_floor(const double (&x)[4], int e, uint32_t (&w)[8]) {
  int h[4];
  unsigned l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) q56_floor(x[i], e, h[i], l[i]);
  constexpr uint32_t m7 = 0x7F7F7F7Fu;
  w[0] = pack4(h[0] >> 21, h[1] >> 21, h[2] >> 21, h[3] >> 21);
  w[1] = pack4(h[0] >> 14, h[1] >> 14, h[2] >> 14, h[3] >> 14) & m7;
  w[2] = pack4(h[0] >> 7, h[1] >> 7, h[2] >> 7, h[3] >> 7) & m7;
  w[3] = pack4(h[0], h[1], h[2], h[3]) & m7;
  w[4] = pack4(l[0] >> 21, l[1] >> 21, l[2] >> 21, l[3] >> 21);
  w[5] = pack4(l[0] >> 14, l[1] >> 14, l[2] >> 14, l[3] >> 14) & m7;
  w[6] = pack4(l[0] >> 7, l[1] >> 7, l[2] >> 7, l[3] >> 7) & m7;
  w[7] = pack4(l[0], l[1], l[2], l[3]) & m7;
}

// Same digits as words8_floor, fewer instructions (rows_slice_kernel):
// q = trunc(x 2^(56-e)) from one exact power-of-two scaling and a truncating
// conversion (|q| < 2^56), its eight base-128 digits spread into the bytes
// of one 64-bit word in three mask/shift steps (byte j = bits 7j..7j+6 of q;
// the top byte also takes the sign bit, i.e. the signed digit q >> 49), and
// four values' words transposed into the eight slice words with byte
// permutes.  s2p = {2^a, 2^b}, a + b = 56 - e, both finite (see pow2_split).
__device__ __forceinline__ unsigned long long spread56(long long q) {
  unsigned long long x = (unsigned long long)q;
  x = (x & 0x000000000FFFFFFFull) | ((x << 4) & 0x0FFFFFFF00000000ull);  // 28 | 28
  x = (x & 0x00003FFF00003FFFull) | ((x << 2) & 0x3FFF00003FFF0000ull);  // 14 x 4
  x = (x & 0x007F007F007F007Full) | ((x << 1) & 0x7F007F007F007F00ull);  // 7 x 8
  return x | ((unsigned long long)q & 0x8000000000000000ull);            // signed top digit
}
__device__ __forceinline__ void transpose4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t& w_b3,
                                           uint32_t& w_b2, uint32_t& w_b1, uint32_t& w_b0) {
  const uint32_t u0 = __byte_perm(a0, a1, 0x5140), u1 = __byte_perm(a0, a1, 0x7362);
  const uint32_t u2 = __byte_perm(a2, a3, 0x5140), u3 = __byte_perm(a2, a3, 0x7362);
  w_b0 = __byte_perm(u0, u2, 0x5410);  // byte 0 of each value
  w_b1 = __byte_perm(u0, u2, 0x7632);
  w_b2 = __byte_perm(u1, u3, 0x5410);
  w_b3 = __byte_perm(u1, u3, 0x7632);
}
// {2^a, 2^b} with a + b = 56 - e and each factor a finite normal double
__device__ __forceinline__ double2 pow2_split(int e) {
  int t = 56 - e;
  const int a = t > 1000 ? 1000 : (t < -1000 ? -1000 : t);
  const int b = t - a;  // |b| <= 1074 + 56 - 1000: finite and normal
  return make_double2(__longlong_as_double((long long)(a + 1023) << 52), __longlong_as_double((long long)(b + 1023) << 52));
}
// FAST: the row exponent is e >= -940, so 2^(56-e) is one finite factor
// (s2p.y == 1) and a subnormal x scales to |q| < 2^(56-e-1022) < 1, i.e.
// truncates to 0 exactly as q56_floor gives -- no per-value checks.
template <bool FAST = false>
__device__ __forceinline__ void words8_fast(const double (&x)[4], double2 s2p, uint32_t (&w)[8]) {
  unsigned long long d[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    long long q;
    if (FAST) {
      q = __double2ll_rz(__dmul_rn(x[i], s2p.x));
    } else {
      // subnormal inputs give q = 0, as q56_floor (which decodes normal numbers only)
      q = fabs(x[i]) < 2.2250738585072014e-308 ? 0ll : __double2ll_rz(__dmul_rn(__dmul_rn(x[i], s2p.x), s2p.y));
    }
    d[i] = spread56(q);
  }
  // slice s word = digit s of the four values; digit s sits in byte 7 - s
  transpose4((uint32_t)(d[0] >> 32), (uint32_t)(d[1] >> 32), (uint32_t)(d[2] >> 32), (uint32_t)(d[3] >> 32),
             w[0], w[1], w[2], w[3]);
  transpose4((uint32_t)d[0], (uint32_t)d[1], (uint32_t)d[2], (uint32_t)d[3], w[4], w[5], w[6], w[7]);
}

}  // namespace oz
}  // namespace cgl
