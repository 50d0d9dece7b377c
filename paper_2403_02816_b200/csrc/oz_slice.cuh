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

}  // namespace oz
}  // namespace cgl
