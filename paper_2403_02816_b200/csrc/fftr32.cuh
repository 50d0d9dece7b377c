// 512-point pencils with 32 points per thread: radix-32 x radix-16, ONE
// shared-memory exchange per transform (the radix-8 x 3 plan of fftpass.cuh
// needs two).  The strided two-transform program G (F^-1, g, F along axis 0)
// is bound by the shared-memory data pipe, not by HBM (profiles/
// r02c_fft_passes.txt: LSU 71 % busy at 44 % of the copy bandwidth), and the
// exchanges are most of its LSU traffic; holding 32 points per thread halves
// them at the price of ~200 registers (2 CTAs x 4 warps per SM, the
// independent butterflies of a thread supplying the parallelism).
//
// Thread (pp, t), pp = 0..7 the pencil within a chunk of 8 adjacent pencils
// (one 128-byte line per axis index), t = 0..15: holds x[t + 16 r], r = 0..31.
//   stage 1:  Y[q] = sum_r x[t + 16 r] W_32^(r q)            (in registers)
//   twiddle:  Y[q] *= W_512^(t q)                            (correctly rounded table)
//   exchange: position (q, t) -> thread t' takes q = t', t' + 16 and every t
//   stage 2:  X[q + 32 p] = sum_t Y_t[q] W_16^(t p)          (in registers)
// so thread t' ends with X[t' + 16 r'], r' = s + 2 p: the distribution it
// started with, and F^-1, g, F chain without further exchanges.
#pragma once
#include "fftpass.cuh"

namespace cgl {
namespace fftp {

// cos(pi k / 16), k = 0..8, correctly rounded
__host__ __device__ constexpr double cos16(int k) {
  return k == 0 ? 1.0
       : k == 1 ? 0.98078528040323044913
       : k == 2 ? 0.92387953251128675613
       : k == 3 ? 0.83146961230254523708
       : k == 4 ? 0.70710678118654752440
       : k == 5 ? 0.55557023301960222474
       : k == 6 ? 0.38268343236508977173
       : k == 7 ? 0.19509032201612826785
                : 0.0;
}
// W_32^e = exp(-2 pi i e / 32): real and imaginary parts (forward sign)
__host__ __device__ constexpr double w32_re(int e) {
  e &= 31;
  const int k = e <= 16 ? e : 32 - e;
  return k <= 8 ? cos16(k) : -cos16(16 - k);
}
__host__ __device__ constexpr double w32_im(int e) {
  e &= 31;
  const int k = e <= 16 ? e : 32 - e;
  const double s = k <= 8 ? cos16(8 - k) : cos16(k - 8);  // sin(pi k / 16)
  return e <= 16 ? -s : s;
}

// a * W_32^E (forward) or its conjugate (inverse), E a compile-time constant
template <int E, bool INV>
__device__ __forceinline__ double2 mulw32(double2 a) {
  constexpr int e = E & 31;
  if constexpr (e == 0) return a;
  else if constexpr (e == 8) return mul_mi(a, INV);
  else if constexpr (e == 16) return make_double2(-a.x, -a.y);
  else if constexpr (e == 24) return mul_mi(a, !INV);
  else {
    constexpr double re = w32_re(e), im = INV ? -w32_im(e) : w32_im(e);
    return cmul(a, make_double2(re, im));
  }
}

template <int J, int M, bool INV>
__device__ __forceinline__ void tw32_row(double2 (&a)[32]) {  // a[J + 8 m] *= W_32^(J m), m = M..3
  if constexpr (M < 4) {
    a[J + 8 * M] = mulw32<J * M, INV>(a[J + 8 * M]);
    tw32_row<J, M + 1, INV>(a);
  }
}
template <int J, bool INV>
__device__ __forceinline__ void tw32_all(double2 (&a)[32]) {
  if constexpr (J < 8) {
    tw32_row<J, 1, INV>(a);
    tw32_all<J + 1, INV>(a);
  }
}

// 32-point DFT in registers: input a[r], r = 0..31; output Y[m + 4 k] in a[k + 8 m]
template <bool INV>
__device__ __forceinline__ void dft32(double2 (&a)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double2 x[4] = {a[j], a[j + 8], a[j + 16], a[j + 24]};
    dft4<INV>(x);
    a[j] = x[0];
    a[j + 8] = x[1];
    a[j + 16] = x[2];
    a[j + 24] = x[3];
  }
  tw32_all<1, INV>(a);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    double2 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = a[8 * m + j];
    dft8<INV>(x);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[8 * m + k] = x[k];
  }
}

template <int J, int M, bool INV>
__device__ __forceinline__ void tw16_row(double2* a) {  // a[J + 4 m] *= W_16^(J m)
  if constexpr (M < 4) {
    a[J + 4 * M] = mulw32<2 * J * M, INV>(a[J + 4 * M]);
    tw16_row<J, M + 1, INV>(a);
  }
}
// 16-point DFT in registers: input a[tt], tt = 0..15; output Z[m + 4 k] in a[k + 4 m]
template <bool INV>
__device__ __forceinline__ void dft16(double2* a) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double2 x[4] = {a[j], a[j + 4], a[j + 8], a[j + 12]};
    dft4<INV>(x);
    a[j] = x[0];
    a[j + 4] = x[1];
    a[j + 8] = x[2];
    a[j + 12] = x[3];
  }
  tw16_row<1, 1, INV>(a);
  tw16_row<2, 1, INV>(a);
  tw16_row<3, 1, INV>(a);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    double2 x[4] = {a[4 * m], a[4 * m + 1], a[4 * m + 2], a[4 * m + 3]};
    dft4<INV>(x);
#pragma unroll
    for (int k = 0; k < 4; ++k) a[4 * m + k] = x[k];
  }
}

// One 512-point transform of the calling thread's pencil: on entry
// v[r] = x[t + 16 r], on exit v[r] = X[t + 16 r].  sm: the chunk's exchange
// buffer [512][8] (conflict-free: a quarter-warp = the 8 pencils of one
// (q, t) position = one 128-byte line); all 128 threads of the chunk call it.
// Exchange slot of position (q, t) of pencil `pp`.  Strided passes (SW = false): the 8
// pencils of a chunk interleaved, [(q, t)][pp]; contiguous passes (SW = true): a pencil
// (= row) owns 512 consecutive slots and t is XOR-swizzled with q, so that both the
// writes (fixed q, t = 0..7 per quarter-warp) and the reads (fixed t, q = 0..7) hit 8
// distinct 16-byte bank groups.
template <bool SW>
__device__ __forceinline__ int r32_slot(int q, int t, int pp) {
  return SW ? pp * 512 + q * 16 + (t ^ (q & 15)) : (q * 16 + t) * 8 + pp;
}

template <bool INV, bool SW = false>
__device__ __forceinline__ void fft512_r32(double2 (&v)[32], int t, int pp, double2* sm) {
  dft32<INV>(v);  // Y[m + 4 k] in v[k + 8 m]
#pragma unroll
  for (int m = 0; m < 4; ++m) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int q = m + 4 * k;
      double2 y = v[k + 8 * m];
      if (q > 0) {
        const double2 w = __ldg(&g_fft_tw512[t * q]);
        y = cmul(y, INV ? make_double2(w.x, -w.y) : w);
      }
      sm[r32_slot<SW>(q, t, pp)] = y;
    }
  }
  if (SW) __syncwarp(); else __syncthreads();  // contiguous: a row's 16 threads share a warp and own their region
  double2 c[32];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
#pragma unroll
    for (int tt = 0; tt < 16; ++tt) c[16 * s + tt] = sm[r32_slot<SW>(t + 16 * s, tt, pp)];
  }
  if (SW) __syncwarp(); else __syncthreads();
  dft16<INV>(c);       // Z_0[m + 4 k] in c[k + 4 m]
  dft16<INV>(c + 16);  // Z_1
#pragma unroll
  for (int s = 0; s < 2; ++s) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[s + 2 * (m + 4 * k)] = c[16 * s + k + 4 * m];
    }
  }
}

// Strided-axis pass with 32 points per thread (L = 512): PLAIN (INV selects
// the direction; measured slower than the 8-point kernel, not launched) or G
// (inverse, x scale, g, forward).  One chunk of 8 adjacent pencils per
// 128-thread CTA, 2 CTAs per SM.  Measured and rejected (profiles/
// r02e_fft_r32.txt): 3 CTAs per SM at 168 registers (spills: 1.34 ms), an L2
// prefetch of a later chunk (no change), persistent CTAs with a cp.async
// prefetch buffer and a two-round 32 KB exchange (1.28 ms).
template <int PROG, bool INV>
__global__ void __launch_bounds__(128, 2) fft_r32_kernel(const Args a, const int nchunks) {
  extern __shared__ double2 sm[];
  pdl_wait();
  const uint64_t step = resolve_pos(a.flag, a.pos) >> 24;
  if (a.flag && flag_skip(a.flag, step << 24)) return;
  const int tid = threadIdx.x;
  const int pp = tid & 7, t = tid >> 3;
  const int cpo = (int)a.I / 8;  // chunks per outer index
  const int c = blockIdx.x;
  if (c >= nchunks) return;
  const int o = c / cpo;
  const int gbase = o * 512 * (int)a.I + (c - o * cpo) * 8 + pp + t * (int)a.I;
  const int gstride = 16 * (int)a.I;
  double2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = ldg_s(a.src + gbase + r * gstride);
  if (PROG == FP_PLAIN) {
    fft512_r32<INV>(v, t, pp, sm);
  } else {  // FP_G
    fft512_r32<true>(v, t, pp, sm);
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      V<1> x;
      x.c[0] = cscale(a.scale, v[r]);
      v[r] = gfun<1>(a.nl, x).c[0];
    }
    fft512_r32<false>(v, t, pp, sm);
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) stg_s(a.dst + gbase + r * gstride, v[r]);
  pdl_trigger();
}

// Contiguous-axis two-transform programs with 32 points per thread (L = 512): G (inverse,
// x scale, g, forward: the slab-sharded plan's fused evaluation) and STR_MID (forward, x E1,
// inverse: strang).  8 rows per 128-thread CTA, 16 threads per row; a half-warp reads 256
// contiguous bytes per load.
template <int PROG>
__global__ void __launch_bounds__(128, 2) fft_c32_kernel(const Args a, const int ntiles) {
  extern __shared__ double2 sm[];
  pdl_wait();
  const uint64_t step = resolve_pos(a.flag, a.pos) >> 24;
  if (a.flag && flag_skip(a.flag, step << 24)) return;
  const int tid = threadIdx.x;
  const int t = tid & 15, pp = tid >> 4;
  const int row = blockIdx.x * 8 + pp;
  const bool valid = blockIdx.x < ntiles && row < (int)a.O;
  const int gbase = row * 512 + t;
  double2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = valid ? ldg_s(a.src + gbase + 16 * r) : make_double2(0.0, 0.0);
  if (PROG == FP_G) {
    fft512_r32<true, true>(v, t, pp, sm);
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      V<1> x;
      x.c[0] = cscale(a.scale, v[r]);
      v[r] = gfun<1>(a.nl, x).c[0];
    }
    fft512_r32<false, true>(v, t, pp, sm);
  } else {  // FP_STR_MID
    fft512_r32<false, true>(v, t, pp, sm);
    double2 rf[2];
    rf[1] = valid ? row_factor(a, 1, row) : make_double2(0.0, 0.0);
    rf[0] = rf[1];
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = cmul(efac(a, 1, rf, t + 16 * r), v[r]);
    fft512_r32<true, true>(v, t, pp, sm);
  }
  if (valid) {
#pragma unroll
    for (int r = 0; r < 32; ++r) stg_s(a.dst + gbase + 16 * r, v[r]);
  }
  pdl_trigger();
}

}  // namespace fftp
}  // namespace cgl
