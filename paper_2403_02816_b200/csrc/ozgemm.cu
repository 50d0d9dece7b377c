// FP64-accurate complex GEMM emulated on the INT8 tensor cores (tcgen05
// kind::i8, TMEM accumulators) by exponent-aligned splitting (Ozaki scheme I).
//
// Why: B200's FP64 tensor path is warp-level DMMA at 37 TFLOP/s; the INT8
// tcgen05 path is ~4.5 POPS dense.  A double with 53 mantissa bits is split
// into S int8 "slices" of 7 bits each relative to a power-of-two scale shared
// by its row (A operand) or column (B operand); slice products are exact in
// INT32, and the products of slice pairs whose weights 2^-7(s+t) are below
// 2^-7(S+1) are dropped.  For S = 8 the dropped/truncated terms are below
// 2^-56 of (row max x column max) per product term, i.e. FP64-level error for
// the dense exp(tau A) factors of the mu-mode products.
//
// Complex -> real: the complex product C = A B (M x K times K x N) is the
// real product of
//   Ahat (2M x 2K): row 2i = [.., Re a_ik, -Im a_ik, ..], row 2i+1 = [.., Im a_ik, Re a_ik, ..]
//   Bhat (2K x N):  row 2k = Re b_k., row 2k+1 = Im b_k.
// so Chat row 2i = Re c_i., row 2i+1 = Im c_i.  Bhat is stored transposed
// (N x 2K, K-major) as UMMA wants both operands K-major.
//
// Operand slices are written by the slicing kernels directly in the UMMA
// canonical no-swizzle K-major layout, tile by tile: a (rows x KC bytes) tile
// is a grid of 8-row x 16-byte core matrices, [row group][k group][8][16], so
// every pipeline stage is a handful of contiguous 1D bulk copies
// (cp.async.bulk + mbarrier complete_tx) -- no tensor maps.
//
// GEMM kernel (one 128 x BN output tile of Chat per CTA, 6 warps):
//   warp 0: producer -- per K chunk, S slices of A and S of B into a stage
//   warp 1: MMA issuer -- for every slice pair (s, t) with s + t <= S + 1,
//           tcgen05.mma into the TMEM accumulator of level d = s + t
//           (S levels x BN int32 columns = 512 columns for S = 8, BN = 64);
//           the B slices of one A slice are issued as ONE wide MMA (N up to
//           256) because their levels are consecutive -- this keeps the SMEM
//           operand reads under the 128 B/clk port (ncu: the narrow-MMA
//           version was bound by sm__mem_tensor_cycles at 93 %)
//   warps 2-5: epilogue -- per level, tcgen05.ld the int32 accumulator, add
//           2^-7d * D_d in FP64, scale by 2^(e_row + e_col), write complex C.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <climits>
#include <cooperative_groups.h>

#include "cgl_common.cuh"
#include "cgl_internal.h"
#include "oz_slice.cuh"
#include "rows_slice.cuh"

namespace cgl {
namespace oz {

constexpr int BM = kOzBM;  // UMMA M (rows of Chat per CTA)

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}
// wait with back-off for roles that do not need sub-100 ns wake-up (keeps
// spinning warps off the shared-memory port the tensor core reads from)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity));
    if (done) return;
    __nanosleep(ns);
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols));
}

// no-swizzle K-major smem descriptor: LBO = K-direction core stride, SBO = 8-row group stride
__device__ __forceinline__ uint64_t make_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  const uint32_t a = smem_u32(smem);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0 (SWIZZLE_NONE)
  return d;
}

// instruction descriptor: kind::i8, s8 x s8 -> s32, both K-major, M x N
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (2u << 4)                       // c_format = S32
         | (1u << 7) | (1u << 10)         // a/b format = signed int8
         | ((uint32_t)(N >> 3) << 17)     // n_dim
         | ((uint32_t)(M >> 4) << 24);    // m_dim
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
// lane predicate of one elected lane (all lanes call; compute once per loop)
__device__ __forceinline__ uint32_t elect_lane() {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, e;\n\t}\n"
      : "=r"(r));
  return r;
}
// all lanes execute with identical operands; the lane with leader != 0 issues
__device__ __forceinline__ void mma_i8_lead(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(leader));
}
__device__ __forceinline__ void mma_commit_lead(uint64_t* bar, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %1, 0;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(bar)), "r"(leader)
      : "memory");
}
// warp-uniform issue: every lane executes the call with identical operands and
// one elected lane issues (keeps descriptors warp-uniform, no per-MMA
// R2UR/ELECT loop around the instruction)
__device__ __forceinline__ void mma_i8_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc));
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

#define LD32x32b_X32(r, taddr)                                                                              \
  asm volatile(                                                                                             \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"      \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                       \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),           \
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),         \
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),         \
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                              \
      : "r"(taddr))

#define ST32x32b_X32(taddr, r)                                                                              \
  asm volatile(                                                                                             \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),                    \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),   \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),       \
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),      \
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))

// 2^e as a double for any frexp exponent (normal range by bit construction,
// subnormal results via one extra exact scaling)
__device__ __forceinline__ double pow2(int e) {
  if (e >= -1022 && e <= 1023) return __longlong_as_double((long long)(e + 1023) << 52);
  if (e > 1023) return __longlong_as_double(0x7ff0000000000000ll);
  return __longlong_as_double((long long)(e + 64 + 1023) << 52) * 5.421010862427522e-20;  // * 2^-64
}

#define LD32x32b_X16(r, taddr)                                                                              \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15])                                                                                     \
               : "r"(taddr))
#define ST32x32b_X16(taddr, r)                                                                              \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),        \
               "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),        \
               "r"(r[15]))

#define LD32x32b_X8(r, taddr)                                                                               \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"                     \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])  \
               : "r"(taddr))
#define ST32x32b_X8(taddr, r)                                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),       \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]))

template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t (&r)[N], uint32_t taddr) {
  static_assert(N == 8 || N == 16, "8 or 16 columns");
  if constexpr (N == 16) LD32x32b_X16(r, taddr); else LD32x32b_X8(r, taddr);
}
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t (&r)[N]) {
  static_assert(N == 8 || N == 16, "8 or 16 columns");
  if constexpr (N == 16) ST32x32b_X16(taddr, r); else ST32x32b_X8(taddr, r);
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

struct SliceArgs {
  const double2* srcs[8];  // per item (blockIdx.z = item * batch + b)
  int8_t* outs[8];
  int* expss[8];
  const double2* src;   // complex matrix Z, element (r, c) at src[r*sr + c*sc]
  int64_t sr, sc;
  int64_t rows, cols;   // complex extents (rows of Z -> operand rows, cols -> K)
  int a_mode;           // 1: A operand (2 real rows per complex row: [re,-im],[im,re]); 0: B operand ([re, im])
  int S;
  int RT;               // row tile (128 for A, BN for B)
  int nchunks;          // K chunks per row tile (2*cols padded to KC)
  int64_t cols_items;   // number of items (grid.z = items * batch)
  int floor_digits;     // 1: floor digits (dense data operand), 0: sign-magnitude (constant operand)
  int64_t rtiles;       // row tiles
  int8_t* out;          // S * rtiles * nchunks * RT * KC bytes
  int* exps;            // per complex row: scale exponent e (values scaled by 2^-e)
};

// ---- coalesced two-pass slicing (used for the per-product data operand) ------
// pass 1: per-row exponent e (max over the row's K entries, |x| 2^-e < 1).
// Rows-contiguous inputs (the transposed data operand of the left form):
// blocks of 32 rows x 8 column groups, each block covering a column range,
// combined with an integer atomicMax (the frexp exponent is monotone in the
// max); exps must be pre-set to a very negative value (0x80 bytes).
__global__ void rowexp_rows_kernel(const SliceArgs a, int64_t sc, int64_t rows, int64_t cols, int64_t batch,
                                   int64_t src_bs, int64_t exp_bs, int64_t cspan) {
  CGL_PROF_SCOPE(KID_ROWEXP);
  __shared__ double red[8][33];
  const int64_t b = blockIdx.z % batch;
  const int item = (int)(blockIdx.z / batch);
  const double2* z = a.srcs[item] + b * src_bs;
  int* exps = a.expss[item];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + tx;
  const int64_t c0 = (int64_t)blockIdx.y * cspan, c1 = c0 + cspan < cols ? c0 + cspan : cols;
  double m = 0.0;
  if (r < rows) {
#pragma unroll 4
    for (int64_t c = c0 + ty; c < c1; c += 8) {
      const double2 v = z[r + c * sc];
      // fmax drops a NaN operand: test both parts explicitly so a NaN sticks
      const bool nan_v = v.x != v.x || v.y != v.y;
      const double av = fmax(fabs(v.x), fabs(v.y));
      m = (nan_v || m != m) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(m, av);
    }
  }
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && r < rows) {
    bool bad = !(m == m) || isinf(m);
    for (int k = 1; k < 8; ++k) {
      const double o = red[k][tx];
      bad |= !(o == o) || isinf(o);
      m = fmax(m, o);
    }
    if (bad) {
      atomicMax(exps + b * exp_bs + r, NONFINITE);
    } else if (m > 0.0) {
      int e;
      frexp(m, &e);
      atomicMax(exps + b * exp_bs + r, e);
    }
  }
}

// K-contiguous rows: warp per row
__global__ void rowexp_kernel(const SliceArgs a, int64_t sr, int64_t sc, int64_t rows, int64_t cols, int64_t batch,
                              int64_t src_bs, int64_t exp_bs) {
  CGL_PROF_SCOPE(KID_ROWEXP);
  const int64_t b = blockIdx.y % batch;
  const int item = (int)(blockIdx.y / batch);
  const double2* z = a.srcs[item] + b * src_bs;
  int* exps = a.expss[item];
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  double m = 0.0;
  bool bad = false;
  for (int64_t c = lane; c < cols; c += 32) {
    const double2 v = z[r * sr + c * sc];
    bad |= !isfinite(v.x) || !isfinite(v.y);
    m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  bad = __any_sync(0xffffffffu, bad);
  int e = 0;
  if (m > 0.0) frexp(m, &e);
  if (lane == 0) exps[b * exp_bs + r] = bad ? NONFINITE : e;
}

// pass 2: one CTA per (row tile, CPB consecutive K chunks, item x batch).
// The Z block is staged through shared memory with loads coalesced along
// whichever of r / c is contiguous; each value is scaled ONCE to a 56-bit
// integer q = trunc(x 2^(56-e)) (exact power-of-two scale, truncation toward
// zero = the Ozaki digit truncation) and its S base-128 digits are peeled
// off with integer shifts (sign applied to every digit).
constexpr int CPB = 4;  // K chunks per CTA

__device__ __forceinline__ void digits8(double x, int e, uint32_t (&w)[8][4], int byte) {
  const double sc = __longlong_as_double((long long)(56 - e + 1023) << 52);  // 2^(56-e), e in (-966, 1079)
  long long q = (long long)(x * sc);                                         // |q| < 2^56
  const bool neg = q < 0;
  unsigned long long m = neg ? (unsigned long long)(-q) : (unsigned long long)q;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int d = (int)((m >> (7 * (7 - s))) & 127ull);
    const uint32_t v = (uint32_t)(uint8_t)(int8_t)(neg ? -d : d);
    w[s][byte >> 2] |= v << (8 * (byte & 3));
  }
}

// Floor ("two's complement") digits for the per-product data operand: the
// top digit is signed (q >> 49 in [-128, 127]), the others in [0, 127]; the
// slices represent the same truncated integer q, with ~half the instructions
// of the sign-magnitude form and no FP64 conversion (q comes from the IEEE
// bits).  Constant operands keep sign-magnitude digits so their small
// entries leave the leading slices exactly zero (block skipping).
__device__ __forceinline__ void digits8_floor(double x, int e, uint32_t (&w)[8][4], int byte) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int E = (int)((bits >> 52) & 0x7FF);
  long long q = 0;
  if (E != 0) {
    const unsigned long long M = (bits & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull;
    const int k = E - 1019 - e;  // q = M 2^k, |q| < 2^56
    const unsigned long long mag = k >= 0 ? (M << k) : (k > -64 ? (M >> (-k)) : 0ull);
    q = (bits >> 63) ? -(long long)mag : (long long)mag;
  }
  const int hi = (int)(q >> 28);                 // signed, 28 bits of magnitude
  const unsigned lo = (unsigned)q & 0x0FFFFFFFu;  // 28 bits
  const unsigned d[8] = {(unsigned)(hi >> 21), ((unsigned)hi >> 14) & 127u, ((unsigned)hi >> 7) & 127u,
                         (unsigned)hi & 127u, (lo >> 21) & 127u, (lo >> 14) & 127u, (lo >> 7) & 127u, lo & 127u};
  const int word = byte >> 2, sh = 8 * (byte & 3);
#pragma unroll
  for (int s = 0; s < 8; ++s) w[s][word] |= (d[s] & 0xFFu) << sh;
}


// FUSED (data operand, B mode): the CTAs of one row tile form a thread-block
// cluster spanning the whole K range; each reduces its staged block to
// partial row exponents, the cluster combines them through distributed
// shared memory, and every CTA slices its block with the row exponents --
// one launch, the data read from HBM once (replaces rowexp_* + this kernel).
template <int S, int AMODE, int CPBT = CPB, bool FUSED = false>
__global__ void __launch_bounds__(256) slice_tile_kernel(const SliceArgs a, int64_t src_bs, int64_t out_bs,
                                                         int64_t exp_bs) {
  CGL_PROF_SCOPE(KID_SLICE);
  constexpr int CC = KC / 2;              // complex columns per chunk
  constexpr int W = CC * CPBT;            // complex columns per CTA
  constexpr int RT = AMODE ? BM : kOzBN;  // real rows per tile
  constexpr int CR = AMODE ? RT / 2 : RT; // complex rows per tile
  extern __shared__ double2 blk_dyn[];    // [CR][W + 1]
  const int64_t batch = gridDim.z / a.cols_items;
  const int64_t b = blockIdx.z % batch;
  const int item = (int)(blockIdx.z / batch);
  const int rt = blockIdx.x, ch0 = blockIdx.y * CPBT;
  const int64_t r0 = (int64_t)rt * CR, c0 = (int64_t)ch0 * CC;
  const double2* z = a.srcs[item] + b * src_bs;
  const int tid = threadIdx.x;
  const int rows_here = (int)min((int64_t)CR, a.rows - r0), cols_here = (int)min((int64_t)W, a.cols - c0);
  if constexpr (FUSED) pdl_wait();  // launched with launch_k: the data come from the previous kernel
  CGL_PROF_MARK(301);
  // all CR*W/256 loads of a thread are issued before any store to smem (the
  // kernel runs as ~one wave: memory-level parallelism decides its speed)
  static_assert((CR * W) % 256 == 0, "staging tile must be a multiple of the CTA size");
  constexpr int NLD = CR * W / 256;
  double2 v[NLD];
  if (a.sc == 1) {
    const double2* zb = z + r0 * a.sr + c0;
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int i = tid + k * 256, rr = i / W, cc = i % W;  // W, CR are powers of two: shifts
      v[k] = (rr < rows_here && cc < cols_here) ? __ldg(zb + rr * a.sr + cc) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int i = tid + k * 256;
      blk_dyn[(i / W) * (W + 1) + i % W] = v[k];
    }
  } else {
    const double2* zb = z + r0 + c0 * a.sc;  // sr == 1
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int i = tid + k * 256, rr = i % CR, cc = i / CR;
      v[k] = (rr < rows_here && cc < cols_here) ? __ldg(zb + rr + (int64_t)cc * a.sc) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int i = tid + k * 256;
      blk_dyn[(i % CR) * (W + 1) + i / CR] = v[k];
    }
  }
  __syncthreads();
  CGL_PROF_MARK(302);
  if constexpr (FUSED) pdl_trigger();  // inputs staged: the GEMM may start its prologue
  int8_t* outb = a.outs[item] + b * out_bs;
  const int* exps = a.expss[item] + b * exp_bs + r0;
  __shared__ int erow[FUSED ? CR : 1];
  if constexpr (FUSED) {
    static_assert(!AMODE && CR == 32, "fused exponents: data operand, 32-row tiles");
    __shared__ double red[8][33];
    __shared__ int redbad[8][32];
    __shared__ int epart[8][32];  // [cluster rank][row]: partials pushed by every CTA of the cluster
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    {
      const int rr = tid & 31, part = tid >> 5;
      double m = 0.0;
      bool bad = false;
      for (int cc = part; cc < cols_here; cc += 8) {
        const double2 v = blk_dyn[rr * (W + 1) + cc];
        bad |= !isfinite(v.x) || !isfinite(v.y);
        m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
      }
      red[part][rr] = m;
      redbad[part][rr] = bad;
    }
    __syncthreads();
    if (tid < 32) {
      double m = red[0][tid];
      int bad = redbad[0][tid];
      for (int k = 1; k < 8; ++k) {
        m = fmax(m, red[k][tid]);
        bad |= redbad[k][tid];
      }
      int e = INT_MIN;
      if (bad) e = NONFINITE;
      else if (m > 0.0) frexp(m, &e);
      // push this CTA's partial into every peer's slot (DSMEM stores), so after
      // ONE cluster barrier each CTA reads only its own shared memory and may
      // exit without waiting for the others
      const unsigned me = cluster.block_rank(), nb = cluster.num_blocks();
      for (unsigned rk = 0; rk < nb; ++rk) cluster.map_shared_rank(&epart[0][0], rk)[me * 32 + tid] = e;
    }
    cluster.sync();
    CGL_PROF_MARK(303);
    if (tid < 32) {
      int e = INT_MIN;
      for (unsigned rk = 0; rk < cluster.num_blocks(); ++rk) e = max(e, epart[rk][tid]);
      if (e == INT_MIN) e = 0;  // all-zero row (same convention as rowexp_kernel)
      erow[tid] = e;
      if (blockIdx.y == 0 && tid < rows_here) a.expss[item][b * exp_bs + r0 + tid] = e;
    }
    __syncthreads();  // erow visible
  }
  constexpr int nreal = AMODE ? 2 : 1;
  constexpr int NG = KC / 16;               // 16-byte groups per chunk
  constexpr int groups = CPBT * NG;
  // consecutive threads take consecutive REAL rows of one 16-byte group, so the
  // slice stores of a warp fill whole 128-byte lines of the core-matrix layout
  constexpr int nrr = CR * nreal;
  // block base of row tile rt, chunk ch: ((rt * nchunks + ch) * S) * RT * KC
  int8_t* tile_base = outb + (int64_t)rt * a.nchunks * S * (RT * KC);
#pragma unroll 2
  for (int w = tid; w < nrr * groups; w += 256) {
    const int rr_real = w % nrr, gg = w / nrr;
    const int rr = AMODE ? rr_real >> 1 : rr_real, part = AMODE ? rr_real & 1 : 0;
    const int ch = ch0 + gg / NG, g = gg % NG;
    if (rr >= rows_here || ch >= a.nchunks) continue;  // padding stays zero (buffer zeroed once)
    const int e_raw = FUSED ? erow[rr] : exps[rr];
    const bool nonfinite = e_raw == NONFINITE;
    uint32_t wv[8][4];
#pragma unroll
    for (int q = 0; q < 8; ++q) wv[q][0] = wv[q][1] = wv[q][2] = wv[q][3] = 0u;
    if (!nonfinite) {
      const double2* row = blk_dyn + rr * (W + 1) + (gg / NG) * CC + g * 8;
      if (!AMODE && S == 8 && a.floor_digits) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 v0 = row[2 * k], v1 = row[2 * k + 1];
          const double x[4] = {v0.x, v0.y, v1.x, v1.y};
          uint32_t ww[8];
          words8_floor(x, e_raw, ww);
#pragma unroll
          for (int q = 0; q < 8; ++q) wv[q][k] = ww[q];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 v = row[j];
          const double x0 = AMODE ? (part ? v.y : v.x) : v.x;
          const double x1 = AMODE ? (part ? v.x : -v.y) : v.y;
          if (a.floor_digits) {
            digits8_floor(x0, e_raw, wv, 2 * j);
            digits8_floor(x1, e_raw, wv, 2 * j + 1);
          } else {
            digits8(x0, e_raw, wv, 2 * j);
            digits8(x1, e_raw, wv, 2 * j + 1);
          }
        }
      }
    }
    const int R = AMODE ? 2 * rr + part : rr;  // real row within the tile
    int8_t* dst = tile_base + (int64_t)ch * S * (RT * KC) + (((R >> 3) * (KC / 16) + g) * 8 + (R & 7)) * 16;
#pragma unroll
    for (int q = 0; q < S; ++q)
      *reinterpret_cast<uint4*>(dst + q * (RT * KC)) = make_uint4(wv[q][0], wv[q][1], wv[q][2], wv[q][3]);
  }
}

// First non-zero slice (1..S, S+1 = all zero) of every (row tile, K chunk)
// block of a sliced CONSTANT operand.  The exp(f tau A_mu) factors are
// numerically banded, so far from the diagonal whole blocks are zero in all
// S slices (entries below 2^-7S of the row max) and near it the leading
// slices vanish first; the GEMM skips those loads and MMAs exactly.
__global__ void zmap_kernel(const int8_t* sl, int S, int64_t slice_stride, int nchunks, int RT, int64_t nblocks,
                            int8_t* z) {
  CGL_PROF_SCOPE(KID_ZMAP);
  const int64_t blk = blockIdx.x;  // = rt * nchunks + chunk
  if (blk >= nblocks) return;
  const int bytes = RT * KC;
  __shared__ int first;
  if (threadIdx.x == 0) first = S + 1;
  __syncthreads();
  for (int s = 0; s < S; ++s) {
    const uint4* p = reinterpret_cast<const uint4*>(sl + (blk * S + s) * (int64_t)bytes);
    int nz = 0;
    for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) {
      const uint4 v = p[i];
      nz |= (v.x | v.y | v.z | v.w) != 0;
    }
    if (__syncthreads_or(nz)) {
      if (threadIdx.x == 0) first = s + 1;
      break;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) z[blk] = (int8_t)first;
}

// ---- the emulated GEMM --------------------------------------------------------
struct OzItem {
  const int8_t* A;   // A-mode slices (batch stride sAb)
  const int* Ae;     // per complex row exponents (batch stride sAeb)
  const int8_t* B;   // B-mode slices (batch stride sBb)
  const int* Be;     // per complex column exponents (batch stride sBeb)
  double2* C;        // output (batch stride sCb), element (i, j) at i*ldc + j
  const int8_t* Az;  // optional [mtiles][nchunks] first non-zero A slice (constant operand), or null
  const int8_t* Bz;  // optional [ntiles][nchunks] first non-zero B slice, or null
};

struct OzArgs {
  int64_t M, N;           // complex output extents
  int mtiles, ntiles, nchunks;
  int64_t sAb, sAeb, sBb, sBeb, sCb, ldc;
  int64_t batch;
  int trans_c;            // 1: element (i, j) stored at C[j*ldc + i] (Out = In E^T computed as E In^T)
  const cgl_flag_t* flag;
  uint64_t pos;
  long long* trace;  // optional: CTA 0 phase timestamps (globaltimer ns), see OZ_TRACE
  int debug;         // CGL_OZ_DEBUG (timing experiments only; results invalid): 1 skip MMAs, 2 skip copies
  int m_fastest;     // tile order (persistent kernel): 1 = row tiles fastest (large data operands)
  OzItem items[kMaxItems];
};

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define OZ_TRACE(slot) \
  do { if (a.trace && blockIdx.x == 0) a.trace[slot] = gtime(); } while (0)

template <int S, int BN, int STAGES>
struct OzCfg {
  static constexpr int A_BYTES = BM * KC;                  // one slice tile of A per chunk
  static constexpr int B_BYTES = BN * KC;
  static constexpr int STAGE_BYTES = S * (A_BYTES + B_BYTES);
  static constexpr int STG_BYTES = BM * (BN + 1) * 8;       // epilogue staging (reuses the stages)
  static constexpr int BODY = STAGES * STAGE_BYTES > STG_BYTES ? STAGES * STAGE_BYTES : STG_BYTES;
  static constexpr int SMEM = BODY + 256;                    // + barriers / tmem slot
  static constexpr int LEVELS = S;                         // d = 2 .. S+1
  static constexpr uint32_t TMEM_COLS = (S * BN <= 256) ? 256 : 512;
  static_assert(S * BN <= 512, "levels x BN must fit the 512 TMEM columns");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
};

constexpr int OZ_THREADS = 320;  // warp 0 producer, warp 1 MMA issuer, warps 2-9 epilogue

template <int S, int BN, int STAGES>
__global__ void __launch_bounds__(OZ_THREADS, (S * BN <= 256 ? 2 : 1)) ozgemm_kernel(const OzArgs a) {
  CGL_PROF_SCOPE(KID_OZ);
  using Cfg = OzCfg<S, BN, STAGES>;
  if (flag_skip(a.flag, resolve_pos(a.flag, a.pos))) return;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BODY);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // decode (item, batch, tm, tn)
  int64_t bid = blockIdx.x;
  const int tn = (int)(bid % a.ntiles);
  bid /= a.ntiles;
  const int tm = (int)(bid % a.mtiles);
  bid /= a.mtiles;
  const int64_t b = bid % a.batch;
  const int item = (int)(bid / a.batch);
  const OzItem& it = a.items[item];

  if (threadIdx.x == 0) OZ_TRACE(0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp >= 2) {
    // zero all level accumulators so every MMA accumulates (blocks may be skipped);
    // epilogue warp pairs share a TMEM lane quadrant and split the columns
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    uint32_t zr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) zr[j] = 0u;
#pragma unroll 1
    for (int level = 0; level < S; ++level)
      ST32x32b_X16(tmem + (q * 32 << 16) + level * BN + half * (BN / 2), zr);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) OZ_TRACE(1);

  const int nch = a.nchunks;
  if (warp == 0 && lane == 0) {
    // ---- producer ----
    const int8_t* A = it.A + b * a.sAb + (int64_t)tm * nch * S * Cfg::A_BYTES;
    const int8_t* B = it.B + b * a.sBb + (int64_t)tn * nch * S * Cfg::B_BYTES;
    int it_n = 0;
    for (int c = 0; c < nch; ++c) {
      const int za = it.Az ? it.Az[(int64_t)tm * nch + c] : 1;
      const int zb = it.Bz ? it.Bz[(int64_t)tn * nch + c] : 1;
      if (za + zb > S + 1) continue;  // every slice pair of this chunk is zero
      const int st = it_n % STAGES;
      const uint32_t ph = (it_n / STAGES) & 1;
      ++it_n;
      mbar_wait(&empty[st], ph ^ 1);
      if (it_n <= 16) OZ_TRACE(2 + it_n);  // producer: chunk issue times (slots 3..18)
      const int na = S + 2 - zb - za, nb = S + 2 - za - zb;  // A slices za..S+1-zb, B slices zb..S+1-za
      mbar_expect_tx(&full[st], na * Cfg::A_BYTES + nb * Cfg::B_BYTES);
      uint8_t* sa = stage_base + st * Cfg::STAGE_BYTES;
      uint8_t* sb = sa + S * Cfg::A_BYTES;
      // one bulk copy per operand: slices za .. S+1-zb of A, zb .. S+1-za of B
      bulk_g2s(sa + (za - 1) * Cfg::A_BYTES, A + ((int64_t)c * S + (za - 1)) * Cfg::A_BYTES, na * Cfg::A_BYTES,
               &full[st]);
      bulk_g2s(sb + (zb - 1) * Cfg::B_BYTES, B + ((int64_t)c * S + (zb - 1)) * Cfg::B_BYTES, nb * Cfg::B_BYTES,
               &full[st]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    constexpr uint32_t LBO = 128, SBO = (KC / 16) * 128;
    int it_n = 0;
    for (int c = 0; c < nch; ++c) {
      const int za = it.Az ? it.Az[(int64_t)tm * nch + c] : 1;
      const int zb = it.Bz ? it.Bz[(int64_t)tn * nch + c] : 1;
      if (za + zb > S + 1) continue;
      const int st = it_n % STAGES;
      const uint32_t ph = (it_n / STAGES) & 1;
      ++it_n;
      mbar_wait(&full[st], ph);
      tc_fence_after();
      if (it_n <= 16) OZ_TRACE(18 + it_n);  // MMA: chunk data-ready times (slots 19..34)
      const uint8_t* sa = stage_base + st * Cfg::STAGE_BYTES;
      const uint8_t* sb = sa + S * Cfg::A_BYTES;
      // descriptors differ only in the start-address field (16-byte units, no
      // carry below 256 KB): build once per stage, then add byte offsets >> 4
      const uint64_t ad0 = make_desc(sa, LBO, SBO), bd0 = make_desc(sb, LBO, SBO);
      constexpr int PER = 256 / BN;
#pragma unroll
      for (int ks = 0; ks < KC / 32; ++ks) {
        // For slice s of A, the B slices t = zb .. S+1-s are consecutive BN-row
        // blocks of one K-major operand (same SBO), and their products land in
        // consecutive level accumulators s+t-2: one MMA covers up to 256/BN
        // slices (N <= 256), cutting the SMEM reads of A by that factor.
#pragma unroll
        for (int s = 1; s <= S; ++s) {
          if (s < za || s > S + 1 - zb) continue;
          const uint64_t ad = ad0 + (uint64_t)((((s - 1) * Cfg::A_BYTES) + ks * 256) >> 4);
#pragma unroll
          for (int blk = 0; blk < (S + PER - 1) / PER; ++blk) {
            const int t0 = zb + blk * PER;
            if (t0 > S + 1 - s) continue;
            const int cnt = (S + 2 - s - t0) < PER ? (S + 2 - s - t0) : PER;
            const uint64_t bd = bd0 + (uint64_t)((((t0 - 1) * Cfg::B_BYTES) + ks * 256) >> 4);
            const uint32_t idesc = make_idesc(BM, BN) + ((uint32_t)((cnt - 1) * BN) >> 3 << 17);
            mma_i8(tmem + (s + t0 - 2) * BN, ad, bd, idesc, 1u);
          }
        }
      }
      if (it_n <= 8) OZ_TRACE(55 + it_n);   // MMA: chunk issue finished (slots 56..63)
      mma_commit(&empty[st]);  // frees the stage when these MMAs complete
    }
    mma_commit(tfull);
  } else if (warp >= 2) {
    // ---- epilogue: 8 warps, warp pairs share a TMEM lane quadrant (BN/2 columns each) ----
    constexpr int HC = BN / 2;
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int row = q * 32 + lane;  // real row of the tile (2i + part)
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (lane == 0 && warp < 6) OZ_TRACE(48 + (warp - 2));
    // Exact integer recombination of the levels: levels 0..3 (d = 2..5) and
    // 4..S-1 (d = 6..S+1) are folded base-128 into two int64 sums, each below
    // 2^53 in magnitude, so the FP64 result is one rounding of
    // hi 2^-35 + lo 2^-7(S+1) (no per-level int->double conversions).
    long long hi[HC], lo[HC];
#pragma unroll
    for (int j = 0; j < HC; ++j) hi[j] = lo[j] = 0;
#pragma unroll
    for (int level = 0; level < S; level += 2) {
      uint32_t r0[HC], r1[HC];
      LD32x32b_X16(r0, tmem + ((uint32_t)(q * 32) << 16) + level * BN + half * HC);
      if (level + 1 < S) LD32x32b_X16(r1, tmem + ((uint32_t)(q * 32) << 16) + (level + 1) * BN + half * HC);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < HC; ++j) {
        const long long d0 = (long long)(int)r0[j];
        if (level < 4) hi[j] = hi[j] * 128 + d0; else lo[j] = lo[j] * 128 + d0;
        if (level + 1 < S) {
          const long long d1 = (long long)(int)r1[j];
          if (level + 1 < 4) hi[j] = hi[j] * 128 + d1; else lo[j] = lo[j] * 128 + d1;
        }
      }
    }
    // hi carries 4 levels (or S if S < 4): weight of its last level
    constexpr int HL = S < 4 ? S : 4;
    const double whi = pow2(-7 * (HL + 1)), wlo = pow2(-7 * (S + 1));
    double acc[HC];
#pragma unroll
    for (int j = 0; j < HC; ++j) acc[j] = fma((double)hi[j], whi, (double)lo[j] * wlo);
    if (lane == 0 && warp < 6) OZ_TRACE(44 + (warp - 2));
    // exact power-of-two scales: rows from Ae, columns broadcast from smem
    __shared__ double colscale[BN];
    const int ct = threadIdx.x - 64;
    if (ct < BN) {
      const int64_t col = (int64_t)tn * BN + ct;
      const int eb = (col < a.N) ? it.Be[b * a.sBeb + col] : 0;
      colscale[ct] = eb == NONFINITE ? __longlong_as_double(0x7ff8000000000000ll) : pow2(eb);
    }
    asm volatile("bar.sync 1, 256;\n" ::);
    const int64_t R = (int64_t)tm * BM + row;
    const int64_t i = R >> 1;
    const int part = lane & 1;  // 0: Re row, 1: Im row (rows 2i, 2i+1 sit in adjacent lanes)
    const int ea = (i < a.M) ? it.Ae[b * a.sAeb + i] : 0;
    const double rs = ea == NONFINITE ? __longlong_as_double(0x7ff8000000000000ll) : pow2(ea);
    double v[HC];
#pragma unroll
    for (int j = 0; j < HC; ++j) v[j] = (acc[j] * rs) * colscale[half * HC + j];
    // lane pairs swap halves: the Re lane writes columns 0..HC/2-1, the Im lane HC/2..HC-1
    double2 out[HC / 2];
#pragma unroll
    for (int c = 0; c < HC / 2; ++c) {
      const double send = part ? v[c] : v[c + HC / 2];
      const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
      out[c] = part ? make_double2(recv, v[c + HC / 2]) : make_double2(v[c], recv);
    }
    double2* C = it.C + b * a.sCb;
    const int64_t col0 = (int64_t)tn * BN + half * HC + part * (HC / 2);
    if (i < a.M) {
      if (!a.trans_c) {
#pragma unroll
        for (int c = 0; c < HC / 2; ++c)
          if (col0 + c < a.N) C[i * a.ldc + col0 + c] = out[c];
      } else {
#pragma unroll
        for (int c = 0; c < HC / 2; ++c)
          if (col0 + c < a.N) C[(col0 + c) * a.ldc + i] = out[c];
      }
    }
    if (threadIdx.x == 64) OZ_TRACE(41);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) OZ_TRACE(42);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}


// ---- persistent variant -------------------------------------------------------
// One CTA per SM walks tiles t = blockIdx.x, +gridDim.x, ...; the S level
// accumulators are double-buffered in TMEM (2 x S x BN <= 512 columns) so the
// epilogue of tile j (TMEM -> registers -> HBM) overlaps the MMAs of tile
// j+1, and the smem ring keeps streaming across tile boundaries.  Same
// operands, zero maps and arithmetic as ozgemm_kernel (bit-identical).
// warps 0, 10, 11, 12: producers (producer p owns ring stage p: bulk copies
// serialise per issuing warp, ~0.4 us each, so one warp per in-flight stage);
// warp 1: MMA issuer; warps 2-9: epilogue
constexpr int OZP_PRODUCERS = 4;
#ifndef OZP_EPI_GROUPS
#define OZP_EPI_GROUPS 4
#endif
constexpr int OZP_EPI = OZP_EPI_GROUPS;       // epilogue warps per TMEM lane quadrant (column groups)
constexpr int OZP_EPI_WARPS = 4 * OZP_EPI;    // warps 2 .. 2 + OZP_EPI_WARPS - 1
constexpr int OZP_THREADS = 32 * (2 + OZP_EPI_WARPS + OZP_PRODUCERS - 1);

template <int S, int BN, int STAGES>
struct OzPCfg {
  static constexpr int A_BYTES = BM * KC;
  static constexpr int B_BYTES = BN * KC;
  static constexpr int STAGE_BYTES = S * (A_BYTES + B_BYTES);
  static constexpr int BODY = STAGES * STAGE_BYTES;
  static constexpr int NTI = 4;          // tile-info ring slots
  static constexpr int KMAXCH = 256;     // max K chunks per tile (K <= 8192 bytes)
  static constexpr int TINFO = BODY + 256;
  static constexpr int SMEM = TINFO + NTI * (KMAXCH + 1) * 4;
  static constexpr uint32_t ACC_COLS = S * BN;
  static_assert(2 * S * BN <= 512, "two level buffers must fit the 512 TMEM columns");
};

// tile t -> (tn fastest, tm, batch b, item); 32-bit (host checks total < 2^31)
struct TileId {
  int tn, tm, b, item;
};
__device__ __forceinline__ TileId decode_tile(const OzArgs& a, uint32_t t) {
  TileId d;
  const uint32_t nt = (uint32_t)a.ntiles, mt = (uint32_t)a.mtiles, nb = (uint32_t)a.batch;
  uint32_t q2;
  if (a.m_fastest) {
    // tm fastest: the CTAs in flight share few B tiles (read from HBM once,
    // then from L2) -- for products whose data slices do not fit in L2
    const uint32_t q = t / mt;
    d.tm = (int)(t - q * mt);
    q2 = q / nt;
    d.tn = (int)(q - q2 * nt);
  } else {
    const uint32_t q = t / nt;
    d.tn = (int)(t - q * nt);
    q2 = q / mt;
    d.tm = (int)(q - q2 * mt);
  }
  const uint32_t q3 = q2 / nb;
  d.b = (int)(q2 - q3 * nb);
  d.item = (int)q3;
  return d;
}

template <int S, int BN, int STAGES>
__global__ void __launch_bounds__(OZP_THREADS, 1) ozgemm_persistent_kernel(const OzArgs a, int64_t total) {
  CGL_PROF_SCOPE(KID_OZP);
  using Cfg = OzPCfg<S, BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BODY);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2] MMAs of the buffer's tile done
  uint64_t* acc_empty = acc_full + 2;   // [2] epilogue has read (and re-zeroed) the buffer
  uint64_t* ti_full = acc_empty + 2;    // [NTI] live-chunk list of a tile written (producer warp 0)
  uint64_t* ti_empty = ti_full + Cfg::NTI;  // [NTI] list consumed (issuer + producer warps 10-12)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ti_empty + Cfg::NTI);
  // tile-info ring: [slot][0] = live chunk count, [slot][1 + e] = c | za << 16 | zb << 24
  uint32_t* tinfo = reinterpret_cast<uint32_t*>(smem + Cfg::TINFO);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) OZ_TRACE(0);
  // item table in shared memory: a dynamically indexed kernel-parameter load
  // misses the constant cache, and the dependent global loads would stall on it
  __shared__ OzItem sitems[kMaxItems];
  static_assert(kMaxItems <= 32, "one warp writes the item table");
  // warp 0: the first tile's zero-map words (constant factors, read before
  // griddepcontrol.wait as below) are loaded first, their latency hidden
  // behind the barrier init
  int pre_za = S + 1, pre_zb = S + 1;
  if (warp == 0 && (int64_t)blockIdx.x < total && lane < a.nchunks) {
    const TileId td0 = decode_tile(a, blockIdx.x);
    const int8_t* az0 = a.items[td0.item].Az;
    const int8_t* bz0 = a.items[td0.item].Bz;
    pre_za = az0 ? az0[(int64_t)td0.tm * a.nchunks + lane] : 1;
    pre_zb = bz0 ? bz0[(int64_t)td0.tn * a.nchunks + lane] : 1;
  }
  if (warp == 0) {
    // warp 0 (barrier init, then producer 0) never touches TMEM: it starts the first tile's live-chunk list and copies right after the
    // barrier init instead of waiting for the TMEM allocation and zeroing
    // (named barrier 1: warp 0 arrives, the other warps sync)
    if (lane < kMaxItems) sitems[lane] = a.items[lane];
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int s = 0; s < 2; ++s) {
        mbar_init(&acc_full[s], 1);
        mbar_init(&acc_empty[s], OZP_EPI_WARPS);
      }
      for (int s = 0; s < Cfg::NTI; ++s) {
        mbar_init(&ti_full[s], 1);
        mbar_init(&ti_empty[s], OZP_PRODUCERS);  // issuer + the 3 other producer warps
      }
      fence_barrier_init();
    }
    __syncwarp();
    CGL_PROF_MARK(109);  // warp 0: barriers initialised
    asm volatile("bar.arrive 1, %0;\n" ::"n"(OZP_THREADS) : "memory");
  } else {
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    asm volatile("bar.sync 1, %0;\n" ::"n"(OZP_THREADS) : "memory");
    tc_fence_after();
  }
  const uint32_t tmem = warp == 0 ? 0u : *tmem_slot;
  if (warp >= 2 && warp < 2 + OZP_EPI_WARPS) {
    constexpr int HC = BN / OZP_EPI;
    const uint32_t q = warp & 3, grp = (warp - 2) >> 2;
    uint32_t zr[HC];
#pragma unroll
    for (int j = 0; j < HC; ++j) zr[j] = 0u;
#pragma unroll 1
    for (int level = 0; level < 2 * S; ++level) tmem_st_cols<HC>(tmem + (q * 32 << 16) + level * BN + grp * HC, zr);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  // zeroed accumulators -> the issuer's first MMA (warps 1 .. last; not warp 0)
  if (warp != 0) asm volatile("bar.sync 2, %0;\n" ::"n"(OZP_THREADS - 32) : "memory");
  tc_fence_after();
  if (threadIdx.x == 0) OZ_TRACE(1);
  if (warp == 1) CGL_PROF_MARK(101);  // setup done (TMEM ready)
  // Everything above and the first tile's live-chunk list (constant zero maps)
  // overlap the previous kernel's tail under PDL; every role executes
  // griddepcontrol.wait before touching the data operand, its exponents or
  // the divergence key (written by earlier kernels).
  const int nch = a.nchunks;
  const int64_t step = gridDim.x;
  if (warp == 0 || warp >= 2 + OZP_EPI_WARPS) {
    // ---- producers: one ring across all tiles of this CTA.  Producer warp 0
    // first lists the live chunks of each tile (zero maps read 32 chunks per
    // load, ballot) into the tile-info ring; all producer warps and the
    // issuer walk that list.  Producer p issues the copies of the live chunks
    // it_n with it_n % STAGES == p (its own stage: bulk copies serialise per
    // issuing warp). ----
    static_assert(STAGES == OZP_PRODUCERS, "one producer warp per stage");
    const int pw = warp == 0 ? 0 : warp - (1 + OZP_EPI_WARPS);
    const int64_t t_end = (a.debug & 4) ? 0 : total;  // debug 4: producers idle
    int it_n = 0, j = 0;
    bool waited = false, stop = false;
    for (int64_t t = blockIdx.x; t < t_end; t += step, ++j) {
      const TileId td = decode_tile(a, (uint32_t)t);
      const int tn = td.tn, tm = td.tm;
      const int64_t b = td.b;
      const OzItem& it = sitems[td.item];
      const int slot = j % Cfg::NTI;
      uint32_t* list = tinfo + slot * (Cfg::KMAXCH + 1);
      if (pw == 0) {
        mbar_wait(&ti_empty[slot], ((j / Cfg::NTI) & 1) ^ 1);
        const int8_t* az = it.Az ? it.Az + (int64_t)tm * nch : nullptr;
        const int8_t* bz = it.Bz ? it.Bz + (int64_t)tn * nch : nullptr;
        int n = 0;
        for (int c0 = 0; c0 < nch; c0 += 32) {
          int zal = S + 1, zbl = S + 1;
          if (j == 0 && c0 == 0) {
            zal = pre_za;  // prefetched at kernel entry
            zbl = pre_zb;
          } else if (c0 + lane < nch) {
            zal = az ? az[c0 + lane] : 1;
            zbl = bz ? bz[c0 + lane] : 1;
          }
          const bool live_me = zal + zbl <= S + 1;
          const unsigned live = __ballot_sync(0xffffffffu, live_me);
          if (live_me)
            list[1 + n + __popc(live & ((1u << lane) - 1u))] =
                (uint32_t)(c0 + lane) | ((uint32_t)zal << 16) | ((uint32_t)zbl << 24);
          n += __popc(live);
        }
        if (lane == 0) list[0] = (uint32_t)n;
        __syncwarp();
        if (lane == 0) mbar_arrive(&ti_full[slot]);
        if (j == 0) CGL_PROF_MARK(114);  // first live-chunk list built
      } else {
        mbar_wait(&ti_full[slot], (j / Cfg::NTI) & 1);
      }
      const int8_t* A = it.A + b * a.sAb + (int64_t)tm * nch * S * Cfg::A_BYTES;
      const int8_t* B = it.B + b * a.sBb + (int64_t)tn * nch * S * Cfg::B_BYTES;
      const int n = (int)list[0];
      // this warp's chunks are every STAGES-th live chunk of the CTA's sequence
      int e = ((pw - it_n) % STAGES + STAGES) % STAGES;
      for (; e < n; e += STAGES) {
        const uint32_t ent = list[1 + e];
        const int c = (int)(ent & 0xFFFFu), za = (int)((ent >> 16) & 0xFF), zb = (int)(ent >> 24);
        const int itc = it_n + e;
        const int st = itc % STAGES;
        const uint32_t ph = (itc / STAGES) & 1;
        const int na = S + 2 - zb - za;
        uint8_t* sa = stage_base + st * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + S * Cfg::A_BYTES;
        // the constant factor slices (A) do not depend on earlier kernels: the
        // first chunk's A copy is issued before griddepcontrol.wait
        if (lane == 0) {
          mbar_wait_sleep(&empty[st], ph ^ 1, 64);
          if (itc < 8) OZ_TRACE(44 + itc);
          if (a.debug & 2) {
            mbar_arrive(&full[st]);
          } else {
            mbar_expect_tx(&full[st], na * (Cfg::A_BYTES + Cfg::B_BYTES));
            bulk_g2s(sa + (za - 1) * Cfg::A_BYTES, A + ((int64_t)c * S + (za - 1)) * Cfg::A_BYTES,
                     na * Cfg::A_BYTES, &full[st]);
          }
        }
        const bool first = !waited;
        if (first && pw == 0) CGL_PROF_MARK(115);  // first constant-factor copy issued
        if (first) {
          pdl_wait();
          if (pw == 0) CGL_PROF_MARK(107);  // producer: pdl wait passed
          waited = true;
        }
        if (lane == 0 && !(a.debug & 2))
          bulk_g2s(sb + (zb - 1) * Cfg::B_BYTES, B + ((int64_t)c * S + (zb - 1)) * Cfg::B_BYTES,
                   na * Cfg::B_BYTES, &full[st]);
        // the divergence key is read after the first data copy is in flight
        // (one L2 round trip off the critical path); the issuer skips too
        const bool skip = first && flag_skip_at(a.flag, a.pos);
        if (first && pw == 0) CGL_PROF_MARK(108);  // producer: flag read
        __syncwarp();
        if (skip) {  // nobody consumes this stage: let its copies land before the CTA exits
          if (lane == 0) mbar_wait(&full[st], ph);
          __syncwarp();
          stop = true;
          break;
        }
      }
      if (stop) break;
      it_n += n;
      __syncwarp();
      if (pw != 0 && lane == 0) mbar_arrive(&ti_empty[slot]);
    }
    if (!waited) pdl_wait();  // (no chunk issued) keep the PDL contract before exiting
    CGL_PROF_MARK(106);  // producer loop done
  } else if (warp == 1) {
    // ---- MMA issuer: the whole warp runs the (warp-uniform) loop over the
    // tile's live-chunk list; one lane, elected once, issues every tcgen05
    // instruction ----
    constexpr uint32_t LBO = 128, SBO = (KC / 16) * 128;
    constexpr int PER = 256 / BN;
    const uint32_t leader = elect_lane();
    pdl_wait();
    const int64_t total_run = flag_skip_at(a.flag, a.pos) ? 0 : total;
    int it_n = 0, j = 0;
    for (int64_t t = blockIdx.x; t < total_run; t += step, ++j) {
      const int buf = j & 1;
      const int slot = j % Cfg::NTI;
      const uint32_t* list = tinfo + slot * (Cfg::KMAXCH + 1);
      if (!(a.debug & 4)) mbar_wait(&ti_full[slot], (j / Cfg::NTI) & 1);
      const int n = (a.debug & 4) ? 0 : (int)list[0];
      mbar_wait(&acc_empty[buf], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0 && j < 8) OZ_TRACE(3 + j);
      const uint32_t dt = tmem + buf * Cfg::ACC_COLS;
      for (int e = 0; e < n; ++e) {
        const uint32_t ent = list[1 + e];
        const int za = (int)((ent >> 16) & 0xFF), zb = (int)(ent >> 24);
        const int st = it_n % STAGES;
        const uint32_t ph = (it_n / STAGES) & 1;
        mbar_wait(&full[st], ph);  // TMA writes -> MMA reads: ordered by complete_tx
        if (it_n == 0) CGL_PROF_MARK(103);  // first data ready
        if (lane == 0 && it_n < 8) OZ_TRACE(52 + it_n);
        if (!(a.debug & 1)) {
          const uint8_t* sa = stage_base + st * Cfg::STAGE_BYTES;
          const uint64_t ad0 = make_desc(sa, LBO, SBO), bd0 = make_desc(sa + S * Cfg::A_BYTES, LBO, SBO);
          if (zb == 1 && KC == 32 && PER >= S) {
            // dense data operand: for A slice s one MMA covers B slices 1..S+1-s
            // (N = (S+1-s) BN) into levels s-1 .. S-1; offsets are compile-time
#pragma unroll
            for (int s = 1; s <= S; ++s) {
              if (s < za) continue;
              mma_i8_lead(dt + (s - 1) * BN, ad0 + (uint64_t)(((s - 1) * Cfg::A_BYTES) >> 4), bd0,
                          make_idesc(BM, (S + 1 - s) * BN), leader);
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < KC / 32; ++ks) {
#pragma unroll
              for (int s = 1; s <= S; ++s) {
                if (s < za || s > S + 1 - zb) continue;
                const uint64_t ad = ad0 + (uint64_t)((((s - 1) * Cfg::A_BYTES) + ks * 256) >> 4);
#pragma unroll
                for (int blk = 0; blk < (S + PER - 1) / PER; ++blk) {
                  const int t0 = zb + blk * PER;
                  if (t0 > S + 1 - s) continue;
                  const int cnt = (S + 2 - s - t0) < PER ? (S + 2 - s - t0) : PER;
                  const uint64_t bd = bd0 + (uint64_t)((((t0 - 1) * Cfg::B_BYTES) + ks * 256) >> 4);
                  const uint32_t idesc = make_idesc(BM, BN) + ((uint32_t)((cnt - 1) * BN) >> 3 << 17);
                  mma_i8_lead(dt + (s + t0 - 2) * BN, ad, bd, idesc, leader);
                }
              }
            }
          }
        }
        mma_commit_lead(&empty[st], leader);
        if (lane == 0 && it_n < 16) OZ_TRACE(64 + it_n);
        ++it_n;
      }
      mma_commit_lead(&acc_full[buf], leader);
      __syncwarp();
      if (lane == 0 && !(a.debug & 4)) mbar_arrive(&ti_empty[slot]);
      if (lane == 0 && j < 8) OZ_TRACE(11 + j);
      if (lane == 0 && j == 0 && a.trace && blockIdx.x == 0) a.trace[63] = it_n;  // chunks of tile 0
    }
    CGL_PROF_MARK(104);  // all MMAs issued
    pdl_trigger();  // all MMAs issued: only this CTA's epilogue tail remains
  } else if (warp >= 2) {
    // ---- epilogue (OZP_EPI warps per TMEM lane quadrant, HC columns each) ----
    constexpr int HC = BN / OZP_EPI;
    const int q = warp & 3, half = (warp - 2) >> 2;  // half = column group
    const int row = q * 32 + lane;
    const int part = lane & 1;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + half * HC;
    pdl_wait();
    const int64_t total_run = flag_skip_at(a.flag, a.pos) ? 0 : total;
    int j = 0;
    for (int64_t t = blockIdx.x; t < total_run; t += step, ++j) {
      const TileId td = decode_tile(a, (uint32_t)t);
      const int tn = td.tn, tm = td.tm;
      const int64_t b = td.b;
      const OzItem& it = sitems[td.item];
      const int buf = j & 1;
      // exponents do not depend on the MMAs: fetch them before waiting
      // (one column exponent per lane, shared through shuffles below)
      const int64_t R = (int64_t)tm * BM + row;
      const int64_t i = R >> 1;
      const int ea = (i < a.M) ? __ldg(it.Ae + b * a.sAeb + i) : 0;
      const int64_t ccol = (int64_t)tn * BN + lane;
      const int eb_lane = (lane < BN && ccol < a.N) ? __ldg(it.Be + b * a.sBeb + ccol) : 0;
      mbar_wait_sleep(&acc_full[buf], (j >> 1) & 1, 32);
      tc_fence_after();
      if (j < 8 && threadIdx.x == 64) OZ_TRACE(19 + j);
      const uint32_t base = lane_base + buf * Cfg::ACC_COLS;
      long long hi[HC], lo[HC];
#pragma unroll
      for (int k = 0; k < HC; ++k) hi[k] = lo[k] = 0;
#pragma unroll
      for (int level = 0; level < S; level += 2) {
        uint32_t r0[HC], r1[HC];
        tmem_ld_cols<HC>(r0, base + level * BN);
        if (level + 1 < S) tmem_ld_cols<HC>(r1, base + (level + 1) * BN);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < HC; ++k) {
          const long long d0 = (long long)(int)r0[k];
          if (level < 4) hi[k] = hi[k] * 128 + d0; else lo[k] = lo[k] * 128 + d0;
          if (level + 1 < S) {
            const long long d1 = (long long)(int)r1[k];
            if (level + 1 < 4) hi[k] = hi[k] * 128 + d1; else lo[k] = lo[k] * 128 + d1;
          }
        }
      }
      if (j < 2 && threadIdx.x == 64) OZ_TRACE(36 + 3 * j);
      {  // re-zero the buffer for the tile after next, then hand it back to the issuer
        uint32_t zr[HC];
#pragma unroll
        for (int k = 0; k < HC; ++k) zr[k] = 0u;
#pragma unroll
        for (int level = 0; level < S; ++level) tmem_st_cols<HC>(base + level * BN, zr);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
      if (j < 2 && threadIdx.x == 64) OZ_TRACE(37 + 3 * j);
      constexpr int HL = S < 4 ? S : 4;
      const double whi = pow2(-7 * (HL + 1)), wlo = pow2(-7 * (S + 1));
      // value = (hi 2^-35 + lo 2^-7(S+1)) 2^(ea+eb): one rounding in the fma,
      // then one power-of-two scaling -- exact, and the same value as scaling
      // by the row and then the column factor, whenever every exponent of the
      // warp lies in [-450, 500] (no subnormal or overflow possible); one FP64
      // multiply fewer per output (FP64 issue is the epilogue's bottleneck
      // while the next tile's MMAs run).  Otherwise (or NONFINITE exponents:
      // NaN) the general two-step path.
      const int64_t cbase = (int64_t)tn * BN + half * HC;
      static_assert(BN <= 32, "one column exponent per lane");
      double v[HC];
      if (__all_sync(0xffffffffu, ea >= -450 && ea <= 500 && eb_lane >= -450 && eb_lane <= 500)) {
#pragma unroll
        for (int k = 0; k < HC; ++k) {
          const int es = ea + __shfl_sync(0xffffffffu, eb_lane, half * HC + k) + 1023;
          const double x = fma((double)hi[k], whi, (double)lo[k] * wlo);
          v[k] = x * __longlong_as_double((long long)es << 52);
        }
      } else {
        const double rs = pow2(ea);
#pragma unroll
        for (int k = 0; k < HC; ++k) {
          const int eb = __shfl_sync(0xffffffffu, eb_lane, half * HC + k);
          const double x = fma((double)hi[k], whi, (double)lo[k] * wlo);
          const double y = (x * rs) * pow2(eb);
          v[k] = (ea == NONFINITE || eb == NONFINITE) ? __longlong_as_double(0x7ff8000000000000ll) : y;
        }
      }
      if (j < 2 && threadIdx.x == 64) OZ_TRACE(38 + 3 * j);
      double2 out[HC / 2];
#pragma unroll
      for (int c = 0; c < HC / 2; ++c) {
        const double send = part ? v[c] : v[c + HC / 2];
        const double recv = __shfl_xor_sync(0xffffffffu, send, 1);
        out[c] = part ? make_double2(recv, v[c + HC / 2]) : make_double2(v[c], recv);
      }
      double2* C = it.C + b * a.sCb;
      const int64_t col0 = cbase + part * (HC / 2);
      if (i < a.M) {
        if (!a.trans_c) {
#pragma unroll
          for (int c = 0; c < HC / 2; ++c)
            if (col0 + c < a.N) C[i * a.ldc + col0 + c] = out[c];
        } else {
#pragma unroll
          for (int c = 0; c < HC / 2; ++c)
            if (col0 + c < a.N) C[(col0 + c) * a.ldc + i] = out[c];
        }
      }
      if (j < 8 && threadIdx.x == 64) OZ_TRACE(27 + j);
    }
    CGL_PROF_MARK(105);  // epilogue done
  }
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) OZ_TRACE(42);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace oz
}  // namespace cgl

namespace cgl {

long long* g_oz_trace = nullptr;

int oz_slice_multi(cudaStream_t st, int S, int nitems, const double* const* srcs, int64_t sr, int64_t sc,
                   int64_t rows, int64_t cols, int64_t batch, int64_t src_bs, int a_mode, int8_t* const* outs,
                   int64_t out_bs, int* const* exps, int64_t exp_bs, int floor_digits) {
  if (S < 1 || S > 8) return set_error(CGL_EINVAL, "oz_slice: S must be 1..8");
  if (nitems < 1 || nitems > 8) return set_error(CGL_EINVAL, "oz_slice: 1..8 items");
  if (rows <= 0 || cols <= 0 || batch <= 0) return 0;
  const int RT = a_mode ? kOzBM : kOzBN;
  oz::SliceArgs a{};
  for (int f = 0; f < nitems; ++f) {
    a.srcs[f] = reinterpret_cast<const double2*>(srcs[f]);
    a.outs[f] = outs[f];
    a.expss[f] = exps[f];
  }
  a.sr = sr;
  a.sc = sc;
  a.rows = rows;
  a.cols = cols;
  a.a_mode = a_mode;
  a.S = S;
  a.RT = RT;
  a.nchunks = (int)((2 * cols + oz::KC - 1) / oz::KC);
  a.rtiles = ((a_mode ? 2 * rows : rows) + RT - 1) / RT;
  a.cols_items = nitems;
  a.floor_digits = floor_digits;
  const int64_t zdim = batch * nitems;
  if (zdim > 65535) return set_error(CGL_ESHAPE, "oz_slice: batch x items too large");
  // full-K rows kernel (stages.cu rows_slice_kernel: one CTA per QC whole rows, the row
  // exponent a CTA-local reduction) for the data operands of the step plans; everything
  // else (A-role slices of the constant factors, S != 8, K > 2048, doubly strided sources)
  // takes the general two-pass path below.  CGL_OZ_FUSED_SLICE=0 sends every call there
  // (the tests compare the two bit for bit).
  const char* ev_fused = getenv("CGL_OZ_FUSED_SLICE");
  const bool rows_ok = !(ev_fused && ev_fused[0] == '0');
  if (rows_ok && !a_mode && floor_digits && S == 8 && (sr == 1 || sc == 1) && rows_slice_ok(cols, false)) {
    // row r of Z = operand row, K = cols
    return rows_slice_plain(st, nitems, srcs, sr, sc, rows, cols, batch, src_bs, outs, out_bs, exps, exp_bs);
  }
  // pass 1: exponents
  if (sr == 1) {
    for (int f = 0; f < nitems; ++f) {
      cudaError_t e = cudaSuccess;
      if (exp_bs == rows) {
        e = cudaMemsetAsync(exps[f], 0x80, (size_t)batch * rows * sizeof(int), st);
      } else {
        for (int64_t bb = 0; bb < batch && e == cudaSuccess; ++bb)
          e = cudaMemsetAsync(exps[f] + bb * exp_bs, 0x80, (size_t)rows * sizeof(int), st);
      }
      if (e != cudaSuccess) return set_cuda_error(e, "oz_slice memset");
    }
    const int64_t rblk = (rows + 31) / 32;
    int64_t csplit = (4 * 148 + rblk * zdim - 1) / (rblk * zdim);
    if (csplit < 1) csplit = 1;
    if (csplit > (cols + 63) / 64) csplit = (cols + 63) / 64;
    const int64_t cspan = (cols + csplit - 1) / csplit;
    dim3 g1((unsigned)rblk, (unsigned)csplit, (unsigned)zdim);
    oz::rowexp_rows_kernel<<<g1, 256, 0, st>>>(a, sc, rows, cols, batch, src_bs, exp_bs, cspan);
  } else {
    dim3 g1((unsigned)((rows + 7) / 8), (unsigned)zdim);
    oz::rowexp_kernel<<<g1, 256, 0, st>>>(a, sr, sc, rows, cols, batch, src_bs, exp_bs);
  }
  int r = check_launch("oz_rowexp");
  if (r) return r;
  dim3 g2((unsigned)a.rtiles, (unsigned)((a.nchunks + oz::CPB - 1) / oz::CPB), (unsigned)zdim);
  const int CR = a_mode ? RT / 2 : RT;
  const size_t smem = (size_t)CR * (oz::CPB * oz::KC / 2 + 1) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
#define OZ_ATTR(S_, A_) cudaFuncSetAttribute(oz::slice_tile_kernel<S_, A_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)
    OZ_ATTR(8, 0); OZ_ATTR(8, 1); OZ_ATTR(7, 0); OZ_ATTR(7, 1); OZ_ATTR(1, 0); OZ_ATTR(1, 1);
#undef OZ_ATTR
    attr = true;
  }
#define OZ_SLICE(S_) (a_mode ? (oz::slice_tile_kernel<S_, 1><<<g2, 256, smem, st>>>(a, src_bs, out_bs, exp_bs)) \
                             : (oz::slice_tile_kernel<S_, 0><<<g2, 256, smem, st>>>(a, src_bs, out_bs, exp_bs)))
  switch (S) {
    case 7: OZ_SLICE(7); break;
    case 8: OZ_SLICE(8); break;
    default: OZ_SLICE(1); break;
  }
#undef OZ_SLICE
  return check_launch("oz_slice");
}

int oz_slice(cudaStream_t st, int S, const double* src, int64_t sr, int64_t sc, int64_t rows, int64_t cols,
             int64_t batch, int64_t src_bs, int a_mode, int RT, int8_t* out, int64_t out_bs, int* exps, int64_t exp_bs) {
  (void)RT;
  return oz_slice_multi(st, S, 1, &src, sr, sc, rows, cols, batch, src_bs, a_mode, &out, out_bs, &exps, exp_bs, 0);
}

template <int S, int BN, int STAGES>
static int oz_launch_cfg(oz::OzArgs& a, int nitems, cudaStream_t st) {
  using Cfg = oz::OzCfg<S, BN, STAGES>;
  auto kern = oz::ozgemm_kernel<S, BN, STAGES>;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(ozgemm)");
    init = true;
  }
  const int64_t blocks = (int64_t)a.mtiles * a.ntiles * a.batch * nitems;
  if (blocks <= 0) return 0;
  kern<<<(unsigned)blocks, oz::OZ_THREADS, Cfg::SMEM, st>>>(a);
  return check_launch("ozgemm_kernel");
}

template <int S, int BN, int STAGES>
static int oz_launch_persistent(oz::OzArgs& a, int nitems, cudaStream_t st) {
  using Cfg = oz::OzPCfg<S, BN, STAGES>;
  auto kern = oz::ozgemm_persistent_kernel<S, BN, STAGES>;
  static int nsm = 0;
  if (!nsm) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(ozgemm_persistent)");
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const int64_t tiles = (int64_t)a.mtiles * a.ntiles * a.batch * nitems;
  if (tiles <= 0) return 0;
  if (tiles >= (1ll << 31)) return set_error(CGL_ESHAPE, "oz_gemm: more than 2^31 tiles in one launch");
  const int64_t grid = tiles < nsm ? tiles : nsm;
  cudaError_t e = launch_k(kern, dim3((unsigned)grid), dim3(oz::OZP_THREADS), Cfg::SMEM, st, dim3(1), a, tiles);
  if (e != cudaSuccess) return set_cuda_error(e, "ozgemm_persistent launch");
  return check_launch("ozgemm_persistent_kernel");
}

static int oz_args(oz::OzArgs& a, cudaStream_t st, int S, int64_t M, int64_t N, int64_t K, int nitems,
                   const int8_t* const* A, const int* const* Ae, const int8_t* const* Az, const int8_t* const* B,
                   const int* const* Be, const int8_t* const* Bz, double* const* C, int64_t ldc, int64_t batch,
                   int64_t sAb, int64_t sAeb, int64_t sBb, int64_t sBeb, int64_t sCb, const cgl_flag_t* flag,
                   uint64_t pos, int trans_c) {
  constexpr int BN = kOzBN;
  (void)S;
  if (nitems < 1 || nitems > kMaxItems) return set_error(CGL_EINVAL, "oz_gemm: 1..8 items");
  a.M = M;
  a.N = N;
  a.mtiles = (int)((2 * M + oz::BM - 1) / oz::BM);
  a.ntiles = (int)((N + BN - 1) / BN);
  a.nchunks = (int)((2 * K + oz::KC - 1) / oz::KC);
  a.sAb = sAb;
  a.sAeb = sAeb;
  a.sBb = sBb;
  a.sBeb = sBeb;
  a.sCb = sCb;
  a.ldc = ldc;
  a.batch = batch;
  a.trans_c = trans_c;
  a.flag = flag;
  a.pos = pos;
  {
    const char* dbg = getenv("CGL_OZ_DEBUG");
    a.debug = dbg ? atoi(dbg) : 0;
  }
  {
    static long long* trace = nullptr;
    const char* e = getenv("CGL_OZ_TRACE");
    if (e && e[0] == '1') {
      if (!trace) cudaMalloc(&trace, 128 * sizeof(long long));
      cudaMemsetAsync(trace, 0, 128 * sizeof(long long), st);
      a.trace = trace;
      g_oz_trace = trace;
    }
  }
  for (int f = 0; f < nitems; ++f)
    a.items[f] = oz::OzItem{A[f], Ae[f], B[f], Be[f], reinterpret_cast<double2*>(C[f]), Az ? Az[f] : nullptr,
                            Bz ? Bz[f] : nullptr};
  // tile order: column tiles fastest.  Row tiles fastest (each B tile fetched from HBM once)
  // was measured on C2/C4 (256^3 / 1024^3 products): no gain (C2 if4 5.82 -> 6.02 ms/step).
  a.m_fastest = 0;
  return 0;
}

int oz_gemm(cudaStream_t st, int S, int64_t M, int64_t N, int64_t K, int nitems, const int8_t* const* A,
            const int* const* Ae, const int8_t* const* Az, const int8_t* const* B, const int* const* Be,
            const int8_t* const* Bz, double* const* C, int64_t ldc, int64_t batch, int64_t sAb, int64_t sAeb,
            int64_t sBb, int64_t sBeb, int64_t sCb, const cgl_flag_t* flag, uint64_t pos, int trans_c) {
  constexpr int BN = kOzBN;
  oz::OzArgs a{};
  int r = oz_args(a, st, S, M, N, K, nitems, A, Ae, Az, B, Be, Bz, C, ldc, batch, sAb, sAeb, sBb, sBeb, sCb, flag,
                  pos, trans_c);
  if (r) return r;
  // persistent TMEM-double-buffered kernel; the one-tile-per-CTA kernel serves S = 7 / 1 and
  // K extents beyond its live-chunk list
  if (S == 8 && a.nchunks <= oz::OzPCfg<8, BN, 4>::KMAXCH) return oz_launch_persistent<8, BN, 4>(a, nitems, st);
  switch (S) {
    case 7: return oz_launch_cfg<7, BN, 2>(a, nitems, st);
    case 8: return oz_launch_cfg<8, BN, 2>(a, nitems, st);
    case 1: return oz_launch_cfg<1, BN, 2>(a, nitems, st);
    default: return set_error(CGL_EINVAL, "oz_gemm: S must be 1, 7 or 8");
  }
}

int oz_zmap(cudaStream_t st, int S, const int8_t* slices, int64_t rows, int64_t cols, int a_mode, int RT, int8_t* z) {
  const int64_t nchunks = (2 * cols + oz::KC - 1) / oz::KC;
  const int64_t rtiles = ((a_mode ? 2 * rows : rows) + RT - 1) / RT;
  const int64_t nblocks = rtiles * nchunks;
  if (nblocks <= 0) return 0;
  oz::zmap_kernel<<<(unsigned)nblocks, 256, 0, st>>>(slices, S, 0, (int)nchunks, RT, nblocks, z);
  return check_launch("oz_zmap");
}

int64_t oz_slice_bytes(int S, int64_t rows, int64_t cols, int a_mode, int RT) {
  const int64_t nchunks = (2 * cols + oz::KC - 1) / oz::KC;
  const int64_t rtiles = ((a_mode ? 2 * rows : rows) + RT - 1) / RT;
  return (int64_t)S * rtiles * nchunks * RT * oz::KC;
}

CGL_PROF_TU(ozgemm)

}  // namespace cgl
