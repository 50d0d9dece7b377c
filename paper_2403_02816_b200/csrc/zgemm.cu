// Complex-FP64 batched GEMM on B200 FP64 tensor cores (DMMA.8x8x4).
//
// This is the mu-mode product engine: np.tensordot -> zgemm in the reference
// (tensors.py:38-59).  On sm_100a FP64 has no tcgen05 path (tcgen05.mma has
// no .kind::f64), so the tensor-core route is warp-level mma.sync
// m8n8k4.f64 (SASS DMMA.8x8x4; measured 37.06 TFLOP/s chip peak, see
// profiles/fp64_peak_r01.txt).  A complex MAC is four real DMMAs:
//     Cr += Ar Br - Ai Bi ,  Ci += Ar Bi + Ai Br    (8 real flops)
// Operands are staged through a multi-stage cp.async pipeline into padded
// shared-memory tiles whose padding makes every 16-byte fragment load
// bank-conflict-free (see the SA/SB derivation below).
//
// Layout (row-major, complex elements):
//   A[m,k] k-contiguous, B[k,n] n-contiguous, C/Y[m,n] n-contiguous.
// Both mode-product forms map onto it: "left" (U_b = M * In_b, A = M) and
// "right" (Out = In * M^T, B = M^T stored explicitly).
#include <cstdint>
#include <cstdio>

#include "cgl_common.cuh"
#include "cgl_internal.h"

namespace cgl {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Shared-memory row strides in 16-byte (complex) units.
//  A fragment (row = lane/4, col k = lane%4): 8 lanes of one 128-bit phase hit
//  (m*SA + k) mod 8 distinct  <=>  SA = 4 (mod 8).
//  B fragment (row k = lane%4, col n = lane/4): (k*SB + n) mod 8 distinct
//  <=>  SB = 2 (mod 8).
template <int BK> struct StrideA { static constexpr int v = BK + 4; };
template <int BN> struct StrideB { static constexpr int v = BN + 2; };

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
struct GemmCfg {
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M;
  static constexpr int WTN = BN / WARPS_N;
  static constexpr int FM = WTM / 8;
  static constexpr int FN = WTN / 8;
  static constexpr int SA = StrideA<BK>::v;
  static constexpr int SB = StrideB<BN>::v;
  static constexpr int A_STAGE = BM * SA;
  static constexpr int B_STAGE = BK * SB;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double2);
  static_assert(BM % (8 * WARPS_M) == 0 && BN % (8 * WARPS_N) == 0, "warp tile");
  static_assert(BK % 8 == 0, "BK multiple of 8");
  static_assert(SA % 8 == 4 && SB % 8 == 2, "conflict-free padding");
};

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    zgemm_kernel(const GemmArgs args) {
  using Cfg = GemmCfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  constexpr int NT = Cfg::NT, FM = Cfg::FM, FN = Cfg::FN, SA = Cfg::SA, SB = Cfg::SB;

  if (flag_skip(args.flag, args.pos)) return;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + STAGES * Cfg::A_STAGE;

  // ---- decode (item, batch, tile) from the linear block index ----
  const int64_t tiles_m = (args.M + BM - 1) / BM;
  const int64_t tiles_n = (args.N + BN - 1) / BN;
  const int64_t tiles = tiles_m * tiles_n;
  int64_t bid = blockIdx.x;
  const int64_t t = bid % tiles;
  bid /= tiles;
  const int64_t b = bid % args.batch;
  const int item = (int)(bid / args.batch);
  int64_t tm, tn;
  if (args.m_fastest) { tm = t % tiles_m; tn = t / tiles_m; }
  else                { tn = t % tiles_n; tm = t / tiles_n; }
  const int64_t m0 = tm * BM, n0 = tn * BN;

  const double2* __restrict__ A = reinterpret_cast<const double2*>(args.items[item].A) + b * args.sA;
  const double2* __restrict__ B = reinterpret_cast<const double2*>(args.items[item].B) + b * args.sB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int64_t M = args.M, N = args.N, K = args.K, lda = args.lda, ldb = args.ldb;
  const int ktiles = (int)((K + BK - 1) / BK);

  auto load_tile = [&](int stage, int kt) {
    const int64_t k0 = (int64_t)kt * BK;
    double2* as = As + stage * Cfg::A_STAGE;
    double2* bs = Bs + stage * Cfg::B_STAGE;
#pragma unroll
    for (int c = tid; c < BM * BK; c += NT) {
      const int r = c / BK, kk = c % BK;
      const int64_t gm = m0 + r, gk = k0 + kk;
      const bool p = gm < M && gk < K;
      cp_async16(as + r * SA + kk, p ? (const void*)(A + gm * lda + gk) : (const void*)A, p);
    }
#pragma unroll
    for (int c = tid; c < BK * BN; c += NT) {
      const int r = c / BN, nn = c % BN;
      const int64_t gk = k0 + r, gn = n0 + nn;
      const bool p = gk < K && gn < N;
      cp_async16(bs + r * SB + nn, p ? (const void*)(B + gk * ldb + gn) : (const void*)B, p);
    }
  };

  double cr[FM][FN][2], ci[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    cp_async_commit();
  }

  const int arow = (wm * Cfg::WTM + (lane >> 2)) * SA + (lane & 3);
  const int bcol = (lane & 3) * SB + wn * Cfg::WTN + (lane >> 2);

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) load_tile(nk % STAGES, nk);
      cp_async_commit();
    }
    const double2* as = As + (kt % STAGES) * Cfg::A_STAGE + arow;
    const double2* bs = Bs + (kt % STAGES) * Cfg::B_STAGE + bcol;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double2 a[FM], bb[FN];
#pragma unroll
      for (int i = 0; i < FM; ++i) a[i] = as[i * 8 * SA + kk * 4];
#pragma unroll
      for (int j = 0; j < FN; ++j) bb[j] = bs[kk * 4 * SB + j * 8];
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const double nai = -a[i].y;
#pragma unroll
        for (int j = 0; j < FN; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], a[i].x, bb[j].x);
          dmma(ci[i][j][0], ci[i][j][1], a[i].x, bb[j].y);
          dmma(ci[i][j][0], ci[i][j][1], a[i].y, bb[j].x);
          dmma(cr[i][j][0], cr[i][j][1], nai, bb[j].y);
        }
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: C = alpha*acc + beta*Y ----
  double2* __restrict__ C = reinterpret_cast<double2*>(args.items[item].C) + b * args.sC;
  const double2* Y = args.items[item].Y ? reinterpret_cast<const double2*>(args.items[item].Y) + b * args.sY : nullptr;
  const double2 al = args.alpha;
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int64_t row = m0 + wm * Cfg::WTM + i * 8 + (lane >> 2);
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < FN; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t col = n0 + wn * Cfg::WTN + j * 8 + (lane & 3) * 2 + e;
        if (col >= N) continue;
        double2 v = make_double2(al.x * cr[i][j][e] - al.y * ci[i][j][e],
                                 al.x * ci[i][j][e] + al.y * cr[i][j][e]);
        if (Y) {
          const double2 y = Y[row * args.ldy + col];
          v.x = fma(args.beta, y.x, v.x);
          v.y = fma(args.beta, y.y, v.y);
        }
        C[row * args.ldc + col] = v;
      }
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int ST>
static int launch_cfg(const GemmArgs& a, int nitems, cudaStream_t s) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, ST>;
  auto kern = zgemm_kernel<BM, BN, BK, WM, WN, ST>;
  static bool attr_done = false;  // per template instance
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(zgemm)");
    attr_done = true;
  }
  const int64_t tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  const int64_t blocks = tiles * a.batch * nitems;
  if (blocks <= 0) return 0;
  if (blocks > 0x7fffffffLL) return set_error(CGL_ESHAPE, "zgemm grid too large");
  kern<<<(unsigned)blocks, Cfg::NT, Cfg::SMEM, s>>>(a);
  return check_launch("zgemm_kernel");
}

// Tile-shape choice: the 64x64 tile (8 warps, 32x16 warp tiles) when it
// yields at least ~one CTA per SM, else the 32x32 tile (4 warps) so small
// grids (128^2 fields) still spread over the 148 SMs.
int zgemm_launch(const GemmArgs& a, int nitems, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return 0;
  const int64_t big = ((a.M + 63) / 64) * ((a.N + 63) / 64) * a.batch * nitems;
  if (big >= 120) return launch_cfg<64, 64, 16, 2, 4, 3>(a, nitems, s);
  return launch_cfg<32, 32, 16, 2, 2, 3>(a, nitems, s);
}

}  // namespace cgl
