// Complex-FP64 batched GEMM on B200 FP64 tensor cores (DMMA.8x8x4).
//
// This is the mu-mode product engine: np.tensordot -> zgemm in the reference
// (tensors.py:38-59).  On sm_100a FP64 has no tcgen05 path (tcgen05.mma has
// no .kind::f64), so the tensor-core route is warp-level mma.sync
// m8n8k4.f64 (SASS DMMA.8x8x4; measured 37.06 TFLOP/s chip peak, see
// profiles/fp64_peak_r01.txt).
//
// Complex product: Gauss/Karatsuba "3M" form, three real DMMAs per complex
// fragment pair instead of four:
//     P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi)
//     Cr = P1 - P2,  Ci = P3 - P1 - P2
// (the operand sums are one DADD per fragment, ~3% of the DMMA issue).
// The algorithmic flop count stays 8 per complex MAC; the executed tensor
// work is 6 — rooflines are reported on the algorithmic count.  The classic
// 4-DMMA form is kept (CGL_ZGEMM_4M=1) for A/B checks.
//
// Decomposition: persistent stream-K.  grid = (#SM x resident CTAs); the
// flattened (tile, k-tile) iteration space is cut into equal contiguous
// ranges, one per CTA, so every SM gets the same MAC count regardless of how
// many 64x64 tiles the problem has (512^2 fields give 64 tiles per field, a
// 0.86-wave grid in the data-parallel form).  A tile split across CTAs is
// finished by its HEAD CTA (the one holding k-tile 0, which reaches the tile
// at the end of its range); the continuing CTAs compute their tail segment
// first and publish it at once (workspace + release/acquire flags), so the
// head finds the partials ready instead of serialising the chain.  The grid
// never exceeds the co-resident CTA count, so every awaited CTA is running.
// The workspace is per device: cgl GEMM launches must be stream-ordered.
//
// Operands are staged through a 3-stage cp.async pipeline into padded
// shared-memory tiles whose padding makes every 16-byte fragment load
// bank-conflict-free (SA/SB derivation below).
//
// Layout (row-major, complex elements):
//   A[m,k] k-contiguous, B[k,n] n-contiguous, C/Y[m,n] n-contiguous.
// Both mode-product forms map onto it: "left" (U_b = M * In_b, A = M) and
// "right" (Out = In * M^T, B = M^T stored explicitly).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <vector>

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

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Shared-memory row strides in 16-byte (complex) units.
//  A fragment (row = lane/4, col k = lane%4): 8 lanes of one 128-bit phase hit
//  (m*SA + k) mod 8 distinct  <=>  SA = 4 (mod 8).
//  B fragment (row k = lane%4, col n = lane/4): (k*SB + n) mod 8 distinct
//  <=>  SB = 2 (mod 8).
template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool M3>
struct GemmCfg {
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M;
  static constexpr int WTN = BN / WARPS_N;
  static constexpr int FM = WTM / 8;
  static constexpr int FN = WTN / 8;
  static constexpr int SA = BK + 4;
  static constexpr int SB = BN + 2;
  static constexpr int A_STAGE = BM * SA;
  static constexpr int B_STAGE = BK * SB;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double2);
  static constexpr int NACC = M3 ? 3 : 2;           // accumulator planes
  static constexpr int PART = FM * FN * 4;          // partial (Cr, Ci) doubles per thread
  static_assert(BM % (8 * WARPS_M) == 0 && BN % (8 * WARPS_N) == 0, "warp tile");
  static_assert(BK % 8 == 0, "BK multiple of 8");
  static_assert(SA % 8 == 4 && SB % 8 == 2, "conflict-free padding");
};

template <class Cfg>
struct Acc {
  double p[Cfg::NACC][Cfg::FM][Cfg::FN][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < Cfg::NACC; ++a)
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) p[a][i][j][0] = p[a][i][j][1] = 0.0;
  }
};

// Accumulate k-tiles [kt0, kt1) of one output tile into acc.
template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool M3, class Cfg>
__device__ __forceinline__ void mainloop(const GemmArgs& args, const double2* __restrict__ A,
                                         const double2* __restrict__ B, int64_t m0, int64_t n0, int kt0, int kt1,
                                         double2* As, double2* Bs, Acc<Cfg>& acc) {
  constexpr int NT = Cfg::NT, FM = Cfg::FM, FN = Cfg::FN, SA = Cfg::SA, SB = Cfg::SB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int64_t M = args.M, N = args.N, K = args.K, lda = args.lda, ldb = args.ldb;

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

  const int nk = kt1 - kt0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_tile(s, kt0 + s);
    cp_async_commit();
  }
  const int arow = (wm * Cfg::WTM + (lane >> 2)) * SA + (lane & 3);
  const int bcol = (lane & 3) * SB + wn * Cfg::WTN + (lane >> 2);

  for (int t = 0; t < nk; ++t) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = t + STAGES - 1;
      if (nt < nk) load_tile(nt % STAGES, kt0 + nt);
      cp_async_commit();
    }
    const double2* as = As + (t % STAGES) * Cfg::A_STAGE + arow;
    const double2* bs = Bs + (t % STAGES) * Cfg::B_STAGE + bcol;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double2 bb[FN];
      double bsum[FN];
#pragma unroll
      for (int j = 0; j < FN; ++j) {
        bb[j] = bs[kk * 4 * SB + j * 8];
        bsum[j] = bb[j].x + bb[j].y;
      }
#pragma unroll
      for (int i = 0; i < FM; ++i) {
        const double2 a = as[i * 8 * SA + kk * 4];
        if (M3) {
          const double asum = a.x + a.y;
#pragma unroll
          for (int j = 0; j < FN; ++j) {
            dmma(acc.p[0][i][j][0], acc.p[0][i][j][1], a.x, bb[j].x);
            dmma(acc.p[1][i][j][0], acc.p[1][i][j][1], a.y, bb[j].y);
            dmma(acc.p[2 % Cfg::NACC][i][j][0], acc.p[2 % Cfg::NACC][i][j][1], asum, bsum[j]);
          }
        } else {
          const double nai = -a.y;
#pragma unroll
          for (int j = 0; j < FN; ++j) {
            dmma(acc.p[0][i][j][0], acc.p[0][i][j][1], a.x, bb[j].x);
            dmma(acc.p[1][i][j][0], acc.p[1][i][j][1], a.x, bb[j].y);
            dmma(acc.p[1][i][j][0], acc.p[1][i][j][1], a.y, bb[j].x);
            dmma(acc.p[0][i][j][0], acc.p[0][i][j][1], nai, bb[j].y);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // the next segment's prologue reuses the stages
}

// Fold the 3M planes into (Cr, Ci) in planes 0 and 1, in place.
template <bool M3, class Cfg>
__device__ __forceinline__ void finalize(Acc<Cfg>& acc) {
  if (!M3) return;
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double p1 = acc.p[0][i][j][e], p2 = acc.p[1][i][j][e], p3 = acc.p[2 % Cfg::NACC][i][j][e];
        acc.p[0][i][j][e] = p1 - p2;
        acc.p[1][i][j][e] = p3 - p1 - p2;
      }
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool M3>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    zgemm_kernel(const GemmArgs args) {
  CGL_PROF_SCOPE(KID_ZGEMM);
  using Cfg = GemmCfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES, M3>;
  constexpr int FM = Cfg::FM, FN = Cfg::FN, NT = Cfg::NT;

  if (flag_skip(args.flag, resolve_pos(args.flag, args.pos))) return;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + STAGES * Cfg::A_STAGE;

  const int64_t tiles_m = (args.M + BM - 1) / BM;
  const int64_t tiles_n = (args.N + BN - 1) / BN;
  const int64_t tiles = tiles_m * tiles_n;
  const int ktiles = max(1, (int)((args.K + BK - 1) / BK));  // K = 0: one zero-filled k-tile
  const int64_t total = args.total_iters;  // (nitems * batch * tiles) * ktiles
  const int64_t G = gridDim.x, g = blockIdx.x;
  const int64_t it_end = (g + 1) * total / G;
  int64_t it = g * total / G;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;

  while (it < it_end) {
    const int64_t tile_id = it / ktiles;
    const int kt0 = (int)(it % ktiles);
    const int64_t rem = it_end - it;
    const int kt1 = (int)((int64_t)kt0 + rem < (int64_t)ktiles ? (int64_t)kt0 + rem : (int64_t)ktiles);
    // decode (item, batch, tile)
    int64_t r = tile_id;
    const int64_t t = r % tiles;
    r /= tiles;
    const int64_t b = r % args.batch;
    const int item = (int)(r / args.batch);
    int64_t tm, tn;
    if (args.m_fastest) { tm = t % tiles_m; tn = t / tiles_m; }
    else                { tn = t % tiles_n; tm = t / tiles_n; }
    const int64_t m0 = tm * BM, n0 = tn * BN;
    const double2* A = reinterpret_cast<const double2*>(args.items[item].A) + b * args.sA;
    const double2* B = reinterpret_cast<const double2*>(args.items[item].B) + b * args.sB;

    Acc<Cfg> acc;
    acc.zero();
    mainloop<BM, BN, BK, WARPS_M, WARPS_N, STAGES, M3, Cfg>(args, A, B, m0, n0, kt0, kt1, As, Bs, acc);
    finalize<M3, Cfg>(acc);
    it += kt1 - kt0;

    if (kt0 > 0) {
      // This segment continues a tile begun by a lower CTA; it is the first
      // thing this CTA computes, so publish it right away.  The tile's head
      // CTA (which reaches the tile at the END of its range) finishes it.
      double* ws = args.workspace + (size_t)g * Cfg::PART * NT;
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = ((i * FN + j) * 2 + e) * 2;
            __stcg(ws + (size_t)q * NT + tid, acc.p[0][i][j][e]);
            __stcg(ws + (size_t)(q + 1) * NT + tid, acc.p[1][i][j][e]);
          }
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release(args.flags + g, args.epoch);
      continue;
    }
    if (kt1 < ktiles) {
      // head segment at the end of this CTA's range: add the tail partials
      // that the following CTAs published at the start of theirs
      const int64_t tile_end = (tile_id + 1) * ktiles;
      for (int64_t h = g + 1; h < G; ++h) {
        if (tid == 0) {
          while (ld_acquire(args.flags + h) != args.epoch) __nanosleep(20);
        }
        __syncthreads();
        const double* wh = args.workspace + (size_t)h * Cfg::PART * NT;
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int q = ((i * FN + j) * 2 + e) * 2;
              acc.p[0][i][j][e] += __ldcg(wh + (size_t)q * NT + tid);
              acc.p[1][i][j][e] += __ldcg(wh + (size_t)(q + 1) * NT + tid);
            }
        __syncthreads();
        if (tid == 0) args.flags[h] = 0;  // single consumer: re-arm for the next launch (graph-replay safe)
        if ((h + 1) * total / G >= tile_end) break;  // CTA h holds the tile's last k-tile
      }
    }

    // epilogue: C = alpha*acc + beta*Y
    double2* __restrict__ C = reinterpret_cast<double2*>(args.items[item].C) + b * args.sC;
    const double2* Y = args.items[item].Y ? reinterpret_cast<const double2*>(args.items[item].Y) + b * args.sY : nullptr;
    const double2 al = args.alpha;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int64_t row = m0 + wm * Cfg::WTM + i * 8 + (lane >> 2);
      if (row >= args.M) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = n0 + wn * Cfg::WTN + j * 8 + (lane & 3) * 2 + e;
          if (col >= args.N) continue;
          const double2 a = make_double2(acc.p[0][i][j][e], acc.p[1][i][j][e]);
          double2 v = make_double2(al.x * a.x - al.y * a.y, al.x * a.y + al.y * a.x);
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
}

// ---------------------------------------------------------------------------
// host side: per-device persistent workspace + flags, grid sizing
// ---------------------------------------------------------------------------
// Stream-K partials + per-CTA flags, one state per device (GEMM launches are
// stream-ordered: the library enqueues every product of a plan on one stream;
// two DMMA products running concurrently on two streams would share the flags
// and are not supported).  Buffers only grow, and a buffer that is
// outgrown is RETIRED, never freed: CUDA graphs captured earlier (the fused step
// plans) bake its pointers and may be replayed at any later time, so freeing it
// would let a replay write into memory torch has reused.  The leak is
// bounded by the geometric growth (x1.5) of the largest configuration used.
struct StreamKState {
  double* ws = nullptr;
  int* flags = nullptr;
  size_t ws_doubles = 0;
  int nflags = 0;
};
static StreamKState g_sk[64];
static std::vector<void*> g_sk_retired;  // kept alive for graphs that captured them
static std::mutex g_sk_mu;

static int ensure_state(int dev, cudaStream_t stream, size_t ws_doubles, int nflags, StreamKState* out) {
  std::lock_guard<std::mutex> lock(g_sk_mu);
  StreamKState& s = g_sk[dev & 63];
  if (s.ws_doubles < ws_doubles) {
    const size_t want = std::max(ws_doubles, s.ws_doubles + s.ws_doubles / 2);
    double* p = nullptr;
    cudaError_t e = cudaMalloc(&p, want * sizeof(double));
    if (e != cudaSuccess) return set_cuda_error(e, "zgemm workspace");
    if (s.ws) g_sk_retired.push_back(s.ws);
    s.ws = p;
    s.ws_doubles = want;
  }
  if (s.nflags < nflags) {
    const int want = std::max(nflags, s.nflags + s.nflags / 2);
    int* p = nullptr;
    cudaError_t e = cudaMalloc(&p, want * sizeof(int));
    // flags are consumed and re-armed to 0 inside the kernel; a fresh buffer
    // starts armed.  The memset is ordered before the launch on `stream`.
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, want * sizeof(int), stream);
    if (e != cudaSuccess) return set_cuda_error(e, "zgemm flags");
    if (s.flags) g_sk_retired.push_back(s.flags);
    s.flags = p;
    s.nflags = want;
  }
  *out = s;
  return 0;
}

static bool use_4m() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CGL_ZGEMM_4M");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <int BM, int BN, int BK, int WM, int WN, int ST, bool M3>
static int launch_cfg(GemmArgs a, int nitems, cudaStream_t s) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, ST, M3>;
  auto kern = zgemm_kernel<BM, BN, BK, WM, WN, ST, M3>;
  static int occ = 0, sms = 0, dev_cached = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (occ == 0 || dev != dev_cached) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(zgemm)");
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::NT, Cfg::SMEM);
    if (e != cudaSuccess || occ < 1) return set_cuda_error(e, "zgemm occupancy");
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dev_cached = dev;
  }
  const int64_t tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  const int64_t ktiles = a.K > 0 ? (a.K + BK - 1) / BK : 1;  // K = 0: one zero-filled k-tile
  const int64_t units = tiles * a.batch * nitems;
  if (units <= 0) return 0;
  a.total_iters = units * ktiles;
  int64_t G = (int64_t)sms * occ;
  if (G > a.total_iters) G = a.total_iters;
  StreamKState st;
  int r = ensure_state(dev, s, (size_t)G * Cfg::PART * Cfg::NT, (int)G, &st);
  if (r) return r;
  a.workspace = st.ws;
  a.flags = st.flags;
  a.epoch = 1;  // flags are re-armed to 0 by their consumer, so a constant works under graph replay
  kern<<<(unsigned)G, Cfg::NT, Cfg::SMEM, s>>>(a);
  return check_launch("zgemm_kernel");
}

static int env_cfg() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("CGL_ZGEMM_CFG");
    v = e ? atoi(e) : -1;
  }
  return v;
}

template <bool M3>
static int launch_big(const GemmArgs& a, int nitems, cudaStream_t s, int cfg) {
  switch (cfg) {
    case 1: return launch_cfg<64, 32, 16, 4, 2, 3, M3>(a, nitems, s);   // 16x16 warp tiles, 8 warps
    case 2: return launch_cfg<64, 64, 16, 4, 4, 3, M3>(a, nitems, s);   // 16x16 warp tiles, 16 warps
    case 3: return launch_cfg<32, 64, 16, 2, 4, 3, M3>(a, nitems, s);   // 16x16 warp tiles, 8 warps
    case 4: return launch_cfg<64, 32, 32, 4, 2, 3, M3>(a, nitems, s);   // BK = 32
    case 0: return launch_cfg<64, 64, 16, 2, 4, 3, M3>(a, nitems, s);   // 32x16 warp tiles, 8 warps
    case 6: return launch_cfg<128, 64, 32, 4, 2, 2, M3>(a, nitems, s);  // 32x32 warp tiles, 8 warps
    case 7: return launch_cfg<64, 64, 48, 4, 4, 2, M3>(a, nitems, s);   // BK = 48, 16 warps
    case 5: return launch_cfg<64, 64, 32, 4, 4, 2, M3>(a, nitems, s);   // 16x16 warp tiles, 16 warps
    case 9: return launch_cfg<32, 64, 32, 2, 4, 3, M3>(a, nitems, s);   // 16x16, 8 warps, 3 stages
    // default (measured best on B200, profiles/r01_zgemm_configs.txt): 64x128 CTA
    // tile, 8 warps of 32x32, BK = 32, double-buffered, 1 CTA/SM (207 KB smem)
    default: return launch_cfg<64, 128, 32, 2, 4, 2, M3>(a, nitems, s);
  }
}

// Tile-shape choice: the 64x64 tile for real work; the 32x32 tile (4 warps)
// when a problem has too few 64x64 tiles to occupy the SMs without splitting
// every tile many ways.
int zgemm_launch(const GemmArgs& a, int nitems, cudaStream_t s) {
  if (a.M <= 0 || a.N <= 0) return 0;
  const int64_t big = ((a.M + 63) / 64) * ((a.N + 63) / 64) * a.batch * nitems;
  const bool m3 = !use_4m();
  if (big >= 32) return m3 ? launch_big<true>(a, nitems, s, env_cfg()) : launch_big<false>(a, nitems, s, env_cfg());
  return m3 ? launch_cfg<32, 32, 16, 2, 2, 3, true>(a, nitems, s)
            : launch_cfg<32, 32, 16, 2, 2, 3, false>(a, nitems, s);
}

CGL_PROF_TU(zgemm)

}  // namespace cgl
