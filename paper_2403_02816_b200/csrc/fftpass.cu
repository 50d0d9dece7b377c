// Pencil-FFT passes for the periodic (Fourier pseudospectral) path, sm_100a.
//
// The reference transforms with numpy's pocketfft (spectral.py:79-86,
// `np.fft.fftn` / `ifftn`) around every pointwise nonlinear evaluation
// (integrators.py:99-120: Problem.g / Problem.flow on a Fourier operator
// are F g F^-1).  A 3D transform of a 512^3 complex128 field cannot be done in
// one HBM pass (a pencil plane is 4 MiB; an SM holds 227 KB), so it is three
// passes, one per axis.  What this file adds over a library FFT is FUSION:
// every pointwise piece of the time step rides inside the first or last pass
// whose data is already in registers:
//   * F g F^-1 of a stage input: the inverse pass along the slowest axis,
//     the 1/N scale, g(.) and the forward pass along the same axis are ONE
//     kernel (the inverse's last radix stage leaves each thread holding
//     exactly the elements the forward's first stage reads);
//   * the Lawson stage combinations (integrators.py:205-215) and the
//     separable exp(f tau symbol) multipliers run between the forward pass of
//     g_i and the inverse pass of the next stage input along the contiguous
//     axis (one kernel: forward -> g_i -> stage -> inverse); the combination
//     u' = E1 (u + t/6 g1) + t/3 E1/2 (g2 + g3) + t/6 g4 accumulates term by
//     term in one field, so a stage reads at most one extra operand;
//   * strang: the end-of-step flow, the finiteness check, the next step's
//     first flow and the forward pass share one kernel along the slowest axis
//     (for the exact cubic flow the two flows are evaluated as one, STR_A0F);
//     E1 rides between the forward and inverse passes of the contiguous axis.
// Per-pass layout:
//   contiguous axis (stride 1): a CTA owns 4096/L whole rows; thread t of a
//     row holds elements t + (L/8) r, r = 0..7; the exchange buffer uses the
//     128-byte XOR swizzle (conflict-free for every radix-8 stage pattern);
//   strided axis (stride I, I % 8 == 0): a CTA owns 512/L chunks of 8
//     adjacent pencils (one 128-byte line per axis index); the 8 threads of a
//     quarter-warp are the 8 pencils of a chunk, so global accesses are whole
//     128-byte lines and the exchange buffer [i][8] is conflict-free.
// Transform: Stockham autosort, radix-8 stages (+ one radix-2/4 stage last
// for L = 2^(3a+1), 2^(3a+2)); every stage reads x[t + (L/8) r], so the
// first stage loads straight from HBM and the last stores straight to HBM;
// two shared-memory exchanges per 512-point pencil.  Twiddles come from one
// correctly rounded 512-entry table (fft_twiddles.h).  Unnormalised both
// ways (the 1/N of ifftn is applied by the program that consumes the inverse).
// The two-transform programs at 512 points (G; STR_MID) are bound by the
// shared-memory data pipe: they run with 32 points per thread, radix-32 x
// radix-16 and ONE exchange per transform (fftr32.cuh).
#include "fftpass.cuh"
#include "fftr32.cuh"

namespace cgl {
namespace fftp {

template <int L, bool CONTIG, int PROG, bool INV, int NT>
__global__ void __launch_bounds__(NT, Occ<PROG, NT, CONTIG>::MINB) fft_pass_kernel(const Args a, const int ntiles) {
  using GE = Geo<L, CONTIG, NT>;
  constexpr int T = GE::T;
  constexpr int NAUX = Aux<PROG>::N;
  extern __shared__ double2 sm[];
  pdl_wait();
  pdl_trigger();
  const uint64_t step = resolve_pos(a.flag, a.pos) >> 24;
  int first = 0;
  if (PROG == FP_STR_A0) first = a.fw;
  if (a.flag && flag_skip(a.flag, (step << 24) | ((uint64_t)first << 8))) return;

  const int tid = threadIdx.x;
  const TileMap<L, CONTIG, NT> map(tid);
  const int t = map.t;
  Lay<L, CONTIG> lay;
  lay.base = map.lay_base();
  lay.cw = CONTIG ? 0 : GE::CW;
  constexpr bool RING = CONTIG;                // strided passes: one tile per CTA, loads straight to registers
  double2* ring[2] = {sm, sm + GE::TILE};
  // per-stage twiddles: staged in shared memory by the persistent (contiguous)
  // CTAs; one-tile strided CTAs read the global table through L1
  double2* tws = sm + (RING ? 2 : 1) * GE::TILE;
  const double2* tw = RING ? tws : g_fft_stage_tw + fft_stage_tw_offset(L);
  double2* aux = tws + (RING ? 512 : 0);       // stage operands of the current tile: [k][r][NT]
  const double2* src = (PROG == FP_IF4_START || PROG == FP_STR_START) ? a.u : a.src;
  uint64_t key = ~0ull;
  const double tau = a.tau;
  const uint64_t check_pos = (step << 24) | (255ull << 8);

  auto issue = [&](int tile, double2* buf) {
    if (!RING) return;
    int gb, gs, rw;
    if (tile < ntiles && map.geo(a, tile, gb, gs, rw)) {
#pragma unroll
      for (int r = 0; r < 8; ++r) cp_async16(buf + lay.at(t + T * r), src + gb + (t + T * r) * gs);
    }
    cp_async_commit();
  };
  // strided passes (one tile per CTA): the tile's loads go out before the
  // twiddle tables are staged, so their latency overlaps the staging
  double2 v[8];
  if (!RING) {
    int gb, gs, rw;
    const bool ok = map.geo(a, blockIdx.x, gb, gs, rw);
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = ok ? ldg_s(src + gb + (t + T * r) * gs) : make_double2(0.0, 0.0);
  }
  issue(blockIdx.x, ring[0]);
  if (RING) {
    stage_twiddles<L>(tws, tid, NT);
    __syncthreads();
  }

  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    double2* sbuf = ring[it & 1];
    int gbase, gstride, row;
    const bool valid = map.geo(a, tile, gbase, gstride, row);
    if (NAUX > 0 && valid) {
      // pointwise operands, needed after the first transform (committed before
      // the next tile's prefetch so that wait_group 1 covers them)
#pragma unroll
      for (int r = 0; r < 8; ++r) cp_async16(aux + r * NT + tid, a.u + gbase + (t + T * r));
      // B2 / B3: the running combination is read straight from global memory after the
      // forward transform; pull its lines into L2 now
      if (PROG == FP_IF4_B2 || PROG == FP_IF4_B3) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
          asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.g[0] + gbase + (t + T * r)));
      }
    }
    cp_async_commit();
    issue(tile + (int)gridDim.x, ring[(it + 1) & 1]);
    if (RING) {
      cp_async_wait<2>();  // this tile's main operand (the two newer groups may still fly)
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = valid ? sbuf[lay.at(t + T * r)] : make_double2(0.0, 0.0);
      pencil_sync<L, CONTIG>(lay);  // the pencil's threads hold their inputs: its buffer becomes the exchange buffer
    }
    if (PROG == FP_STR_START) {
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = cscale(a.scale, v[r]);
    }
    bool store = true;
    if (PROG == FP_PLAIN) {
      fft_pencil<L, CONTIG, INV>(v, t, sbuf, lay, tw);
    } else if (PROG == FP_IF4_START) {
      fft_pencil<L, CONTIG, true>(v, t, sbuf, lay, tw);
    } else if (PROG == FP_G) {
      fft_pencil<L, CONTIG, true>(v, t, sbuf, lay, tw);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        V<1> x;
        x.c[0] = cscale(a.scale, v[r]);
        v[r] = gfun<1>(a.nl, x).c[0];
      }
      pencil_sync<L, CONTIG>(lay);
      fft_pencil<L, CONTIG, false>(v, t, sbuf, lay, tw);
    } else if (PROG == FP_IF4_B1 || PROG == FP_IF4_B2 || PROG == FP_IF4_B3 || PROG == FP_IF4_B4) {
      if constexpr (CONTIG) store = contig_program<L, PROG, NT>(v, a, valid, row, gbase, t, tid, aux, sbuf, lay, tw, key, check_pos);
    } else if (PROG == FP_STR_START) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        V<1> x;
        x.c[0] = v[r];
        v[r] = flow<1>(a.nl, x, 0.5 * tau, step, 0, key).c[0];
      }
      fft_pencil<L, CONTIG, false>(v, t, sbuf, lay, tw);
    } else if (PROG == FP_STR_A0) {
      fft_pencil<L, CONTIG, true>(v, t, sbuf, lay, tw);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        V<1> x;
        x.c[0] = cscale(a.scale, v[r]);
        const double2 out = flow<1>(a.nl, x, 0.5 * tau, step, a.fw, key).c[0];
        if (!cfinite(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        if (valid) stg_s(a.u_out + gbase + (t + T * r) * gstride, out);
        x.c[0] = out;
        v[r] = flow<1>(a.nl, x, 0.5 * tau, step + 1, 0, key).c[0];
      }
      if (a.dst == nullptr) {
        store = false;
      } else {
        __syncthreads();
        fft_pencil<L, CONTIG, false>(v, t, sbuf, lay, tw);
      }
    } else if (PROG == FP_STR_MID) {
      if constexpr (CONTIG) store = contig_program<L, PROG, NT>(v, a, valid, row, gbase, t, tid, aux, sbuf, lay, tw, key, check_pos);
    }
    if (valid && store) {
#pragma unroll
      for (int r = 0; r < 8; ++r) stg_s(a.dst + gbase + (t + T * r) * gstride, v[r]);
    }
    if (!valid) key = ~0ull;
    pencil_sync<L, CONTIG>(lay);  // the pencil's exchange reads are done before its buffer is refilled
  }
  cp_async_wait<0>();
  if (PROG == FP_IF4_B4 || PROG == FP_STR_START || PROG == FP_STR_A0) raise_min(a.flag, key);
}

// Strided-axis pass: one tile (G chunks of CW adjacent pencils) per CTA,
// straight-line -- loads go to registers first, the per-stage twiddles come
// from the global table through L1, the tile buffer is the exchange buffer.
// (A persistent ring does not pay here: the 64-byte chunks at an 8 KB / 4 MB
// stride are DRAM-activation-bound, and the ring's registers cost occupancy.)
template <int L, int PROG, bool INV, int NT>
__global__ void __launch_bounds__(NT, Occ<PROG, NT, false>::MINB) fft_strided_kernel(const Args a, const int ntiles) {
  using GE = Geo<L, false, NT>;
  constexpr int T = GE::T;
  extern __shared__ double2 sm[];
  // dependents are released only when this CTA is done: with tens of
  // thousands of CTAs an early trigger would let the next grid's waiting CTAs
  // take the slots this grid's remaining CTAs need
  pdl_wait();
  const uint64_t step = resolve_pos(a.flag, a.pos) >> 24;
  if (a.flag && flag_skip(a.flag, (step << 24) | ((uint64_t)((PROG == FP_STR_A0 || PROG == FP_STR_A0F) ? a.fw : 0) << 8)))
    return;
  const int tid = threadIdx.x;
  const TileMap<L, false, NT> map(tid);
  const int t = map.t;
  Lay<L, false> lay;
  lay.base = map.lay_base();
  lay.cw = GE::CW;
  const double2* tw = g_fft_stage_tw + fft_stage_tw_offset(L);
  int gbase, gstride, row;
  const bool valid = map.geo(a, blockIdx.x, gbase, gstride, row);
  const double2* src = PROG == FP_STR_START ? a.u : a.src;
  double2 v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) v[r] = valid ? ldg_s(src + gbase + (t + T * r) * gstride) : make_double2(0.0, 0.0);
  uint64_t key = ~0ull;
  const double tau = a.tau;
  if (PROG == FP_PLAIN) {
    fft_pencil<L, false, INV>(v, t, sm, lay, tw);
  } else if (PROG == FP_G) {
    fft_pencil<L, false, true>(v, t, sm, lay, tw);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      V<1> x;
      x.c[0] = cscale(a.scale, v[r]);
      v[r] = gfun<1>(a.nl, x).c[0];
    }
    __syncthreads();
    fft_pencil<L, false, false>(v, t, sm, lay, tw);
  } else if (PROG == FP_STR_START) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      V<1> x;
      x.c[0] = cscale(a.scale, v[r]);
      v[r] = flow<1>(a.nl, x, 0.5 * tau, step, 0, key).c[0];
    }
    fft_pencil<L, false, false>(v, t, sm, lay, tw);
  } else if (PROG == FP_STR_A0) {
    const uint64_t check_pos = (step << 24) | (255ull << 8);
    fft_pencil<L, false, true>(v, t, sm, lay, tw);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      V<1> x;
      x.c[0] = cscale(a.scale, v[r]);
      const double2 out = flow<1>(a.nl, x, 0.5 * tau, step, a.fw, key).c[0];
      if (!cfinite(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      if (valid) stg_s(a.u_out + gbase + (t + T * r) * gstride, out);
      x.c[0] = out;
      v[r] = flow<1>(a.nl, x, 0.5 * tau, step + 1, 0, key).c[0];
    }
    if (a.dst == nullptr) {
      raise_min(a.flag, valid ? key : ~0ull);
      pdl_trigger();
      return;
    }
    __syncthreads();
    fft_pencil<L, false, false>(v, t, sm, lay, tw);
  } else if (PROG == FP_STR_A0F) {
    fft_pencil<L, false, true>(v, t, sm, lay, tw);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double2 w = cscale(a.scale, v[r]);
      if (valid) stg_s(a.u_out + gbase + (t + T * r) * gstride, w);
      v[r] = cubic_boundary(a.nl, w, 0.5 * tau, step, a.fw, key);
    }
    if (a.dst == nullptr) {
      raise_min(a.flag, valid ? key : ~0ull);
      pdl_trigger();
      return;
    }
    __syncthreads();
    fft_pencil<L, false, false>(v, t, sm, lay, tw);
  }
  if (valid) {
#pragma unroll
    for (int r = 0; r < 8; ++r) stg_s(a.dst + gbase + (t + T * r) * gstride, v[r]);
  }
  if (PROG == FP_STR_START || PROG == FP_STR_A0 || PROG == FP_STR_A0F) raise_min(a.flag, valid ? key : ~0ull);
  pdl_trigger();
}

// Threads per CTA, chosen by same-box A/B at 512^3 (tools/fft_probe.py,
// profiles/r02_fft_passes.txt):
//  * contiguous ring: 256 (92% of HBM; 77% at 512);
//  * strided 512-point passes: 512, so a chunk is 8 pencils = one 128-byte
//    line per axis index (plain 81% / 76% on axes 1 / 0 vs 72% / 46% with
//    64-byte chunks at 256); the fused g pass at 2 CTAs x 64 registers
//    (1.50 ms, vs 1.63 at 1 CTA and 1.67 at 256 threads);
//  * strided strang flow passes: 256 x 3 CTAs (3.67 ms vs 4.64 at 512): the
//    two exact flows per point are FP64-latency-bound and want warps more
//    than 128-byte chunks.
static int threads_for(int L, bool contig, int prog) {
  if (prog == FP_STR_A0 || prog == FP_STR_A0F || prog == FP_STR_START) return 256;
  return (!contig && L == 512) ? 512 : 256;
}

template <int L, bool CONTIG, int PROG, bool INV, int NT>
static int launch_nt(const Args& a, cudaStream_t st) {
  using GE = Geo<L, CONTIG, NT>;
  void (*kern)(const Args, const int);
  if constexpr (CONTIG) kern = fft_pass_kernel<L, true, PROG, INV, NT>;
  else kern = fft_strided_kernel<L, PROG, INV, NT>;
  static int blocks_per_sm = 0, sms = 0;
  const int smem = CONTIG ? (2 * GE::TILE + 512 + Aux<PROG>::N * 8 * NT) * (int)sizeof(double2)
                          : GE::TILE * (int)sizeof(double2);
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, NT, smem);
    if (e != cudaSuccess || blocks_per_sm < 1) return set_cuda_error(e, "fft_pass occupancy");
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t tiles = CONTIG ? (a.O + GE::ROWS - 1) / GE::ROWS : ((a.O * (a.I / GE::CW)) + GE::G - 1) / GE::G;
  if (tiles <= 0) return 0;
  // contiguous passes: persistent CTAs over the tile ring; strided passes: one tile per CTA
  int64_t grid = CONTIG ? (int64_t)sms * blocks_per_sm : tiles;
  if (grid > tiles) grid = tiles;
  cudaError_t e = launch_k(kern, dim3((unsigned)grid), dim3(NT), (size_t)smem, st, dim3(1), a, tiles);
  if (e != cudaSuccess) return set_cuda_error(e, "fft_pass launch");
  return check_launch("fft_pass_kernel");
}

// 32 points per thread (fftr32.cuh): the 512-point strided G pass, one chunk per CTA
template <int PROG, bool INV>
static int launch_r32(const Args& a, cudaStream_t st) {
  auto kern = fft_r32_kernel<PROG, INV>;
  const int smem = 4096 * (int)sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "fft_r32 attribute");
    attr = true;
  }
  const int64_t chunks = a.O * (a.I / 8);
  if (chunks <= 0) return 0;
  cudaError_t e = launch_k(kern, dim3((unsigned)chunks), dim3(128), (size_t)smem, st, dim3(1), a, (int)chunks);
  if (e != cudaSuccess) return set_cuda_error(e, "fft_r32 launch");
  return check_launch("fft_r32_kernel");
}

template <int PROG>
static int launch_c32(const Args& a, cudaStream_t st) {
  auto kern = fft_c32_kernel<PROG>;
  const int smem = 4096 * (int)sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "fft_c32 attribute");
    attr = true;
  }
  const int64_t tiles = (a.O + 7) / 8;
  if (tiles <= 0) return 0;
  cudaError_t e = launch_k(kern, dim3((unsigned)tiles), dim3(128), (size_t)smem, st, dim3(1), a, (int)tiles);
  if (e != cudaSuccess) return set_cuda_error(e, "fft_c32 launch");
  return check_launch("fft_c32_kernel");
}

template <int L, bool CONTIG, int PROG, bool INV>
static int launch_one(const Args& a, cudaStream_t st) {
  // two-transform programs at 512 points: 32 points per thread, one exchange per transform
  // (contiguous: STR_MID 1131 vs 1413 us with the radix-8 ring kernel, profiles/r02j_fft_probe.txt)
  if constexpr (L == 512 && CONTIG && (PROG == FP_G || PROG == FP_STR_MID)) return launch_c32<PROG>(a, st);
  // the two-transform G pass is bound by the shared-memory data pipe: 32 points per thread
  // (one exchange per transform) take 1.15 ms at 512^3 against 1.50 ms for the radix-8 plan;
  // the single-transform passes are HBM/latency-bound and keep the 8-point kernel (0.76-0.87
  // vs 0.85-1.0 ms), profiles/r02e_fft_r32.txt
  if constexpr (L == 512 && !CONTIG && PROG == FP_G) return launch_r32<PROG, INV>(a, st);
  if constexpr (L == 512 && !CONTIG) {
    if (threads_for(L, CONTIG, PROG) == 512) return launch_nt<L, CONTIG, PROG, INV, 512>(a, st);
  }
  return launch_nt<L, CONTIG, PROG, INV, 256>(a, st);
}

template <int L>
static int launch_L(int prog, bool contig, bool inv, const Args& a, cudaStream_t st) {
  if (contig) {
    switch (prog) {
      case FP_PLAIN: return inv ? launch_one<L, true, FP_PLAIN, true>(a, st) : launch_one<L, true, FP_PLAIN, false>(a, st);
      case FP_IF4_START: return launch_one<L, true, FP_IF4_START, true>(a, st);
      case FP_IF4_B1: return launch_one<L, true, FP_IF4_B1, false>(a, st);
      case FP_IF4_B2: return launch_one<L, true, FP_IF4_B2, false>(a, st);
      case FP_IF4_B3: return launch_one<L, true, FP_IF4_B3, false>(a, st);
      case FP_IF4_B4: return launch_one<L, true, FP_IF4_B4, false>(a, st);
      case FP_G: return launch_one<L, true, FP_G, false>(a, st);
      case FP_STR_MID: return launch_one<L, true, FP_STR_MID, false>(a, st);
      default: return set_error(CGL_EINVAL, "fft_pass: program needs a strided axis");
    }
  }
  switch (prog) {
    case FP_PLAIN: return inv ? launch_one<L, false, FP_PLAIN, true>(a, st) : launch_one<L, false, FP_PLAIN, false>(a, st);
    case FP_G: return launch_one<L, false, FP_G, false>(a, st);
    case FP_STR_START: return launch_one<L, false, FP_STR_START, false>(a, st);
    case FP_STR_A0: return launch_one<L, false, FP_STR_A0, false>(a, st);
    case FP_STR_A0F: return launch_one<L, false, FP_STR_A0F, false>(a, st);
    default: return set_error(CGL_EINVAL, "fft_pass: program needs the contiguous axis");
  }
}

}  // namespace fftp

bool fft_pass_supported(int ndim, const int64_t* shape) {
  if (ndim < 2 || ndim > 3) return false;
  for (int d = 0; d < ndim; ++d) {
    const int64_t n = shape[d];
    if (n < 16 || n > 512 || (n & (n - 1))) return false;
  }
  return true;
}

int fft_pass_launch(cudaStream_t st, int program, int ndim, const int64_t* shape, int axis, int inverse,
                    const double* src, double* dst, const cgl_fft_ops_t* ops) {
  using namespace fftp;
  if (program < 0 || program >= FP_NPROG) return set_error(CGL_EINVAL, "fft_pass: unknown program");
  if (!fft_pass_supported(ndim, shape)) return set_error(CGL_ESHAPE, "fft_pass: 2D/3D, power-of-two extents 16..512");
  if (axis < 0 || axis >= ndim) return set_error(CGL_EINVAL, "fft_pass: bad axis");
  Args a{};
  a.src = reinterpret_cast<const double2*>(src);
  a.dst = reinterpret_cast<double2*>(dst);
  a.O = 1;
  a.I = 1;
  for (int d = 0; d < axis; ++d) a.O *= shape[d];
  for (int d = axis + 1; d < ndim; ++d) a.I *= shape[d];
  const bool contig = axis == ndim - 1;
  const int L = (int)shape[axis];
  a.nd = ndim;
  a.lg1 = 0;
  if (ndim == 3)
    while ((1ll << a.lg1) < shape[1]) ++a.lg1;
  if (ops) {
    a.u = reinterpret_cast<const double2*>(ops->u);
    a.u_out = reinterpret_cast<double2*>(ops->u_out);
    for (int q = 0; q < 3; ++q) a.g[q] = reinterpret_cast<const double2*>(ops->g[q]);
    a.g_out = reinterpret_cast<double2*>(ops->g_out);
    for (int fr = 0; fr < 2; ++fr)
      for (int d = 0; d < ndim; ++d) a.tab[fr][d] = reinterpret_cast<const double2*>(ops->tables[fr][d]);
    a.tau = ops->tau;
    a.scale = ops->scale;
    const cgl_nonlinear_t& nl = ops->nl;
    a.nl = StageNL{nl.alpha3, nl.beta3, nl.alpha4, nl.beta4, nl.alpha5, nl.kind};
    if (nl.kind >= 2) return set_error(CGL_EINVAL, "fft_pass: scalar two-term kinds only");
    a.fw = 1;
    a.flag = ops->flag;
    a.pos = ops->pos;
  } else if (program != FP_PLAIN) {
    return set_error(CGL_EINVAL, "fft_pass: program needs its operands");
  }
  // operand checks per program
  const bool need_src = !(program == FP_IF4_START || program == FP_STR_START);
  if (need_src && !src) return set_error(CGL_EINVAL, "fft_pass: null src");
  const bool dst_optional = program == FP_IF4_B4 || program == FP_STR_A0 || program == FP_STR_A0F;
  if (!dst && !dst_optional) return set_error(CGL_EINVAL, "fft_pass: null dst");
  if ((program >= FP_IF4_START && program <= FP_IF4_B4 || program == FP_STR_START) && !a.u)
    return set_error(CGL_EINVAL, "fft_pass: program needs u");
  if ((program >= FP_IF4_B1 && program <= FP_IF4_B3) && !a.g_out) return set_error(CGL_EINVAL, "fft_pass: needs g_out");
  if ((program == FP_IF4_B2 || program == FP_IF4_B3) && !a.g[0])
    return set_error(CGL_EINVAL, "fft_pass: B2 / B3 need the running combination g[0]");
  if (program == FP_IF4_B4 && !a.u_out) return set_error(CGL_EINVAL, "fft_pass: B4 needs u_out");
  if ((program == FP_STR_A0 || program == FP_STR_A0F) && !a.u_out) return set_error(CGL_EINVAL, "fft_pass: needs u_out");
  if (program == FP_STR_A0F && a.nl.kind != 0) return set_error(CGL_EINVAL, "fft_pass: STR_A0F is for the exact cubic flow");
  if ((program >= FP_IF4_B1 && program <= FP_IF4_B4) || program == FP_STR_MID)
    for (int fr = 0; fr < 2; ++fr)
      for (int d = 0; d < ndim; ++d)
        if (!a.tab[fr][d]) return set_error(CGL_EINVAL, "fft_pass: program needs the exp tables");
  if (!contig && a.I % 8) return set_error(CGL_ESHAPE, "fft_pass: strided axis needs inner extent % 8 == 0");
  // 32-bit element offsets in the kernels: extents <= 512 in <= 3D keep N <= 2^27
  switch (L) {
    case 16: return launch_L<16>(program, contig, inverse != 0, a, st);
    case 32: return launch_L<32>(program, contig, inverse != 0, a, st);
    case 64: return launch_L<64>(program, contig, inverse != 0, a, st);
    case 128: return launch_L<128>(program, contig, inverse != 0, a, st);
    case 256: return launch_L<256>(program, contig, inverse != 0, a, st);
    case 512: return launch_L<512>(program, contig, inverse != 0, a, st);
    default: return set_error(CGL_ESHAPE, "fft_pass: extent");
  }
}

CGL_PROF_TU(fftpass)

}  // namespace cgl
