// Plane-chunked pencil-FFT passes: three passes of a 3D Fourier step in ONE
// persistent launch, with the intermediate fields held in L2.
//
// In the periodic steppers (integrators.py:99-120, 161-164, 205-215 around
// spectral.py:79-86) every contiguous-axis program of fftpass.cu (IF4_B1..B4,
// STR_MID: F_2, pointwise stage, F_2^-1 on whole rows) sits between a forward
// and an inverse transform along axis 1.  All three act inside one axis-0
// plane (n1 x n2 points, 4 MiB at 512^2), so a plane can go
//     F_1 (strided pencils)  ->  program (rows)  ->  F_1^-1 (strided pencils)
// while it is resident in the 126 MB L2: HBM sees one read of the plane, the
// program's own operand streams, and one write -- 64..112 B per point for
// the if4 programs instead of 128..176 B with three separate launches.
//
// One launch runs every plane.  CTAs are persistent and take TICKETS from a
// global counter; a ticket is one tile (8 x threads points) of one phase of
// one plane, and tickets are ordered so that every tile a ticket depends on
// has a smaller ticket:
//     round r:  phase 0 of plane r,  phase 1 of plane r - D,  phase 2 of plane r - 2 D
// (D planes of lag, so that the producer tiles of a phase were handed out two
// grid-widths earlier and a consumer hardly ever waits).  A phase-1 tile needs
// ALL phase-0 tiles of its plane, a phase-2 tile all phase-1 tiles: per-plane
// counters, bumped with release semantics after a tile's stores, read with
// acquire semantics before a tile's loads.  Running CTAs only ever wait on
// smaller tickets, which are held by running CTAs: no co-residency is assumed
// and there is no deadlock.  The next ticket's tile is prefetched (cp.async,
// L2 -> shared, bypassing the non-coherent L1) into the other half of a
// two-tile ring while the current tile is transformed, if its plane is ready.
// The control block is caller-owned (zeroed once); the last CTA re-zeroes it.
//
// Arithmetic is that of the separate passes (same fft_pencil / contig_program
// templates), so results are bit-identical to them.
#include "fftpass.cuh"

namespace cgl {
namespace fftp {

constexpr int kPlaneMax = 512;
struct PlaneCtl {
  unsigned ticket;
  unsigned finished;
  unsigned pad[2];
  unsigned done[2 * kPlaneMax];  // [plane][0]: F_1 tiles stored, [plane][1]: program tiles stored
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int L, int PROG, int NT>
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : 2)
    fft_plane_kernel(const Args a, PlaneCtl* __restrict__ ctl, const int P, const int D) {
  using GS = Geo<L, false, NT>;
  using GC = Geo<L, true, NT>;
  constexpr int T = L / 8;
  constexpr int TILE = NT * 8;
  constexpr int TPP = L * L / TILE;  // tiles per plane and phase
  constexpr int NAUX = Aux<PROG>::N;
  static_assert(TPP >= 1 && TPP * TILE == L * L, "plane = whole tiles");
  extern __shared__ double2 sm[];
  __shared__ int s_tk[2][2];
  __shared__ int s_last;
  pdl_wait();
  const uint64_t step = resolve_pos(a.flag, a.pos) >> 24;
  if (a.flag && flag_skip(a.flag, step << 24)) return;

  const int tid = threadIdx.x;
  const TileMap<L, true, NT> mc(tid);
  const TileMap<L, false, NT> ms(tid);
  Lay<L, true> lc;
  lc.base = mc.lay_base();
  lc.cw = 0;
  Lay<L, false> ls;
  ls.base = ms.lay_base();
  ls.cw = GS::CW;
  double2* ring[2] = {sm, sm + TILE};
  double2* tws = sm + 2 * TILE;
  double2* aux = tws + 512;  // stage operand u of the current program tile: [r][NT]
  stage_twiddles<L>(tws, tid, NT);  // visible after the first barrier below
  uint64_t key = ~0ull;
  const uint64_t check_pos = (step << 24) | (255ull << 8);
  double2* const field = a.dst;

  // a ticket is a BATCH of KB consecutive tiles of one phase of one plane
  constexpr int KB = TPP < 4 ? TPP : 4;
  constexpr int BPP = TPP / KB;  // batches per plane and phase
  static_assert(KB >= 2 && BPP * KB == TPP, "batches");
  const int total_b = (P + 2 * D) * 3 * BPP;
  auto decode = [&](int tk, int& phase, int& plane, int& batch) -> bool {
    constexpr int per = 3 * BPP;
    const int r = tk / per, rem = tk - r * per;
    phase = rem / BPP;
    batch = rem - phase * BPP;
    plane = r - phase * D;
    return plane >= 0 && plane < P;
  };
  auto plane_ready = [&](int ph, int pl) -> bool {  // thread 0
    if (ph == 0) return true;
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(&ctl->done[2 * pl + ph - 1]) : "memory");
    if (v < (unsigned)BPP) return false;
    __threadfence();  // acquire: the plane's tiles, stored before their batches were counted, are visible
    return true;
  };
  // thread 0: next valid ticket from `first` on (-1: none left)
  auto next_valid = [&](int first) -> int {
    int tk = first, ph, pl, b;
    for (;;) {
      if (tk >= total_b) return -1;
      if (decode(tk, ph, pl, b)) return tk;
      tk = (int)atomicAdd(&ctl->ticket, 1u);
    }
  };
  auto wait_plane = [&](int ph, int pl) {
    if (ph > 0) {
      if (tid == 0)
        while (!plane_ready(ph, pl)) __nanosleep(64);
      __syncthreads();
    }
  };
  // global offset of this thread's element 0, tile gt of a phase
  auto strided_base = [&](int gt) {
    constexpr int cpo = L / GS::CW;
    const int c = gt * GS::G + ms.p_or_g;
    const int o = c / cpo;
    return o * L * L + (c - o * cpo) * GS::CW + ms.pp;
  };
  auto contig_row = [&](int gt) { return gt * GC::ROWS + mc.p_or_g; };
  auto issue = [&](int ph, int gt, double2* buf) {
    if (ph == 1) {
      const double2* g = field + contig_row(gt) * L + mc.t;
#pragma unroll
      for (int r = 0; r < 8; ++r) cp_async16(buf + lc.at(mc.t + T * r), g + T * r);
    } else {
      const double2* g = field + strided_base(gt) + ms.t * L;
#pragma unroll
      for (int r = 0; r < 8; ++r) cp_async16(buf + ls.at(ms.t + T * r), g + (T * r) * L);
    }
  };

  // s_tk[0]: the next batch's ticket, s_tk[1]: its plane was ready when polled
  int* s_nt = &s_tk[0][0];
  if (tid == 0) s_nt[0] = next_valid((int)atomicAdd(&ctl->ticket, 1u));
  __syncthreads();
  int tk = s_nt[0], ph = 0, pl = 0, bt = 0;
  if (tk >= 0) {
    decode(tk, ph, pl, bt);
    wait_plane(ph, pl);
    issue(ph, pl * TPP + bt * KB, ring[0]);
  }
  cp_async_commit();
  int r_tk = 0;  // thread 0: the ticket taken at a batch's first tile (consumed one tile later)
  int j = 0;     // tile within the batch
  for (int it = 0; tk >= 0; ++it) {
    const int gt = pl * TPP + bt * KB + j;
    double2* sbuf = ring[it & 1];
    const int row = contig_row(gt);
    const int gbase_c = row * L;
    if (tid == 0 && j == 0) r_tk = (int)atomicAdd(&ctl->ticket, 1u);  // in flight through this tile
    if (NAUX > 0 && ph == 1) {
#pragma unroll
      for (int r = 0; r < 8; ++r) cp_async16(aux + r * NT + tid, a.u + gbase_c + mc.t + T * r);
    }
    cp_async_commit();  // group A: stage operands of this tile
    // the next tile: in this batch (ready by construction), or the next batch's first
    int ntk = tk, nph = ph, npl = pl, nbt = bt;
    bool nready = true;
    if (j == KB - 1) {
      ntk = s_nt[0];
      nready = s_nt[1] != 0;
      if (ntk >= 0) decode(ntk, nph, npl, nbt);
    }
    const int nj = j == KB - 1 ? 0 : j + 1;
    if (ntk >= 0 && nready) issue(nph, npl * TPP + nbt * KB + nj, ring[(it + 1) & 1]);
    cp_async_commit();  // group B: the next tile, if its plane is ready
    cp_async_wait<2>();  // this tile's main operand
    double2 v[8];
    if (ph == 1) {
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = sbuf[lc.at(mc.t + T * r)];
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = sbuf[ls.at(ms.t + T * r)];
    }
    __syncthreads();  // every thread holds its inputs: the tile buffer becomes the exchange buffer
    if (ph == 0) {
      fft_pencil<L, false, false>(v, ms.t, sbuf, ls, tws);
      double2* g = field + strided_base(gt) + ms.t * L;
#pragma unroll
      for (int r = 0; r < 8; ++r) g[(T * r) * L] = v[r];  // stays in L2 for phase 1
    } else if (ph == 1) {
      contig_program<L, PROG, NT>(v, a, true, row, gbase_c, mc.t, tid, aux, sbuf, lc, tws, key, check_pos);
      double2* g = field + gbase_c + mc.t;
#pragma unroll
      for (int r = 0; r < 8; ++r) g[T * r] = v[r];        // stays in L2 for phase 2
    } else {
      fft_pencil<L, false, true>(v, ms.t, sbuf, ls, tws);
      double2* g = field + strided_base(gt) + ms.t * L;
#pragma unroll
      for (int r = 0; r < 8; ++r) stg_s(g + (T * r) * L, v[r]);
    }
    if (j == KB - 1 && ph < 2) __threadfence();  // the batch's stores are visible device-wide before it is counted
    if (tid == 0) {
      if (j == 0) s_nt[0] = next_valid(r_tk);
      if (j == KB - 2) {
        int xp, xl, xb;
        const int x = s_nt[0];
        s_nt[1] = x >= 0 && decode(x, xp, xl, xb) && plane_ready(xp, xl);
      }
    }
    __syncthreads();   // exchange reads done before the buffer is refilled; s_nt published
    if (j == KB - 1) {
      if (tid == 0 && ph < 2) atomicAdd(&ctl->done[2 * pl + ph], 1u);
      if (ntk >= 0 && !nready) {
        wait_plane(nph, npl);
        issue(nph, npl * TPP + nbt * KB, ring[(it + 1) & 1]);
      }
    }
    cp_async_commit();  // group C: the next batch's first tile, if it had to wait
    tk = ntk;
    ph = nph;
    pl = npl;
    bt = nbt;
    j = nj;
  }
  cp_async_wait<0>();
  if (PROG == FP_IF4_B4) raise_min(a.flag, key);
  pdl_trigger();
  // the last CTA out leaves the control block zeroed for the next launch
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&ctl->finished, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (int i = tid; i < 2 * P; i += NT) ctl->done[i] = 0;
    if (tid == 0) {
      ctl->ticket = 0;
      ctl->finished = 0;
    }
  }
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

template <int L, int PROG, int NT>
static int launch_plane_nt(const Args& a, PlaneCtl* ctl, int P, cudaStream_t st) {
  constexpr int TILE = NT * 8;
  constexpr int TPP = L * L / TILE;
  auto kern = fft_plane_kernel<L, PROG, NT>;
  static int blocks_per_sm = 0, sms = 0;
  const int smem = (2 * TILE + 512 + Aux<PROG>::N * TILE) * (int)sizeof(double2);
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, NT, smem);
    if (e != cudaSuccess || blocks_per_sm < 1) return set_cuda_error(e, "fft_plane occupancy");
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t grid = (int64_t)sms * blocks_per_sm;
  const int64_t batches = (int64_t)P * 3 * (TPP / (TPP < 4 ? TPP : 4));
  if (grid > batches) grid = batches;
  // lag in planes: a phase's producer tiles were handed out >= 2 grid-widths earlier
  int D = env_int("CGL_PLANE_LAG", 0);
  if (D <= 0) D = (int)((2 * grid + 3 * TPP - 1) / (3 * TPP));
  if (D < 1) D = 1;
  if (D > P) D = P;
  cudaError_t e = launch_k(kern, dim3((unsigned)grid), dim3(NT), (size_t)smem, st, dim3(1), a, ctl, P, D);
  if (e != cudaSuccess) return set_cuda_error(e, "fft_plane launch");
  return check_launch("fft_plane_kernel");
}

template <int L, int PROG>
static int launch_plane_prog(const Args& a, PlaneCtl* ctl, int P, cudaStream_t st) {
  if constexpr (L == 512) {
    if (env_int("CGL_PLANE_NT", 256) == 512) return launch_plane_nt<L, PROG, 512>(a, ctl, P, st);
  }
  return launch_plane_nt<L, PROG, 256>(a, ctl, P, st);
}

template <int L>
static int launch_plane_L(int prog, const Args& a, PlaneCtl* ctl, int P, cudaStream_t st) {
  switch (prog) {
    case FP_IF4_B1: return launch_plane_prog<L, FP_IF4_B1>(a, ctl, P, st);
    case FP_IF4_B2: return launch_plane_prog<L, FP_IF4_B2>(a, ctl, P, st);
    case FP_IF4_B3: return launch_plane_prog<L, FP_IF4_B3>(a, ctl, P, st);
    case FP_IF4_B4: return launch_plane_prog<L, FP_IF4_B4>(a, ctl, P, st);
    case FP_STR_MID: return launch_plane_prog<L, FP_STR_MID>(a, ctl, P, st);
    default: return set_error(CGL_EINVAL, "fft_plane: program must be IF4_B1..B4 or STR_MID");
  }
}

}  // namespace fftp

size_t fft_plane_workspace_bytes() { return sizeof(fftp::PlaneCtl); }

bool fft_plane_supported(int ndim, const int64_t* shape) {
  if (ndim != 3 || !fft_pass_supported(ndim, shape)) return false;
  return shape[1] == shape[2] && shape[1] >= 64 && shape[0] <= fftp::kPlaneMax;
}

int fft_plane_launch(cudaStream_t st, int program, int ndim, const int64_t* shape, double* field,
                     const cgl_fft_ops_t* ops, void* workspace) {
  using namespace fftp;
  if (!fft_plane_supported(ndim, shape)) return set_error(CGL_ESHAPE, "fft_plane: 3D, shape[1] == shape[2] in 64..512");
  if (!field || !ops || !workspace) return set_error(CGL_EINVAL, "fft_plane: null field / operands / workspace");
  if (reinterpret_cast<uintptr_t>(workspace) & 15) return set_error(CGL_EINVAL, "fft_plane: workspace alignment");
  Args a{};
  a.src = reinterpret_cast<const double2*>(field);
  a.dst = reinterpret_cast<double2*>(field);
  a.O = shape[0] * shape[1];
  a.I = 1;
  a.nd = 3;
  a.lg1 = 0;
  while ((1ll << a.lg1) < shape[1]) ++a.lg1;
  a.u = reinterpret_cast<const double2*>(ops->u);
  a.u_out = reinterpret_cast<double2*>(ops->u_out);
  for (int q = 0; q < 3; ++q) a.g[q] = reinterpret_cast<const double2*>(ops->g[q]);
  a.g_out = reinterpret_cast<double2*>(ops->g_out);
  for (int fr = 0; fr < 2; ++fr)
    for (int d = 0; d < 3; ++d) a.tab[fr][d] = reinterpret_cast<const double2*>(ops->tables[fr][d]);
  a.tau = ops->tau;
  a.scale = ops->scale;
  const cgl_nonlinear_t& nl = ops->nl;
  a.nl = StageNL{nl.alpha3, nl.beta3, nl.alpha4, nl.beta4, nl.alpha5, nl.kind};
  a.fw = 1;
  a.flag = ops->flag;
  a.pos = ops->pos;
  if (program >= FP_IF4_B1 && program <= FP_IF4_B4 && !a.u) return set_error(CGL_EINVAL, "fft_plane: program needs u");
  if (program >= FP_IF4_B1 && program <= FP_IF4_B3 && !a.g_out) return set_error(CGL_EINVAL, "fft_plane: needs g_out");
  if (program == FP_IF4_B4 && (!a.g[0] || !a.g[1] || !a.g[2] || !a.u_out))
    return set_error(CGL_EINVAL, "fft_plane: B4 needs g1..g3 and u_out");
  for (int fr = 0; fr < 2; ++fr)
    for (int d = 0; d < 3; ++d)
      if (!a.tab[fr][d]) return set_error(CGL_EINVAL, "fft_plane: program needs the exp tables");
  PlaneCtl* ctl = static_cast<PlaneCtl*>(workspace);
  const int P = (int)shape[0];
  switch ((int)shape[1]) {
    case 64: return launch_plane_L<64>(program, a, ctl, P, st);
    case 128: return launch_plane_L<128>(program, a, ctl, P, st);
    case 256: return launch_plane_L<256>(program, a, ctl, P, st);
    case 512: return launch_plane_L<512>(program, a, ctl, P, st);
    default: return set_error(CGL_ESHAPE, "fft_plane: extent");
  }
}

}  // namespace cgl
