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
//     axis (one kernel: forward -> g_i -> stage -> inverse);
//   * strang: the end-of-step flow, the finiteness check, the next step's
//     first flow and the forward pass share one kernel along the slowest axis;
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
#include <cstdlib>

#include <cuda_runtime.h>

#include "cgl_common.cuh"
#include "cgl_internal.h"
#include "fft_twiddles.h"
#include "stage_ops.cuh"


namespace cgl {
namespace fftp {


enum Prog {
  FP_PLAIN = 0,     // transform only
  FP_IF4_START,     // contiguous, inverse: src = spectral state u
  FP_IF4_B1,        // contiguous: g1 = F(src); u2 = E1/2 (u + t/2 g1); dst = F^-1 u2
  FP_IF4_B2,        // g2 = F(src); u3 = E1/2 u + t/2 g2
  FP_IF4_B3,        // g3 = F(src); u4 = t E1/2 g3 + E1 u
  FP_IF4_B4,        // g4 = F(src); out = E1 (u + t/6 g1) + t/3 E1/2 (g2 + g3) + t/6 g4 -> u; check;
                    // dst = F^-1 out (the next step's first inverse pass) when dst != null
  FP_G,             // inverse, x scale, g(.), forward (any axis)
  FP_STR_START,     // strided, forward: src = physical u (x scale); v = flow(u, t/2) [seq 0]
  FP_STR_A0,        // strided: w = F^-1(src) x scale; out = flow(w, t/2) [seq w]; check; u_out = out;
                    // v = flow(out, t/2) [step + 1, seq 0]; dst = F(v) when dst != null
  FP_STR_MID,       // contiguous: F, x E1, F^-1
  FP_NPROG
};

struct Args {
  const double2* src;
  double2* dst;
  int64_t O, I;  // outer count, inner stride of the transform axis (I = 1: contiguous)
  const double2* u;
  double2* u_out;
  const double2* g[3];
  double2* g_out;
  const double2* tab[2][3];  // separable exp(f tau symbol): [fraction 1/2, 1][axis]
  int nd;
  int lg1;        // log2 n1 (3D row decode: i0 = row >> lg1, i1 = row & (n1 - 1))
  double tau, scale;
  StageNL nl;
  cgl_flag_t* flag;
  uint64_t pos;
  int fw;
};

__device__ __forceinline__ double2 mul_mi(double2 a, bool inv) {  // a * (-i) forward, a * (+i) inverse
  return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
__device__ __forceinline__ double2 mul_w8(double2 a, bool inv) {  // a * exp(-+ i pi / 4)
  const double s = 0.70710678118654752440;
  return inv ? make_double2(__dmul_rn(s, __dsub_rn(a.x, a.y)), __dmul_rn(s, __dadd_rn(a.x, a.y)))
             : make_double2(__dmul_rn(s, __dadd_rn(a.x, a.y)), __dmul_rn(s, __dsub_rn(a.y, a.x)));
}
__device__ __forceinline__ double2 mul_w83(double2 a, bool inv) {  // a * exp(-+ 3 i pi / 4)
  const double s = 0.70710678118654752440;
  return inv ? make_double2(__dmul_rn(-s, __dadd_rn(a.x, a.y)), __dmul_rn(s, __dsub_rn(a.x, a.y)))
             : make_double2(__dmul_rn(s, __dsub_rn(a.y, a.x)), __dmul_rn(-s, __dadd_rn(a.x, a.y)));
}

template <bool INV>
__device__ __forceinline__ void dft8(double2 (&a)[8]) {
  const double2 b0 = cadd(a[0], a[4]), b4 = csub(a[0], a[4]);
  const double2 b1 = cadd(a[1], a[5]), b5 = mul_w8(csub(a[1], a[5]), INV);
  const double2 b2 = cadd(a[2], a[6]), b6 = mul_mi(csub(a[2], a[6]), INV);
  const double2 b3 = cadd(a[3], a[7]), b7 = mul_w83(csub(a[3], a[7]), INV);
  const double2 c0 = cadd(b0, b2), c2 = csub(b0, b2), c1 = cadd(b1, b3), c3 = mul_mi(csub(b1, b3), INV);
  const double2 c4 = cadd(b4, b6), c6 = csub(b4, b6), c5 = cadd(b5, b7), c7 = mul_mi(csub(b5, b7), INV);
  a[0] = cadd(c0, c1);
  a[4] = csub(c0, c1);
  a[2] = cadd(c2, c3);
  a[6] = csub(c2, c3);
  a[1] = cadd(c4, c5);
  a[5] = csub(c4, c5);
  a[3] = cadd(c6, c7);
  a[7] = csub(c6, c7);
}
template <bool INV>
__device__ __forceinline__ void dft4(double2 (&a)[4]) {
  const double2 b0 = cadd(a[0], a[2]), b2 = csub(a[0], a[2]);
  const double2 b1 = cadd(a[1], a[3]), b3 = mul_mi(csub(a[1], a[3]), INV);
  a[0] = cadd(b0, b1);
  a[2] = csub(b0, b1);
  a[1] = cadd(b2, b3);
  a[3] = csub(b2, b3);
}

// twiddles: staged once per CTA in shared memory as per-stage tables
// tw[base(s) + (m - 1) Ns + k] = W_{Ns R}^{m k}, so the threads of a
// quarter-warp (consecutive k) read consecutive 16-byte words: no bank
// conflicts (a 512-entry table indexed by m k 512/(Ns R) puts them 8 words
// apart).
__device__ __forceinline__ double2 twiddle(const double2* tw, int idx, bool inv) {
  const double2 w = tw[idx];  // shared (persistent CTAs) or the global table through L1
  return inv ? make_double2(w.x, -w.y) : w;
}

// log2 and radix plan of a power-of-two length 8 <= L <= 512
template <int L>
struct Plan {
  static constexpr int p = L == 8 ? 3 : L == 16 ? 4 : L == 32 ? 5 : L == 64 ? 6 : L == 128 ? 7 : L == 256 ? 8 : 9;
  static constexpr int n8 = p / 3;          // radix-8 stages
  static constexpr int tail = p % 3;        // 0: none, 1: radix-2, 2: radix-4 (last stage)
  static constexpr int nstages = n8 + (tail ? 1 : 0);
  static constexpr int T = L / 8;           // threads per pencil
  static constexpr int radix(int s) { return s < n8 ? 8 : (tail == 1 ? 2 : 4); }
  static constexpr int ns(int s) { return s == 0 ? 1 : ns(s - 1) * radix(s - 1); }
  // first twiddle of stage s (stage 0 has Ns = 1: no twiddles)
  static constexpr int twbase(int s) { return s <= 1 ? 0 : twbase(s - 1) + (radix(s - 1) - 1) * ns(s - 1); }
  static constexpr int twsize() { return twbase(nstages); }
};

// per-stage twiddle tables of a length-L transform (see twiddle()), copied
// from the generated global table into shared memory by persistent CTAs
template <int L>
__device__ __forceinline__ void stage_twiddles(double2* tw, int tid, int nt) {
  for (int e = tid; e < Plan<L>::twsize(); e += nt) tw[e] = __ldg(&g_fft_stage_tw[fft_stage_tw_offset(L) + e]);
}

// shared-memory slot of element i of the calling thread's pencil
template <int L, bool CONTIG>
struct Lay {
  int base;  // CONTIG: pencil * L; strided: chunk * L * CW + pencil-in-chunk
  int cw;    // strided: pencils per chunk
  __device__ __forceinline__ int at(int i) const {
    if (CONTIG) return base + ((i & ~7) | ((i ^ (i >> 3)) & 7));
    // 4-pencil chunks: a quarter-warp covers rows of two threads t, t + 1;
    // swapping rows 2q, 2q + 1 when bit 3 of i is set puts those two rows in
    // different halves of a 128-byte line for every stage pattern
    if (cw == 4) return base + ((i ^ ((i >> 3) & 1)) << 2);
    return base + i * cw;
  }
};

// In-register transform of one pencil: on entry v[r] = x[t + T r]; on exit
// v[r] = X[t + T r].  sm: the CTA's exchange buffer.
template <int L, bool CONTIG, bool INV>
__device__ __forceinline__ void fft_pencil(double2 (&v)[8], int t, double2* sm, const Lay<L, CONTIG>& lay,
                                           const double2* tw) {
  using PL = Plan<L>;
  constexpr int T = PL::T;
  int Ns = 1;
#pragma unroll
  for (int s = 0; s < PL::nstages; ++s) {
    const int R = s < PL::n8 ? 8 : (PL::tail == 1 ? 2 : 4);
    const bool last = s == PL::nstages - 1;
    // twiddle W_{Ns R}^{m k} = W_512^{m k 512 / (Ns R)}
    if (R == 8) {
      const int j = t;
      const int k = j & (Ns - 1);
      double2 a[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = v[m];
      if (Ns > 1) {
#pragma unroll
        for (int m = 1; m < 8; ++m) a[m] = cmul(a[m], twiddle(tw, PL::twbase(s) + (m - 1) * Ns + k, INV));
      }
      dft8<INV>(a);
      if (last) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = a[q];
      } else {
        const int o = (j / Ns) * Ns * 8 + k;
#pragma unroll
        for (int q = 0; q < 8; ++q) sm[lay.at(o + q * Ns)] = a[q];
      }
    } else if (R == 4) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = t + h * T;
        const int k = j & (Ns - 1);
        double2 a[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) a[m] = v[h + 2 * m];
        if (Ns > 1) {
#pragma unroll
          for (int m = 1; m < 4; ++m) a[m] = cmul(a[m], twiddle(tw, PL::twbase(s) + (m - 1) * Ns + k, INV));
        }
        dft4<INV>(a);
        // radix-4 only ever runs last (L = 2^(3a+2)): out[j + q Ns] = v[h + 2 q]
#pragma unroll
        for (int q = 0; q < 4; ++q) v[h + 2 * q] = a[q];
      }
    } else {
      // radix 2, last stage
      double2 a[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = v[r];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int j = t + h * T;
        const int k = j & (Ns - 1);
        double2 x0 = a[h], x1 = a[h + 4];
        if (Ns > 1) x1 = cmul(x1, twiddle(tw, PL::twbase(s) + k, INV));
        v[h] = cadd(x0, x1);
        v[h + 4] = csub(x0, x1);
      }
    }
    if (!last) {
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = sm[lay.at(t + T * r)];
      __syncthreads();
    }
    Ns *= R;
  }
}

// separable exp(f tau symbol) of a contiguous-axis row: every element of a
// thread lies in one row, so the product of the row's slower-axis factors is
// formed once (rf[fr]) and each element costs one table load and one cmul.
__device__ __forceinline__ double2 row_factor(const Args& a, int fr, int row) {
  if (a.nd == 3) return cmul(ld2(a.tab[fr][1] + (row & ((1 << a.lg1) - 1))), ld2(a.tab[fr][0] + (row >> a.lg1)));
  return ld2(a.tab[fr][0] + row);
}
__device__ __forceinline__ double2 efac(const Args& a, int fr, const double2 (&rf)[2], int i) {
  return cmul(ld2(a.tab[fr][a.nd - 1] + i), rf[fr]);
}

// operands prefetched into shared memory by the stage programs
template <int PROG>
struct Aux {
  static constexpr int N = (PROG >= FP_IF4_B1 && PROG <= FP_IF4_B4) ? 1 : 0;
};
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// streaming global accesses: every pass touches each element once
__device__ __forceinline__ double2 ldg_s(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void stg_s(double2* p, double2 v) { __stcs(p, v); }

// CTA geometry for threads NT and pencil length L
template <int L, bool CONTIG, int NT>
struct Geo {
  static constexpr int T = L / 8;                                  // threads per pencil
  static constexpr int TILE = NT * 8;                              // elements per CTA
  static constexpr int ROWS = CONTIG ? TILE / L : 0;               // contiguous: rows per CTA
  static constexpr int CW = CONTIG ? 0 : (NT / T < 8 ? NT / T : 8);  // strided: pencils per chunk
  static constexpr int G = CONTIG ? 0 : NT / (T * CW);             // strided: chunks per CTA
};

// registers per thread the program needs to co-reside MINB CTAs per SM
template <int PROG, int NT, bool CONTIG>
struct Occ {
  // shared memory: 2 tiles of 32 KB + 8 KB twiddles (+ 32 KB stage operands for B1..B4)
  static constexpr int MINB = NT >= 512                                   ? ((PROG == FP_PLAIN || PROG == FP_G) ? 2 : 1)
                              : (PROG >= FP_IF4_B1 && PROG <= FP_IF4_B4)   ? 2
                              : (PROG == FP_PLAIN && !CONTIG)              ? 4
                                                                           : 3;
};

// Persistent pass kernel: each CTA walks tiles blockIdx.x, +gridDim.x, ...
// The main operand of tile i+1 is copied (cp.async, L2 -> shared, no
// registers) into the other half of a two-tile ring while tile i is
// transformed, so HBM reads stay in flight through the compute phase; each
// thread copies exactly the elements it will read (its own slots of the
// exchange layout), so the copy needs no barrier, and the tile buffer doubles
// as the exchange buffer of the transform.
template <int L, bool CONTIG, int NT>
struct TileMap {
  using GE = Geo<L, CONTIG, NT>;
  static constexpr int T = GE::T;
  int t, p_or_g, pp;
  __device__ __forceinline__ explicit TileMap(int tid) {
    if constexpr (CONTIG) {
      p_or_g = tid / T;
      t = tid % T;
      pp = 0;
    } else {
      pp = tid % GE::CW;
      p_or_g = (tid / GE::CW) / T;
      t = (tid / GE::CW) % T;
    }
  }
  // element (t + T r) of this thread's pencil in tile `tile` sits at gbase + (t + T r) * gstride
  __device__ __forceinline__ bool geo(const Args& a, int64_t tile, int& gbase, int& gstride, int& row) const {
    if (CONTIG) {
      row = tile * GE::ROWS + p_or_g;
      gbase = row * L;
      gstride = 1;
      return row < (int)a.O;
    } else {
    const int cpo = (int)a.I / GE::CW;
    const int c = tile * GE::G + p_or_g;
    const int o = c / cpo;
    gbase = o * L * (int)a.I + (c % cpo) * GE::CW + pp;
    gstride = (int)a.I;
    row = 0;
    return c < (int)a.O * cpo;
    }
  }
  __device__ __forceinline__ int lay_base() const {
    return CONTIG ? p_or_g * L : p_or_g * L * GE::CW + pp;
  }
};

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
    }
    cp_async_commit();
    issue(tile + (int)gridDim.x, ring[(it + 1) & 1]);
    if (RING) {
      cp_async_wait<2>();  // this tile's main operand (the two newer groups may still fly)
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = valid ? sbuf[lay.at(t + T * r)] : make_double2(0.0, 0.0);
      __syncthreads();  // every thread holds its inputs: the tile buffer becomes the exchange buffer
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
      __syncthreads();
      fft_pencil<L, CONTIG, false>(v, t, sbuf, lay, tw);
    } else if (PROG == FP_IF4_B1 || PROG == FP_IF4_B2 || PROG == FP_IF4_B3 || PROG == FP_IF4_B4) {
      fft_pencil<L, CONTIG, false>(v, t, sbuf, lay, tw);  // v = g_i (spectral)
      cp_async_wait<RING ? 1 : 0>();                      // the stage operands (the prefetch may fly)
      double2 rf[2];
      rf[0] = valid ? row_factor(a, 0, row) : make_double2(0.0, 0.0);
      rf[1] = (valid && (PROG == FP_IF4_B3 || PROG == FP_IF4_B4)) ? row_factor(a, 1, row) : rf[0];
      if (valid) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int i = t + T * r;
          const int gi = gbase + i;
          const double2 gi_v = v[r];
          const double2 u = aux[r * NT + tid];
          if (PROG == FP_IF4_B1) {
            stg_s(a.g_out + gi, gi_v);
            v[r] = cmul(efac(a, 0, rf, i), caxpy(0.5 * tau, gi_v, u));
          } else if (PROG == FP_IF4_B2) {
            stg_s(a.g_out + gi, gi_v);
            v[r] = caxpy(0.5 * tau, gi_v, cmul(efac(a, 0, rf, i), u));
          } else if (PROG == FP_IF4_B3) {
            stg_s(a.g_out + gi, gi_v);
            v[r] = caxpy(tau, cmul(efac(a, 0, rf, i), gi_v), cmul(efac(a, 1, rf, i), u));
          } else {
            const double2 g1 = ldg_s(a.g[0] + gi), g2 = ldg_s(a.g[1] + gi), g3 = ldg_s(a.g[2] + gi);
            const double2 out =
                caxpy(tau / 6.0, gi_v,
                      caxpy(tau / 3.0, cmul(efac(a, 0, rf, i), caxpy(1.0, g2, g3)),
                            cmul(efac(a, 1, rf, i), caxpy(tau / 6.0, g1, u))));
            if (!cfinite(out)) note(key, check_pos, CGL_NONFINITE_STATE);
            stg_s(a.u_out + gi, out);
            v[r] = out;
          }
        }
      }
      if (PROG == FP_IF4_B4 && a.dst == nullptr) {
        store = false;
      } else {
        __syncthreads();
        fft_pencil<L, CONTIG, true>(v, t, sbuf, lay, tw);
      }
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
      fft_pencil<L, CONTIG, false>(v, t, sbuf, lay, tw);
      double2 rf[2];
      rf[1] = valid ? row_factor(a, 1, row) : make_double2(0.0, 0.0);
      rf[0] = rf[1];
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = cmul(efac(a, 1, rf, t + T * r), v[r]);
      __syncthreads();
      fft_pencil<L, CONTIG, true>(v, t, sbuf, lay, tw);
    }
    if (valid && store) {
#pragma unroll
      for (int r = 0; r < 8; ++r) stg_s(a.dst + gbase + (t + T * r) * gstride, v[r]);
    }
    if (!valid) key = ~0ull;
    __syncthreads();  // the exchange reads of this tile are done before its buffer is refilled
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
  if (a.flag && flag_skip(a.flag, (step << 24) | ((uint64_t)(PROG == FP_STR_A0 ? a.fw : 0) << 8))) return;
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
  }
  if (valid) {
#pragma unroll
    for (int r = 0; r < 8; ++r) stg_s(a.dst + gbase + (t + T * r) * gstride, v[r]);
  }
  if (PROG == FP_STR_START || PROG == FP_STR_A0) raise_min(a.flag, valid ? key : ~0ull);
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
  if (prog == FP_STR_A0 || prog == FP_STR_START) return 256;
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

template <int L, bool CONTIG, int PROG, bool INV>
static int launch_one(const Args& a, cudaStream_t st) {
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
    if (nl.kind == 2) return set_error(CGL_EINVAL, "fft_pass: scalar fields only");
    a.fw = 1;
    a.flag = ops->flag;
    a.pos = ops->pos;
  } else if (program != FP_PLAIN) {
    return set_error(CGL_EINVAL, "fft_pass: program needs its operands");
  }
  // operand checks per program
  const bool need_src = !(program == FP_IF4_START || program == FP_STR_START);
  if (need_src && !src) return set_error(CGL_EINVAL, "fft_pass: null src");
  const bool dst_optional = program == FP_IF4_B4 || program == FP_STR_A0;
  if (!dst && !dst_optional) return set_error(CGL_EINVAL, "fft_pass: null dst");
  if ((program >= FP_IF4_START && program <= FP_IF4_B4 || program == FP_STR_START) && !a.u)
    return set_error(CGL_EINVAL, "fft_pass: program needs u");
  if ((program >= FP_IF4_B1 && program <= FP_IF4_B3) && !a.g_out) return set_error(CGL_EINVAL, "fft_pass: needs g_out");
  if (program == FP_IF4_B4 && (!a.g[0] || !a.g[1] || !a.g[2] || !a.u_out))
    return set_error(CGL_EINVAL, "fft_pass: B4 needs g1..g3 and u_out");
  if (program == FP_STR_A0 && !a.u_out) return set_error(CGL_EINVAL, "fft_pass: needs u_out");
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
