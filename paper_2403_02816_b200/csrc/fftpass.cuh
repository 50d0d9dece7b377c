// Shared device templates of the pencil-FFT kernels (fftpass.cu: one pass per
// launch; fftplane.cu: three passes per plane in one persistent launch).
#pragma once
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
  FP_IF4_B1,        // contiguous: g1 = F(src); acc = E1 (u + t/6 g1) -> g_out; u2 = E1/2 (u + t/2 g1); dst = F^-1 u2
  FP_IF4_B2,        // g2 = F(src); acc = g[0] + t/3 E1/2 g2 -> g_out; u3 = E1/2 u + t/2 g2
  FP_IF4_B3,        // g3 = F(src); acc = g[0] + t/3 E1/2 g3 -> g_out; u4 = t E1/2 g3 + E1 u
  FP_IF4_B4,        // g4 = F(src); out = u + t/6 g4 with u = acc -> u_out; check;
                    // dst = F^-1 out (the next step's first inverse pass) when dst != null
  FP_G,             // inverse, x scale, g(.), forward (any axis)
  FP_STR_START,     // strided, forward: src = physical u (x scale); v = flow(u, t/2) [seq 0]
  FP_STR_A0,        // strided: w = F^-1(src) x scale; out = flow(w, t/2) [seq w]; check; u_out = out;
                    // v = flow(out, t/2) [step + 1, seq 0]; dst = F(v) when dst != null
  FP_STR_MID,       // contiguous: F, x E1, F^-1
  FP_STR_A0F,       // as STR_A0 for the exact cubic flow with the two boundary flows fused (cubic_boundary):
                    // u_out = w (the step's state is flow(u_out, t/2), evaluated on demand); dst = F(flow(w, t))
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

// Barrier among the threads that exchange data through a pencil's buffer.
// Contiguous passes: a pencil is L/8 consecutive threads with its own L-element
// region, so the threads of ONE pencil suffice -- a warp barrier up to L = 256,
// a 64-thread named barrier (id 1 + pencil) at L = 512; the other pencils of the
// CTA run on unhindered.  Strided passes interleave the pencils of a chunk over
// all warps: CTA barrier.
template <int L, bool CONTIG>
__device__ __forceinline__ void pencil_sync(const Lay<L, CONTIG>& lay) {
  if constexpr (!CONTIG) {
    __syncthreads();
  } else if constexpr (L / 8 <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + lay.base / L), "n"(L / 8) : "memory");
  }
}

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
      pencil_sync<L, CONTIG>(lay);
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = sm[lay.at(t + T * r)];
      pencil_sync<L, CONTIG>(lay);
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


// Contiguous-axis step programs (IF4_B1..B4, STR_MID) between "tile in
// registers" and "tile ready to store": forward transform, the pointwise
// stage with its operands (u from the shared-memory operand tile `aux`,
// committed one cp.async group before the newest), inverse transform.
// Returns false when the tile is not to be stored (B4 without dst).
template <int L, int PROG, int NT>
__device__ __forceinline__ bool contig_program(double2 (&v)[8], const Args& a, bool valid, int row, int gbase, int t,
                                               int tid, const double2* aux, double2* sbuf, const Lay<L, true>& lay,
                                               const double2* tw, uint64_t& key, uint64_t check_pos) {
  constexpr int T = L / 8;
  const double tau = a.tau;
  if (PROG == FP_STR_MID) {
    fft_pencil<L, true, false>(v, t, sbuf, lay, tw);
    double2 rf[2];
    rf[1] = valid ? row_factor(a, 1, row) : make_double2(0.0, 0.0);
    rf[0] = rf[1];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = cmul(efac(a, 1, rf, t + T * r), v[r]);
    pencil_sync<L, true>(lay);
    fft_pencil<L, true, true>(v, t, sbuf, lay, tw);
    return true;
  }
  fft_pencil<L, true, false>(v, t, sbuf, lay, tw);  // v = g_i (spectral)
  cp_async_wait<1>();                               // the stage operand (the prefetch may fly)
  // The Lawson combination out = E1 (u + t/6 g1) + t/3 E1/2 (g2 + g3) + t/6 g4
  // (integrators.py:205-215) is ACCUMULATED stage by stage in one field `acc`
  // (B1 starts it, B2 and B3 add their term, B4 adds the last and checks), so
  // no stage reads more than one extra operand and g1..g3 are never stored.
  // E1 = E1/2 E1/2 is formed as the square of the E1/2 entry (semigroup property, the same
  // few-ulp difference from a separately rounded E1 table as the FD path's quad form): the
  // passes are LSU-bound and a second table walk per point costs more than four multiplies
  double2 rf[2];
  rf[0] = (valid && PROG != FP_IF4_B4) ? row_factor(a, 0, row) : make_double2(0.0, 0.0);
  rf[1] = rf[0];
  if (valid) {
    // B2 / B3: the running combination of this tile, loaded before the arithmetic needs it
    double2 acc[8];
    if (PROG == FP_IF4_B2 || PROG == FP_IF4_B3) {
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] = ldg_s(a.g[0] + gbase + t + T * r);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = t + T * r;
      const int gi = gbase + i;
      const double2 gi_v = v[r];
      const double2 u = aux[r * NT + tid];  // B1..B3: the state u; B4: the accumulated combination
      if (PROG == FP_IF4_B1) {
        const double2 eh = efac(a, 0, rf, i);
        stg_s(a.g_out + gi, cmul(cmul(eh, eh), caxpy(tau / 6.0, gi_v, u)));
        v[r] = cmul(eh, caxpy(0.5 * tau, gi_v, u));
      } else if (PROG == FP_IF4_B2) {
        const double2 eh = efac(a, 0, rf, i);
        stg_s(a.g_out + gi, caxpy(tau / 3.0, cmul(eh, gi_v), acc[r]));
        v[r] = caxpy(0.5 * tau, gi_v, cmul(eh, u));
      } else if (PROG == FP_IF4_B3) {
        const double2 eh = efac(a, 0, rf, i);
        const double2 ehg = cmul(eh, gi_v);
        stg_s(a.g_out + gi, caxpy(tau / 3.0, ehg, acc[r]));
        v[r] = caxpy(tau, ehg, cmul(cmul(eh, eh), u));
      } else {
        const double2 out = caxpy(tau / 6.0, gi_v, u);
        if (!cfinite(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        stg_s(a.u_out + gi, out);
        v[r] = out;
      }
    }
  }
  if (PROG == FP_IF4_B4 && a.dst == nullptr) return false;
  pencil_sync<L, true>(lay);
  fft_pencil<L, true, true>(v, t, sbuf, lay, tw);
  return true;
}

}  // namespace fftp
}  // namespace cgl
