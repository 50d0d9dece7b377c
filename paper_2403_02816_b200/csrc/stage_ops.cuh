// Pointwise stage building blocks shared by the stage kernels (stages.cu)
// and the stage / slicing prologues of the fused GEMM (ozgemm.cu):
// nonlinearity g, exact cubic and RK4 flows with the reference's divergence
// positions (flows.py:62-133), stage-combination helpers, the stage program
// ids.  See stages.cu for the per-scheme programs.
#pragma once
#include <cstdint>

#include "cgl_common.cuh"

namespace cgl {

constexpr int kStageThreads = 256;

struct StageNL {
  double a3, b3, a4, b4, a5;
  int kind;  // 0 cubic (exact flow), 1 cubic_quintic, 2 coupled, 3 cubic_quintic with the
             // three-term splitting: every flow is a pair of exact flows (strang_3t / split4_3t)
};
constexpr int kKindThreeTerm = 3;

template <int NF>
struct V {
  double2 c[NF];
};

template <int NF>
__device__ __forceinline__ V<NF> load(const double2* const* p, int base, int64_t i, double s) {
  V<NF> v;
#pragma unroll
  for (int c = 0; c < NF; ++c) v.c[c] = cscale(s, ld2(p[base + c] + i));
  return v;
}
template <int NF>
__device__ __forceinline__ void store(double2* const* p, int base, int64_t i, const V<NF>& v) {
#pragma unroll
  for (int c = 0; c < NF; ++c) p[base + c][i] = v.c[c];
}
template <int NF>
__device__ __forceinline__ V<NF> axpy(double s, const V<NF>& x, const V<NF>& y) {  // s*x + y
  V<NF> r;
#pragma unroll
  for (int c = 0; c < NF; ++c) r.c[c] = caxpy(s, x.c[c], y.c[c]);
  return r;
}

template <int NF>
__device__ __forceinline__ V<NF> gfun(const StageNL& p, const V<NF>& u) {
  double m[NF];
#pragma unroll
  for (int c = 0; c < NF; ++c) m[c] = cabs2(u.c[c]);
  V<NF> g;
#pragma unroll
  for (int c = 0; c < NF; ++c) {
    double2 r = cmul(make_double2(p.a3 * m[c], p.b3 * m[c]), u.c[c]);
    if (p.kind != 0) r = cadd(r, cmul(make_double2(p.a4 * (m[c] * m[c]), p.b4 * (m[c] * m[c])), u.c[c]));
    if (p.kind == 2 && NF == 2) r = cadd(r, cscale(p.a5 * m[1 - c], u.c[c]));
    g.c[c] = r;
  }
  return g;
}

__device__ __forceinline__ void note(uint64_t& key, uint64_t pos, unsigned reason) {
  const uint64_t k = pos | reason;
  if (k < key) key = k;
}

// exact cubic flow (flows.py:87-100) of one component at position pos
__device__ __forceinline__ double2 cubic_exact(const StageNL& p, double2 u, double t, uint64_t pos, uint64_t& key) {
  const double m = cabs2(u);
  if (fabs(p.a3) < 1e-14) {
    double sn, cs;
    sincos(p.b3 * m * t, &sn, &cs);
    return cmul(u, make_double2(cs, sn));
  }
  const double y = 2.0 * p.a3 * m * t;
  if (y >= 1.0) note(key, pos, CGL_BLOWUP_CUBIC);
  const double L = log1p(-y);
  // |exp(-L/2)| = (1 - y)^(-1/2): one rsqrt instead of exp (same value to ~1 ulp;
  // 1 - y is exact for y >= 1/2 and rounds once below); the phase needs L
  double sn, cs;
  sincos((-p.b3 / (2.0 * p.a3)) * L, &sn, &cs);
  const double r = rsqrt(1.0 - y);
  const double2 v = cmul(u, make_double2(__dmul_rn(r, cs), __dmul_rn(r, sn)));
  if (!cfinite(v)) note(key, pos, CGL_NONFINITE_CUBIC);
  return v;
}

// exact quintic flow (flows.py:103-115) of one component at position pos;
// |exp(-L/4)| = (1 - y)^(-1/4) as sqrt(rsqrt(1 - y)), the phase from L (as cubic_exact)
__device__ __forceinline__ double2 quintic_exact(const StageNL& p, double2 u, double t, uint64_t pos, uint64_t& key) {
  const double m = cabs2(u), m4 = m * m;
  if (fabs(p.a4) < 1e-14) {
    double sn, cs;
    sincos(p.b4 * m4 * t, &sn, &cs);
    return cmul(u, make_double2(cs, sn));
  }
  const double y = 4.0 * p.a4 * m4 * t;
  if (y >= 1.0) note(key, pos, CGL_BLOWUP_QUINTIC);
  const double L = log1p(-y);
  double sn, cs;
  sincos((-p.b4 / (4.0 * p.a4)) * L, &sn, &cs);
  const double r = sqrt(rsqrt(1.0 - y));
  const double2 v = cmul(u, make_double2(__dmul_rn(r, cs), __dmul_rn(r, sn)));
  if (!cfinite(v)) note(key, pos, CGL_NONFINITE_QUINTIC);
  return v;
}

// one flow call of the scheme: seq positions seq0, seq0+1, ... (exact) or seq0 (rk4).
// Three-term splitting (kind 3, integrators.py:178-195 `_strang3`): the flow over t is
// quintic(t) then cubic(t) at seq0, seq0 + 1 in the first half of a Strang step and
// cubic(t) then quintic(t) in the second half (`second`).
template <int NF>
__device__ __forceinline__ V<NF> flow(const StageNL& p, const V<NF>& u, double t, uint64_t step, int seq0,
                                      uint64_t& key, bool second = false) {
  V<NF> r;
  if (p.kind == kKindThreeTerm) {
    const uint64_t p0 = (step << 24) | ((uint64_t)seq0 << 8), p1 = (step << 24) | ((uint64_t)(seq0 + 1) << 8);
#pragma unroll
    for (int c = 0; c < NF; ++c)
      r.c[c] = second ? quintic_exact(p, cubic_exact(p, u.c[c], t, p0, key), t, p1, key)
                      : cubic_exact(p, quintic_exact(p, u.c[c], t, p0, key), t, p1, key);
    return r;
  }
  if (p.kind == 0) {
#pragma unroll
    for (int c = 0; c < NF; ++c) r.c[c] = cubic_exact(p, u.c[c], t, (step << 24) | ((uint64_t)(seq0 + c) << 8), key);
    return r;
  }
  const double h = 0.5 * t, t6 = t / 6.0;
  const V<NF> k1 = gfun<NF>(p, u);
  const V<NF> k2 = gfun<NF>(p, axpy<NF>(h, k1, u));
  const V<NF> k3 = gfun<NF>(p, axpy<NF>(h, k2, u));
  const V<NF> k4 = gfun<NF>(p, axpy<NF>(t, k3, u));
  bool bad = false;
#pragma unroll
  for (int c = 0; c < NF; ++c) {
    const double2 acc = cadd(cadd(cadd(k1.c[c], cscale(2.0, k2.c[c])), cscale(2.0, k3.c[c])), k4.c[c]);
    r.c[c] = cadd(u.c[c], cscale(t6, acc));
    bad |= !cfinite(r.c[c]);
  }
  if (bad) note(key, (step << 24) | ((uint64_t)seq0 << 8), CGL_NONFINITE_RK4);
  return r;
}

// Boundary of two Strang steps on the exact cubic flow (kind 0).  The reference evaluates
//   out = flow(w, h) at (step, seq1), checks the state, then v = flow(out, h) at (step + 1, 0)
// (integrators.py:161-164 at consecutive steps; flows.py:87-100).  By the semigroup property
// v = flow(w, 2 h): one log1p, one sincos and one rsqrt instead of two of each.  With
// y1 = 2 a3 |w|^2 h computed as the reference computes it, none of its four checks (blow-up
// and non-finite output of either flow, non-finite state) can fire while w is finite and
// y1 < 1/2 (then y2 = 2 a3 |out|^2 h = y1 / (1 - y1) < 1); a guard band of 1e-9 below that
// threshold and every other case take the reference's own two evaluations, so the recorded
// (step, seq, reason) is the reference's.  Returns v; the step's state is flow(w, h), which
// the caller keeps as w and evaluates on demand.
__device__ __forceinline__ double2 cubic_boundary(const StageNL& p, double2 w, double h, uint64_t step, int seq1,
                                                  uint64_t& key) {
  const double m = cabs2(w);
  const double y1 = 2.0 * p.a3 * m * h;
  const bool phase_only = fabs(p.a3) < 1e-14;
  if (cfinite(w) && (phase_only || y1 < 0.5 - 1e-9)) {
    double sn, cs;
    if (phase_only) {
      sincos(p.b3 * m * (2.0 * h), &sn, &cs);
      return cmul(w, make_double2(cs, sn));
    }
    const double y = 2.0 * y1;  // 2 a3 |w|^2 (2 h)
    const double L = log1p(-y);
    sincos((-p.b3 / (2.0 * p.a3)) * L, &sn, &cs);
    const double r = rsqrt(1.0 - y);
    return cmul(w, make_double2(__dmul_rn(r, cs), __dmul_rn(r, sn)));
  }
  const double2 out = cubic_exact(p, w, h, (step << 24) | ((uint64_t)seq1 << 8), key);
  if (!cfinite(out)) note(key, (step << 24) | (255ull << 8), CGL_NONFINITE_STATE);
  return cubic_exact(p, out, h, (step + 1) << 24, key);
}

template <int NF>
__device__ __forceinline__ bool finite_all(const V<NF>& v) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < NF; ++c) ok &= cfinite(v.c[c]);
  return ok;
}

struct StageArgs {
  const double2* in[12];  // up to 5 operands x 2 components (FIF4_S4, coupled)
  double2* out[8];
  int64_t n;
  double tau;
  double in_scale;
  StageNL nl;
  cgl_flag_t* flag;
  uint64_t pos;  // CGL_POS_DEVICE form allowed; low bits ignored (each program knows its seqs)
  int fw;        // flow width: calls per flow() = NF for the exact cubic flow, 1 for RK4
  // Fourier programs: separable exp(f tau symbol) tables, [fraction 1/2, 1][component][axis]
  const double2* tab[2][2][4];
  int64_t ext[4];
  int nd;
  int lg[4];   // log2 ext[d] when every extent is a power of two (pow2), for shift/mask indexing
  int pow2;
  // column-block (transposed) layout of a slab-sharded spectral field: local
  // element (k0, c) of an (n0 x tm) block is global flat k0*t12 + toff + c
  int64_t tm, toff, t12;
};

// exp(f tau symbol) at flat index i (C order) for fraction slot fr, component c
__device__ __forceinline__ double2 sep_factor(const StageArgs& a, int fr, int c, int64_t i) {
  double2 e = make_double2(1.0, 0.0);
  if (a.pow2 && a.tm == 0) {  // power-of-two extents: shifts and masks, no 64-bit divisions
    uint64_t r = (uint64_t)i;
    for (int d = a.nd - 1; d >= 0; --d) {
      e = cmul(e, ld2(a.tab[fr][c][d] + (r & ((1ull << a.lg[d]) - 1ull))));
      r >>= a.lg[d];
    }
    return e;
  }
  int64_t r = a.tm > 0 ? (i / a.tm) * a.t12 + a.toff + (i % a.tm) : i;
  for (int d = a.nd - 1; d >= 0; --d) {
    const int64_t j = r % a.ext[d];
    r /= a.ext[d];
    e = cmul(e, ld2(a.tab[fr][c][d] + j));
  }
  return e;
}

template <int NF>
__device__ __forceinline__ V<NF> emul(const StageArgs& a, int fr, int64_t i, const V<NF>& x) {
  V<NF> r;
#pragma unroll
  for (int c = 0; c < NF; ++c) r.c[c] = cmul(sep_factor(a, fr, c, i), x.c[c]);
  return r;
}

__device__ __forceinline__ void raise_min(cgl_flag_t* f, uint64_t key) {
  // warp-min then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t other = __shfl_xor_sync(0xffffffffu, key, o);
    key = other < key ? other : key;
  }
  if ((threadIdx.x & 31) == 0 && key != ~0ull && f) atomicMin(reinterpret_cast<unsigned long long*>(&f->key),
                                                              (unsigned long long)key);
}

#define STAGE_LOOP for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; \
                        i += (int64_t)gridDim.x * blockDim.x)

enum Prog {
  P_IF4_PRE = 0, P_IF4_MID, P_IF4_END, P_FLOW1, P_FLOW2, P_SPLIT4_MID, P_SPLIT4_END, P_STRANG_END,
  P_IF2_PRE, P_IF2_END,
  // Fourier (spectral-space) programs; g / flows run in physical space between cuFFT calls
  P_FIF4_S1, P_FIF4_S2, P_FIF4_S3, P_FIF4_S4, P_FLOW_END,
  // if4 by the semigroup property E1 = E1/2 E1/2 and linearity (E1/2 X1 = E1/2 u + t/2 E1/2 g1,
  // same for X5); ids 15, 16 are retired (an intermediate five-Tucker form):
  //   [A, G] = E1/2 [u, g1]
  //   MIDQ: u2 = A + t/2 G, w = A + t/6 G; g2 = g(u2); u3 = A + t/2 g2; g3 = g(u3); s = g2 + g3;
  //         p = A + t g3; r = w + t/3 s
  //   [u4, q] = E1/2 [p, r]
  //   ENDQ: out = q + t/6 g(u4); check; g1' = g(out)        -> four half-step Tuckers per step
  P_IF4_MIDQ = 17, P_IF4_ENDQ = 18, P_NPROG
};

}  // namespace cgl
