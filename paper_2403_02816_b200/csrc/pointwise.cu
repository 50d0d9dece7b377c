// Pointwise kernels: nonlinearity, exact/RK4 flows, stage combinations,
// finiteness checks and Fourier multipliers.  All HBM-bound, one 16-byte
// load/store per complex value per operand, grid-stride loops sized to the
// 148 SMs (cgl_common.cuh:grid_for).
//
// Reference call sites restated here (paths under pkg/src/cglsolve/):
//   eval_g            flows.py:62-78
//   cubic_flow        flows.py:87-100
//   quintic_flow      flows.py:103-115
//   rk4_flow          flows.py:118-133
//   _axpy/_add/_scale integrators.py:130-143
//   isfinite check    integrators.py:274-278
//   pointwise_apply   spectral.py:123-129, symbol_exponential :116-120
#include <cstdint>

#include "cgl_common.cuh"
#include "cgl_internal.h"

namespace cgl {

constexpr int kThreads = 256;
constexpr double kRealCoeffFloor = 1e-14;  // flows.py:29

struct NL {
  double a3, b3, a4, b4, a5;
  int kind;
};
static NL to_nl(const cgl_nonlinear_t* p) {
  NL n{p->alpha3, p->beta3, p->alpha4, p->beta4, p->alpha5, p->kind};
  return n;
}

// g for component with modulus^2 m and the other component's modulus^2 mo
__device__ __forceinline__ double2 g_one(const NL& p, double2 u, double m, double mo) {
  double2 g = cmul(make_double2(p.a3 * m, p.b3 * m), u);
  if (p.kind != 0) g = cadd(g, cmul(make_double2(p.a4 * (m * m), p.b4 * (m * m)), u));
  if (p.kind == 2) g = cadd(g, cscale(p.a5 * mo, u));
  return g;
}

template <int NF>
__device__ __forceinline__ void g_all(const NL& p, const double2 (&u)[NF], double2 (&g)[NF]) {
  double m[NF];
#pragma unroll
  for (int c = 0; c < NF; ++c) m[c] = cabs2(u[c]);
#pragma unroll
  for (int c = 0; c < NF; ++c) g[c] = g_one(p, u[c], m[c], NF == 2 ? m[1 - c] : 0.0);
}

// ---------------------------------------------------------------------------
struct LinArgs {
  const double2* x[6];
  double c[6];
  int nterms;
};

__global__ void lincomb_kernel(int64_t n, LinArgs a, double2* out, const cgl_flag_t* flag, uint64_t pos) {
  CGL_PROF_SCOPE(KID_LINCOMB);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = cscale(a.c[0], ld2(a.x[0] + i));
    for (int t = 1; t < a.nterms; ++t) acc = caxpy(a.c[t], ld2(a.x[t] + i), acc);
    out[i] = acc;
  }
}

template <int NF>
__global__ void eval_g_kernel(int64_t n, NL p, const double2* in0, const double2* in1, double s,
                              double2* out0, double2* out1, const cgl_flag_t* flag, uint64_t pos) {
  CGL_PROF_SCOPE(KID_POINTWISE);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 u[NF], g[NF];
    u[0] = cscale(s, ld2(in0 + i));
    if (NF == 2) u[NF - 1] = cscale(s, ld2(in1 + i));
    g_all<NF>(p, u, g);
    out0[i] = g[0];
    if (NF == 2) out1[i] = g[NF - 1];
  }
}

// Exact flow u * exp(-(a + i b)/(q a) * log1p(-q a |u|^(2r) t)), q = 2 (cubic,
// r = 1) or 4 (quintic, r = 2); phase rotation when |a| < 1e-14.
template <int Q>
__global__ void exact_flow_kernel(int64_t n, double t, double a, double b, const double2* in, double s,
                                  double2* out, cgl_flag_t* flag, uint64_t pos, unsigned r_blow, unsigned r_nonfinite) {
  CGL_PROF_SCOPE(KID_POINTWISE);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  bool blow = false, bad = false;
  const bool phase_only = fabs(a) < kRealCoeffFloor;
  const double fi = -b / (Q * a);  // Im of -(a + i b)/(Q a)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 u = cscale(s, ld2(in + i));
    double m = cabs2(u);
    if (Q == 4) m = m * m;
    double2 v;
    if (phase_only) {
      double sn, cs;
      sincos(b * m * t, &sn, &cs);
      v = cmul(u, make_double2(cs, sn));
    } else {
      const double y = (double)Q * a * m * t;
      if (y >= 1.0) blow = true;
      const double L = log1p(-y);
      // exp((fr + i fi) * L) with fr = -1/2 (cubic: -(a)/(2a)) or -1/4
      v = cmul(u, cexp(make_double2((Q == 2 ? -0.5 : -0.25) * L, fi * L)));
      if (!cfinite(v)) bad = true;
    }
    out[i] = v;
  }
  flag_raise_warp(flag, pos, blow, r_blow);
  flag_raise_warp(flag, pos, bad, r_nonfinite);
}

template <int NF>
__global__ void rk4_flow_kernel(int64_t n, double t, NL p, const double2* in0, const double2* in1, double s,
                                double2* out0, double2* out1, cgl_flag_t* flag, uint64_t pos) {
  CGL_PROF_SCOPE(KID_POINTWISE);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  bool bad = false;
  const double h = 0.5 * t, t6 = t / 6.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 u[NF], k1[NF], k2[NF], k3[NF], k4[NF], w[NF];
    u[0] = cscale(s, ld2(in0 + i));
    if (NF == 2) u[NF - 1] = cscale(s, ld2(in1 + i));
    g_all<NF>(p, u, k1);
#pragma unroll
    for (int c = 0; c < NF; ++c) w[c] = cadd(u[c], cscale(h, k1[c]));
    g_all<NF>(p, w, k2);
#pragma unroll
    for (int c = 0; c < NF; ++c) w[c] = cadd(u[c], cscale(h, k2[c]));
    g_all<NF>(p, w, k3);
#pragma unroll
    for (int c = 0; c < NF; ++c) w[c] = cadd(u[c], cscale(t, k3[c]));
    g_all<NF>(p, w, k4);
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      double2 acc = cadd(cadd(cadd(k1[c], cscale(2.0, k2[c])), cscale(2.0, k3[c])), k4[c]);
      double2 v = cadd(u[c], cscale(t6, acc));
      if (!cfinite(v)) bad = true;
      if (c == 0) out0[i] = v; else out1[i] = v;
    }
  }
  flag_raise_warp(flag, pos, bad, CGL_NONFINITE_RK4);
}

struct FinArgs { const double2* x[4]; int nf; };

__global__ void check_finite_kernel(int64_t n, FinArgs a, cgl_flag_t* flag, uint64_t pos) {
  CGL_PROF_SCOPE(KID_POINTWISE);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < a.nf; ++c) bad |= !cfinite(ld2(a.x[c] + i));
  flag_raise_warp(flag, pos, bad, CGL_NONFINITE_STATE);
}

__global__ void flag_reset_kernel(cgl_flag_t* f) { f->key = ~0ull; }
__global__ void flag_advance_kernel(cgl_flag_t* f, unsigned long long n) {
  CGL_PROF_SCOPE(KID_FLAG_ADV);
  pdl_wait();
  f->step += n;
  pdl_trigger();
}

__global__ void mul_kernel(int64_t n, const double2* f, const double2* in, double2* out, const cgl_flag_t* flag, uint64_t pos) {
  CGL_PROF_SCOPE(KID_POINTWISE);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cmul(ld2(f + i), ld2(in + i));
}

__global__ void symexp_kernel(int64_t n, double s, const double2* sym, double2* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 z = ld2(sym + i);
    out[i] = cexp(make_double2(s * z.x, s * z.y));
  }
}

struct SepArgs {
  const double2* tab[4];
  int64_t ext[4];
  int nd;
  int lg[4], pow2;  // power-of-two extents: shift/mask indexing
  int64_t tm, toff, t12;  // optional column-block layout (see stages.cu)
};

// out[j] = s * prod_mu tab_mu[j_mu] * in[j] (C order: last axis fastest)
__global__ void separable_kernel(int64_t n, SepArgs a, double s, const double2* in, double2* out,
                                 const cgl_flag_t* flag, uint64_t pos) {
  CGL_PROF_SCOPE(KID_SEPARABLE);
  pos = resolve_pos(flag, pos);
  if (flag_skip(flag, pos)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 e = make_double2(s, 0.0);
    if (a.pow2 && a.tm == 0) {
      uint64_t r = (uint64_t)i;
      for (int d = a.nd - 1; d >= 0; --d) {
        e = cmul(e, ld2(a.tab[d] + (r & ((1ull << a.lg[d]) - 1ull))));
        r >>= a.lg[d];
      }
    } else {
      int64_t r = a.tm > 0 ? (i / a.tm) * a.t12 + a.toff + (i % a.tm) : i;
      for (int d = a.nd - 1; d >= 0; --d) {
        const int64_t j = r % a.ext[d];
        r /= a.ext[d];
        e = cmul(e, ld2(a.tab[d] + j));
      }
    }
    out[i] = cmul(e, ld2(in + i));
  }
}

// ---------------------------------------------------------------------------
// launchers (called from capi.cu)
// ---------------------------------------------------------------------------
int pw_lincomb(cudaStream_t st, int64_t n, int nterms, const double* coef, const double* const* x, double* out,
               const cgl_flag_t* flag, uint64_t pos) {
  if (nterms < 1 || nterms > 6) return set_error(CGL_EINVAL, "lincomb: 1..6 terms");
  LinArgs a{};
  a.nterms = nterms;
  for (int t = 0; t < nterms; ++t) { a.x[t] = reinterpret_cast<const double2*>(x[t]); a.c[t] = coef[t]; }
  if (n <= 0) return 0;
  lincomb_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, a, reinterpret_cast<double2*>(out), flag, pos);
  return check_launch("lincomb");
}

int pw_eval_g(cudaStream_t st, int64_t n, const cgl_nonlinear_t* nl, int nf, const double* const* in, double s,
              double* const* out, const cgl_flag_t* flag, uint64_t pos) {
  if (nf != 1 && nf != 2) return set_error(CGL_EINVAL, "eval_g: 1 or 2 components");
  if ((nl->kind == 2) != (nf == 2)) return set_error(CGL_EINVAL, "eval_g: component count does not match kind");
  if (n <= 0) return 0;
  NL p = to_nl(nl);
  auto i0 = reinterpret_cast<const double2*>(in[0]);
  auto o0 = reinterpret_cast<double2*>(out[0]);
  if (nf == 1)
    eval_g_kernel<1><<<grid_for(n, kThreads), kThreads, 0, st>>>(n, p, i0, nullptr, s, o0, nullptr, flag, pos);
  else
    eval_g_kernel<2><<<grid_for(n, kThreads), kThreads, 0, st>>>(n, p, i0, reinterpret_cast<const double2*>(in[1]), s, o0,
                                                                 reinterpret_cast<double2*>(out[1]), flag, pos);
  return check_launch("eval_g");
}

int pw_exact_flow(cudaStream_t st, int quintic, int64_t n, double t, const cgl_nonlinear_t* nl, const double* in,
                  double s, double* out, cgl_flag_t* flag, uint64_t pos) {
  if (n <= 0) return 0;
  auto i0 = reinterpret_cast<const double2*>(in);
  auto o0 = reinterpret_cast<double2*>(out);
  if (!quintic)
    exact_flow_kernel<2><<<grid_for(n, kThreads), kThreads, 0, st>>>(n, t, nl->alpha3, nl->beta3, i0, s, o0, flag, pos,
                                                                      CGL_BLOWUP_CUBIC, CGL_NONFINITE_CUBIC);
  else
    exact_flow_kernel<4><<<grid_for(n, kThreads), kThreads, 0, st>>>(n, t, nl->alpha4, nl->beta4, i0, s, o0, flag, pos,
                                                                      CGL_BLOWUP_QUINTIC, CGL_NONFINITE_QUINTIC);
  return check_launch("exact_flow");
}

int pw_rk4_flow(cudaStream_t st, int64_t n, double t, const cgl_nonlinear_t* nl, int nf, const double* const* in,
                double s, double* const* out, cgl_flag_t* flag, uint64_t pos) {
  if (nf != 1 && nf != 2) return set_error(CGL_EINVAL, "rk4_flow: 1 or 2 components");
  if ((nl->kind == 2) != (nf == 2)) return set_error(CGL_EINVAL, "rk4_flow: component count does not match kind");
  if (n <= 0) return 0;
  NL p = to_nl(nl);
  auto i0 = reinterpret_cast<const double2*>(in[0]);
  auto o0 = reinterpret_cast<double2*>(out[0]);
  if (nf == 1)
    rk4_flow_kernel<1><<<grid_for(n, kThreads), kThreads, 0, st>>>(n, t, p, i0, nullptr, s, o0, nullptr, flag, pos);
  else
    rk4_flow_kernel<2><<<grid_for(n, kThreads), kThreads, 0, st>>>(n, t, p, i0, reinterpret_cast<const double2*>(in[1]), s,
                                                                   o0, reinterpret_cast<double2*>(out[1]), flag, pos);
  return check_launch("rk4_flow");
}

int pw_check_finite(cudaStream_t st, int64_t n, int nf, const double* const* x, cgl_flag_t* flag, uint64_t pos) {
  if (nf < 1 || nf > 4) return set_error(CGL_EINVAL, "check_finite: 1..4 fields");
  if (n <= 0) return 0;
  FinArgs a{};
  a.nf = nf;
  for (int c = 0; c < nf; ++c) a.x[c] = reinterpret_cast<const double2*>(x[c]);
  check_finite_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, a, flag, pos);
  return check_launch("check_finite");
}

int pw_flag_reset(cudaStream_t st, cgl_flag_t* f) {
  flag_reset_kernel<<<1, 1, 0, st>>>(f);
  return check_launch("flag_reset");
}

int pw_flag_advance(cudaStream_t st, cgl_flag_t* f, unsigned long long n) {
  cudaError_t e = launch_k(flag_advance_kernel, dim3(1), dim3(1), 0, st, dim3(1), f, n);
  if (e != cudaSuccess) return set_cuda_error(e, "flag_advance launch");
  return check_launch("flag_advance");
}

int pw_mul(cudaStream_t st, int64_t n, const double* f, const double* in, double* out, const cgl_flag_t* flag, uint64_t pos) {
  if (n <= 0) return 0;
  mul_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, reinterpret_cast<const double2*>(f),
                                                         reinterpret_cast<const double2*>(in),
                                                         reinterpret_cast<double2*>(out), flag, pos);
  return check_launch("pointwise_mul");
}

int pw_symexp(cudaStream_t st, int64_t n, double s, const double* sym, double* out) {
  if (n <= 0) return 0;
  symexp_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, s, reinterpret_cast<const double2*>(sym),
                                                            reinterpret_cast<double2*>(out));
  return check_launch("symbol_exp");
}

int pw_separable(cudaStream_t st, int nd, const int64_t* shape, const double* const* tabs, double s, const double* in,
                 double* out, const cgl_flag_t* flag, uint64_t pos, int64_t tm, int64_t toff) {
  if (nd < 1 || nd > 4) return set_error(CGL_EINVAL, "separable_mul: 1..4 dims");
  SepArgs a{};
  a.nd = nd;
  int64_t n = 1;
  a.pow2 = 1;
  for (int d = 0; d < nd; ++d) {
    a.tab[d] = reinterpret_cast<const double2*>(tabs[d]);
    a.ext[d] = shape[d];
    n *= shape[d];
    int lg = 0;
    while ((1ll << lg) < shape[d]) ++lg;
    a.lg[d] = lg;
    a.pow2 &= (1ll << lg) == shape[d];
  }
  if (tm > 0) {
    a.tm = tm;
    a.toff = toff;
    a.t12 = n / shape[0];
    if (toff + tm > a.t12) return set_error(CGL_ESHAPE, "separable_mul: bad column block");
    n = shape[0] * tm;
  }
  if (n <= 0) return 0;
  separable_kernel<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, a, s, reinterpret_cast<const double2*>(in),
                                                               reinterpret_cast<double2*>(out), flag, pos);
  return check_launch("separable_mul");
}

CGL_PROF_TU(pointwise)

}  // namespace cgl
