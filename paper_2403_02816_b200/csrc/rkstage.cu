// Explicit Runge-Kutta stages on a finite-difference (Kronecker-sum) operator
// with banded per-direction factors, one launch per stage.
//
// The reference evaluates rhs(u) = K u + g(u) with K u = sum_mu A_mu x_mu u as
// one dense matrix product per direction (integrators.py:146-158 `_step_rk2` /
// `_step_rk4` over Problem.rhs, tensors.py:72-84 `kron_sum_apply`).  The FD
// factors are banded (half-bandwidth 1 or 2: operators.py:40-113), and a dense
// product with an exactly-zero entry adds an exact zero, so the products
// reduce to a (2 b + 1)-point contraction per direction: the stage
//     f = sum_mu A_mu x_mu x + g(x);  x_out = u + cx f;  acc_out = acc_in + ca f
// is ONE pass over the fields (the neighbours come from L1/L2), instead of
// d dense GEMMs, a g kernel and a linear combination.  The host detects the
// bandwidth from the matrices themselves (plan.BandedRKPlan); wider factors
// stay on the generic GEMM path.
//
// Band storage per direction: band[i * (2 b + 1) + d] = A[i][i + d - b]
// (zero outside the matrix).  Fields are C-order complex128, 1..3 dimensions,
// 1 or 2 components (the coupled system carries one operator per component).
#include <cuda_runtime.h>

#include "cgl_common.cuh"
#include "cgl_internal.h"
#include "stage_ops.cuh"

namespace cgl {

constexpr int kRkMaxBand = 8;
constexpr int kRkThreads = 256;

struct RkArgs {
  int nd, nf;
  int n[3];
  int b[3];
  int64_t stride[3];
  int64_t N;
  const double2* band[2][3];
  const double2* x[2];
  const double2* u[2];
  const double2* acc_in[2];
  double2* x_out[2];
  double2* acc_out[2];
  double cx, ca;
  int check;
  StageNL nl;
  cgl_flag_t* flag;
  uint64_t pos;
};

template <int NF>
__global__ void __launch_bounds__(kRkThreads) rk_stage_kernel(const RkArgs a) {
  pdl_wait();
  pdl_trigger();
  const uint64_t step = resolve_pos(a.flag, a.pos) >> 24;
  if (flag_skip(a.flag, step << 24)) return;  // uniform over the grid (the key only grows later)
  uint64_t key = ~0ull;
  const uint64_t check_pos = (step << 24) | (255ull << 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.N; i += (int64_t)gridDim.x * blockDim.x) {
    int idx[3] = {0, 0, 0};
    if (a.N <= 0x7fffffff) {  // 32-bit divisions (every grid up to 1024^3 but itself)
      unsigned r = (unsigned)i;
      for (int mu = a.nd - 1; mu >= 0; --mu) {
        const unsigned q = r / (unsigned)a.n[mu];
        idx[mu] = (int)(r - q * (unsigned)a.n[mu]);
        r = q;
      }
    } else {
      int64_t r = i;
      for (int mu = a.nd - 1; mu >= 0; --mu) {
        idx[mu] = (int)(r % a.n[mu]);
        r /= a.n[mu];
      }
    }
    V<NF> xv, f;
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      xv.c[c] = a.x[c][i];
      double2 s = make_double2(0.0, 0.0);
      for (int mu = 0; mu < a.nd; ++mu) {
        const int b = a.b[mu], w = 2 * b + 1, im = idx[mu];
        const double2* band = a.band[c][mu] + (int64_t)im * w;
        const int d0 = im - b < 0 ? b - im : 0;
        const int d1 = im + b >= a.n[mu] ? a.n[mu] - 1 - im + b : 2 * b;
        double2 t = make_double2(0.0, 0.0);
        for (int d = d0; d <= d1; ++d) {
          const double2 coef = ld2(band + d);
          const double2 v = d == b ? xv.c[c] : ld2(a.x[c] + i + (int64_t)(d - b) * a.stride[mu]);
          // t += coef * v (complex multiply-add, fixed rounding structure)
          t.x = fma(coef.x, v.x, fma(-coef.y, v.y, t.x));
          t.y = fma(coef.x, v.y, fma(coef.y, v.x, t.y));
        }
        s = cadd(s, t);
      }
      f.c[c] = s;
    }
    const V<NF> g = gfun<NF>(a.nl, xv);
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      const double2 fc = cadd(f.c[c], g.c[c]);
      if (a.x_out[c]) a.x_out[c][i] = caxpy(a.cx, fc, a.u[c][i]);
      if (a.acc_out[c]) {
        const double2 base = a.acc_in[c] ? a.acc_in[c][i] : a.u[c][i];
        const double2 out = caxpy(a.ca, fc, base);
        if (a.check && !cfinite(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        a.acc_out[c][i] = out;
      }
    }
  }
  if (a.check) raise_min(a.flag, key);
}

int rk_stage_launch(cudaStream_t st, int ndim, const int64_t* shape, int nf, const int* halfband,
                    const double* const* bands, const cgl_nonlinear_t* nl, const double* const* x,
                    const double* const* u, const double* const* acc_in, double* const* x_out,
                    double* const* acc_out, double cx, double ca, int check, cgl_flag_t* flag, uint64_t pos) {
  if (ndim < 1 || ndim > 3) return set_error(CGL_ESHAPE, "rk_stage: 1..3 dimensions");
  if (nf != 1 && nf != 2) return set_error(CGL_EINVAL, "rk_stage: 1 or 2 components");
  if (!shape || !halfband || !bands || !nl || !x || !u) return set_error(CGL_EINVAL, "rk_stage: null argument");
  if ((nl->kind == 2) != (nf == 2)) return set_error(CGL_EINVAL, "rk_stage: component count does not match kind");
  if (!x_out && !acc_out) return set_error(CGL_EINVAL, "rk_stage: no output");
  RkArgs a{};
  a.nd = ndim;
  a.nf = nf;
  a.N = 1;
  for (int mu = 0; mu < ndim; ++mu) {
    if (shape[mu] < 1 || shape[mu] > (1 << 20)) return set_error(CGL_ESHAPE, "rk_stage: extent");
    if (halfband[mu] < 0 || halfband[mu] > kRkMaxBand) return set_error(CGL_EINVAL, "rk_stage: half-bandwidth 0..8");
    a.n[mu] = (int)shape[mu];
    a.b[mu] = halfband[mu];
    a.N *= shape[mu];
  }
  int64_t s = 1;
  for (int mu = ndim - 1; mu >= 0; --mu) {
    a.stride[mu] = s;
    s *= shape[mu];
  }
  for (int c = 0; c < nf; ++c) {
    for (int mu = 0; mu < ndim; ++mu) {
      a.band[c][mu] = reinterpret_cast<const double2*>(bands[c * ndim + mu]);
      if (!a.band[c][mu]) return set_error(CGL_EINVAL, "rk_stage: null band");
    }
    a.x[c] = reinterpret_cast<const double2*>(x[c]);
    a.u[c] = reinterpret_cast<const double2*>(u[c]);
    a.acc_in[c] = acc_in ? reinterpret_cast<const double2*>(acc_in[c]) : nullptr;
    a.x_out[c] = x_out ? reinterpret_cast<double2*>(x_out[c]) : nullptr;
    a.acc_out[c] = acc_out ? reinterpret_cast<double2*>(acc_out[c]) : nullptr;
    if (!a.x[c] || !a.u[c]) return set_error(CGL_EINVAL, "rk_stage: null field");
    // the contraction reads neighbours of x: it cannot be updated in place
    if ((const void*)a.x[c] == (const void*)a.x_out[c] || (const void*)a.x[c] == (const void*)a.acc_out[c])
      return set_error(CGL_EINVAL, "rk_stage: output aliases the stage input");
  }
  a.cx = cx;
  a.ca = ca;
  a.check = check;
  a.nl = StageNL{nl->alpha3, nl->beta3, nl->alpha4, nl->beta4, nl->alpha5, nl->kind};
  a.flag = flag;
  a.pos = pos;
  const int grid = grid_for(a.N, kRkThreads);
  cudaError_t e = nf == 1 ? launch_k(rk_stage_kernel<1>, dim3(grid), dim3(kRkThreads), 0, st, dim3(1), a)
                          : launch_k(rk_stage_kernel<2>, dim3(grid), dim3(kRkThreads), 0, st, dim3(1), a);
  if (e != cudaSuccess) return set_cuda_error(e, "rk_stage launch");
  return check_launch("rk_stage_kernel");
}

}  // namespace cgl
