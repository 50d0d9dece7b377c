// Cross-mode fused 2D Tucker for small grids (N1 of the scope table; the
// reference chain is tucker_apply, tensors.py:62-69: mode 0 then mode 1).
//
// Out = E0 * In * E1^T for an (n0 x n1) field in ONE launch: CTA i owns output
// row i; phase 1 forms row i of the intermediate T = E0 In in shared memory
// (it never touches HBM), phase 2 contracts it with E1.  The step plans of
// grids below the INT8-emulated engine's threshold (C0: 128^2, where the step
// is launch-latency bound) use it; strang's end-of-step program (flow, check,
// next step's flow) runs in the same kernel, so a C0 strang step is one launch.
//
// The factors exp(f tau A_mu) are numerically banded.  Each output row i of
// E0 reads only its significant band k in [lo_i, hi_i] -- entries below
// 2^-60 of the row's largest magnitude are dropped, a relative change below
// n 2^-60 ~ 1e-16, the same order as the INT8-emulated engine's truncation
// (ozaki.py) and far inside the 1e-10 parity bar; the bands come from
// KroneckerOperator.tucker2d_bands.  FP64 FMA in ascending k.
#include "cgl_common.cuh"
#include "cgl_internal.h"
#include "stage_ops.cuh"

namespace cgl {

constexpr int kT2Threads = 128;
constexpr int kT2MaxN = 1024;

struct T2Item {
  const double2* in;
  double2* out;
  double2* out2;        // STRANG_END: next step's v
  const double2* e0;    // n0 x n0 (row-major)
  const double2* e1t;   // E1^T, n1 x n1 (row k = column k of E1)
  const int2* band0;    // per row i of E0: [lo, hi]
  const int2* band1;    // per row j of E1: [lo, hi]
};

struct T2Args {
  T2Item it[kMaxItems];
  int64_t n0, n1;
  StageNL nl;
  double tau;
  cgl_flag_t* flag;
  uint64_t pos;
  int fw;
};

template <int PROG>
__global__ void __launch_bounds__(kT2Threads) tucker2d_kernel(const T2Args a) {
  __shared__ double2 trow[kT2MaxN];
  __shared__ double2 erow[kT2MaxN];  // row i of E0 inside its band
  pdl_wait();
  pdl_trigger();
  const T2Item& it = a.it[blockIdx.y];
  const uint64_t rpos = resolve_pos(a.flag, a.pos);
  const uint64_t step = rpos >> 24;
  if (PROG == P_STRANG_END) {
    if (flag_skip(a.flag, (step << 24) | ((uint64_t)a.fw << 8))) return;
  } else if (flag_skip(a.flag, rpos)) {
    return;
  }
  const int64_t n0 = a.n0, n1 = a.n1;
  const int64_t i = blockIdx.x;
  // phase 1: T[i, :] = sum_k E0[i, k] In[k, :]
  const int2 b0 = __ldg(it.band0 + i);
  // the band of E0's row is read once, coalesced (constant factor: it does not
  // wait for the previous kernel's data); the loop below then has one
  // independent global load per term and runs 8 terms deep
  for (int k = b0.x + (int)threadIdx.x; k <= b0.y; k += blockDim.x) erow[k - b0.x] = ld2(it.e0 + i * n0 + k);
  __syncthreads();
  for (int64_t j = threadIdx.x; j < n1; j += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 8
    for (int k = b0.x; k <= b0.y; ++k) {
      const double2 e = erow[k - b0.x];
      const double2 x = ld2(it.in + (int64_t)k * n1 + j);
      acc.x = fma(e.x, x.x, fma(-e.y, x.y, acc.x));
      acc.y = fma(e.x, x.y, fma(e.y, x.x, acc.y));
    }
    trow[j] = acc;
  }
  __syncthreads();
  // phase 2: Out[i, j] = sum_k T[i, k] E1[j, k]; a warp walks the union of its
  // columns' bands (in-band entries outside one column's own band are the
  // tiny tails, included exactly)
  uint64_t key = ~0ull;
  for (int64_t j0 = threadIdx.x - (threadIdx.x & 31); j0 < n1; j0 += blockDim.x) {
    const int64_t j = j0 + (threadIdx.x & 31);
    int lo = 1 << 30, hi = -1;
    if (j < n1) {
      const int2 b1 = __ldg(it.band1 + j);
      lo = b1.x;
      hi = b1.y;
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (j >= n1) continue;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 8
    for (int k = lo; k <= hi; ++k) {
      const double2 t = trow[k];
      const double2 e = ld2(it.e1t + (int64_t)k * n1 + j);
      acc.x = fma(t.x, e.x, fma(-t.y, e.y, acc.x));
      acc.y = fma(t.x, e.y, fma(t.y, e.x, acc.y));
    }
    if (PROG == P_STRANG_END) {
      V<1> x;
      x.c[0] = acc;
      const double2 out = flow<1>(a.nl, x, 0.5 * a.tau, step, a.fw, key).c[0];
      if (!cfinite(out)) note(key, (step << 24) | (255ull << 8), CGL_NONFINITE_STATE);
      it.out[i * n1 + j] = out;
      x.c[0] = out;
      it.out2[i * n1 + j] = flow<1>(a.nl, x, 0.5 * a.tau, step + 1, 0, key).c[0];
    } else {
      it.out[i * n1 + j] = acc;
    }
  }
  if (PROG == P_STRANG_END) raise_min(a.flag, key);
}

int tucker2d_launch(cudaStream_t st, int program, int nitems, int64_t n0, int64_t n1, const double* const* in,
                    double* const* out, const double* const* e0, const double* const* e1t, const int* const* band0,
                    const int* const* band1, const cgl_nonlinear_t* nl, double tau, cgl_flag_t* flag,
                    uint64_t pos) {
  if (nitems < 1 || nitems > kMaxItems) return set_error(CGL_EINVAL, "tucker2d: 1..8 items");
  if (n0 < 1 || n1 < 1 || n0 > kT2MaxN || n1 > kT2MaxN) return set_error(CGL_ESHAPE, "tucker2d: n0, n1 <= 1024");
  if (program != 0 && program != 1) return set_error(CGL_EINVAL, "tucker2d: program 0 (plain) or 1 (strang end)");
  program = program == 1 ? P_STRANG_END : -1;
  if (program == P_STRANG_END && (nitems != 1 || !nl || nl->kind >= 2))
    return set_error(CGL_EINVAL, "tucker2d: STRANG_END takes one scalar field");
  T2Args a{};
  for (int q = 0; q < nitems; ++q) {
    if (!in[q] || !out[q] || !e0[q] || !e1t[q] || !band0[q] || !band1[q])
      return set_error(CGL_EINVAL, "tucker2d: null operand");
    a.it[q].in = reinterpret_cast<const double2*>(in[q]);
    a.it[q].out = reinterpret_cast<double2*>(out[q]);
    a.it[q].out2 = program == P_STRANG_END ? reinterpret_cast<double2*>(out[1]) : nullptr;
    a.it[q].e0 = reinterpret_cast<const double2*>(e0[q]);
    a.it[q].e1t = reinterpret_cast<const double2*>(e1t[q]);
    a.it[q].band0 = reinterpret_cast<const int2*>(band0[q]);
    a.it[q].band1 = reinterpret_cast<const int2*>(band1[q]);
  }
  a.n0 = n0;
  a.n1 = n1;
  if (nl) a.nl = StageNL{nl->alpha3, nl->beta3, nl->alpha4, nl->beta4, nl->alpha5, nl->kind};
  a.tau = tau;
  a.flag = flag;
  a.pos = pos;
  a.fw = 1;
  cudaError_t e;
  if (program == P_STRANG_END)
    e = launch_k(tucker2d_kernel<P_STRANG_END>, dim3((unsigned)n0, nitems), dim3(kT2Threads), 0, st, dim3(1), a);
  else
    e = launch_k(tucker2d_kernel<0>, dim3((unsigned)n0, nitems), dim3(kT2Threads), 0, st, dim3(1), a);
  if (e != cudaSuccess) return set_cuda_error(e, "tucker2d launch");
  return check_launch("tucker2d_kernel");
}

CGL_PROF_TU(tucker2d)

}  // namespace cgl
