// cuFFT Z2Z plans for the periodic (Fourier pseudospectral) path:
// dft_forward / dft_inverse of spectral.py:79-86.  cuFFT's backward
// transform is unnormalised; the 1/N of ifftn is folded by the caller into
// the next pointwise kernel (its in_scale argument), so no extra pass.
#include <cufft.h>

#include "cgl_common.cuh"
#include "cgl_internal.h"

namespace cgl {

struct FftPlan {
  cufftHandle h;
  int64_t n;
};

int fft_plan(int ndim, const int64_t* shape, void** out) {
  if (ndim < 1 || ndim > 3) return set_error(CGL_EINVAL, "fft_plan: 1..3 dims");
  long long dims[3];
  int64_t n = 1;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] < 1) return set_error(CGL_ESHAPE, "fft_plan: empty extent");
    dims[d] = shape[d];
    n *= shape[d];
  }
  auto* p = new FftPlan{};
  p->n = n;
  size_t work = 0;
  cufftResult r = cufftCreate(&p->h);
  if (r == CUFFT_SUCCESS)
    r = cufftMakePlanMany64(p->h, ndim, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 1, &work);
  if (r != CUFFT_SUCCESS) {
    delete p;
    return set_error(CGL_ECUFFT, "cufftMakePlanMany64 failed");
  }
  *out = p;
  return 0;
}

// General batched plan (advanced layout): used by the slab-sharded 3D FFT --
// 2D transforms of the local x0-planes and 1D transforms along x0 of the
// transposed (n0 x m) column blocks (istride = m, idist = 1).
int fft_plan_many(int rank, const int64_t* n, int64_t batch, int64_t istride, int64_t idist, int64_t ostride,
                  int64_t odist, void** out) {
  if (rank < 1 || rank > 3) return set_error(CGL_EINVAL, "fft_plan_many: rank 1..3");
  long long dims[3], emb[3];
  int64_t tot = 1;
  for (int d = 0; d < rank; ++d) {
    if (n[d] < 1) return set_error(CGL_ESHAPE, "fft_plan_many: empty extent");
    dims[d] = emb[d] = n[d];
    tot *= n[d];
  }
  auto* p = new FftPlan{};
  p->n = tot;
  size_t work = 0;
  cufftResult r = cufftCreate(&p->h);
  if (r == CUFFT_SUCCESS)
    r = cufftMakePlanMany64(p->h, rank, dims, emb, istride, idist, emb, ostride, odist, CUFFT_Z2Z, batch, &work);
  if (r != CUFFT_SUCCESS) {
    delete p;
    return set_error(CGL_ECUFFT, "cufftMakePlanMany64 (advanced) failed");
  }
  *out = p;
  return 0;
}

int fft_exec(void* plan, cudaStream_t st, const double* in, double* out, int inverse) {
  auto* p = static_cast<FftPlan*>(plan);
  if (!p) return set_error(CGL_EINVAL, "fft_exec: null plan");
  if (cufftSetStream(p->h, st) != CUFFT_SUCCESS) return set_error(CGL_ECUFFT, "cufftSetStream failed");
  cufftResult r = cufftExecZ2Z(p->h, reinterpret_cast<cufftDoubleComplex*>(const_cast<double*>(in)),
                               reinterpret_cast<cufftDoubleComplex*>(out), inverse ? CUFFT_INVERSE : CUFFT_FORWARD);
  if (r != CUFFT_SUCCESS) return set_error(CGL_ECUFFT, "cufftExecZ2Z failed");
  return 0;
}

int fft_destroy(void* plan) {
  auto* p = static_cast<FftPlan*>(plan);
  if (!p) return 0;
  cufftDestroy(p->h);
  delete p;
  return 0;
}

}  // namespace cgl
