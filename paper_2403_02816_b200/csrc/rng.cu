// Seeded inputs on the device: the reference's counter-based stream
// (rng.py:21-64, restated in oracle/cgl_oracle.py): value i of stream `seed`
// is splitmix64(seed + (i + 1) * golden), its top 53 bits -> (0, 1]; normals
// by Box-Muller on consecutive pairs (2k, 2k+1); normal_tensor fills a shape
// in Fortran order.  The integer stream and the uniforms are bit-identical to
// the host; the normals use the device log/sqrt/sin/cos (a few ulp from
// numpy's).  The initial-condition recipes of the workloads (experiments.py
// ICs restated in workloads.py) are evaluated per point from 1D coordinate
// tables, so no N-sized host array is built or copied.
#include <cstdint>

#include "cgl_common.cuh"
#include "cgl_internal.h"

namespace cgl {

__device__ __forceinline__ double stream_uniform(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return ((double)(z >> 11) + 1.0) * (1.0 / 9007199254740992.0);
}

// normal number i of stream seed (pair k = i/2: cos branch for even i, sin for odd)
__device__ __forceinline__ double stream_normal(uint64_t seed, uint64_t i) {
  const uint64_t k = i >> 1;
  const double u1 = stream_uniform(seed, 2 * k), u2 = stream_uniform(seed, 2 * k + 1);
  const double rad = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.141592653589793 * u2;
  return (i & 1) ? rad * sin(ang) : rad * cos(ang);
}

__global__ void uniforms_kernel(uint64_t seed, uint64_t start, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = stream_uniform(seed, start + (uint64_t)i);
}

struct IcArgs {
  int ndim;
  int64_t ext[4];
  const double* axis[4];  // per-axis coordinates
  uint64_t seed;
  int kind;  // 0 sech_noise, 1 gauss_noise, 2 random_phase, 3 noise only (xi_r + i xi_i)
};

// out[c] (C order) = recipe(x) with xi at the Fortran-order stream index of c
__global__ void seeded_ic_kernel(const IcArgs a, int64_t n, double2* out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = c, f = 0, fstride = 1;
    int64_t idx[4];
    for (int d = a.ndim - 1; d >= 0; --d) {
      idx[d] = rem % a.ext[d];
      rem /= a.ext[d];
    }
    for (int d = 0; d < a.ndim; ++d) {
      f += idx[d] * fstride;
      fstride *= a.ext[d];
    }
    const double xr = stream_normal(a.seed, (uint64_t)f), xi = stream_normal(a.seed + 1, (uint64_t)f);
    double r2 = 0.0;
    for (int d = 0; d < a.ndim; ++d) {
      const double x = a.axis[d] ? a.axis[d][idx[d]] : 0.0;
      r2 = r2 + x * x;
    }
    double2 v;
    if (a.kind == 0 || a.kind == 1) {
      // profile * (1 + 0.01 xi), as numpy evaluates real * complex
      const double p = a.kind == 0 ? 1.0 / cosh(sqrt(r2)) : 2.0 * exp(-r2 / 4.0);
      v = make_double2(p * (1.0 + 0.01 * xr), p * (0.01 * xi));
    } else if (a.kind == 2) {
      v = make_double2(0.1 * xr, 0.1 * xi);
    } else {
      v = make_double2(xr, xi);
    }
    out[c] = v;
  }
}

int rng_uniforms(cudaStream_t st, uint64_t seed, uint64_t start, int64_t n, double* out) {
  if (n <= 0) return 0;
  uniforms_kernel<<<grid_for(n, 256), 256, 0, st>>>(seed, start, n, out);
  return check_launch("uniforms_kernel");
}

int rng_seeded_ic(cudaStream_t st, int kind, uint64_t seed, int ndim, const int64_t* shape,
                  const double* const* axes, double* out) {
  if (ndim < 1 || ndim > 4) return set_error(CGL_EINVAL, "seeded_ic: 1..4 dimensions");
  if (kind < 0 || kind > 3) return set_error(CGL_EINVAL, "seeded_ic: unknown recipe");
  IcArgs a{};
  a.ndim = ndim;
  int64_t n = 1;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] <= 0) return 0;
    a.ext[d] = shape[d];
    a.axis[d] = axes ? axes[d] : nullptr;
    n *= shape[d];
  }
  if ((kind == 0 || kind == 1) && !axes) return set_error(CGL_EINVAL, "seeded_ic: profile recipes need axes");
  a.seed = seed;
  a.kind = kind;
  seeded_ic_kernel<<<grid_for(n, 256), 256, 0, st>>>(a, n, reinterpret_cast<double2*>(out));
  return check_launch("seeded_ic_kernel");
}

}  // namespace cgl
