// Shared device helpers for the B200 CGL integrator (sm_100a).
//
// Field data is complex128 stored as interleaved (re, im) double pairs,
// i.e. `double2` per grid point, C-contiguous (last axis fastest) exactly as
// torch/numpy hold a complex128 tensor of shape (n_1, ..., n_d).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/cgl_b200.h"

namespace cgl {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 caxpy(double s, double2 x, double2 y) {  // s*x + y
  return make_double2(fma(s, x.x, y.x), fma(s, x.y, y.y));
}
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }
// exp(z) for complex z
__device__ __forceinline__ double2 cexp(double2 z) {
  double s, c;
  sincos(z.y, &s, &c);
  double e = exp(z.x);
  return make_double2(e * c, e * s);
}

__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }

// Programmatic dependent launch (kernels launched through launch_k): wait
// until the preceding kernel in the stream has completed and its writes are
// visible (a no-op without the launch attribute); trigger lets the next
// kernel's CTAs start their prologue while this grid finishes.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Sticky divergence record (see include/cgl_b200.h, cgl_flag_t).
//
// key = (step << 24) | (seq << 8) | reason; all-ones = "no divergence".
// A kernel sitting at position `pos` = (step << 24) | (seq << 8) skips its
// work iff an EARLIER position already diverged (key < pos); divergences
// recorded by the kernel's own blocks never make it skip, so every kernel
// either runs completely or not at all.
// ---------------------------------------------------------------------------
// Device-relative positions: step = flag->step (a base advanced once per
// captured chunk of steps) + the local step index baked into pos bits 24..62.
__device__ __forceinline__ uint64_t resolve_pos(const cgl_flag_t* f, uint64_t pos) {
  if (f != nullptr && (pos & CGL_POS_DEVICE)) {
    const uint64_t base = *reinterpret_cast<const volatile unsigned long long*>(&f->step);
    const uint64_t local = (pos & ~CGL_POS_DEVICE) >> 24;
    return ((base + local) << 24) | (pos & 0xFFFFFFull);
  }
  return pos & ~CGL_POS_DEVICE;
}

// pos must already be resolved (resolve_pos)
__device__ __forceinline__ bool flag_skip(const cgl_flag_t* f, uint64_t pos) {
  if (f == nullptr) return false;
  uint64_t k = *reinterpret_cast<const volatile unsigned long long*>(&f->key);
  return k < pos;
}

__device__ __forceinline__ void flag_raise(cgl_flag_t* f, uint64_t pos, unsigned reason) {
  if (f != nullptr) atomicMin(reinterpret_cast<unsigned long long*>(&f->key),
                              (unsigned long long)(pos | reason));
}

// Warp-aggregated raise: one atomic per warp that saw a bad value.
__device__ __forceinline__ void flag_raise_warp(cgl_flag_t* f, uint64_t pos, bool bad, unsigned reason) {
  unsigned m = __ballot_sync(0xffffffffu, bad);
  if (m && (threadIdx.x & 31) == (__ffs(m) - 1)) flag_raise(f, pos, reason);
}

inline int grid_for(int64_t n, int threads, int per_thread = 1) {
  int64_t b = (n + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  // 148 SMs x 8 resident 256-thread CTAs; grid-stride beyond that
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace cgl
