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

// Complex helpers with an explicit rounding structure: every multiply-add is
// either a written fma() or a non-contractible __dmul_rn/__dadd_rn pair, so
// the same expression gives the same bits in every kernel it is inlined
// into (the fused stage+slicing kernels are bit-identical to stage_kernel +
// slicing; compiler FMA contraction would otherwise depend on the context).
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(__dmul_rn(s, a.x), __dmul_rn(s, a.y)); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -__dmul_rn(a.y, b.y)), fma(a.x, b.y, __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 caxpy(double s, double2 x, double2 y) {  // s*x + y
  return make_double2(fma(s, x.x, y.x), fma(s, x.y, y.y));
}
__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, __dmul_rn(a.y, a.y)); }
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

// flag_skip(f, resolve_pos(f, pos)) with key and step read by one 16-byte load
__device__ __forceinline__ bool flag_skip_at(const cgl_flag_t* f, uint64_t pos) {
  if (f == nullptr) return false;
  if (reinterpret_cast<uintptr_t>(f) & 15) return flag_skip(f, resolve_pos(f, pos));  // C callers: 8-byte aligned
  unsigned long long key, base;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(key), "=l"(base) : "l"(f) : "memory");
  if (pos & CGL_POS_DEVICE) pos = ((base + ((pos & ~CGL_POS_DEVICE) >> 24)) << 24) | (pos & 0xFFFFFFull);
  return key < pos;
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

// ---------------------------------------------------------------------------
// In-graph timeline profiling (profiling builds only: -DCGL_PROF, see
// tools/timeline.py).  Every warp of an instrumented kernel appends one
// record {kernel id, block, warp, start, end} (globaltimer ns) when it
// leaves the kernel, so per-launch spans, PDL overlap and per-role warp
// times are visible inside a replayed CUDA graph.  Each translation unit
// holds its own copy of the buffer pointer; cgl_prof_set() fills them all.
// ---------------------------------------------------------------------------
struct CglProfRec {
  long long t0, t1;
  int kid, blk;
  int warp, pad;
};
#ifdef CGL_PROF
static __device__ CglProfRec* g_prof_buf = nullptr;
static __device__ unsigned long long* g_prof_n = nullptr;
static __device__ unsigned g_prof_cap = 0;
struct ProfScope {
  long long t0;
  int kid;
  __device__ __forceinline__ explicit ProfScope(int k) : kid(k) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  }
  __device__ __forceinline__ ~ProfScope() { mark(kid); }
  // one record {t0 = warp start, t1 = now} under id k (lane 0 of the calling warp)
  __device__ __forceinline__ void mark(int k) const {
    if ((threadIdx.x & 31) == 0 && g_prof_buf != nullptr) {
      long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      sm &= 255u;
      // per-SM counters and buffer regions: no cross-SM atomic contention
      const unsigned per = g_prof_cap / 256u;
      const unsigned long long s = atomicAdd(g_prof_n + sm, 1ull);
      if (s < per) {
        CglProfRec r;
        r.t0 = t0;
        r.t1 = t1;
        r.kid = k;
        r.blk = (int)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
        r.warp = (int)(threadIdx.x >> 5);
        r.pad = 0;
        g_prof_buf[(unsigned long long)sm * per + s] = r;
      }
    }
  }
};
#define CGL_PROF_SCOPE(k) ::cgl::ProfScope cgl_prof_scope_(k)
#define CGL_PROF_MARK(k) cgl_prof_scope_.mark(k)
#define CGL_PROF_TU(name)                                                                    \
  int cgl_prof_set_##name(void* buf, void* n, unsigned cap) {                                \
    CglProfRec* b = static_cast<CglProfRec*>(buf);                                           \
    unsigned long long* c = static_cast<unsigned long long*>(n);                             \
    if (cudaMemcpyToSymbol(g_prof_buf, &b, sizeof(b)) != cudaSuccess) return -1;             \
    if (cudaMemcpyToSymbol(g_prof_n, &c, sizeof(c)) != cudaSuccess) return -1;               \
    if (cudaMemcpyToSymbol(g_prof_cap, &cap, sizeof(cap)) != cudaSuccess) return -1;         \
    return 0;                                                                                \
  }
#else
#define CGL_PROF_SCOPE(k) ((void)0)
#define CGL_PROF_MARK(k) ((void)0)
#define CGL_PROF_TU(name) \
  int cgl_prof_set_##name(void*, void*, unsigned) { return -1; }
#endif
// kernel ids (tools/timeline.py)
enum ProfKid {
  KID_SLICE = 1, KID_OZP = 2, KID_STAGE = 3, KID_STAGE_SLICE = 4, KID_FLAG_ADV = 5, KID_SEPARABLE = 6,
  KID_ZGEMM = 7, KID_OZ = 8, KID_ROWEXP = 9, KID_ZMAP = 10, KID_LINCOMB = 11, KID_POINTWISE = 12
};

inline int grid_for(int64_t n, int threads, int per_thread = 1) {
  int64_t b = (n + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  // 148 SMs x 8 resident 256-thread CTAs; grid-stride beyond that
  const int64_t cap = 148 * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace cgl
