// Fused per-scheme stage kernels: every pointwise piece of a time step
// between two exponential (Tucker / Fourier-multiplier) applications runs as
// ONE pass over the grid, reading each operand once and writing each result
// once, with the nonlinearity, the exact / RK4 substep flows, the stage
// combination, the end-of-step finiteness check and the next step's
// prologue all in registers.  Step bodies restated (integrators.py):
//
//   if4   (:205-215)  PRE:  g1 = g(u); X1 = u + t/2 g1; X5 = u + t/6 g1
//                     [u2, a, b, c] = expk([1/2, 1/2, 1, 1], [X1, u, u, X5])
//                     MID:  g2 = g(u2); u3 = a + t/2 g2; g3 = g(u3); s = g2 + g3
//                     [d, e] = expk(1/2, [g3, s])
//                     END:  u4 = b + t d; g4 = g(u4); out = c + t/3 e + t/6 g4
//                           check(out); PRE(out) for the next step
//   strang (:161-164) FLOW1: v = flow(u, t/2)          expk(1, v) -> w
//                     END:  out = flow(w, t/2); check; v' = flow(out, t/2)
//   split4 (:167-175) FLOW2: v = flow(u, t/2) [seq 0], f = flow(u, t/4) [seq 2]
//                     [v, f] = expk([1, 1/2], [v, f])
//                     MID:  c = flow(v, t/2) [seq 1]; f = flow(f, t/2) [seq 3]
//                     f = expk(1/2, f)
//                     END:  fine = flow(f, t/4) [seq 4]; out = 4/3 fine - 1/3 c;
//                           check; FLOW2(out) for the next step
//   if2   (:198-202)  PRE:  g1 = g(u); X = u + t g1; Y = u + t/2 g1
//                     [u2, o] = expk(1, [X, Y])
//                     END:  out = o + t/2 g(u2); check; PRE(out)
//
// "flow" is the exact cubic flow for the cubic kind and one RK4 substep on
// g otherwise (integrators.py:103-110).  Flow seq numbers follow the
// reference's call order (one per component for the exact flow), so the
// recorded first failure is the one the reference would raise.  A kernel
// skips if a failure was recorded before its FIRST flow position.
#include <cstdint>

#include <climits>
#include <cstdlib>
#include <cooperative_groups.h>

#include "cgl_common.cuh"
#include "cgl_internal.h"
#include "oz_slice.cuh"
#include "stage_ops.cuh"
#include "rows_slice.cuh"

namespace cgl {



template <int NF, int PROG>
__global__ void __launch_bounds__(kStageThreads) stage_kernel(const StageArgs a) {
  CGL_PROF_SCOPE(KID_STAGE);
  pdl_wait();  // inputs and the divergence key come from earlier kernels
  pdl_trigger();  // the next kernel may take SMs as this grid drains (its own wait orders the data)
  const cgl_flag_t* cf = a.flag;
  const uint64_t step = resolve_pos(cf, a.pos) >> 24;
  // first flow seq of the program (skip position); non-flow programs: 0
  int first = 0;
  if (PROG == P_SPLIT4_MID) first = a.fw;           // seq w (coarse second flow)
  if (PROG == P_SPLIT4_END) first = (a.nl.kind == kKindThreeTerm ? 5 : 4) * a.fw;  // seq 4w (three-term: 5w)
  if (PROG == P_STRANG_END || PROG == P_FLOW_END) first = a.fw;  // seq w
  const bool is_end = (PROG == P_IF4_END || PROG == P_SPLIT4_END || PROG == P_STRANG_END || PROG == P_IF2_END ||
                       PROG == P_FIF4_S4 || PROG == P_FLOW_END || PROG == P_IF4_ENDH || PROG == P_IF4_ENDQ);
  if (flag_skip(cf, (step << 24) | ((uint64_t)first << 8))) return;  // all CTAs agree (key only grows later)

  uint64_t key = ~0ull;
  const double t = a.tau, s = a.in_scale;
  const uint64_t check_pos = (step << 24) | (255ull << 8);
  STAGE_LOOP {
    if (PROG == P_IF4_PRE || PROG == P_IF2_PRE) {
      const V<NF> u = load<NF>(a.in, 0, i, s);
      const V<NF> g1 = gfun<NF>(a.nl, u);
      store<NF>(a.out, 0, i, axpy<NF>(PROG == P_IF4_PRE ? 0.5 * t : t, g1, u));
      store<NF>(a.out, NF, i, axpy<NF>(PROG == P_IF4_PRE ? t / 6.0 : 0.5 * t, g1, u));
    } else if (PROG == P_IF4_MID) {
      const V<NF> u2 = load<NF>(a.in, 0, i, s), av = load<NF>(a.in, NF, i, s);
      const V<NF> g2 = gfun<NF>(a.nl, u2);
      const V<NF> g3 = gfun<NF>(a.nl, axpy<NF>(0.5 * t, g2, av));
      store<NF>(a.out, 0, i, g3);
      store<NF>(a.out, NF, i, axpy<NF>(1.0, g2, g3));
    } else if (PROG == P_IF4_END) {
      const V<NF> b = load<NF>(a.in, 0, i, s), c = load<NF>(a.in, NF, i, s);
      const V<NF> d = load<NF>(a.in, 2 * NF, i, s), e = load<NF>(a.in, 3 * NF, i, s);
      const V<NF> g4 = gfun<NF>(a.nl, axpy<NF>(t, d, b));
      const V<NF> out = axpy<NF>(t / 6.0, g4, axpy<NF>(t / 3.0, e, c));
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
      const V<NF> g1 = gfun<NF>(a.nl, out);
      store<NF>(a.out, NF, i, axpy<NF>(0.5 * t, g1, out));
      store<NF>(a.out, 2 * NF, i, axpy<NF>(t / 6.0, g1, out));
    } else if (PROG == P_IF4_MIDQ) {
      // semigroup + linearity form: [A, G] = E1/2 [u, g1] -> p, r   (stage_ops.cuh Prog)
      const V<NF> A = load<NF>(a.in, 0, i, s), G = load<NF>(a.in, NF, i, s);
      const V<NF> u2 = axpy<NF>(0.5 * t, G, A), w = axpy<NF>(t / 6.0, G, A);
      const V<NF> g2 = gfun<NF>(a.nl, u2);
      const V<NF> g3 = gfun<NF>(a.nl, axpy<NF>(0.5 * t, g2, A));
      store<NF>(a.out, 0, i, axpy<NF>(t, g3, A));
      store<NF>(a.out, NF, i, axpy<NF>(t / 3.0, axpy<NF>(1.0, g2, g3), w));
    } else if (PROG == P_IF4_ENDQ) {
      // out = q + t/6 g(u4); check; g1 of the next step
      const V<NF> u4 = load<NF>(a.in, 0, i, s), q = load<NF>(a.in, NF, i, s);
      const V<NF> out = axpy<NF>(t / 6.0, gfun<NF>(a.nl, u4), q);
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
      store<NF>(a.out, NF, i, gfun<NF>(a.nl, out));
    } else if (PROG == P_IF4_MIDH) {
      // semigroup form: p = a + t g3, r = w + t/3 (g2 + g3)   (stage_ops.cuh Prog)
      const V<NF> u2 = load<NF>(a.in, 0, i, s), av = load<NF>(a.in, NF, i, s), w = load<NF>(a.in, 2 * NF, i, s);
      const V<NF> g2 = gfun<NF>(a.nl, u2);
      const V<NF> g3 = gfun<NF>(a.nl, axpy<NF>(0.5 * t, g2, av));
      store<NF>(a.out, 0, i, axpy<NF>(t, g3, av));
      store<NF>(a.out, NF, i, axpy<NF>(t / 3.0, axpy<NF>(1.0, g2, g3), w));
    } else if (PROG == P_IF4_ENDH) {
      // semigroup form: out = q + t/6 g(u4); check; PRE(out)
      const V<NF> u4 = load<NF>(a.in, 0, i, s), q = load<NF>(a.in, NF, i, s);
      const V<NF> out = axpy<NF>(t / 6.0, gfun<NF>(a.nl, u4), q);
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
      const V<NF> g1 = gfun<NF>(a.nl, out);
      store<NF>(a.out, NF, i, axpy<NF>(0.5 * t, g1, out));
      store<NF>(a.out, 2 * NF, i, axpy<NF>(t / 6.0, g1, out));
    } else if (PROG == P_FLOW1) {
      // strang prologue: v = flow(u, t/2) at seq 0 of `step`
      const V<NF> u = load<NF>(a.in, 0, i, s);
      store<NF>(a.out, 0, i, flow<NF>(a.nl, u, 0.5 * t, step, 0, key));
    } else if (PROG == P_FLOW2) {
      // split4 prologue: v = flow(u, t/2) [seq 0], f = flow(u, t/4) [seq 2w]
      const V<NF> u = load<NF>(a.in, 0, i, s);
      store<NF>(a.out, 0, i, flow<NF>(a.nl, u, 0.5 * t, step, 0, key));
      store<NF>(a.out, NF, i, flow<NF>(a.nl, u, 0.25 * t, step, 2 * a.fw, key));
    } else if (PROG == P_SPLIT4_MID) {
      const V<NF> v = load<NF>(a.in, 0, i, s), f = load<NF>(a.in, NF, i, s);
      store<NF>(a.out, 0, i, flow<NF>(a.nl, v, 0.5 * t, step, a.fw, key, true));
      if (a.nl.kind == kKindThreeTerm) {
        // the two quarter-step flows either side of the fine substep boundary do not
        // merge: end of fine substep 1 (seq 3w), start of fine substep 2 (seq 4w)
        const V<NF> f1 = flow<NF>(a.nl, f, 0.25 * t, step, 3 * a.fw, key, true);
        store<NF>(a.out, NF, i, flow<NF>(a.nl, f1, 0.25 * t, step, 4 * a.fw, key));
      } else {
        store<NF>(a.out, NF, i, flow<NF>(a.nl, f, 0.5 * t, step, 3 * a.fw, key));
      }
    } else if (PROG == P_SPLIT4_END) {
      const V<NF> f = load<NF>(a.in, 0, i, s), c = load<NF>(a.in, NF, i, s);
      const V<NF> fine = flow<NF>(a.nl, f, 0.25 * t, step, (a.nl.kind == kKindThreeTerm ? 5 : 4) * a.fw, key, true);
      V<NF> out;
#pragma unroll
      for (int q = 0; q < NF; ++q) out.c[q] = cadd(cscale(4.0 / 3.0, fine.c[q]), cscale(-1.0 / 3.0, c.c[q]));
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
      store<NF>(a.out, NF, i, flow<NF>(a.nl, out, 0.5 * t, step + 1, 0, key));
      store<NF>(a.out, 2 * NF, i, flow<NF>(a.nl, out, 0.25 * t, step + 1, 2 * a.fw, key));
    } else if (PROG == P_STRANG_END) {
      const V<NF> w = load<NF>(a.in, 0, i, s);
      const V<NF> out = flow<NF>(a.nl, w, 0.5 * t, step, a.fw, key, true);
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
      store<NF>(a.out, NF, i, flow<NF>(a.nl, out, 0.5 * t, step + 1, 0, key));
    } else if (PROG == P_FIF4_S1) {
      // u2 = E1/2 (u + t/2 g1)
      const V<NF> u = load<NF>(a.in, 0, i, s), g1 = load<NF>(a.in, NF, i, s);
      store<NF>(a.out, 0, i, emul<NF>(a, 0, i, axpy<NF>(0.5 * t, g1, u)));
    } else if (PROG == P_FIF4_S2) {
      // u3 = E1/2 u + t/2 g2
      const V<NF> u = load<NF>(a.in, 0, i, s), g2 = load<NF>(a.in, NF, i, s);
      store<NF>(a.out, 0, i, axpy<NF>(0.5 * t, g2, emul<NF>(a, 0, i, u)));
    } else if (PROG == P_FIF4_S3) {
      // u4 = t E1/2 g3 + E1 u
      const V<NF> u = load<NF>(a.in, 0, i, s), g3 = load<NF>(a.in, NF, i, s);
      store<NF>(a.out, 0, i, axpy<NF>(t, emul<NF>(a, 0, i, g3), emul<NF>(a, 1, i, u)));
    } else if (PROG == P_FIF4_S4) {
      // out = E1 (u + t/6 g1) + t/3 E1/2 (g2 + g3) + t/6 g4
      const V<NF> u = load<NF>(a.in, 0, i, s), g1 = load<NF>(a.in, NF, i, s);
      const V<NF> g2 = load<NF>(a.in, 2 * NF, i, s), g3 = load<NF>(a.in, 3 * NF, i, s);
      const V<NF> g4 = load<NF>(a.in, 4 * NF, i, s);
      const V<NF> out = axpy<NF>(t / 6.0, g4, axpy<NF>(t / 3.0, emul<NF>(a, 0, i, axpy<NF>(1.0, g2, g3)),
                                                       emul<NF>(a, 1, i, axpy<NF>(t / 6.0, g1, u))));
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
    } else if (PROG == P_FLOW_END) {
      // out = flow(w, t/2) at seq w; finiteness of the physical result stands in for the
      // spectral state's (an FFT of finite values is finite barring overflow)
      const V<NF> w = load<NF>(a.in, 0, i, s);
      const V<NF> out = flow<NF>(a.nl, w, 0.5 * t, step, a.fw, key, true);
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
    } else if (PROG == P_IF2_END) {
      const V<NF> u2 = load<NF>(a.in, 0, i, s), o = load<NF>(a.in, NF, i, s);
      const V<NF> out = axpy<NF>(0.5 * t, gfun<NF>(a.nl, u2), o);
      if (!finite_all<NF>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
      store<NF>(a.out, 0, i, out);
      const V<NF> g1 = gfun<NF>(a.nl, out);
      store<NF>(a.out, NF, i, axpy<NF>(t, g1, out));
      store<NF>(a.out, 2 * NF, i, axpy<NF>(0.5 * t, g1, out));
    }
  }
  raise_min(a.flag, key);
  (void)is_end;
}

// ---- fused stage + data slicing (INT8-emulated products, if4 on FD grids) ----
// The if4 stage outputs X1, X5 (END) and g3, s (MID) are consumed only as the
// data operands of the next axis-0 mu-mode products, so they are never stored
// in FP64: a cluster of CTAs spanning the axis-0 range of 32 consecutive
// columns q of the (n0 x Q) field view computes the stage pointwise on its
// block, stores the state u (END) in FP64, keeps the sliced outputs in shared
// memory, exchanges partial column exponents through DSMEM (one cluster
// barrier) and emits the floor-digit slices in the GEMM's B-operand layout
// (Z = In^T: rows q, K = axis-0 index; exactly what cgl_oz_slice_multi
// produces for the same field).  One pass instead of a stage kernel plus a
// slicing kernel per field.
struct StageSliceArgs {
  StageArgs s;        // inputs; s.out[0] = u (END only)
  int8_t* slices[3];  // per sliced output: B-mode slices (rows Q, K n0)
  int* exps[3];       // per sliced output: row (= column q) exponents
  int64_t Q, n0;
  int nchunks;
};

#ifndef SS_THREADS
#define SS_THREADS 256
#endif
constexpr int kSSThreads = SS_THREADS;  // threads per CTA of the fused stage+slicing kernel
constexpr int kSSParts = kSSThreads / 32;

template <int PROG, int NSL, int CPBT>
__global__ void __launch_bounds__(kSSThreads) stage_slice_kernel(const StageSliceArgs A) {
  CGL_PROF_SCOPE(KID_STAGE_SLICE);
  namespace cg = cooperative_groups;
  using oz::KC;
  using oz::NONFINITE;
  constexpr int CR = 32;                 // Z rows (columns q) per tile = the GEMM's B row tile
  constexpr int CC = KC / 2;             // complex K per chunk
  constexpr int W = CC * CPBT;           // complex K per CTA
  constexpr int PT = CR * W / kSSThreads;  // points per thread
  static_assert(PT >= 1 && CR * W % kSSThreads == 0, "tile / CTA size");
  static_assert(kOzBN == CR, "B row tile");
  pdl_wait();
  pdl_trigger();  // as rows_slice_kernel: the GEMM's setup overlaps this grid's tail
  CGL_PROF_MARK(201);
  const StageArgs& a = A.s;
  const cgl_flag_t* cf = a.flag;
  const uint64_t step = resolve_pos(cf, a.pos) >> 24;
  int first = 0;  // first flow seq of the program (as stage_kernel)
  if (PROG == P_SPLIT4_MID || PROG == P_STRANG_END) first = a.fw;
  if (PROG == P_SPLIT4_END) first = 4 * a.fw;
  if (flag_skip(cf, (step << 24) | ((uint64_t)first << 8))) return;  // uniform over the grid
  uint64_t key = ~0ull;
  const uint64_t check_pos = (step << 24) | (255ull << 8);
  const double t = a.tau, sc = a.in_scale;
  extern __shared__ double2 blk[];  // [NSL][CR][W + 1]
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * CR, c0 = (int64_t)blockIdx.y * W;
  const int rows_here = (int)min((int64_t)CR, A.Q - r0), cols_here = (int)min((int64_t)W, A.n0 - c0);
  // ---- stage, pointwise (consecutive threads: consecutive q, coalesced) ----
#pragma unroll 2
  for (int j = 0; j < PT; ++j) {
    const int k = tid + kSSThreads * j, rr = k % CR, cc = k / CR;
    double2 o[NSL];
#pragma unroll
    for (int q = 0; q < NSL; ++q) o[q] = make_double2(0.0, 0.0);
    if (rr < rows_here && cc < cols_here) {
      const int64_t i = (c0 + cc) * A.Q + (r0 + rr);
      if (PROG == P_IF4_MID) {
        const V<1> u2 = load<1>(a.in, 0, i, sc), av = load<1>(a.in, 1, i, sc);
        const V<1> g2 = gfun<1>(a.nl, u2);
        const V<1> g3 = gfun<1>(a.nl, axpy<1>(0.5 * t, g2, av));
        o[0] = g3.c[0];
        o[1] = axpy<1>(1.0, g2, g3).c[0];
      } else if (PROG == P_STRANG_END) {
        const V<1> w = load<1>(a.in, 0, i, sc);
        const V<1> out = flow<1>(a.nl, w, 0.5 * t, step, a.fw, key);
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        store<1>(a.out, 0, i, out);
        o[0] = flow<1>(a.nl, out, 0.5 * t, step + 1, 0, key).c[0];              // v of step + 1
      } else if (PROG == P_SPLIT4_MID) {
        const V<1> v = load<1>(a.in, 0, i, sc), f = load<1>(a.in, 1, i, sc);
        store<1>(a.out, 0, i, flow<1>(a.nl, v, 0.5 * t, step, a.fw, key));     // coarse c (FP64)
        o[0] = flow<1>(a.nl, f, 0.5 * t, step, 3 * a.fw, key).c[0];             // f (sliced only)
      } else if (PROG == P_SPLIT4_END) {
        const V<1> f = load<1>(a.in, 0, i, sc), c = load<1>(a.in, 1, i, sc);
        const V<1> fine = flow<1>(a.nl, f, 0.25 * t, step, 4 * a.fw, key);
        V<1> out;
        out.c[0] = cadd(cscale(4.0 / 3.0, fine.c[0]), cscale(-1.0 / 3.0, c.c[0]));
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        store<1>(a.out, 0, i, out);
        o[0] = flow<1>(a.nl, out, 0.5 * t, step + 1, 0, key).c[0];              // v of step + 1
        o[1] = flow<1>(a.nl, out, 0.25 * t, step + 1, 2 * a.fw, key).c[0];      // f of step + 1
      } else {  // P_IF4_END
        const V<1> b = load<1>(a.in, 0, i, sc), c = load<1>(a.in, 1, i, sc);
        const V<1> d = load<1>(a.in, 2, i, sc), e = load<1>(a.in, 3, i, sc);
        const V<1> g4 = gfun<1>(a.nl, axpy<1>(t, d, b));
        const V<1> out = axpy<1>(t / 6.0, g4, axpy<1>(t / 3.0, e, c));
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        store<1>(a.out, 0, i, out);
        const V<1> g1 = gfun<1>(a.nl, out);
        o[0] = axpy<1>(0.5 * t, g1, out).c[0];   // X1
        o[1] = out.c[0];                          // u
        o[2] = axpy<1>(t / 6.0, g1, out).c[0];    // X5
      }
    }
#pragma unroll
    for (int q = 0; q < NSL; ++q) blk[(q * CR + rr) * (W + 1) + cc] = o[q];
  }
  __syncthreads();
  CGL_PROF_MARK(202);
  // ---- partial exponents of the 32 Z rows per output, exchanged in the cluster ----
  __shared__ double red[NSL][kSSParts][33];
  __shared__ int redbad[NSL][kSSParts][32];
  __shared__ int epart[NSL][16][32];  // [output][cluster rank][row]
  __shared__ int erow[NSL][32];
  cg::cluster_group cluster = cg::this_cluster();
  {
    const int rr = tid & 31, part = tid >> 5;
#pragma unroll
    for (int q = 0; q < NSL; ++q) {
      double m = 0.0;
      bool bad = false;
      for (int cc = part; cc < cols_here; cc += kSSParts) {
        const double2 v = blk[(q * CR + rr) * (W + 1) + cc];
        bad |= !isfinite(v.x) || !isfinite(v.y);
        m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
      }
      red[q][part][rr] = m;
      redbad[q][part][rr] = bad;
    }
  }
  __syncthreads();
  if (tid < 32 * NSL) {
    const int q = tid >> 5, rr = tid & 31;
    double m = red[q][0][rr];
    int bad = redbad[q][0][rr];
    for (int k = 1; k < kSSParts; ++k) {
      m = fmax(m, red[q][k][rr]);
      bad |= redbad[q][k][rr];
    }
    int e = INT_MIN;
    if (bad) e = NONFINITE;
    else if (m > 0.0) frexp(m, &e);
    const unsigned me = cluster.block_rank(), nb = cluster.num_blocks();
    for (unsigned rk = 0; rk < nb; ++rk) cluster.map_shared_rank(&epart[0][0][0], rk)[(q * 16 + me) * 32 + rr] = e;
  }
  cluster.sync();
  CGL_PROF_MARK(203);
  if (tid < 32 * NSL) {
    const int q = tid >> 5, rr = tid & 31;
    int e = INT_MIN;
    for (unsigned rk = 0; rk < cluster.num_blocks(); ++rk) e = max(e, epart[q][rk][rr]);
    if (e == INT_MIN) e = 0;  // all-zero row (same convention as the slicing kernels)
    erow[q][rr] = e;
    if (blockIdx.y == 0 && rr < rows_here) A.exps[q][r0 + rr] = e;
  }
  __syncthreads();
  // ---- slices (same digits and layout as slice_tile_kernel<8, 0>) ----
  constexpr int NG = KC / 16, groups = CPBT * NG;
  const int ch0 = blockIdx.y * CPBT;
  for (int w = tid; w < NSL * CR * groups; w += kSSThreads) {
    const int q = w / (CR * groups), rem = w % (CR * groups);
    const int rr = rem % CR, gg = rem / CR;
    const int ch = ch0 + gg / NG, g = gg % NG;
    if (rr >= rows_here || ch >= A.nchunks) continue;
    const int e = erow[q][rr];
    uint32_t wv[8][4];
#pragma unroll
    for (int s8 = 0; s8 < 8; ++s8) wv[s8][0] = wv[s8][1] = wv[s8][2] = wv[s8][3] = 0u;
    if (e != NONFINITE) {
      const double2* row = blk + (q * CR + rr) * (W + 1) + (gg / NG) * CC + g * 8;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 v0 = row[2 * k], v1 = row[2 * k + 1];
        const double x[4] = {v0.x, v0.y, v1.x, v1.y};
        uint32_t ww[8];
        oz::words8_floor(x, e, ww);
#pragma unroll
        for (int s8 = 0; s8 < 8; ++s8) wv[s8][k] = ww[s8];
      }
    }
    int8_t* dst = A.slices[q] + oz::tile_offset(r0 + rr, (int64_t)ch * KC + g * 16, CR, A.nchunks, 8);
#pragma unroll
    for (int s8 = 0; s8 < 8; ++s8)
      *reinterpret_cast<uint4*>(dst + s8 * (CR * KC)) = make_uint4(wv[s8][0], wv[s8][1], wv[s8][2], wv[s8][3]);
  }
  raise_min(a.flag, key);
}


template <int PROG, int NSL, int TPT, int PP = 8, int NT = kRSThreads>
__global__ void __launch_bounds__(NT) rows_slice_kernel(const RowsSliceArgs A) {
  CGL_PROF_SCOPE(PROG == P_SLICE ? KID_SLICE : KID_STAGE_SLICE);
  __shared__ RowsSliceSmem sm;
  pdl_wait();
  // every CTA of this grid is resident by now at the step sizes: let the next
  // kernel (the GEMM) take SMs as they drain -- its setup (barriers, TMEM,
  // first live-chunk list, constant-factor copy) then overlaps this tail
  pdl_trigger();
  CGL_PROF_MARK(201);
  if (A.debug & 8) return;  // timing experiment: launch + wait only
  rows_slice_block<PROG, NSL, TPT, PP, NT>(A, blockIdx.x, blockIdx.y, threadIdx.x, 0, sm);
}

// QC rows per CTA: NT threads cover QC * KG tasks (PP complex each) in TPT
// rounds; the smallest QC that fills the threads (measured: fewer, larger CTAs
// are slower; CGL_RS_TARGET > 0 grows QC until the grid is about that many CTAs).
int rows_slice_qc(int64_t K, int64_t rows_total, int tpt_max, int* tpt, int pp, int nt) {
  const int64_t KG = (K + pp - 1) / pp;
  static const int target = [] {
    const char* e = getenv("CGL_RS_TARGET");
    return e ? atoi(e) : 0;
  }();
  int qc = 2;
  while (qc < 32 && qc * KG < nt) qc <<= 1;
  while (target > 0 && qc < 32 && rows_total / qc > target && (2 * qc) * KG <= (int64_t)tpt_max * nt) qc <<= 1;
  *tpt = (int)((qc * KG + nt - 1) / nt);
  return qc;
}
int rows_slice_qc(int64_t K, int64_t rows_total, int tpt_max, int* tpt) {
  return rows_slice_qc(K, rows_total, tpt_max, tpt, 8, kRSThreads);
}

// 4-point tasks on 256-thread CTAs: twice the warps of the 8-point /
// 128-thread form at the same rows per CTA.  Measured on C1: MIDQ 7.4 -> 6.4,
// ENDQ 7.6 -> 7.1, MID 6.6 -> 6.2, END 10.6 -> 9.6, 2-field slicing 5.9 -> 5.0
// us; at 256^3 the stage programs are 3-11 % faster but the HBM-bound plain
// slicing slower (90 -> 80 % of HBM).  Stage programs: always; plain slicing:
// when the launch's data are L2-sized.  CGL_RS_PP (stage) / CGL_RS_PP_SLICE
// (plain) = 4 or 8 force.
static int rows_pp(bool stage, double bytes) {
  static const int pp_stage = [] {
    const char* e = getenv("CGL_RS_PP");
    return e ? atoi(e) : 4;
  }();
  static const int pp_slice = [] {
    const char* e = getenv("CGL_RS_PP_SLICE");
    return e ? atoi(e) : 0;
  }();
  if (stage) return pp_stage;
  return pp_slice ? pp_slice : (bytes <= 64.0 * (1 << 20) ? 4 : 8);
}

template <int PROG, int NSL>
static cudaError_t launch_rows_slice(RowsSliceArgs& A, int64_t gy, cudaStream_t st) {
  int tpt = 1;
  {
    const double bytes = 16.0 * (double)A.rows * (double)gy * (double)A.K;
    int tpt4 = 1;
    const int qc4 = rows_slice_qc(A.K, A.rows * gy, 2, &tpt4, 4, 256);
    if (rows_pp(PROG != P_SLICE, bytes) == 4 && tpt4 <= 2) {
      A.QC = qc4;
      tpt = tpt4;
      const dim3 grid((unsigned)((A.rows + A.QC - 1) / A.QC), (unsigned)gy, 1);
      if (tpt == 1) return launch_k(rows_slice_kernel<PROG, NSL, 1, 4, 256>, grid, dim3(256), 0, st, dim3(1), A);
      if (tpt == 2) return launch_k(rows_slice_kernel<PROG, NSL, 2, 4, 256>, grid, dim3(256), 0, st, dim3(1), A);
      return cudaErrorInvalidValue;
    }
  }
  A.QC = rows_slice_qc(A.K, A.rows * gy, PROG == P_SLICE ? 4 : 2, &tpt);
  const dim3 grid((unsigned)((A.rows + A.QC - 1) / A.QC), (unsigned)gy, 1);
  switch (tpt) {
    case 1: return launch_k(rows_slice_kernel<PROG, NSL, 1>, grid, dim3(kRSThreads), 0, st, dim3(1), A);
    case 2: return launch_k(rows_slice_kernel<PROG, NSL, 2>, grid, dim3(kRSThreads), 0, st, dim3(1), A);
    default: break;
  }
  if constexpr (PROG == P_SLICE) {  // stage programs stop at TPT = 2 (register-resident stage outputs)
    if (tpt == 3) return launch_k(rows_slice_kernel<PROG, NSL, 3>, grid, dim3(kRSThreads), 0, st, dim3(1), A);
    if (tpt == 4) return launch_k(rows_slice_kernel<PROG, NSL, 4>, grid, dim3(kRSThreads), 0, st, dim3(1), A);
  }
  return cudaErrorInvalidValue;
}

// plain slicing: K <= 2048 (TPT <= 4); stage programs: K <= 1024 (TPT <= 2)
bool rows_slice_ok(int64_t K, bool stage) { return K >= 1 && (K + 7) / 8 <= (stage ? 2 : 4) * kRSThreads / 2; }

int rows_slice_plain(cudaStream_t st, int nitems, const double* const* srcs, int64_t sr, int64_t sk, int64_t rows,
                     int64_t K, int64_t batch, int64_t src_bs, int8_t* const* outs, int64_t out_bs,
                     int* const* exps, int64_t exp_bs) {
  if (!rows_slice_ok(K, false)) return set_error(CGL_ESHAPE, "rows_slice: K extent too large");
  if (batch * nitems > 65535) return set_error(CGL_ESHAPE, "rows_slice: batch x items too large");
  RowsSliceArgs A{};
  for (int f = 0; f < nitems; ++f) {
    A.srcs[f] = reinterpret_cast<const double2*>(srcs[f]);
    A.slices[f] = outs[f];
    A.exps[f] = exps[f];
  }
  A.src_bs = src_bs;
  A.out_bs = out_bs;
  A.exp_bs = exp_bs;
  A.batch = batch;
  A.rows = rows;
  A.K = K;
  A.sr = sr;
  A.sk = sk;
  A.nchunks = (int)((2 * K + oz::KC - 1) / oz::KC);
  {
    const char* d = getenv("CGL_RS_DEBUG");
    A.debug = d ? atoi(d) : 0;
  }
  cudaError_t e = launch_rows_slice<P_SLICE, 1>(A, batch * nitems, st);
  if (e != cudaSuccess) return set_cuda_error(e, "rows_slice launch");
  return check_launch("rows_slice_kernel");
}

template <int PROG, int NSL, int CPBT>
static cudaError_t launch_stage_slice(const StageSliceArgs& A, cudaStream_t st) {
  constexpr int W = (oz::KC / 2) * CPBT;
  const int cy = (A.nchunks + CPBT - 1) / CPBT;
  const size_t smem = (size_t)NSL * 32 * (W + 1) * sizeof(double2);
  auto kern = stage_slice_kernel<PROG, NSL, CPBT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  const dim3 grid((unsigned)((A.Q + 31) / 32), (unsigned)cy, 1);
  return launch_k(kern, grid, dim3(kSSThreads), smem, st, dim3(1, (unsigned)cy, 1), A);
}

int stage_slice_launch(cudaStream_t st, int prog, int64_t n0, int64_t Q, const cgl_nonlinear_t* nl, double tau,
                       double in_scale, const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos,
                       int8_t* const* slices, int* const* exps) {
  int nin, nsl, nout;
  switch (prog) {
    case P_IF4_MID: nin = 2; nsl = 2; nout = 0; break;
    case P_IF4_END: nin = 4; nsl = 3; nout = 1; break;
    case P_IF4_MIDH: nin = 3; nsl = 2; nout = 0; break;
    case P_IF4_ENDH: nin = 2; nsl = 3; nout = 1; break;
    case P_IF4_MIDQ: nin = 2; nsl = 2; nout = 0; break;
    case P_IF4_ENDQ: nin = 2; nsl = 2; nout = 1; break;
    case P_STRANG_END: nin = 1; nsl = 1; nout = 1; break;
    case P_SPLIT4_MID: nin = 2; nsl = 1; nout = 1; break;
    case P_SPLIT4_END: nin = 2; nsl = 2; nout = 1; break;
    default: return set_error(CGL_EINVAL, "stage_slice: if4 MID/END (+ half-step forms), strang END, split4 MID/END only");
  }
  if (n0 <= 0 || Q <= 0) return 0;
  if (nout && (!out || !out[0])) return set_error(CGL_EINVAL, "stage_slice: program writes an FP64 output");
  StageSliceArgs A{};
  StageArgs& a = A.s;
  for (int k = 0; k < nin; ++k) a.in[k] = reinterpret_cast<const double2*>(in[k]);
  if (nout) a.out[0] = reinterpret_cast<double2*>(out[0]);
  a.n = n0 * Q;
  a.tau = tau;
  a.in_scale = in_scale;
  a.nl.a3 = nl->alpha3;
  a.nl.b3 = nl->beta3;
  a.nl.a4 = nl->alpha4;
  a.nl.b4 = nl->beta4;
  a.nl.a5 = nl->alpha5;
  a.nl.kind = nl->kind;
  if (nl->kind == 2 || nl->kind == kKindThreeTerm)
    return set_error(CGL_EINVAL, "stage_slice: single-component two-term nonlinearities only");
  a.flag = flag;
  a.pos = pos;
  a.fw = 1;
  for (int q = 0; q < nsl; ++q) {
    A.slices[q] = slices[q];
    A.exps[q] = exps[q];
  }
  A.Q = Q;
  A.n0 = n0;
  A.nchunks = (int)((2 * n0 + oz::KC - 1) / oz::KC);
  // full-K rows kernel for every program (measured: if4 MID 6.6 vs 9.8 us, END
  // 10.6 vs 14.7 us on C1; split4 END 517 vs 611 us at 256^3; since its 4-point
  // tasks on 256-thread CTAs and the early PDL trigger also the exact cubic
  // flows: C1 strang 0.0417 -> 0.0354, split4 0.0947 -> 0.0813 ms/step, C2
  // split4 3.67 -> 3.32 ms/step).  CGL_SS_CLUSTER=1 forces the cluster kernel
  // (A/B and tests; not for the half-step if4 programs, rows kernel only).
  const char* ev = getenv("CGL_SS_CLUSTER");
  const bool half = prog == P_IF4_MIDH || prog == P_IF4_ENDH || prog == P_IF4_MIDQ || prog == P_IF4_ENDQ;  // rows kernel only
  const bool old_kernel = !half && ev != nullptr && ev[0] == '1';
  if (!old_kernel && rows_slice_ok(n0, true)) {
    // full-K CTAs (rows_slice_kernel): element (q, i) of the axis-0 data at i * Q + q
    RowsSliceArgs R{};
    R.s = a;
    for (int q = 0; q < nsl; ++q) {
      R.slices[q] = slices[q];
      R.exps[q] = exps[q];
    }
    R.batch = 1;
    R.rows = Q;
    R.K = n0;
    R.sr = 1;
    R.sk = Q;
    R.nchunks = A.nchunks;
    cudaError_t e;
    switch (prog) {
      case P_IF4_MID: e = launch_rows_slice<P_IF4_MID, 2>(R, 1, st); break;
      case P_IF4_END: e = launch_rows_slice<P_IF4_END, 3>(R, 1, st); break;
      case P_IF4_MIDH: e = launch_rows_slice<P_IF4_MIDH, 2>(R, 1, st); break;
      case P_IF4_ENDH: e = launch_rows_slice<P_IF4_ENDH, 3>(R, 1, st); break;
      case P_IF4_MIDQ: e = launch_rows_slice<P_IF4_MIDQ, 2>(R, 1, st); break;
      case P_IF4_ENDQ: e = launch_rows_slice<P_IF4_ENDQ, 2>(R, 1, st); break;
      case P_STRANG_END: e = launch_rows_slice<P_STRANG_END, 1>(R, 1, st); break;
      case P_SPLIT4_MID: e = launch_rows_slice<P_SPLIT4_MID, 1>(R, 1, st); break;
      default: e = launch_rows_slice<P_SPLIT4_END, 2>(R, 1, st); break;
    }
    if (e != cudaSuccess) return set_cuda_error(e, "stage_slice (rows) launch");
    return check_launch("rows_slice_kernel");
  }
  if (half) return set_error(CGL_ESHAPE, "stage_slice: the if4 half-step programs need an axis-0 extent <= 1024");
  // CTAs of a tile's cluster cover all K chunks: <= 16 CTAs (non-portable beyond 8)
  if (A.nchunks > 64) return set_error(CGL_ESHAPE, "stage_slice: axis-0 extent above 1024");
  const bool small = A.nchunks <= 32;
#define SS_LAUNCH(P_, N_) (small ? launch_stage_slice<P_, N_, 2>(A, st) : launch_stage_slice<P_, N_, 4>(A, st))
  cudaError_t e;
  switch (prog) {
    case P_IF4_MID: e = SS_LAUNCH(P_IF4_MID, 2); break;
    case P_IF4_END: e = SS_LAUNCH(P_IF4_END, 3); break;
    case P_STRANG_END: e = SS_LAUNCH(P_STRANG_END, 1); break;
    case P_SPLIT4_MID: e = SS_LAUNCH(P_SPLIT4_MID, 1); break;
    default: e = SS_LAUNCH(P_SPLIT4_END, 2); break;
  }
#undef SS_LAUNCH
  if (e != cudaSuccess) return set_cuda_error(e, "stage_slice launch");
  return check_launch("stage_slice_kernel");
}

template <int NF>
static int launch_prog(int prog, const StageArgs& a, cudaStream_t st) {
  const int grid = grid_for(a.n, kStageThreads);
  cudaError_t e = cudaSuccess;
  switch (prog) {
    case P_IF4_PRE: e = launch_k(stage_kernel<NF, P_IF4_PRE>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_MID: e = launch_k(stage_kernel<NF, P_IF4_MID>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_END: e = launch_k(stage_kernel<NF, P_IF4_END>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FLOW1: e = launch_k(stage_kernel<NF, P_FLOW1>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FLOW2: e = launch_k(stage_kernel<NF, P_FLOW2>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_SPLIT4_MID: e = launch_k(stage_kernel<NF, P_SPLIT4_MID>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_SPLIT4_END: e = launch_k(stage_kernel<NF, P_SPLIT4_END>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_STRANG_END: e = launch_k(stage_kernel<NF, P_STRANG_END>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF2_PRE: e = launch_k(stage_kernel<NF, P_IF2_PRE>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF2_END: e = launch_k(stage_kernel<NF, P_IF2_END>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FIF4_S1: e = launch_k(stage_kernel<NF, P_FIF4_S1>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FIF4_S2: e = launch_k(stage_kernel<NF, P_FIF4_S2>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FIF4_S3: e = launch_k(stage_kernel<NF, P_FIF4_S3>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FIF4_S4: e = launch_k(stage_kernel<NF, P_FIF4_S4>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_FLOW_END: e = launch_k(stage_kernel<NF, P_FLOW_END>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_MIDH: e = launch_k(stage_kernel<NF, P_IF4_MIDH>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_ENDH: e = launch_k(stage_kernel<NF, P_IF4_ENDH>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_MIDQ: e = launch_k(stage_kernel<NF, P_IF4_MIDQ>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_ENDQ: e = launch_k(stage_kernel<NF, P_IF4_ENDQ>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    default: return set_error(CGL_EINVAL, "stage: unknown program");
  }
  if (e != cudaSuccess) return set_cuda_error(e, "stage_kernel launch");
  return check_launch("stage_kernel");
}

// inputs/outputs per program, in units of component groups
static const int kIns[P_NPROG] = {1, 2, 4, 1, 1, 2, 2, 1, 1, 2, 2, 2, 2, 5, 1, 3, 2, 2, 2};
static const int kOuts[P_NPROG] = {2, 2, 3, 1, 2, 2, 3, 2, 2, 3, 1, 1, 1, 1, 1, 2, 3, 2, 2};

int stage_launch(cudaStream_t st, int prog, int nf, int64_t n, const cgl_nonlinear_t* nl, double tau,
                 double in_scale, const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos,
                 int ndim, const int64_t* shape, const double* const* tables, int64_t tm, int64_t toff) {
  if (prog < 0 || prog >= P_NPROG) return set_error(CGL_EINVAL, "stage: unknown program");
  if (nf != 1 && nf != 2) return set_error(CGL_EINVAL, "stage: 1 or 2 components");
  static_assert(sizeof(((StageArgs*)0)->in) / sizeof(void*) >= 10, "in[] holds 5 operands x 2 components");
  if ((nl->kind == 2) != (nf == 2)) return set_error(CGL_EINVAL, "stage: component count does not match kind");
  if (n <= 0) return 0;
  StageArgs a{};
  for (int q = 0; q < kIns[prog] * nf; ++q) a.in[q] = reinterpret_cast<const double2*>(in[q]);
  for (int q = 0; q < kOuts[prog] * nf; ++q) a.out[q] = reinterpret_cast<double2*>(out[q]);
  a.n = n;
  a.tau = tau;
  a.in_scale = in_scale;
  a.nl = StageNL{nl->alpha3, nl->beta3, nl->alpha4, nl->beta4, nl->alpha5, nl->kind};
  a.flag = flag;
  a.pos = pos;
  if (nl->kind < 0 || nl->kind > kKindThreeTerm) return set_error(CGL_EINVAL, "stage: unknown nonlinearity kind");
  a.fw = nl->kind == 0 ? nf : (nl->kind == kKindThreeTerm ? 2 : 1);
  if (prog >= P_FIF4_S1 && prog <= P_FIF4_S4) {
    if (ndim < 1 || ndim > 4 || !shape || !tables) return set_error(CGL_EINVAL, "stage: Fourier programs need tables");
    a.nd = ndim;
    int64_t tot = 1;
    a.pow2 = 1;
    for (int d = 0; d < ndim; ++d) {
      a.ext[d] = shape[d];
      tot *= shape[d];
      int lg = 0;
      while ((1ll << lg) < shape[d]) ++lg;
      a.lg[d] = lg;
      a.pow2 &= (1ll << lg) == shape[d];
    }
    if (tm > 0) {
      // local (n0 x tm) column block of a global shape (sharded spectral layout)
      a.tm = tm;
      a.toff = toff;
      a.t12 = tot / shape[0];
      if (n != shape[0] * tm || toff + tm > a.t12) return set_error(CGL_ESHAPE, "stage: bad column block");
    } else if (tot != n) {
      return set_error(CGL_ESHAPE, "stage: shape does not match n");
    }
    // tables: [fraction(2)][component(nf)][axis(ndim)]
    for (int fr = 0; fr < 2; ++fr)
      for (int c = 0; c < nf; ++c)
        for (int d = 0; d < ndim; ++d)
          a.tab[fr][c][d] = reinterpret_cast<const double2*>(tables[(fr * nf + c) * ndim + d]);
  }
  return nf == 1 ? launch_prog<1>(prog, a, st) : launch_prog<2>(prog, a, st);
}

CGL_PROF_TU(stages)

}  // namespace cgl
