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
                       PROG == P_FIF4_S4 || PROG == P_FLOW_END || PROG == P_IF4_ENDQ);
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

// ---- fused stage + data slicing (INT8-emulated products on FD grids) ----
// The stage outputs consumed only as the data operands of the next axis-0
// mu-mode products (if4: p, r / u, g1'; strang: v'; split4: f, v', f') are
// never stored in FP64: the stage program runs inside the full-K rows slicing
// kernel (rows_slice.cuh), which stores the state in FP64 and emits the
// floor-digit slices in the GEMM's B-operand layout (Z = In^T: rows q, K =
// axis-0 index; exactly what cgl_oz_slice_multi produces for the same field).
// (A cluster/DSMEM kernel covering 32 columns per cluster was the first
// version; the rows kernel beat it on every program -- if4 MID 6.6 vs 9.8 us,
// END 10.6 vs 14.7 us on C1, split4 END 517 vs 611 us at 256^3 -- and replaced it.)
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
  rows_slice_block<PROG, NSL, TPT, PP, NT>(A, blockIdx.x, blockIdx.y, threadIdx.x, 0, sm);
}

// QC rows per CTA: NT threads cover QC * KG tasks (PP complex each) in TPT
// rounds; the smallest QC that fills the threads (measured: fewer, larger CTAs
// are slower).
int rows_slice_qc(int64_t K, int64_t rows_total, int tpt_max, int* tpt, int pp, int nt) {
  const int64_t KG = (K + pp - 1) / pp;
  (void)rows_total;
  (void)tpt_max;
  int qc = 2;
  while (qc < 32 && qc * KG < nt) qc <<= 1;
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
// when the launch's data are L2-sized.
static int rows_pp(bool stage, double bytes) {
  if (stage) return 4;
  return bytes <= 64.0 * (1 << 20) ? 4 : 8;
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
  cudaError_t e = launch_rows_slice<P_SLICE, 1>(A, batch * nitems, st);
  if (e != cudaSuccess) return set_cuda_error(e, "rows_slice launch");
  return check_launch("rows_slice_kernel");
}

int stage_slice_launch(cudaStream_t st, int prog, int64_t n0, int64_t Q, const cgl_nonlinear_t* nl, double tau,
                       double in_scale, const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos,
                       int8_t* const* slices, int* const* exps) {
  int nin, nsl, nout;
  switch (prog) {
    case P_IF4_MID: nin = 2; nsl = 2; nout = 0; break;
    case P_IF4_END: nin = 4; nsl = 3; nout = 1; break;
    case P_IF4_MIDQ: nin = 2; nsl = 2; nout = 0; break;
    case P_IF4_ENDQ: nin = 2; nsl = 2; nout = 1; break;
    case P_STRANG_END: nin = 1; nsl = 1; nout = 1; break;
    case P_SPLIT4_MID: nin = 2; nsl = 1; nout = 1; break;
    case P_SPLIT4_END: nin = 2; nsl = 2; nout = 1; break;
    default: return set_error(CGL_EINVAL, "stage_slice: if4 MID/END (reference or quad form), strang END, split4 MID/END only");
  }
  if (n0 <= 0 || Q <= 0) return 0;
  if (nout && (!out || !out[0])) return set_error(CGL_EINVAL, "stage_slice: program writes an FP64 output");
  if (nl->kind == 2 || nl->kind == kKindThreeTerm)
    return set_error(CGL_EINVAL, "stage_slice: single-component two-term nonlinearities only");
  if (!rows_slice_ok(n0, true)) return set_error(CGL_ESHAPE, "stage_slice: axis-0 extent above 1024");
  // full-K CTAs (rows_slice_kernel): element (q, i) of the axis-0 data at i * Q + q
  RowsSliceArgs R{};
  StageArgs& a = R.s;
  for (int k = 0; k < nin; ++k) a.in[k] = reinterpret_cast<const double2*>(in[k]);
  if (nout) a.out[0] = reinterpret_cast<double2*>(out[0]);
  a.n = n0 * Q;
  a.tau = tau;
  a.in_scale = in_scale;
  a.nl = StageNL{nl->alpha3, nl->beta3, nl->alpha4, nl->beta4, nl->alpha5, nl->kind};
  a.flag = flag;
  a.pos = pos;
  a.fw = 1;
  for (int q = 0; q < nsl; ++q) {
    R.slices[q] = slices[q];
    R.exps[q] = exps[q];
  }
  R.batch = 1;
  R.rows = Q;
  R.K = n0;
  R.sr = 1;
  R.sk = Q;
  R.nchunks = (int)((2 * n0 + oz::KC - 1) / oz::KC);
  cudaError_t e;
  switch (prog) {
    case P_IF4_MID: e = launch_rows_slice<P_IF4_MID, 2>(R, 1, st); break;
    case P_IF4_END: e = launch_rows_slice<P_IF4_END, 3>(R, 1, st); break;
    case P_IF4_MIDQ: e = launch_rows_slice<P_IF4_MIDQ, 2>(R, 1, st); break;
    case P_IF4_ENDQ: e = launch_rows_slice<P_IF4_ENDQ, 2>(R, 1, st); break;
    case P_STRANG_END: e = launch_rows_slice<P_STRANG_END, 1>(R, 1, st); break;
    case P_SPLIT4_MID: e = launch_rows_slice<P_SPLIT4_MID, 1>(R, 1, st); break;
    default: e = launch_rows_slice<P_SPLIT4_END, 2>(R, 1, st); break;
  }
  if (e != cudaSuccess) return set_cuda_error(e, "stage_slice (rows) launch");
  return check_launch("rows_slice_kernel");
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
    case P_IF4_MIDQ: e = launch_k(stage_kernel<NF, P_IF4_MIDQ>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    case P_IF4_ENDQ: e = launch_k(stage_kernel<NF, P_IF4_ENDQ>, dim3(grid), dim3(kStageThreads), 0, st, dim3(1), a); break;
    default: return set_error(CGL_EINVAL, "stage: unknown program");
  }
  if (e != cudaSuccess) return set_cuda_error(e, "stage_kernel launch");
  return check_launch("stage_kernel");
}

// inputs/outputs per program, in units of component groups
static const int kIns[P_NPROG] = {1, 2, 4, 1, 1, 2, 2, 1, 1, 2, 2, 2, 2, 5, 1, 0, 0, 2, 2};  // 15, 16: retired ids
static const int kOuts[P_NPROG] = {2, 2, 3, 1, 2, 2, 3, 2, 2, 3, 1, 1, 1, 1, 1, 0, 0, 2, 2};

int stage_launch(cudaStream_t st, int prog, int nf, int64_t n, const cgl_nonlinear_t* nl, double tau,
                 double in_scale, const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos,
                 int ndim, const int64_t* shape, const double* const* tables, int64_t tm, int64_t toff) {
  if (prog < 0 || prog >= P_NPROG || kIns[prog] == 0) return set_error(CGL_EINVAL, "stage: unknown program");
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
