// Full-K data slicing of the INT8-emulated GEMM's B operand, optionally
// fused with a stage program (stage_ops.cuh): the block-level body shared by
// the standalone kernel (stages.cu) and the prologue phase of the fused GEMM
// (ozgemm.cu).
#pragma once
#include <climits>
#include <cstdint>

#include "cgl_common.cuh"
#include "cgl_internal.h"
#include "oz_slice.cuh"
#include "stage_ops.cuh"

namespace cgl {

// ---- full-K data slicing (no cluster) -------------------------------------
// One CTA owns QC whole operand rows R (columns q of the field for the axis-0
// data, rows p for the last-axis data) over the ENTIRE K range, so the row
// exponent is a CTA-local reduction: no cluster, no DSMEM exchange, no
// shared-memory staging of the values.  Thread task = (row qi, 16-byte K
// group g = 8 complex k's): its 8 points are loaded once (all loads in flight
// together with the flag reads), the stage program runs in registers, the
// per-row max is reduced with shuffles + one __syncthreads, and the thread
// writes its group's S = 8 slices as 16-byte stores.  QC adjacent rows make
// every warp store / load sector-complete (rows R, R+1 are adjacent 16-byte
// rows of a core matrix; the QC q's of one k are contiguous in the field).
// Element (R, k) of the operand is at R * sr + k * sk in each source.
// Same digits, exponents and layout as slice_tile_kernel<8, 0, *, *> /
// stage_slice_kernel (bit-identical; tests/test_gpu_parity.py).
constexpr int P_SLICE = 100;  // plain slicing of up to 8 items (no stage program)
constexpr int kRSThreads = 128;

struct RowsSliceArgs {
  StageArgs s;              // stage programs: inputs (s.in), FP64 outputs (s.out), flag
  const double2* srcs[8];   // P_SLICE: per item source (blockIdx.y = item * batch + b)
  int8_t* slices[8];        // per sliced output (stage) / per item (P_SLICE)
  int* exps[8];
  int64_t src_bs, out_bs, exp_bs;  // P_SLICE batch strides (elements / bytes / ints)
  int64_t batch;
  int64_t rows, K;          // operand rows R, complex K extent
  int64_t sr, sk;           // element (R, k) at R * sr + k * sk
  int nchunks, QC;
};

// Shared-memory scratch of one 128-thread group.
struct RowsSliceSmem {
  double red[3][8][32];   // up to 8 warps per group (NT <= 256)
  int redbad[3][8][32];
  int erow[3][32];
};

__device__ __forceinline__ void group_bar(int id, int nt = kRSThreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nt) : "memory");
}

// One virtual CTA (bx = row block, by = item * batch + b) of the full-K
// slicing, run by a 128-thread group (tid 0..127) synchronising on named
// barrier `bar`.  Returns false iff the stage program skips (a failure was
// recorded before its first flow position; uniform over the grid).  The
// caller has executed griddepcontrol.wait.
// masked high word of |x|: unsigned order = order of |x| (finite), exponent
// field 0x7FF (>= 0x7FF00000) marks Inf/NaN
__device__ __forceinline__ unsigned absbits_hi(double x) { return (unsigned)__double2hiint(x) & 0x7FFFFFFFu; }

template <int PROG, int NSL, int TPT, int PP = 8, int NT = kRSThreads>
__device__ __forceinline__ bool rows_slice_block(const RowsSliceArgs& A, int64_t bx, int64_t by, int tid, int bar,
                                                 RowsSliceSmem& sm) {
  using oz::KC;
  using oz::NONFINITE;
  constexpr int NO = PROG == P_SLICE ? 1 : NSL;  // sliced outputs per task
  constexpr int NIN = PROG == P_SLICE ? 1
                      : (PROG == P_IF4_END ? 4 : (PROG == P_STRANG_END ? 1 : 2));
  const StageArgs& a = A.s;
  const int lane = tid & 31, wid = tid >> 5;
  const int QC = A.QC, lqc = __ffs(QC) - 1;  // QC is a power of two
  const int64_t R0 = bx * QC;
  const int item = PROG == P_SLICE ? (A.batch == 1 ? (int)by : (int)(by / A.batch)) : 0;
  const int64_t bb = PROG == P_SLICE ? (A.batch == 1 ? 0 : (int64_t)(by % A.batch)) : 0;
  static_assert(PP == 8 || PP == 4, "points per task: one 16-byte (PP = 8) or 8-byte (PP = 4) K group");
  const int64_t KG = (A.K + PP - 1) / PP;  // K groups of PP complex
  const int64_t sk = A.sk;
  // flag state (written by earlier kernels: plain loads after griddepcontrol.wait)
  uint64_t step = 0, fkey = ~0ull;
  const cgl_flag_t* cf = a.flag;
  if (PROG != P_SLICE && cf != nullptr) {
    fkey = __ldcg(reinterpret_cast<const unsigned long long*>(&cf->key));
    const uint64_t base = __ldcg(reinterpret_cast<const unsigned long long*>(&cf->step));
    step = (a.pos & CGL_POS_DEVICE) ? base + ((a.pos & ~CGL_POS_DEVICE) >> 24) : (a.pos >> 24);
  }
  double2 o[TPT][NO][PP];
  const double t = a.tau, sc = a.in_scale;
  uint64_t key = ~0ull;
  const uint64_t check_pos = (step << 24) | (255ull << 8);
  (void)t;
  (void)sc;
  (void)check_pos;
#pragma unroll
  for (int j = 0; j < TPT; ++j) {
    const int task = tid + NT * j;
    const int qi = task & (QC - 1);
    const int64_t g = task >> lqc, R = R0 + qi;
    const bool live = g < KG && R < A.rows;
    const bool full = live && PP * g + PP - 1 < A.K;  // common case: no per-point bounds
    const int64_t i0 = live ? R * A.sr + PP * g * sk : 0;  // element offset of the task's first point
    // ---- loads (the first task's are in flight together with the flag reads) ----
    double2 in[NIN][PP];
    const double2* srcs[NIN];
#pragma unroll
    for (int q = 0; q < NIN; ++q) srcs[q] = (PROG == P_SLICE ? A.srcs[item] + bb * A.src_bs : a.in[q]) + i0;
    if (full) {
#pragma unroll
      for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int q = 0; q < NIN; ++q) in[q][p] = __ldg(srcs[q] + p * sk);
    } else {
      const int64_t nk = live ? A.K - PP * g : 0;  // points of this task inside K
#pragma unroll
      for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int q = 0; q < NIN; ++q) in[q][p] = p < nk ? __ldg(srcs[q] + p * sk) : make_double2(0.0, 0.0);
    }
    // skip (uniform over the grid) if a failure was recorded before this
    // program's first flow position: nothing is written, as stage_kernel
    if (PROG != P_SLICE && j == 0) {
      int first = 0;
      if (PROG == P_SPLIT4_MID || PROG == P_STRANG_END) first = a.fw;
      if (PROG == P_SPLIT4_END) first = 4 * a.fw;
      if (fkey < ((step << 24) | ((uint64_t)first << 8))) return false;
    }
    if (PROG == P_SLICE) {
#pragma unroll
      for (int p = 0; p < PP; ++p) o[j][0][p] = in[0][p];
      continue;
    }
    // ---- stage program in registers; FP64 outputs stored here ----
    double2* dout = a.out[0] + i0;
#pragma unroll
    const int64_t nk = full ? PP : (live ? A.K - PP * g : 0);
#pragma unroll
    for (int p = 0; p < PP; ++p, dout += sk) {
      const bool ok = p < nk;
#pragma unroll
      for (int q = 0; q < NO; ++q) o[j][q][p] = make_double2(0.0, 0.0);
      if (!ok) continue;
      if (PROG == P_IF4_MIDQ) {
        V<1> A, G;
        A.c[0] = cscale(sc, in[0][p]);
        G.c[0] = cscale(sc, in[NIN > 1 ? 1 : 0][p]);
        const V<1> u2 = axpy<1>(0.5 * t, G, A), w = axpy<1>(t / 6.0, G, A);
        const V<1> g2 = gfun<1>(a.nl, u2);
        const V<1> g3 = gfun<1>(a.nl, axpy<1>(0.5 * t, g2, A));
        const V<1> sv = axpy<1>(1.0, g2, g3);
        o[j][0][p] = axpy<1>(t, g3, A).c[0];                     // p = a + t g3
        o[j][NO > 1 ? 1 : 0][p] = axpy<1>(t / 3.0, sv, w).c[0];  // r = w + t/3 s
      } else if (PROG == P_IF4_ENDQ) {
        V<1> u4, q;
        u4.c[0] = cscale(sc, in[0][p]);
        q.c[0] = cscale(sc, in[NIN > 1 ? 1 : 0][p]);
        const V<1> out = axpy<1>(t / 6.0, gfun<1>(a.nl, u4), q);
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        *dout = out.c[0];
        o[j][0][p] = out.c[0];                                   // u
        o[j][NO > 1 ? 1 : 0][p] = gfun<1>(a.nl, out).c[0];       // g1 of the next step
      } else if (PROG == P_IF4_MID) {
        V<1> u2, av;
        u2.c[0] = cscale(sc, in[0][p]);
        av.c[0] = cscale(sc, in[NIN > 1 ? 1 : 0][p]);
        const V<1> g2 = gfun<1>(a.nl, u2);
        const V<1> g3 = gfun<1>(a.nl, axpy<1>(0.5 * t, g2, av));
        o[j][0][p] = g3.c[0];
        o[j][NO > 1 ? 1 : 0][p] = axpy<1>(1.0, g2, g3).c[0];
      } else if (PROG == P_STRANG_END) {
        V<1> w;
        w.c[0] = cscale(sc, in[0][p]);
        const V<1> out = flow<1>(a.nl, w, 0.5 * t, step, a.fw, key);
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        *dout = out.c[0];
        o[j][0][p] = flow<1>(a.nl, out, 0.5 * t, step + 1, 0, key).c[0];
      } else if (PROG == P_SPLIT4_MID) {
        V<1> v, f;
        v.c[0] = cscale(sc, in[0][p]);
        f.c[0] = cscale(sc, in[NIN > 1 ? 1 : 0][p]);
        *dout = flow<1>(a.nl, v, 0.5 * t, step, a.fw, key).c[0];
        o[j][0][p] = flow<1>(a.nl, f, 0.5 * t, step, 3 * a.fw, key).c[0];
      } else if (PROG == P_SPLIT4_END) {
        V<1> f, c;
        f.c[0] = cscale(sc, in[0][p]);
        c.c[0] = cscale(sc, in[NIN > 1 ? 1 : 0][p]);
        const V<1> fine = flow<1>(a.nl, f, 0.25 * t, step, 4 * a.fw, key);
        V<1> out;
        out.c[0] = cadd(cscale(4.0 / 3.0, fine.c[0]), cscale(-1.0 / 3.0, c.c[0]));
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        *dout = out.c[0];
        o[j][0][p] = flow<1>(a.nl, out, 0.5 * t, step + 1, 0, key).c[0];
        o[j][NO > 1 ? 1 : 0][p] = flow<1>(a.nl, out, 0.25 * t, step + 1, 2 * a.fw, key).c[0];
      } else {  // P_IF4_END
        V<1> b, c, d, e;
        b.c[0] = cscale(sc, in[0][p]);
        c.c[0] = cscale(sc, in[NIN > 1 ? 1 : 0][p]);
        d.c[0] = cscale(sc, in[NIN > 2 ? 2 : 0][p]);
        e.c[0] = cscale(sc, in[NIN > 3 ? 3 : 0][p]);
        const V<1> g4 = gfun<1>(a.nl, axpy<1>(t, d, b));
        const V<1> out = axpy<1>(t / 6.0, g4, axpy<1>(t / 3.0, e, c));
        if (!finite_all<1>(out)) note(key, check_pos, CGL_NONFINITE_STATE);
        *dout = out.c[0];
        const V<1> g1 = gfun<1>(a.nl, out);
        o[j][0][p] = axpy<1>(0.5 * t, g1, out).c[0];
        o[j][NO > 1 ? 1 : 0][p] = out.c[0];
        o[j][NO > 2 ? 2 : 0][p] = axpy<1>(t / 6.0, g1, out).c[0];
      }
    }
  }
  // ---- per-row max over the group (rows qi = tid % QC): the frexp exponent of
  // max|x| is the exponent field of the largest masked high word ----
  auto& red = sm.red;
  auto& redbad = sm.redbad;
  auto& erow = sm.erow;
  (void)red;
#pragma unroll
  for (int q = 0; q < NO; ++q) {
    unsigned mh = 0;
#pragma unroll
    for (int j = 0; j < TPT; ++j)
#pragma unroll
      for (int p = 0; p < PP; ++p) mh = max(mh, max(absbits_hi(o[j][q][p].x), absbits_hi(o[j][q][p].y)));
    for (int off = 16; off >= QC; off >>= 1) mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, off));
    if (lane < QC) redbad[q][wid][lane] = (int)mh;
  }
  group_bar(bar, NT);
  if (tid < QC * NO) {
    const int q = tid >> lqc, qi = tid & (QC - 1);
    unsigned mh = (unsigned)redbad[q][0][qi];
    for (int k = 1; k < NT / 32; ++k) mh = max(mh, (unsigned)redbad[q][k][qi]);
    // normal max: frexp exponent = E - 1022; all zero / subnormal (E = 0): resolved below
    const int E = (int)(mh >> 20);
    erow[q][qi] = E == 0x7FF ? NONFINITE : (E == 0 ? INT_MIN : E - 1022);
  }
  group_bar(bar, NT);
  // rows whose max is zero or subnormal (rare): the exact frexp of the double max
  bool sub = false;
#pragma unroll
  for (int q = 0; q < NO; ++q)
    for (int qi = 0; qi < QC; ++qi) sub |= erow[q][qi] == INT_MIN;
  if (sub) {  // uniform over the group
#pragma unroll
    for (int q = 0; q < NO; ++q) {
      double m = 0.0;
#pragma unroll
      for (int j = 0; j < TPT; ++j)
#pragma unroll
        for (int p = 0; p < PP; ++p) m = fmax(m, fmax(fabs(o[j][q][p].x), fabs(o[j][q][p].y)));
      for (int off = 16; off >= QC; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
      if (lane < QC) red[q][wid][lane] = m;
    }
    group_bar(bar, NT);
    if (tid < QC * NO) {
      const int q = tid >> lqc, qi = tid & (QC - 1);
      if (erow[q][qi] == INT_MIN) {
        double m = red[q][0][qi];
        for (int k = 1; k < NT / 32; ++k) m = fmax(m, red[q][k][qi]);
        int e = 0;  // all-zero row: 0 (same convention as the slicing kernels)
        if (m > 0.0) frexp(m, &e);
        erow[q][qi] = e;
      }
    }
    group_bar(bar, NT);
  }
  if (tid < QC * NO) {
    const int q = tid >> lqc, qi = tid & (QC - 1);
    if (R0 + qi < A.rows) {
      if (PROG == P_SLICE) A.exps[item][bb * A.exp_bs + R0 + qi] = erow[q][qi];
      else A.exps[q][R0 + qi] = erow[q][qi];
    }
  }
  // ---- digits: one 16-byte (PP = 8) or 8-byte (PP = 4) store per slice and task ----
  constexpr int NW = PP / 2;  // 32-bit words per slice per task (two complex per word)
#pragma unroll
  for (int j = 0; j < TPT; ++j) {
    const int task = tid + NT * j;
    const int qi = task & (QC - 1);
    const int64_t g = task >> lqc, R = R0 + qi;
    if (g >= KG || R >= A.rows) continue;  // padding stays zero (buffer zeroed once)
#pragma unroll
    for (int q = 0; q < NO; ++q) {
      const int e = erow[q][qi];
      uint32_t wv[8][NW];
#pragma unroll
      for (int s8 = 0; s8 < 8; ++s8)
#pragma unroll
        for (int k = 0; k < NW; ++k) wv[s8][k] = 0u;
      if (e != NONFINITE) {
        const double2 s2p = oz::pow2_split(e);
        if (e >= -940) {  // uniform per row: one scaling factor, no subnormal checks
#pragma unroll
          for (int k = 0; k < NW; ++k) {
            const double2 v0 = o[j][q][2 * k], v1 = o[j][q][2 * k + 1];
            const double x[4] = {v0.x, v0.y, v1.x, v1.y};
            uint32_t ww[8];
            oz::words8_fast<true>(x, s2p, ww);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) wv[s8][k] = ww[s8];
          }
        } else {
#pragma unroll
          for (int k = 0; k < NW; ++k) {
            const double2 v0 = o[j][q][2 * k], v1 = o[j][q][2 * k + 1];
            const double x[4] = {v0.x, v0.y, v1.x, v1.y};
            uint32_t ww[8];
            oz::words8_fast<false>(x, s2p, ww);
#pragma unroll
            for (int s8 = 0; s8 < 8; ++s8) wv[s8][k] = ww[s8];
          }
        }
      }
      int8_t* base = PROG == P_SLICE ? A.slices[item] + bb * A.out_bs : A.slices[q];
      int8_t* dst = base + oz::tile_offset(R, 2 * PP * g, kOzBN, A.nchunks, 8);
      {
#pragma unroll
        for (int s8 = 0; s8 < 8; ++s8) {
          if constexpr (PP == 8)
            *reinterpret_cast<uint4*>(dst + s8 * (kOzBN * KC)) = make_uint4(wv[s8][0], wv[s8][1], wv[s8][2], wv[s8][NW - 1]);
          else
            *reinterpret_cast<uint2*>(dst + s8 * (kOzBN * KC)) = make_uint2(wv[s8][0], wv[s8][NW - 1]);
        }
      }
    }
  }
  if (PROG != P_SLICE) raise_min(a.flag, key);
  return true;
}

}  // namespace cgl
