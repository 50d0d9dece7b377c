/*
 * cgl_b200.h — C ABI of the B200-native CGL time-integration hot path.
 *
 * Drop-in boundary for the reference package `cglsolve` (arXiv 2403.02816,
 * /root/reference/pkg/src/cglsolve).  The reference has no FFI: its seam is
 * the Python operator protocol (operators.py:106-208) and the stepper bodies
 * (integrators.py:130-227).  Each entry point below replaces the numpy call
 * site named in its comment; the Python package `paper_2403_02816_b200`
 * binds them with ctypes behind the same Python API.
 *
 * Conventions (all entry points):
 *   - complex128 data = interleaved (re, im) doubles, C-contiguous tensors of
 *     shape (n_1, ..., n_d) (last axis fastest), device pointers;
 *   - `stream` is a cudaStream_t passed as void*; work is enqueued, never
 *     synchronised;
 *   - return 0 on success, a negative CGL_E* code on argument errors, or a
 *     positive cudaError_t; cgl_last_error() has the message;
 *   - `flag`/`pos` implement the sticky divergence record (may be NULL/0):
 *     a kernel at position pos skips when an earlier position diverged.
 */
#ifndef CGL_B200_H
#define CGL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: cgl_oz_gemm_fused removed; cgl_rk_stage, CGL_FFT_STR_A0F, nonlinearity kind 3 added; the
 * IF4_B1..B4 pass programs accumulate the Lawson combination in one field */
#define CGL_ABI_VERSION 2

#define CGL_EINVAL (-1)
#define CGL_ESHAPE (-2)
#define CGL_ECUFFT (-3)
#define CGL_ENCCL (-4)       /* an NCCL call failed                                 */
#define CGL_EUNAVAILABLE (-5) /* NCCL is not loaded in this process                  */

/* Sticky divergence record + device step base (24 bytes, device memory).
 * key = (step << 24) | (seq << 8) | reason, atomically min-reduced, so it
 * holds the first (step, call) that failed; mirrors DivergenceError(reason)
 * + diverged_at of integrators.py:264-278 and flows.py:32-39,95-132.
 * Init: key = all ones, step = 0 (base), done = 0 (reserved).
 * A `pos` with CGL_POS_DEVICE set is relative: step = flag->step + the local
 * step index in pos bits 24..62 (seq << 8 in the low bits), so a captured
 * CUDA graph of a chunk of steps replays unchanged; cgl_flag_advance moves
 * the base at the end of each chunk. */
typedef struct cgl_flag_t {
  unsigned long long key;
  unsigned long long step;
  unsigned int done;
  unsigned int reserved;
} cgl_flag_t;

#define CGL_POS_DEVICE (1ull << 63)

enum cgl_reason {
  CGL_BLOWUP_CUBIC = 0,      /* flows.py:95-96  "finite-time blow-up in cubic flow" */
  CGL_NONFINITE_CUBIC = 1,   /* flows.py:99-100 "non-finite cubic flow output" */
  CGL_BLOWUP_QUINTIC = 2,    /* flows.py:111-112 */
  CGL_NONFINITE_QUINTIC = 3, /* flows.py:114-115 */
  CGL_NONFINITE_RK4 = 4,     /* flows.py:131-132 "non-finite RK4 flow output" */
  CGL_NONFINITE_STATE = 5    /* integrators.py:274-278 "non-finite state" */
};

/* Nonlinearity (flows.py:42-78). kind: 0 cubic, 1 cubic_quintic,
 * 2 coupled_cubic_quintic (two components); 3 (cgl_stage flow programs only):
 * cubic_quintic under the three-term splitting -- every flow of a strang /
 * split4 program is the pair of exact flows of integrators.py:178-195
 * (quintic then cubic in the first half of a Strang step, cubic then quintic
 * in the second), two sequence positions per flow. */
typedef struct cgl_nonlinear_t {
  double alpha3, beta3, alpha4, beta4, alpha5;
  int kind;
} cgl_nonlinear_t;

const char* cgl_version(void);
const char* cgl_last_error(void);
int cgl_abi_version(void);

/* Number of kernels this library has launched in this process (evidence
 * counter for benchmarks; cuFFT's own kernels are not counted). */
unsigned long long cgl_launch_count(void);

/* FP64 tensor-pipe probe: a register-resident DMMA.8x8x4 loop on all SMs;
 * returns the flops one launch performs (time it with events on `stream`).
 * Used to report mu-mode-product rooflines against a measured FP64 peak. */
double cgl_probe_dmma(void* stream, int iters);

/* ---- dense complex-FP64 contractions (DMMA tensor cores) ---------------- */

/* Batched complex GEMM, row-major:
 *   C_b[m,n] = alpha * sum_k A_b[m,k] B_b[k,n] + beta * Y_b[m,n]
 * A_b = A + b*sA (element (m,k) at m*lda+k), likewise B, C, Y (Y may be NULL,
 * may alias C).  Strides/leading dims are in complex elements.
 * Replaces the zgemm under np.tensordot (tensors.py:59). */
int cgl_zgemm(void* stream, int64_t M, int64_t N, int64_t K,
              const double* A, int64_t lda, int64_t sA,
              const double* B, int64_t ldb, int64_t sB,
              double* C, int64_t ldc, int64_t sC, int64_t batch,
              double alpha_re, double alpha_im,
              const double* Y, int64_t ldy, int64_t sY, double beta,
              const cgl_flag_t* flag, uint64_t pos);

/* mu-mode product out = u x_axis mat (tensors.py:38-59), plus optional
 * out = alpha*(...) + beta*y.  mat is m_out x shape[axis] row-major; mat_t is
 * its transpose (shape[axis] x m_out row-major), used when axis is the
 * contiguous (last) axis. */
int cgl_mode_product(void* stream, int ndim, const int64_t* shape, int axis,
                     const double* mat, const double* mat_t, int64_t m_out,
                     const double* in, double* out,
                     double alpha, const double* y, double beta,
                     const cgl_flag_t* flag, uint64_t pos);

/* The same for nfields fields with per-field matrices in ONE GEMM launch
 * (mats/mats_t/ins/outs/ys: arrays of nfields pointers, ys may be NULL). */
int cgl_mode_product_batch(void* stream, int ndim, const int64_t* shape, int axis,
                           int nfields, const double* const* mats,
                           const double* const* mats_t, int64_t m_out,
                           const double* const* ins, double* const* outs,
                           double alpha, const double* const* ys, double beta,
                           const cgl_flag_t* flag, uint64_t pos);

/* Tucker chain out_f = in_f x_1 M_{f,1} ... x_d M_{f,d} for nfields fields
 * in one launch per mode (tensors.py:62-69 / operators.py:134-139).
 * mats/mats_t: nfields*ndim square matrices (field-major); work: nfields
 * scratch fields (may be NULL when ndim == 1). in may not alias out. */
int cgl_tucker(void* stream, int ndim, const int64_t* shape, int nfields,
               const double* const* mats, const double* const* mats_t,
               const double* const* in, double* const* out,
               double* const* work, const cgl_flag_t* flag, uint64_t pos);

/* ---- FP64-accurate complex GEMM on the INT8 tensor cores (Ozaki I) ------- */
/* (csrc/ozgemm.cu) C = A B with complex A (M x K), B (K x N), computed from
 * S int8 slices per operand on tcgen05 kind::i8 with TMEM accumulators.
 * Operands are pre-sliced into the UMMA tile layout:
 *   A side ("a_mode" = 1): slices of the complex M x K matrix A,
 *   B side ("a_mode" = 0): slices of Z = B^T (N x K), i.e. rows = output columns.
 * cgl_oz_slice reads complex Z(r, c) = src[r*sr + c*sc] (rows x cols, per
 * batch + src_batch_stride), writes S slices (cgl_oz_slice_bytes per batch,
 * zero-initialise once: padding is never written) and one exponent per row.
 * A row holding NaN/Inf gets the exponent 0x7fffffff and the GEMM returns
 * NaN for its outputs (non-finite states propagate as in an FP64 GEMM). */
int64_t cgl_oz_slice_bytes(int S, int64_t rows, int64_t cols, int a_mode);
int cgl_oz_slice(void* stream, int S, const double* src, int64_t sr, int64_t sc,
                 int64_t rows, int64_t cols, int64_t batch, int64_t src_batch_stride,
                 int a_mode, int8_t* out, int64_t out_batch_stride, int* exps,
                 int64_t exp_batch_stride);
/* The same for nitems equally shaped matrices in one launch pair, for the
 * per-product (dense) data operand: digits in floor form (signed top digit,
 * others in [0, 127]) -- cgl_oz_slice uses sign-magnitude digits, which keep
 * the leading slices of small entries zero for cgl_oz_zmap skipping. */
int cgl_oz_slice_multi(void* stream, int S, int nitems, const double* const* srcs,
                       int64_t sr, int64_t sc, int64_t rows, int64_t cols, int64_t batch,
                       int64_t src_batch_stride, int a_mode, int8_t* const* outs,
                       int64_t out_batch_stride, int* const* exps, int64_t exp_batch_stride);
/* As cgl_oz_gemm but C stored transposed: element (i, j) at C[j*ldc + i].
 * The last-axis product Out = In E^T runs as Out^T = E In^T with the
 * constant E on the (block-skipped) A side and the data on the B side. */
int cgl_oz_gemm_t(void* stream, int S, int64_t M, int64_t N, int64_t K, int nitems,
                  const int8_t* const* A, const int* const* Aexp, const int8_t* const* Azmap,
                  const int8_t* const* B, const int* const* Bexp, const int8_t* const* Bzmap,
                  double* const* C, int64_t ldc, int64_t batch,
                  int64_t sA, int64_t sAexp, int64_t sB, int64_t sBexp, int64_t sC,
                  const cgl_flag_t* flag, uint64_t pos);
/* Fused if4 stage + data slicing on a finite-difference grid viewed as
 * (n0 x Q) (axis 0 x the rest), single-component nonlinearities:
 *   program CGL_STAGE IF4_MID (1): in = {u2, a}; sliced outputs {g3, s}
 *     (g2 = g(u2), g3 = g(a + t/2 g2), s = g2 + g3);
 *   program IF4_END (2): in = {b, c, d, e}; out[0] = u (FP64 state, checked
 *     finite as cgl_stage); sliced outputs {X1, u, X5} of the next step.
 * Each sliced output is written as the B-operand slices + row exponents of
 * the next axis-0 product (exactly cgl_oz_slice_multi's result for Z = In^T,
 * rows Q, K n0), so X1/X5/g3/s never exist in FP64.  Replaces
 * integrators.py:205-215 stage arithmetic + the read of the matmul input.
 * Requires n0 <= 1024. */
int cgl_stage_slice(void* stream, int program, int64_t n0, int64_t Q, const cgl_nonlinear_t* nl,
                    double tau, double in_scale, const double* const* in, double* const* out,
                    cgl_flag_t* flag, uint64_t pos, int8_t* const* slices, int* const* exps);
/* Seeded inputs on the device (rng.py:21-64): uniforms start..start+count-1
 * of stream `seed` (bit-identical to the host stream). */
int cgl_uniforms(void* stream, uint64_t seed, uint64_t start, int64_t count, double* out);
/* Seeded complex initial condition of a C-order shape (complex128 out):
 * recipe 0 sech(r)(1 + 0.01 xi), 1 2 exp(-r^2/4)(1 + 0.01 xi), 2 0.1 xi,
 * 3 xi; xi = xi_r + i xi_i with xi_r = normal_tensor(seed),
 * xi_i = normal_tensor(seed + 1) (Fortran-order streams, Box-Muller on the
 * device: a few ulp from numpy); r^2 from the per-axis coordinates axes[d]
 * (recipes 0 and 1).  Replaces experiments.py's host IC construction. */
int cgl_seeded_ic(void* stream, int recipe, uint64_t seed, int ndim, const int64_t* shape,
                  const double* const* axes, double* out);
/* Tile geometry of the emulated GEMM: A row tile, B row tile, K chunk bytes. */
int cgl_oz_geometry(int* bm, int* bn, int* kc);
/* Debug: with CGL_OZ_TRACE=1 in the environment, CTA 0 of the last
 * cgl_oz_gemm records phase timestamps (ns); copies 64 slots to host64. */
int cgl_oz_trace(long long* host128);
/* Profiling builds only (-DCGL_PROF, tools/timeline.py): every warp of the
 * instrumented kernels appends {t0, t1 (globaltimer ns), kernel id, block,
 * warp} records (32 B) to `records` (device, `capacity` entries split in
 * 256 per-SM regions), counting in `counter` (device, 256 u64, one per SM).
 * Returns CGL_EINVAL in product builds. */
int cgl_prof_set(void* records, void* counter, unsigned capacity);
/* Block sparsity of a sliced CONSTANT operand: zmap[tile][chunk] = first
 * non-zero slice (S+1: block all zero); rows/cols/a_mode as in cgl_oz_slice. */
int cgl_oz_zmap(void* stream, int S, const int8_t* slices, int64_t rows, int64_t cols,
                int a_mode, int8_t* zmap);
/* nitems independent batched products (S = 7 or 8); C[f] + b*sC, element
 * (i, j) at i*ldc + j (complex elements); strides of A/B slices in bytes,
 * of exponents in ints.  Azmap/Bzmap (arrays of nitems, or NULL) let the
 * kernel skip the zero slice blocks of a constant operand exactly. */
int cgl_oz_gemm(void* stream, int S, int64_t M, int64_t N, int64_t K, int nitems,
                const int8_t* const* A, const int* const* Aexp, const int8_t* const* Azmap,
                const int8_t* const* B, const int* const* Bexp, const int8_t* const* Bzmap,
                double* const* C, int64_t ldc, int64_t batch,
                int64_t sA, int64_t sAexp, int64_t sB, int64_t sBexp, int64_t sC,
                const cgl_flag_t* flag, uint64_t pos);

/* ---- pointwise kernels (HBM-bound) --------------------------------------- */

/* out = sum_i coef[i] * x[i] (nterms <= 6, real coefficients) —
 * integrators.py:130-143 (_axpy/_add/_scale). out may alias an x[i]. */
int cgl_lincomb(void* stream, int64_t n, int nterms, const double* coef,
                const double* const* x, double* out,
                const cgl_flag_t* flag, uint64_t pos);

/* out_c = g_c(in_scale * in) per component (flows.py:62-78). */
int cgl_eval_g(void* stream, int64_t n, const cgl_nonlinear_t* nl, int nfields,
               const double* const* in, double in_scale, double* const* out,
               const cgl_flag_t* flag, uint64_t pos);

/* Exact cubic / quintic flows over time t of in_scale*in (flows.py:87-115);
 * raise CGL_BLOWUP_* / CGL_NONFINITE_* at pos. */
int cgl_cubic_flow(void* stream, int64_t n, double t, const cgl_nonlinear_t* nl,
                   const double* in, double in_scale, double* out,
                   cgl_flag_t* flag, uint64_t pos);
int cgl_quintic_flow(void* stream, int64_t n, double t, const cgl_nonlinear_t* nl,
                     const double* in, double in_scale, double* out,
                     cgl_flag_t* flag, uint64_t pos);

/* One fused RK4 step of size t on u' = g(u) (flows.py:118-133): one read and
 * one write per component, all four stages in registers. */
int cgl_rk4_flow(void* stream, int64_t n, double t, const cgl_nonlinear_t* nl,
                 int nfields, const double* const* in, double in_scale,
                 double* const* out, cgl_flag_t* flag, uint64_t pos);

/* Raise CGL_NONFINITE_STATE at pos if any value of any field is NaN/Inf
 * (integrators.py:274-278). */
int cgl_check_finite(void* stream, int64_t n, int nfields,
                     const double* const* x, cgl_flag_t* flag, uint64_t pos);

int cgl_flag_reset(void* stream, cgl_flag_t* flag);
int cgl_flag_advance(void* stream, cgl_flag_t* flag, unsigned long long nsteps);

/* ---- fused per-scheme stage kernels (csrc/stages.cu) -------------------- */
enum cgl_stage_program {
  CGL_STAGE_IF4_PRE = 0,    /* in u            -> out X1, X5           */
  CGL_STAGE_IF4_MID = 1,    /* in u2, a        -> out g3, s            */
  CGL_STAGE_IF4_END = 2,    /* in b, c, d, e   -> out u', X1', X5'     */
  CGL_STAGE_FLOW1 = 3,      /* in u            -> out v                */
  CGL_STAGE_FLOW2 = 4,      /* in u            -> out v, f             */
  CGL_STAGE_SPLIT4_MID = 5, /* in v, f         -> out c, f'            */
  CGL_STAGE_SPLIT4_END = 6, /* in f, c         -> out u', v', f'       */
  CGL_STAGE_STRANG_END = 7, /* in w            -> out u', v'           */
  CGL_STAGE_IF2_PRE = 8,    /* in u            -> out X, Y             */
  CGL_STAGE_IF2_END = 9,    /* in u2, o        -> out u', X', Y'       */
  /* Fourier if4 (spectral space, integrators.py:205-215 with E = exp(f tau symbol)) */
  CGL_STAGE_FIF4_S1 = 10,   /* in u, g1        -> out E1/2 (u + t/2 g1)            */
  CGL_STAGE_FIF4_S2 = 11,   /* in u, g2        -> out E1/2 u + t/2 g2              */
  CGL_STAGE_FIF4_S3 = 12,   /* in u, g3        -> out t E1/2 g3 + E1 u             */
  CGL_STAGE_FIF4_S4 = 13,   /* in u,g1,g2,g3,g4 -> out u' (+ check, step++)        */
  CGL_STAGE_FLOW_END = 14   /* in w (physical) -> out flow(w, t/2) (+ check, step++) */
};
/* One fused pass of a step body (integrators.py:146-215): see the program
 * table in csrc/stages.cu.  in/out: (#operands x nfields) pointers, operand
 * major.  *_END programs check finiteness and run the next step's prologue;
 * the step comes from pos (relative to flag->step when CGL_POS_DEVICE is
 * set).  in/out may alias elementwise (each point is read before written). */
int cgl_stage(void* stream, int program, int nfields, int64_t n,
              const cgl_nonlinear_t* nl, double tau, double in_scale,
              const double* const* in, double* const* out,
              cgl_flag_t* flag, uint64_t pos);

/* Fourier stage programs (CGL_STAGE_FIF4_*): the separable multipliers are
 * evaluated in-kernel from per-axis tables, tables[(fr*nfields + c)*ndim + d]
 * for fraction slot fr (0: 1/2, 1: 1), component c, axis d. */
int cgl_stage_fourier(void* stream, int program, int nfields, int ndim,
                      const int64_t* shape, const cgl_nonlinear_t* nl, double tau,
                      double in_scale, const double* const* tables,
                      const double* const* in, double* const* out,
                      cgl_flag_t* flag, uint64_t pos);

/* Column-block variants for the slab-sharded spectral layout: the local
 * field is the (shape[0] x cols) block of columns col_offset .. +cols of the
 * global (shape[0] x prod(shape[1:])) matrix (after the axis-0 transpose). */
int cgl_stage_fourier_cols(void* stream, int program, int nfields, int ndim,
                           const int64_t* shape, int64_t cols, int64_t col_offset,
                           const cgl_nonlinear_t* nl, double tau, double in_scale,
                           const double* const* tables, const double* const* in,
                           double* const* out, cgl_flag_t* flag, uint64_t pos);
int cgl_separable_mul_cols(void* stream, int ndim, const int64_t* shape, int64_t cols,
                           int64_t col_offset, const double* const* tables, double in_scale,
                           const double* in, double* out, const cgl_flag_t* flag, uint64_t pos);

/* Hadamard product out = factor .* in (spectral.py:123-129). */
int cgl_pointwise_mul(void* stream, int64_t n, const double* factor,
                      const double* in, double* out,
                      const cgl_flag_t* flag, uint64_t pos);

/* out = exp(s * symbol) elementwise (spectral.py:116-120). */
int cgl_symbol_exp(void* stream, int64_t n, double s, const double* symbol,
                   double* out);

/* Separable Fourier multiplier: out[j] = in_scale * prod_mu table_mu[j_mu] * in[j],
 * the factorised exp(f tau symbol) of spectral.py:89-120 (never reads an
 * N-sized E). tables: ndim device arrays of shape[mu] complex values. */
int cgl_separable_mul(void* stream, int ndim, const int64_t* shape,
                      const double* const* tables, double in_scale,
                      const double* in, double* out,
                      const cgl_flag_t* flag, uint64_t pos);

/* ---- FFT (cuFFT Z2Z) — spectral.py:79-86 --------------------------------- */
/* Forward is unnormalised; "inverse" here is the unnormalised backward
 * transform: callers fold the 1/N of dft_inverse into the next kernel's
 * in_scale. */
int cgl_fft_plan(int ndim, const int64_t* shape, void** plan);
int cgl_fft_exec(void* plan, void* stream, const double* in, double* out, int inverse);
/* Batched plan with advanced layout (cufftPlanMany semantics, embeds = n):
 * 2D slab transforms and strided 1D transforms along axis 0 of the
 * transposed column blocks in the slab-sharded 3D FFT. */
int cgl_fft_plan_many(int rank, const int64_t* n, int64_t batch, int64_t istride,
                      int64_t idist, int64_t ostride, int64_t odist, void** plan);
int cgl_fft_destroy(void* plan);

/* ---- Pencil-FFT passes with fused step programs (csrc/fftpass.cu) -------- */
/* One HBM pass of unnormalised length-shape[axis] transforms along `axis` of a
 * C-order complex128 field (2D/3D, power-of-two extents 16..512), with the
 * pointwise pieces of the Fourier steppers fused in (spectral.py:79-86 around
 * integrators.py:99-120, 161-164, 205-215).  A 3D transform is three passes
 * (axis 2 contiguous, axes 1 and 0 strided); the programs below fuse the
 * Lawson stage combinations, g, the exact flows, the finiteness check and
 * the separable exp(f tau symbol) multipliers into the first/last pass. */
enum cgl_fft_program {
  CGL_FFT_PLAIN = 0,      /* transform src -> dst (direction from `inverse`)         */
  CGL_FFT_IF4_START = 1,  /* last axis, inverse: u (spectral state) -> dst             */
  /* B1..B4 accumulate the Lawson combination out = E1 (u + t/6 g1) + t/3 E1/2 (g2 + g3)
   * + t/6 g4 (integrators.py:205-215) in ONE field acc, one term per stage:          */
  CGL_FFT_IF4_B1 = 2,     /* last axis: g1 = F src; g_out = acc = E1 (u + t/6 g1);
                             dst = F^-1 E1/2 (u + t/2 g1)                              */
  CGL_FFT_IF4_B2 = 3,     /* g2 = F src; g_out = g[0] + t/3 E1/2 g2; dst = F^-1 (E1/2 u + t/2 g2) */
  CGL_FFT_IF4_B3 = 4,     /* g3 = F src; g_out = g[0] + t/3 E1/2 g3; dst = F^-1 (t E1/2 g3 + E1 u) */
  CGL_FFT_IF4_B4 = 5,     /* g4 = F src; u_out = u + t/6 g4 with u = acc (checked);
                             dst = F^-1 u_out unless dst == NULL                       */
  CGL_FFT_G = 6,          /* dst = F g(scale * F^-1 src) along one axis                */
  CGL_FFT_STR_START = 7,  /* strided: dst = F flow(scale * u, t/2)  [step, seq 0]      */
  CGL_FFT_STR_A0 = 8,     /* strided: w = scale F^-1 src; u_out = flow(w, t/2) [seq 1],
                             checked; dst = F flow(u_out, t/2) [step + 1] unless NULL  */
  CGL_FFT_STR_MID = 9,    /* last axis: dst = F^-1 (E1 .* F src)                       */
  CGL_FFT_STR_A0F = 10    /* STR_A0 for the exact cubic flow (kind 0) with the two flows at the
                             step boundary evaluated as one (semigroup; the reference's checks
                             and positions kept): u_out = w = scale F^-1 src, the step's state
                             being flow(u_out, t/2); dst = F flow(w, t) unless NULL          */
};
typedef struct {
  const double* u;           /* state operand (spectral for if4, physical for strang) */
  double* u_out;             /* state output                                        */
  const double* g[3];        /* g[0]: running combination acc (IF4_B2, B3); g[1..2] unused */
  double* g_out;             /* acc output (IF4_B1..B3; may alias g[0])              */
  const double* tables[2][3];/* separable exp(f tau symbol): [1/2, 1][axis]           */
  double tau, scale;
  cgl_nonlinear_t nl;        /* scalar kinds only (cubic / cubic_quintic)            */
  cgl_flag_t* flag;
  uint64_t pos;
} cgl_fft_ops_t;
/* 1 when the pass kernels support this grid, else 0 (no error set). */
int cgl_fft_pass_supported(int ndim, const int64_t* shape);
int cgl_fft_pass(void* stream, int program, int ndim, const int64_t* shape, int axis, int inverse,
                 const double* src, double* dst, const cgl_fft_ops_t* ops);

/* ---- Explicit Runge-Kutta stage on banded Kronecker-sum operators (csrc/rkstage.cu) ----
 * One stage of rk2 / rk4 (integrators.py:146-158 over Problem.rhs, tensors.py:72-84):
 *   f = sum_mu A_mu x_mu x + g(x);   x_out = u + cx f;   acc_out = (acc_in ? acc_in : u) + ca f
 * for per-direction factors A_mu of half-bandwidth halfband[mu] <= 8 (the FD
 * operators: 1 or 2), as ONE pass: the dense products of the reference reduce
 * exactly to (2 b + 1)-point contractions.  bands[c * ndim + mu]: complex
 * (shape[mu] x (2 b + 1)) array, band[i][d] = A[i][i + d - b] (zero outside);
 * x, u, acc_in, x_out, acc_out: arrays of nf (1 or 2) field pointers; acc_in,
 * x_out, acc_out may be NULL (not both outputs); x must not alias an output.
 * check != 0: acc_out is the step's new state, checked finite at (step, 255). */
int cgl_rk_stage(void* stream, int ndim, const int64_t* shape, int nf, const int* halfband,
                 const double* const* bands, const cgl_nonlinear_t* nl, const double* const* x,
                 const double* const* u, const double* const* acc_in, double* const* x_out,
                 double* const* acc_out, double cx, double ca, int check, cgl_flag_t* flag, uint64_t pos);

/* ---- Slab-sharded axis-0 transposes (csrc/slab.cu) ------------------------
 * A rank's slab of a global (world*planes, world*cols) field (axis 0 split,
 * C order) <-> its (world*planes, cols) column block, so the mu-mode product
 * along the sharded axis 0 (tensors.py:38-59, mu = 0) runs on whole fibres.
 * pack:   slab (planes, world, cols) -> blocks [world][planes][cols]
 * unpack: blocks [world][planes][cols] -> slab (planes, world, cols) */
int cgl_slab_pack(void* stream, int64_t world, int64_t planes, int64_t cols, const double* slab, double* blocks);
int cgl_slab_unpack(void* stream, int64_t world, int64_t planes, int64_t cols, const double* blocks,
                    double* slab);
/* dir 0: slab -> column block (pack into work, all-to-all into out);
 * dir 1: column block -> slab (all-to-all into work, unpack into out).
 * comm: the caller's ncclComm_t (world ranks); NCCL is resolved at run time
 * from the process (CGL_EUNAVAILABLE if none is loaded).  work: scratch of
 * planes*world*cols complex values.  in/out/work must not overlap. */
int cgl_slab_transpose(void* stream, void* comm, int world, int dir, int64_t planes, int64_t cols,
                       const double* in, double* out, double* work);

/* ---- Cross-mode fused 2D Tucker (csrc/tucker2d.cu) ------------------------
 * out_q = E0_q in_q E1_q^T for (n0 x n1) fields (n0, n1 <= 1024), mode 0 then
 * mode 1 (tensors.py:62-69) in ONE launch, the intermediate row in shared
 * memory.  e1t = E1^T.  band0/band1: int pairs [lo, hi] per row of E0 / E1,
 * the significant band (entries >= 2^-60 of the row max).
 * program 0: plain (1..8 items); 1: strang end-of-step (one scalar field):
 * out[0] = flow(E0 in E1^T, t/2) checked, out[1] = flow(out[0], t/2) of the
 * next step (integrators.py:161-164), positions as CGL_STAGE_STRANG_END. */
int cgl_tucker2d(void* stream, int program, int nitems, int64_t n0, int64_t n1, const double* const* in,
                 double* const* out, const double* const* e0, const double* const* e1t,
                 const int* const* band0, const int* const* band1, const cgl_nonlinear_t* nl, double tau,
                 cgl_flag_t* flag, uint64_t pos);

#ifdef __cplusplus
}
#endif

#endif /* CGL_B200_H */
