#include <cstdlib>
// extern "C" boundary (include/cgl_b200.h): argument validation, layout
// mapping of mu-mode products onto the batched GEMM, and error plumbing.
#include <cstdio>
#include <cstring>
#include <string>

#include "cgl_common.cuh"
#include "cgl_internal.h"

namespace cgl {

// launchers from pointwise.cu / fft.cu
int pw_lincomb(cudaStream_t, int64_t, int, const double*, const double* const*, double*, const cgl_flag_t*, uint64_t);
int pw_eval_g(cudaStream_t, int64_t, const cgl_nonlinear_t*, int, const double* const*, double, double* const*,
              const cgl_flag_t*, uint64_t);
int pw_exact_flow(cudaStream_t, int, int64_t, double, const cgl_nonlinear_t*, const double*, double, double*,
                  cgl_flag_t*, uint64_t);
int pw_rk4_flow(cudaStream_t, int64_t, double, const cgl_nonlinear_t*, int, const double* const*, double,
                double* const*, cgl_flag_t*, uint64_t);
int pw_check_finite(cudaStream_t, int64_t, int, const double* const*, cgl_flag_t*, uint64_t);
int pw_flag_reset(cudaStream_t, cgl_flag_t*);
int pw_flag_advance(cudaStream_t, cgl_flag_t*, unsigned long long);
int pw_mul(cudaStream_t, int64_t, const double*, const double*, double*, const cgl_flag_t*, uint64_t);
int pw_symexp(cudaStream_t, int64_t, double, const double*, double*);
int pw_separable(cudaStream_t, int, const int64_t*, const double* const*, double, const double*, double*,
                 const cgl_flag_t*, uint64_t, int64_t, int64_t);
int fft_plan_many(int, const int64_t*, int64_t, int64_t, int64_t, int64_t, int64_t, void**);
int fft_plan(int, const int64_t*, void**);
extern long long* g_oz_trace;
int fft_exec(void*, cudaStream_t, const double*, double*, int);
int fft_destroy(void*);
int oz_slice(cudaStream_t, int, const double*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int8_t*,
             int64_t, int*, int64_t);
int oz_gemm(cudaStream_t, int, int64_t, int64_t, int64_t, int, const int8_t* const*, const int* const*,
            const int8_t* const*, const int8_t* const*, const int* const*, const int8_t* const*, double* const*,
            int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, const cgl_flag_t*, uint64_t, int);
int oz_zmap(cudaStream_t, int, const int8_t*, int64_t, int64_t, int, int, int8_t*);
int oz_slice_multi(cudaStream_t, int, int, const double* const*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                   int, int8_t* const*, int64_t, int* const*, int64_t, int);
int64_t oz_slice_bytes(int, int64_t, int64_t, int, int);
int stage_launch(cudaStream_t, int, int, int64_t, const cgl_nonlinear_t*, double, double, const double* const*,
                 double* const*, cgl_flag_t*, uint64_t, int, const int64_t*, const double* const*, int64_t, int64_t);
int rng_uniforms(cudaStream_t, uint64_t, uint64_t, int64_t, double*);
int rng_seeded_ic(cudaStream_t, int, uint64_t, int, const int64_t*, const double* const*, double*);
int stage_slice_launch(cudaStream_t, int, int64_t, int64_t, const cgl_nonlinear_t*, double, double,
                       const double* const*, double* const*, cgl_flag_t*, uint64_t, int8_t* const*, int* const*);

static thread_local std::string g_err;
static unsigned long long g_launches = 0;

__global__ void dmma_probe_kernel(double* sink, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
  for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
  if (r == 1234.5) *sink = r;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("CGL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}
int set_cuda_error(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return (int)e;
}
int check_launch(const char* name) {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, name);
  return 0;
}

// Map out_f = alpha * (in_f x_axis mat_f) + beta * y_f onto one batched GEMM
// launch over nitems fields.  shape is the input shape; out replaces
// shape[axis] by m_out.
static int mode_product_multi(cudaStream_t st, int ndim, const int64_t* shape, int axis, int64_t m_out, int nitems,
                              const double* const* mats, const double* const* mats_t, const double* const* ins,
                              double* const* outs, double alpha, const double* const* ys, double beta,
                              const cgl_flag_t* flag, uint64_t pos) {
  if (ndim < 1 || ndim > 8) return set_error(CGL_ESHAPE, "mode_product: ndim must be 1..8");
  if (axis < 0 || axis >= ndim) return set_error(CGL_ESHAPE, "mode_product: axis out of range");
  if (nitems < 1 || nitems > kMaxItems) return set_error(CGL_EINVAL, "mode_product: 1..8 fields per launch");
  int64_t P = 1, Q = 1;
  for (int d = 0; d < axis; ++d) P *= shape[d];
  for (int d = axis + 1; d < ndim; ++d) Q *= shape[d];
  const int64_t n = shape[axis];
  for (int d = 0; d < ndim; ++d)
    if (shape[d] < 0) return set_error(CGL_ESHAPE, "mode_product: negative extent");
  if (m_out < 0) return set_error(CGL_ESHAPE, "mode_product: negative m_out");
  GemmArgs a{};
  a.alpha = make_double2(alpha, 0.0);
  a.beta = beta;
  a.flag = flag;
  a.pos = pos;
  bool have_y = false;
  for (int f = 0; f < nitems; ++f) {
    if (ins[f] == outs[f] && n > 0) return set_error(CGL_EINVAL, "mode_product: in and out must not alias");
    have_y |= (ys && ys[f]);
  }
  if (Q == 1) {
    // contiguous axis: Out (P x m) = In (P x n) * M^T
    a.M = P; a.N = m_out; a.K = n;
    a.lda = n; a.ldb = m_out; a.ldc = m_out; a.ldy = m_out;
    a.sA = a.sB = a.sC = a.sY = 0;
    a.batch = 1;
    a.m_fastest = 0;
    for (int f = 0; f < nitems; ++f) {
      if (!mats_t || !mats_t[f]) return set_error(CGL_EINVAL, "mode_product: last-axis product needs mat_t");
      a.items[f] = GemmItem{ins[f], mats_t[f], outs[f], have_y ? ys[f] : nullptr};
    }
  } else {
    // Out_p (m x Q) = M (m x n) * In_p (n x Q), batched over the P leading slabs
    a.M = m_out; a.N = Q; a.K = n;
    a.lda = n; a.ldb = Q; a.ldc = Q; a.ldy = Q;
    a.sA = 0; a.sB = n * Q; a.sC = m_out * Q; a.sY = m_out * Q;
    a.batch = P;
    a.m_fastest = 1;
    for (int f = 0; f < nitems; ++f) {
      if (!mats || !mats[f]) return set_error(CGL_EINVAL, "mode_product: null matrix");
      a.items[f] = GemmItem{mats[f], ins[f], outs[f], have_y ? ys[f] : nullptr};
    }
  }
  if (a.batch == 0) return 0;
  return zgemm_launch(a, nitems, st);
}

int cgl_prof_set_ozgemm(void*, void*, unsigned);
int cgl_prof_set_stages(void*, void*, unsigned);
int cgl_prof_set_pointwise(void*, void*, unsigned);
int cgl_prof_set_zgemm(void*, void*, unsigned);

}  // namespace cgl

using namespace cgl;

extern "C" {

const char* cgl_version(void) { return "cgl_b200 1.0 (sm_100a, DMMA complex-FP64)"; }
const char* cgl_last_error(void) { return g_err.c_str(); }
int cgl_abi_version(void) { return CGL_ABI_VERSION; }
unsigned long long cgl_launch_count(void) { return g_launches; }

int cgl_prof_set(void* records, void* counter, unsigned capacity) {
  // every translation unit holds its own copy of the record pointers
  static char msg[160];
  msg[0] = 0;
  if (cgl_prof_set_ozgemm(records, counter, capacity)) strcat(msg, " ozgemm");
  if (cgl_prof_set_stages(records, counter, capacity)) strcat(msg, " stages");
  if (cgl_prof_set_pointwise(records, counter, capacity)) strcat(msg, " pointwise");
  if (cgl_prof_set_zgemm(records, counter, capacity)) strcat(msg, " zgemm");
  if (!msg[0]) return 0;
  static char full[256];
  snprintf(full, sizeof full, "cgl_prof_set: not a profiling build (-DCGL_PROF) or symbol copy failed in:%s (%s)",
           msg, cudaGetErrorString(cudaGetLastError()));
  return set_error(CGL_EINVAL, full);
}

double cgl_probe_dmma(void* stream, int iters) {
  static double* sink = nullptr;
  if (!sink && cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return -1.0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256;
  dmma_probe_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(sink, iters);
  if (check_launch("dmma_probe")) return -1.0;
  // 8 DMMA.8x8x4 per iteration per warp, 2*8*8*4 flops each
  return (double)blocks * (threads / 32) * iters * 8.0 * 512.0;
}

int cgl_zgemm(void* stream, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int64_t sA, const double* B,
              int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC, int64_t batch, double alpha_re,
              double alpha_im, const double* Y, int64_t ldy, int64_t sY, double beta, const cgl_flag_t* flag,
              uint64_t pos) {
  if (M < 0 || N < 0 || K < 0 || batch < 0) return set_error(CGL_ESHAPE, "zgemm: negative size");
  if (lda < K || ldb < N || ldc < N || (Y && ldy < N)) return set_error(CGL_ESHAPE, "zgemm: leading dimension too small");
  GemmArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.lda = lda; a.ldb = ldb; a.ldc = ldc; a.ldy = ldy;
  a.sA = sA; a.sB = sB; a.sC = sC; a.sY = sY;
  a.batch = batch;
  a.alpha = make_double2(alpha_re, alpha_im);
  a.beta = beta;
  a.m_fastest = 1;
  a.flag = flag;
  a.pos = pos;
  a.items[0] = GemmItem{A, B, C, Y};
  if (batch == 0) return 0;
  return zgemm_launch(a, 1, (cudaStream_t)stream);
}

int cgl_mode_product(void* stream, int ndim, const int64_t* shape, int axis, const double* mat, const double* mat_t,
                     int64_t m_out, const double* in, double* out, double alpha, const double* y, double beta,
                     const cgl_flag_t* flag, uint64_t pos) {
  const double* ys[1] = {y};
  return mode_product_multi((cudaStream_t)stream, ndim, shape, axis, m_out, 1, &mat, &mat_t, &in, &out, alpha,
                            y ? ys : nullptr, beta, flag, pos);
}

int cgl_mode_product_batch(void* stream, int ndim, const int64_t* shape, int axis, int nfields,
                           const double* const* mats, const double* const* mats_t, int64_t m_out,
                           const double* const* ins, double* const* outs, double alpha, const double* const* ys,
                           double beta, const cgl_flag_t* flag, uint64_t pos) {
  return mode_product_multi((cudaStream_t)stream, ndim, shape, axis, m_out, nfields, mats, mats_t, ins, outs, alpha,
                            ys, beta, flag, pos);
}

int cgl_tucker(void* stream, int ndim, const int64_t* shape, int nfields, const double* const* mats,
               const double* const* mats_t, const double* const* in, double* const* out, double* const* work,
               const cgl_flag_t* flag, uint64_t pos) {
  if (nfields < 1 || nfields > kMaxItems) return set_error(CGL_EINVAL, "tucker: 1..8 fields per launch");
  if (ndim < 1 || ndim > 8) return set_error(CGL_ESHAPE, "tucker: ndim must be 1..8");
  if (ndim > 1 && !work) return set_error(CGL_EINVAL, "tucker: work buffers required for ndim > 1");
  const double* src[kMaxItems];
  double* dst[kMaxItems];
  const double* m[kMaxItems];
  const double* mt[kMaxItems];
  for (int f = 0; f < nfields; ++f) {
    if (in[f] == out[f]) return set_error(CGL_EINVAL, "tucker: in and out must not alias");
    src[f] = in[f];
  }
  for (int axis = 0; axis < ndim; ++axis) {
    const bool to_out = ((ndim - axis) % 2) == 1;  // the last product lands in out
    for (int f = 0; f < nfields; ++f) {
      dst[f] = to_out ? out[f] : work[f];
      m[f] = mats[f * ndim + axis];
      mt[f] = mats_t ? mats_t[f * ndim + axis] : nullptr;
    }
    int r = mode_product_multi((cudaStream_t)stream, ndim, shape, axis, shape[axis], nfields, m, mt, src, dst, 1.0,
                               nullptr, 0.0, flag, pos);
    if (r) return r;
    for (int f = 0; f < nfields; ++f) src[f] = dst[f];
  }
  return 0;
}

int cgl_lincomb(void* stream, int64_t n, int nterms, const double* coef, const double* const* x, double* out,
                const cgl_flag_t* flag, uint64_t pos) {
  return pw_lincomb((cudaStream_t)stream, n, nterms, coef, x, out, flag, pos);
}

int cgl_eval_g(void* stream, int64_t n, const cgl_nonlinear_t* nl, int nfields, const double* const* in,
               double in_scale, double* const* out, const cgl_flag_t* flag, uint64_t pos) {
  return pw_eval_g((cudaStream_t)stream, n, nl, nfields, in, in_scale, out, flag, pos);
}

int cgl_cubic_flow(void* stream, int64_t n, double t, const cgl_nonlinear_t* nl, const double* in, double in_scale,
                   double* out, cgl_flag_t* flag, uint64_t pos) {
  return pw_exact_flow((cudaStream_t)stream, 0, n, t, nl, in, in_scale, out, flag, pos);
}

int cgl_quintic_flow(void* stream, int64_t n, double t, const cgl_nonlinear_t* nl, const double* in, double in_scale,
                     double* out, cgl_flag_t* flag, uint64_t pos) {
  return pw_exact_flow((cudaStream_t)stream, 1, n, t, nl, in, in_scale, out, flag, pos);
}

int cgl_rk4_flow(void* stream, int64_t n, double t, const cgl_nonlinear_t* nl, int nfields, const double* const* in,
                 double in_scale, double* const* out, cgl_flag_t* flag, uint64_t pos) {
  return pw_rk4_flow((cudaStream_t)stream, n, t, nl, nfields, in, in_scale, out, flag, pos);
}

int cgl_check_finite(void* stream, int64_t n, int nfields, const double* const* x, cgl_flag_t* flag, uint64_t pos) {
  return pw_check_finite((cudaStream_t)stream, n, nfields, x, flag, pos);
}

int cgl_flag_reset(void* stream, cgl_flag_t* flag) { return pw_flag_reset((cudaStream_t)stream, flag); }
int cgl_flag_advance(void* stream, cgl_flag_t* flag, unsigned long long nsteps) {
  return pw_flag_advance((cudaStream_t)stream, flag, nsteps);
}

int cgl_pointwise_mul(void* stream, int64_t n, const double* factor, const double* in, double* out,
                      const cgl_flag_t* flag, uint64_t pos) {
  return pw_mul((cudaStream_t)stream, n, factor, in, out, flag, pos);
}

int cgl_symbol_exp(void* stream, int64_t n, double s, const double* symbol, double* out) {
  return pw_symexp((cudaStream_t)stream, n, s, symbol, out);
}

int cgl_separable_mul(void* stream, int ndim, const int64_t* shape, const double* const* tables, double in_scale,
                      const double* in, double* out, const cgl_flag_t* flag, uint64_t pos) {
  return pw_separable((cudaStream_t)stream, ndim, shape, tables, in_scale, in, out, flag, pos, 0, 0);
}

int cgl_separable_mul_cols(void* stream, int ndim, const int64_t* shape, int64_t cols, int64_t col_offset,
                           const double* const* tables, double in_scale, const double* in, double* out,
                           const cgl_flag_t* flag, uint64_t pos) {
  return pw_separable((cudaStream_t)stream, ndim, shape, tables, in_scale, in, out, flag, pos, cols, col_offset);
}

int cgl_fft_plan_many(int rank, const int64_t* n, int64_t batch, int64_t istride, int64_t idist, int64_t ostride,
                      int64_t odist, void** plan) {
  return fft_plan_many(rank, n, batch, istride, idist, ostride, odist, plan);
}

int cgl_stage(void* stream, int program, int nfields, int64_t n, const cgl_nonlinear_t* nl, double tau,
              double in_scale, const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos) {
  return stage_launch((cudaStream_t)stream, program, nfields, n, nl, tau, in_scale, in, out, flag, pos, 0, nullptr,
                      nullptr, 0, 0);
}

int cgl_stage_fourier(void* stream, int program, int nfields, int ndim, const int64_t* shape,
                      const cgl_nonlinear_t* nl, double tau, double in_scale, const double* const* tables,
                      const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos) {
  int64_t n = 1;
  for (int d = 0; d < ndim; ++d) n *= shape[d];
  return stage_launch((cudaStream_t)stream, program, nfields, n, nl, tau, in_scale, in, out, flag, pos, ndim, shape,
                      tables, 0, 0);
}

int cgl_stage_fourier_cols(void* stream, int program, int nfields, int ndim, const int64_t* shape, int64_t cols,
                           int64_t col_offset, const cgl_nonlinear_t* nl, double tau, double in_scale,
                           const double* const* tables, const double* const* in, double* const* out, cgl_flag_t* flag,
                           uint64_t pos) {
  return stage_launch((cudaStream_t)stream, program, nfields, shape[0] * cols, nl, tau, in_scale, in, out, flag, pos,
                      ndim, shape, tables, cols, col_offset);
}

int cgl_tucker2d(void* stream, int program, int nitems, int64_t n0, int64_t n1, const double* const* in,
                 double* const* out, const double* const* e0, const double* const* e1t, const int* const* band0,
                 const int* const* band1, const cgl_nonlinear_t* nl, double tau, cgl_flag_t* flag, uint64_t pos) {
  if (!in || !out || !e0 || !e1t || !band0 || !band1) return set_error(CGL_EINVAL, "tucker2d: null array");
  return tucker2d_launch((cudaStream_t)stream, program, nitems, n0, n1, in, out, e0, e1t, band0, band1, nl, tau,
                         flag, pos);
}

int cgl_slab_pack(void* stream, int64_t world, int64_t planes, int64_t cols, const double* slab, double* blocks) {
  return slab_rows((cudaStream_t)stream, slab, blocks, world, planes, cols, 0);
}

int cgl_slab_unpack(void* stream, int64_t world, int64_t planes, int64_t cols, const double* blocks, double* slab) {
  return slab_rows((cudaStream_t)stream, blocks, slab, world, planes, cols, 1);
}

int cgl_slab_transpose(void* stream, void* comm, int world, int dir, int64_t planes, int64_t cols, const double* in,
                       double* out, double* work) {
  if (world < 1 || (dir != 0 && dir != 1)) return set_error(CGL_EINVAL, "slab_transpose: world >= 1, dir 0/1");
  if (!comm) return set_error(CGL_EINVAL, "slab_transpose: null communicator");
  if (!in || !out || !work || in == out || in == work || out == work)
    return set_error(CGL_EINVAL, "slab_transpose: in/out/work must be distinct buffers");
  const size_t count = (size_t)planes * (size_t)cols * 2;  // doubles per block
  cudaStream_t st = (cudaStream_t)stream;
  if (dir == 0) {
    int r = slab_rows(st, in, work, world, planes, cols, 0);
    return r ? r : nccl_all_to_all(st, comm, world, work, out, count);
  }
  int r = nccl_all_to_all(st, comm, world, in, work, count);
  return r ? r : slab_rows(st, work, out, world, planes, cols, 1);
}

int cgl_fft_pass_supported(int ndim, const int64_t* shape) {
  return shape && fft_pass_supported(ndim, shape) ? 1 : 0;
}

int cgl_rk_stage(void* stream, int ndim, const int64_t* shape, int nf, const int* halfband,
                 const double* const* bands, const cgl_nonlinear_t* nl, const double* const* x,
                 const double* const* u, const double* const* acc_in, double* const* x_out,
                 double* const* acc_out, double cx, double ca, int check, cgl_flag_t* flag, uint64_t pos) {
  return rk_stage_launch((cudaStream_t)stream, ndim, shape, nf, halfband, bands, nl, x, u, acc_in, x_out, acc_out, cx,
                         ca, check, flag, pos);
}

int cgl_fft_pass(void* stream, int program, int ndim, const int64_t* shape, int axis, int inverse, const double* src,
                 double* dst, const cgl_fft_ops_t* ops) {
  if (!shape) return set_error(CGL_EINVAL, "fft_pass: null shape");
  return fft_pass_launch((cudaStream_t)stream, program, ndim, shape, axis, inverse, src, dst, ops);
}

int64_t cgl_oz_slice_bytes(int S, int64_t rows, int64_t cols, int a_mode) {
  return oz_slice_bytes(S, rows, cols, a_mode, a_mode ? kOzBM : kOzBN);
}

int cgl_oz_slice(void* stream, int S, const double* src, int64_t sr, int64_t sc, int64_t rows, int64_t cols,
                 int64_t batch, int64_t src_batch_stride, int a_mode, int8_t* out, int64_t out_batch_stride, int* exps,
                 int64_t exp_batch_stride) {
  return oz_slice((cudaStream_t)stream, S, src, sr, sc, rows, cols, batch, src_batch_stride, a_mode, a_mode ? kOzBM : kOzBN,
                  out, out_batch_stride, exps, exp_batch_stride);
}

int cgl_oz_gemm(void* stream, int S, int64_t M, int64_t N, int64_t K, int nitems, const int8_t* const* A,
                const int* const* Aexp, const int8_t* const* Azmap, const int8_t* const* B, const int* const* Bexp,
                const int8_t* const* Bzmap, double* const* C, int64_t ldc, int64_t batch, int64_t sA, int64_t sAexp,
                int64_t sB, int64_t sBexp, int64_t sC, const cgl_flag_t* flag, uint64_t pos) {
  return oz_gemm((cudaStream_t)stream, S, M, N, K, nitems, A, Aexp, Azmap, B, Bexp, Bzmap, C, ldc, batch, sA, sAexp,
                 sB, sBexp, sC, flag, pos, 0);
}

int cgl_oz_gemm_t(void* stream, int S, int64_t M, int64_t N, int64_t K, int nitems, const int8_t* const* A,
                  const int* const* Aexp, const int8_t* const* Azmap, const int8_t* const* B, const int* const* Bexp,
                  const int8_t* const* Bzmap, double* const* C, int64_t ldc, int64_t batch, int64_t sA, int64_t sAexp,
                  int64_t sB, int64_t sBexp, int64_t sC, const cgl_flag_t* flag, uint64_t pos) {
  return oz_gemm((cudaStream_t)stream, S, M, N, K, nitems, A, Aexp, Azmap, B, Bexp, Bzmap, C, ldc, batch, sA, sAexp,
                 sB, sBexp, sC, flag, pos, 1);
}

int cgl_oz_slice_multi(void* stream, int S, int nitems, const double* const* srcs, int64_t sr, int64_t sc,
                       int64_t rows, int64_t cols, int64_t batch, int64_t src_batch_stride, int a_mode,
                       int8_t* const* outs, int64_t out_batch_stride, int* const* exps, int64_t exp_batch_stride) {
  return oz_slice_multi((cudaStream_t)stream, S, nitems, srcs, sr, sc, rows, cols, batch, src_batch_stride, a_mode,
                        outs, out_batch_stride, exps, exp_batch_stride, 1);
}

int cgl_stage_slice(void* stream, int program, int64_t n0, int64_t Q, const cgl_nonlinear_t* nl, double tau,
                    double in_scale, const double* const* in, double* const* out, cgl_flag_t* flag, uint64_t pos,
                    int8_t* const* slices, int* const* exps) {
  if (!nl || !in || !slices || !exps) return set_error(CGL_EINVAL, "cgl_stage_slice: null argument");
  return stage_slice_launch((cudaStream_t)stream, program, n0, Q, nl, tau, in_scale, in, out, flag, pos, slices,
                            exps);
}

int cgl_uniforms(void* stream, uint64_t seed, uint64_t start, int64_t count, double* out) {
  if (count > 0 && !out) return set_error(CGL_EINVAL, "cgl_uniforms: null output");
  return rng_uniforms((cudaStream_t)stream, seed, start, count, out);
}

int cgl_seeded_ic(void* stream, int recipe, uint64_t seed, int ndim, const int64_t* shape,
                  const double* const* axes, double* out) {
  if (!shape || !out) return set_error(CGL_EINVAL, "cgl_seeded_ic: null argument");
  return rng_seeded_ic((cudaStream_t)stream, recipe, seed, ndim, shape, axes, out);
}

int cgl_oz_geometry(int* bm, int* bn, int* kc) {
  *bm = kOzBM;
  *bn = kOzBN;
  *kc = kOzKC;
  return 0;
}

int cgl_oz_trace(long long* host128) {
  if (!g_oz_trace) return -1;
  cudaError_t e = cudaMemcpy(host128, g_oz_trace, 128 * sizeof(long long), cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? 0 : (int)e;
}

int cgl_oz_zmap(void* stream, int S, const int8_t* slices, int64_t rows, int64_t cols, int a_mode, int8_t* zmap) {
  return oz_zmap((cudaStream_t)stream, S, slices, rows, cols, a_mode, a_mode ? kOzBM : kOzBN, zmap);
}

int cgl_fft_plan(int ndim, const int64_t* shape, void** plan) { return fft_plan(ndim, shape, plan); }
int cgl_fft_exec(void* plan, void* stream, const double* in, double* out, int inverse) {
  return fft_exec(plan, (cudaStream_t)stream, in, out, inverse);
}
int cgl_fft_destroy(void* plan) { return fft_destroy(plan); }

}  // extern "C"
