// Internal (C++) declarations shared by the CUDA translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/cgl_b200.h"

namespace cgl {

constexpr int kMaxItems = 8;

// INT8-emulated GEMM (ozgemm.cu) tile geometry, shared by the slicing layout
constexpr int kOzBM = 128;  // A-operand row tile (UMMA M)
constexpr int kOzBN = 32;   // B-operand row tile (output columns per CTA)
constexpr int kOzKC = 32;   // K bytes per pipeline chunk

struct GemmItem {
  const double* A;
  const double* B;
  double* C;
  const double* Y;
};

// One launch = nitems independent batched GEMMs of identical shape.
struct GemmArgs {
  int64_t M, N, K;
  int64_t lda, ldb, ldc, ldy;
  int64_t sA, sB, sC, sY;
  int64_t batch;
  double2 alpha;
  double beta;
  int m_fastest;  // tile order: consecutive CTAs walk M (reuse the B tile in L2)
  const cgl_flag_t* flag;
  uint64_t pos;
  // stream-K bookkeeping (filled by the launcher)
  int64_t total_iters;
  double* workspace;
  int* flags;
  int epoch;
  GemmItem items[kMaxItems];
};

int zgemm_launch(const GemmArgs& a, int nitems, cudaStream_t s);

// full-K data slicing (stages.cu): rows x K complex operand, element (r, k) at
// src[r * sr + k * sk]; same slices/exponents as the B-mode floor-digit slicing
bool rows_slice_ok(int64_t K, bool stage);
int rows_slice_qc(int64_t K, int64_t rows_total, int tpt_max, int* tpt);
int rows_slice_plain(cudaStream_t st, int nitems, const double* const* srcs, int64_t sr, int64_t sk, int64_t rows,
                     int64_t K, int64_t batch, int64_t src_bs, int8_t* const* outs, int64_t out_bs,
                     int* const* exps, int64_t exp_bs);

// pencil-FFT passes (fftpass.cu)
bool fft_pass_supported(int ndim, const int64_t* shape);
int fft_pass_launch(cudaStream_t st, int program, int ndim, const int64_t* shape, int axis, int inverse,
                    const double* src, double* dst, const cgl_fft_ops_t* ops);

// banded Kronecker-sum RK stage (rkstage.cu)
int rk_stage_launch(cudaStream_t st, int ndim, const int64_t* shape, int nf, const int* halfband,
                    const double* const* bands, const cgl_nonlinear_t* nl, const double* const* x,
                    const double* const* u, const double* const* acc_in, double* const* x_out,
                    double* const* acc_out, double cx, double ca, int check, cgl_flag_t* flag, uint64_t pos);

// slab transposes (slab.cu)
int slab_rows(cudaStream_t st, const double* src, double* dst, int64_t P, int64_t p0, int64_t m, int unpack);
int nccl_all_to_all(cudaStream_t st, void* comm, int world, const double* send, double* recv, size_t count);

// cross-mode fused 2D Tucker (tucker2d.cu)
int tucker2d_launch(cudaStream_t st, int program, int nitems, int64_t n0, int64_t n1, const double* const* in,
                    double* const* out, const double* const* e0, const double* const* e1t, const int* const* band0,
                    const int* const* band1, const cgl_nonlinear_t* nl, double tau, cgl_flag_t* flag, uint64_t pos);

// error plumbing (capi.cu)
// Launch with the programmatic-dependent-launch attribute (CGL_PDL=0
// disables) and an optional thread-block cluster shape.  Every kernel
// launched this way calls pdl_wait() before reading data produced by
// earlier kernels in the stream.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, dim3 cluster,
                     Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  unsigned na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster.x * cluster.y * cluster.z > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster.x;
    at[na].val.clusterDim.y = cluster.y;
    at[na].val.clusterDim.z = cluster.z;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_launch(const char* name);

}  // namespace cgl
