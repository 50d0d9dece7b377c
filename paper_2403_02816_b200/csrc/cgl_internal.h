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

// error plumbing (capi.cu)
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_launch(const char* name);

}  // namespace cgl
