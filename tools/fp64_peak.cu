// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) shapes.
// Reports achieved TFLOP/s for register-resident loops; used to pin the FP64
// roofline denominator that MEASURED_PEAKS.json does not carry.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dfma(double* out, double s) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  double b = 1.0000001, c = 0.9999999;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double r = 0; for (int i = 0; i < 8; ++i) r += a[i];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m8n8k4(double* out, double s) {
  double a = s + threadIdx.x, b = 1.0 - s;
  double c[4][2] = {};
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0; for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m16n8k4(double* out, double s) {
  double a0 = s + threadIdx.x, a1 = s, b = 1.0 - s;
  double c[4][4] = {};
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0; for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m16n8k8(double* out, double s) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = s + threadIdx.x + i;
  b[0] = 1 - s; b[1] = s;
  double c[4][4] = {};
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double r = 0; for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.0) out[0] = r;
}

__global__ void k_m16n8k16(double* out, double s) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = s + threadIdx.x + i;
  for (int i = 0; i < 4; ++i) b[i] = 1 - s * i;
  double c[4][4] = {};
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0; for (int i = 0; i < 4; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.0) out[0] = r;
}

template <typename K>
double run(K kern, int blocks, int threads, double flops_per_thread_iter, const char* name, double* d) {
  kern<<<blocks, threads>>>(d, 0.5);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, 0.5);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double fl = flops_per_thread_iter * ITERS * (double)blocks * threads;
  double tf = fl / (best * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", name, blocks, threads, best, tf);
  return tf;
}

int main() {
  double* d; cudaMalloc(&d, 64);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  printf("# %s sms=%d clock_khz=%d\n", p.name, sms, p.clockRate);
  for (int w : {4, 8, 16}) {
    int t = 32 * w;
    // flops per thread-iteration: DFMA 8 fma * 2; mma: shape flops*4 / 32 threads
    run(k_dfma, sms * 2, t, 16.0, "dfma", d);
    run(k_m8n8k4, sms * 2, t, 4.0 * 2 * 8 * 8 * 4 / 32.0, "mma_m8n8k4", d);
    run(k_m16n8k4, sms * 2, t, 4.0 * 2 * 16 * 8 * 4 / 32.0, "mma_m16n8k4", d);
    run(k_m16n8k8, sms * 2, t, 4.0 * 2 * 16 * 8 * 8 / 32.0, "mma_m16n8k8", d);
    run(k_m16n8k16, sms * 2, t, 4.0 * 2 * 16 * 8 * 16 / 32.0, "mma_m16n8k16", d);
  }
  cudaError_t e = cudaGetLastError();
  printf("# err=%s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
