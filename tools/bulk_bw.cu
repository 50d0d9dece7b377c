// Per-SM cp.async.bulk ingress: grid CTAs each stream `iters` chunks of CHUNK
// bytes from an L2-resident source into a STAGES-deep smem ring, the chunk
// split into `pieces` bulk copies.  Prints GB/s per SM and chip-wide.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}\n" ::"r"(smem_u32(bar)), "r"(parity));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void kern(const uint8_t* src, size_t src_bytes, int chunk, int pieces, int iters, int nthreads_issue, int STAGES) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  const int piece = chunk / pieces;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
      const int st = i % STAGES;
      if (i >= STAGES) mbar_wait(&full[st], ((i / STAGES) - 1) & 1);
      __syncwarp();
      if (lane == 0) mbar_expect_tx(&full[st], chunk);
      __syncwarp();
      const size_t off = ((size_t)(blockIdx.x * 7919 + i * 104729) * chunk) % (src_bytes - chunk);
      for (int p = lane; p < pieces; p += nthreads_issue) {
        if (lane < nthreads_issue)
          bulk_g2s(smem + st * chunk + p * piece, src + (off & ~(size_t)1023) + p * piece, piece, &full[st]);
      }
    }
    for (int i = iters; i < iters + STAGES; ++i) {
      const int st = i % STAGES;
      mbar_wait(&full[st], ((i / STAGES) - 1) & 1);
    }
  }
}


// every warp of the CTA streams its own ring (stages per warp) with lane 0 issuing
__global__ void kern_warps(const uint8_t* src, size_t src_bytes, int chunk, int iters, int STAGES) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int nw = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nw * STAGES * chunk) + w * STAGES;
  uint8_t* ring = smem + (size_t)w * STAGES * chunk;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncwarp();
  if (lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int st = i % STAGES;
      if (i >= STAGES) mbar_wait(&full[st], ((i / STAGES) - 1) & 1);
      mbar_expect_tx(&full[st], chunk);
      const size_t off = ((size_t)((blockIdx.x * nw + w) * 7919 + i * 104729) * chunk) % (src_bytes - chunk);
      bulk_g2s(ring + st * chunk, src + (off & ~(size_t)1023), chunk, &full[st]);
    }
    for (int i = iters; i < iters + STAGES; ++i) mbar_wait(&full[i % STAGES], ((i / STAGES) - 1) & 1);
  }
}

int main(int argc, char** argv) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  size_t src_bytes = (size_t)(argc > 1 ? atoi(argv[1]) : 32) << 20;
  uint8_t* src;
  cudaMalloc(&src, src_bytes);
  cudaMemset(src, 1, src_bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case { int chunk, stages, per_sm; };
  const Case cases[] = {{8192, 4, 1}, {8192, 8, 1}, {8192, 16, 1}, {8192, 4, 2}, {8192, 4, 4},
                        {40960, 2, 1}, {40960, 4, 1}, {40960, 4, 2}, {40960, 5, 1},
                        {65536, 2, 1}, {65536, 3, 1}, {98304, 2, 1}, {20480, 8, 1}, {20480, 4, 2}};
  for (const Case& c : cases) {
    const int grid = nsm * c.per_sm, iters = 1000;
    const int smem = c.stages * c.chunk + 256;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) continue;
    kern<<<grid, 32, smem>>>(src, src_bytes, c.chunk, 1, 50, 1, c.stages);
    cudaEventRecord(e0);
    kern<<<grid, 32, smem>>>(src, src_bytes, c.chunk, 1, iters, 1, c.stages);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)grid * iters * c.chunk;
    printf("chunk %6d stages %2d ctas/SM %d : %7.1f GB/s per SM, %8.1f GB/s chip, %.3f us per chunk per CTA (%s)\n",
           c.chunk, c.stages, c.per_sm, bytes / nsm / (ms * 1e6), bytes / (ms * 1e6), ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int chunk : {8192, 20480, 40960}) {
    for (int nw : {1, 2, 4, 8}) {
      const int stages = 2, iters = 1000;
      const size_t smem = (size_t)nw * stages * chunk + nw * stages * 8 + 64;
      if (smem > 227 * 1024) continue;
      cudaFuncSetAttribute(kern_warps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern_warps<<<nsm, 32 * nw, smem>>>(src, src_bytes, chunk, 50, stages);
      cudaEventRecord(e0);
      kern_warps<<<nsm, 32 * nw, smem>>>(src, src_bytes, chunk, iters, stages);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)nsm * nw * iters * chunk;
      printf("warps %d chunk %6d: %7.1f GB/s per SM, %8.1f GB/s chip (%s)\n", nw, chunk, bytes / nsm / (ms * 1e6),
             bytes / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
