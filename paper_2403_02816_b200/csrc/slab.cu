// Axis-0 slab <-> column-block transposes of the slab-sharded 3D path.
//
// The mu-mode product along the sharded axis (reference tensors.py:38-59 with
// mu = 0) needs whole axis-0 fibres.  A rank holds the slab (p0, P, m) of a
// global field (n0, n1 n2) = (P p0, P m) in C order; the exchange gives rank
// r the column block (n0, m) = [P][p0][m] of columns r m .. r m + m - 1:
//   pack     slab (p0, P, m)   -> send [P][p0][m]   (rows of m elements permuted)
//   all-to-all (P blocks of p0 m elements per rank; receive = column block)
//   ... product on the column block ...
//   all-to-all back,  unpack [P][p0][m] -> slab (p0, P, m)
// Per-rank send volume 16 n0 n1 n2 (P - 1) / P^2 bytes per transpose.
//
// cgl_slab_transpose runs pack + exchange (+ unpack) for a C caller that owns
// an NCCL communicator.  NCCL is resolved at run time (dlsym on the NCCL the
// process has loaded -- the caller created its communicator with it), so the
// library has no link-time NCCL dependency and a caller's ncclComm_t is always
// used with the NCCL that made it.  The Python host (distributed.py) uses the
// same pack / unpack kernels with torch.distributed for the exchange.
#include <dlfcn.h>

#include "cgl_common.cuh"
#include "cgl_internal.h"

namespace cgl {

// dst row d = s p0 + i  <-  src row i P + s   (pack: slab -> [P][p0][m])
// dst row d = i P + s   <-  src row s p0 + i  (unpack)
// One CTA moves whole rows with 16-byte accesses; rows are m complex long.
__global__ void __launch_bounds__(256) slab_rows_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                                        int64_t P, int64_t p0, int64_t m, int unpack) {
  pdl_wait();
  const int64_t rows = P * p0;
  for (int64_t d = blockIdx.y; d < rows; d += gridDim.y) {
    const int64_t s = unpack ? d % P : d / p0;
    const int64_t i = unpack ? d / P : d % p0;
    const int64_t srow = unpack ? s * p0 + i : i * P + s;
    const double2* a = src + srow * m;
    double2* b = dst + d * m;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x)
      __stcs(b + c, __ldcs(a + c));
  }
  pdl_trigger();
}

int slab_rows(cudaStream_t st, const double* src, double* dst, int64_t P, int64_t p0, int64_t m, int unpack) {
  if (P < 1 || p0 < 1 || m < 1) return set_error(CGL_ESHAPE, "slab: empty extent");
  if (!src || !dst) return set_error(CGL_EINVAL, "slab: null buffer");
  if (src == dst && P > 1) return set_error(CGL_EINVAL, "slab: pack/unpack cannot run in place");
  const int64_t rows = P * p0;
  const int64_t bx = (m + 255) / 256 < 8 ? (m + 255) / 256 : 8;
  const int64_t by = rows < 65535 ? rows : 65535;
  cudaError_t e = launch_k(slab_rows_kernel, dim3((unsigned)bx, (unsigned)by), dim3(256), 0, st, dim3(1),
                           reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), P, p0, m, unpack);
  if (e != cudaSuccess) return set_cuda_error(e, "slab_rows launch");
  return check_launch("slab_rows_kernel");
}

// ---- NCCL, resolved at run time -----------------------------------------------
namespace {
typedef int (*nccl_send_t)(const void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_recv_t)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_t)();
constexpr int kNcclDouble = 8;  // ncclFloat64 (nccl.h)

struct NcclFns {
  nccl_send_t send = nullptr;
  nccl_recv_t recv = nullptr;
  nccl_group_t start = nullptr, end = nullptr;
  bool ok() const { return send && recv && start && end; }
};

NcclFns nccl_fns() {
  NcclFns f;
  f.send = reinterpret_cast<nccl_send_t>(dlsym(RTLD_DEFAULT, "ncclSend"));
  f.recv = reinterpret_cast<nccl_recv_t>(dlsym(RTLD_DEFAULT, "ncclRecv"));
  f.start = reinterpret_cast<nccl_group_t>(dlsym(RTLD_DEFAULT, "ncclGroupStart"));
  f.end = reinterpret_cast<nccl_group_t>(dlsym(RTLD_DEFAULT, "ncclGroupEnd"));
  if (!f.ok()) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (h) {
      f.send = reinterpret_cast<nccl_send_t>(dlsym(h, "ncclSend"));
      f.recv = reinterpret_cast<nccl_recv_t>(dlsym(h, "ncclRecv"));
      f.start = reinterpret_cast<nccl_group_t>(dlsym(h, "ncclGroupStart"));
      f.end = reinterpret_cast<nccl_group_t>(dlsym(h, "ncclGroupEnd"));
    }
  }
  return f;
}
}  // namespace

// All-to-all of P equal blocks of `count` doubles: block s of `send` goes to
// rank s, block s of `recv` comes from rank s.
int nccl_all_to_all(cudaStream_t st, void* comm, int world, const double* send, double* recv, size_t count) {
  static NcclFns f;
  if (!f.ok()) f = nccl_fns();  // resolved once NCCL is in the process
  if (!f.ok()) return set_error(CGL_EUNAVAILABLE, "slab_transpose: no NCCL loaded in this process");
  if (f.start() != 0) return set_error(CGL_ENCCL, "ncclGroupStart failed");
  for (int s = 0; s < world; ++s) {
    if (f.send(send + (size_t)s * count, count, kNcclDouble, s, comm, st) != 0 ||
        f.recv(recv + (size_t)s * count, count, kNcclDouble, s, comm, st) != 0) {
      f.end();
      return set_error(CGL_ENCCL, "ncclSend/ncclRecv failed");
    }
  }
  if (f.end() != 0) return set_error(CGL_ENCCL, "ncclGroupEnd failed");
  return 0;
}

}  // namespace cgl
