// tp_emu.cu -- the exchange step of tensor-parallel decode for T ranks that
// live in ONE process on one device (TpEmu: single-GPU validation of the
// sharding).  Same semantics as the NCCL path: allreduce = elementwise sum over
// ranks written back to every rank (here in rank order), allgather = rank-
// ordered concatenation.
#include "kernels.h"

namespace grt {

__global__ void emu_allreduce_kernel(TpPtrs bufs, int T, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float s = 0.0f;
    for (int r = 0; r < T; ++r) s += bufs.p[r][i];
    for (int r = 0; r < T; ++r) bufs.p[r][i] = s;
  }
}

__global__ void emu_allgather_kernel(TpPtrs in, TpPtrs out, int T, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n * T;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int src = static_cast<int>(i / n);
    const float v = in.p[src][i - static_cast<size_t>(src) * n];
    for (int r = 0; r < T; ++r) out.p[r][i] = v;
  }
}

cudaError_t launch_emu_allreduce(const TpPtrs& bufs, int T, size_t n, cudaStream_t s) {
  if (T < 1 || T > TP_MAX) return cudaErrorInvalidValue;
  emu_allreduce_kernel<<<static_cast<unsigned>((n + 255) / 256 > 1024 ? 1024 : (n + 255) / 256), 256, 0, s>>>(bufs, T, n);
  return cudaGetLastError();
}

cudaError_t launch_emu_allgather(const TpPtrs& in, const TpPtrs& out, int T, size_t n, cudaStream_t s) {
  if (T < 1 || T > TP_MAX) return cudaErrorInvalidValue;
  const size_t tot = n * T;
  emu_allgather_kernel<<<static_cast<unsigned>((tot + 255) / 256 > 1024 ? 1024 : (tot + 255) / 256), 256, 0, s>>>(
      in, out, T, n);
  return cudaGetLastError();
}

}  // namespace grt
