// init.cu -- weight materialisation into the device layout.
//
// Reference init_model (model.cpp:30-76) fills every tensor with
// uniform_symmetric(0.1) draws (prng.hpp:33-35).  Two schemes are supported:
//   * mt19937_64 in the reference draw order: generated on the host (the stream
//     is serial), uploaded with launch_map_copy;
//   * counter-based Philox4x32-10 keyed by (seed, tensor id, logical index):
//     generated directly on the device here, bit-identical to
//     oracle.c:oc_philox_weight, so a 13 GB LLaMA-2 7B needs no host upload.
// Either way the logical [k,n] reference tensor is scattered into the device
// layout ([n,k] rows, RoPE pair permutation, gate/up interleave) by MapDesc.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace grt {

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0;
    const uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__device__ __forceinline__ float philox_weight(uint64_t seed, uint32_t tid, uint64_t idx) {
  uint32_t c[4] = {static_cast<uint32_t>(idx), static_cast<uint32_t>(idx >> 32), tid, 0x67724954u};
  philox4x32_10(c, static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const uint64_t bits = ((static_cast<uint64_t>(c[1]) << 32) | c[0]) >> 11;
  const double u = static_cast<double>(bits) * 0x1.0p-53;
  return static_cast<float>((2.0 * u - 1.0) * static_cast<double>(0.1f));
}

__host__ __device__ __forceinline__ int64_t win_p1(const MapDesc& d) { return d.p1 > 0 ? d.p1 : d.rows; }
__host__ __device__ __forceinline__ int64_t win_j1(const MapDesc& d) { return d.j1 > 0 ? d.j1 : d.cols; }

// Physical element index of logical (p, j) of a [rows=k, cols=n] tensor
// (inside the shard window).
__device__ __forceinline__ int64_t phys_index(const MapDesc& d, int64_t p, int64_t j) {
  p -= d.p0;
  j -= d.j0;
  if (!d.transpose) return p * (win_j1(d) - d.j0) + j;
  int64_t jj = j;
  if (d.rope_pair) {
    const int64_t dh = d.head_dim, half = dh >> 1;
    const int64_t head = j / dh, e = j - head * dh;
    jj = head * dh + (e < half ? 2 * e : 2 * (e - half) + 1);
  }
  const int64_t row = d.row_base + jj * d.row_stride + d.row_offset;
  return row * d.ld + p;
}

__device__ __forceinline__ void store_dt(void* dst, int64_t i, float v, int dt) {
  if (dt == static_cast<int>(Dt::BF16))
    reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(dst)[i] = v;
}

__device__ __forceinline__ float load_dt(const void* src, int64_t i, int dt) {
  if (dt == static_cast<int>(Dt::BF16)) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(src)[i]);
  if (dt == 2) return __half2float(reinterpret_cast<const __half*>(src)[i]);  // f16 (checkpoints only)
  return reinterpret_cast<const float*>(src)[i];
}

// Iterate the logical tensor with p (the reduction index) fastest, so writes of
// a transposed matrix stay coalesced along the physical row.
__device__ __forceinline__ void window_coords(const MapDesc& d, int64_t t, int64_t& p, int64_t& j) {
  const int64_t wr = win_p1(d) - d.p0, wc = win_j1(d) - d.j0;
  if (d.transpose) {
    j = t / wr;
    p = t - j * wr;
  } else {
    p = t / wc;
    j = t - p * wc;
  }
  p += d.p0;
  j += d.j0;
}

__global__ void map_init_kernel(MapDesc d, void* dst, uint64_t seed, uint32_t tid) {
  const int64_t n = (win_p1(d) - d.p0) * (win_j1(d) - d.j0);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t p, j;
    window_coords(d, t, p, j);
    store_dt(dst, phys_index(d, p, j), philox_weight(seed, tid, p * d.cols + j), d.dst_dtype);
  }
}

__global__ void map_copy_kernel(MapDesc d, void* dst, const void* src, int src_dt, int src_out_in) {
  const int64_t n = (win_p1(d) - d.p0) * (win_j1(d) - d.j0);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t p, j;
    window_coords(d, t, p, j);
    const int64_t si = src_out_in ? j * d.rows + p : p * d.cols + j;
    store_dt(dst, phys_index(d, p, j), load_dt(src, si, src_dt), d.dst_dtype);
  }
}

// writes the shard window into `out` at its logical positions (full [rows, cols])
__global__ void map_read_kernel(MapDesc d, const void* dst, float* out) {
  const int64_t wc = win_j1(d) - d.j0;
  const int64_t n = (win_p1(d) - d.p0) * wc;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t p = d.p0 + t / wc, j = d.j0 + (t - (t / wc) * wc);
    out[p * d.cols + j] = load_dt(dst, phys_index(d, p, j), d.dst_dtype);
  }
}

static dim3 grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 64) b = 148 * 64;
  if (b < 1) b = 1;
  return dim3(static_cast<unsigned>(b));
}

cudaError_t launch_map_init(const MapDesc& d, void* dst, uint64_t seed, uint32_t tensor_id, cudaStream_t s) {
  map_init_kernel<<<grid_for((win_p1(d) - d.p0) * (win_j1(d) - d.j0)), 256, 0, s>>>(d, dst, seed, tensor_id);
  return cudaGetLastError();
}

cudaError_t launch_map_copy(const MapDesc& d, void* dst, const void* src, int src_dtype, bool src_out_in,
                            cudaStream_t s) {
  map_copy_kernel<<<grid_for(d.rows * d.cols), 256, 0, s>>>(d, dst, src, src_dtype, src_out_in ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_map_read(const MapDesc& d, const void* dst, float* out, cudaStream_t s) {
  map_read_kernel<<<grid_for(d.rows * d.cols), 256, 0, s>>>(d, dst, out);
  return cudaGetLastError();
}

}  // namespace grt
