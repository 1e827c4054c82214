// stream_bench.cu -- design-space probe for the weight-streaming loop of the
// decode GEMVs (not part of the product).  Streams a 1 GiB buffer once per
// launch and reports GB/s for:
//   bulk  : per-warp rings of cp.async.bulk stages (stage bytes x depth x warps)
//   ldg   : ld.global.nc.L1::no_allocate.v4 with UNROLL loads in flight per lane
// Optional dot product against a shared-memory vector (compute=1) to see
// whether consumption keeps up.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(512, 1) bulk_stream(const uint8_t* __restrict__ src, size_t bytes, int stage_bytes,
                                                       int depth, int compute, float* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[16][16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const size_t n_stages = bytes / stage_bytes;
  const size_t gw = static_cast<size_t>(blockIdx.x) * nw + warp;
  const size_t tw = static_cast<size_t>(gridDim.x) * nw;
  uint8_t* ring = smem + static_cast<size_t>(warp) * depth * stage_bytes;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0) {
    for (int s = 0; s < depth; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  // this warp's stages: gw, gw+tw, ...
  const size_t mine = gw < n_stages ? (n_stages - gw + tw - 1) / tw : 0;
  auto issue = [&](size_t i) {
    const int slot = i % depth;
    uint64_t* bar = &bars[warp][slot];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(stage_bytes));
    const uint8_t* g = src + (gw + i * tw) * stage_bytes;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(ring + slot * stage_bytes)),
        "l"(g), "r"(stage_bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  };
  if (lane == 0)
    for (size_t i = 0; i < mine && i < static_cast<size_t>(depth); ++i) issue(i);
  float acc = 0.f;
  for (size_t i = 0; i < mine; ++i) {
    const int slot = i % depth;
    const uint32_t par = (i / depth) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bars[warp][slot])), "r"(par)
                   : "memory");
    if (compute) {
      const uint4* w = reinterpret_cast<const uint4*>(ring + slot * stage_bytes);
      for (int g = lane; g < stage_bytes / 16; g += 32) {
        const uint4 u = w[g];
        acc += __uint_as_float(u.x << 16) + __uint_as_float(u.y & 0xffff0000u) + __uint_as_float(u.z << 16) +
               __uint_as_float(u.w & 0xffff0000u);
      }
    }
    __syncwarp();
    if (lane == 0 && i + depth < mine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + depth);
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

// One producer thread (last warp) feeds a CTA ring of `depth` stages; consumer
// warp w takes stages w, w+nc, ...  (the decode_pass v4 structure).
__global__ void __launch_bounds__(544, 1) central_stream(const uint8_t* __restrict__ src, size_t bytes,
                                                          int stage_bytes, int depth, int nc, int compute,
                                                          float* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[32], empty[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t n_stages = bytes / stage_bytes;
  // this CTA's contiguous share of stages
  const size_t s0 = n_stages * blockIdx.x / gridDim.x, s1 = n_stages * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto wait = [&](uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok)
                   : "r"(smem_u32(b)), "r"(par)
                   : "memory");
  };
  if (warp == nc) {
    if (lane != 0) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (size_t i = s0; i < s1; ++i) {
      const uint32_t t = static_cast<uint32_t>(i - s0);
      const int slot = t % depth;
      wait(&empty[slot], ((t / depth) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])),
                   "r"(stage_bytes));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
          "%4;" ::"r"(smem_u32(smem + slot * stage_bytes)),
          "l"(src + i * stage_bytes), "r"(stage_bytes), "r"(smem_u32(&full[slot])), "l"(pol)
          : "memory");
    }
    return;
  }
  float acc = 0.f;
  for (size_t i = s0 + warp; i < s1; i += nc) {
    const uint32_t t = static_cast<uint32_t>(i - s0);
    const int slot = t % depth;
    wait(&full[slot], (t / depth) & 1);
    if (compute) {
      const uint4* w = reinterpret_cast<const uint4*>(smem + slot * stage_bytes);
      for (int g = lane; g < stage_bytes / 16; g += 32) {
        const uint4 u = w[g];
        acc += __uint_as_float(u.x << 16) + __uint_as_float(u.y & 0xffff0000u) + __uint_as_float(u.z << 16) +
               __uint_as_float(u.w & 0xffff0000u);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[slot])) : "memory");
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int UNROLL>
__global__ void __launch_bounds__(512) ldg_stream(const int4* __restrict__ src, size_t n16, float* out) {
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t nt = static_cast<size_t>(gridDim.x) * blockDim.x;
  float acc = 0.f;
  for (size_t base = tid; base < n16; base += nt * UNROLL) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const size_t i = base + u * nt;
      if (i < n16)
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(src + i));
      else
        v[u] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += __int_as_float(v[u].x) + __int_as_float(v[u].w);
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const size_t bytes = 1ull << 30;
  uint8_t* buf;
  float* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto&& fn) {
    fn();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes * 5 / (ms * 1e-3) / 1e9;
  };
  const int cfgs[][3] = {{8192, 1, 8},  {8192, 2, 8},  {8192, 3, 8},  {4096, 2, 8},  {4096, 4, 8},
                         {4096, 6, 8},  {2048, 4, 8},  {2048, 8, 8},  {16384, 1, 8}, {16384, 2, 8},
                         {8192, 1, 16}, {8192, 2, 16}, {4096, 2, 16}, {4096, 3, 16}, {2048, 6, 16},
                         {32768, 3, 2}, {16384, 3, 4}, {8192, 6, 4},  {8192, 4, 4},  {8192, 2, 4}};
  for (int compute = 0; compute < 2; ++compute)
    for (auto& c : cfgs) {
      const int sb = c[0], depth = c[1], nw = c[2];
      const size_t smem = static_cast<size_t>(sb) * depth * nw;
      if (smem > 220 * 1024) continue;
      double gbs = timeit([&] { bulk_stream<<<sms, nw * 32, smem>>>(buf, bytes, sb, depth, compute, out); });
      printf("bulk stage=%6d depth=%2d warps=%2d ring=%3zu KB compute=%d : %7.1f GB/s\n", sb, depth, nw, smem / 1024,
             compute, gbs);
    }
  cudaFuncSetAttribute(central_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int ccfgs[][3] = {{8192, 20, 12}, {8192, 20, 8}, {16384, 10, 8}, {16384, 12, 12}, {32768, 6, 8},
                          {4096, 32, 8},  {8192, 26, 12}};
  for (int compute = 0; compute < 2; ++compute)
    for (auto& c : ccfgs) {
      const int sb = c[0], depth = c[1], nc = c[2];
      const size_t smem = static_cast<size_t>(sb) * depth;
      double gbs = timeit([&] { central_stream<<<sms, (nc + 1) * 32, smem>>>(buf, bytes, sb, depth, nc, compute, out); });
      printf("central stage=%6d depth=%2d consumers=%2d ring=%3zu KB compute=%d : %7.1f GB/s\n", sb, depth, nc,
             smem / 1024, compute, gbs);
    }
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    double g4 = timeit([&] { ldg_stream<4><<<sms * blocks_per_sm, 512>>>((const int4*)buf, bytes / 16, out); });
    double g8 = timeit([&] { ldg_stream<8><<<sms * blocks_per_sm, 512>>>((const int4*)buf, bytes / 16, out); });
    printf("ldg 512thr x %d/SM : unroll4 %7.1f GB/s  unroll8 %7.1f GB/s\n", blocks_per_sm, g4, g8);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
