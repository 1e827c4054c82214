// ring_bench.cu -- design probe for the decode GEMV's weight ring (not part of
// the product).  Streams a [rows, 4096] bf16 matrix once per launch the way
// gemv_kernel does -- each CTA owns a contiguous range of row PAIRS, its
// (pair, k-chunk) tasks are dealt round-robin to 8 warps, a task = two
// cp.async.bulk copies (rows 2p and 2p+1, `ch` elements each) into one ring
// slot, dot products against an fp32 x row in shared memory -- and reports GB/s
// for ring depth x chunk size x CTAs per SM (2: two independent CTAs share an
// SM, as two consecutive kernels would under PDL).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ring_bench tools/ring_bench.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int K = 4096, WARPS = 8;

__global__ void __launch_bounds__(WARPS * 32) ring(const __nv_bfloat16* __restrict__ w, int n_pairs, int ch, int depth,
                                                   float* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[WARPS][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = K / ch;
  const uint32_t rowb = ch * 2, stageb = 2 * rowb;
  uint8_t* mine = smem + warp * depth * stageb;
  float* xs = reinterpret_cast<float*>(smem + WARPS * depth * stageb);
  for (int j = threadIdx.x; j < K; j += blockDim.x) xs[j] = 1.0f / (1 + j);
  const int pb = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
  const int pe = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
  const int tc = (pe - pb) * nch;
  const int nt = tc > warp ? (tc - warp + WARPS - 1) / WARPS : 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0) {
    for (int s = 0; s < depth; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int t = warp + i * WARPS, pl = t / nch, c = t - pl * nch;
    const int slot = i % depth;
    uint64_t* bar = &bars[warp][slot];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(stageb));
    const __nv_bfloat16* src = w + static_cast<int64_t>(2 * (pb + pl)) * K + c * ch;
    for (int r = 0; r < 2; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
              smem_u32(mine + slot * stageb + r * rowb)),
          "l"(src + r * K), "r"(rowb), "r"(smem_u32(bar)), "l"(pol)
          : "memory");
  };
  if (lane == 0)
    for (int i = 0; i < nt && i < depth; ++i) issue(i);
  float acc = 0.f;
  for (int i = 0; i < nt; ++i) {
    const int slot = i % depth;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bars[warp][slot])), "r"((i / depth) & 1)
                   : "memory");
    const int t = warp + i * WARPS, c = t % nch;
    const uint4* a = reinterpret_cast<const uint4*>(mine + slot * stageb);
    const uint4* b = reinterpret_cast<const uint4*>(mine + slot * stageb + rowb);
    const float4* x = reinterpret_cast<const float4*>(xs + c * ch);
    for (int g = lane; g < ch / 8; g += 32) {
      const uint4 u = a[g], v = b[g];
      const float4 x0 = x[2 * g], x1 = x[2 * g + 1];
      acc += __uint_as_float(u.x << 16) * x0.x + __uint_as_float(u.y << 16) * x0.z + __uint_as_float(u.z << 16) * x1.x +
             __uint_as_float(u.w << 16) * x1.z + __uint_as_float(v.x << 16) * x0.y + __uint_as_float(v.w << 16) * x1.w;
    }
    __syncwarp();
    if (lane == 0 && i + depth < nt) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(i + depth);
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const int rows = 2 * 131072;  // 2 GiB of bf16 weights
  __nv_bfloat16* w;
  float* out;
  cudaMalloc(&w, static_cast<size_t>(rows) * K * 2);
  cudaMalloc(&out, 4);
  cudaMemset(w, 0x3c, static_cast<size_t>(rows) * K * 2);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int cfg[][3] = {{2048, 3, 1}, {2048, 2, 1}, {2048, 1, 1}, {1024, 3, 1}, {1024, 6, 1}, {4096, 1, 1},
                        {2048, 1, 2}, {1024, 2, 2}, {1024, 3, 2}, {2048, 2, 2}, {4096, 1, 2}, {1024, 1, 2}};
  for (auto& c : cfg) {
    const int ch = c[0], depth = c[1], bps = c[2];
    const size_t smem = static_cast<size_t>(WARPS) * depth * 2 * ch * 2 + K * 4;
    if (smem * bps > 226 * 1024) continue;
    auto run = [&] { ring<<<sms * bps, WARPS * 32, smem>>>(w, rows / 2, ch, depth, out); };
    run();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring, WARPS * 32, smem);
    printf("chunk=%5d B/row  depth=%d  CTAs/SM=%d (resident %d)  ring=%3zu KB/CTA : %7.1f GB/s\n", ch * 2, depth, bps,
           occ, smem / 1024, static_cast<double>(rows) * K * 2 * 5 / (ms * 1e-3) / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
