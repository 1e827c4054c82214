// tma_bench.cu -- design probe for the short-prompt prefill GEMM's weight
// stream (not part of the product).  Persistent CTAs stream a [R, K] bf16 weight
// matrix as (128-row tile, K split) items through a 3-stage ring of 4 TMA boxes
// (64 x 128, SWIZZLE_128B) per stage -- the prefill_gemm_kernel pattern at P <= 64
// -- from (a) the row-major layout (each box = 128 rows x 128 B, rows K*2 bytes
// apart) and (b) a tiled copy where each box is 16 KB contiguous.  No MMA: the
// consumer only waits and frees the slots.  Reports GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
               : "=r"(ok)
               : "r"(smem_u32(b)), "r"(par)
               : "memory");
  return ok;
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

constexpr int SMAX = 12, BOX = 128 * 64 * 2;

__global__ void __launch_bounds__(64) stream(const __grid_constant__ CUtensorMap map, int m_tiles, int nkb, int ks,
                                             int tiled, int S, int KBOX) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[SMAX], empty[SMAX];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int n_items = m_tiles * ks;
  const int nst = nkb / KBOX;  // ring stages per tile
  if (threadIdx.x == 0) {
    int i = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int mt = w / ks, sp = w % ks;
      const int s0 = sp * nst / ks, s1 = (sp + 1) * nst / ks;
      for (int st = s0; st < s1; ++st, ++i) {
        const int s = i % S;
        while (!mbar_try(&empty[s], ((i / S) & 1) ^ 1)) {
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(KBOX * BOX));
        for (int j = 0; j < KBOX; ++j) {
          const int kb = st * KBOX + j;
          if (tiled)
            tma2d(sm + s * KBOX * BOX + j * BOX, &map, 0, (mt * nkb + kb) * 128, &full[s]);
          else
            tma2d(sm + s * KBOX * BOX + j * BOX, &map, kb * 64, mt * 128, &full[s]);
        }
      }
    }
  } else if (threadIdx.x == 32) {
    int i = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int sp = w % ks;
      const int s0 = sp * nst / ks, s1 = (sp + 1) * nst / ks;
      for (int st = s0; st < s1; ++st, ++i) {
        const int s = i % S;
        while (!mbar_try(&full[s], (i / S) & 1)) {
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      }
    }
  }
}


// the decode GEMV's pattern: 8 warps, each with a private ring of `depth`
// slots of 2 rows x `ch` elements, filled by cp.async.bulk (1D, contiguous)
__global__ void __launch_bounds__(256) bulk_stream(const __nv_bfloat16* __restrict__ w, int R, int K, int ch, int depth) {
  extern __shared__ __align__(128) uint8_t raw[];
  __shared__ uint64_t bars[8][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = K / ch;
  const uint32_t rowb = ch * 2, stageb = 2 * rowb;
  uint8_t* mine = raw + warp * depth * stageb;
  const int n_pairs = R / 2;
  const int pb = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
  const int pe = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
  const int tc = (pe - pb) * nch;
  const int nt = tc > warp ? (tc - warp + 7) / 8 : 0;
  if (lane == 0) {
    for (int s = 0; s < depth; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto issue = [&](int i) {
    const int t = warp + i * 8, pl = t / nch, c = t - pl * nch;
    const int slot = i % depth;
    uint64_t* bar = &bars[warp][slot];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(stageb));
    const __nv_bfloat16* src = w + static_cast<int64_t>(2 * (pb + pl)) * K + c * ch;
    for (int r = 0; r < 2; ++r)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(mine + slot * stageb + r * rowb)),
                   "l"(src + r * K), "r"(rowb), "r"(smem_u32(bar))
                   : "memory");
  };
  if (lane == 0)
    for (int i = 0; i < nt && i < depth; ++i) issue(i);
  for (int i = 0; i < nt; ++i) {
    while (!mbar_try(&bars[warp][i % depth], (i / depth) & 1)) {
    }
    __syncwarp();
    if (lane == 0 && i + depth < nt) issue(i + depth);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // ring geometry: stages x boxes per stage, CTAs per SM
  const int geo[][3] = {{3, 4, 1}, {6, 2, 1}, {12, 1, 1}, {2, 4, 1}, {3, 2, 2}, {6, 1, 2}, {2, 2, 3}, {3, 1, 4}};
  const int shapes[][3] = {{12288, 4096, 3}, {4096, 11008, 4}};
  void* flush = nullptr;
  cudaMalloc(&flush, 256u << 20);
  for (auto& sh : shapes) {
    const int R = sh[0], K = sh[1];
    const int Kp = (K + 255) / 256 * 256;
    const int m_tiles = R / 128, nkb = Kp / 64;
    void* w = nullptr;
    const size_t bytes = static_cast<size_t>(R) * Kp * 2;
    cudaMalloc(&w, bytes);
    cudaMemset(w, 0x3c, bytes);
    CUtensorMap map;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(R)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * 2};
    const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (auto& g : geo) {
      const int S = g[0], KB = g[1], cps = g[2];
      for (int ks : {sh[2], 2 * sh[2], 4 * sh[2]}) {
        if ((nkb / KB) < ks) continue;
        const int items = m_tiles * ks;
        const int grid = items < sms * cps ? items : sms * cps;
        const size_t smem = static_cast<size_t>(S) * KB * BOX + 1024;
        float tot = 0;
        for (int r = 0; r < 6; ++r) {
          cudaMemsetAsync(flush, r, 256u << 20);
          cudaEventRecord(e0);
          stream<<<grid, 64, smem>>>(map, m_tiles, nkb, ks, 0, S, KB);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (r > 0) tot += ms;
        }
        printf("R=%5d K=%5d stages=%2d boxes=%d ring=%3zu KB ctas/SM=%d ks=%2d items=%4d : %7.2f us %7.1f GB/s\n", R, K, S,
               KB, smem / 1024, cps, ks, items, tot / 5 * 1e3, bytes / (tot / 5 * 1e-3) / 1e9);
      }
    }
    cudaFree(w);
  }
  // decode-GEMV-style bulk rings on the same shapes
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int bshapes[][2] = {{12288, 4096}, {4096, 11008}, {22016, 4096}};
  for (auto& sh : bshapes) {
    const int R = sh[0], K = sh[1];
    void* w = nullptr;
    const size_t bytes = static_cast<size_t>(R) * K * 2;
    cudaMalloc(&w, bytes);
    cudaMemset(w, 0x3c, bytes);
    for (int ch : {2048, 1376, 1024, 512}) {
      if (K % ch) continue;
      for (int depth : {3, 2}) {
        const size_t smem = static_cast<size_t>(8) * depth * 2 * ch * 2;
        if (smem > 200 * 1024) continue;
        float tot = 0;
        for (int r = 0; r < 6; ++r) {
          cudaMemsetAsync(flush, r, 256u << 20);
          cudaEventRecord(e0);
          bulk_stream<<<sms, 256, smem>>>(static_cast<const __nv_bfloat16*>(w), R, K, ch, depth);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (r > 0) tot += ms;
        }
        printf("bulk R=%5d K=%5d chunk=%5d B depth=%d : %7.2f us %7.1f GB/s\n", R, K, ch * 2, depth, tot / 5 * 1e3,
               bytes / (tot / 5 * 1e-3) / 1e9);
      }
    }
    cudaFree(w);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
