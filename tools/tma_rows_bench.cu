// tma_rows_bench.cu -- design probe (not part of the product): is the large-prompt
// prefill GEMM's operand feed bound by the 2D tensor TMA's per-row requests?
// 148 persistent CTAs run the GEMM's ring (S stages; one producer thread, one
// consumer thread that frees each slot as soon as it lands, no MMA) over
//   (a) 2D tensor boxes {64 K, BR rows}, SWIZZLE_128B -- BR row requests of 128 B
//       per box, the prefill_gemm_kernel pattern;
//   (b) 2D tensor boxes {32 K, BR rows}, SWIZZLE_64B  -- 64-byte rows;
//   (c) one 1D cp.async.bulk of the same bytes from a contiguous (pre-tiled) copy.
// Two operands: "tokens" (a [512, 4096] bf16 matrix every CTA reads, L2-resident,
// like the B operand) and "weights" (a [12288, 4096] matrix each CTA streams its
// own 128-row tiles of, HBM, like the A operand).  Reports aggregate GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rows_bench tools/tma_rows_bench.cu -lcuda
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
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int SMAX = 16;

// mode 0/1: tensor boxes (kbw K elements wide, br rows); mode 2: 1D bulk.
// own_rows: each CTA streams its own row tiles (weights) instead of shared ones.
// nprod producer warps (lane 0 each) take the stages i % nprod == w in turn.
__global__ void __launch_bounds__(160) feed(const __grid_constant__ CUtensorMap map, const uint8_t* lin, int mode, int br,
                                           int kbw, int S, int iters, int own_rows, int row_tiles, int K, int nprod) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[SMAX], empty[SMAX];
  const uint32_t box_bytes = static_cast<uint32_t>(br) * kbw * 2;
  const int nkb = K / kbw;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int pw = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && pw >= 1 && pw <= nprod) {
    for (int i = pw - 1; i < iters; i += nprod) {
      const int s = i % S;
      while (!mbar_try(&empty[s], ((i / S) & 1) ^ 1)) {
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(box_bytes));
      const int kb = i % nkb;
      const int rt = own_rows ? (blockIdx.x + (i / nkb) * gridDim.x) % row_tiles : 0;
      if (mode < 2) {
        tma2d(sm + s * box_bytes, &map, kb * kbw, rt * br, &full[s]);
      } else {  // tile (rt, kb) stored contiguously
        bulk1d(sm + s * box_bytes, lin + (static_cast<int64_t>(rt) * nkb + kb) * box_bytes, box_bytes, &full[s]);
      }
    }
  } else if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      while (!mbar_try(&full[s], (i / S) & 1)) {
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
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
  cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int K = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int own = 0; own < 2; ++own) {
    const int rows = own ? 12288 : 512;
    void* buf = nullptr;
    const size_t bytes = static_cast<size_t>(rows) * K * 2;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    for (int br : {128, 256}) {
      if (own && br != 128) continue;  // weights: 128-row tiles (UMMA M)
      for (int mode = 0; mode < 3; ++mode) {
        const int kbw = mode == 1 ? 32 : 64;
        const uint32_t box_bytes = br * kbw * 2;
        for (int nprod : {1, 2, 4}) {
          const int ring_kb = 192;
          const int S = ring_kb * 1024 / box_bytes;
          if (S < 2 || S > SMAX) continue;
          CUtensorMap map;
          const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
          const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
          const cuuint32_t box[2] = {static_cast<cuuint32_t>(kbw), static_cast<cuuint32_t>(br)};
          const cuuint32_t estr[2] = {1, 1};
          enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              mode == 1 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          const int row_tiles = rows / br;
          const int iters = own ? (row_tiles * (K / kbw)) / sms : 4096;
          const size_t smem = static_cast<size_t>(S) * box_bytes + 1024;
          feed<<<sms, 160, smem>>>(map, static_cast<const uint8_t*>(buf), mode, br, kbw, S, iters, own, row_tiles, K, nprod);
          cudaEventRecord(e0);
          for (int r = 0; r < 5; ++r)
            feed<<<sms, 160, smem>>>(map, static_cast<const uint8_t*>(buf), mode, br, kbw, S, iters, own, row_tiles, K,
                                     nprod);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double gb = 5.0 * sms * iters * static_cast<double>(box_bytes) / 1e9;
          printf("%-8s %s box=%3d rows x %3d B  ring=%3d KB (%2d stages) producers=%d: %8.1f GB/s  %6.0f cycles/box/SM (%s)\n",
                 own ? "weights" : "tokens", mode == 2 ? "1D bulk  " : "2D tensor", br, kbw * 2, ring_kb, S, nprod,
                 gb / (ms / 1e3), (ms / 1e3) * 1.965e9 / (5.0 * iters), cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
    cudaFree(buf);
  }
  return 0;
}
