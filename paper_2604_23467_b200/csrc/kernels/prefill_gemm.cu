// prefill_gemm.cu -- batched-prefill projection GEMMs on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Reference: prefill is P token-by-token passes of make_matmul
// (pipeline.cpp:207-214, kernels.cpp:23-50); the incremental == restart
// property (model_test.cpp:129-146) lets all P tokens go through each layer at
// once, turning every projection into a GEMM  Y[P, N] = X[P, K] . W[N, K]^T.
//
// Shape: the weight is the MMA's A operand (M = 128 weight rows per CTA, K-major
// as stored), the P tokens are B (N = up to 256 tokens per MMA, K-major bf16
// activations) -- weights are streamed from HBM exactly once per GEMM however
// many tokens there are (two N tiles / TMEM accumulators cover P <= 512).
//   * warp 0: TMA producer (cp.async.bulk.tensor.2d, SWIZZLE_128B, 64-wide K
//     blocks) into a `stages`-deep ring, mbarrier full/empty handshakes;
//   * warp 1: allocates TMEM and issues tcgen05.mma.cta_group::1.kind::f16
//     (bf16 x bf16 -> fp32, M=128, N=ntile, K=16 per instruction) from one
//     elected lane; tcgen05.commit frees ring slots and signals the epilogue;
//   * warps 2-5: epilogue -- tcgen05.ld 32x32b (one weight row per thread, 16
//     tokens per load) -> fused RoPE/KV-cache write, SwiGLU, residual add;
//   * small-M GEMMs (Wo, down) split K over several CTAs; partials go to a
//     global scratch and the last CTA of a tile sums them in split order
//     (deterministic).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace grt {

constexpr int PG_BM = 128;        // weight rows per CTA (UMMA M)
constexpr int PG_BK = 64;         // K elements per stage (one 128-byte swizzle row)
constexpr int PG_UK = 16;         // K per tcgen05.mma (kind::f16)
constexpr int PG_THREADS = 192;   // 6 warps
constexpr int PG_MAX_NT = 256;    // tokens per N tile (UMMA N max)

// ---- tcgen05 / TMA primitives (inline PTX) --------------------------------------

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: 8-row x 128-byte
// atoms, stride between atoms (SBO) 1024 B, LBO unused (1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (ignored for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO
  d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N=n.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(PG_BM >> 4) << 24);
}

// ---- epilogue -------------------------------------------------------------------

// Value v of weight row m (global) for token n; vp is row m^1's value (the
// RoPE / SwiGLU partner, adjacent TMEM lane).
__device__ __forceinline__ void pg_epilogue(const PrefillGemmParams& p, int m, int n, float v, float vp) {
  if (m >= p.M || n >= p.P) return;
  switch (p.epi) {
    case PG_EPI_STORE:
      p.out[static_cast<int64_t>(n) * p.M + m] = v;
      break;
    case PG_EPI_RESID: {
      float* o = p.out + static_cast<int64_t>(n) * p.M + m;
      *o = *o + v;
      break;
    }
    case PG_EPI_SWIGLU:
      if ((m & 1) == 0) {
        const float s = v / (1.0f + expf(-v));
        static_cast<__nv_bfloat16*>(p.out_bf16)[static_cast<int64_t>(n) * (p.M >> 1) + (m >> 1)] = __float2bfloat16_rn(s * vp);
      }
      break;
    default: {  // PG_EPI_QKV / PG_EPI_QKV_ROPE: same index math as the decode epilogue (gemv_core.cuh)
      if (m & 1) return;
      const int d = p.d_model, dh = p.head_dim;
      const int pos = p.start_pos + n;
      const int sec = m / d;
      const int lp = (m >> 1) - sec * (d >> 1);
      float ra = v, rb = vp;
      int e0, e1, head;
      if (p.epi == PG_EPI_QKV_ROPE && sec < 2) {
        const int half = dh >> 1;
        head = lp / half;
        const int i = lp - head * half;
        const float c = p.rope_cos[static_cast<int64_t>(pos) * half + i];
        const float s = p.rope_sin[static_cast<int64_t>(pos) * half + i];
        ra = v * c - vp * s;
        rb = vp * c + v * s;
        e0 = i;
        e1 = i + half;
      } else {
        const int e = 2 * lp;
        head = e / dh;
        e0 = e - head * dh;
        e1 = e0 + 1;
      }
      if (sec == 0) {
        float* q = p.q_out + static_cast<int64_t>(n) * d + head * dh;
        q[e0] = ra;
        q[e1] = rb;
      } else {
        void* cache = sec == 1 ? p.k_cache : p.v_cache;
        const int64_t base = (static_cast<int64_t>(head) * p.max_seq + pos) * dh;
        if (p.kv_bf16) {
          __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(cache) + base;
          c[e0] = __float2bfloat16_rn(ra);
          c[e1] = __float2bfloat16_rn(rb);
        } else {
          float* c = reinterpret_cast<float*>(cache) + base;
          c[e0] = ra;
          c[e1] = rb;
        }
      }
    }
  }
}

// ---- the kernel -----------------------------------------------------------------

__global__ void __launch_bounds__(PG_THREADS, 1)
    prefill_gemm_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                        const PrefillGemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[8], empty[8], acc_bar;
  __shared__ uint32_t tmem_base;
  __shared__ int s_last;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x / p.ksplit, split = blockIdx.x - m_tile * p.ksplit;
  const int m0 = m_tile * PG_BM;
  const int nkb = p.K / PG_BK;
  const int kb0 = static_cast<int>(static_cast<int64_t>(split) * nkb / p.ksplit);
  const int kb1 = static_cast<int>(static_cast<int64_t>(split + 1) * nkb / p.ksplit);
  const int S = p.stages;
  const uint32_t a_bytes = PG_BM * PG_BK * 2;
  const uint32_t b_tile_bytes = static_cast<uint32_t>(p.ntile) * PG_BK * 2;
  const uint32_t stage_bytes = a_bytes + p.n_ntiles * b_tile_bytes;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_bar, 1);
    mbar_fence_init();
  }
  if (warp == 1) {  // TMEM: one fp32 column per token, n_ntiles accumulators of ntile columns
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(p.n_ntiles * p.ntile)) cols <<= 1;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  griddep_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {
      // weights do not depend on the previous kernel: the first ring fill of W
      // could start before the wait, but the activation tile shares the stage
      // barrier, so wait first (prefill is not latency critical per kernel).
      griddep_wait();
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
        uint8_t* st = smem + static_cast<size_t>(s) * stage_bytes;
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        tma_load_2d(st, &map_w, kb * PG_BK, m0, &full[s]);
        for (int t = 0; t < p.n_ntiles; ++t)
          tma_load_2d(st + a_bytes + t * b_tile_bytes, &map_x, kb * PG_BK, t * p.ntile, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(p.ntile);
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + static_cast<size_t>(s) * stage_bytes);
#pragma unroll
        for (int k = 0; k < PG_BK / PG_UK; ++k) {
          const uint64_t ad = sw128_desc(sa + k * PG_UK * 2);
          for (int t = 0; t < p.n_ntiles; ++t) {
            const uint64_t bd = sw128_desc(sa + a_bytes + t * b_tile_bytes + k * PG_UK * 2);
            tc_mma_bf16(tmem + t * p.ntile, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
          }
        }
        tc_commit(&empty[s]);  // frees the slot once these MMAs have read it
      }
      tc_commit(&acc_bar);  // accumulators complete
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31 = weight rows
    const int lane_base = 32 * (warp & 3);
    const int m = m0 + lane_base + lane;
    mbar_wait(&acc_bar, 0);
    tc_fence_after();
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(lane_base) << 16);
    const bool split_k = p.ksplit > 1;
    const int P_pad = p.n_ntiles * p.ntile;
    float* mypart = split_k ? p.part + (static_cast<int64_t>(m_tile) * p.ksplit + split) * P_pad * PG_BM : nullptr;
    for (int t = 0; t < p.n_ntiles; ++t) {
      for (int c0 = 0; c0 < p.ntile; c0 += 16) {
        float v[16];
        tc_ld16(t_lane + t * p.ntile + c0, v);
        const int nb = t * p.ntile + c0;
        if (split_k) {
#pragma unroll
          for (int j = 0; j < 16; ++j) mypart[static_cast<int64_t>(nb + j) * PG_BM + lane_base + lane] = v[j];
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float vp = __shfl_xor_sync(0xffffffffu, v[j], 1);
            pg_epilogue(p, m, nb + j, v[j], vp);
          }
        }
      }
    }
    if (split_k) {
      // last CTA of this M tile sums the partials in split order
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 2 && lane == 0) s_last = atomicAdd(p.counters + m_tile, 1) == p.ksplit - 1;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (s_last) {
        __threadfence();
        const float* base = p.part + static_cast<int64_t>(m_tile) * p.ksplit * P_pad * PG_BM;
        for (int n = 0; n < p.P; ++n) {
          float v = 0.0f;
          for (int s = 0; s < p.ksplit; ++s) v += __ldcg(base + (static_cast<int64_t>(s) * P_pad + n) * PG_BM + lane_base + lane);
          const float vp = __shfl_xor_sync(0xffffffffu, v, 1);
          pg_epilogue(p, m, n, v, vp);
        }
        if (warp == 2 && lane == 0) p.counters[m_tile] = 0;  // self-reset
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(p.n_ntiles * p.ntile)) cols <<= 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols) : "memory");
  }
}

// ---- host side --------------------------------------------------------------------

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2D bf16 row-major [rows, cols] tensor, box [box_rows, 64 cols], 128-byte swizzle;
// rows beyond `rows` read as zero (token padding).
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {PG_BK, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

int prefill_gemm_ksplit(int M, int K, int sms) {
  const int m_tiles = (M + PG_BM - 1) / PG_BM;
  const int nkb = K / PG_BK;
  int ks = std::max(1, (sms + m_tiles - 1) / m_tiles);
  if (m_tiles * 2 > sms) ks = 1;  // already >= half a wave: no split
  return std::max(1, std::min(ks, std::min(nkb, 8)));
}

size_t prefill_gemm_part_floats(int M, int K, int P, int sms) {
  const int m_tiles = (M + PG_BM - 1) / PG_BM;
  const int ks = prefill_gemm_ksplit(M, K, sms);
  if (ks == 1) return 0;
  const int nt = P > PG_MAX_NT ? 2 : 1;
  const int ntile = ((P + nt - 1) / nt + 15) / 16 * 16;
  return static_cast<size_t>(m_tiles) * ks * nt * ntile * PG_BM;
}

cudaError_t prefill_gemm_prepare() {
  return cudaFuncSetAttribute(prefill_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
}

cudaError_t launch_prefill_gemm(const void* w, const void* x, PrefillGemmParams p, cudaStream_t s, bool pdl) {
  if (p.K % PG_BK != 0 || p.P < 1 || p.P > 2 * PG_MAX_NT || p.M < 1) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = num_sms(dev);
  p.n_ntiles = p.P > PG_MAX_NT ? 2 : 1;
  p.ntile = ((p.P + p.n_ntiles - 1) / p.n_ntiles + 15) / 16 * 16;
  p.ksplit = prefill_gemm_ksplit(p.M, p.K, sms);
  if (p.ksplit > 1 && (!p.part || !p.counters)) return cudaErrorInvalidValue;
  const int stage_bytes = PG_BM * PG_BK * 2 + p.n_ntiles * p.ntile * PG_BK * 2;
  const int budget = 220 * 1024 - 1024;
  p.stages = std::max(2, std::min(8, budget / stage_bytes));
  CUtensorMap mw, mx;
  if (!make_map(&mw, w, p.M, p.K, PG_BM)) return cudaErrorInvalidValue;
  if (!make_map(&mx, x, p.P, p.K, p.ntile)) return cudaErrorInvalidValue;
  const int m_tiles = (p.M + PG_BM - 1) / PG_BM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(m_tiles * p.ksplit);
  cfg.blockDim = dim3(PG_THREADS);
  cfg.dynamicSmemBytes = static_cast<size_t>(p.stages) * stage_bytes + 1024;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, prefill_gemm_kernel, mw, mx, p);
}

}  // namespace grt
