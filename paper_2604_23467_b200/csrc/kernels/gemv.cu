// gemv.cu -- the fused batch-1 GEMV family (K1 QKV, K4 Wo, K5 gate/up, K6 down,
// K7 LM head) for sm_100a.
//
// Reference ops replaced: make_layernorm (kernels.cpp:52-85) + make_matmul
// (kernels.cpp:23-50) + make_kv_write (kernels.cpp:188-203) + make_residual_add
// (kernels.cpp:162-174) + make_relu (kernels.cpp:176-186); LLaMA adds RMSNorm,
// RoPE and SwiGLU.  The reference computes out[j] = sum_p a[p] * W[p*n+j] with W
// stored [k,n]; the device stores W transposed ([n,k], row = output) so one
// output is one contiguous row.
//
// Memory-bound design (decode is ~1 flop/byte; tensor cores stay idle):
//  * each warp owns a private ring of GEMV_STAGES shared-memory slots; lane 0
//    streams weight row chunks with cp.async.bulk (TMA engine) under an
//    evict-first L2 policy, completion tracked by an mbarrier per slot;
//  * rows are consumed in adjacent pairs (2p, 2p+1) so RoPE / SwiGLU epilogues
//    see both operands in one warp; dot products reduce with warp shuffles;
//  * the first ring fill is issued BEFORE griddepcontrol.wait, so weight
//    streaming overlaps the previous kernel (Programmatic Dependent Launch);
//  * the normalised activation lives in shared memory as fp32 ("plane" layout
//    for bf16 weights so the two float4 reads per lane are conflict-free).
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace grt {

constexpr int GEMV_WARPS = 8;
constexpr int GEMV_STAGES = 2;
constexpr int GEMV_THREADS = GEMV_WARPS * 32;

template <typename WT>
struct WTraits;
template <>
struct WTraits<__nv_bfloat16> {
  static constexpr int VEC = 8;     // elements per 16-byte lane load
  static constexpr int CH = 2048;   // elements per row chunk (4 KB)
};
template <>
struct WTraits<float> {
  static constexpr int VEC = 4;
  static constexpr int CH = 1024;
};

// Index of element j in the shared-memory activation buffer.
template <typename WT>
__device__ __forceinline__ int xs_index(int j, int k) {
  if constexpr (WTraits<WT>::VEC == 8) {
    const int g = j >> 3, w = j & 7;
    return (w >> 2) * (k >> 1) + g * 4 + (w & 3);
  } else {
    return j;
  }
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();  // red reuse
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.0f;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// Activation prologue: xs = norm(x) (or x).  Loop shapes follow the reference
// layernorm (kernels.cpp:66-83); RMSNorm drops the mean and beta.
template <typename WT, int NORM>
__device__ __forceinline__ void load_x(const GemvParams& p, float* xs, float* red) {
  const int k = p.k;
  if constexpr (NORM == NORM_NONE) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) xs[xs_index<WT>(j, k)] = p.x[j];
  } else if constexpr (NORM == NORM_RMS) {
    float ss = 0.0f;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      const float v = p.x[j];
      ss += v * v;
    }
    ss = block_sum(ss, red);
    const float inv = 1.0f / sqrtf(ss / static_cast<float>(k) + p.eps);
    for (int j = threadIdx.x; j < k; j += blockDim.x) xs[xs_index<WT>(j, k)] = p.x[j] * inv * p.gamma[j];
  } else {
    float s = 0.0f;
    for (int j = threadIdx.x; j < k; j += blockDim.x) s += p.x[j];
    const float mean = block_sum(s, red) / static_cast<float>(k);
    float v = 0.0f;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      const float c = p.x[j] - mean;
      v += c * c;
    }
    const float var = block_sum(v, red) / static_cast<float>(k);
    const float inv = 1.0f / sqrtf(var + p.eps);
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      xs[xs_index<WT>(j, k)] = (p.x[j] - mean) * inv * p.gamma[j] + p.beta[j];
  }
  __syncthreads();
}

// Partial dot products of one row pair over one chunk [c0, c0+ce).
template <typename WT>
__device__ __forceinline__ void dot_chunk(const uint8_t* sa, const uint8_t* sb, const float* xs, int k, int c0,
                                          int ce, float& acc_a, float& acc_b) {
  const int lane = threadIdx.x & 31;
  if constexpr (WTraits<WT>::VEC == 8) {
    const uint4* wa = reinterpret_cast<const uint4*>(sa);
    const uint4* wb = reinterpret_cast<const uint4*>(sb);
    const float4* xa = reinterpret_cast<const float4*>(xs) + (c0 >> 3);
    const float4* xb = reinterpret_cast<const float4*>(xs + (k >> 1)) + (c0 >> 3);
    const int groups = ce >> 3;
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 4
    for (int g = lane; g < groups; g += 32) {
      const uint4 u = wa[g];
      const uint4 v = wb[g];
      const float4 x0 = xa[g];
      const float4 x1 = xb[g];
      a0 = fmaf(bf16lo(u.x), x0.x, a0);
      a1 = fmaf(bf16hi(u.x), x0.y, a1);
      a0 = fmaf(bf16lo(u.y), x0.z, a0);
      a1 = fmaf(bf16hi(u.y), x0.w, a1);
      a0 = fmaf(bf16lo(u.z), x1.x, a0);
      a1 = fmaf(bf16hi(u.z), x1.y, a1);
      a0 = fmaf(bf16lo(u.w), x1.z, a0);
      a1 = fmaf(bf16hi(u.w), x1.w, a1);
      b0 = fmaf(bf16lo(v.x), x0.x, b0);
      b1 = fmaf(bf16hi(v.x), x0.y, b1);
      b0 = fmaf(bf16lo(v.y), x0.z, b0);
      b1 = fmaf(bf16hi(v.y), x0.w, b1);
      b0 = fmaf(bf16lo(v.z), x1.x, b0);
      b1 = fmaf(bf16hi(v.z), x1.y, b1);
      b0 = fmaf(bf16lo(v.w), x1.z, b0);
      b1 = fmaf(bf16hi(v.w), x1.w, b1);
    }
    acc_a += a0 + a1;
    acc_b += b0 + b1;
  } else {
    const float4* wa = reinterpret_cast<const float4*>(sa);
    const float4* wb = reinterpret_cast<const float4*>(sb);
    const float4* xv = reinterpret_cast<const float4*>(xs) + (c0 >> 2);
    const int groups = ce >> 2;
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 4
    for (int g = lane; g < groups; g += 32) {
      const float4 u = wa[g];
      const float4 v = wb[g];
      const float4 x = xv[g];
      a0 = fmaf(u.x, x.x, a0);
      a1 = fmaf(u.y, x.y, a1);
      a0 = fmaf(u.z, x.z, a0);
      a1 = fmaf(u.w, x.w, a1);
      b0 = fmaf(v.x, x.x, b0);
      b1 = fmaf(v.y, x.y, b1);
      b0 = fmaf(v.z, x.z, b0);
      b1 = fmaf(v.w, x.w, b1);
    }
    acc_a += a0 + a1;
    acc_b += b0 + b1;
  }
}

template <typename KT>
__device__ __forceinline__ void kv_store(void* base, int64_t idx, float v) {
  store_cast(reinterpret_cast<KT*>(base) + idx, v);
}

template <int EPI>
__device__ __forceinline__ void epilogue(const GemvParams& p, int pair, float va, float vb, bool has_b) {
  const int row0 = 2 * pair;
  if constexpr (EPI == EPI_STORE) {
    p.out[row0] = va;
    if (has_b) p.out[row0 + 1] = vb;
  } else if constexpr (EPI == EPI_RESID) {
    p.out[row0] += va;
    if (has_b) p.out[row0 + 1] += vb;
  } else if constexpr (EPI == EPI_RELU) {
    p.out[row0] = fmaxf(va, 0.0f);
    if (has_b) p.out[row0 + 1] = fmaxf(vb, 0.0f);
  } else if constexpr (EPI == EPI_SWIGLU) {
    const float s = va / (1.0f + expf(-va));
    p.out[pair] = s * vb;
  } else {  // EPI_QKV / EPI_QKV_ROPE
    const int d = p.d_model, dh = p.head_dim;
    const int pos = *p.seq_len - 1;
    const int sec = row0 / d;
    const int lp = pair - sec * (d >> 1);
    float ra = va, rb = vb;
    int e0, e1, head;
    if (EPI == EPI_QKV_ROPE && sec < 2) {
      const int half = dh >> 1;
      head = lp / half;
      const int i = lp - head * half;
      const float c = p.rope_cos[static_cast<int64_t>(pos) * half + i];
      const float s = p.rope_sin[static_cast<int64_t>(pos) * half + i];
      ra = va * c - vb * s;
      rb = vb * c + va * s;
      e0 = i;
      e1 = i + half;
    } else {
      const int e = 2 * lp;
      head = e / dh;
      e0 = e - head * dh;
      e1 = e0 + 1;
    }
    if (sec == 0) {
      p.q_out[head * dh + e0] = ra;
      p.q_out[head * dh + e1] = rb;
    } else {
      void* cache = sec == 1 ? p.k_cache : p.v_cache;
      const int64_t base = (static_cast<int64_t>(head) * p.max_seq + pos) * dh;
      if (p.kv_bf16) {
        kv_store<__nv_bfloat16>(cache, base + e0, ra);
        kv_store<__nv_bfloat16>(cache, base + e1, rb);
      } else {
        kv_store<float>(cache, base + e0, ra);
        kv_store<float>(cache, base + e1, rb);
      }
    }
  }
}

template <typename WT, int NORM, int EPI>
__global__ void __launch_bounds__(GEMV_THREADS, 1) gemv_kernel(const GemvParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[GEMV_WARPS][GEMV_STAGES];
  __shared__ float red[32];
  constexpr int CH = WTraits<WT>::CH;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rowb = static_cast<uint32_t>(p.rowb);
  const uint32_t stageb = 2 * rowb;
  uint8_t* mystage = smem + static_cast<size_t>(warp) * GEMV_STAGES * stageb;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(GEMV_WARPS) * GEMV_STAGES * stageb);

  const int n_pairs = (p.n_rows + 1) >> 1;
  const int pair_begin = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
  const int pair_end = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
  const int nch = (p.k + CH - 1) / CH;
  const int span = pair_end - pair_begin - warp;
  const int my_pairs = span <= 0 ? 0 : (span + GEMV_WARPS - 1) / GEMV_WARPS;
  const int n_tasks = my_pairs * nch;
  uint64_t* mybar = bars[warp];
  const uint64_t pol = l2_evict_first_policy();
  const WT* W = reinterpret_cast<const WT*>(p.w);

  auto issue = [&](int t) {
    const int pi = t / nch, c = t - pi * nch;
    const int row0 = 2 * (pair_begin + warp + pi * GEMV_WARPS);
    const int c0 = c * CH;
    const int ce = min(CH, p.k - c0);
    const uint32_t bytes = static_cast<uint32_t>(ce) * sizeof(WT);
    const bool has_b = row0 + 1 < p.n_rows;
    const int slot = t % GEMV_STAGES;
    uint64_t* bar = &mybar[slot];
    uint8_t* dst = mystage + slot * stageb;
    mbar_arrive_expect_tx(bar, has_b ? 2 * bytes : bytes);
    const WT* src = W + static_cast<int64_t>(row0) * p.k + c0;
    bulk_g2s(dst, src, bytes, bar, pol);
    if (has_b) bulk_g2s(dst + rowb, src + p.k, bytes, bar, pol);
  };

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < GEMV_STAGES; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  griddep_launch_dependents();
  // Weights never depend on the previous kernel: start streaming now.
  if (lane == 0) {
    const int pre = min(GEMV_STAGES, n_tasks);
    for (int t = 0; t < pre; ++t) issue(t);
  }
  griddep_wait();
  load_x<WT, NORM>(p, xs, red);

  float acc_a = 0.0f, acc_b = 0.0f;
  for (int t = 0; t < n_tasks; ++t) {
    const int slot = t % GEMV_STAGES;
    mbar_wait(&mybar[slot], static_cast<uint32_t>((t / GEMV_STAGES) & 1));
    const int pi = t / nch, c = t - pi * nch;
    const int pair = pair_begin + warp + pi * GEMV_WARPS;
    const int c0 = c * CH;
    const int ce = min(CH, p.k - c0);
    const uint8_t* st = mystage + slot * stageb;
    dot_chunk<WT>(st, st + rowb, xs, p.k, c0, ce, acc_a, acc_b);
    __syncwarp();
    if (lane == 0 && t + GEMV_STAGES < n_tasks) {
      fence_proxy_async_smem();
      issue(t + GEMV_STAGES);
    }
    if (c == nch - 1) {
      const float va = warp_sum(acc_a);
      const float vb = warp_sum(acc_b);
      if (lane == 0) epilogue<EPI>(p, pair, va, vb, 2 * pair + 1 < p.n_rows);
      acc_a = 0.0f;
      acc_b = 0.0f;
    }
  }
}

// ---------------------------------------------------------------------------
// Host side

int num_sms(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    cached[device] = n > 0 ? n : 148;
  }
  return cached[device];
}

template <typename WT>
static int rowb_for(int k) {
  const int ce = std::min(WTraits<WT>::CH, k);
  return ((ce * static_cast<int>(sizeof(WT)) + 15) / 16) * 16;
}

size_t gemv_smem_bytes(Dt wdt, int k) {
  const int rowb = wdt == Dt::BF16 ? rowb_for<__nv_bfloat16>(k) : rowb_for<float>(k);
  return static_cast<size_t>(GEMV_WARPS) * GEMV_STAGES * 2 * rowb + static_cast<size_t>(k) * sizeof(float);
}

using GemvFn = void (*)(const GemvParams);

template <typename WT>
static GemvFn pick(int norm, int epi) {
#define GRT_CASE(N, E) \
  if (norm == N && epi == E) return gemv_kernel<WT, N, E>;
  GRT_CASE(NORM_NONE, EPI_STORE)
  GRT_CASE(NORM_NONE, EPI_RESID)
  GRT_CASE(NORM_LN, EPI_QKV)
  GRT_CASE(NORM_RMS, EPI_QKV_ROPE)
  GRT_CASE(NORM_RMS, EPI_QKV)
  GRT_CASE(NORM_LN, EPI_RELU)
  GRT_CASE(NORM_RMS, EPI_SWIGLU)
  GRT_CASE(NORM_LN, EPI_STORE)
  GRT_CASE(NORM_RMS, EPI_STORE)
#undef GRT_CASE
  return nullptr;
}

static GemvFn pick_any(Dt wdt, int norm, int epi) {
  return wdt == Dt::BF16 ? pick<__nv_bfloat16>(norm, epi) : pick<float>(norm, epi);
}

cudaError_t gemv_prepare(int device) {
  int optin = 0;
  cudaError_t err = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (err != cudaSuccess) return err;
  const int norms[] = {NORM_NONE, NORM_LN, NORM_RMS};
  const int epis[] = {EPI_STORE, EPI_RESID, EPI_QKV, EPI_QKV_ROPE, EPI_SWIGLU, EPI_RELU};
  for (Dt dt : {Dt::F32, Dt::BF16})
    for (int n : norms)
      for (int e : epis) {
        GemvFn f = pick_any(dt, n, e);
        if (!f) continue;
        cudaFuncAttributes fa;
        err = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
        if (err != cudaSuccess) return err;
        err = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   optin - static_cast<int>(fa.sharedSizeBytes));
        if (err != cudaSuccess) return err;
      }
  return cudaSuccess;
}

cudaError_t launch_gemv(Dt wdt, int norm, int epi, GemvParams p, cudaStream_t s, bool pdl, int grid_ctas) {
  GemvFn f = pick_any(wdt, norm, epi);
  if (!f) return cudaErrorInvalidValue;
  if (p.k % 8 != 0 || p.n_rows < 1) return cudaErrorInvalidValue;
  p.rowb = wdt == Dt::BF16 ? rowb_for<__nv_bfloat16>(p.k) : rowb_for<float>(p.k);
  int dev = 0;
  cudaGetDevice(&dev);
  const int n_pairs = (p.n_rows + 1) / 2;
  int grid = grid_ctas > 0 ? grid_ctas : num_sms(dev);
  grid = std::max(1, std::min(grid, (n_pairs + GEMV_WARPS - 1) / GEMV_WARPS));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMV_THREADS);
  cfg.dynamicSmemBytes = gemv_smem_bytes(wdt, p.k);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, f, p);
}

}  // namespace grt
