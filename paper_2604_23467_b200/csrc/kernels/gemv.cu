// gemv.cu -- per-op fused GEMV kernels (K1 QKV, K4 Wo, K5 gate/up, K6 down,
// K7 LM head) for sm_100a.  Used by the per-op plan (eager-launch ablation and
// op-level tests); the default static pass is the persistent decode_pass.cu,
// built from the same device functions (gemv_core.cuh).
//
// Memory-bound design (decode is ~1 flop/byte; tensor cores stay idle):
//  * each warp owns a private ring of GEMV_STAGES shared-memory slots; lane 0
//    streams weight row chunks with cp.async.bulk (TMA engine, SASS UBLKCP)
//    under an evict-first L2 policy, completion tracked by an mbarrier per slot;
//  * the first ring fill is issued BEFORE griddepcontrol.wait, so weight
//    streaming overlaps the previous kernel (Programmatic Dependent Launch).
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int GEMV_WARPS = 8;
constexpr int GEMV_STAGES = 2;
constexpr int GEMV_THREADS = GEMV_WARPS * 32;

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
  load_x<WT, NORM, false>(p.x, p.gamma, p.beta, p.eps, p.k, xs, red);

  EpiArgs ea;
  ea.out = p.out;
  ea.q_out = p.q_out;
  ea.k_cache = p.k_cache;
  ea.v_cache = p.v_cache;
  ea.pos = p.seq_len ? *p.seq_len - 1 : 0;
  ea.rope_cos = p.rope_cos;
  ea.rope_sin = p.rope_sin;
  ea.head_dim = p.head_dim;
  ea.max_seq = p.max_seq;
  ea.d_model = p.d_model;
  ea.kv_bf16 = p.kv_bf16;

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
      if (lane == 0) epilogue<EPI>(ea, pair, va, vb, 2 * pair + 1 < p.n_rows);
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
