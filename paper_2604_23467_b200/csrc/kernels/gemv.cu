// gemv.cu -- per-op fused GEMV kernels (K1 QKV, K4 Wo, K5 gate/up, K6 down,
// K7 LM head) for sm_100a: the static decode pass is a
// graph of these plus the split-K attention kernel.
//
// Memory-bound design (decode is ~1 flop/byte; tensor cores stay idle):
//  * each warp owns a private ring of `stages` shared-memory slots (as deep as
//    the 227 KB opt-in budget allows after the activation row, up to
//    GEMV_MAX_STAGES); lane 0 streams weight row chunks with cp.async.bulk (TMA
//    engine, SASS UBLKCP) under an evict-first L2 policy, completion tracked by
//    one mbarrier per slot;
//  * the whole first ring fill -- and the norm weights -- are loaded BEFORE
//    griddepcontrol.wait, so with Programmatic Dependent Launch the kernel
//    streams its weights while the previous kernel drains;
//  * a CTA owns a contiguous range of row PAIRS (2p, 2p+1); its (pair, k-chunk)
//    tasks are dealt round-robin to the warps (equal bytes per warp), partial
//    dot products are summed per pair in shared memory, and the epilogues run
//    thread-parallel at the end; pairs let RoPE (rotate-half) and SwiGLU
//    finish in one epilogue;
//  * the QKV kernel prefetches this layer's K/V rows [0, seq_len) into L2 (and
//    warms their TLB entries) for the attention kernel that follows.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int GEMV_WARPS = 8;
constexpr int GEMV_MAX_STAGES = 8;
constexpr int GEMV_THREADS = GEMV_WARPS * 32;

// Activation prologue with the norm weights already in registers (they are
// weights, so they are loaded before griddepcontrol.wait): x is pulled into
// registers with independent 16-byte loads, reduced, normalised (reference
// layernorm kernels.cpp:66-83; RMSNorm drops mean and beta) and stored in the
// shared-memory layout dot_chunk expects.
template <typename WT, int NORM>
__device__ __forceinline__ void load_x_pre(const float* x, const float4* gv, const float4* bv, float eps, int k,
                                           float* xs, float* red) {
  const int n4 = k >> 2;
  float4 v[LOADX_MAXV];
#pragma unroll
  for (int i = 0; i < LOADX_MAXV; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    v[i] = j4 < n4 ? *reinterpret_cast<const float4*>(x + 4 * j4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float mean = 0.0f, inv = 1.0f;
  if constexpr (NORM == NORM_RMS) {
    float ss = 0.0f;
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    ss = block_sum(ss, red);
    inv = 1.0f / sqrtf(ss / static_cast<float>(k) + eps);
  } else if constexpr (NORM == NORM_LN) {
    float sm = 0.0f;
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) sm += v[i].x + v[i].y + v[i].z + v[i].w;
    mean = block_sum(sm, red) / static_cast<float>(k);
    float var = 0.0f;
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) {
      const int j4 = threadIdx.x + i * CONSUMER_THREADS;
      if (j4 < n4) {
        const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
        var += a * a + b * b + c * c + d * d;
      }
    }
    var = block_sum(var, red) / static_cast<float>(k);
    inv = 1.0f / sqrtf(var + eps);
  }
#pragma unroll
  for (int i = 0; i < LOADX_MAXV; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    if (j4 >= n4) continue;
    float4 o = v[i];
    if constexpr (NORM == NORM_RMS) {
      const float4 g = gv[i];
      o = make_float4(o.x * inv * g.x, o.y * inv * g.y, o.z * inv * g.z, o.w * inv * g.w);
    } else if constexpr (NORM == NORM_LN) {
      const float4 g = gv[i], b = bv[i];
      o = make_float4((o.x - mean) * inv * g.x + b.x, (o.y - mean) * inv * g.y + b.y, (o.z - mean) * inv * g.z + b.z,
                      (o.w - mean) * inv * g.w + b.w);
    }
    xs_store4<WT>(xs, j4, k, o);
  }
  consumer_sync();
}

// RMSNorm with the scale deferred: xs = x * gamma right away (the dots start
// after ONE barrier), the per-thread sum of squares is reduced after the
// streaming loop and 1/rms is applied to the finished dot products in the
// epilogue: out = inv * sum_k W_k (x_k g_k) == sum_k W_k (x_k inv g_k).
template <typename WT>
__device__ __forceinline__ float load_x_rms_deferred(const float* x, const float4* gv, int k, float* xs) {
  const int n4 = k >> 2;
  float4 v[LOADX_MAXV];
#pragma unroll
  for (int i = 0; i < LOADX_MAXV; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    v[i] = j4 < n4 ? *reinterpret_cast<const float4*>(x + 4 * j4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float ss = 0.0f;
#pragma unroll
  for (int i = 0; i < LOADX_MAXV; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    if (j4 < n4) {
      const float4 g = gv[i];
      xs_store4<WT>(xs, j4, k, make_float4(v[i].x * g.x, v[i].y * g.y, v[i].z * g.z, v[i].w * g.w));
    }
  }
  consumer_sync();
  return ss;
}

template <typename WT, int NORM, int EPI>
__global__ void __launch_bounds__(GEMV_THREADS, 1) gemv_kernel(const GemvParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[GEMV_WARPS][GEMV_MAX_STAGES];
  __shared__ float red[32];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.stages;
  const uint32_t rowb = static_cast<uint32_t>(p.rowb);
  const uint32_t stageb = 2 * rowb;
  uint8_t* mystage = smem + static_cast<size_t>(warp) * S * stageb;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(GEMV_WARPS) * S * stageb);

  const int CH = p.ch, nch = p.nch;
  const int n_pairs = (p.n_rows + 1) >> 1;
  const int pair_begin = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
  const int pair_end = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
  // The CTA's (pair, chunk) tasks are dealt round-robin to its warps: every
  // warp streams the same bytes (+-1 chunk) and at any moment the 8 warps read
  // 8 adjacent chunks.  Per-task dot products go to shared memory and are
  // summed per pair in chunk order at the end (deterministic).
  const int Tc = (pair_end - pair_begin) * nch;
  const int n_tasks = Tc > warp ? (Tc - warp + GEMV_WARPS - 1) / GEMV_WARPS : 0;
  float* part = xs + p.k;  // [pairs of this CTA][nch][2]
  uint64_t* mybar = bars[warp];
  const uint64_t pol = l2_evict_first_policy();
  const WT* Wt = reinterpret_cast<const WT*>(p.w);

  auto issue = [&](int i) {
    const int t = warp + i * GEMV_WARPS;
    const int pl = t / nch, c = t - pl * nch;
    const int row0 = 2 * (pair_begin + pl);
    const int c0 = c * CH;
    const int ce = min(CH, p.k - c0);
    const uint32_t bytes = static_cast<uint32_t>(ce) * sizeof(WT);
    const bool has_b = row0 + 1 < p.n_rows;
    const int slot = i % S;
    uint64_t* bar = &mybar[slot];
    uint8_t* dst = mystage + slot * stageb;
    mbar_arrive_expect_tx(bar, has_b ? 2 * bytes : bytes);
    const WT* src = Wt + static_cast<int64_t>(row0) * p.k + c0;
    bulk_g2s(dst, src, bytes, bar, pol);
    if (has_b) bulk_g2s(dst + rowb, src + p.k, bytes, bar, pol);
  };
  auto prefetch_l2 = [&](int i) {  // task i's rows into L2 only (keeps HBM busy while x is loaded)
    const int t = warp + i * GEMV_WARPS;
    const int pl = t / nch, c = t - pl * nch;
    const int row0 = 2 * (pair_begin + pl);
    const int c0 = c * CH;
    const uint32_t bytes = static_cast<uint32_t>(min(CH, p.k - c0)) * sizeof(WT);
    const WT* src = Wt + static_cast<int64_t>(row0) * p.k + c0;
    prefetch_l2_bulk(src, bytes);
    if (row0 + 1 < p.n_rows) prefetch_l2_bulk(src + p.k, bytes);
  };

  op_stamp(p.trace, 0);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  griddep_launch_dependents();
  // norm weights are weights too: in registers before the dependency wait, and
  // requested BEFORE the ring fill so they do not queue behind 190 KB of weights
  constexpr bool HAS_G = NORM == NORM_RMS || NORM == NORM_LN;
  float4 gv[HAS_G ? LOADX_MAXV : 1], bv[NORM == NORM_LN ? LOADX_MAXV : 1];
  const bool pre_norm = p.k <= LOADX_MAXV * 4 * CONSUMER_THREADS;
  if constexpr (HAS_G) {
    if (pre_norm) {
      const int n4 = p.k >> 2;
#pragma unroll
      for (int i = 0; i < LOADX_MAXV; ++i) {
        const int j4 = threadIdx.x + i * CONSUMER_THREADS;
        gv[i] = j4 < n4 ? __ldg(reinterpret_cast<const float4*>(p.gamma) + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (NORM == NORM_LN)
          bv[i] = j4 < n4 ? __ldg(reinterpret_cast<const float4*>(p.beta) + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  // Weights never depend on the previous kernel: start filling the ring now
  // (`pre_stages` slots; the rest right after the activation is in, so the
  // successor's whole-grid burst does not delay its own activation load).
  const int pre = min(min(S, p.pre_stages > 0 ? p.pre_stages : S), n_tasks);
  if (lane == 0) {
    for (int i = 0; i < pre; ++i) issue(i);
    if (pre == min(S, n_tasks))
      for (int i = pre; i < min(pre + p.l2_pre, n_tasks); ++i) prefetch_l2(i);
  }
  griddep_wait();
  op_stamp(p.trace, 1);
  const bool defer = NORM == NORM_RMS && pre_norm && p.rms_defer;
  float ss_part = 0.0f;
  if (defer)
    ss_part = load_x_rms_deferred<WT>(p.x, gv, p.k, xs);
  else if (HAS_G && pre_norm)
    load_x_pre<WT, (HAS_G ? NORM : NORM_RMS)>(p.x, gv, bv, p.eps, p.k, xs, red);
  else
    load_x<WT, NORM, false>(p.x, p.gamma, p.beta, p.eps, p.k, xs, red);
  op_stamp(p.trace, 2);
  if (lane == 0)
    for (int i = pre; i < min(S, n_tasks); ++i) issue(i);
  if constexpr (EPI == EPI_QKV || EPI == EPI_QKV_ROPE) {
    // (after the activation load, off its critical path) L2 prefetch (and TLB warm-up) of this layer's K/V rows [0, seq_len-1) for
    // the attention kernel: one contiguous [len, dh] run per (head, K|V).
    if (threadIdx.x == 0 && p.seq_len && static_cast<int>(blockIdx.x) < 2 * p.n_heads) {
      kv_prefetch_l2((blockIdx.x & 1) ? p.v_cache : p.k_cache, p.kvp, blockIdx.x >> 1, p.max_seq, p.head_dim,
                     p.kv_bf16 ? 2 : 4, max(0, *p.seq_len - 1));
    }
  }

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
  ea.kvp = p.kvp;

  for (int i = 0; i < n_tasks; ++i) {
    const int slot = i % S;
    mbar_wait(&mybar[slot], static_cast<uint32_t>((i / S) & 1));
    if (i == 0 && warp == 0) op_stamp(p.trace, 4);
    const int t = warp + i * GEMV_WARPS;
    const int c = t % nch;
    const int c0 = c * CH;
    const int ce = min(CH, p.k - c0);
    const uint8_t* st = mystage + slot * stageb;
    float acc_a = 0.0f, acc_b = 0.0f;
    dot_chunk<WT>(st, st + rowb, xs, p.k, c0, ce, acc_a, acc_b);
    __syncwarp();
    if (lane == 0 && i + S < n_tasks) {
      fence_proxy_async_smem();
      issue(i + S);
    }
    acc_a = warp_sum(acc_a);
    acc_b = warp_sum(acc_b);
    if (lane == 0) {
      part[2 * t] = acc_a;
      part[2 * t + 1] = acc_b;
    }
  }
  if (warp == 0) op_stamp(p.trace, 5);
  consumer_sync();
  float inv = 1.0f;
  if (defer) inv = 1.0f / sqrtf(block_sum(ss_part, red) / static_cast<float>(p.k) + p.eps);
  // Epilogues run thread-parallel (one pair per thread): their own memory
  // round trips (residual read, RoPE table) are paid once per CTA.
  for (int pl = threadIdx.x; pl < pair_end - pair_begin; pl += CONSUMER_THREADS) {
    float va = 0.0f, vb = 0.0f;
    for (int c = 0; c < nch; ++c) {
      va += part[2 * (pl * nch + c)];
      vb += part[2 * (pl * nch + c) + 1];
    }
    const int pair = pair_begin + pl;
    epilogue<EPI>(ea, pair, va * inv, vb * inv, 2 * pair + 1 < p.n_rows);
  }
  if (p.trace) {
    consumer_sync();
    op_stamp(p.trace, 3);
  }
}

// pairs a CTA owns at most (sizes the per-task partial sums in shared memory)
static int max_pairs_per_cta(int n_pairs, int grid) { return (n_pairs + grid - 1) / grid; }

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

static int smem_optin(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 227 * 1024;
  if (!cached[device]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cached[device] = n > 0 ? n : 227 * 1024;
  }
  return cached[device];
}

// chunking of a k-long row: near-equal chunks of <= CH elements, multiple of 8

static void chunking(Dt wdt, int k, int* ch, int* nch, int* rowb, int chmax_hint = 0) {
  int chmax = wdt == Dt::BF16 ? WTraits<__nv_bfloat16>::CH : WTraits<float>::CH;
  if (chmax_hint > 0 && wdt == Dt::BF16) chmax = chmax_hint;
  *nch = (k + chmax - 1) / chmax;
  *ch = ((k + *nch - 1) / *nch + 7) / 8 * 8;
  *rowb = ((*ch * (wdt == Dt::BF16 ? 2 : 4) + 15) / 16) * 16;
}

static constexpr int kStaticSmemReserve = 1024;  // bars + red + alignment

int gemv_max_stages() { return GEMV_MAX_STAGES; }

static int stages_for(int device, int rowb, int k, int part_bytes) {
  const int budget = smem_optin(device) - kStaticSmemReserve - k * 4 - part_bytes;
  const int s = budget / (GEMV_WARPS * 2 * rowb);
  return std::max(1, std::min(gemv_max_stages(), s));
}

size_t gemv_smem_bytes(Dt wdt, int k) {
  int ch, nch, rowb, dev = 0;
  chunking(wdt, k, &ch, &nch, &rowb);
  cudaGetDevice(&dev);
  return static_cast<size_t>(GEMV_WARPS) * stages_for(dev, rowb, k, 0) * 2 * rowb + static_cast<size_t>(k) * sizeof(float);
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
  const int optin = smem_optin(device);
  const int norms[] = {NORM_NONE, NORM_LN, NORM_RMS};
  const int epis[] = {EPI_STORE, EPI_RESID, EPI_QKV, EPI_QKV_ROPE, EPI_SWIGLU, EPI_RELU};
  for (Dt dt : {Dt::F32, Dt::BF16})
    for (int n : norms)
      for (int e : epis) {
        GemvFn f = pick_any(dt, n, e);
        if (!f) continue;
        cudaFuncAttributes fa;
        cudaError_t err = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
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
  int dev = 0;
  cudaGetDevice(&dev);
  chunking(wdt, p.k, &p.ch, &p.nch, &p.rowb, p.chmax);
  const int n_pairs = (p.n_rows + 1) / 2;
  int grid = grid_ctas > 0 ? grid_ctas : num_sms(dev);
  grid = std::max(1, std::min(grid, (n_pairs * p.nch + GEMV_WARPS - 1) / GEMV_WARPS));
  const int part_bytes = max_pairs_per_cta(n_pairs, grid) * p.nch * 2 * 4;
  p.stages = stages_for(dev, p.rowb, p.k, part_bytes);
  // the whole first ring fill goes out before the dependency wait; no L2
  // prefetch beyond the ring (measured slower: 2.63-2.73 vs 2.58 ms/token);
  // RMSNorm's 1/rms applied to the finished dot products
  p.pre_stages = 0;
  p.l2_pre = 0;
  p.rms_defer = 1;
  if (static_cast<int64_t>(GEMV_WARPS) * p.stages * 2 * p.rowb + p.k * 4 + part_bytes >
      smem_optin(dev) - kStaticSmemReserve)
    return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMV_THREADS);
  cfg.dynamicSmemBytes = static_cast<size_t>(GEMV_WARPS) * p.stages * 2 * p.rowb + static_cast<size_t>(p.k) * 4 + part_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, f, p);
}

}  // namespace grt
