// decode_pass.cu -- the static pass of one decode step as ONE persistent kernel.
//
// Reference: Model::build_plan (model.cpp:118-143) -- 14 kernels per layer, each
// a separate closure.  Batch-1 decode is bandwidth bound (13.2 GB of weights per
// token for LLaMA-2 7B), so what limits it on a B200 is not arithmetic but the
// bubbles between ~160 dependent kernels.  Here the whole pass is one launch:
//
//   * grid = one CTA per SM, 8 warps; every warp owns a ring of DP_STAGES
//     shared-memory slots that its lane 0 fills with cp.async.bulk (TMA engine)
//     copies of the weight-row chunks it will consume, in consumption order,
//     ACROSS phase and layer boundaries -- weights never depend on activations,
//     so the ring keeps HBM busy while the CTA waits for a dependency;
//   * phases per layer: QKV(+norm, RoPE, KV write) | attention | Wo(+residual) |
//     gate/up(+norm, SwiGLU) | down(+residual); the boundaries are device-side
//     dependency counters (release: __threadfence + atomicAdd; acquire: spin +
//     __threadfence); the last CTA out resets them for the next pass;
//   * activations produced by other CTAs in the same launch are read with
//     ld.global.cg (L2), never through a possibly stale L1 line;
//   * a watchdog turns a missing arrival into DEVERR_TIMEOUT instead of a hang.
#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int DP_WARPS = 8;
constexpr int DP_THREADS = DP_WARPS * 32;
constexpr int DP_STAGES = 5;
constexpr int DP_CH_BF16 = 1024;  // elements per row chunk: 2 KB -> 4 KB stages (row pair)
constexpr int DP_CH_F32 = 512;
constexpr uint32_t DP_STAGE_BYTES = 4096;
constexpr unsigned long long DP_WATCHDOG_NS = 2000000000ull;  // 2 s

enum SyncSlot { SY_QKV = 0, SY_ATTN = 1, SY_WO = 2, SY_UP = 3, SY_DOWN = 4, SY_HEADS = 8 };

int decode_pass_sync_stride(int n_heads) { return ((SY_HEADS + n_heads + 31) / 32) * 32; }

template <typename WT>
constexpr int dp_ch() {
  return sizeof(WT) == 2 ? DP_CH_BF16 : DP_CH_F32;
}

struct GemvPhase {
  const void* w;
  int n_rows;
  int k;
};

template <bool LLAMA>
__device__ __forceinline__ GemvPhase phase_desc(const PassParams& p, int ph) {
  if (ph >= 4 * p.n_layers) return {p.head, p.V, p.d};
  const PassLayer* L = p.layers + (ph >> 2);
  switch (ph & 3) {
    case 0: return {L->w_qkv, 3 * p.d, p.d};
    case 1: return {L->w_o, p.d, p.d};
    case 2: return {L->w_up, LLAMA ? 2 * p.ff : p.ff, p.d};
    default: return {L->w_down, p.d, p.ff};
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-warp producer state: walks (phase, pair, chunk) in consumption order.
template <typename WT, bool LLAMA>
struct Producer {
  int ph = 0, pi = 0, c = 0;
  int nch = 0, my_pairs = 0, pair_begin = 0, n_last = 0;
  GemvPhase g{};
  bool done = false;
  int t = 0;  // tasks issued

  __device__ void load_phase(const PassParams& p, int warp) {
    const int n_ph = 4 * p.n_layers + 1;
    for (; ph < n_ph; ++ph) {
      g = phase_desc<LLAMA>(p, ph);
      const int n_pairs = (g.n_rows + 1) >> 1;
      pair_begin = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
      const int pair_end = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
      const int span = pair_end - pair_begin - warp;
      my_pairs = span <= 0 ? 0 : (span + DP_WARPS - 1) / DP_WARPS;
      nch = (g.k + dp_ch<WT>() - 1) / dp_ch<WT>();
      if (my_pairs > 0) {
        pi = 0;
        c = 0;
        return;
      }
    }
    done = true;
  }

  // lane 0 only
  __device__ void issue(uint8_t* ring, uint64_t* bars, int warp, uint64_t pol) {
    constexpr int CH = dp_ch<WT>();
    const int row0 = 2 * (pair_begin + warp + pi * DP_WARPS);
    const int c0 = c * CH;
    const int ce = min(CH, g.k - c0);
    const uint32_t bytes = static_cast<uint32_t>(ce) * sizeof(WT);
    const bool has_b = row0 + 1 < g.n_rows;
    const int slot = t % DP_STAGES;
    uint64_t* bar = &bars[slot];
    uint8_t* dst = ring + slot * DP_STAGE_BYTES;
    mbar_arrive_expect_tx(bar, has_b ? 2 * bytes : bytes);
    const WT* src = reinterpret_cast<const WT*>(g.w) + static_cast<int64_t>(row0) * g.k + c0;
    bulk_g2s(dst, src, bytes, bar, pol);
    if (has_b) bulk_g2s(dst + DP_STAGE_BYTES / 2, src + g.k, bytes, bar, pol);
  }

  __device__ void advance(const PassParams& p, int warp) {
    ++t;
    if (++c < nch) return;
    c = 0;
    if (++pi < my_pairs) return;
    ++ph;
    load_phase(p, warp);
  }
};

// ---- dependency counters ------------------------------------------------------

__device__ __forceinline__ void phase_arrive(int* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
  }
}

// returns false on watchdog expiry (uniform across the CTA)
__device__ __forceinline__ bool phase_wait(int* ctr, int target, int* err, int* s_ok) {
  if (threadIdx.x == 0) {
    int ok = 1;
    const volatile int* v = ctr;
    if (*v < target) {
      const unsigned long long t0 = globaltimer();
      while (*v < target) {
        __nanosleep(64);
        if (globaltimer() - t0 > DP_WATCHDOG_NS) {
          atomicOr(err, DEVERR_TIMEOUT);
          ok = 0;
          break;
        }
      }
    }
    __threadfence();
    *s_ok = ok;
  }
  __syncthreads();
  return *s_ok != 0;
}

// ---- attention (one (head, split) work item per call; kernels.cpp:87-137) ----

template <typename KT>
__device__ __forceinline__ float4 kv_load4(const KT* p);
template <>
__device__ __forceinline__ float4 kv_load4<float>(const float* p) {
  return __ldcg(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 kv_load4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = __ldcg(reinterpret_cast<const uint2*>(p));
  return make_float4(bf16lo(u.x), bf16hi(u.x), bf16lo(u.y), bf16hi(u.y));
}

__device__ __forceinline__ float block_max_256(float v, float* red) {
  v = warp_max(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < DP_WARPS ? red[threadIdx.x] : -INFINITY;
    t = warp_max(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

template <typename KT>
__device__ void attention_item(const PassParams& p, const PassLayer& L, int layer, int head, int split, int len,
                               float* sm, float* red, int* s_last) {
  const int dh = p.dh, ns = p.nsplit;
  const int gs = dh >> 2;              // lanes per position
  const int npg = DP_THREADS / gs;     // position groups
  const int span = (len + ns - 1) / ns;
  const int j0 = split * span;
  const int n = max(0, min(len, j0 + span) - j0);
  float* qs = sm;
  float* sc = qs + dh;
  float* op = sc + p.span_cap;
  for (int d = threadIdx.x; d < dh; d += DP_THREADS) qs[d] = __ldcg(p.q + head * dh + d);
  __syncthreads();
  const KT* K = reinterpret_cast<const KT*>(L.k) + static_cast<int64_t>(head) * p.max_seq * dh;
  const KT* V = reinterpret_cast<const KT*>(L.v) + static_cast<int64_t>(head) * p.max_seq * dh;
  const int grp = threadIdx.x / gs, gl = threadIdx.x - grp * gs;
  const float4 q4 = reinterpret_cast<const float4*>(qs)[gl];
  for (int jb = 0; jb < n; jb += npg) {
    const int jj = jb + grp;
    float s = 0.0f;
    if (jj < n) {
      const float4 k4 = kv_load4<KT>(K + static_cast<int64_t>(j0 + jj) * dh + 4 * gl);
      s = q4.x * k4.x + q4.y * k4.y + q4.z * k4.z + q4.w * k4.w;
    }
    for (int o = gs >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (jj < n && gl == 0) sc[jj] = s * p.scale;
  }
  __syncthreads();
  float m = -INFINITY;
  for (int jj = threadIdx.x; jj < n; jj += DP_THREADS) m = fmaxf(m, sc[jj]);
  m = block_max_256(m, red);
  float l = 0.0f;
  for (int jj = threadIdx.x; jj < n; jj += DP_THREADS) {
    const float e = expf(sc[jj] - m);
    sc[jj] = e;
    l += e;
  }
  l = block_sum(l, red);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int jj = grp; jj < n; jj += npg) {
    const float e = sc[jj];
    const float4 v4 = kv_load4<KT>(V + static_cast<int64_t>(j0 + jj) * dh + 4 * gl);
    acc.x = fmaf(e, v4.x, acc.x);
    acc.y = fmaf(e, v4.y, acc.y);
    acc.z = fmaf(e, v4.z, acc.z);
    acc.w = fmaf(e, v4.w, acc.w);
  }
  reinterpret_cast<float4*>(op + grp * dh)[gl] = acc;
  __syncthreads();
  int* head_ctr = p.sync + layer * p.sync_stride + SY_HEADS + head;
  int* attn_ctr = p.sync + layer * p.sync_stride + SY_ATTN;
  if (ns == 1) {
    const float inv = 1.0f / l;
    for (int d = threadIdx.x; d < dh; d += DP_THREADS) {
      float o = 0.0f;
      for (int g = 0; g < npg; ++g) o += op[g * dh + d];
      p.attn[head * dh + d] = o * inv;
    }
    phase_arrive(attn_ctr);
    __syncthreads();
    return;
  }
  const int stride = dh + 2;
  float* mine = p.part + (static_cast<int64_t>(head) * ns + split) * stride;
  for (int d = threadIdx.x; d < dh; d += DP_THREADS) {
    float o = 0.0f;
    for (int g = 0; g < npg; ++g) o += op[g * dh + d];
    mine[d] = o;
  }
  if (threadIdx.x == 0) {
    mine[dh] = n > 0 ? m : -INFINITY;
    mine[dh + 1] = n > 0 ? l : 0.0f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *s_last = (atomicAdd(head_ctr, 1) == ns - 1);
    if (*s_last) __threadfence();
  }
  __syncthreads();
  if (!*s_last) return;
  // merge the splits in order (deterministic)
  const float* base = p.part + static_cast<int64_t>(head) * ns * stride;
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s)
    if (__ldcg(base + s * stride + dh + 1) > 0.0f) M = fmaxf(M, __ldcg(base + s * stride + dh));
  float Lsum = 0.0f;
  for (int s = 0; s < ns; ++s) {
    const float ls = __ldcg(base + s * stride + dh + 1);
    if (ls > 0.0f) Lsum += ls * expf(__ldcg(base + s * stride + dh) - M);
  }
  const float invL = 1.0f / Lsum;
  for (int d = threadIdx.x; d < dh; d += DP_THREADS) {
    float o = 0.0f;
    for (int s = 0; s < ns; ++s) {
      const float ls = __ldcg(base + s * stride + dh + 1);
      if (ls > 0.0f) o += __ldcg(base + s * stride + d) * expf(__ldcg(base + s * stride + dh) - M);
    }
    p.attn[head * dh + d] = o * invL;
  }
  phase_arrive(attn_ctr);
  __syncthreads();
}

// ---- the kernel -------------------------------------------------------------------

template <typename WT, typename KT, bool LLAMA>
__global__ void __launch_bounds__(DP_THREADS, 1) decode_pass_kernel(const PassParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[DP_WARPS][DP_STAGES];
  __shared__ float red[32];
  __shared__ int s_ok, s_last;
  constexpr int CH = dp_ch<WT>();
  constexpr int NORM = LLAMA ? NORM_RMS : NORM_LN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  uint8_t* ring = smem + static_cast<size_t>(warp) * DP_STAGES * DP_STAGE_BYTES;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(DP_WARPS) * DP_STAGES * DP_STAGE_BYTES);
  float* asm_ = xs + max(p.d, p.ff);  // attention scratch
  uint64_t* mybar = bars[warp];
  const uint64_t pol = l2_evict_first_policy();

  Producer<WT, LLAMA> prod;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < DP_STAGES; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  prod.load_phase(p, warp);
  // Weights do not depend on the previous kernel: fill the ring before waiting.
  for (int s = 0; s < DP_STAGES && !prod.done; ++s) {
    if (lane == 0) prod.issue(ring, mybar, warp, pol);
    prod.advance(p, warp);
  }
  griddep_wait();
  if (p.trace && threadIdx.x == 0)
    p.trace[static_cast<int64_t>(blockIdx.x) * p.trace_stride + p.n_layers * PASS_TRACE_PER_LAYER + 2] = globaltimer();

  const int len = *p.seq_len;
  EpiArgs ea;
  ea.pos = len - 1;
  ea.rope_cos = p.rope_cos;
  ea.rope_sin = p.rope_sin;
  ea.head_dim = p.dh;
  ea.max_seq = p.max_seq;
  ea.d_model = p.d;
  ea.kv_bf16 = sizeof(KT) == 2;
  ea.q_out = p.q;

  int t = 0;  // tasks consumed by this warp
  // Consume every task of GEMV phase `ph` with epilogue EPI.
  auto run_phase = [&](int ph, auto epi_tag) {
    constexpr int EPI = decltype(epi_tag)::value;
    const GemvPhase g = phase_desc<LLAMA>(p, ph);
    const int n_pairs = (g.n_rows + 1) >> 1;
    const int pb = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / G);
    const int pe = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / G);
    const int span = pe - pb - warp;
    const int my_pairs = span <= 0 ? 0 : (span + DP_WARPS - 1) / DP_WARPS;
    const int nch = (g.k + CH - 1) / CH;
    for (int pi = 0; pi < my_pairs; ++pi) {
      const int pair = pb + warp + pi * DP_WARPS;
      float acc_a = 0.0f, acc_b = 0.0f;
      for (int c = 0; c < nch; ++c, ++t) {
        const int slot = t % DP_STAGES;
        mbar_wait(&mybar[slot], static_cast<uint32_t>((t / DP_STAGES) & 1));
        const int c0 = c * CH;
        const uint8_t* st = ring + slot * DP_STAGE_BYTES;
        dot_chunk<WT>(st, st + DP_STAGE_BYTES / 2, xs, g.k, c0, min(CH, g.k - c0), acc_a, acc_b);
        __syncwarp();
        if (!prod.done) {
          if (lane == 0) {
            fence_proxy_async_smem();
            prod.issue(ring, mybar, warp, pol);
          }
          prod.advance(p, warp);
        }
      }
      const float va = warp_sum(acc_a);
      const float vb = warp_sum(acc_b);
      if (lane == 0) epilogue<EPI>(ea, pair, va, vb, 2 * pair + 1 < g.n_rows);
    }
  };
  using QkvTag = std::integral_constant<int, LLAMA ? EPI_QKV_ROPE : EPI_QKV>;
  using ResidTag = std::integral_constant<int, EPI_RESID>;
  using UpTag = std::integral_constant<int, LLAMA ? EPI_SWIGLU : EPI_RELU>;
  using StoreTag = std::integral_constant<int, EPI_STORE>;

  if (len < 1 || len > p.max_seq || (len + p.nsplit - 1) / p.nsplit > p.span_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.err, DEVERR_WRONG_LENGTH);
    // drain the prefetched stages so no bulk copy is outstanding at exit
    for (int s = 0; s < min(DP_STAGES, prod.t); ++s) mbar_wait(&mybar[s], 0);
    return;
  }

  unsigned long long* trace = p.trace ? p.trace + static_cast<int64_t>(blockIdx.x) * p.trace_stride : nullptr;
  auto stamp = [&](int ev) {
    if (trace && threadIdx.x == 0) trace[ev] = globaltimer();
  };

  for (int l = 0; l < p.n_layers; ++l) {
    const PassLayer L = p.layers[l];
    int* sy = p.sync + l * p.sync_stride;
    const int tb = l * PASS_TRACE_PER_LAYER;
    // ---- QKV: norm1 + q,k,v (+RoPE) + KV row write
    if (l > 0 && !phase_wait(p.sync + (l - 1) * p.sync_stride + SY_DOWN, G, p.err, &s_ok)) return;
    stamp(tb + 0);
    load_x<WT, NORM, true>(p.x, L.ln1_g, L.ln1_b, p.eps, p.d, xs, red);
    ea.k_cache = L.k;
    ea.v_cache = L.v;
    run_phase(4 * l + 0, QkvTag{});
    phase_arrive(sy + SY_QKV);
    stamp(tb + 1);
    // ---- attention over [0, len)
    if (!phase_wait(sy + SY_QKV, G, p.err, &s_ok)) return;
    stamp(tb + 2);
    const int items = p.h * p.nsplit;
    for (int it = blockIdx.x; it < items; it += G) {
      if (sizeof(KT) == 2)
        attention_item<__nv_bfloat16>(p, L, l, it / p.nsplit, it % p.nsplit, len, asm_, red, &s_last);
      else
        attention_item<float>(p, L, l, it / p.nsplit, it % p.nsplit, len, asm_, red, &s_last);
    }
    stamp(tb + 3);
    // ---- Wo + residual
    if (!phase_wait(sy + SY_ATTN, p.h, p.err, &s_ok)) return;
    stamp(tb + 4);
    load_x<WT, NORM_NONE, true>(p.attn, nullptr, nullptr, 0.f, p.d, xs, red);
    ea.out = p.x;
    run_phase(4 * l + 1, ResidTag{});
    phase_arrive(sy + SY_WO);
    stamp(tb + 5);
    // ---- norm2 + gate/up (SwiGLU) | W1 (ReLU)
    if (!phase_wait(sy + SY_WO, G, p.err, &s_ok)) return;
    stamp(tb + 6);
    load_x<WT, NORM, true>(p.x, L.ln2_g, L.ln2_b, p.eps, p.d, xs, red);
    ea.out = p.act;
    run_phase(4 * l + 2, UpTag{});
    phase_arrive(sy + SY_UP);
    stamp(tb + 7);
    // ---- down + residual
    if (!phase_wait(sy + SY_UP, G, p.err, &s_ok)) return;
    stamp(tb + 8);
    load_x<WT, NORM_NONE, true>(p.act, nullptr, nullptr, 0.f, p.ff, xs, red);
    ea.out = p.x;
    run_phase(4 * l + 3, ResidTag{});
    phase_arrive(sy + SY_DOWN);
    stamp(tb + 9);
  }
  // ---- ln_f + head
  if (!phase_wait(p.sync + (p.n_layers - 1) * p.sync_stride + SY_DOWN, G, p.err, &s_ok)) return;
  stamp(p.n_layers * PASS_TRACE_PER_LAYER + 0);
  load_x<WT, NORM, true>(p.x, p.lnf_g, p.lnf_b, p.eps, p.d, xs, red);
  ea.out = p.logits;
  run_phase(4 * p.n_layers, StoreTag{});
  stamp(p.n_layers * PASS_TRACE_PER_LAYER + 1);

  // Self-reset: the last CTA out zeroes every counter for the next pass (all
  // other CTAs have passed their last wait when they arrive here).
  __syncthreads();
  int* exit_ctr = p.sync + p.n_layers * p.sync_stride;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(exit_ctr, 1) == G - 1;
  }
  __syncthreads();
  if (s_last) {
    const int total = p.n_layers * p.sync_stride + 1;
    for (int i = threadIdx.x; i < total; i += DP_THREADS) p.sync[i] = 0;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------

using PassFn = void (*)(const PassParams);

static PassFn pick_pass(Dt wdt, Dt kvdt, bool llama) {
  if (wdt == Dt::BF16) {
    if (kvdt == Dt::BF16) return llama ? decode_pass_kernel<__nv_bfloat16, __nv_bfloat16, true>
                                       : decode_pass_kernel<__nv_bfloat16, __nv_bfloat16, false>;
    return llama ? decode_pass_kernel<__nv_bfloat16, float, true> : decode_pass_kernel<__nv_bfloat16, float, false>;
  }
  if (kvdt == Dt::BF16) return llama ? decode_pass_kernel<float, __nv_bfloat16, true>
                                     : decode_pass_kernel<float, __nv_bfloat16, false>;
  return llama ? decode_pass_kernel<float, float, true> : decode_pass_kernel<float, float, false>;
}

static size_t pass_smem(const PassParams& p) {
  const int npg = DP_THREADS / std::max(1, p.dh / 4);
  return static_cast<size_t>(DP_WARPS) * DP_STAGES * DP_STAGE_BYTES +
         static_cast<size_t>(std::max(p.d, p.ff)) * 4 + (static_cast<size_t>(p.dh) + p.span_cap + npg * p.dh) * 4;
}

cudaError_t decode_pass_prepare(int device) {
  int optin = 0;
  cudaError_t err = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (err != cudaSuccess) return err;
  for (Dt w : {Dt::F32, Dt::BF16})
    for (Dt k : {Dt::F32, Dt::BF16})
      for (bool l : {false, true}) {
        PassFn f = pick_pass(w, k, l);
        cudaFuncAttributes fa;
        err = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
        if (err != cudaSuccess) return err;
        err = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   optin - static_cast<int>(fa.sharedSizeBytes));
        if (err != cudaSuccess) return err;
      }
  return cudaSuccess;
}

cudaError_t launch_decode_pass(Dt wdt, Dt kvdt, bool arch_llama, const PassParams& p, cudaStream_t s, bool pdl) {
  if (p.d % 8 || p.ff % 8 || p.dh % 4 || p.dh > 128) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t smem = pass_smem(p);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms(dev));  // one persistent CTA per SM (smem forces 1/SM)
  cfg.blockDim = dim3(DP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, pick_pass(wdt, kvdt, arch_llama), p);
}

}  // namespace grt
