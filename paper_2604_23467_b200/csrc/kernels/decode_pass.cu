// decode_pass.cu -- the static pass of one decode step as ONE persistent kernel.
//
// Reference: Model::build_plan (model.cpp:118-143) -- 14 kernels per layer, each
// a separate closure.  Batch-1 decode is bandwidth bound (13.2 GB of weights per
// token for LLaMA-2 7B), so on a B200 what limits it is not arithmetic but the
// bubbles between ~160 dependent kernels.  Here the whole pass is one launch:
//
//   * grid = one CTA per SM, 8 warps.  Every warp owns a ring of DP_STAGES
//     8 KB shared-memory slots; its lane 0 CLAIMS the next row pair of the
//     current GEMV phase from a global counter (dynamic load balance: fast SMs
//     take more rows) and streams it with cp.async.bulk (TMA engine) in 8 KB
//     stages.  Claims run ahead of consumption ACROSS phase and layer
//     boundaries -- weights never depend on activations -- so HBM stays busy
//     while the CTA waits for a dependency;
//   * phases per layer: QKV(+norm, RoPE, KV write) | attention | Wo(+residual) |
//     gate/up(+norm, SwiGLU) | down(+residual); boundaries are device-side
//     dependency counters (release: __threadfence + atomicAdd; acquire: spin +
//     __threadfence); the last CTA out resets all counters for the next pass;
//   * activations produced by other CTAs in the same launch are read with
//     ld.global.cg (L2), never through a possibly stale L1 line;
//   * a watchdog turns a missing arrival into DEVERR_TIMEOUT instead of a hang.
#include <cuda_bf16.h>

#include <algorithm>
#include <climits>
#include <type_traits>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int DP_WARPS = 8;
constexpr int DP_THREADS = DP_WARPS * 32;
constexpr int DP_STAGES = 2;
constexpr uint32_t DP_STAGE_BYTES = 8192;
constexpr unsigned long long DP_WATCHDOG_NS = 2000000000ull;  // 2 s

enum SyncSlot { SY_QKV = 0, SY_ATTN = 1, SY_WO = 2, SY_UP = 3, SY_DOWN = 4, SY_HEADS = 8 };

int decode_pass_sync_stride(int n_heads) { return ((SY_HEADS + n_heads + 31) / 32) * 32; }
// sync array: [n_layers][stride] phase counters | [4L+1] row-pair claim counters | exit counter
static __host__ __device__ int sync_total(int n_layers, int stride) { return n_layers * stride + 4 * n_layers + 2; }
int decode_pass_sync_ints(int n_layers, int n_heads) { return sync_total(n_layers, decode_pass_sync_stride(n_heads)); }

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

// Per-stage metadata (written by the producer lane, read by the warp).
struct StageMeta {
  int ph;    // phase of the stage; -1 = slot empty
  int pair;  // row pair
  int off;   // byte offset in the pair's contiguous 2-row stream
  int len;   // bytes in this stage
};

// Per-warp producer: claims row pairs phase by phase and issues 8 KB stages.
// All lanes keep identical state (claims are broadcast from lane 0).
template <typename WT, bool LLAMA>
struct Producer {
  int ph = 0;        // phase being claimed; > 4L = done
  int pair = -1;     // claimed pair (-1: claim next)
  int off = 0;       // next byte offset in the pair stream
  int pair_bytes = 0;
  GemvPhase g{};
  int n_pairs = 0;
  int t = 0;         // stages issued
  bool done = false;

  __device__ void set_phase(const PassParams& p, int new_ph) {
    ph = new_ph;
    if (ph > 4 * p.n_layers) {
      done = true;
      return;
    }
    g = phase_desc<LLAMA>(p, ph);
    n_pairs = (g.n_rows + 1) >> 1;
  }

  // Issues the next stage into slot t % DP_STAGES; returns false when exhausted.
  __device__ bool issue(const PassParams& p, int* claims, uint8_t* ring, uint64_t* bars, StageMeta* meta,
                        uint64_t pol) {
    const int lane = threadIdx.x & 31;
    while (!done && pair < 0) {
      int c = 0;
      if (lane == 0) c = atomicAdd(claims + ph, 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c < n_pairs) {
        pair = c;
        off = 0;
        const int rows = (2 * c + 1 < g.n_rows) ? 2 : 1;
        pair_bytes = rows * g.k * static_cast<int>(sizeof(WT));
      } else {
        set_phase(p, ph + 1);
      }
    }
    if (done) return false;
    const int slot = t % DP_STAGES;
    const int len = min(static_cast<int>(DP_STAGE_BYTES), pair_bytes - off);
    if (lane == 0) {
      meta[slot] = StageMeta{ph, pair, off, len};
      uint64_t* bar = &bars[slot];
      mbar_arrive_expect_tx(bar, static_cast<uint32_t>(len));
      const uint8_t* src = reinterpret_cast<const uint8_t*>(g.w) +
                           static_cast<int64_t>(2 * pair) * g.k * static_cast<int64_t>(sizeof(WT)) + off;
      bulk_g2s(ring + slot * DP_STAGE_BYTES, src, static_cast<uint32_t>(len), bar, pol);
    }
    off += len;
    if (off >= pair_bytes) pair = -1;
    ++t;
    return true;
  }
};

// Dot of one stage of a pair stream: elements [e0, e0 + len/sizeof) of the
// concatenation row_a | row_b (each of length k).
template <typename WT>
__device__ __forceinline__ void dot_stage(const uint8_t* st, int e0, int len, int k, const float* xs, float& acc_a,
                                          float& acc_b) {
  const int lane = threadIdx.x & 31;
  const int groups = len >> 4;  // 16-byte groups
  float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
  if constexpr (sizeof(WT) == 2) {
    const uint4* w = reinterpret_cast<const uint4*>(st);
    const float4* xa = reinterpret_cast<const float4*>(xs);
    const float4* xb = reinterpret_cast<const float4*>(xs + (k >> 1));
#pragma unroll 4
    for (int q = lane; q < groups; q += 32) {
      const int e = e0 + q * 8;
      const bool isb = e >= k;
      const int gi = (isb ? e - k : e) >> 3;
      const uint4 u = w[q];
      const float4 x0 = xa[gi];
      const float4 x1 = xb[gi];
      float s0 = bf16lo(u.x) * x0.x;
      float s1 = bf16hi(u.x) * x0.y;
      s0 = fmaf(bf16lo(u.y), x0.z, s0);
      s1 = fmaf(bf16hi(u.y), x0.w, s1);
      s0 = fmaf(bf16lo(u.z), x1.x, s0);
      s1 = fmaf(bf16hi(u.z), x1.y, s1);
      s0 = fmaf(bf16lo(u.w), x1.z, s0);
      s1 = fmaf(bf16hi(u.w), x1.w, s1);
      if (isb) {
        b0 += s0;
        b1 += s1;
      } else {
        a0 += s0;
        a1 += s1;
      }
    }
  } else {
    const float4* w = reinterpret_cast<const float4*>(st);
    const float4* xv = reinterpret_cast<const float4*>(xs);
#pragma unroll 4
    for (int q = lane; q < groups; q += 32) {
      const int e = e0 + q * 4;
      const bool isb = e >= k;
      const int gi = (isb ? e - k : e) >> 2;
      const float4 u = w[q];
      const float4 x = xv[gi];
      float s0 = u.x * x.x;
      float s1 = u.y * x.y;
      s0 = fmaf(u.z, x.z, s0);
      s1 = fmaf(u.w, x.w, s1);
      if (isb) {
        b0 += s0;
        b1 += s1;
      } else {
        a0 += s0;
        a1 += s1;
      }
    }
  }
  acc_a += a0 + a1;
  acc_b += b0 + b1;
}

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

__device__ __forceinline__ float block_max_all(float v, float* red) {
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
  const int gs = dh >> 2;           // lanes per position
  const int npg = DP_THREADS / gs;  // position groups
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
  m = block_max_all(m, red);
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
  __shared__ StageMeta metas[DP_WARPS][DP_STAGES];
  __shared__ float red[32];
  __shared__ int s_ok, s_last;
  constexpr int NORM = LLAMA ? NORM_RMS : NORM_LN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  uint8_t* ring = smem + static_cast<size_t>(warp) * DP_STAGES * DP_STAGE_BYTES;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(DP_WARPS) * DP_STAGES * DP_STAGE_BYTES);
  float* asm_ = xs + max(p.d, p.ff);  // attention scratch
  uint64_t* mybar = bars[warp];
  StageMeta* meta = metas[warp];
  const uint64_t pol = l2_evict_first_policy();
  int* claims = p.sync + p.n_layers * p.sync_stride;

  Producer<WT, LLAMA> prod;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < DP_STAGES; ++s) {
      mbar_init(&mybar[s], 1);
      meta[s].ph = -1;
    }
    mbar_fence_init();
  }
  __syncwarp();
  prod.set_phase(p, 0);
  // Weights do not depend on the previous kernel: fill the ring before waiting.
  for (int s = 0; s < DP_STAGES; ++s)
    if (!prod.issue(p, claims, ring, mybar, meta, pol)) break;
  __syncwarp();
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

  int t = 0;  // stages consumed by this warp
  // Consume every stage this warp claimed in GEMV phase `ph`.
  auto run_phase = [&](int ph, auto epi_tag) {
    constexpr int EPI = decltype(epi_tag)::value;
    const GemvPhase g = phase_desc<LLAMA>(p, ph);
    float acc_a = 0.0f, acc_b = 0.0f;
    for (;;) {
      const int slot = t % DP_STAGES;
      const StageMeta m = meta[slot];
      if (m.ph != ph) break;  // ring moved on to a later phase (or ran dry)
      mbar_wait(&mybar[slot], static_cast<uint32_t>((t / DP_STAGES) & 1));
      dot_stage<WT>(ring + slot * DP_STAGE_BYTES, m.off / static_cast<int>(sizeof(WT)), m.len, g.k, xs, acc_a,
                    acc_b);
      __syncwarp();
      if (lane == 0) {
        meta[slot].ph = -1;
        fence_proxy_async_smem();
      }
      __syncwarp();
      prod.issue(p, claims, ring, mybar, meta, pol);
      __syncwarp();
      ++t;
      const int rows = (2 * m.pair + 1 < g.n_rows) ? 2 : 1;
      if (m.off + m.len >= rows * g.k * static_cast<int>(sizeof(WT))) {
        const float va = warp_sum(acc_a);
        const float vb = warp_sum(acc_b);
        if (lane == 0) epilogue<EPI>(ea, m.pair, va, vb, rows == 2);
        acc_a = 0.0f;
        acc_b = 0.0f;
      }
    }
  };
  using QkvTag = std::integral_constant<int, LLAMA ? EPI_QKV_ROPE : EPI_QKV>;
  using ResidTag = std::integral_constant<int, EPI_RESID>;
  using UpTag = std::integral_constant<int, LLAMA ? EPI_SWIGLU : EPI_RELU>;
  using StoreTag = std::integral_constant<int, EPI_STORE>;

  unsigned long long* trace = p.trace ? p.trace + static_cast<int64_t>(blockIdx.x) * p.trace_stride : nullptr;
  auto stamp = [&](int ev) {
    if (trace && threadIdx.x == 0) trace[ev] = globaltimer();
  };

  if (len < 1 || len > p.max_seq || (len + p.nsplit - 1) / p.nsplit > p.span_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.err, DEVERR_WRONG_LENGTH);
    // drain the prefetched stages so no bulk copy is outstanding at exit
    for (int s = 0; s < min(DP_STAGES, prod.t); ++s) mbar_wait(&mybar[s], 0);
    return;
  }

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

  // Self-reset: the last CTA out zeroes every counter (phase, head, claim) for
  // the next pass; all other CTAs have passed their last wait and claim.
  __syncthreads();
  const int total = sync_total(p.n_layers, p.sync_stride);
  int* exit_ctr = p.sync + total - 1;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(exit_ctr, 1) == G - 1;
  }
  __syncthreads();
  if (s_last) {
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
