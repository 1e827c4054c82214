// decode_pass.cu -- the static pass of one decode step as ONE persistent kernel.
//
// Reference: Model::build_plan (model.cpp:118-143) -- 14 kernels per layer, each
// a separate closure.  Batch-1 decode is bandwidth bound (13.2 GB of weights per
// token for LLaMA-2 7B), so on a B200 what limits it is not arithmetic but the
// bubbles between ~160 dependent kernels.  Here the whole pass is one launch,
// warp-specialised:
//
//   * grid = one CTA per SM.  Warp 8 is the PRODUCER: one lane walks every GEMV
//     phase of the pass (QKV, Wo, gate/up, down per layer, then the LM head),
//     takes its CTA's row pairs (a static share plus dynamically claimed tail
//     pairs for load balance) and streams them into a 16-slot x 8 KB ring with
//     cp.async.bulk (TMA engine) under an evict-first L2 policy.  Weights never
//     depend on activations, so it runs ahead ACROSS phase and layer boundaries,
//     throttled only by free slots -- HBM stays busy while the CTA waits.
//   * warps 0-7 are CONSUMERS: each stage is split across the 8 warps (1 KB
//     each); per row pair the warp partials are reduced in a fixed order, so
//     results are deterministic.  Between phases the consumers wait on
//     device-side dependency counters (release: __threadfence + atomicAdd;
//     acquire: spin + __threadfence); the last CTA out resets every counter.
//   * phases per layer: QKV(+norm, RoPE, KV write) | attention | Wo(+residual) |
//     gate/up(+norm, SwiGLU) | down(+residual); activations written by other
//     CTAs in this launch are read with ld.global.cg (L2), never a stale L1 line;
//   * watchdogs turn a missing arrival into DEVERR_TIMEOUT instead of a hang.
#include <cuda_bf16.h>

#include <algorithm>
#include <climits>
#include <type_traits>

#define GRT_CONSUMER_THREADS 384  // 12 consumer warps (3 per SM sub-partition)
#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int DP_CWARPS = CONSUMER_THREADS / 32;   // consumer warps
constexpr int DP_THREADS = (DP_CWARPS + 1) * 32;   // + producer warp
#ifndef GRT_DP_STAGES
#define GRT_DP_STAGES 20
#endif
#ifndef GRT_DP_STAGE_KB
#define GRT_DP_STAGE_KB 8
#endif
constexpr int DP_STAGES = GRT_DP_STAGES;
constexpr uint32_t DP_STAGE_BYTES = GRT_DP_STAGE_KB * 1024;  // 16 KB = one LLaMA-7B row pair (k=4096)
constexpr int DP_PARTS = 64;  // per-stage partial-sum slots (> DP_STAGES + max stages per pair)
constexpr unsigned long long DP_WATCHDOG_NS = 2000000000ull;  // 2 s
constexpr int DP_END = INT_MAX;

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

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// wait with a watchdog; returns false on expiry
__device__ __forceinline__ bool mbar_wait_wd(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return true;
  const unsigned long long t0 = globaltimer();
  while (!mbar_try_wait(bar, parity))
    if (globaltimer() - t0 > DP_WATCHDOG_NS) return false;
  return true;
}

struct StageMeta {
  int ph;    // phase of the stage; DP_END after the last one
  int pair;  // row pair
  int off;   // byte offset in the pair's contiguous 2-row stream
  int len;   // bytes in this stage
};

// Static share: 4/5 of the pairs in contiguous blocks per CTA; the rest are
// claimed one pair at a time by whichever CTA is ready first.
__device__ __forceinline__ int static_share(int n_pairs, int G) { return (n_pairs * 4 / 5) / G; }

// ---- producer (warp 8, lane 0) ---------------------------------------------------

template <typename WT, bool LLAMA>
__device__ void producer(const PassParams& p, uint8_t* ring, uint64_t* full, uint64_t* empty, StageMeta* meta) {
  const uint64_t pol = l2_evict_first_policy();
  int* claims = p.sync + p.n_layers * p.sync_stride;
  const int G = gridDim.x;
  uint32_t t = 0;
  auto next_slot = [&](int& slot) -> bool {
    slot = t % DP_STAGES;
    // the first pass over the ring finds every slot free
    return mbar_wait_wd(&empty[slot], ((t / DP_STAGES) & 1) ^ 1);
  };
  auto stream_pair = [&](int ph, const GemvPhase& g, int pair) -> bool {
    const int rows = (2 * pair + 1 < g.n_rows) ? 2 : 1;
    const int bytes = rows * g.k * static_cast<int>(sizeof(WT));
    const uint8_t* src = reinterpret_cast<const uint8_t*>(g.w) +
                         static_cast<int64_t>(2 * pair) * g.k * static_cast<int64_t>(sizeof(WT));
    for (int off = 0; off < bytes; off += DP_STAGE_BYTES) {
      int slot;
      if (!next_slot(slot)) return false;
      const int len = min(static_cast<int>(DP_STAGE_BYTES), bytes - off);
      meta[slot] = StageMeta{ph, pair, off, len};
      mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(len));
      bulk_g2s(ring + slot * DP_STAGE_BYTES, src + off, static_cast<uint32_t>(len), &full[slot], pol);
      ++t;
    }
    return true;
  };
  const int n_ph = 4 * p.n_layers + 1;
  for (int ph = 0; ph < n_ph; ++ph) {
    const GemvPhase g = phase_desc<LLAMA>(p, ph);
    const int n_pairs = (g.n_rows + 1) >> 1;
    const int s0 = static_share(n_pairs, G);
    // The first tail claim is put in flight before the static share is
    // streamed, and every later one before the pair it follows: the atomic's
    // round trip overlaps the copies instead of stalling the producer.
    int nxt = atomicAdd(claims + ph, 1);
    for (int pr = blockIdx.x * s0; pr < (blockIdx.x + 1) * s0; ++pr)
      if (!stream_pair(ph, g, pr)) return;
    for (;;) {
      const int pr = G * s0 + nxt;
      if (pr >= n_pairs) break;
      nxt = atomicAdd(claims + ph, 1);
      if (!stream_pair(ph, g, pr)) return;
    }
  }
  // one end marker per consumer warp (warp w owns stages w, w+8, ...)
  for (int w = 0; w < DP_CWARPS; ++w) {
    int slot;
    if (!next_slot(slot)) return;
    meta[slot] = StageMeta{DP_END, 0, 0, 0};
    mbar_arrive(&full[slot]);
    ++t;
  }
}

// ---- consumer-side helpers ------------------------------------------------------

// Dot of one whole stage (one warp): bytes [0, len) of the stage are elements
// stage_e0 + ... of the concatenation row_a | row_b (length k each).
// Dot of bytes [b_lo, b_hi) of a stage that all belong to ONE row, whose first
// byte b_lo corresponds to column col0; 16-byte groups, lane-strided.
template <typename WT>
__device__ __forceinline__ float dot_run(const uint8_t* st, int b_lo, int b_hi, int col0, int k, const float* xs) {
  const int lane = threadIdx.x & 31;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if constexpr (sizeof(WT) == 2) {
    // group q covers columns col0 + 8q .. +7 -> float4 #(col0/8 + q) of each x plane
    const uint4* w = reinterpret_cast<const uint4*>(st + b_lo);
    const float4* xa = reinterpret_cast<const float4*>(xs) + (col0 >> 3);
    const float4* xb = reinterpret_cast<const float4*>(xs + (k >> 1)) + (col0 >> 3);
    const int groups = (b_hi - b_lo) >> 4;
#pragma unroll 4
    for (int q = lane; q < groups; q += 32) {
      const uint4 u = w[q];
      const float4 x0 = xa[q];
      const float4 x1 = xb[q];
      a0 = fmaf(bf16lo(u.x), x0.x, a0);
      a1 = fmaf(bf16hi(u.x), x0.y, a1);
      a2 = fmaf(bf16lo(u.y), x0.z, a2);
      a3 = fmaf(bf16hi(u.y), x0.w, a3);
      a0 = fmaf(bf16lo(u.z), x1.x, a0);
      a1 = fmaf(bf16hi(u.z), x1.y, a1);
      a2 = fmaf(bf16lo(u.w), x1.z, a2);
      a3 = fmaf(bf16hi(u.w), x1.w, a3);
    }
  } else {
    const float4* w = reinterpret_cast<const float4*>(st + b_lo);
    const float4* xv = reinterpret_cast<const float4*>(xs) + (col0 >> 2);
    const int groups = (b_hi - b_lo) >> 4;
#pragma unroll 4
    for (int q = lane; q < groups; q += 32) {
      const float4 u = w[q];
      const float4 x = xv[q];
      a0 = fmaf(u.x, x.x, a0);
      a1 = fmaf(u.y, x.y, a1);
      a2 = fmaf(u.z, x.z, a2);
      a3 = fmaf(u.w, x.w, a3);
    }
  }
  return (a0 + a1) + (a2 + a3);
}

// Dot of one whole stage (one warp): bytes [0, len) of the stage are elements
// stage_e0 + ... of the concatenation row_a | row_b (length k each).  The row
// boundary is crossed at most once, so the stage splits into <= 2 linear runs.
template <typename WT>
__device__ __forceinline__ void dot_stage(const uint8_t* st, int stage_e0, int len, int k, const float* xs,
                                          float& acc_a, float& acc_b) {
  const int sz = static_cast<int>(sizeof(WT));
  const int e_end = stage_e0 + len / sz;
  if (stage_e0 < k) {
    const int hi = min(e_end, k);
    acc_a += dot_run<WT>(st, 0, (hi - stage_e0) * sz, stage_e0, k, xs);
  }
  if (e_end > k) {
    const int lo = max(stage_e0, k);
    acc_b += dot_run<WT>(st, (lo - stage_e0) * sz, len, lo - k, k, xs);
  }
}

__device__ __forceinline__ void phase_arrive(int* ctr) {
  consumer_sync();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
  }
}

// returns false on watchdog expiry (uniform across the consumer warps)
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
  consumer_sync();
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
  consumer_sync();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  consumer_sync();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < DP_CWARPS ? red[threadIdx.x] : -INFINITY;
    t = warp_max(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  consumer_sync();
  return red[0];
}

template <typename KT>
__device__ void attention_item(const PassParams& p, const PassLayer& L, int layer, int head, int split, int len,
                               float* sm, float* red, int* s_last) {
  constexpr int NT = CONSUMER_THREADS;
  const int dh = p.dh, ns = p.nsplit;
  const int gs = dh >> 2;   // lanes per position
  const int npg = NT / gs;  // position groups
  const int span = (len + ns - 1) / ns;
  const int j0 = split * span;
  const int n = max(0, min(len, j0 + span) - j0);
  // Latency-oriented: q comes straight from L2, and each thread issues the K and
  // V loads of a batch of positions together before using any of them; an
  // online softmax per position group avoids a scores round trip through smem.
  float* op = sm;                 // [npg][dh] group partial outputs
  float* gmax = op + npg * dh;    // [npg]
  float* gsum = gmax + npg;       // [npg]
  const KT* K = reinterpret_cast<const KT*>(L.k) + static_cast<int64_t>(head) * p.max_seq * dh;
  const KT* V = reinterpret_cast<const KT*>(L.v) + static_cast<int64_t>(head) * p.max_seq * dh;
  const int grp = threadIdx.x / gs, gl = threadIdx.x - grp * gs;
  const float4 q4 = __ldcg(reinterpret_cast<const float4*>(p.q + head * dh) + gl);
  constexpr int BATCH = 4;
  float mt = -INFINITY, lt = 0.0f;
  float4 ot = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int jb = 0; jb < n; jb += BATCH * npg) {  // trip count uniform across the CTA
    float4 kk[BATCH], vv[BATCH];
#pragma unroll
    for (int i = 0; i < BATCH; ++i) {
      const int jj = jb + grp + i * npg;
      if (jj < n) {
        kk[i] = kv_load4<KT>(K + static_cast<int64_t>(j0 + jj) * dh + 4 * gl);
        vv[i] = kv_load4<KT>(V + static_cast<int64_t>(j0 + jj) * dh + 4 * gl);
      } else {
        kk[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        vv[i] = kk[i];
      }
    }
    float s[BATCH];
    float bmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < BATCH; ++i) {
      float v = q4.x * kk[i].x + q4.y * kk[i].y + q4.z * kk[i].z + q4.w * kk[i].w;
      for (int o = gs >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      s[i] = (jb + grp + i * npg < n) ? v * p.scale : -INFINITY;
      bmax = fmaxf(bmax, s[i]);
    }
    if (bmax > -INFINITY) {
      const float mnew = fmaxf(mt, bmax);
      const float c = mt > -INFINITY ? expf(mt - mnew) : 0.0f;
      lt *= c;
      ot.x *= c;
      ot.y *= c;
      ot.z *= c;
      ot.w *= c;
#pragma unroll
      for (int i = 0; i < BATCH; ++i) {
        const float e = s[i] > -INFINITY ? expf(s[i] - mnew) : 0.0f;
        lt += e;
        ot.x = fmaf(e, vv[i].x, ot.x);
        ot.y = fmaf(e, vv[i].y, ot.y);
        ot.z = fmaf(e, vv[i].z, ot.z);
        ot.w = fmaf(e, vv[i].w, ot.w);
      }
      mt = mnew;
    }
  }
  if (gl == 0) {
    gmax[grp] = mt;
    gsum[grp] = lt;
  }
  reinterpret_cast<float4*>(op + grp * dh)[gl] = ot;
  consumer_sync();
  float m = -INFINITY;
  for (int g = 0; g < npg; ++g) m = fmaxf(m, gmax[g]);
  float l = 0.0f;
  for (int g = 0; g < npg; ++g)
    if (gmax[g] > -INFINITY) l += gsum[g] * expf(gmax[g] - m);
  {  // rescale this thread's own group partial to the CTA max
    const float c = mt > -INFINITY ? expf(mt - m) : 0.0f;
    float4* mine4 = reinterpret_cast<float4*>(op + grp * dh) + gl;
    float4 v = *mine4;
    *mine4 = make_float4(v.x * c, v.y * c, v.z * c, v.w * c);
  }
  consumer_sync();
  int* head_ctr = p.sync + layer * p.sync_stride + SY_HEADS + head;
  int* attn_ctr = p.sync + layer * p.sync_stride + SY_ATTN;
  if (ns == 1) {
    const float inv = 1.0f / l;
    for (int d = threadIdx.x; d < dh; d += NT) {
      float o = 0.0f;
      for (int g = 0; g < npg; ++g) o += op[g * dh + d];
      p.attn[head * dh + d] = o * inv;
    }
    phase_arrive(attn_ctr);
    consumer_sync();
    return;
  }
  const int stride = dh + 2;
  float* mine = p.part + (static_cast<int64_t>(head) * ns + split) * stride;
  for (int d = threadIdx.x; d < dh; d += NT) {
    float o = 0.0f;
    for (int g = 0; g < npg; ++g) o += op[g * dh + d];
    mine[d] = o;
  }
  if (threadIdx.x == 0) {
    mine[dh] = n > 0 ? m : -INFINITY;
    mine[dh + 1] = n > 0 ? l : 0.0f;
  }
  consumer_sync();
  if (threadIdx.x == 0) {
    __threadfence();
    *s_last = (atomicAdd(head_ctr, 1) == ns - 1);
    if (*s_last) __threadfence();
  }
  consumer_sync();
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
  for (int d = threadIdx.x; d < dh; d += NT) {
    float o = 0.0f;
    for (int s = 0; s < ns; ++s) {
      const float ls = __ldcg(base + s * stride + dh + 1);
      if (ls > 0.0f) o += __ldcg(base + s * stride + d) * expf(__ldcg(base + s * stride + dh) - M);
    }
    p.attn[head * dh + d] = o * invL;
  }
  phase_arrive(attn_ctr);
  consumer_sync();
}

// ---- the kernel -------------------------------------------------------------------

template <typename WT, typename KT, bool LLAMA>
__global__ void __launch_bounds__(DP_THREADS, 1) decode_pass_kernel(const PassParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[DP_STAGES], empty[DP_STAGES];
  __shared__ StageMeta meta[DP_STAGES];
  __shared__ float red[32];
  __shared__ float2 part_sum[DP_PARTS];
  __shared__ int part_seq[DP_PARTS];
  __shared__ int s_ok, s_last;
  __shared__ int s_ready, s_waited;  // trace only: stages already landed when a consumer arrived vs not
  constexpr int NORM = LLAMA ? NORM_RMS : NORM_LN;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  uint8_t* ring = smem;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(DP_STAGES) * DP_STAGE_BYTES);
  float* asm_ = xs + max(p.d, p.ff);  // attention scratch

  if (threadIdx.x == 0) {
    for (int s = 0; s < DP_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < DP_PARTS; ++s) part_seq[s] = -1;
    s_ready = 0;
    s_waited = 0;
    mbar_fence_init();
  }
  __syncthreads();  // all 9 warps: barriers initialised

  if (warp == DP_CWARPS) {  // ---------------- producer warp
    if (lane == 0) producer<WT, LLAMA>(p, ring, full, empty, meta);
    return;
  }

  // ---------------- consumer warps 0..7
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

  // Warp w consumes the CTA's stages w, w+8, w+16, ... (whole 8 KB stages).  A
  // row pair spans 1..6 consecutive stages, so its partial sums come from
  // several warps: each warp posts its stage partial in part_sum[t % 64] with
  // the stage number in part_seq; the warp holding the pair's LAST stage waits
  // for the others, adds them in stage order (deterministic) and runs the
  // epilogue.  It releases its own ring slot only afterwards, which bounds how
  // far the producer can run ahead and keeps the 64 partial slots from wrapping.
  int t = warp;  // next stage of this warp
  bool alive = true;
  auto run_phase = [&](int ph, auto epi_tag) {
    constexpr int EPI = decltype(epi_tag)::value;
    const GemvPhase g = phase_desc<LLAMA>(p, ph);
    const int sz = static_cast<int>(sizeof(WT));
    for (;;) {
      const int slot = t % DP_STAGES;
      if (p.trace && lane == 0) atomicAdd(mbar_try_wait(&full[slot], (t / DP_STAGES) & 1) ? &s_ready : &s_waited, 1);
      if (!mbar_wait_wd(&full[slot], (t / DP_STAGES) & 1)) {
        if (threadIdx.x == 0) atomicOr(p.err, DEVERR_TIMEOUT);
        alive = false;
        return;
      }
      const StageMeta m = meta[slot];
      if (m.ph != ph) return;  // stage of a later phase (or the end marker): leave it
      float acc_a = 0.0f, acc_b = 0.0f;
      dot_stage<WT>(ring + slot * DP_STAGE_BYTES, m.off / sz, m.len, g.k, xs, acc_a, acc_b);
      const float va = warp_sum(acc_a);
      const float vb = warp_sum(acc_b);
      const int rows = (2 * m.pair + 1 < g.n_rows) ? 2 : 1;
      const int pair_bytes = rows * g.k * sz;
      if (m.off + m.len < pair_bytes) {  // not the pair's last stage: post the partial
        if (lane == 0) {
          part_sum[t % DP_PARTS] = make_float2(va, vb);
          __threadfence_block();
          reinterpret_cast<volatile int*>(part_seq)[t % DP_PARTS] = t;
          mbar_arrive(&empty[slot]);
        }
      } else {
        if (lane == 0) {
          const int n_prev = m.off / static_cast<int>(DP_STAGE_BYTES);  // earlier stages of this pair
          float sa = 0.0f, sb = 0.0f;
          for (int j = n_prev; j >= 1; --j) {
            const int ts = t - j;
            volatile int* seq = reinterpret_cast<volatile int*>(part_seq);
            while (seq[ts % DP_PARTS] != ts) {
            }
            __threadfence_block();
            const float2 ps = part_sum[ts % DP_PARTS];
            sa += ps.x;
            sb += ps.y;
          }
          epilogue<EPI>(ea, m.pair, sa + va, sb + vb, rows == 2);
          mbar_arrive(&empty[slot]);
        }
      }
      __syncwarp();
      t += DP_CWARPS;
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
    // Invalid live length for this bucket: flag it and drain the stream so the
    // producer finishes and no bulk copy is outstanding at exit.
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.err, DEVERR_WRONG_LENGTH);
    for (;;) {
      const int slot = t % DP_STAGES;
      if (!mbar_wait_wd(&full[slot], (t / DP_STAGES) & 1)) return;
      if (meta[slot].ph == DP_END) return;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      t += DP_CWARPS;
    }
  }

  for (int l = 0; l < p.n_layers && alive; ++l) {
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
  if (!alive) return;
  // ---- ln_f + head
  if (!phase_wait(p.sync + (p.n_layers - 1) * p.sync_stride + SY_DOWN, G, p.err, &s_ok)) return;
  stamp(p.n_layers * PASS_TRACE_PER_LAYER + 0);
  load_x<WT, NORM, true>(p.x, p.lnf_g, p.lnf_b, p.eps, p.d, xs, red);
  ea.out = p.logits;
  run_phase(4 * p.n_layers, StoreTag{});
  stamp(p.n_layers * PASS_TRACE_PER_LAYER + 1);
  consumer_sync();
  if (trace && threadIdx.x == 0) {
    trace[p.n_layers * PASS_TRACE_PER_LAYER + 3] = static_cast<unsigned long long>(s_ready);
    trace[p.n_layers * PASS_TRACE_PER_LAYER + 4] = static_cast<unsigned long long>(s_waited);
  }

  // Self-reset: the last CTA out zeroes every counter (phase, head, claim) for
  // the next pass; all other CTAs have passed their last wait and claim.
  consumer_sync();
  const int total = sync_total(p.n_layers, p.sync_stride);
  int* exit_ctr = p.sync + total - 1;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(exit_ctr, 1) == G - 1;
  }
  consumer_sync();
  if (s_last) {
    for (int i = threadIdx.x; i < total; i += CONSUMER_THREADS) p.sync[i] = 0;
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
  const int npg = CONSUMER_THREADS / std::max(1, p.dh / 4);
  return static_cast<size_t>(DP_STAGES) * DP_STAGE_BYTES + static_cast<size_t>(std::max(p.d, p.ff)) * 4 +
         (static_cast<size_t>(npg) * p.dh + 2 * npg + 32) * 4;
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
