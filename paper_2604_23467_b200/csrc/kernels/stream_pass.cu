// stream_pass.cu -- the static pass of one decode step as ONE persistent launch
// whose weight stream never stops (pass_impl 2, LLaMA arch, bf16 weights + KV).
//
// Reference: Model::build_plan (model.cpp:118-143) -- per layer ln1, q, k, v,
// kv_write, attention, wo, +res, ln2, w1, relu, w2, +res; then ln_f, head.
// Batch-1 decode reads 13.2 GB of weights per token and does ~1 flop per byte,
// so the step is an HBM stream; what costs time is every place the stream
// pauses.  With one kernel per op each boundary drains the old grid, launches
// the new one, refills its rings and reloads its activation (~3-5 us of HBM
// idle per boundary, 4 per layer).  Here:
//
//   * grid = one CTA per SM (co-residency checked at launch), 8 warps, each warp
//     with a private ring of `stages` shared-memory slots fed by cp.async.bulk
//     (TMA engine) under an evict-first L2 policy -- the gemv.cu / gemv_pair.cu
//     building blocks;
//   * every warp owns a STATIC task list over the whole pass: per layer its
//     (row pair, k chunk) tasks of QKV, Wo, gate/up and down, then the LM head.
//     Weights never depend on activations, so a slot freed by task i is
//     immediately refilled with task i+stages -- whichever phase or layer that
//     is.  Across a dependency wait the ring keeps streaming the NEXT phase's
//     rows; only the activation row (16-44 KB, L2) is loaded after the wait;
//   * phases are separated by grid barriers (monotonic arrival counter,
//     release/acquire at gpu scope, watchdog -> DEVERR_TIMEOUT); activations
//     written by other CTAs in this launch are read through L2 (ld.global.cg);
//   * attention is a phase of its own: CTA b < h*ns computes the split-softmax
//     partial of head b/ns (pair_attn.cuh), and after a barrier every CTA merges
//     all heads into its Wo activation row;
//   * the arithmetic per output is that of the per-op kernels (pair rows, chunk
//     partials summed in chunk order, deferred RMSNorm scale), so results are
//     identical to pass_impl 1 bit for bit.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"
#include "pair_attn.cuh"

namespace grt {

constexpr int SP_WARPS = GP_WARPS;  // 8 consumer warps (CONSUMER_THREADS = 256)
constexpr int SP_MAX_STAGES = 8;
constexpr unsigned long long SP_WATCHDOG_NS = 2000000000ull;  // 2 s
// The down projection (k = d_ff) runs as two phases over the two halves of k,
// so its activation row needs only half the shared memory (a third ring stage
// for every phase); the partials of both halves are summed in chunk order.
enum SpKind : int { SK_QKV = 0, SK_WO = 1, SK_UP = 2, SK_DNA = 3, SK_DNB = 4, SK_HEAD = 5, SK_N = 6 };

struct SpGeom {
  int k, n_rows, ch, nch, pair_begin, pair_end, n_tasks;
  int ld, kofs;  // row stride of the weight matrix; first k element of this phase
};

__device__ __forceinline__ SpGeom sp_geom(int k, int n_rows, int ch, int nch, int warp, int ld = 0, int kofs = 0) {
  SpGeom g;
  g.ld = ld > 0 ? ld : k;
  g.kofs = kofs;
  g.k = k;
  g.n_rows = n_rows;
  g.ch = ch;
  g.nch = nch;
  const int n_pairs = (n_rows + 1) >> 1;
  g.pair_begin = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
  g.pair_end = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
  const int Tc = (g.pair_end - g.pair_begin) * nch;
  g.n_tasks = Tc > warp ? (Tc - warp + SP_WARPS - 1) / SP_WARPS : 0;
  return g;
}

// xs = x (* gamma); returns this thread's sum of squares of x (deferred RMSNorm:
// 1/rms multiplies the finished dot products).  x was written by other CTAs of
// this launch: L2 loads, every load of a thread issued before any is used.
__device__ __forceinline__ float sp_load_x(const float* x, const float* gamma, int k, float* xs) {
  const int n4 = k >> 2;
  float4 v[LOADX_MAXV], gv[LOADX_MAXV];
#pragma unroll
  for (int i = 0; i < LOADX_MAXV; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    v[i] = j4 < n4 ? __ldcg(reinterpret_cast<const float4*>(x) + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
    gv[i] = (gamma && j4 < n4) ? __ldg(reinterpret_cast<const float4*>(gamma) + j4) : make_float4(1.f, 1.f, 1.f, 1.f);
  }
  float ss = 0.0f;
#pragma unroll
  for (int i = 0; i < LOADX_MAXV; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    if (j4 < n4)
      xs_store4<__nv_bfloat16>(xs, j4, k,
                               gamma ? make_float4(v[i].x * gv[i].x, v[i].y * gv[i].y, v[i].z * gv[i].z, v[i].w * gv[i].w)
                                     : v[i]);
  }
  consumer_sync();
  return ss;
}

__global__ void __launch_bounds__(SP_WARPS * 32, 1) stream_pass_kernel(const StreamPassParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[SP_WARPS][SP_MAX_STAGES];
  __shared__ float red[32];
  const PassParams& p = P.p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = P.stages;
  const uint32_t rowb = static_cast<uint32_t>(P.rowb), stageb = 2 * rowb;
  uint8_t* mystage = smem + static_cast<size_t>(warp) * S * stageb;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(SP_WARPS) * S * stageb);
  float* part = xs + P.xs_floats;
  uint64_t* mybar = bars[warp];
  const uint64_t pol = l2_evict_first_policy();
  const int L = p.n_layers, d = p.d, ff = p.ff;

  SpGeom G[SK_N];
  G[SK_QKV] = sp_geom(d, 3 * d, P.ch_d, P.nch_d, warp);
  G[SK_WO] = sp_geom(d, d, P.ch_d, P.nch_d, warp);
  G[SK_UP] = sp_geom(d, 2 * ff, P.ch_d, P.nch_d, warp);
  G[SK_DNA] = sp_geom(P.k_split, d, P.ch_f, P.nch_fa, warp, ff, 0);
  G[SK_DNB] = sp_geom(ff - P.k_split, d, P.ch_f, P.nch_fb, warp, ff, P.k_split);
  G[SK_HEAD] = sp_geom(d, p.V, P.ch_d, P.nch_d, warp);
  const int n_qkv = G[SK_QKV].n_tasks, n_wo = G[SK_WO].n_tasks, n_up = G[SK_UP].n_tasks;
  const int n_dna = G[SK_DNA].n_tasks, n_dnb = G[SK_DNB].n_tasks;
  const int NL = n_qkv + n_wo + n_up + n_dna + n_dnb;  // this warp's tasks per layer
  float* part_b = part + P.part_a_floats;  // down, second half
  const int n_all = L * NL + G[SK_HEAD].n_tasks;

  // global task i of this warp -> (weights, geometry, task index within its phase);
  // prefetch_only: the task's rows go to L2 (cp.async.bulk.prefetch) instead of the ring
  struct Loc {
    const __nv_bfloat16* src;
    uint32_t bytes;
    int ld;
    bool has_b;
  };
  auto locate = [&](int i) -> Loc {
    int kind, j;
    const void* w;
    if (i < L * NL) {
      const int l = i / NL;
      j = i - l * NL;
      const PassLayer& Ly = p.layers[l];
      if (j < n_qkv) {
        kind = SK_QKV;
        w = Ly.w_qkv;
      } else if ((j -= n_qkv) < n_wo) {
        kind = SK_WO;
        w = Ly.w_o;
      } else if ((j -= n_wo) < n_up) {
        kind = SK_UP;
        w = Ly.w_up;
      } else if ((j -= n_up) < n_dna) {
        kind = SK_DNA;
        w = Ly.w_down;
      } else {
        j -= n_dna;
        kind = SK_DNB;
        w = Ly.w_down;
      }
    } else {
      kind = SK_HEAD;
      j = i - L * NL;
      w = p.head;
    }
    const SpGeom& g = G[kind];
    const int t = warp + j * SP_WARPS;
    const int pl = t / g.nch, c = t - pl * g.nch;
    const int row0 = 2 * (g.pair_begin + pl);
    const int c0 = c * g.ch;
    Loc r;
    r.src = static_cast<const __nv_bfloat16*>(w) + static_cast<int64_t>(row0) * g.ld + g.kofs + c0;
    r.bytes = static_cast<uint32_t>(min(g.ch, g.k - c0)) * 2;
    r.ld = g.ld;
    r.has_b = row0 + 1 < g.n_rows;
    return r;
  };
  int pf_next = 0;  // (lane 0) first task neither issued nor L2-prefetched
  auto issue = [&](int i) {
    const Loc t = locate(i);
    const int slot = i % S;
    uint64_t* bar = &mybar[slot];
    uint8_t* dst = mystage + slot * stageb;
    mbar_arrive_expect_tx(bar, t.has_b ? 2 * t.bytes : t.bytes);
    bulk_g2s(dst, t.src, t.bytes, bar, pol);
    if (t.has_b) bulk_g2s(dst + rowb, t.src + t.ld, t.bytes, bar, pol);
    pf_next = max(pf_next, i + 1);
  };
  // Before a dependency wait the HBM would idle once the rings are full: the
  // next n tasks beyond the ring are requested into L2, so after the wait the
  // ring refills from L2 instead of HBM.
  auto prefetch_ahead = [&](int from, int n) {
    if (lane != 0) return;
    const int hi = min(from + n, n_all);
    for (int i = max(pf_next, from); i < hi; ++i) {
      const Loc t = locate(i);
      prefetch_l2_bulk(t.src, t.bytes);
      if (t.has_b) prefetch_l2_bulk(t.src + t.ld, t.bytes);
    }
    pf_next = max(pf_next, hi);
  };
  int gi = 0;  // next global task this warp consumes
  // consume one phase's tasks into `part`, refilling the ring as slots free
  auto run_phase = [&](const SpGeom& g, float* pt) {
    for (int j = 0; j < g.n_tasks; ++j, ++gi) {
      const int slot = gi % S;
      mbar_wait(&mybar[slot], static_cast<uint32_t>((gi / S) & 1));
      const int t = warp + j * SP_WARPS;
      const int c = t % g.nch;
      const int c0 = c * g.ch;
      const int ce = min(g.ch, g.k - c0);
      const uint8_t* st = mystage + slot * stageb;
      float acc_a = 0.0f, acc_b = 0.0f;
      dot_chunk<__nv_bfloat16>(st, st + rowb, xs, g.k, c0, ce, acc_a, acc_b);
      __syncwarp();
      if (lane == 0 && gi + S < n_all) {
        fence_proxy_async_smem();
        issue(gi + S);
      }
      acc_a = warp_sum(acc_a);
      acc_b = warp_sum(acc_b);
      if (lane == 0) {
        pt[2 * t] = acc_a;
        pt[2 * t + 1] = acc_b;
      }
    }
    consumer_sync();
  };
  auto stamp = [&](int idx) {
    if (P.trace && threadIdx.x == 0) P.trace[static_cast<size_t>(blockIdx.x) * P.trace_stride + idx] = gtimer();
  };

  EpiArgs ea;  // QKV epilogue arguments (cache pointers per layer below)
  ea.rope_cos = p.rope_cos;
  ea.rope_sin = p.rope_sin;
  ea.head_dim = p.dh;
  ea.max_seq = p.max_seq;
  ea.d_model = d;
  ea.kv_bf16 = 1;
  ea.kvp = P.att.kvp;
  ea.q_out = p.q;
  auto epilogue_phase = [&](const SpGeom& g, auto epi_tag, float inv) {
    constexpr int EPI = decltype(epi_tag)::value;
    for (int pl = threadIdx.x; pl < g.pair_end - g.pair_begin; pl += CONSUMER_THREADS) {
      float va = 0.0f, vb = 0.0f;
      for (int c = 0; c < g.nch; ++c) {
        va += part[2 * (pl * g.nch + c)];
        vb += part[2 * (pl * g.nch + c) + 1];
      }
      const int pair = g.pair_begin + pl;
      epilogue<EPI>(ea, pair, va * inv, vb * inv, 2 * pair + 1 < g.n_rows);
    }
  };

  int nb = 0;  // grid barriers passed
  auto grid_barrier = [&]() {
    ++nb;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(P.bar, 1);
      const unsigned long long t0 = gtimer();
      int seen;
      do {
        asm volatile("ld.acquire.gpu.b32 %0, [%1];" : "=r"(seen) : "l"(P.bar) : "memory");
        if (seen >= nb * static_cast<int>(gridDim.x)) break;
        if (gtimer() - t0 > SP_WATCHDOG_NS) {
          if (p.err) atomicOr(p.err, DEVERR_TIMEOUT);
          break;
        }
      } while (true);
    }
    __syncthreads();
  };

  stamp(0);
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  // weights never depend on the previous kernel: the whole first ring fill
  // goes out before the dependency wait
  if (lane == 0)
    for (int i = 0; i < min(S, n_all); ++i) issue(i);
  griddep_wait();
  const int len = __ldcg(p.seq_len);
  stamp(1);

  PairAttn A = P.att;
  for (int l = 0; l < L; ++l) {
    const PassLayer& Ly = p.layers[l];
    // ---- QKV (+ ln1 RMSNorm, RoPE, KV row write) ----
    {
      float ss = sp_load_x(p.x, Ly.ln1_g, d, xs);
      if (threadIdx.x == 0 && static_cast<int>(blockIdx.x) < 2 * p.h)
        kv_prefetch_l2((blockIdx.x & 1) ? Ly.v : Ly.k, P.att.kvp, blockIdx.x >> 1, p.max_seq, p.dh, 2, max(0, len - 1));
      run_phase(G[SK_QKV], part);
      const float inv = 1.0f / sqrtf(block_sum(ss, red) / static_cast<float>(d) + p.eps);
      ea.k_cache = Ly.k;
      ea.v_cache = Ly.v;
      ea.pos = len - 1;
      epilogue_phase(G[SK_QKV], std::integral_constant<int, EPI_QKV_ROPE>{}, inv);
    }
    stamp(2 + 8 * l);
    prefetch_ahead(gi + S, P.pf_att);
    grid_barrier();
    // ---- attention: split partials, barrier, merge into Wo's activation row ----
    A.k_cache = Ly.k;
    A.v_cache = Ly.v;
    if (static_cast<int>(blockIdx.x) < A.n_heads * A.ns) pair_attn_partial<true>(A, xs, p.err);
    stamp(3 + 8 * l);
    grid_barrier();
    pair_attn_merge(A, d, xs, part);
    stamp(4 + 8 * l);
    // ---- Wo + residual ----
    run_phase(G[SK_WO], part);
    ea.out = p.x;
    epilogue_phase(G[SK_WO], std::integral_constant<int, EPI_RESID>{}, 1.0f);
    stamp(5 + 8 * l);
    prefetch_ahead(gi + S, P.pf_bar);
    grid_barrier();
    // ---- ln2 RMSNorm + gate/up + SwiGLU ----
    {
      float ss = sp_load_x(p.x, Ly.ln2_g, d, xs);
      run_phase(G[SK_UP], part);
      const float inv = 1.0f / sqrtf(block_sum(ss, red) / static_cast<float>(d) + p.eps);
      ea.out = p.act;
      epilogue_phase(G[SK_UP], std::integral_constant<int, EPI_SWIGLU>{}, inv);
    }
    stamp(6 + 8 * l);
    prefetch_ahead(gi + S, P.pf_bar);
    grid_barrier();
    // ---- down + residual, over the two halves of k ----
    sp_load_x(p.act, nullptr, P.k_split, xs);
    run_phase(G[SK_DNA], part);
    sp_load_x(p.act + P.k_split, nullptr, ff - P.k_split, xs);
    run_phase(G[SK_DNB], part_b);
    {
      const SpGeom& ga = G[SK_DNA];
      const SpGeom& gb = G[SK_DNB];
      ea.out = p.x;
      for (int pl = threadIdx.x; pl < ga.pair_end - ga.pair_begin; pl += CONSUMER_THREADS) {
        float va = 0.0f, vb = 0.0f;
        for (int c = 0; c < ga.nch; ++c) {
          va += part[2 * (pl * ga.nch + c)];
          vb += part[2 * (pl * ga.nch + c) + 1];
        }
        for (int c = 0; c < gb.nch; ++c) {
          va += part_b[2 * (pl * gb.nch + c)];
          vb += part_b[2 * (pl * gb.nch + c) + 1];
        }
        const int pair = ga.pair_begin + pl;
        epilogue<EPI_RESID>(ea, pair, va, vb, 2 * pair + 1 < ga.n_rows);
      }
    }
    stamp(7 + 8 * l);
    prefetch_ahead(gi + S, P.pf_bar);
    grid_barrier();
  }
  // ---- ln_f RMSNorm + LM head ----
  griddep_launch_dependents();
  {
    float ss = sp_load_x(p.x, p.lnf_g, d, xs);
    run_phase(G[SK_HEAD], part);
    const float inv = 1.0f / sqrtf(block_sum(ss, red) / static_cast<float>(d) + p.eps);
    ea.out = p.logits;
    epilogue_phase(G[SK_HEAD], std::integral_constant<int, EPI_STORE>{}, inv);
  }
  stamp(2 + 8 * L);
  // departure: the last CTA out re-arms the barrier for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(P.bar + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      P.bar[0] = 0;
      P.bar[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------

static int sp_optin_smem(int dev) {
  static int v[64] = {0};
  if (!v[dev]) cudaDeviceGetAttribute(&v[dev], cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v[dev];
}

// chunks of exactly ch elements (the last one shorter): with ch % 64 == 0 every
// bulk copy starts on a 128-byte line of the row
static void sp_chunking(int k, int chmax, int* ch, int* nch, int* rowb) {
  if (chmax % 64 == 0) {
    *ch = chmax;
  } else {
    const int n = (k + chmax - 1) / chmax;
    *ch = ((k + n - 1) / n + 7) / 8 * 8;
  }
  *nch = (k + *ch - 1) / *ch;
  *rowb = ((*ch * 2 + 15) / 16) * 16;
}

cudaError_t stream_pass_prepare() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(stream_pass_kernel));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(stream_pass_kernel),
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              sp_optin_smem(dev) - static_cast<int>(fa.sharedSizeBytes));
}

cudaError_t stream_pass_configure(StreamPassParams* P, int chmax) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int G = num_sms(dev);
  const PassParams& p = P->p;
  if (p.d % 8 || p.ff % 8 || p.d > LOADX_MAXV * 4 * CONSUMER_THREADS || p.ff > LOADX_MAXV * 4 * CONSUMER_THREADS ||
      !P->bar || !P->att.part)
    return cudaErrorInvalidValue;
  int rowb_d, rowb_f;
  sp_chunking(p.d, chmax, &P->ch_d, &P->nch_d, &rowb_d);
  int nch_f;
  sp_chunking(p.ff, chmax, &P->ch_f, &nch_f, &rowb_f);
  P->rowb = std::max(rowb_d, rowb_f);
  if (nch_f < 2) {  // one chunk covers d_ff: split it in two
    P->ch_f = ((p.ff + 1) / 2 + 7) / 8 * 8;
    nch_f = 2;
  }
  P->nch_fa = (nch_f + 1) / 2;  // down: first half of the chunks, then the rest
  P->k_split = std::min(p.ff, P->nch_fa * P->ch_f);
  P->nch_fb = (p.ff - P->k_split + P->ch_f - 1) / P->ch_f;
  if (P->nch_fb < 1 || P->k_split % 8 || (p.ff - P->k_split) % 8) return cudaErrorInvalidValue;
  const PairAttn& A = P->att;
  if (A.head_dim % 4 || A.head_dim > 128 || (32 % (A.head_dim / 4)) || A.n_heads * A.ns > G ||
      A.n_heads * A.head_dim != p.d || A.ns > GP_ATT_MAX_NS || p.d > GP_MERGE_V * 4 * CONSUMER_THREADS)
    return cudaErrorInvalidValue;
  P->xs_floats = std::max({p.d, P->k_split, p.ff - P->k_split, SP_WARPS * (A.head_dim + 4)});
  auto part_floats = [&](int n_rows, int nch) { return ((n_rows + 1) / 2 + G - 1) / G * nch * 2; };
  P->part_a_floats = part_floats(p.d, P->nch_fa);
  const int part = std::max({part_floats(3 * p.d, P->nch_d), part_floats(2 * p.ff, P->nch_d),
                             P->part_a_floats + part_floats(p.d, P->nch_fb), part_floats(p.V, P->nch_d),
                             A.n_heads * A.ns});
  P->part_floats = part;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(stream_pass_kernel));
  if (e != cudaSuccess) return e;
  const int budget = sp_optin_smem(dev) - static_cast<int>(fa.sharedSizeBytes) - (P->xs_floats + part) * 4;
  P->stages = std::min({SP_MAX_STAGES, P->max_stages > 0 ? P->max_stages : SP_MAX_STAGES,
                        budget / (SP_WARPS * 2 * P->rowb)});
  if (P->stages < 1) return cudaErrorInvalidValue;
  P->smem_bytes = static_cast<size_t>(SP_WARPS) * P->stages * 2 * P->rowb + static_cast<size_t>(P->xs_floats + part) * 4;
  // the grid barrier needs every CTA resident at once: one CTA per SM must fit
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stream_pass_kernel, SP_WARPS * 32, P->smem_bytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  P->grid = G;
  return cudaSuccess;
}

cudaError_t launch_stream_pass(const StreamPassParams& P, cudaStream_t s, bool pdl) {
  if (P.grid < 1 || P.stages < 1) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.grid);
  cfg.blockDim = dim3(SP_WARPS * 32);
  cfg.dynamicSmemBytes = P.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, stream_pass_kernel, P);
}

}  // namespace grt
