// gemv_pair.cu -- two consecutive decode GEMVs in ONE launch: the residual Wo
// GEMV (phase A) and the normed gate/up GEMV that consumes its output (phase
// B), separated by a grid-wide barrier.
//
// Why: between two per-op kernels the successor's CTAs only become resident
// when the predecessor's exit, and then pay the dependency release, the
// activation load and the norm before their weight ring runs (per-op trace:
// ~4-5 us per boundary, HBM partly idle).  Here every warp's weight ring runs
// straight from phase A's rows into phase B's rows (task numbering continues
// across the phase boundary), so phase B's first stages are in shared memory
// before the barrier releases; only the activation row (16 KB, L2) is loaded
// after it.  Same building blocks and arithmetic as gemv.cu (pair rows,
// round-robin (pair, chunk) tasks, per-task partials summed in chunk order,
// deferred RMSNorm scale) -- results are identical to the two per-op kernels.
//
// Co-residency: grid = one CTA per SM holding the SM's whole shared memory
// (occupancy checked at launch), and the kernel triggers its dependents only
// after the barrier, so every CTA of the grid is resident before any successor
// can take an SM; a watchdog turns a barrier that never completes into
// DEVERR_TIMEOUT instead of a hang.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int GP_WARPS = 8;
constexpr int GP_MAX_STAGES = 8;
constexpr unsigned long long GP_WATCHDOG_NS = 1000000000ull;  // 1 s

struct PhaseGeom {
  const __nv_bfloat16* w;
  int k, n_rows, ch, nch, pair_begin, pair_end, n_tasks;
};

__device__ __forceinline__ PhaseGeom phase_geom(const GemvParams& p, int warp) {
  PhaseGeom g;
  g.w = reinterpret_cast<const __nv_bfloat16*>(p.w);
  g.k = p.k;
  g.n_rows = p.n_rows;
  g.ch = p.ch;
  g.nch = p.nch;
  const int n_pairs = (p.n_rows + 1) >> 1;
  g.pair_begin = static_cast<int>(static_cast<int64_t>(blockIdx.x) * n_pairs / gridDim.x);
  g.pair_end = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * n_pairs / gridDim.x);
  const int Tc = (g.pair_end - g.pair_begin) * g.nch;
  g.n_tasks = Tc > warp ? (Tc - warp + GP_WARPS - 1) / GP_WARPS : 0;
  return g;
}

__device__ __forceinline__ unsigned long long gp_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int EB>
__global__ void __launch_bounds__(GP_WARPS * 32, 1) gemv_pair_kernel(const GemvPairParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[GP_WARPS][GP_MAX_STAGES];
  __shared__ float red[32];
  const GemvParams& pa = P.a;
  const GemvParams& pb = P.b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = P.stages;
  const uint32_t rowb = static_cast<uint32_t>(P.rowb), stageb = 2 * rowb;
  uint8_t* mystage = smem + static_cast<size_t>(warp) * S * stageb;
  float* xs = reinterpret_cast<float*>(smem + static_cast<size_t>(GP_WARPS) * S * stageb);
  float* part = xs + P.xs_floats;
  uint64_t* mybar = bars[warp];
  const uint64_t pol = l2_evict_first_policy();
  const PhaseGeom ga = phase_geom(pa, warp), gb = phase_geom(pb, warp);
  const int na = ga.n_tasks, n_all = na + gb.n_tasks;

  // global task i: phase A's tasks first, then phase B's (same slot sequence)
  auto issue = [&](int i) {
    const PhaseGeom& g = i < na ? ga : gb;
    const int t = warp + (i < na ? i : i - na) * GP_WARPS;
    const int pl = t / g.nch, c = t - pl * g.nch;
    const int row0 = 2 * (g.pair_begin + pl);
    const int c0 = c * g.ch;
    const int ce = min(g.ch, g.k - c0);
    const uint32_t bytes = static_cast<uint32_t>(ce) * 2;
    const bool has_b = row0 + 1 < g.n_rows;
    const int slot = i % S;
    uint64_t* bar = &mybar[slot];
    uint8_t* dst = mystage + slot * stageb;
    mbar_arrive_expect_tx(bar, has_b ? 2 * bytes : bytes);
    const __nv_bfloat16* src = g.w + static_cast<int64_t>(row0) * g.k + c0;
    bulk_g2s(dst, src, bytes, bar, pol);
    if (has_b) bulk_g2s(dst + rowb, src + g.k, bytes, bar, pol);
  };
  // consume tasks [i0, i1) of one phase into `part`, refilling the ring
  auto run_phase = [&](const PhaseGeom& g, int i0, int i1) {
    for (int i = i0; i < i1; ++i) {
      const int slot = i % S;
      mbar_wait(&mybar[slot], static_cast<uint32_t>((i / S) & 1));
      const int t = warp + (i - i0) * GP_WARPS;
      const int c = t % g.nch;
      const int c0 = c * g.ch;
      const int ce = min(g.ch, g.k - c0);
      const uint8_t* st = mystage + slot * stageb;
      float acc_a = 0.0f, acc_b = 0.0f;
      dot_chunk<__nv_bfloat16>(st, st + rowb, xs, g.k, c0, ce, acc_a, acc_b);
      __syncwarp();
      if (lane == 0 && i + S < n_all) {
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
    consumer_sync();
  };
  auto epi_args = [](const GemvParams& p) {
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
    return ea;
  };

  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  // phase B's norm weights, then the ring (its tail may already be phase B rows)
  float4 gv[LOADX_MAXV];
  {
    const int n4 = pb.k >> 2;
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) {
      const int j4 = threadIdx.x + i * CONSUMER_THREADS;
      gv[i] = j4 < n4 ? __ldg(reinterpret_cast<const float4*>(pb.gamma) + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (lane == 0) {
    for (int i = 0; i < min(S, n_all); ++i) issue(i);
  }
  griddep_wait();

  // grid-wide barrier number `nb` (co-resident grid, see the header comment)
  auto grid_barrier = [&](int nb) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(P.bar, 1);
      const unsigned long long t0 = gp_timer();
      int seen;
      do {
        asm volatile("ld.acquire.gpu.b32 %0, [%1];" : "=r"(seen) : "l"(P.bar) : "memory");
        if (gp_timer() - t0 > GP_WATCHDOG_NS) {
          if (P.err) atomicOr(P.err, DEVERR_TIMEOUT);
          break;
        }
      } while (seen < nb * static_cast<int>(gridDim.x));
    }
    __syncthreads();
  };

  // ---- phase A: residual GEMV (x_a produced by the previous kernel) ----
  load_x<__nv_bfloat16, NORM_NONE, false>(pa.x, nullptr, nullptr, 0.0f, pa.k, xs, red);
  run_phase(ga, 0, na);
  {
    const EpiArgs ea = epi_args(pa);
    for (int pl = threadIdx.x; pl < ga.pair_end - ga.pair_begin; pl += CONSUMER_THREADS) {
      float va = 0.0f, vb = 0.0f;
      for (int c = 0; c < ga.nch; ++c) {
        va += part[2 * (pl * ga.nch + c)];
        vb += part[2 * (pl * ga.nch + c) + 1];
      }
      const int pair = ga.pair_begin + pl;
      epilogue<EPI_RESID>(ea, pair, va, vb, 2 * pair + 1 < pa.n_rows);
    }
  }

  // ---- grid barrier: phase B reads the residual rows every CTA just wrote ----
  grid_barrier(1);
  griddep_launch_dependents();  // only now: every CTA of this grid is resident

  // ---- phase B: normed GEMV on the fresh residual (L2, bypass L1) ----
  float ss = 0.0f;
  {
    const int n4 = pb.k >> 2;
    float4 v[LOADX_MAXV];
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) {
      const int j4 = threadIdx.x + i * CONSUMER_THREADS;
      v[i] = j4 < n4 ? __ldcg(reinterpret_cast<const float4*>(pb.x) + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) {
      const int j4 = threadIdx.x + i * CONSUMER_THREADS;
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
      if (j4 < n4) {
        const float4 g = gv[i];
        xs_store4<__nv_bfloat16>(xs, j4, pb.k, make_float4(v[i].x * g.x, v[i].y * g.y, v[i].z * g.z, v[i].w * g.w));
      }
    }
    consumer_sync();
  }
  if constexpr (EB == EPI_QKV_ROPE) {  // K/V rows of this layer into L2 for the attention kernel
    if (threadIdx.x == 0 && pb.seq_len && static_cast<int>(blockIdx.x) < 2 * pb.n_heads) {
      kv_prefetch_l2((blockIdx.x & 1) ? pb.v_cache : pb.k_cache, pb.kvp, blockIdx.x >> 1, pb.max_seq, pb.head_dim,
                     pb.kv_bf16 ? 2 : 4, max(0, *pb.seq_len - 1));
    }
  }
  run_phase(gb, na, n_all);
  const float inv = 1.0f / sqrtf(block_sum(ss, red) / static_cast<float>(pb.k) + pb.eps);
  {
    const EpiArgs eb = epi_args(pb);
    for (int pl = threadIdx.x; pl < gb.pair_end - gb.pair_begin; pl += CONSUMER_THREADS) {
      float va = 0.0f, vb = 0.0f;
      for (int c = 0; c < gb.nch; ++c) {
        va += part[2 * (pl * gb.nch + c)];
        vb += part[2 * (pl * gb.nch + c) + 1];
      }
      const int pair = gb.pair_begin + pl;
      epilogue<EB>(eb, pair, va * inv, vb * inv, 2 * pair + 1 < pb.n_rows);
    }
  }
  // departure: the last CTA out re-arms the barrier for the next replay
  if (threadIdx.x == 0) {
    if (atomicAdd(P.bar + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      P.bar[0] = 0;
      P.bar[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------

static int optin_smem(int dev) {
  static int v[64] = {0};
  if (!v[dev]) cudaDeviceGetAttribute(&v[dev], cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v[dev];
}

static void pair_chunking(int k, int chmax, int* ch, int* nch, int* rowb) {
  *nch = (k + chmax - 1) / chmax;
  *ch = ((k + *nch - 1) / *nch + 7) / 8 * 8;
  *rowb = ((*ch * 2 + 15) / 16) * 16;
}

cudaError_t gemv_pair_prepare() {
  int dev = 0;
  cudaGetDevice(&dev);
  const void* f = reinterpret_cast<const void*>(gemv_pair_kernel<EPI_SWIGLU>);
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, f);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin_smem(dev) - static_cast<int>(fa.sharedSizeBytes));
}

// Wo + gate/up (epi_b = EPI_SWIGLU) -- the only pairing the plan uses.
cudaError_t launch_gemv_pair(int epi_b, GemvPairParams P, cudaStream_t s, bool pdl) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int G = num_sms(dev);
  if (epi_b != EPI_SWIGLU || P.a.k % 8 || P.b.k % 8 || !P.bar) return cudaErrorInvalidValue;
  pair_chunking(P.a.k, P.a.chmax > 0 ? P.a.chmax : 2048, &P.a.ch, &P.a.nch, &P.a.rowb);
  pair_chunking(P.b.k, P.b.chmax > 0 ? P.b.chmax : 2048, &P.b.ch, &P.b.nch, &P.b.rowb);
  P.rowb = std::max(P.a.rowb, P.b.rowb);
  P.xs_floats = std::max(P.a.k, P.b.k);
  auto part_floats = [&](const GemvParams& p) { return ((p.n_rows + 1) / 2 + G - 1) / G * p.nch * 2; };
  const int part = std::max(part_floats(P.a), part_floats(P.b));
  const int budget = optin_smem(dev) - 1024 - (P.xs_floats + part) * 4;
  P.stages = std::max(1, std::min(GP_MAX_STAGES, budget / (GP_WARPS * 2 * P.rowb)));
  if (P.stages < 2) return cudaErrorInvalidValue;
  const size_t smem = static_cast<size_t>(GP_WARPS) * P.stages * 2 * P.rowb + (P.xs_floats + part) * 4;
  // The grid barrier needs all G CTAs resident at once: one CTA per SM must
  // fit this configuration (checked here), and the kernel holds each SM's
  // whole shared memory, so no two of its CTAs share an SM.  Not a cooperative
  // launch: that is refused the early (PDL) launch during the attention
  // kernel, which is what lets every CTA fill its weight ring ahead (measured
  // 2.556 vs 2.467 ms/token).  Sharing the GPU with another context (MPS)
  // can still starve the barrier; the watchdog then reports DEVERR_TIMEOUT.
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemv_pair_kernel<EPI_SWIGLU>, GP_WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(GP_WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gemv_pair_kernel<EPI_SWIGLU>, P);
}

}  // namespace grt
