// attention.cu -- split-K flash-decode over the device KV cache (K3).
//
// Replaces make_attention (kernels.cpp:87-137): per head, s_j = (q . K_j) * scale
// over j in [0, len), max-subtracted softmax, out = sum_j p_j V_j.  The length is
// read from device memory (seq_len) instead of being baked into the plan
// (model.cpp:118-131), so one captured graph serves every length in its bucket.
//
// One thread-block cluster per head, sized for the graph's length bucket; see
// attn_decode_kernel.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace grt {

constexpr int ATTN_THREADS = 512;

template <typename KT>
__device__ __forceinline__ float4 load4(const KT* p);
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(bf16lo(u.x), bf16hi(u.x), bf16lo(u.y), bf16hi(u.y));
}

__device__ __forceinline__ float group_sum(float v, int gs) {
  for (int o = gs >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Decode attention for one head = one thread-block CLUSTER of `ns` CTAs
// (ns = 1..16, sized for the graph's bucket); CTA r of the cluster owns
// positions [r*span, (r+1)*span) in `rounds` passes of ATTN_WARPS warps x
// ATTN_UNROLL row groups.  A row of dh elements is read by G = dh/4 lanes
// (4 elements each), so one warp load covers RPW = 32/G positions.
//  * every K and V row of a pass is requested at once, right after the
//    dependency wait and in parallel with the seq_len / q loads (the rows are
//    addressed by bucket position, masked by the live length afterwards): one
//    memory round trip instead of three -- the kernel is latency bound;
//  * scores, max-subtracted softmax and P.V per warp (online across passes),
//    merged across warps in shared memory in warp order;
//  * the cluster's CTAs merge their partials {o[dh], m, l} through distributed
//    shared memory in rank order (deterministic, no global fences/atomics) and
//    rank 0 writes out[head] -- Wo reads a plain activation row.
constexpr int ATTN_UNROLL = 8;
constexpr int ATTN_WARPS = ATTN_THREADS / 32;
constexpr int ATTN_MAX_CLUSTER = 16;
constexpr size_t ATTN_STAGE_SMEM = 192 * 1024;  // dynamic smem for staged rounds (3 x 64 KB at dh 128)
__host__ __device__ constexpr int attn_pass_span(int dh) { return ATTN_WARPS * ATTN_UNROLL * (32 / (dh / 4)); }

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// generic address of `p` (this CTA's shared memory) in CTA `rank` of the cluster
template <typename T>
__device__ __forceinline__ const T* dsmem_map(const T* p, uint32_t rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const T*>(out);
}

template <typename KT>
__global__ void __launch_bounds__(ATTN_THREADS, 1) attn_decode_kernel(const AttnParams p) {
  __shared__ float s_m[ATTN_WARPS], s_l[ATTN_WARPS];
  __shared__ __align__(16) float s_o[ATTN_WARPS][256];
  __shared__ __align__(16) float c_o[256];  // this CTA's partial, read by rank 0 over DSMEM
  __shared__ float c_ml[2];
  op_stamp(p.trace, 0);
  const int dh = p.head_dim;
  const int G = dh >> 2, RPW = 32 / G;
  const int ns = static_cast<int>(cluster_nctarank());
  const int rank = static_cast<int>(cluster_ctarank());
  const int head = blockIdx.x / ns;
  const int pass = ATTN_WARPS * ATTN_UNROLL * RPW;
  const int rounds = p.rounds;
  const int span = pass * rounds;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, c = lane - g * G;
  const KT* K = reinterpret_cast<const KT*>(p.k_cache) + 4 * c;
  const KT* V = reinterpret_cast<const KT*>(p.v_cache) + 4 * c;
  // element offsets of this lane's rows in round r (bucket positions, masked below)
  auto rows_of = [&](int jw, int64_t* row) {
    if (p.kvp.page == 0) {
#pragma unroll
      for (int u = 0; u < ATTN_UNROLL; ++u)
        row[u] = (static_cast<int64_t>(head) * p.max_seq + min(jw + u * RPW + g, p.max_seq - 1)) * dh;
    } else {
#pragma unroll
      for (int u = 0; u < ATTN_UNROLL; ++u) row[u] = kv_row(p.kvp, head, p.max_seq, min(jw + u * RPW + g, p.max_seq - 1)) * dh;
    }
  };
  // Every row of round 0 except the current step's (position len-1, written by
  // the QKV kernel this kernel depends on) holds data of EARLIER steps or lies
  // past the live length (masked, never read into the result), so the whole
  // round is requested before the dependency wait -- overlapping the QKV
  // kernel's tail -- and only the new row is re-read after it.
  float4 kv[ATTN_UNROLL], vv[ATTN_UNROLL];
  const bool pre = p.prefetch && p.seq_len;
  if (pre) {
    int64_t row[ATTN_UNROLL];
    rows_of(rank * span + warp * ATTN_UNROLL * RPW, row);
#pragma unroll
    for (int u = 0; u < ATTN_UNROLL; ++u) {
      kv[u] = load4<KT>(K + row[u]);
      vv[u] = load4<KT>(V + row[u]);
    }
  }
  // Rounds 1.. (bf16, contiguous cache): their rows are staged into shared
  // memory by the TMA engine before the wait as well (p.smem_rounds of them).
  extern __shared__ __align__(128) uint8_t att_dyn[];  // [round-1][K|V][pass][dh] bf16
  __shared__ uint64_t rbar;
  const bool stage = pre && p.smem_rounds > 0 && p.kvp.page == 0 && sizeof(KT) == 2;
  const size_t rstride = static_cast<size_t>(pass) * dh * sizeof(KT);  // bytes of one K (or V) round
  if (stage) {
    if (threadIdx.x == 0) {
      mbar_init(&rbar, 1);
      mbar_fence_init();
      uint32_t total = 0;
      for (int r = 1; r <= p.smem_rounds; ++r) {
        const int j0 = rank * span + r * pass;
        const int nr = max(0, min(pass, p.max_seq - j0));
        total += 2u * static_cast<uint32_t>(nr) * dh * sizeof(KT);
      }
      mbar_arrive_expect_tx(&rbar, total);
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      for (int r = 1; r <= p.smem_rounds; ++r) {
        const int j0 = rank * span + r * pass;
        const int nr = max(0, min(pass, p.max_seq - j0));
        if (nr == 0) continue;
        const uint32_t bytes = static_cast<uint32_t>(nr) * dh * sizeof(KT);
        const int64_t off = (static_cast<int64_t>(head) * p.max_seq + j0) * dh;
        uint8_t* dst = att_dyn + static_cast<size_t>(r - 1) * 2 * rstride;
        bulk_g2s(dst, reinterpret_cast<const KT*>(p.k_cache) + off, bytes, &rbar, pol);
        bulk_g2s(dst + rstride, reinterpret_cast<const KT*>(p.v_cache) + off, bytes, &rbar, pol);
      }
    }
    __syncthreads();  // barrier initialised before anyone waits on it
  }
  griddep_wait();
  op_stamp(p.trace, 1);
  if (p.trigger == 0) griddep_launch_dependents();

  const int len = p.seq_len ? *p.seq_len : p.len_fixed;
  const float4 q4 = __ldcg(reinterpret_cast<const float4*>(p.q + head * dh) + c);
  float m = -INFINITY, l = 0.0f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int r = 0; r < rounds; ++r) {
    const int jw = rank * span + r * pass + warp * ATTN_UNROLL * RPW;  // first position of this warp
    int64_t row[ATTN_UNROLL];
    rows_of(jw, row);
    const bool from_smem = stage && r >= 1 && r <= p.smem_rounds;
    if (from_smem && r == 1) mbar_wait(&rbar, 0);
#pragma unroll
    for (int u = 0; u < ATTN_UNROLL; ++u) {
      const int jp = jw + u * RPW + g;
      if (r == 0 && pre && jp != len - 1) continue;  // requested before the wait
      if (from_smem && jp != len - 1 && jp < p.max_seq) {  // staged before the wait
        const int rr = jp - (rank * span + r * pass);
        const uint8_t* bk = att_dyn + static_cast<size_t>(r - 1) * 2 * rstride;
        kv[u] = load4<KT>(reinterpret_cast<const KT*>(bk) + rr * dh + 4 * c);
        vv[u] = load4<KT>(reinterpret_cast<const KT*>(bk + rstride) + rr * dh + 4 * c);
        continue;
      }
      kv[u] = load4<KT>(K + row[u]);
      vv[u] = load4<KT>(V + row[u]);
    }
    float sc[ATTN_UNROLL];
    float mr = -INFINITY;
#pragma unroll
    for (int u = 0; u < ATTN_UNROLL; ++u) {
      float sv = q4.x * kv[u].x + q4.y * kv[u].y + q4.z * kv[u].z + q4.w * kv[u].w;
      sv = group_sum(sv, G);  // lanes of one row share the score
      sc[u] = jw + u * RPW + g < len ? sv * p.scale : -INFINITY;
      mr = fmaxf(mr, sc[u]);
    }
    for (int o = G; o < 32; o <<= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));  // across row groups
    if (r == 0 && p.trace && warp == 0) op_stamp(p.trace, 2);
    if (mr != -INFINITY) {
      const float mn = fmaxf(m, mr);
      const float f = m == -INFINITY ? 0.0f : __expf(m - mn);
      l *= f;
      acc = make_float4(acc.x * f, acc.y * f, acc.z * f, acc.w * f);
      m = mn;
#pragma unroll
      for (int u = 0; u < ATTN_UNROLL; ++u) {
        if (sc[u] == -INFINITY) continue;  // masked rows never touch V (it may be stale)
        const float e = __expf(sc[u] - m);
        l += e;
        acc.x = fmaf(e, vv[u].x, acc.x);
        acc.y = fmaf(e, vv[u].y, acc.y);
        acc.z = fmaf(e, vv[u].z, acc.z);
        acc.w = fmaf(e, vv[u].w, acc.w);
      }
    }
  }
  if (p.trigger == 1) griddep_launch_dependents();
  // the warp's m is uniform; l and acc are per row group: reduce over groups
  for (int o = G; o < 32; o <<= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (lane < G) reinterpret_cast<float4*>(s_o[warp])[c] = acc;
  if (lane == 0) {
    s_m[warp] = m;
    s_l[warp] = l;
  }
  __syncthreads();

  // CTA merge (fixed warp order) -> this CTA's partial {o, m, l}
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < ATTN_WARPS; ++w) M = fmaxf(M, s_m[w]);
  float L = 0.0f, f[ATTN_WARPS];
#pragma unroll
  for (int w = 0; w < ATTN_WARPS; ++w) {
    f[w] = s_m[w] == -INFINITY ? 0.0f : __expf(s_m[w] - M);
    L += s_l[w] * f[w];
  }
  for (int d = threadIdx.x; d < dh; d += ATTN_THREADS) {
    float o = 0.0f;
#pragma unroll
    for (int w = 0; w < ATTN_WARPS; ++w) o += s_o[w][d] * f[w];
    c_o[d] = o;
  }
  if (threadIdx.x == 0) {
    c_ml[0] = M;
    c_ml[1] = L;
  }
  // live length outside the bucket this graph was built for (lengths below the
  // bucket are served correctly -- masked -- so only the upper end is unsafe)
  if (len < 1 || len > ns * span || (p.max_len > 0 && len > p.max_len)) {
    if (threadIdx.x == 0 && rank == 0 && head == 0 && p.err) atomicOr(p.err, DEVERR_WRONG_LENGTH);
  }
  op_stamp(p.trace, 4);
  if (ns == 1) {  // whole head in this CTA: no cluster exchange
    for (int d = threadIdx.x; d < dh; d += ATTN_THREADS) p.out[head * dh + d] = c_o[d] / L;  // own c_o[d], own L
    op_stamp(p.trace, 3);
    return;
  }
  cluster_sync_all();  // partials visible cluster-wide
  op_stamp(p.trace, 5);
  if (rank == 0) {
    float MM = -INFINITY;
    for (int r = 0; r < ns; ++r) MM = fmaxf(MM, *dsmem_map(&c_ml[0], r));
    float LL = 0.0f;
    for (int r = 0; r < ns; ++r) {
      const float mr = *dsmem_map(&c_ml[0], r);
      if (mr != -INFINITY) LL += *dsmem_map(&c_ml[1], r) * __expf(mr - MM);
    }
    const float inv = 1.0f / LL;
    // every remote read happens before rank 0's arrive; the global store of the
    // result comes after it, so the barrier's release never waits on it
    float res = 0.0f;
    const int d = threadIdx.x;
    if (d < dh) {
      for (int r = 0; r < ns; ++r) {
        const float mr = *dsmem_map(&c_ml[0], r);
        if (mr != -INFINITY) res += *dsmem_map(&c_o[d], r) * __expf(mr - MM);
      }
    }
    op_stamp(p.trace, 6);
    cluster_arrive();  // the other CTAs may now exit (their shared memory was read)
    if (d < dh) p.out[head * dh + d] = res * inv;
    cluster_wait();
  } else {
    op_stamp(p.trace, 6);
    cluster_sync_all();  // keep this CTA's shared memory alive until rank 0 has read it
  }
  op_stamp(p.trace, 3);
  // (trigger 2: the successor launches when this CTA exits)
}

// Cluster size and passes for a bucket of max_len positions.
// Each CTA takes up to `per_cta` passes before the head is split over a
// cluster: a pass costs one memory round trip, a cluster costs two cluster
// barriers and a DSMEM merge (measured: ~1 round trip each while the next
// kernel's CTAs are being launched).
static int attn_rounds_per_cta() {
  return 1;  // measured: 2-CTA clusters beat 2 rounds in one CTA (p99 2.56 vs 2.58 ms)
}

// cap: the largest cluster for which all n_heads clusters fit on the SMs at once
// (one 512-thread CTA per SM): a second wave would double the latency.
static int attn_cluster_cap(int n_heads) {
  if (n_heads <= 0) return ATTN_MAX_CLUSTER;
  int dev = 0;
  cudaGetDevice(&dev);
  int c = 1;
  while (2 * c <= ATTN_MAX_CLUSTER && 2 * c * n_heads <= num_sms(dev)) c <<= 1;
  return c;
}

static void attn_shape(int max_len, int head_dim, int* ns, int* rounds, int n_heads = 0) {
  const int pass = attn_pass_span(head_dim);
  const int need = std::max(1, (max_len + pass - 1) / pass);  // passes over the whole bucket
  const int want = (need + attn_rounds_per_cta() - 1) / attn_rounds_per_cta();
  const int cap = attn_cluster_cap(n_heads);
  int c = 1;
  while (c < want && c < cap) c <<= 1;
  *ns = c;
  *rounds = (need + c - 1) / c;
}

int attention_splits(int max_len, int head_dim) {
  int ns, rounds;
  attn_shape(max_len, head_dim, &ns, &rounds);
  return ns;
}

int attention_nsplit(int max_len, int n_heads, int sms) {
  // persistent pass: aim for ~one wave of CTAs and >= 32 positions per CTA.
  int ns = std::max(1, std::min((max_len + 31) / 32, std::max(1, (2 * sms) / std::max(1, n_heads))));
  return std::min(ns, 64);
}

cudaError_t launch_attention(Dt kvdt, AttnParams p, int max_len, cudaStream_t s, bool pdl) {
  const int gs = p.head_dim / 4;
  if (p.head_dim % 4 != 0 || gs < 1 || gs > 32 || (gs & (gs - 1)) != 0 || p.head_dim > 256)
    return cudaErrorInvalidValue;
  int ns, rounds;
  attn_shape(max_len, p.head_dim, &ns, &rounds, p.n_heads);
  p.rounds = rounds;
  p.max_len = max_len;
  // 0 (default): the successor (Wo + gate/up) launches at once and fills its
  // weight ring on the SMs this small grid leaves free (measured fastest)
  p.trigger = 0;
  p.prefetch = 1;  // round 0's old rows requested before the dependency wait (2.588 -> 2.442 ms/token)
  const int stage_max = 3;  // rounds >= 1 staged through shared memory before the wait (P=500: 2.745 -> 2.681 ms)
  const int pref = p.prefetch;
  const size_t rbytes = static_cast<size_t>(attn_pass_span(p.head_dim)) * p.head_dim * 2 * 2;  // K+V of a round
  // bulk copies need 16-byte aligned sources and sizes: rows of dh bf16 with dh % 8 == 0
  p.smem_rounds = (kvdt == Dt::BF16 && p.kvp.page == 0 && pref && p.head_dim % 8 == 0)
                      ? std::min(rounds - 1, stage_max) : 0;
  while (p.smem_rounds > 0 && static_cast<size_t>(p.smem_rounds) * rbytes > ATTN_STAGE_SMEM) --p.smem_rounds;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_heads * ns);
  cfg.blockDim = dim3(ATTN_THREADS);
  cfg.dynamicSmemBytes = static_cast<size_t>(p.smem_rounds) * rbytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ns;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  if (kvdt == Dt::BF16) return cudaLaunchKernelEx(&cfg, attn_decode_kernel<__nv_bfloat16>, p);
  return cudaLaunchKernelEx(&cfg, attn_decode_kernel<float>, p);
}

cudaError_t attention_prepare() {
  for (const void* f : {reinterpret_cast<const void*>(attn_decode_kernel<__nv_bfloat16>),
                        reinterpret_cast<const void*>(attn_decode_kernel<float>)}) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ATTN_STAGE_SMEM));
    if (e != cudaSuccess) return e;
    // same L1/shared carveout as the GEMVs, so the next GEMV's CTAs can become
    // resident next to attention CTAs (PDL) without an SM reconfiguration
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace grt
