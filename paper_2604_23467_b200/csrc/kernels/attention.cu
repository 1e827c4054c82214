// attention.cu -- split-K flash-decode over the device KV cache (K3).
//
// Replaces make_attention (kernels.cpp:87-137): per head, s_j = (q . K_j) * scale
// over j in [0, len), max-subtracted softmax, out = sum_j p_j V_j.  The length is
// read from device memory (seq_len) instead of being baked into the plan
// (model.cpp:118-131), so one captured graph serves every length in its bucket.
//
// Grid = (n_heads, nsplit).  Each CTA scores its span of positions (a group of
// head_dim/4 lanes per position, coalesced row reads of the [h][max_seq][dh]
// cache), does a local softmax, accumulates P.V and, when nsplit > 1, publishes
// (m, l, o) partials; the LAST CTA of a head (arrival counter) merges the
// partials in split order, so results are deterministic run to run.
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace grt {

constexpr int ATTN_THREADS = 128;

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

__device__ __forceinline__ float block_reduce(float v, float* red, bool is_max) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (ATTN_THREADS / 32) ? red[threadIdx.x] : (is_max ? -INFINITY : 0.0f);
    t = is_max ? warp_max(t) : warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

template <typename KT>
__global__ void __launch_bounds__(ATTN_THREADS) attn_decode_kernel(const AttnParams p) {
  extern __shared__ __align__(16) float sm[];
  __shared__ float red[32];
  __shared__ int s_last;
  griddep_launch_dependents();
  griddep_wait();

  const int len = p.seq_len ? *p.seq_len : p.len_fixed;
  const int head = blockIdx.x, split = blockIdx.y, ns = gridDim.y;
  const int dh = p.head_dim;
  const int gs = dh >> 2;                  // lanes per position (4 dims per lane)
  const int npg = ATTN_THREADS / gs;       // position groups per CTA
  const int span = (len + ns - 1) / ns;
  if (len < 1 || span > p.span_cap) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && p.err) atomicOr(p.err, DEVERR_WRONG_LENGTH);
    return;  // uniform across the grid: every CTA sees the same len
  }
  const int j0 = split * span;
  const int j1 = min(len, j0 + span);
  const int n = max(0, j1 - j0);

  float* qs = sm;                  // [dh]
  float* sc = qs + dh;             // [span_cap]
  float* op = sc + p.span_cap;     // [npg][dh]
  for (int d = threadIdx.x; d < dh; d += ATTN_THREADS) qs[d] = p.q[head * dh + d];
  __syncthreads();

  const KT* K = reinterpret_cast<const KT*>(p.k_cache) + static_cast<int64_t>(head) * p.max_seq * dh;
  const KT* V = reinterpret_cast<const KT*>(p.v_cache) + static_cast<int64_t>(head) * p.max_seq * dh;
  const int grp = threadIdx.x / gs, gl = threadIdx.x - grp * gs;
  const float4 q4 = reinterpret_cast<const float4*>(qs)[gl];

  // scores
  for (int jb = 0; jb < n; jb += npg) {  // warp-uniform trip count (shuffles below)
    const int jj = jb + grp;
    float s = 0.0f;
    if (jj < n) {
      const float4 k4 = load4<KT>(K + static_cast<int64_t>(j0 + jj) * dh + 4 * gl);
      s = q4.x * k4.x + q4.y * k4.y + q4.z * k4.z + q4.w * k4.w;
    }
    s = group_sum(s, gs);
    if (jj < n && gl == 0) sc[jj] = s * p.scale;
  }
  __syncthreads();
  float m = -INFINITY;
  for (int jj = threadIdx.x; jj < n; jj += ATTN_THREADS) m = fmaxf(m, sc[jj]);
  m = block_reduce(m, red, true);
  float l = 0.0f;
  for (int jj = threadIdx.x; jj < n; jj += ATTN_THREADS) {
    const float e = expf(sc[jj] - m);
    sc[jj] = e;
    l += e;
  }
  l = block_reduce(l, red, false);  // ends with __syncthreads: sc visible

  // o = sum_j e_j V_j
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int jj = grp; jj < n; jj += npg) {
    const float e = sc[jj];
    const float4 v4 = load4<KT>(V + static_cast<int64_t>(j0 + jj) * dh + 4 * gl);
    acc.x = fmaf(e, v4.x, acc.x);
    acc.y = fmaf(e, v4.y, acc.y);
    acc.z = fmaf(e, v4.z, acc.z);
    acc.w = fmaf(e, v4.w, acc.w);
  }
  reinterpret_cast<float4*>(op + grp * dh)[gl] = acc;
  __syncthreads();

  if (ns == 1) {
    const float inv = 1.0f / l;
    for (int d = threadIdx.x; d < dh; d += ATTN_THREADS) {
      float o = 0.0f;
      for (int g = 0; g < npg; ++g) o += op[g * dh + d];
      p.out[head * dh + d] = o * inv;
    }
    return;
  }

  // publish this split's partial
  const int stride = dh + 2;
  float* mine = p.part + (static_cast<int64_t>(head) * ns + split) * stride;
  for (int d = threadIdx.x; d < dh; d += ATTN_THREADS) {
    float o = 0.0f;
    for (int g = 0; g < npg; ++g) o += op[g * dh + d];
    mine[d] = o;
  }
  if (threadIdx.x == 0) {
    mine[dh] = n > 0 ? m : -INFINITY;
    mine[dh + 1] = n > 0 ? l : 0.0f;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&p.counters[head], 1) == ns - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // merge in split order (deterministic)
  const float* base = p.part + static_cast<int64_t>(head) * ns * stride;
  float M = -INFINITY;
  for (int s = 0; s < ns; ++s) {
    const float ls = __ldcg(base + s * stride + dh + 1);
    if (ls > 0.0f) M = fmaxf(M, __ldcg(base + s * stride + dh));
  }
  float L = 0.0f;
  for (int s = 0; s < ns; ++s) {
    const float ls = __ldcg(base + s * stride + dh + 1);
    if (ls > 0.0f) L += ls * expf(__ldcg(base + s * stride + dh) - M);
  }
  const float invL = 1.0f / L;
  for (int d = threadIdx.x; d < dh; d += ATTN_THREADS) {
    float o = 0.0f;
    for (int s = 0; s < ns; ++s) {
      const float ls = __ldcg(base + s * stride + dh + 1);
      if (ls > 0.0f) o += __ldcg(base + s * stride + d) * expf(__ldcg(base + s * stride + dh) - M);
    }
    p.out[head * dh + d] = o * invL;
  }
  if (threadIdx.x == 0) p.counters[head] = 0;  // self-reset for the next replay
}

int attention_nsplit(int max_len, int n_heads, int sms) {
  // Aim for ~one wave of CTAs and >= 32 positions per CTA.
  int ns = std::max(1, std::min((max_len + 31) / 32, std::max(1, (2 * sms) / std::max(1, n_heads))));
  return std::min(ns, 64);
}

cudaError_t launch_attention(Dt kvdt, AttnParams p, int nsplit, cudaStream_t s, bool pdl) {
  const int gs = p.head_dim / 4;
  if (p.head_dim % 4 != 0 || gs < 1 || gs > 32 || (gs & (gs - 1)) != 0) return cudaErrorInvalidValue;
  const int npg = ATTN_THREADS / gs;
  const size_t smem = (static_cast<size_t>(p.head_dim) + p.span_cap + static_cast<size_t>(npg) * p.head_dim) * 4;
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_heads, nsplit);
  cfg.blockDim = dim3(ATTN_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (kvdt == Dt::BF16) return cudaLaunchKernelEx(&cfg, attn_decode_kernel<__nv_bfloat16>, p);
  return cudaLaunchKernelEx(&cfg, attn_decode_kernel<float>, p);
}

cudaError_t attention_prepare() {
  cudaError_t e = cudaFuncSetAttribute(attn_decode_kernel<__nv_bfloat16>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_decode_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}
// (200 KB + the 132 B of static shared memory stays below the 227 KB opt-in limit)

}  // namespace grt
