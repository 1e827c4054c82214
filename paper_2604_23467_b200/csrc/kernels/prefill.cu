// prefill.cu -- the non-GEMM kernels of the batched prefill (sm_100a):
// embedding gather for P tokens, per-token RMSNorm into bf16 GEMM operands,
// causal attention over the KV cache for P queries, and the hand-off to the
// decode state (last row -> residual buffer, device seq_len).
//
// Reference: prefill = P sequential passes (pipeline.cpp:207-214); each pass's
// extend_position (kernels.cpp:238-259), layernorm (kernels.cpp:52-85, RMSNorm
// for LLaMA) and attention (kernels.cpp:87-137) become one launch over all P
// tokens.  Attention of query i sees keys [0, start+i] -- the causal mask is
// exactly the reference's per-pass length.
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace grt {

// x[i][:] = emb[tokens[start+i]][:]  (LLaMA: no position table)
template <typename WT>
__global__ void prefill_embed_kernel(const int* tokens, int start, int P, const WT* emb, int d, float* X, int vocab,
                                     int* err) {
  const int i = blockIdx.x;
  if (i >= P) return;
  const int tok = tokens[start + i];
  if (tok < 0 || tok >= vocab) {
    if (threadIdx.x == 0 && err) atomicOr(err, DEVERR_TOKEN_RANGE);
    return;
  }
  const WT* row = emb + static_cast<int64_t>(tok) * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) X[static_cast<int64_t>(i) * d + j] = to_f32(row[j]);
}

// Xn[i] = bf16(rmsnorm(X[i]) * gamma): ss = sum x^2 ; inv = 1/sqrt(ss/d + eps)
__global__ void prefill_rmsnorm_kernel(const float* X, const float* gamma, float eps, int d, __nv_bfloat16* Xn) {
  __shared__ float red[32];
  const int i = blockIdx.x;
  const float* x = X + static_cast<int64_t>(i) * d;
  float ss = 0.0f;
  for (int j = threadIdx.x; j < d; j += blockDim.x) ss += x[j] * x[j];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / static_cast<float>(d) + eps);
  for (int j = threadIdx.x; j < d; j += blockDim.x)
    Xn[static_cast<int64_t>(i) * d + j] = __float2bfloat16_rn(x[j] * inv * gamma[j]);
}

template <typename KT>
__device__ __forceinline__ float4 ld4(const KT* p);
template <>
__device__ __forceinline__ float4 ld4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  return make_float4(bf16lo(u.x), bf16hi(u.x), bf16lo(u.y), bf16hi(u.y));
}

// One warp per (query, head); G = dh/4 lanes per key row, RPW = 32/G rows per
// load, 8 row groups in flight, online softmax.  Output bf16 (Wo GEMM operand).
constexpr int PA_WARPS = 4;
constexpr int PA_UNROLL = 8;
template <typename KT>
__global__ void __launch_bounds__(PA_WARPS * 32)
    prefill_attn_kernel(const float* Q, const void* k_cache, const void* v_cache, int start, int P, int d, int dh,
                        int max_seq, float scale, __nv_bfloat16* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * PA_WARPS + warp;
  const int head = blockIdx.y;
  if (i >= P) return;
  const int G = dh >> 2, RPW = 32 / G;
  const int g = lane / G, c = lane - g * G;
  const int last = start + i;  // keys [0, last]
  const KT* K = reinterpret_cast<const KT*>(k_cache) + static_cast<int64_t>(head) * max_seq * dh + 4 * c;
  const KT* V = reinterpret_cast<const KT*>(v_cache) + static_cast<int64_t>(head) * max_seq * dh + 4 * c;
  const float4 q4 = *reinterpret_cast<const float4*>(Q + static_cast<int64_t>(i) * d + head * dh + 4 * c);
  float m = -INFINITY, l = 0.0f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int jb = 0; jb <= last; jb += RPW * PA_UNROLL) {
    float4 kv[PA_UNROLL], vv[PA_UNROLL];
#pragma unroll
    for (int u = 0; u < PA_UNROLL; ++u) {
      const int j = min(jb + u * RPW + g, last);
      kv[u] = ld4<KT>(K + static_cast<int64_t>(j) * dh);
      vv[u] = ld4<KT>(V + static_cast<int64_t>(j) * dh);
    }
    float sc[PA_UNROLL];
    float mr = -INFINITY;
#pragma unroll
    for (int u = 0; u < PA_UNROLL; ++u) {
      float sv = q4.x * kv[u].x + q4.y * kv[u].y + q4.z * kv[u].z + q4.w * kv[u].w;
      for (int o = G >> 1; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
      sc[u] = jb + u * RPW + g <= last ? sv * scale : -INFINITY;
      mr = fmaxf(mr, sc[u]);
    }
    for (int o = G; o < 32; o <<= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    const float mn = fmaxf(m, mr);
    const float f = m == -INFINITY ? 0.0f : __expf(m - mn);
    l *= f;
    acc = make_float4(acc.x * f, acc.y * f, acc.z * f, acc.w * f);
    m = mn;
#pragma unroll
    for (int u = 0; u < PA_UNROLL; ++u) {
      if (sc[u] == -INFINITY) continue;
      const float e = __expf(sc[u] - m);
      l += e;
      acc.x = fmaf(e, vv[u].x, acc.x);
      acc.y = fmaf(e, vv[u].y, acc.y);
      acc.z = fmaf(e, vv[u].z, acc.z);
      acc.w = fmaf(e, vv[u].w, acc.w);
    }
  }
  for (int o = G; o < 32; o <<= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (lane < G) {
    const float inv = 1.0f / l;
    __nv_bfloat16* o = out + static_cast<int64_t>(i) * d + head * dh + 4 * c;
    o[0] = __float2bfloat16_rn(acc.x * inv);
    o[1] = __float2bfloat16_rn(acc.y * inv);
    o[2] = __float2bfloat16_rn(acc.z * inv);
    o[3] = __float2bfloat16_rn(acc.w * inv);
  }
}

// decode hand-off: residual row of the last prompt token -> x, seq_len = len
__global__ void prefill_handoff_kernel(const float* X_last, int d, float* x, int* seq_len, int len) {
  for (int j = threadIdx.x; j < d; j += blockDim.x) x[j] = X_last[j];
  if (threadIdx.x == 0) *seq_len = len;
}

// ---- host -----------------------------------------------------------------------

cudaError_t launch_prefill_embed(Dt wdt, const int* tokens, int start, int P, const void* emb, int d, float* X,
                                 int vocab, int* err, cudaStream_t s) {
  if (wdt == Dt::BF16)
    prefill_embed_kernel<<<P, 256, 0, s>>>(tokens, start, P, static_cast<const __nv_bfloat16*>(emb), d, X, vocab, err);
  else
    prefill_embed_kernel<<<P, 256, 0, s>>>(tokens, start, P, static_cast<const float*>(emb), d, X, vocab, err);
  return cudaGetLastError();
}

cudaError_t launch_prefill_rmsnorm(const float* X, int P, const float* gamma, float eps, int d, void* Xn,
                                   cudaStream_t s) {
  prefill_rmsnorm_kernel<<<P, 256, 0, s>>>(X, gamma, eps, d, static_cast<__nv_bfloat16*>(Xn));
  return cudaGetLastError();
}

cudaError_t launch_prefill_attention(Dt kvdt, const float* Q, const void* k, const void* v, int start, int P, int d,
                                     int n_heads, int dh, int max_seq, float scale, void* out, cudaStream_t s) {
  const int gs = dh / 4;
  if (dh % 4 != 0 || gs < 1 || gs > 32 || (gs & (gs - 1)) != 0) return cudaErrorInvalidValue;
  dim3 grid((P + PA_WARPS - 1) / PA_WARPS, n_heads);
  if (kvdt == Dt::BF16)
    prefill_attn_kernel<__nv_bfloat16><<<grid, PA_WARPS * 32, 0, s>>>(Q, k, v, start, P, d, dh, max_seq, scale,
                                                                      static_cast<__nv_bfloat16*>(out));
  else
    prefill_attn_kernel<float><<<grid, PA_WARPS * 32, 0, s>>>(Q, k, v, start, P, d, dh, max_seq, scale,
                                                              static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

cudaError_t launch_prefill_handoff(const float* X_last, int d, float* x, int* seq_len, int len, cudaStream_t s) {
  prefill_handoff_kernel<<<1, 256, 0, s>>>(X_last, d, x, seq_len, len);
  return cudaGetLastError();
}

}  // namespace grt
