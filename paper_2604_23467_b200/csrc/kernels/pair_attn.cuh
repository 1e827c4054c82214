// pair_attn.cuh -- decode attention as a phase of a persistent launch (the
// fused pair kernel, gemv_pair.cu, and the streaming pass, stream_pass.cu):
// split partials by a subset of the grid, then (after a grid barrier) a merge
// of every head's partials into the next GEMV's activation row.
// Reference: make_attention (kernels.cpp:87-137).
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "gemv_core.cuh"
#include "kernels.h"

namespace grt {

constexpr int GP_WARPS = 8;

// ---- phase 0: decode attention (make_attention, kernels.cpp:87-137) ---------
// Partial of head b/ns over positions [s*span, min(len, (s+1)*span)), s = b%ns:
// every K and V row of a 64-position step is requested at once (G = dh/4 lanes
// per row, 4 elements each), scores masked by the live length, online
// max-subtracted softmax per warp, warps merged in warp order.  Writes
// {o[dh], m, l} (o unnormalised) to part[(head*ns + s) * (dh+4)].
constexpr int GP_ATT_UNROLL = 8;

template <bool CG = false>
__device__ __forceinline__ float4 ld_bf16x4(const __nv_bfloat16* p) {
  uint2 u;
  if constexpr (CG)
    u = __ldcg(reinterpret_cast<const uint2*>(p));
  else
    u = *reinterpret_cast<const uint2*>(p);
  return make_float4(bf16lo(u.x), bf16hi(u.x), bf16lo(u.y), bf16hi(u.y));
}

// CG: K/V rows written earlier in the SAME launch (streaming pass) are read
// through L2 (ld.global.cg), never a stale L1 line.
template <bool CG = false>
__device__ __forceinline__ void pair_attn_partial(const PairAttn& A, float* scratch, int* err) {
  const int dh = A.head_dim, G = dh >> 2, RPW = 32 / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / G, c = lane - g * G;
  const int head = blockIdx.x / A.ns, split = blockIdx.x - head * A.ns;
  const int len = __ldcg(A.seq_len);
  if ((len < 1 || len > A.ns * A.span) && blockIdx.x == 0 && threadIdx.x == 0 && err)
    atomicOr(err, DEVERR_WRONG_LENGTH);  // live length outside the bucket this graph was built for
  const int j0 = split * A.span, j1 = min(len, j0 + A.span);
  const __nv_bfloat16* K = static_cast<const __nv_bfloat16*>(A.k_cache) + 4 * c;
  const __nv_bfloat16* V = static_cast<const __nv_bfloat16*>(A.v_cache) + 4 * c;
  const float4 q4 = __ldcg(reinterpret_cast<const float4*>(A.q + head * dh) + c);
  float m = -INFINITY, l = 0.0f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int step = GP_WARPS * GP_ATT_UNROLL * RPW;
  for (int base = j0; base < j1; base += step) {
    const int jw = base + warp * GP_ATT_UNROLL * RPW;
    float4 kv[GP_ATT_UNROLL], vv[GP_ATT_UNROLL];
    int64_t row[GP_ATT_UNROLL];  // masked below
    if (A.kvp.page == 0) {
#pragma unroll
      for (int u = 0; u < GP_ATT_UNROLL; ++u)
        row[u] = (static_cast<int64_t>(head) * A.max_seq + min(jw + u * RPW + g, A.max_seq - 1)) * dh;
    } else {
#pragma unroll
      for (int u = 0; u < GP_ATT_UNROLL; ++u) row[u] = kv_row(A.kvp, head, A.max_seq, min(jw + u * RPW + g, A.max_seq - 1)) * dh;
    }
#pragma unroll
    for (int u = 0; u < GP_ATT_UNROLL; ++u) {
      kv[u] = ld_bf16x4<CG>(K + row[u]);
      vv[u] = ld_bf16x4<CG>(V + row[u]);
    }
    float sc[GP_ATT_UNROLL];
    float mr = -INFINITY;
#pragma unroll
    for (int u = 0; u < GP_ATT_UNROLL; ++u) {
      float sv = q4.x * kv[u].x + q4.y * kv[u].y + q4.z * kv[u].z + q4.w * kv[u].w;
      for (int o = G >> 1; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
      sc[u] = jw + u * RPW + g < j1 ? sv * A.scale : -INFINITY;
      mr = fmaxf(mr, sc[u]);
    }
    for (int o = G; o < 32; o <<= 1) mr = fmaxf(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    if (mr != -INFINITY) {
      const float mn = fmaxf(m, mr);
      const float f = m == -INFINITY ? 0.0f : __expf(m - mn);
      l *= f;
      acc = make_float4(acc.x * f, acc.y * f, acc.z * f, acc.w * f);
      m = mn;
#pragma unroll
      for (int u = 0; u < GP_ATT_UNROLL; ++u) {
        if (sc[u] == -INFINITY) continue;
        const float e = __expf(sc[u] - m);
        l += e;
        acc.x = fmaf(e, vv[u].x, acc.x);
        acc.y = fmaf(e, vv[u].y, acc.y);
        acc.z = fmaf(e, vv[u].z, acc.z);
        acc.w = fmaf(e, vv[u].w, acc.w);
      }
    }
  }
  for (int o = G; o < 32; o <<= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, o);
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  const int ld = dh + 4;
  if (lane < G) reinterpret_cast<float4*>(scratch + warp * ld)[c] = acc;
  if (lane == 0) {
    scratch[warp * ld + dh] = m;
    scratch[warp * ld + dh + 1] = l;
  }
  consumer_sync();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < GP_WARPS; ++w) M = fmaxf(M, scratch[w * ld + dh]);
  float* out = A.part + static_cast<int64_t>(head * A.ns + split) * ld;
  for (int d = threadIdx.x; d < dh; d += CONSUMER_THREADS) {
    float o = 0.0f;
#pragma unroll
    for (int w = 0; w < GP_WARPS; ++w) {
      const float mw = scratch[w * ld + dh];
      if (mw != -INFINITY) o += scratch[w * ld + d] * __expf(mw - M);
    }
    out[d] = o;
  }
  if (threadIdx.x == 0) {
    float L = 0.0f;
#pragma unroll
    for (int w = 0; w < GP_WARPS; ++w) {
      const float mw = scratch[w * ld + dh];
      if (mw != -INFINITY) L += scratch[w * ld + dh + 1] * __expf(mw - M);
    }
    out[dh] = M;
    out[dh + 1] = L;
  }
}

// Merge of every head's split partials into the Wo activation row (k = h*dh),
// in the xs layout; split order is fixed, so the result is deterministic.  All
// partial loads of a thread are issued before any is used (one L2 round trip).
constexpr int GP_ATT_MAX_NS = 4;
constexpr int GP_MERGE_V = 4;  // float4 outputs per thread: k <= 4096

__device__ __forceinline__ void pair_attn_merge(const PairAttn& A, int k, float* xs, float* tbl) {
  const int dh = A.head_dim, ns = A.ns, ld = dh + 4;
  for (int hh = threadIdx.x; hh < A.n_heads; hh += CONSUMER_THREADS) {
    float ms[GP_ATT_MAX_NS], ls[GP_ATT_MAX_NS];
#pragma unroll
    for (int s2 = 0; s2 < GP_ATT_MAX_NS; ++s2) {
      const float* pp = A.part + static_cast<int64_t>(hh * ns + s2) * ld;
      ms[s2] = s2 < ns ? __ldcg(pp + dh) : -INFINITY;
      ls[s2] = s2 < ns ? __ldcg(pp + dh + 1) : 0.0f;
    }
    float M = -INFINITY;
#pragma unroll
    for (int s2 = 0; s2 < GP_ATT_MAX_NS; ++s2) M = fmaxf(M, ms[s2]);
    float L = 0.0f, f[GP_ATT_MAX_NS];
#pragma unroll
    for (int s2 = 0; s2 < GP_ATT_MAX_NS; ++s2) {
      f[s2] = ms[s2] == -INFINITY ? 0.0f : __expf(ms[s2] - M);
      L += ls[s2] * f[s2];
    }
    const float inv = 1.0f / L;
#pragma unroll
    for (int s2 = 0; s2 < GP_ATT_MAX_NS; ++s2)
      if (s2 < ns) tbl[hh * ns + s2] = f[s2] * inv;
  }
  float4 v[GP_MERGE_V][GP_ATT_MAX_NS];
#pragma unroll
  for (int i = 0; i < GP_MERGE_V; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    const int idx = 4 * j4, hh = idx / dh, d = idx - hh * dh;
#pragma unroll
    for (int s2 = 0; s2 < GP_ATT_MAX_NS; ++s2)
      v[i][s2] = (j4 < (k >> 2) && s2 < ns)
                     ? __ldcg(reinterpret_cast<const float4*>(A.part + static_cast<int64_t>(hh * ns + s2) * ld + d))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  consumer_sync();  // tbl complete
#pragma unroll
  for (int i = 0; i < GP_MERGE_V; ++i) {
    const int j4 = threadIdx.x + i * CONSUMER_THREADS;
    if (j4 >= (k >> 2)) continue;
    const int hh = (4 * j4) / dh;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int s2 = 0; s2 < GP_ATT_MAX_NS; ++s2) {
      if (s2 >= ns) break;
      const float w = tbl[hh * ns + s2];
      o.x = fmaf(w, v[i][s2].x, o.x);
      o.y = fmaf(w, v[i][s2].y, o.y);
      o.z = fmaf(w, v[i][s2].z, o.z);
      o.w = fmaf(w, v[i][s2].w, o.w);
    }
    xs_store4<__nv_bfloat16>(xs, j4, k, o);
  }
  consumer_sync();
}

}  // namespace grt
