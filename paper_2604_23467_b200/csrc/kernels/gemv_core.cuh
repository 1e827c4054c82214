// gemv_core.cuh -- device building blocks of the batch-1 GEMV family, shared by
// the per-op kernels (gemv.cu) and the fused pair kernel (gemv_pair.cu).
//
// Reference ops: make_layernorm (kernels.cpp:52-85) + make_matmul
// (kernels.cpp:23-50) + make_kv_write (kernels.cpp:188-203) + make_residual_add /
// make_relu (kernels.cpp:162-186); LLaMA adds RMSNorm, RoPE and SwiGLU.  Weights
// are stored [n,k] (transposed reference [k,n]) so one output is one contiguous
// row; rows are consumed in adjacent PAIRS (2p, 2p+1) so RoPE (rotate-half, rows
// permuted so (i, i+dh/2) are adjacent) and SwiGLU (gate/up interleaved) finish
// inside one warp.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"

namespace grt {

template <typename WT>
struct WTraits;
template <>
struct WTraits<__nv_bfloat16> {
  static constexpr int VEC = 8;    // elements per 16-byte lane load
  static constexpr int CH = 2048;  // elements per row chunk (4 KB)
};
template <>
struct WTraits<float> {
  static constexpr int VEC = 4;
  static constexpr int CH = 1024;
};

// Index of element j in the shared-memory activation buffer.  For bf16 weights
// each lane multiplies 8 consecutive elements, so x is split into two planes
// (elements 0-3 and 4-7 of every group of 8) and both float4 reads of a warp are
// contiguous 512-byte rows -- no bank conflicts.
template <typename WT>
__device__ __forceinline__ int xs_index(int j, int k) {
  if constexpr (WTraits<WT>::VEC == 8) {
    const int g = j >> 3, w = j & 7;
    return (w >> 2) * (k >> 1) + g * 4 + (w & 3);
  } else {
    return j;
  }
}

// The compute ("consumer") warps of a CTA: 8 warps.  They synchronise on named
// barrier 1, so the block-wide syncs never involve a non-consumer warp.
#ifndef GRT_CONSUMER_THREADS
#define GRT_CONSUMER_THREADS 256
#endif
constexpr int CONSUMER_THREADS = GRT_CONSUMER_THREADS;
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(CONSUMER_THREADS) : "memory"); }

__device__ __forceinline__ float block_sum(float v, float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum(v);
  consumer_sync();  // red reuse
  if (lane == 0) red[warp] = v;
  consumer_sync();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (CONSUMER_THREADS >> 5) ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  consumer_sync();
  return red[0];
}

// L2-coherent activation load (the persistent pass reads values other CTAs
// wrote in the same launch, so L1 must be bypassed).
template <bool CG>
__device__ __forceinline__ float act_ld(const float* p) {
  if constexpr (CG) return __ldcg(p);
  return *p;
}

template <typename WT, int NORM, bool CG>
__device__ __noinline__ void load_x_slow(const float* x, const float* gamma, const float* beta, float eps, int k,
                                         float* xs, float* red);

template <bool CG>
__device__ __forceinline__ float4 act_ld4(const float* p) {
  if constexpr (CG) return __ldcg(reinterpret_cast<const float4*>(p));
  return *reinterpret_cast<const float4*>(p);
}

// Writes float4 #j4 of the activation into the shared-memory layout (for bf16
// weights an aligned float4 of x is exactly one float4 of plane j4&1).
template <typename WT>
__device__ __forceinline__ void xs_store4(float* xs, int j4, int k, float4 v) {
  if constexpr (WTraits<WT>::VEC == 8)
    reinterpret_cast<float4*>(xs + (j4 & 1) * (k >> 1))[j4 >> 1] = v;
  else
    reinterpret_cast<float4*>(xs)[j4] = v;
}

// float4 per thread kept in registers: covers k <= 12288 (LLaMA-2 7B d_ff = 11008)
constexpr int LOADX_MAXV = (12288 / 4 + CONSUMER_THREADS - 1) / CONSUMER_THREADS;

// Activation prologue: xs = norm(x) (or x).  The whole activation row is pulled
// into registers with independent 16-byte loads first (latency paid once, not
// per element), then reduced, normalised and stored.  Norm arithmetic follows
// the reference layernorm (kernels.cpp:66-83): sum -> mean, sum of squared
// deviations -> variance, inv = 1/sqrt(var + eps); RMSNorm drops mean and beta.
template <typename WT, int NORM, bool CG>
__device__ __forceinline__ void load_x(const float* x, const float* gamma, const float* beta, float eps, int k,
                                       float* xs, float* red) {
  const int n4 = k >> 2;
  if (n4 <= LOADX_MAXV * static_cast<int>(CONSUMER_THREADS)) {
    float4 v[LOADX_MAXV];
#pragma unroll
    for (int i = 0; i < LOADX_MAXV; ++i) {
      const int j4 = threadIdx.x + i * CONSUMER_THREADS;
      v[i] = j4 < n4 ? act_ld4<CG>(x + 4 * j4) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float mean = 0.0f, inv = 1.0f;
    if constexpr (NORM == NORM_RMS) {
      float ss = 0.0f;
#pragma unroll
      for (int i = 0; i < LOADX_MAXV; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
      ss = block_sum(ss, red);
      inv = 1.0f / sqrtf(ss / static_cast<float>(k) + eps);
    } else if constexpr (NORM == NORM_LN) {
      float s = 0.0f;
#pragma unroll
      for (int i = 0; i < LOADX_MAXV; ++i) s += v[i].x + v[i].y + v[i].z + v[i].w;
      mean = block_sum(s, red) / static_cast<float>(k);
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
        const float4 g = *reinterpret_cast<const float4*>(gamma + 4 * j4);
        o = make_float4(o.x * inv * g.x, o.y * inv * g.y, o.z * inv * g.z, o.w * inv * g.w);
      } else if constexpr (NORM == NORM_LN) {
        const float4 g = *reinterpret_cast<const float4*>(gamma + 4 * j4);
        const float4 b = *reinterpret_cast<const float4*>(beta + 4 * j4);
        o = make_float4((o.x - mean) * inv * g.x + b.x, (o.y - mean) * inv * g.y + b.y,
                        (o.z - mean) * inv * g.z + b.z, (o.w - mean) * inv * g.w + b.w);
      }
      xs_store4<WT>(xs, j4, k, o);
    }
    consumer_sync();
    return;
  }
  load_x_slow<WT, NORM, CG>(x, gamma, beta, eps, k, xs, red);
}

// Generic fallback for very wide activations (k > 12*4*blockDim).
template <typename WT, int NORM, bool CG>
__device__ __noinline__ void load_x_slow(const float* x, const float* gamma, const float* beta, float eps, int k,
                                         float* xs, float* red) {
  if constexpr (NORM == NORM_NONE) {
    for (int j = threadIdx.x; j < k; j += CONSUMER_THREADS) xs[xs_index<WT>(j, k)] = act_ld<CG>(x + j);
  } else if constexpr (NORM == NORM_RMS) {
    float ss = 0.0f;
    for (int j = threadIdx.x; j < k; j += CONSUMER_THREADS) {
      const float v = act_ld<CG>(x + j);
      xs[xs_index<WT>(j, k)] = v;
      ss += v * v;
    }
    ss = block_sum(ss, red);  // also orders the xs writes above
    const float inv = 1.0f / sqrtf(ss / static_cast<float>(k) + eps);
    for (int j = threadIdx.x; j < k; j += CONSUMER_THREADS) {
      const int i = xs_index<WT>(j, k);
      xs[i] = xs[i] * inv * gamma[j];
    }
  } else {
    float s = 0.0f;
    for (int j = threadIdx.x; j < k; j += CONSUMER_THREADS) {
      const float v = act_ld<CG>(x + j);
      xs[xs_index<WT>(j, k)] = v;
      s += v;
    }
    const float mean = block_sum(s, red) / static_cast<float>(k);
    float var = 0.0f;
    for (int j = threadIdx.x; j < k; j += CONSUMER_THREADS) {
      const float c = xs[xs_index<WT>(j, k)] - mean;
      var += c * c;
    }
    var = block_sum(var, red) / static_cast<float>(k);
    const float inv = 1.0f / sqrtf(var + eps);
    for (int j = threadIdx.x; j < k; j += CONSUMER_THREADS) {
      const int i = xs_index<WT>(j, k);
      xs[i] = (xs[i] - mean) * inv * gamma[j] + beta[j];
    }
  }
  consumer_sync();
}

// Partial dot products of one row pair over one chunk [c0, c0+ce).
template <typename WT>
__device__ __forceinline__ void dot_chunk(const uint8_t* sa, const uint8_t* sb, const float* xs, int k, int c0,
                                          int ce, float& acc_a, float& acc_b) {
  const int lane = threadIdx.x & 31;
  if constexpr (WTraits<WT>::VEC == 8) {
    const uint4* wa = reinterpret_cast<const uint4*>(sa);
    const uint4* wb = reinterpret_cast<const uint4*>(sb);
    const float4* xa = reinterpret_cast<const float4*>(xs) + (c0 >> 3);
    const float4* xb = reinterpret_cast<const float4*>(xs + (k >> 1)) + (c0 >> 3);
    const int groups = ce >> 3;
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 4
    for (int g = lane; g < groups; g += 32) {
      const uint4 u = wa[g];
      const uint4 v = wb[g];
      const float4 x0 = xa[g];
      const float4 x1 = xb[g];
      a0 = fmaf(bf16lo(u.x), x0.x, a0);
      a1 = fmaf(bf16hi(u.x), x0.y, a1);
      a0 = fmaf(bf16lo(u.y), x0.z, a0);
      a1 = fmaf(bf16hi(u.y), x0.w, a1);
      a0 = fmaf(bf16lo(u.z), x1.x, a0);
      a1 = fmaf(bf16hi(u.z), x1.y, a1);
      a0 = fmaf(bf16lo(u.w), x1.z, a0);
      a1 = fmaf(bf16hi(u.w), x1.w, a1);
      b0 = fmaf(bf16lo(v.x), x0.x, b0);
      b1 = fmaf(bf16hi(v.x), x0.y, b1);
      b0 = fmaf(bf16lo(v.y), x0.z, b0);
      b1 = fmaf(bf16hi(v.y), x0.w, b1);
      b0 = fmaf(bf16lo(v.z), x1.x, b0);
      b1 = fmaf(bf16hi(v.z), x1.y, b1);
      b0 = fmaf(bf16lo(v.w), x1.z, b0);
      b1 = fmaf(bf16hi(v.w), x1.w, b1);
    }
    acc_a += a0 + a1;
    acc_b += b0 + b1;
  } else {
    const float4* wa = reinterpret_cast<const float4*>(sa);
    const float4* wb = reinterpret_cast<const float4*>(sb);
    const float4* xv = reinterpret_cast<const float4*>(xs) + (c0 >> 2);
    const int groups = ce >> 2;
    float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 4
    for (int g = lane; g < groups; g += 32) {
      const float4 u = wa[g];
      const float4 v = wb[g];
      const float4 x = xv[g];
      a0 = fmaf(u.x, x.x, a0);
      a1 = fmaf(u.y, x.y, a1);
      a0 = fmaf(u.z, x.z, a0);
      a1 = fmaf(u.w, x.w, a1);
      b0 = fmaf(v.x, x.x, b0);
      b1 = fmaf(v.y, x.y, b1);
      b0 = fmaf(v.z, x.z, b0);
      b1 = fmaf(v.w, x.w, b1);
    }
    acc_a += a0 + a1;
    acc_b += b0 + b1;
  }
}

// Epilogue arguments (a view of GemvParams that the persistent pass can fill
// per phase).
struct EpiArgs {
  float* out = nullptr;
  float* q_out = nullptr;
  void* k_cache = nullptr;
  void* v_cache = nullptr;
  int pos = 0;  // KV row (seq_len - 1)
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int head_dim = 0, max_seq = 0, d_model = 0;
  int kv_bf16 = 0;
  KvPaging kvp;
};

template <int EPI>
__device__ __forceinline__ void epilogue(const EpiArgs& p, int pair, float va, float vb, bool has_b) {
  const int row0 = 2 * pair;
  if constexpr (EPI == EPI_STORE) {
    p.out[row0] = va;
    if (has_b) p.out[row0 + 1] = vb;
  } else if constexpr (EPI == EPI_RESID) {
    // x is owned row-wise by this warp for the whole phase: plain RMW is safe
    p.out[row0] = __ldcg(p.out + row0) + va;
    if (has_b) p.out[row0 + 1] = __ldcg(p.out + row0 + 1) + vb;
  } else if constexpr (EPI == EPI_RELU) {
    p.out[row0] = fmaxf(va, 0.0f);
    if (has_b) p.out[row0 + 1] = fmaxf(vb, 0.0f);
  } else if constexpr (EPI == EPI_SWIGLU) {
    const float s = va / (1.0f + expf(-va));
    p.out[pair] = s * vb;
  } else {  // EPI_QKV / EPI_QKV_ROPE
    const int d = p.d_model, dh = p.head_dim;
    const int pos = p.pos;
    const int sec = row0 / d;
    const int lp = pair - sec * (d >> 1);
    float ra = va, rb = vb;
    int e0, e1, head;
    if (EPI == EPI_QKV_ROPE && sec < 2) {
      const int half = dh >> 1;
      head = lp / half;
      const int i = lp - head * half;
      const float c = p.rope_cos[static_cast<int64_t>(pos) * half + i];
      const float s = p.rope_sin[static_cast<int64_t>(pos) * half + i];
      ra = va * c - vb * s;
      rb = vb * c + va * s;
      e0 = i;
      e1 = i + half;
    } else {
      const int e = 2 * lp;
      head = e / dh;
      e0 = e - head * dh;
      e1 = e0 + 1;
    }
    if (sec == 0) {
      p.q_out[head * dh + e0] = ra;
      p.q_out[head * dh + e1] = rb;
    } else {
      void* cache = sec == 1 ? p.k_cache : p.v_cache;
      const int64_t base = kv_row(p.kvp, head, p.max_seq, pos) * dh;
      if (p.kv_bf16) {
        store_cast(reinterpret_cast<__nv_bfloat16*>(cache) + base + e0, ra);
        store_cast(reinterpret_cast<__nv_bfloat16*>(cache) + base + e1, rb);
      } else {
        store_cast(reinterpret_cast<float*>(cache) + base + e0, ra);
        store_cast(reinterpret_cast<float*>(cache) + base + e1, rb);
      }
    }
  }
}

}  // namespace grt
