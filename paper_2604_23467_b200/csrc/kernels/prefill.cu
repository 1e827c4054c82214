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
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc05.cuh"

namespace grt {

// x[i][:] = emb[tokens[start+i]][:] (+ pos[start+i][:] in the reference arch,
// extend_position kernels.cpp:238-259; LLaMA: no position table)
template <typename WT>
__global__ void prefill_embed_kernel(const int* tokens, int start, int P, const WT* __restrict__ emb,
                                     const WT* __restrict__ pos, int d, float* __restrict__ X, int vocab, int* err) {
  griddep_launch_dependents();  // PDL successors wait for this grid before reading X
  const int i = blockIdx.x;
  if (i >= P) return;
  const int tok = tokens[start + i];
  if (tok < 0 || tok >= vocab) {
    if (threadIdx.x == 0 && err) atomicOr(err, DEVERR_TOKEN_RANGE);
    return;
  }
  const WT* row = emb + static_cast<int64_t>(tok) * d;
  const WT* prow = pos ? pos + static_cast<int64_t>(start + i) * d : nullptr;
  float* out = X + static_cast<int64_t>(i) * d;
  constexpr int U = 8;  // a thread's loads of the row issued together
  for (int j0 = threadIdx.x; j0 < d; j0 += U * blockDim.x) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * blockDim.x;
      v[u] = j < d ? to_f32(row[j]) + (prow ? to_f32(prow[j]) : 0.0f) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u * blockDim.x < d) out[j0 + u * blockDim.x] = v[u];
  }
}

// Xn[i] = bf16(rmsnorm(X[i]) * gamma): ss = sum x^2 ; inv = 1/sqrt(ss/d + eps).
// The row is pulled into registers with independent 16-byte loads (d <= 16 KB).
constexpr int PN_THREADS = 256, PN_MAXV = 16;  // d <= 16384
__global__ void __launch_bounds__(PN_THREADS) prefill_rmsnorm_kernel(const float* X, const float* gamma, float eps, int d,
                                                                     __nv_bfloat16* Xn) {
  griddep_launch_dependents();  // the next GEMM may start its weight stream
  __shared__ float red[32];
  const int i = blockIdx.x;
  const float4* x = reinterpret_cast<const float4*>(X + static_cast<int64_t>(i) * d);
  const int n4 = d >> 2;
  float4 v[PN_MAXV], g[PN_MAXV];
  float ss = 0.0f;
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) {
    const int j = threadIdx.x + u * PN_THREADS;
    v[u] = j < n4 ? x[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    g[u] = j < n4 ? reinterpret_cast<const float4*>(gamma)[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) ss = __fadd_rn(ss, sumsq4(v[u]));
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (PN_THREADS >> 5) ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / static_cast<float>(d) + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(Xn + static_cast<int64_t>(i) * d);
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) {
    const int j = threadIdx.x + u * PN_THREADS;
    if (j >= n4) continue;
    o[2 * j] = __floats2bfloat162_rn(v[u].x * inv * g[u].x, v[u].y * inv * g[u].y);
    o[2 * j + 1] = __floats2bfloat162_rn(v[u].z * inv * g[u].z, v[u].w * inv * g[u].w);
  }
}

// Xn[i] = bf16((X[i] - mean) / sqrt(var + eps) * gamma + beta): the reference
// arch's make_layernorm (kernels.cpp:52-85) for all P rows, one CTA per row.
__global__ void __launch_bounds__(PN_THREADS) prefill_layernorm_kernel(const float* X, const float* gamma,
                                                                       const float* beta, float eps, int d,
                                                                       __nv_bfloat16* Xn) {
  griddep_launch_dependents();
  __shared__ float red[32];
  const int i = blockIdx.x;
  const float4* x = reinterpret_cast<const float4*>(X + static_cast<int64_t>(i) * d);
  const int n4 = d >> 2;
  float4 v[PN_MAXV];
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) {
    const int j = threadIdx.x + u * PN_THREADS;
    v[u] = j < n4 ? x[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  auto block_sum = [&](float t) {
    t = warp_sum(t);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x < 32) {
      float a = threadIdx.x < (PN_THREADS >> 5) ? red[threadIdx.x] : 0.0f;
      a = warp_sum(a);
      if (threadIdx.x == 0) red[0] = a;
    }
    __syncthreads();
    return red[0];
  };
  float s = 0.0f;
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) s += (v[u].x + v[u].y) + (v[u].z + v[u].w);
  const float mean = block_sum(s) / static_cast<float>(d);
  float q = 0.0f;
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) {
    const int j = threadIdx.x + u * PN_THREADS;
    if (j >= n4) continue;
    const float a = v[u].x - mean, b = v[u].y - mean, c = v[u].z - mean, e = v[u].w - mean;
    q += (a * a + b * b) + (c * c + e * e);
  }
  const float inv = 1.0f / sqrtf(block_sum(q) / static_cast<float>(d) + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(Xn + static_cast<int64_t>(i) * d);
#pragma unroll
  for (int u = 0; u < PN_MAXV; ++u) {
    const int j = threadIdx.x + u * PN_THREADS;
    if (j >= n4) continue;
    const float4 g = reinterpret_cast<const float4*>(gamma)[j], b = reinterpret_cast<const float4*>(beta)[j];
    o[2 * j] = __floats2bfloat162_rn((v[u].x - mean) * inv * g.x + b.x, (v[u].y - mean) * inv * g.y + b.y);
    o[2 * j + 1] = __floats2bfloat162_rn((v[u].z - mean) * inv * g.z + b.z, (v[u].w - mean) * inv * g.w + b.w);
  }
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

// Causal prefill attention, flash style on CUDA cores: one CTA = one head x a
// block of PA_QB queries; key/value tiles of PA_KB rows are staged in shared
// memory once and reused by all PA_QB queries (instead of every query reading
// every key row from L2).  256 threads; thread (tq, tk) owns queries 4tq..4tq+3
// and keys tk + 16r (scores) / dims tk*DH/16.. (output), so every shared-memory
// load feeds 2-4 FMAs.  Online softmax per query row across key tiles.
constexpr int PA_QB = 64, PA_KB = 64, PA_THREADS = 256;

template <typename KT, int DH>
__global__ void __launch_bounds__(PA_THREADS)
    prefill_attn_kernel(const float* Q, const void* k_cache, const void* v_cache, int start, int P, int d,
                        int max_seq, float scale, __nv_bfloat16* out, KvPaging kvp) {
  griddep_launch_dependents();
  extern __shared__ __align__(16) float sm[];
  constexpr int KS = DH + 1;   // odd row stride: conflict-free column reads of K
  constexpr int DPT = DH / 16; // output dims per thread
  float* Qs = sm;                       // [QB][DH]
  float* Ks = Qs + PA_QB * DH;          // [KB][DH+1]
  float* Vs = Ks + PA_KB * KS;          // [KB][DH]
  float* Ps = Vs + PA_KB * DH;          // [QB][KB+1]
  const int head = blockIdx.y, q0 = blockIdx.x * PA_QB;
  const int t = threadIdx.x, tq = t >> 4, tk = t & 15;
  const int nq = min(PA_QB, P - q0);
  const KT* Kb = reinterpret_cast<const KT*>(k_cache);
  const KT* Vb = reinterpret_cast<const KT*>(v_cache);

  for (int e = t; e < PA_QB * DH; e += PA_THREADS) {
    const int qi = e / DH, dd = e - qi * DH;
    Qs[e] = qi < nq ? Q[static_cast<int64_t>(q0 + qi) * d + head * DH + dd] : 0.0f;
  }
  float m[4], l[4], o[4][DPT];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.0f;
#pragma unroll
    for (int j = 0; j < DPT; ++j) o[r][j] = 0.0f;
  }
  const int last_pos = start + q0 + nq - 1;
  for (int kb = 0; kb <= last_pos; kb += PA_KB) {
    __syncthreads();  // previous tile fully consumed (and Qs written, first time)
    for (int e = t; e < PA_KB * DH; e += PA_THREADS) {
      const int kk = e / DH, dd = e - kk * DH;
      const int pos = min(kb + kk, last_pos);
      const int64_t row = kv_row(kvp, head, max_seq, pos) * DH;
      Ks[kk * KS + dd] = to_f32(Kb[row + dd]);
      Vs[kk * DH + dd] = to_f32(Vb[row + dd]);
    }
    __syncthreads();
    // scores S[4 queries][4 keys]
    float sc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) sc[r][c] = 0.0f;
#pragma unroll 8
    for (int dd = 0; dd < DH; ++dd) {
      float qv[4], kv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) qv[r] = Qs[(4 * tq + r) * DH + dd];
#pragma unroll
      for (int c = 0; c < 4; ++c) kv[c] = Ks[(tk + 16 * c) * KS + dd];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) sc[r][c] = fmaf(qv[r], kv[c], sc[r][c]);
    }
    // scale, causal mask, online softmax (a query row lives in 16 lanes)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qpos = start + q0 + 4 * tq + r;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int kpos = kb + tk + 16 * c;
        sc[r][c] = (kpos <= qpos) ? sc[r][c] * scale : -INFINITY;
        mx = fmaxf(mx, sc[r][c]);
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mn = fmaxf(m[r], mx);
      const float f = (m[r] == -INFINITY || mn == -INFINITY) ? 0.0f : __expf(m[r] - mn);
      float rs = 0.0f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float pv = sc[r][c] == -INFINITY ? 0.0f : __expf(sc[r][c] - mn);
        Ps[(4 * tq + r) * (PA_KB + 1) + tk + 16 * c] = pv;
        rs += pv;
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      l[r] = l[r] * f + rs;
      m[r] = mn;
#pragma unroll
      for (int j = 0; j < DPT; ++j) o[r][j] *= f;
    }
    __syncwarp();  // Ps rows of this thread's queries are written by its own half-warp
    // O += P V
#pragma unroll 4
    for (int kk = 0; kk < PA_KB; ++kk) {
      float pv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pv[r] = Ps[(4 * tq + r) * (PA_KB + 1) + kk];
      float vv[DPT];
#pragma unroll
      for (int j = 0; j < DPT; ++j) vv[j] = Vs[kk * DH + tk * DPT + j];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < DPT; ++j) o[r][j] = fmaf(pv[r], vv[j], o[r][j]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = 4 * tq + r;
    if (qi >= nq) continue;
    const float inv = 1.0f / l[r];
    __nv_bfloat16* op = out + static_cast<int64_t>(q0 + qi) * d + head * DH + tk * DPT;
#pragma unroll
    for (int j = 0; j < DPT; ++j) op[j] = __float2bfloat16_rn(o[r][j] * inv);
  }
}

// decode hand-off: residual row of the last prompt token -> x, seq_len = len
__global__ void prefill_handoff_kernel(const float* X_last, int d, float* x, int* seq_len, int len) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;  // one element per thread: one memory round trip
  if (j < d) x[j] = X_last[j];
  if (j == 0) *seq_len = len;
}

// ---- host -----------------------------------------------------------------------

cudaError_t launch_prefill_embed(Dt wdt, const int* tokens, int start, int P, const void* emb, const void* pos, int d,
                                 float* X, int vocab, int* err, cudaStream_t s) {
  if (wdt == Dt::BF16)
    prefill_embed_kernel<<<P, 256, 0, s>>>(tokens, start, P, static_cast<const __nv_bfloat16*>(emb),
                                           static_cast<const __nv_bfloat16*>(pos), d, X, vocab, err);
  else
    prefill_embed_kernel<<<P, 256, 0, s>>>(tokens, start, P, static_cast<const float*>(emb),
                                           static_cast<const float*>(pos), d, X, vocab, err);
  return cudaGetLastError();
}

cudaError_t launch_prefill_layernorm(const float* X, int P, const float* gamma, const float* beta, float eps, int d,
                                     void* Xn, cudaStream_t s) {
  if (d % 4 != 0 || d > 4 * PN_MAXV * PN_THREADS || !beta) return cudaErrorInvalidValue;
  prefill_layernorm_kernel<<<P, PN_THREADS, 0, s>>>(X, gamma, beta, eps, d, static_cast<__nv_bfloat16*>(Xn));
  return cudaGetLastError();
}

cudaError_t launch_prefill_rmsnorm(const float* X, int P, const float* gamma, float eps, int d, void* Xn,
                                   cudaStream_t s) {
  if (d % 4 != 0 || d > 4 * PN_MAXV * PN_THREADS) return cudaErrorInvalidValue;
  prefill_rmsnorm_kernel<<<P, PN_THREADS, 0, s>>>(X, gamma, eps, d, static_cast<__nv_bfloat16*>(Xn));
  return cudaGetLastError();
}

// ---- tensor-core flash attention (bf16 KV), short prompts and head_dim 64 -----
// FA2-style on mma.sync.m16n8k16 (bf16 in, fp32 accumulate): a CTA = one head x
// 64 queries (4 warps x 16 rows); 64-key K/V tiles staged in shared memory
// (zero rows past the causal end); S = Q K^T and O += P V from ldmatrix
// fragments, the S accumulator re-packed in registers as the P operand; online
// softmax per row.  head_dim 128 with a full 128-key block goes to the tcgen05
// kernel below (prefill_fa_tc_kernel).
constexpr int FA_WARPS = 4, FA_QB = 64, FA_KB = 64;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 16-byte global -> shared copy (LDGSTS), zero-filled when !valid
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <int DH>
__global__ void __launch_bounds__(FA_WARPS * 32)
    prefill_fa_kernel(const float* Q, const __nv_bfloat16* k_cache, const __nv_bfloat16* v_cache, int start, int P,
                      int d, int max_seq, float scale, __nv_bfloat16* out, KvPaging kvp) {
  constexpr int LD = DH + 8;  // bf16 row stride: 16-byte aligned, conflict-free ldmatrix
  constexpr int KS = DH / 16, NB = DH / 8;
  griddep_launch_dependents();  // the Wo GEMM's CTAs may take the SMs this grid leaves free
  extern __shared__ __align__(16) uint8_t fa_smem[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(fa_smem);
  __nv_bfloat16* Kb = Qs + FA_QB * LD;      // [2][FA_KB][LD] double-buffered K tiles
  __nv_bfloat16* Vb = Kb + 2 * FA_KB * LD;  // [2][FA_KB][LD] V tiles
  // the q tiles with the most key blocks (causal) are scheduled first
  const int head = blockIdx.y, q0 = (gridDim.x - 1 - blockIdx.x) * FA_QB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int nq = min(FA_QB, P - q0);

  // Q (fp32) -> bf16: 16-byte loads, 8 in flight per thread
  constexpr int QV = FA_QB * DH / 4 / (FA_WARPS * 32);  // float4s per thread
#pragma unroll
  for (int h = 0; h < QV; h += 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + (h + u) * FA_WARPS * 32, r = e / (DH / 4), c = 4 * (e - r * (DH / 4));
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nq) v[u] = *reinterpret_cast<const float4*>(Q + static_cast<int64_t>(q0 + r) * d + head * DH + c);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = threadIdx.x + (h + u) * FA_WARPS * 32, r = e / (DH / 4), c = 4 * (e - r * (DH / 4));
      *reinterpret_cast<uint2*>(&Qs[r * LD + c]) = make_uint2(pack_bf16(v[u].x, v[u].y), pack_bf16(v[u].z, v[u].w));
    }
  }
  __syncthreads();
  uint32_t qf[KS][4];
  {
    const int r = 16 * warp + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int c = (lane >> 4) * 8;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
      ldsm_x4(smem_u32(&Qs[r * LD + 16 * ks + c]), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float o[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0f;
  const int qpos0 = start + q0 + 16 * warp + g;  // rows g and g+8 of this warp
  const int last_pos = start + q0 + nq - 1;

  // K/V tiles stream in with cp.async, double-buffered: the next tile's loads
  // are in flight while this one's MMAs run (rows past the live end are
  // zero-filled: their scores are masked, and 0 * V must stay finite)
  auto load_kv = [&](int kb, int buf) {
    __nv_bfloat16* Ks = Kb + buf * FA_KB * LD;
    __nv_bfloat16* Vs = Vb + buf * FA_KB * LD;
    for (int e = threadIdx.x; e < FA_KB * DH / 8; e += FA_WARPS * 32) {
      const int r = e / (DH / 8), c = 8 * (e - r * (DH / 8));
      const bool ok = kb + r <= last_pos;
      const int64_t row = ok ? kv_row(kvp, head, max_seq, kb + r) * DH : 0;
      cp_async16(&Ks[r * LD + c], k_cache + row + c, ok);
      cp_async16(&Vs[r * LD + c], v_cache + row + c, ok);
    }
    cp_async_commit();
  };
  load_kv(0, 0);
  for (int kb = 0, it = 0; kb <= last_pos; kb += FA_KB, ++it) {
    const int buf = it & 1;
    const bool more = kb + FA_KB <= last_pos;
    if (more) load_kv(kb + FA_KB, buf ^ 1);  // that buffer was released by the barrier ending the last iteration
    if (more)
      cp_async_wait<1>();
    else
      cp_async_wait<0>();
    __syncthreads();
    const __nv_bfloat16* Ks = Kb + buf * FA_KB * LD;
    const __nv_bfloat16* Vs = Vb + buf * FA_KB * LD;
    float sacc[FA_KB / 8][4];
#pragma unroll
    for (int nb = 0; nb < FA_KB / 8; ++nb) sacc[nb][0] = sacc[nb][1] = sacc[nb][2] = sacc[nb][3] = 0.0f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int nb = 0; nb < FA_KB / 8; nb += 2) {
        // matrices: (keys 8nb.., dh 16ks..), (keys 8nb.., dh 16ks+8..), then nb+1
        const int r = 8 * nb + (lane & 7) + (lane >> 4) * 8;
        const int c = 16 * ks + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(&Ks[r * LD + c]), b0, b1, b2, b3);
        mma_bf16(sacc[nb], qf[ks], b0, b1);
        mma_bf16(sacc[nb + 1], qf[ks], b2, b3);
      }
    }
    // scale, causal mask, online softmax over rows g (i=0) and g+8 (i=1)
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nb = 0; nb < FA_KB / 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = e >> 1;
        const int key = kb + 8 * nb + 2 * t + (e & 1);
        const float v = key <= qpos0 + 8 * i ? sacc[nb][e] * scale : -INFINITY;
        sacc[nb][e] = v;
        mx[i] = fmaxf(mx[i], v);
      }
    float f[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
      mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
      const float mn = fmaxf(m[i], mx[i]);
      f[i] = (m[i] == -INFINITY) ? 0.0f : __expf(m[i] - mn);
      m[i] = mn;
      l[i] *= f[i];
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      o[j][0] *= f[0];
      o[j][1] *= f[0];
      o[j][2] *= f[1];
      o[j][3] *= f[1];
    }
#pragma unroll
    for (int nb = 0; nb < FA_KB / 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = e >> 1;
        const float pv = sacc[nb][e] == -INFINITY ? 0.0f : __expf(sacc[nb][e] - m[i]);
        sacc[nb][e] = pv;
        l[i] += pv;
      }
    // O += P V  (P re-packed from the S accumulators as m16n8k16 A fragments)
#pragma unroll
    for (int kk = 0; kk < FA_KB / 16; ++kk) {
      const uint32_t a[4] = {pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]), pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]),
                             pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]),
                             pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3])};
#pragma unroll
      for (int jn = 0; jn < NB; jn += 2) {
        // transposed matrices: (keys 16kk.., dh 8jn..), (keys 16kk+8.., dh 8jn..), then dh 8jn+8
        const int r = 16 * kk + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = 8 * jn + (lane >> 4) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_u32(&Vs[r * LD + c]), b0, b1, b2, b3);
        mma_bf16(o[jn], a, b0, b1);
        mma_bf16(o[jn + 1], a, b2, b3);
      }
    }
    __syncthreads();  // every warp is done with `buf` before it is refilled
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    l[i] += __shfl_xor_sync(0xffffffffu, l[i], 1);
    l[i] += __shfl_xor_sync(0xffffffffu, l[i], 2);
  }
  const int r0 = 16 * warp + g;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + 8 * i;
    if (r >= nq) continue;
    const float inv = 1.0f / l[i];
    __nv_bfloat16* op = out + static_cast<int64_t>(q0 + r) * d + head * DH + 2 * t;
#pragma unroll
    for (int j = 0; j < NB; ++j)
      *reinterpret_cast<__nv_bfloat162*>(op + 8 * j) = __floats2bfloat162_rn(o[j][2 * i] * inv, o[j][2 * i + 1] * inv);
  }
}

// ---- causal attention on the 5th-generation tensor cores (head_dim 128) ------
// One CTA = 128 queries of one head, 4 warps; warp w owns TMEM lanes 32w..32w+31,
// i.e. thread = query row.  Per 128-key block:
//   S = Q K^T     tcgen05.mma (M=128 queries, N=128 keys, K=head_dim) -> TMEM cols [0,128)
//   softmax       the thread's S row in 4 tcgen05.ld x32 (one wait), online max /
//                 sum in the log2 domain (ft_softmax), P (bf16) into shared memory
//                 as the next A operand
//   O += P V      tcgen05.mma (M=128 queries, N=128 head_dim, K=128 keys) into the
//                 TMEM accumulator, cols [128,256); when a row's reference max
//                 moves, the warp rescales its rows in place (tcgen05.ld/st).
// The next block's S MMA is issued before this block's P V is waited on.
// Q, K, V and P tiles are [128][128] bf16 in the K-major 128-byte swizzled layout
// (two [128][64] halves).  K and V are both copied row by row (key = row, head
// dim contiguous) with 16-byte cp.async through the page table; V is therefore
// the MN-major B operand of the second MMA (N = head dim contiguous).  The next
// block's K/V copies overlap this block's MMAs and softmax.
constexpr int FT_ROWS = 128, FT_THREADS = 128;
constexpr uint32_t FT_TILE = FT_ROWS * 128 * 2;  // 32 KB

// byte offset of element (row r, col c) of a [128][128] bf16 tile, 128-byte swizzle
__device__ __forceinline__ uint32_t ft_off(int r, int c) {
  return static_cast<uint32_t>((c >> 6) * (FT_TILE / 2) + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + (c & 7) * 2);
}

// 32 consecutive fp32 columns of this thread's TMEM lane; no wait (batch several,
// then tc_wait_ld once)
#define FT_R32(r) "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
    "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),          \
    "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),        \
    "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define FT_W32(r) "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), \
    "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),      \
    "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),      \
    "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
__device__ __forceinline__ void tc_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : FT_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tc_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      FT_W32(r)
      : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Online-softmax update of one query row over a 128-key block (log2 domain).
// m = the row's reference max of s * sl2, moved only when the block max exceeds
// it by more than FT_RESCALE (FlashAttention-4's conditional rescale: P values
// up to 2^FT_RESCALE are exact in fp32/bf16 range, and most blocks then leave
// the output accumulator alone); alpha = exp2(m_old - m_new) (1 if unmoved);
// P = exp2(s * sl2 - m) as bf16 into the swizzled P tile; ls = sum of this
// block's P.  MASK: keys c > lim are masked out (causal diagonal).  Independent
// partial max / sum accumulators keep the dependency chains short.
constexpr float FT_RESCALE = 8.0f;
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <bool MASK>
__device__ __forceinline__ void ft_softmax(const uint32_t (&s)[128], int lim, float sl2, float& m, float& alpha,
                                           float& ls, uint8_t* Ps, int r) {
  float mx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) mx[k] = -INFINITY;
#pragma unroll
  for (int i = 0; i < 128; ++i) {
    const float v = __uint_as_float(s[i]);
    if (!MASK || i <= lim) mx[i & 7] = fmaxf(mx[i & 7], v);
  }
  const float bm = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
  const float cand = bm * sl2;
  alpha = 1.0f;
  if (m == -INFINITY) {
    m = cand;  // first block (key 0 is visible to every row)
  } else if (cand > m + FT_RESCALE) {
    alpha = ex2_approx(m - cand);
    m = cand;
  }
  const float mn = m;
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
#pragma unroll
  for (int cc = 0; cc < 16; ++cc) {
    uint32_t pk[4];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const int c = 8 * cc + i;
      float p0 = ex2_approx(fmaf(__uint_as_float(s[c]), sl2, -mn));
      float p1 = ex2_approx(fmaf(__uint_as_float(s[c + 1]), sl2, -mn));
      if (MASK) {
        p0 = c <= lim ? p0 : 0.0f;
        p1 = c + 1 <= lim ? p1 : 0.0f;
      }
      acc[i] += p0;
      acc[i + 1] += p1;
      pk[i / 2] = pack_bf16(p0, p1);
    }
    *reinterpret_cast<uint4*>(Ps + ft_off(r, 8 * cc)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  ls = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

__global__ void __launch_bounds__(FT_THREADS, 1)
    prefill_fa_tc_kernel(const float* Q, const __nv_bfloat16* k_cache, const __nv_bfloat16* v_cache, int start, int P,
                          int d, int max_seq, float scale, __nv_bfloat16* out, KvPaging kvp) {
  griddep_launch_dependents();  // the Wo GEMM's CTAs may take the SMs this grid leaves free
  extern __shared__ __align__(1024) uint8_t ft_raw[];
  __shared__ uint64_t bar_s, bar_o;
  __shared__ uint32_t tmem_base;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ft_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = sm;
  uint8_t* Ks = sm + FT_TILE;
  uint8_t* Vs = sm + 3 * FT_TILE;
  uint8_t* Ps = sm + 5 * FT_TILE;
  const int head = blockIdx.y, q0 = (gridDim.x - 1 - blockIdx.x) * FT_ROWS;
  const int tid = threadIdx.x, warp = tid >> 5, r = tid;
  const int nq = min(FT_ROWS, P - q0);
  const int last_pos = start + q0 + nq - 1;
  const int qpos = start + q0 + r;

  if (tid == 0) {
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // K/V copies: thread = one 16-byte column chunk of rows tid/16 + 8i, so its
  // swizzled shared offset is fixed up to i * 1024 B
  const int ld_row = tid >> 4, ld_c = (tid & 15) * 8;
  const uint32_t ld_off = ft_off(ld_row, ld_c);
  auto load_kv = [&](int kb, int buf) {
    uint8_t* ks = Ks + buf * FT_TILE + ld_off;
    uint8_t* vs = Vs + buf * FT_TILE + ld_off;
    if (kvp.page == 0) {
      const int64_t g0 = (static_cast<int64_t>(head) * max_seq + kb + ld_row) * 128 + ld_c;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const bool ok = kb + ld_row + 8 * i <= last_pos;
        const int64_t g = ok ? g0 + i * 1024 : 0;
        cp_async16(ks + i * 1024, k_cache + g, ok);
        cp_async16(vs + i * 1024, v_cache + g, ok);
      }
    } else {
      for (int i = 0; i < 16; ++i) {
        const bool ok = kb + ld_row + 8 * i <= last_pos;
        const int64_t g = ok ? kv_row(kvp, head, max_seq, kb + ld_row + 8 * i) * 128 + ld_c : 0;
        cp_async16(ks + i * 1024, k_cache + g, ok);
        cp_async16(vs + i * 1024, v_cache + g, ok);
      }
    }
    cp_async_commit();
  };
  load_kv(0, 0);
  // Q (fp32, just written by the QKV GEMM) -> bf16 tile: 8 rows' loads in flight per thread
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float4 a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + (8 * h + u) * FT_THREADS, row = e >> 4, c = (e & 15) * 8;
      a[u] = b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < nq) {
        const float4* src = reinterpret_cast<const float4*>(Q + static_cast<int64_t>(q0 + row) * d + head * 128 + c);
        a[u] = src[0];
        b[u] = src[1];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + (8 * h + u) * FT_THREADS, row = e >> 4, c = (e & 15) * 8;
      *reinterpret_cast<uint4*>(Qs + ft_off(row, c)) = make_uint4(pack_bf16(a[u].x, a[u].y), pack_bf16(a[u].z, a[u].w),
                                                                  pack_bf16(b[u].x, b[u].y), pack_bf16(b[u].z, b[u].w));
    }
  }
  const uint32_t sQ = smem_u32(Qs), sK = smem_u32(Ks), sV = smem_u32(Vs), sP = smem_u32(Ps);
  constexpr uint32_t idesc_s = idesc_bf16(128), idesc_o = idesc_bf16(128) | IDESC_B_MN_MAJOR;
  const float sl2 = scale * 1.4426950408889634f;  // scores in log2 units: p = exp2(s * sl2 - m)
  float m = -INFINITY, l = 0.0f;
  int j = 0;
  for (int kb = 0; kb <= last_pos; kb += FT_ROWS, ++j) {
    const int buf = j & 1;
    cp_async_wait<0>();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base + (static_cast<uint32_t>(32 * warp) << 16);
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t off = (ks >> 2) * (FT_TILE / 2) + (ks & 3) * 32;
        tc_mma_bf16(tmem_base, sw128_desc(sQ + off), sw128_desc(sK + buf * FT_TILE + off), idesc_s, ks > 0);
      }
      tc_commit(&bar_s);
    }
    if (j > 0) mbar_wait(&bar_o, (j - 1) & 1);  // P V of block j-1: Ps and buffer buf^1 free, O settled
    if (kb + FT_ROWS <= last_pos) load_kv(kb + FT_ROWS, buf ^ 1);
    mbar_wait(&bar_s, j & 1);
    tc_fence_after();
    uint32_t s[128];  // this query's 128 scores: 4 TMEM loads in flight, one wait
#pragma unroll
    for (int q = 0; q < 4; ++q) tc_ld32_nowait(tm + 32 * q, s + 32 * q);
    tc_wait_ld();
    float alpha, ls;
    if (kb + FT_ROWS - 1 <= start + q0)  // block entirely below the diagonal for every row: no mask
      ft_softmax<false>(s, 0, sl2, m, alpha, ls, Ps, r);
    else
      ft_softmax<true>(s, qpos - kb, sl2, m, alpha, ls, Ps, r);
    l = l * alpha + ls;
    if (j > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {  // rescale the running output in TMEM
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v[64];
        tc_ld32_nowait(tm + 128 + 64 * h, v);
        tc_ld32_nowait(tm + 128 + 64 * h + 32, v + 32);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 64; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
        tc_st32(tm + 128 + 64 * h, v);
        tc_st32(tm + 128 + 64 * h + 32, v + 32);
      }
      tc_wait_st();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint32_t pa = (ks >> 2) * (FT_TILE / 2) + (ks & 3) * 32;
        tc_mma_bf16(tmem_base + 128, sw128_desc(sP + pa), sw128_desc_mn(sV + buf * FT_TILE + ks * 2048, FT_TILE / 2, 1024),
                    idesc_o, (j > 0 || ks > 0) ? 1u : 0u);
      }
      tc_commit(&bar_o);
    }
  }
  mbar_wait(&bar_o, (j - 1) & 1);
  tc_fence_after();
  const uint32_t tm = tmem_base + (static_cast<uint32_t>(32 * warp) << 16);
  const float inv = 1.0f / l;
  uint4* op = reinterpret_cast<uint4*>(out + static_cast<int64_t>(q0 + r) * d + head * 128);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t v[64];
    tc_ld32_nowait(tm + 128 + 64 * h, v);
    tc_ld32_nowait(tm + 128 + 64 * h + 32, v + 32);
    tc_wait_ld();
    if (r < nq) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float* f = reinterpret_cast<const float*>(v + 8 * c);
        op[8 * h + c] = make_uint4(pack_bf16(f[0] * inv, f[1] * inv), pack_bf16(f[2] * inv, f[3] * inv),
                                   pack_bf16(f[4] * inv, f[5] * inv), pack_bf16(f[6] * inv, f[7] * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256) : "memory");
  }
}

static cudaError_t fa_tc_launch(const float* Q, const void* k, const void* v, int start, int P, int d, int n_heads,
                                int max_seq, float scale, void* out, cudaStream_t s, KvPaging kvp) {
  const size_t smem = 6 * FT_TILE + 1024;  // Q, 2 x K, 2 x V, P tiles + 1 KB alignment slack
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_fa_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((P + FT_ROWS - 1) / FT_ROWS, n_heads);
  prefill_fa_tc_kernel<<<grid, FT_THREADS, smem, s>>>(Q, static_cast<const __nv_bfloat16*>(k),
                                                      static_cast<const __nv_bfloat16*>(v), start, P, d, max_seq, scale,
                                                      static_cast<__nv_bfloat16*>(out), kvp);
  return cudaGetLastError();
}

template <typename KT, int DH>
static cudaError_t attn_launch(const float* Q, const void* k, const void* v, int start, int P, int d, int n_heads,
                               int max_seq, float scale, void* out, cudaStream_t s, KvPaging kvp) {
  const size_t smem = (static_cast<size_t>(PA_QB) * DH + PA_KB * (DH + 1) + PA_KB * DH + PA_QB * (PA_KB + 1)) * 4;
  static bool attr_set = false;  // idempotent
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_kernel<KT, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((P + PA_QB - 1) / PA_QB, n_heads);
  prefill_attn_kernel<KT, DH><<<grid, PA_THREADS, smem, s>>>(Q, k, v, start, P, d, max_seq, scale,
                                                               static_cast<__nv_bfloat16*>(out), kvp);
  return cudaGetLastError();
}

template <typename KT>
static cudaError_t attn_dispatch(int dh, const float* Q, const void* k, const void* v, int start, int P, int d,
                                 int n_heads, int max_seq, float scale, void* out, cudaStream_t s, KvPaging kvp) {
  switch (dh) {
    case 16: return attn_launch<KT, 16>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    case 32: return attn_launch<KT, 32>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    case 64: return attn_launch<KT, 64>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    case 128: return attn_launch<KT, 128>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    default: return cudaErrorInvalidValue;
  }
}

template <int DH>
static cudaError_t fa_launch(const float* Q, const void* k, const void* v, int start, int P, int d, int n_heads,
                             int max_seq, float scale, void* out, cudaStream_t s, KvPaging kvp) {
  const size_t smem = static_cast<size_t>(FA_QB + 4 * FA_KB) * (DH + 8) * 2;  // Q + 2 x (K, V)
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_fa_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((P + FA_QB - 1) / FA_QB, n_heads);
  prefill_fa_kernel<DH><<<grid, FA_WARPS * 32, smem, s>>>(Q, static_cast<const __nv_bfloat16*>(k),
                                                        static_cast<const __nv_bfloat16*>(v), start, P, d, max_seq,
                                                        scale, static_cast<__nv_bfloat16*>(out), kvp);
  return cudaGetLastError();
}

cudaError_t launch_prefill_attention(Dt kvdt, const float* Q, const void* k, const void* v, int start, int P, int d,
                                     int n_heads, int dh, int max_seq, float scale, void* out, cudaStream_t s,
                                     KvPaging kvp) {
  if (kvdt == Dt::BF16) {  // tensor cores for bf16 KV
    // tcgen05 once there is a full 128-key block to attend over; a short prompt's
    // single partial tile is cheaper on the mma.sync kernel's 64 x 64 tiles
    if (dh == 128 && start + P >= FT_ROWS) return fa_tc_launch(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    if (dh == 64) return fa_launch<64>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    if (dh == 128) return fa_launch<128>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
  }
  if (kvdt == Dt::BF16) return attn_dispatch<__nv_bfloat16>(dh, Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
  return attn_dispatch<float>(dh, Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
}

cudaError_t launch_prefill_handoff(const float* X_last, int d, float* x, int* seq_len, int len, cudaStream_t s) {
  prefill_handoff_kernel<<<(d + 255) / 256, 256, 0, s>>>(X_last, d, x, seq_len, len);
  return cudaGetLastError();
}

}  // namespace grt
