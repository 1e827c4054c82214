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

// Xn[i] = bf16(rmsnorm(X[i]) * gamma): ss = sum x^2 ; inv = 1/sqrt(ss/d + eps).
// The row is pulled into registers with independent 16-byte loads (d <= 16 KB).
constexpr int PN_THREADS = 256, PN_MAXV = 16;  // d <= 16384
__global__ void __launch_bounds__(PN_THREADS) prefill_rmsnorm_kernel(const float* X, const float* gamma, float eps, int d,
                                                                     __nv_bfloat16* Xn) {
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
  if (d % 4 != 0 || d > 4 * PN_MAXV * PN_THREADS) return cudaErrorInvalidValue;
  prefill_rmsnorm_kernel<<<P, PN_THREADS, 0, s>>>(X, gamma, eps, d, static_cast<__nv_bfloat16*>(Xn));
  return cudaGetLastError();
}

// ---- tensor-core flash attention (bf16 KV) ------------------------------------
// FA2-style on mma.sync.m16n8k16 (bf16 in, fp32 accumulate): a CTA = one head x
// 64 queries (4 warps x 16 rows); 64-key K/V tiles staged in shared memory
// (zero rows past the causal end); S = Q K^T and O += P V from ldmatrix
// fragments, the S accumulator re-packed in registers as the P operand; online
// softmax per row.  Attention is ~1% of the prefill flops, so the
// legacy tensor path is enough here; the projections are the tcgen05 GEMMs.
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
  extern __shared__ __align__(16) uint8_t fa_smem[];
  __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(fa_smem);
  __nv_bfloat16* Kb = Qs + FA_QB * LD;      // [2][FA_KB][LD] double-buffered K tiles
  __nv_bfloat16* Vb = Kb + 2 * FA_KB * LD;  // [2][FA_KB][LD] V tiles
  // the q tiles with the most key blocks (causal) are scheduled first
  const int head = blockIdx.y, q0 = (gridDim.x - 1 - blockIdx.x) * FA_QB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int nq = min(FA_QB, P - q0);

  for (int e = threadIdx.x; e < FA_QB * DH / 2; e += FA_WARPS * 32) {
    const int r = e / (DH / 2), c = 2 * (e - r * (DH / 2));
    float2 v = make_float2(0.f, 0.f);
    if (r < nq) v = *reinterpret_cast<const float2*>(Q + static_cast<int64_t>(q0 + r) * d + head * DH + c);
    *reinterpret_cast<__nv_bfloat162*>(&Qs[r * LD + c]) = __floats2bfloat162_rn(v.x, v.y);
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
    if (dh == 64) return fa_launch<64>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
    if (dh == 128) return fa_launch<128>(Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
  }
  if (kvdt == Dt::BF16) return attn_dispatch<__nv_bfloat16>(dh, Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
  return attn_dispatch<float>(dh, Q, k, v, start, P, d, n_heads, max_seq, scale, out, s, kvp);
}

cudaError_t launch_prefill_handoff(const float* X_last, int d, float* x, int* seq_len, int len, cudaStream_t s) {
  prefill_handoff_kernel<<<1, 256, 0, s>>>(X_last, d, x, seq_len, len);
  return cudaGetLastError();
}

}  // namespace grt
