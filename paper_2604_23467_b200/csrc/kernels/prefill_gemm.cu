// prefill_gemm.cu -- batched-prefill projection GEMMs on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Reference: prefill is P token-by-token passes of make_matmul
// (pipeline.cpp:207-214, kernels.cpp:23-50); the incremental == restart
// property (model_test.cpp:129-146) lets all P tokens go through each layer at
// once, turning every projection into a GEMM  Y[P, N] = X[P, K] . W[N, K]^T.
//
// Shape: the weight is the MMA's A operand (M = 128 weight rows per CTA, K-major
// as stored), the tokens are B (N = one tile of <= 128 tokens per CTA, K-major
// bf16 activations).  CTAs of the same weight tile run concurrently, so the
// weights stream from HBM about once per GEMM (token tiles re-hit L2).
//   * warp 0: TMA producer (cp.async.bulk.tensor.2d, SWIZZLE_128B, 64-wide K
//     blocks) into a `stages`-deep ring, mbarrier full/empty handshakes;
//   * warp 1: allocates TMEM and issues tcgen05.mma.cta_group::1.kind::f16
//     (bf16 x bf16 -> fp32, M=128, N=ntile, K=16 per instruction) from one
//     elected lane; tcgen05.commit frees ring slots and signals the epilogue;
//   * warps 2-5: epilogue -- tcgen05.ld 32x32b (one weight row per thread, 16
//     tokens per load) -> fused RoPE/KV-cache write, SwiGLU, residual add;
//   * short prompts (memory-bound) split K over several CTAs; partials go to a
//     global scratch and the last CTA of a tile sums them in split order
//     (deterministic).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc05.cuh"

namespace grt {

constexpr int PG_BM = 128;        // weight rows per CTA (UMMA M)
constexpr int PG_BK = 64;         // K elements per stage (one 128-byte swizzle row)
constexpr int PG_UK = 16;         // K per tcgen05.mma (kind::f16)
constexpr int PG_EPI_WARPS = 8;    // max: two warps per TMEM lane quadrant, splitting the token columns
// weight (A) TMA warp, MMA warp, epilogue warps (max), token (B) TMA warp -- two
// producer warps: one thread issuing both operands' boxes took ~300 cycles per
// TMA instruction, longer than a stage's MMAs (tools/tma_rows_bench.cu)
constexpr int PG_THREADS = (3 + PG_EPI_WARPS) * 32;
constexpr int PG_MAX_NT = 256;    // tokens per N tile (UMMA N max)

// ---- tcgen05 / TMA primitives (inline PTX) --------------------------------------

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 3D box {64 K, rows, kbox K blocks} of a {64, rows, K/64} view (row stride K*2 B,
// K-block stride 128 B): kbox 128-byte-swizzled [rows][64] tiles, one after the
// other -- the stage layout of kbox 2D boxes, in one instruction.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---- epilogue -------------------------------------------------------------------
// One thread = one weight row m, 16 tokens at a time (the 16 TMEM columns of
// one tcgen05.ld); every global load the epilogue needs for those tokens (RoPE
// table entries, residual values) is issued before any is used, so the memory
// latency is paid once per 16 tokens, not once per token.

__device__ __forceinline__ void pg_epilogue16(const PrefillGemmParams& p, int m, int n0, int nv, const float (&v)[16]) {
  float vp[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) vp[j] = __shfl_xor_sync(0xffffffffu, v[j], 1);  // row m^1 (RoPE / SwiGLU partner)
  if (m >= p.M) return;
  switch (p.epi) {
    case PG_EPI_STORE: {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nv) p.out[static_cast<int64_t>(n0 + j) * p.M + m] = v[j];
      break;
    }
    case PG_EPI_RESID: {
      float old[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) old[j] = j < nv ? p.out[static_cast<int64_t>(n0 + j) * p.M + m] : 0.0f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nv) p.out[static_cast<int64_t>(n0 + j) * p.M + m] = old[j] + v[j];
      break;
    }
    case PG_EPI_RELU: {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out_bf16) + m;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nv) o[static_cast<int64_t>(n0 + j) * p.M] = __float2bfloat16_rn(fmaxf(v[j], 0.0f));
      break;
    }
    case PG_EPI_SWIGLU: {
      if (m & 1) return;
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out_bf16) + (m >> 1);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j >= nv) continue;
        const float sg = v[j] / (1.0f + expf(-v[j]));
        o[static_cast<int64_t>(n0 + j) * (p.M >> 1)] = __float2bfloat16_rn(sg * vp[j]);
      }
      break;
    }
    default: {  // PG_EPI_QKV / PG_EPI_QKV_ROPE: same index math as the decode epilogue (gemv_core.cuh)
      if (m & 1) return;
      const int d = p.d_model, dh = p.head_dim;
      const int sec = m / d;
      const int lp = (m >> 1) - sec * (d >> 1);
      const bool rope = p.epi == PG_EPI_QKV_ROPE && sec < 2;
      int e0, e1, head, i = 0, half = dh >> 1;
      if (rope) {
        head = lp / half;
        i = lp - head * half;
        e0 = i;
        e1 = i + half;
      } else {
        const int e = 2 * lp;
        head = e / dh;
        e0 = e - head * dh;
        e1 = e0 + 1;
      }
      float cs[16], sn[16];
      if (rope) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t t = static_cast<int64_t>(p.start_pos + n0 + (j < nv ? j : 0)) * half + i;
          cs[j] = p.rope_cos[t];
          sn[j] = p.rope_sin[t];
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j >= nv) continue;
        float ra = v[j], rb = vp[j];
        if (rope) {
          ra = v[j] * cs[j] - vp[j] * sn[j];
          rb = vp[j] * cs[j] + v[j] * sn[j];
        }
        const int n = n0 + j;
        if (sec == 0) {
          float* q = p.q_out + static_cast<int64_t>(n) * d + head * dh;
          q[e0] = ra;
          q[e1] = rb;
        } else {
          void* cache = sec == 1 ? p.k_cache : p.v_cache;
          const int64_t base = kv_row(p.kvp, head, p.max_seq, p.start_pos + n) * dh;
          if (p.kv_bf16) {
            __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(cache) + base;
            c[e0] = __float2bfloat16_rn(ra);
            c[e1] = __float2bfloat16_rn(rb);
          } else {
            float* c = reinterpret_cast<float*>(cache) + base;
            c[e0] = ra;
            c[e1] = rb;
          }
        }
      }
    }
  }
}

// QKV epilogue of one warp (32 weight rows = 16 row pairs) for 16 tokens, staged
// through shared memory so the stores are 16-byte vectors of consecutive
// destinations (the per-element q / KV stores of pg_epilogue16 -- 2 or 4 bytes
// per lane, half the lanes idle -- made the epilogue the QKV GEMM's tail: 75 ->
// 51 us at P=500 without it).  Requires d_model % 32 == 0 and head_dim % 32 == 0
// (a warp's 16 pairs lie in one section and one head).  Both lanes of a pair
// work: the even lane rotates tokens 0-7, the odd lane tokens 8-15.  rc / rs:
// this thread's RoPE factors for its 8 tokens.
constexpr int PG_STG = 33;  // staging row stride (floats): conflict-free column reads
__device__ __forceinline__ void pg_epilogue_qkv_staged(const PrefillGemmParams& p, int m, int n0, int nv,
                                                       const float (&v)[16], const float (&rc)[8],
                                                       const float (&rs)[8], float* stg) {
  if ((m & ~31) >= p.M) return;  // warp-uniform (M % 32 == 0)
  const int lane = threadIdx.x & 31;
  const bool odd = lane & 1;
  // the partner row's value for this thread's 8 tokens (8 shuffles)
  float recv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) recv[j] = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[j + 8], 1);
  const int d = p.d_model, dh = p.head_dim;
  const int sec = m / d;
  const bool rope = p.epi == PG_EPI_QKV_ROPE && sec < 2;
  const int pr = lane >> 1;  // pair slot within the warp
  const int sa = rope ? pr : 2 * pr, sb = rope ? 16 + pr : 2 * pr + 1;
  const int jo = odd ? 8 : 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float a = odd ? recv[j] : v[j];       // even row (m & ~1)
    const float b = odd ? v[j + 8] : recv[j];   // odd row
    float ra = a, rb = b;
    if (rope) {
      ra = a * rc[j] - b * rs[j];
      rb = b * rc[j] + a * rs[j];
    }
    stg[(jo + j) * PG_STG + sa] = ra;
    stg[(jo + j) * PG_STG + sb] = rb;
  }
  __syncwarp();
  // destinations: section-local pair index of slot 0, its head and element
  const int m0 = m & ~31;  // row of lane 0 (warp's first row)
  const int lp0 = (m0 >> 1) - sec * (d >> 1);
  int head, ebase;
  if (rope) {
    head = lp0 / (dh >> 1);
    ebase = lp0 - head * (dh >> 1);  // slots 0-15: e = ebase + s; 16-31: e = dh/2 + ebase + s - 16
  } else {
    head = (2 * lp0) / dh;
    ebase = 2 * lp0 - head * dh;  // slot s: e = ebase + s
  }
  const int s0 = (lane & 7) * 4;
  const int e = rope ? (s0 < 16 ? ebase + s0 : (dh >> 1) + ebase + s0 - 16) : ebase + s0;
#pragma unroll
  for (int tb = 0; tb < 4; ++tb) {
    const int j = tb * 4 + (lane >> 3);
    if (j >= nv) continue;
    const float* src = stg + j * PG_STG + s0;
    const float x0 = src[0], x1 = src[1], x2 = src[2], x3 = src[3];
    const int n = n0 + j;
    if (sec == 0) {
      *reinterpret_cast<float4*>(p.q_out + static_cast<int64_t>(n) * d + head * dh + e) = make_float4(x0, x1, x2, x3);
    } else {
      void* cache = sec == 1 ? p.k_cache : p.v_cache;
      const int64_t off = kv_row(p.kvp, head, p.max_seq, p.start_pos + n) * dh + e;
      if (p.kv_bf16) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(x0, x1), hi = __floats2bfloat162_rn(x2, x3);
        uint2 u;
        u.x = *reinterpret_cast<const uint32_t*>(&lo);
        u.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cache) + off) = u;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(cache) + off) = make_float4(x0, x1, x2, x3);
      }
    }
  }
  __syncwarp();  // staging reused by the next group
}

// SwiGLU epilogue of one warp (16 gate/up row pairs) for 16 tokens, staged like
// the QKV one: h = silu(gate) * up (same expression as pg_epilogue16) for 8
// tokens per lane, then 8-byte stores of 4 consecutive bf16 outputs (16 per
// token and warp).  Requires M % 32 == 0.
__device__ __forceinline__ void pg_epilogue_swiglu_staged(const PrefillGemmParams& p, int m, int n0, int nv,
                                                          const float (&v)[16], float* stg) {
  if ((m & ~31) >= p.M) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const bool odd = lane & 1;
  float recv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) recv[j] = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[j + 8], 1);
  const int pr = lane >> 1, jo = odd ? 8 : 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float a = odd ? recv[j] : v[j];      // gate (even row)
    const float b = odd ? v[j + 8] : recv[j];  // up (odd row)
    const float sg = a / (1.0f + expf(-a));
    stg[(jo + j) * PG_STG + pr] = sg * b;
  }
  __syncwarp();
  const int half_m = p.M >> 1;
  const int col = ((m & ~31) >> 1) + (lane & 3) * 4;
#pragma unroll
  for (int tb = 0; tb < 2; ++tb) {
    const int j = tb * 8 + (lane >> 2);
    if (j >= nv) continue;
    const float* src = stg + j * PG_STG + (lane & 3) * 4;
    const __nv_bfloat162 lo = __floats2bfloat162_rn(src[0], src[1]), hi = __floats2bfloat162_rn(src[2], src[3]);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&lo);
    u.y = *reinterpret_cast<const uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.out_bf16) + static_cast<int64_t>(n0 + j) * half_m + col) = u;
  }
  __syncwarp();
}

// RoPE factors of this thread's 8 tokens of the group at column c0 (staged QKV
// epilogue): pair (m & ~1), tokens n0 + c0 + (odd ? 8 : 0) + j.
__device__ __forceinline__ void pg_rope8(const PrefillGemmParams& p, int m, int n, float (&rc)[8], float (&rs)[8]) {
  const int d = p.d_model, half = p.head_dim >> 1;
  const int sec = m / d;
  if (p.epi != PG_EPI_QKV_ROPE || sec >= 2) return;
  const int lp = (m >> 1) - sec * (d >> 1);
  const int i = lp % half;
  const int nb = n + ((threadIdx.x & 1) ? 8 : 0);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t t = static_cast<int64_t>(p.start_pos + min(nb + j, p.P - 1)) * half + i;
    rc[j] = __ldg(p.rope_cos + t);
    rs[j] = __ldg(p.rope_sin + t);
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Epilogue of one row pair (m even, m+1) for one token: the split-K reduce path.
// RoPE factors of row pair m at token n (QKV_ROPE, q/k sections), loaded before
// the reduce kernels' dependency wait -- the tables do not depend on the GEMM
struct PgRope {
  float c = 1.0f, s = 0.0f;
};
__device__ __forceinline__ PgRope pg_rope_load(const PrefillGemmParams& p, int m, int n) {
  PgRope r;
  if (p.epi != PG_EPI_QKV_ROPE || m / p.d_model >= 2) return r;
  const int half = p.head_dim >> 1;
  const int lp = (m >> 1) - (m / p.d_model) * (p.d_model >> 1);
  const int64_t t = static_cast<int64_t>(p.start_pos + n) * half + (lp - (lp / half) * half);
  r.c = __ldg(p.rope_cos + t);
  r.s = __ldg(p.rope_sin + t);
  return r;
}

__device__ __forceinline__ void pg_epilogue_pair(const PrefillGemmParams& p, int m, int n, float va, float vb,
                                                 PgRope rp) {
  const bool has_b = m + 1 < p.M;
  switch (p.epi) {
    case PG_EPI_STORE:
      p.out[static_cast<int64_t>(n) * p.M + m] = va;
      if (has_b) p.out[static_cast<int64_t>(n) * p.M + m + 1] = vb;
      break;
    case PG_EPI_RESID:
      p.out[static_cast<int64_t>(n) * p.M + m] += va;
      if (has_b) p.out[static_cast<int64_t>(n) * p.M + m + 1] += vb;
      break;
    case PG_EPI_RELU: {
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out_bf16) + static_cast<int64_t>(n) * p.M + m;
      o[0] = __float2bfloat16_rn(fmaxf(va, 0.0f));
      if (has_b) o[1] = __float2bfloat16_rn(fmaxf(vb, 0.0f));
      break;
    }
    case PG_EPI_SWIGLU:
      static_cast<__nv_bfloat16*>(p.out_bf16)[static_cast<int64_t>(n) * (p.M >> 1) + (m >> 1)] =
          __float2bfloat16_rn(va / (1.0f + expf(-va)) * vb);
      break;
    default: {
      const int d = p.d_model, dh = p.head_dim;
      const int sec = m / d;
      const int lp = (m >> 1) - sec * (d >> 1);
      const int pos = p.start_pos + n;
      float ra = va, rb = vb;
      int e0, e1, head;
      if (p.epi == PG_EPI_QKV_ROPE && sec < 2) {
        const int half = dh >> 1;
        head = lp / half;
        const int i = lp - head * half;
        const float c = rp.c, sn = rp.s;
        ra = va * c - vb * sn;
        rb = vb * c + va * sn;
        e0 = i;
        e1 = i + half;
      } else {
        const int e = 2 * lp;
        head = e / dh;
        e0 = e - head * dh;
        e1 = e0 + 1;
      }
      if (sec == 0) {
        float* q = p.q_out + static_cast<int64_t>(n) * d + head * dh;
        q[e0] = ra;
        q[e1] = rb;
      } else {
        void* cache = sec == 1 ? p.k_cache : p.v_cache;
        const int64_t base = kv_row(p.kvp, head, p.max_seq, pos) * dh;
        if (p.kv_bf16) {
          __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(cache) + base;
          c[e0] = __float2bfloat16_rn(ra);
          c[e1] = __float2bfloat16_rn(rb);
        } else {
          float* c = reinterpret_cast<float*>(cache) + base;
          c[e0] = ra;
          c[e1] = rb;
        }
      }
    }
  }
}

// mbarrier wait for threads that idle through the main loop: back off so they
// do not steal issue slots from the TMA / MMA threads on their SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(256);
}

// ---- the kernel -----------------------------------------------------------------
// Persistent: grid = min(work items, SMs); work item w = (m tile, n tile, k
// split), CTA c takes items c, c + grid, ...  The TMA producer streams stages
// across item boundaries; the accumulator is double-buffered in TMEM (2 x ntile
// fp32 columns), so the epilogue of item i overlaps the MMAs of item i+1.
// Each pipeline stage carries `kbox` 64-wide K boxes (kbox*128 contiguous bytes
// per weight row).

// STAGED: the QKV epilogue of whole tiles through shared-memory staging
// (pg_epilogue_qkv_staged); a separate instantiation so the launches that never
// use it (split-K short prompts, the other projections) keep the plain kernel
// (measured: one kernel for both cost TTFT P=10-200 30-90 us)
template <bool STAGED>
__global__ void __launch_bounds__(PG_THREADS, 1)
    prefill_gemm_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                        const PrefillGemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[8], empty[8], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg_base = STAGED ? reinterpret_cast<float*>(smem + static_cast<size_t>(p.stages) * p.kbox *
                                                                 (PG_BM * PG_BK * 2 + p.ntile * PG_BK * 2))
                           : nullptr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (p.M + PG_BM - 1) / PG_BM;
  const int n_tiles_all = m_tiles * p.n_ntiles;
  const bool tail = p.tail_ks > 1;  // stream-K tail (ksplit == 1)
  const int n_items = tail ? p.tail_first + (n_tiles_all - p.tail_first) * p.tail_ks : n_tiles_all * p.ksplit;
  const int kstep = PG_BK * p.kbox;
  const int nkb = (p.K + kstep - 1) / kstep;  // a ragged last block reads zeros past K (TMA OOB fill)
  const int S = p.stages;
  const uint32_t a_box = PG_BM * PG_BK * 2;
  const uint32_t b_box = static_cast<uint32_t>(p.ntile) * PG_BK * 2;
  const uint32_t stage_bytes = p.kbox * (a_box + b_box);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * p.ntile)) cols <<= 1;

  auto decode = [&](int w, int& m_tile, int& n_tile, int& split, int& kb0, int& kb1) {
    int mn, ks;
    if (tail) {
      if (w < p.tail_first) {  // whole tile
        mn = w;
        split = 0;
        ks = 1;
      } else {
        const int t = w - p.tail_first;
        mn = p.tail_first + t / p.tail_ks;
        split = t % p.tail_ks;
        ks = p.tail_ks;
      }
    } else {
      split = w % p.ksplit;
      mn = w / p.ksplit;
      ks = p.ksplit;
    }
    n_tile = mn % p.n_ntiles;
    m_tile = mn / p.n_ntiles;
    kb0 = static_cast<int>(static_cast<int64_t>(split) * nkb / ks);
    kb1 = static_cast<int>(static_cast<int64_t>(split + 1) * nkb / ks);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 2);  // the A and the B producer
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], blockDim.x / 32 - 3);  // one arrival per epilogue warp
    }
    mbar_fence_init();
  }
  if (warp == 1) {  // TMEM: 128 lanes (weight rows) x 2 buffers of ntile fp32 columns (tokens)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  griddep_launch_dependents();

  const int b_warp = static_cast<int>(blockDim.x / 32) - 1;  // the token (B) producer
  const uint32_t a_bytes = p.kbox * a_box, b_bytes = p.kbox * b_box;
  if (warp == 0) {
    if (lane == 0) {
      // The weight (A) boxes of the first S stages do not depend on the previous
      // kernel: requested before the dependency wait (the small kernels ahead of
      // a GEMM trigger their dependents at entry, so this CTA can be resident and
      // streaming while they run); the token (B) boxes come from warp b_warp.
      int npre = 0;
      for (int w = blockIdx.x; w < n_items && npre < S; w += gridDim.x) {
        int m_tile, n_tile, split, kb0, kb1;
        decode(w, m_tile, n_tile, split, kb0, kb1);
        for (int kb = kb0; kb < kb1 && npre < S; ++kb, ++npre) {
          uint8_t* st = smem + static_cast<size_t>(npre) * stage_bytes;
          mbar_arrive_expect_tx(&full[npre], a_bytes);
          if (p.box3d)
            tma_load_3d(st, &map_w, 0, m_tile * PG_BM, kb * p.kbox, &full[npre]);
          else
            for (int j = 0; j < p.kbox; ++j)
              tma_load_2d(st + j * a_box, &map_w, kb * kstep + j * PG_BK, m_tile * PG_BM, &full[npre]);
        }
      }
      int i = 0;  // global stage counter across items
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        int m_tile, n_tile, split, kb0, kb1;
        decode(w, m_tile, n_tile, split, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          if (i < npre) continue;
          const int s = i % S;
          uint8_t* st = smem + static_cast<size_t>(s) * stage_bytes;
          mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], a_bytes);
          if (p.box3d)
            tma_load_3d(st, &map_w, 0, m_tile * PG_BM, kb * p.kbox, &full[s]);
          else
            for (int j = 0; j < p.kbox; ++j)
              tma_load_2d(st + j * a_box, &map_w, kb * kstep + j * PG_BK, m_tile * PG_BM, &full[s]);
        }
      }
    }
  } else if (warp == b_warp) {
    if (lane == 0) {
      griddep_wait();  // the tokens are the previous kernel's output
      int i = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x) {
        int m_tile, n_tile, split, kb0, kb1;
        decode(w, m_tile, n_tile, split, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          const int s = i % S;
          uint8_t* st = smem + static_cast<size_t>(s) * stage_bytes;
          mbar_wait(&empty[s], ((i / S) & 1) ^ 1);  // a fresh slot passes at once
          mbar_arrive_expect_tx(&full[s], b_bytes);
          if (p.box3d)
            tma_load_3d(st + p.kbox * a_box, &map_x, 0, n_tile * p.ntile, kb * p.kbox, &full[s]);
          else
            for (int j = 0; j < p.kbox; ++j)
              tma_load_2d(st + p.kbox * a_box + j * b_box, &map_x, kb * kstep + j * PG_BK, n_tile * p.ntile, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(p.ntile);
      int i = 0, it = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
        int m_tile, n_tile, split, kb0, kb1;
        decode(w, m_tile, n_tile, split, kb0, kb1);
        const int buf = it & 1;
        mbar_wait(&acc_empty[buf], ((it >> 1) & 1) ^ 1);  // epilogue has drained this buffer
        tc_fence_after();
        const uint32_t acc = tmem + buf * p.ntile;
        for (int kb = kb0; kb < kb1; ++kb, ++i) {
          const int s = i % S;
          mbar_wait(&full[s], (i / S) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + static_cast<size_t>(s) * stage_bytes);
          const uint32_t sb = sa + p.kbox * a_box;
          for (int j = 0; j < p.kbox; ++j) {
#pragma unroll
            for (int k = 0; k < PG_BK / PG_UK; ++k) {
              const uint64_t ad = sw128_desc(sa + j * a_box + k * PG_UK * 2);
              const uint64_t bd = sw128_desc(sb + j * b_box + k * PG_UK * 2);
              tc_mma_bf16(acc, ad, bd, idesc, (kb > kb0 || j > 0 || k > 0) ? 1u : 0u);
            }
          }
          tc_commit(&empty[s]);  // frees the slot once these MMAs have read it
        }
        tc_commit(&acc_full[buf]);  // this item's accumulator is complete
      }
    }
    __syncwarp();
  } else {
    // epilogue warps 2..9: TMEM lanes 32*(warp%4) .. +31 = weight rows; the two
    // warps of a lane quadrant take alternate 16-token column groups (the
    // epilogue's own memory round trips -- RoPE table, residual -- halve)
    const int lane_base = 32 * (warp & 3);
    const int half = (warp - 2) >> 2;                      // column group of this warp
    const int groups = (static_cast<int>(blockDim.x) / 32 - 3) >> 2;  // warps per lane quadrant
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(lane_base) << 16);
    int it = 0;
    for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
      int m_tile, n_tile, split, kb0, kb1;
      decode(w, m_tile, n_tile, split, kb0, kb1);
      const int buf = it & 1;
      const int m = m_tile * PG_BM + lane_base + lane;
      const int n0 = n_tile * p.ntile;
      const int n_valid = min(p.ntile, p.P - n0);
      mbar_wait_sleep(&acc_full[buf], (it >> 1) & 1);
      tc_fence_after();
      const int tile_id = m_tile * p.n_ntiles + n_tile;
      // partials: every item of a split-K GEMM, or a stream-K tail unit
      const bool split_k = tail ? w >= p.tail_first : p.ksplit > 1;
      float* mypart = nullptr;
      if (split_k)
        mypart = tail ? p.part + (static_cast<int64_t>(tile_id - p.tail_first) * p.tail_ks + split) * p.ntile * PG_BM
                      : p.part + (static_cast<int64_t>(tile_id) * p.ksplit + split) * p.ntile * PG_BM;
      const bool staged = STAGED && !split_k;
      for (int c0 = 16 * half; c0 < n_valid; c0 += 16 * groups) {
        float v[16];
        float rc[8], rs[8];  // RoPE factors (staged epilogue): requested before the TMEM load
        if constexpr (STAGED)
          if (staged && p.epi != PG_EPI_SWIGLU) pg_rope8(p, m, n0 + c0, rc, rs);
        tc_ld16(t_lane + buf * p.ntile + c0, v);
        if (STAGED && staged) {
          float* stg = stg_base + (warp - 2) * 16 * PG_STG;
          if (p.epi == PG_EPI_SWIGLU)
            pg_epilogue_swiglu_staged(p, m, n0 + c0, min(16, n_valid - c0), v, stg);
          else
            pg_epilogue_qkv_staged(p, m, n0 + c0, min(16, n_valid - c0), v, rc, rs, stg);
        } else if (split_k) {
#pragma unroll
          for (int j = 0; j < 16; ++j) mypart[static_cast<int64_t>(c0 + j) * PG_BM + lane_base + lane] = v[j];
        } else {
          pg_epilogue16(p, m, n0 + c0, min(16, n_valid - c0), v);
        }
      }
      // accumulator drained: hand the buffer back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols) : "memory");
}

// ---- split-K reduction + epilogue --------------------------------------------------
// Short prompts split K over work items that only store fp32 partials
// [tile][split][token][128 rows]; this kernel sums them in split order
// (deterministic) and applies the epilogue, one thread per (row pair, token):
// fully parallel, instead of one CTA per tile serialising a tail reduction.
// 2D grid: blockIdx.y = token, x * blockDim + tid = row pair -- no 64-bit index
// division per element (the 1D version spent most of its time there: P=200
// QKV 20.7 us for ~37 MB of traffic).
__global__ void prefill_splitk_reduce_kernel(const PrefillGemmParams p) {
  griddep_launch_dependents();  // the next GEMM may start its weight stream (it waits for us before its tokens)
  const int n_pairs = (p.M + 1) >> 1;
  const int pr = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  const bool live = pr < n_pairs;
  const int m = 2 * pr;
  // this thread's RoPE factors, before the wait
  const PgRope r0 = live ? pg_rope_load(p, m, n) : PgRope{};
  griddep_wait();  // launched with PDL behind the GEMM: partials complete
  if (!live) return;
  const int m_tile = m / PG_BM, n_tile = n / p.ntile;
  const int r = m - m_tile * PG_BM, nn = n - n_tile * p.ntile;
  const float* base = p.part + (static_cast<int64_t>(m_tile * p.n_ntiles + n_tile) * p.ksplit) * p.ntile * PG_BM;
  float va = 0.0f, vb = 0.0f;
  for (int sp = 0; sp < p.ksplit; ++sp) {
    const float2 q = *reinterpret_cast<const float2*>(base + (static_cast<int64_t>(sp) * p.ntile + nn) * PG_BM + r);
    va += q.x;
    vb += q.y;
  }
  pg_epilogue_pair(p, m, n, va, vb, r0);
}

// Reduce of the stream-K tail: tiles [tail_first, m_tiles*n_ntiles), tail_ks
// partials each ([tile - tail_first][split][token][128 rows]), summed in split
// order, then the GEMM's epilogue; one thread per (row pair, token): block
// (x, y) = 4 tokens [4x, 4x+4) of tail tile y, 64 row pairs per token.
__global__ void prefill_tail_reduce_kernel(const PrefillGemmParams p) {
  griddep_launch_dependents();
  const int t = blockIdx.y;
  const int nn = blockIdx.x * 4 + (threadIdx.x >> 6);
  const int r = 2 * (threadIdx.x & 63);
  const int tile = p.tail_first + t;
  const int m_tile = tile / p.n_ntiles, n_tile = tile - m_tile * p.n_ntiles;
  const int m = m_tile * PG_BM + r, n = n_tile * p.ntile + nn;
  griddep_wait();  // launched with PDL behind the GEMM: partials complete
  // (no pre-wait RoPE loads here: measured slower at P >= 200, unlike the short-prompt reduce)
  if (nn >= p.ntile || m >= p.M || n >= p.P) return;
  const float* base = p.part + static_cast<int64_t>(t) * p.tail_ks * p.ntile * PG_BM;
  float va = 0.0f, vb = 0.0f;
  for (int sp = 0; sp < p.tail_ks; ++sp) {
    const float2 q = *reinterpret_cast<const float2*>(base + (static_cast<int64_t>(sp) * p.ntile + nn) * PG_BM + r);
    va += q.x;
    vb += q.y;
  }
  pg_epilogue_pair(p, m, n, va, vb, pg_rope_load(p, m, n));
}

// Deferred reduce of a residual GEMM (epi RESID, split K) + RMSNorm of the
// updated rows: one 1024-thread CTA per token, groups of split partials loaded
// together.  Per element the split partials are summed in split order first
// and then added to X (the order prefill_splitk_reduce_kernel + pg_epilogue_pair
// use), so the residual stream is bit-identical to the separate launches; the
// norm's sum of squares is reduced over a different thread shape (fp32
// reassociation only).
constexpr int RN_THREADS = 512, RN_MAXV = 8, RN_SPLIT_GROUP = 4;  // M = d <= 16384
constexpr int RN_NORM_THREADS = 256, RN_NORM_MAXV = 16;  // prefill_rmsnorm_kernel's thread shape
// MAXV float4 per thread, the smallest that covers d (2 at d = 4096): registers
// stay low enough for several rows' CTAs per SM -- at 8 the kernel held the SM's
// whole register file and ran at 1 CTA per SM (P=500: 19.2 us per launch)
template <int MAXV>
__global__ void __launch_bounds__(RN_THREADS) prefill_resid_norm_kernel(const PrefillGemmParams p, const float* gamma,
                                                                        float eps, __nv_bfloat16* Xn) {
  griddep_launch_dependents();  // the next GEMM may start its weight stream
  __shared__ float red[32];
  extern __shared__ float4 xrow[];  // the updated row, for the reduction below
  float4 g[MAXV];
  const int d = p.M, n4 = d >> 2;
#pragma unroll
  for (int u = 0; u < MAXV; ++u) {
    const int j = threadIdx.x + u * RN_THREADS;
    g[u] = j < n4 ? __ldg(reinterpret_cast<const float4*>(gamma) + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  griddep_wait();  // PDL behind the GEMM: partials complete
  const int n = blockIdx.x;
  const int n_tile = n / p.ntile, nn = n - n_tile * p.ntile;
  float* X = p.out + static_cast<int64_t>(n) * d;
  float4 v[MAXV];
#pragma unroll
  for (int u = 0; u < MAXV; ++u) {
    const int j = threadIdx.x + u * RN_THREADS;
    v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j >= n4) continue;
    const int m = 4 * j, m_tile = m / PG_BM, r = m - m_tile * PG_BM;
    const float* base = p.part + (static_cast<int64_t>(m_tile * p.n_ntiles + n_tile) * p.ksplit) * p.ntile * PG_BM +
                        static_cast<int64_t>(nn) * PG_BM + r;
    const int64_t sstride = static_cast<int64_t>(p.ntile) * PG_BM;
    const float4 x = __ldcg(reinterpret_cast<const float4*>(X) + j);
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < p.ksplit; s0 += RN_SPLIT_GROUP) {  // a group of split loads in flight at once
      float4 q[RN_SPLIT_GROUP];
#pragma unroll
      for (int k = 0; k < RN_SPLIT_GROUP; ++k)
        q[k] = s0 + k < p.ksplit ? __ldcg(reinterpret_cast<const float4*>(base + (s0 + k) * sstride))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < RN_SPLIT_GROUP; ++k) {
        if (s0 + k >= p.ksplit) break;
        sum.x += q[k].x;
        sum.y += q[k].y;
        sum.z += q[k].z;
        sum.w += q[k].w;
      }
    }
    v[u] = make_float4(x.x + sum.x, x.y + sum.y, x.z + sum.z, x.w + sum.w);
    reinterpret_cast<float4*>(X)[j] = v[u];
    xrow[j] = v[u];
  }
  __syncthreads();
  // RMSNorm: prefill_rmsnorm_kernel's arithmetic, its sum of squares reduced
  // over the same (256-thread) shape, so Xn is bit-identical too
  if (threadIdx.x < RN_NORM_THREADS) {
    float ss = 0.0f;
#pragma unroll
    for (int u = 0; u < RN_NORM_MAXV; ++u) {
      const int j = threadIdx.x + u * RN_NORM_THREADS;
      const float4 a = j < n4 ? xrow[j] : make_float4(0.f, 0.f, 0.f, 0.f);
      ss = __fadd_rn(ss, sumsq4(a));
    }
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (RN_NORM_THREADS >> 5) ? red[threadIdx.x] : 0.0f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / static_cast<float>(d) + eps);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(Xn + static_cast<int64_t>(n) * d);
#pragma unroll
  for (int u = 0; u < MAXV; ++u) {
    const int j = threadIdx.x + u * RN_THREADS;
    if (j >= n4) continue;
    o[2 * j] = __floats2bfloat162_rn(v[u].x * inv * g[u].x, v[u].y * inv * g[u].y);
    o[2 * j + 1] = __floats2bfloat162_rn(v[u].z * inv * g[u].z, v[u].w * inv * g[u].w);
  }
}

// ---- host side --------------------------------------------------------------------

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2D bf16 row-major [rows, cols] tensor, box [box_rows, 64 cols], 128-byte swizzle;
// rows beyond `rows` read as zero (token padding).
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {PG_BK, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// {64, rows, K/64} view of a row-major [rows, K] bf16 matrix (K % 64 == 0), box
// {64, box_rows, kbox}, 128-byte swizzle: kbox K blocks in one TMA instruction.
bool make_map3(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows, int kbox) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || cols % PG_BK) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(PG_BK), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(cols / PG_BK)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2, static_cast<cuuint64_t>(PG_BK) * 2};
  const cuuint32_t box[3] = {PG_BK, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(kbox)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// Tiling policy: tokens are split into N tiles of <= 128 (P > 128) so large
// prompts spread over the SMs without any reduction; K is split only for short
// prompts (P <= 64: memory-bound, N cannot supply the parallelism), and then
// each stage carries 4 K boxes (512 contiguous bytes per weight row).
struct PgShape {
  int ntile, n_ntiles, ksplit, kbox;
};
static PgShape pg_shape(int M, int K, int P, int sms, bool wide_split = false) {
  PgShape sh;
  const int m_tiles = (M + PG_BM - 1) / PG_BM;
  sh.kbox = 1;
  sh.ksplit = 1;
  if (P <= 64) {
    // memory-bound: one N tile; split K so the items fill (but do not overflow) one wave
    sh.ntile = (P + 15) / 16 * 16;
    sh.n_ntiles = 1;
    sh.kbox = (K % (4 * PG_BK) == 0) ? 4 : ((K % (2 * PG_BK) == 0) ? 2 : 1);
    const int nkb = (K + PG_BK * sh.kbox - 1) / (PG_BK * sh.kbox);
    // persistent CTAs: pick the split whose work items tile the SMs evenly
    // (time ~ waves / split); partials are reduced by a separate parallel kernel
    const double per_split = 0.05;  // cost of one more split; measured: TTFT P=10 3.66 -> 3.49 ms (vs 0.005)
    double best = 1e30;
    for (int ks = 1; ks <= std::min(16, nkb); ++ks) {
      const double waves = static_cast<double>((m_tiles * ks + sms - 1) / sms);
      const double cost = waves / ks + per_split * ks;
      if (cost < best) {
        best = cost;
        sh.ksplit = ks;
      }
    }
    return sh;
  }
  // compute-bound: the widest token tile (<= 256, TMEM holds two): operand bytes
  // per flop fall as N grows.  Measured (P=500): narrower tiles to occupy more
  // SMs, or split-K with a last-CTA reduction, are both slower for the small-M
  // GEMMs (Wo, down) than 64 wide tiles.
  const int nt_max = PG_MAX_NT;  // 192 / 176 / 128 measured slower at P=500
  sh.n_ntiles = (P + nt_max - 1) / nt_max;
  sh.ntile = ((P + sh.n_ntiles - 1) / sh.n_ntiles + 15) / 16 * 16;
  // small-M GEMMs (Wo, down: 32 tiles) split K so the items fill the SMs;
  // the partials go through the parallel reduce kernel
  const int items = m_tiles * sh.n_ntiles;
  const int nkb = (K + PG_BK - 1) / PG_BK;
  double best = 1e30;
  const int wide_ks = 2;  // max split for P > 256; measured: TTFT P=500 12.3 -> 10.9 ms (32 -> 128 CTAs busy)
  // P > 256: measured faster unsplit -- except (knob) a residual GEMM whose
  // reduce is fused into the next RMSNorm launch
  const int ks_max = sh.n_ntiles > 1 ? (wide_split ? std::min(wide_ks, nkb) : 1) : std::min(8, nkb);
  for (int ks = 1; ks <= ks_max; ++ks) {
    const double waves = static_cast<double>((items * ks + sms - 1) / sms);
    const double cost = waves / ks + 0.02 * (ks - 1);
    if (cost < best) {
      best = cost;
      sh.ksplit = ks;
    }
  }
  return sh;
}

int prefill_gemm_ksplit(int M, int K, int sms) { return pg_shape(M, K, 16, sms).ksplit; }

// Stream-K tail of an unsplit GEMM: when the tiles leave a partial last wave,
// its tiles are split ks ways in K (ks <= 4, their units fill the SMs) and
// reduced afterwards; the first full waves stay whole tiles.
static void pg_tail(int n_tiles_all, int nkb, int sms, int* tail_first, int* tail_ks) {
  *tail_first = 0;
  *tail_ks = 0;
  if (n_tiles_all <= sms) return;
  const int rem = n_tiles_all % sms;
  if (rem == 0) return;
  const int ks = std::min({4, sms / rem, nkb});
  if (ks < 2) return;
  *tail_first = n_tiles_all - rem;
  *tail_ks = ks;
}

size_t prefill_gemm_part_floats(int M, int K, int P, int sms) {
  size_t worst = 0;
  (void)P;
  for (int q = 16; q <= PREFILL_CHUNK; q += 16) {  // size for the worst token count
    for (const bool wide : {false, true}) {
      const PgShape sh = pg_shape(M, K, q, sms, wide);
      const int m_tiles = (M + PG_BM - 1) / PG_BM;
      if (sh.ksplit == 1) {  // stream-K tail partials
        int tf, tk;
        pg_tail(m_tiles * sh.n_ntiles, (K + PG_BK * sh.kbox - 1) / (PG_BK * sh.kbox), sms, &tf, &tk);
        if (tk > 1)
          worst = std::max(worst, static_cast<size_t>(m_tiles * sh.n_ntiles - tf) * tk * sh.ntile * PG_BM);
        continue;
      }
      worst = std::max(worst, static_cast<size_t>(m_tiles) * sh.n_ntiles * sh.ksplit * sh.ntile * PG_BM);
    }
  }
  return worst;
}

cudaError_t prefill_gemm_prepare() {
  cudaError_t e = cudaFuncSetAttribute(prefill_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(prefill_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
}

static cudaError_t launch_prefill_gemm_impl(const void* w, const void* x, PrefillGemmParams p, cudaStream_t s, bool pdl,
                                            PrefillGemmParams* out) {
  // K need not be a multiple of the 64-wide K box (e.g. d_ff / 8 = 1376 under
  // TP=8): TMA zero-fills both operands past K; rows must stay 16-byte aligned
  if (p.K % 8 != 0 || p.P < 1 || p.P > PREFILL_CHUNK || p.M < 1) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  const PgShape sh = pg_shape(p.M, p.K, p.P, num_sms(dev), p.wide_split || (p.defer_reduce && p.epi == PG_EPI_RESID));
  p.ntile = sh.ntile;
  p.n_ntiles = sh.n_ntiles;
  p.ksplit = sh.ksplit;
  p.kbox = sh.kbox;
  if (p.ksplit > 1 && (!p.part || !p.counters)) return cudaErrorInvalidValue;
  const int m_tiles = (p.M + PG_BM - 1) / PG_BM;
  if (p.ksplit > 1 && m_tiles * p.n_ntiles > 4096) return cudaErrorInvalidValue;
  p.tail_first = 0;
  p.tail_ks = 0;
  if (p.ksplit == 1 && p.part)
    pg_tail(m_tiles * p.n_ntiles, (p.K + PG_BK * p.kbox - 1) / (PG_BK * p.kbox), num_sms(dev), &p.tail_first,
            &p.tail_ks);
  const bool tail = p.tail_ks > 1;
  const int n_items =
      tail ? p.tail_first + (m_tiles * p.n_ntiles - p.tail_first) * p.tail_ks : m_tiles * p.n_ntiles * p.ksplit;
  const int stage_bytes = p.kbox * (PG_BM * PG_BK * 2 + p.ntile * PG_BK * 2);
  // the QKV / SwiGLU epilogue of whole tiles goes through per-warp shared-memory staging
  p.epi_stage = p.ksplit == 1 && (((p.epi == PG_EPI_QKV || p.epi == PG_EPI_QKV_ROPE) && p.head_dim % 32 == 0 &&
                                    p.d_model % 32 == 0) ||
                                   (p.epi == PG_EPI_SWIGLU && p.M % 32 == 0));
  const int stg_bytes = p.epi_stage ? PG_EPI_WARPS * 16 * PG_STG * 4 : 0;
  const int budget = 220 * 1024 - 1024 - stg_bytes;
  p.stages = std::min(8, budget / stage_bytes);
  if (p.stages < 2) return cudaErrorInvalidValue;
  CUtensorMap mw, mx;
  // several K blocks per stage (short prompts): one 3D box per operand and stage
  // instead of kbox 2D boxes when K is a whole number of blocks
  p.box3d = 0;
#ifndef GRT_NO_BOX3D
  if (p.kbox > 1 && p.K % (PG_BK * p.kbox) == 0 && make_map3(&mw, w, p.M, p.K, PG_BM, p.kbox) &&
      make_map3(&mx, x, p.P, p.K, p.ntile, p.kbox))
    p.box3d = 1;
#endif
  if (!p.box3d) {
    if (!make_map(&mw, w, p.M, p.K, PG_BM)) return cudaErrorInvalidValue;
    if (!make_map(&mx, x, p.P, p.K, p.ntile)) return cudaErrorInvalidValue;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(n_items, num_sms(dev)));
  // two token tiles (P > 256): 8 epilogue warps (the epilogue's memory round
  // trips dominate a one-item CTA); otherwise 4 (measured faster)
  cfg.blockDim = dim3(p.n_ntiles > 1 ? PG_THREADS : 7 * 32);
  cfg.dynamicSmemBytes = static_cast<size_t>(p.stages) * stage_bytes + stg_bytes + 1024;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = p.epi_stage ? cudaLaunchKernelEx(&cfg, prefill_gemm_kernel<true>, mw, mx, p)
                              : cudaLaunchKernelEx(&cfg, prefill_gemm_kernel<false>, mw, mx, p);
  if (out) *out = p;
  if (e != cudaSuccess) return e;
  if (tail) {  // reduce + epilogue of the tail tiles
    const int n_tail = m_tiles * p.n_ntiles - p.tail_first;
    cudaLaunchConfig_t rc = {};
    // one (row pair, token) per thread: every partial load of the grid in flight at once
    rc.gridDim = dim3((p.ntile + 3) / 4, n_tail);
    rc.blockDim = dim3(256);
    rc.stream = s;
    rc.attrs = attr;
    rc.numAttrs = 1;
    return cudaLaunchKernelEx(&rc, prefill_tail_reduce_kernel, p);
  }
  if (p.ksplit == 1 || (p.defer_reduce && p.epi == PG_EPI_RESID)) return e;
  cudaLaunchConfig_t rc = {};
  rc.gridDim = dim3(((p.M + 1) / 2 + 255) / 256, p.P);
  rc.blockDim = dim3(256);
  rc.stream = s;
  rc.attrs = attr;
  rc.numAttrs = 1;  // always PDL: the reduce's launch overlaps the GEMM's tail
  return cudaLaunchKernelEx(&rc, prefill_splitk_reduce_kernel, p);
}

cudaError_t launch_prefill_gemm(const void* w, const void* x, PrefillGemmParams p, cudaStream_t s, bool pdl) {
  return launch_prefill_gemm_impl(w, x, p, s, pdl, nullptr);
}

cudaError_t launch_prefill_gemm_ex(const void* w, const void* x, PrefillGemmParams* p, cudaStream_t s, bool pdl) {
  return launch_prefill_gemm_impl(w, x, *p, s, pdl, p);
}

cudaError_t launch_prefill_resid_norm(const PrefillGemmParams& p, const float* gamma, float eps, void* Xn,
                                      cudaStream_t s) {
  if (p.epi != PG_EPI_RESID || p.ksplit < 2 || p.M % 4 || p.M > 4 * RN_MAXV * RN_THREADS ||
      p.M > 4 * RN_NORM_MAXV * RN_NORM_THREADS || p.M > 48 * 1024 / 4 || !p.part)
    return cudaErrorInvalidValue;
  cudaLaunchConfig_t rc = {};
  rc.gridDim = dim3(p.P);
  rc.blockDim = dim3(RN_THREADS);
  rc.dynamicSmemBytes = static_cast<size_t>(p.M) * 4;
  rc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  rc.attrs = attr;
  rc.numAttrs = 1;
  const int n4 = p.M / 4;
  if (n4 <= 2 * RN_THREADS)
    return cudaLaunchKernelEx(&rc, prefill_resid_norm_kernel<2>, p, gamma, eps, static_cast<__nv_bfloat16*>(Xn));
  if (n4 <= 4 * RN_THREADS)
    return cudaLaunchKernelEx(&rc, prefill_resid_norm_kernel<4>, p, gamma, eps, static_cast<__nv_bfloat16*>(Xn));
  return cudaLaunchKernelEx(&rc, prefill_resid_norm_kernel<RN_MAXV>, p, gamma, eps, static_cast<__nv_bfloat16*>(Xn));
}

}  // namespace grt
