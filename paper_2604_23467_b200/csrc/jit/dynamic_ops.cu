// dynamic_ops.cu -- NVRTC source of the DYNAMIC ops (the JIT context path).
//
// The reference's dynamic set is exactly {extend_position, kv_append,
// sample_token} (kernels.hpp:14-19).  Here they are hand-written
// CUDA compiled at session start by NVRTC for sm_100a, specialised on the model
// shape through -D defines (GRT_D, GRT_V, GRT_MAXSEQ, GRT_WBF16, GRT_ARCH_REF).
// They read every runtime value (token, position, RNG state) from the device
// control block (ctrl.h), so they are capturable into the step graph.
//
// Compiled with --fmad=false: the integer-CDF sampler must reproduce
// oracle.c:oc_sample_topkp bit for bit.
#include "ctrl.h"

#ifndef GRT_D
#error "GRT_D must be defined"
#endif
#ifndef GRT_V
#error "GRT_V must be defined"
#endif

typedef unsigned long long u64;
typedef unsigned int u32;

#define GRT_SAMPLE_THREADS 1024
// top-k/top-p: the per-token weights are computed once into dynamic shared
// memory (u32: w = e * 2^31 <= 2^31) when they fit; the host launches the
// sampler kernels with GRT_V * 4 bytes of dynamic shared memory then (jit.cpp)
#define GRT_SAMPLE_SMEM_MAX 196608
// 2: weights + a u16 candidate list (radix select with compaction, below);
// 1: weights only (8-bit radix passes over the whole vocabulary); 0: recomputed
#if GRT_V * 6 <= GRT_SAMPLE_SMEM_MAX && GRT_V <= 32768
#define GRT_TOPKP_SMEM 2
#elif GRT_V * 4 <= GRT_SAMPLE_SMEM_MAX
#define GRT_TOPKP_SMEM 1
#else
#define GRT_TOPKP_SMEM 0
#endif
#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif
// phase stamps for the sampler timing probe (tools/sampler_timing.cu); no-op here
#ifndef GRT_STAMP
#define GRT_STAMP(i)
#endif

__device__ __forceinline__ void grt_griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grt_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ u64 grt_globaltimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float grt_bf16_to_f32(unsigned short h) { return __uint_as_float(((u32)h) << 16); }

// ---------------------------------------------------------------------------
// extend_position + slot append (kernels.cpp:238-259, :205-236; model.cpp:156-162)
//   x = emb[token] (+ pos_table[position] in the reference arch); cur_len++.
// The zero rows the reference appends are overwritten by the static pass before
// they are read (build_plan writes row length-1 before attention), so the
// append reduces to the length bump.
// x = emb[tok] (+ pos_table[pos]); then cur_len = pos + 1.
__device__ __forceinline__ void gather_row(GrtCtrl* ctrl, int pos, int tok, const void* emb, const void* pos_table,
                                           float* x) {
  const long long erow = (long long)tok * GRT_D;
#if GRT_WBF16 && !GRT_ARCH_REF && (GRT_D % 8 == 0)
  (void)pos_table;
  // 16-byte loads (8 bf16) -> two float4 stores
  for (int j8 = threadIdx.x; j8 < GRT_D / 8; j8 += blockDim.x) {
    const uint4 u = ((const uint4*)((const unsigned short*)emb + erow))[j8];
    float4 a, b;
    a.x = __uint_as_float(u.x << 16); a.y = __uint_as_float(u.x & 0xFFFF0000u);
    a.z = __uint_as_float(u.y << 16); a.w = __uint_as_float(u.y & 0xFFFF0000u);
    b.x = __uint_as_float(u.z << 16); b.y = __uint_as_float(u.z & 0xFFFF0000u);
    b.z = __uint_as_float(u.w << 16); b.w = __uint_as_float(u.w & 0xFFFF0000u);
    ((float4*)x)[2 * j8] = a;
    ((float4*)x)[2 * j8 + 1] = b;
  }
#else
#if GRT_ARCH_REF
  const long long prow = (long long)pos * GRT_D;
#else
  (void)pos_table;
#endif
  for (int j = threadIdx.x; j < GRT_D; j += blockDim.x) {
#if GRT_WBF16
    float e = grt_bf16_to_f32(((const unsigned short*)emb)[erow + j]);
#if GRT_ARCH_REF
    e = e + grt_bf16_to_f32(((const unsigned short*)pos_table)[prow + j]);
#endif
#else
    float e = ((const float*)emb)[erow + j];
#if GRT_ARCH_REF
    e = e + ((const float*)pos_table)[prow + j];
#endif
#endif
    x[j] = e;
  }
#endif
  __syncthreads();
  if (threadIdx.x == 0) ctrl->seq_len = pos + 1;
}

__device__ __forceinline__ void preprocess_impl(GrtCtrl* ctrl, const void* emb, const void* pos_table, float* x) {
  __shared__ int s_pos, s_tok, s_ok;
  if (threadIdx.x == 0) {
    const int pos = ctrl->seq_len;
    int ok = 1;
    int tok = 0;
    if (pos >= GRT_MAXSEQ || pos < 0) {
      atomicOr(&ctrl->err, 2); /* CacheFull / position outside table */
      ok = 0;
    } else {
      tok = ctrl->tokens[pos];
      if (tok < 0 || tok >= GRT_V) {
        atomicOr(&ctrl->err, 4); /* TokenOutOfRange */
        ok = 0;
      }
    }
    s_pos = pos;
    s_tok = tok;
    s_ok = ok;
  }
  __syncthreads();
  if (!s_ok) return;
  gather_row(ctrl, s_pos, s_tok, emb, pos_table, x);
}

extern "C" __global__ void grt_preprocess(GrtCtrl* ctrl, const void* emb, const void* pos_table, float* x) {
  grt_launch_dependents();
  grt_griddep_wait();
  preprocess_impl(ctrl, emb, pos_table, x);
}

// ---------------------------------------------------------------------------
// Sampler (run_sampler, kernels.cpp:263-289, plus the integer-CDF top-k/top-p).

__device__ __forceinline__ void philox4x32_10(u32 c[4], u32 k0, u32 k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u32 hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const u32 hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const u32 n0 = hi1 ^ c[1] ^ k0;
    const u32 n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Twin of oracle.c:oc_grt_expf -- every step an explicit fmaf or one rounded op.
__device__ __forceinline__ float grt_expf(float z) {
  if (!(z > -30.0f)) return 0.0f;
  if (z > 0.0f) z = 0.0f;
  const float n = rintf(z * 1.44269504088896341f);
  float r = fmaf(n, -0.693145751953125f, z);
  r = fmaf(n, -1.428606765330187e-06f, r);
  float p = 1.3981999507e-3f;
  p = fmaf(p, r, 8.3334519073e-3f);
  p = fmaf(p, r, 4.1665795894e-2f);
  p = fmaf(p, r, 1.6666665459e-1f);
  p = fmaf(p, r, 5.0000001201e-1f);
  const float r2 = r * r;
  float y = fmaf(p, r2, r);
  y = y + 1.0f;
  // y * 2^n with n in [-44, 0] and y in [0.7, 1.5): always a normal float, so
  // adding n to the exponent field is ldexpf's result exactly
  return __int_as_float(__float_as_int(y) + ((int)n << 23));
}

__device__ __forceinline__ u64 topkp_weight_v(float logit, float m, float t) {
  const float z = (logit - m) / t;
  const float e = grt_expf(z);
  return (u64)(u32)(e * 2147483648.0f);  // e <= 1: the product fits 32 bits (same truncation)
}
__device__ __forceinline__ u64 topkp_weight(const float* logits, int i, float m, float t) {
  const float z = (logits[i] - m) / t;
  const float e = grt_expf(z);
  return (u64)(e * 2147483648.0f);
}
__device__ __forceinline__ u64 topkp_key(u64 w, int i) { return (w << 16) | (u64)(0xFFFF - i); }

__device__ float block_max_f(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) t = fmaxf(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

__device__ u64 block_sum_u64(u64 v, u64* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    u64 t = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

// Finds, among keys with (key & mask) == prefix and key >= floor, the digit
// bucket where the descending cumulative (count or weight) reaches `need`:
// the highest digit dg >= 1 whose inclusive suffix sum reaches `need` (else 0),
// and the remainder need - (sum of the buckets above dg).  Warp 0 scans the
// 256 buckets in parallel (lane l owns buckets 8l..8l+7); integer sums, so the
// result equals the serial top-down walk exactly.
__device__ void radix_pick(u64* hist, int shift, u64& prefix, u64& mask, u64& need) {
  __shared__ u64 s_prefix, s_need;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    u64 hb[8];
    u64 tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      hb[k] = hist[8 * lane + k];
      tot += hb[k];
    }
    u64 suf = tot;  // inclusive suffix over lanes >= lane
    for (int o = 1; o < 32; o <<= 1) {
      const u64 n = __shfl_down_sync(0xffffffffu, suf, o);
      if (lane + o < 32) suf += n;
    }
    u64 run = suf - tot;  // buckets above this lane's range
    int best = -1;
    u64 excl = 0;
#pragma unroll
    for (int k = 7; k >= 0; --k) {
      const int d = 8 * lane + k;
      if (best < 0 && d >= 1) {
        if (run + hb[k] >= need) {
          best = d;
          excl = run;
        }
      }
      run += hb[k];
    }
    const unsigned hit = __ballot_sync(0xffffffffu, best >= 1);
    int dg;
    u64 above;
    if (hit) {
      const int src = 31 - __clz(hit);
      dg = __shfl_sync(0xffffffffu, best, src);
      above = __shfl_sync(0xffffffffu, excl, src);
    } else {  // fall through to digit 0: every bucket above it is consumed
      dg = 0;
      above = __shfl_sync(0xffffffffu, suf - hb[0], 0);
    }
    if (lane == 0) {
      s_prefix = prefix | ((u64)dg << shift);
      s_need = need - above;
    }
  }
  __syncthreads();
  prefix = s_prefix;
  need = s_need;
  mask |= (u64)255 << shift;
  __syncthreads();
}

#if GRT_TOPKP_SMEM == 2
// ---- radix select with candidate compaction (11-bit digits) -------------------
// The threshold key of oc_sample_topkp (oracle.c) -- walking the rank keys in
// descending order, the key at which the running total of `val` (1 for top-k,
// the weight for top-p) first reaches `need` -- found digit by digit from the
// top (bits 37-47, 26-36, 15-25, 4-14, 0-10; the last pass overlaps bits already
// fixed, which every candidate shares).  Pass 0 scans the whole vocabulary
// (keys >= kfloor); every pass keeps only the keys in the chosen digit bucket,
// compacted into a u16 list in shared memory, so later passes touch a handful
// of candidates instead of 32000 keys.  Integer sums throughout: the result is
// the serial walk's exactly.
#define RS_B 2048
#define RS_PER ((GRT_V + GRT_SAMPLE_THREADS - 1) / GRT_SAMPLE_THREADS)

__device__ __forceinline__ u64 rs_key(const u32* wsm, int i) { return ((u64)wsm[i] << 16) | (u64)(0xFFFF - i); }
// key(w, i) >= floor with 32-bit compares: key = w << 16 | (0xFFFF - i)
__device__ __forceinline__ bool rs_ge(u32 w, int i, u64 floor) {
  const u32 fw = (u32)(floor >> 16), fl = (u32)(floor & 0xFFFFu);
  return w > fw || (w == fw && (u32)(0xFFFF - i) >= fl);
}

// block-wide exclusive scan of one int per thread; returns the total
__device__ __forceinline__ int rs_scan(int v, int* excl, int* warp_tot) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += n;
  }
  if (lane == 31) warp_tot[wp] = x;
  __syncthreads();
  if (wp == 0) {
    int t = lane < (GRT_SAMPLE_THREADS >> 5) ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += n;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  *excl = x - v + (wp > 0 ? warp_tot[wp - 1] : 0);
  const int total = warp_tot[31];
  __syncthreads();
  return total;
}

// bucket b's total: hist[b] + 2^16 * hist[RS_B + b] (the low and high 16 bits of
// every weight are summed separately with native 32-bit shared-memory atomics --
// a 64-bit atomicAdd compiles to a CAS spin loop; both sums stay below 2^31
// for V <= 32768)
__device__ __forceinline__ u64 rs_bucket(const u32* hist, int b) { return (u64)hist[b] + ((u64)hist[RS_B + b] << 16); }

// the highest digit whose inclusive descending cumulative reaches need (else 0)
// and the cumulative above it; thread t owns buckets 2t, 2t+1
__device__ __forceinline__ void rs_pick(const u32* hist, u64 need, int* s_dg, u64* s_above, u64* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const u64 h0 = rs_bucket(hist, 2 * tid), h1 = rs_bucket(hist, 2 * tid + 1), sm = h0 + h1;
  u64 v = sm;  // inclusive suffix within the warp
  for (int o = 1; o < 32; o <<= 1) {
    const u64 n = __shfl_down_sync(0xffffffffu, v, o);
    if (lane + o < 32) v += n;
  }
  if (lane == 0) wsum[wp] = v;
  if (tid == 0) *s_dg = 0;
  __syncthreads();
  if (wp == 0) {  // exclusive suffix over the warps
    u64 t = wsum[lane];
    u64 incl = t;
    for (int o = 1; o < 32; o <<= 1) {
      const u64 n = __shfl_down_sync(0xffffffffu, incl, o);
      if (lane + o < 32) incl += n;
    }
    wsum[lane] = incl - t;
  }
  __syncthreads();
  const u64 S = v + wsum[wp];  // cumulative from bucket 2*tid upward
  const u64 E = S - sm;        // above bucket 2*tid+1
  int b = -1;
  if (E + h1 >= need) b = 2 * tid + 1;
  else if (tid > 0 && S >= need) b = 2 * tid;
  if (b >= 1) atomicMax(s_dg, b);
  __syncthreads();
  const int dg = *s_dg;
  if (dg >= 1 && (dg >> 1) == tid) *s_above = (dg & 1) ? E : E + h1;
  if (dg == 0 && tid == 0) *s_above = E + h1;  // total - hist[0]
  __syncthreads();
}

// hist_ready: pass 0's histogram was accumulated by the caller (while it
// computed the weights, kfloor == 0)
__device__ u64 radix_select_compact(const u32* wsm, unsigned short* cand, u64 kfloor, bool by_weight, u64 need,
                                    u32* hist, bool hist_ready = false) {
  __shared__ int s_dg, s_n, warp_tot[32];
  __shared__ u64 s_above, wsum[32];
  const int tid = threadIdx.x;
  int n = -1;  // -1: every index of the vocabulary with key >= kfloor
  u64 prefix = 0;
  const int shifts[5] = {37, 26, 15, 4, 0};
#pragma unroll 1
  for (int ps = 0; ps < 5; ++ps) {
    const int sh = shifts[ps];
    const bool built = ps == 0 && hist_ready;
    if (!built) {
      for (int b = tid; b < 2 * RS_B; b += GRT_SAMPLE_THREADS) hist[b] = 0;
      __syncthreads();
    }
    auto add = [&](int i, u64 key) {
      const int b = (int)((key >> sh) & (RS_B - 1));
      if (!by_weight) {
        atomicAdd(&hist[b], 1u);
      } else {
        const u32 w = wsm[i];
        atomicAdd(&hist[b], w & 0xFFFFu);
        if (w >> 16) atomicAdd(&hist[RS_B + b], w >> 16);
      }
    };
    if (built) {
      // histogram already complete (the caller synchronised)
    } else if (n < 0) {  // pass 0 (sh = 37 >= 16): the digit is w's top bits, 32-bit arithmetic
      // digit 0 (weights below 2^21: most of the vocabulary) is summed per thread
      // and added once per warp -- 32000 atomics on one shared word serialise
      u32 z_lo = 0, z_hi = 0;
      for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) {
        const u32 w = wsm[i];
        if (kfloor == 0 || rs_ge(w, i, kfloor)) {
          const int b = (int)((w >> (sh - 16)) & (RS_B - 1));
          if (b == 0) {
            z_lo += by_weight ? (w & 0xFFFFu) : 1u;
            z_hi += by_weight ? (w >> 16) : 0u;
          } else if (!by_weight) {
            atomicAdd(&hist[b], 1u);
          } else {
            atomicAdd(&hist[b], w & 0xFFFFu);
            if (w >> 16) atomicAdd(&hist[RS_B + b], w >> 16);
          }
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        z_lo += __shfl_xor_sync(0xffffffffu, z_lo, o);
        z_hi += __shfl_xor_sync(0xffffffffu, z_hi, o);
      }
      if ((tid & 31) == 0) {
        if (z_lo) atomicAdd(&hist[0], z_lo);
        if (z_hi) atomicAdd(&hist[RS_B], z_hi);
      }
    } else {
      for (int j = tid; j < n; j += GRT_SAMPLE_THREADS) {
        const int i = cand[j];
        add(i, rs_key(wsm, i));
      }
    }
    __syncthreads();
    rs_pick(hist, need, &s_dg, &s_above, wsum);
    const u64 dg = (u64)s_dg;
    need -= s_above;
    prefix |= dg << sh;
    // keep the keys of bucket dg, compacted into cand (order is irrelevant: the
    // select works on the candidate SET, so warp-aggregated slots are fine)
    if (n < 0) {
      if (tid == 0) s_n = 0;
      __syncthreads();
      const int lane = tid & 31;
      for (int base = 0; base < GRT_V; base += GRT_SAMPLE_THREADS) {
        const int i = base + tid;  // consecutive indices per warp: no bank conflicts
        bool f = false;
        if (i < GRT_V) {
          const u32 w = wsm[i];
          f = ((w >> (sh - 16)) & (RS_B - 1)) == (u32)dg && (kfloor == 0 || rs_ge(w, i, kfloor));
        }
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        int slot = 0;
        if (lane == 0 && bal) slot = atomicAdd(&s_n, __popc(bal));
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (f) cand[slot + __popc(bal & ((1u << lane) - 1))] = (unsigned short)i;
      }
      __syncthreads();
      n = s_n;
    } else {
      int out = 0;
      for (int base = 0; base < n; base += GRT_SAMPLE_THREADS) {  // tile: read all, then write
        const int j = base + tid;
        const int i = j < n ? cand[j] : 0;
        const int f = j < n && ((rs_key(wsm, i) >> sh) & (RS_B - 1)) == dg;
        int pos;
        const int total = rs_scan(f, &pos, warp_tot);  // (its barriers order the reads before the writes)
        if (f) cand[out + pos] = (unsigned short)i;
        out += total;
        __syncthreads();
      }
      n = out;
    }
    if (tid == 0) s_n = n;
    __syncthreads();
    n = s_n;
    GRT_STAMP(9 + ps);
    // one candidate left: it is the threshold key (the running total reaches
    // `need` inside its bucket); the remaining passes would only re-derive its
    // low digits.  n <= 0 cannot happen (need <= total at every pass).
    if (n <= 1) break;
  }
  const u64 r = n == 1 ? rs_key(wsm, cand[0]) : prefix;
  __syncthreads();
  return r;
}
#endif

// Returns the sampled token (block-uniform) or -1 on a prefill pass.  With
// fence == false the caller issues the system fence for the host-mapped slots.
__device__ __forceinline__ int sample_impl(GrtCtrl* ctrl, const float* logits, bool fence = true) {
  __shared__ float redf[32];
  __shared__ u64 redu[32];
  __shared__ u64 hist[256];
  __shared__ int s_tok;
  __shared__ u64 s_t0;
  const int pos = ctrl->seq_len;
  if (pos < ctrl->prompt_len) return -1;  // prefill pass: the token is given
  const int step = pos - ctrl->prompt_len;
  if (threadIdx.x == 0) s_t0 = grt_globaltimer();
  const int kind = ctrl->sample_kind;
  const int tid = threadIdx.x;
  const float temperature = ctrl->temperature;

  if (kind == 0 || !(temperature > 0.0f)) {
    // greedy: strict >, lowest index wins ties (kernels.cpp:265-270)
    // every logit load of a thread is issued before the first compare (one
    // memory round trip, not GRT_V / threads dependent ones)
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    constexpr int NV4 = GRT_V / 4;
    constexpr int PER = NV4 > 0 ? (NV4 + GRT_SAMPLE_THREADS - 1) / GRT_SAMPLE_THREADS : 1;
    float4 lv[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j4 = tid + k * GRT_SAMPLE_THREADS;
      lv[k] = j4 < NV4 ? reinterpret_cast<const float4*>(logits)[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j4 = tid + k * GRT_SAMPLE_THREADS;
      if (j4 >= NV4) continue;
      const float e[4] = {lv[k].x, lv[k].y, lv[k].z, lv[k].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (e[c] > bv || bi == 0x7fffffff) {
          bv = e[c];
          bi = 4 * j4 + c;
        }
      }
    }
    for (int i = 4 * NV4 + tid; i < GRT_V; i += GRT_SAMPLE_THREADS) {  // V % 4 tail
      const float v = logits[i];
      if (v > bv || bi == 0x7fffffff) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    __shared__ float sv[32];
    __shared__ int si[32];
    if ((tid & 31) == 0) {
      sv[tid >> 5] = bv;
      si[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid < 32) {
      bv = sv[tid];
      bi = si[tid];
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (tid == 0) s_tok = bi;
    }
    __syncthreads();
  } else if (kind == 1) {
    // temperature, reference-compatible (kernels.cpp:271-288): one uniform01
    // draw per sample (pre-generated by the host from mt19937_64(seed) in step
    // order), fp32 softmax numerators, fp32 denominator summed in ascending
    // index order (serial, as in the reference), inverse CDF walked in double.
    float m = -INFINITY;
    for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) m = fmaxf(m, logits[i]);
    m = block_max_f(m, redf);
    float* probs = ctrl->scratch;
    for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) probs[i] = expf((logits[i] - m) / temperature);
    __syncthreads();
    __shared__ float s_denom;
    if (tid == 0) {
      float denom = 0.0f;
      for (int i = 0; i < GRT_V; ++i) denom += probs[i];
      s_denom = denom;
    }
    __syncthreads();
    const double u = ctrl->uniforms[step] * (double)s_denom;
    // inclusive prefix sums in double over contiguous per-thread blocks
    const int per = (GRT_V + GRT_SAMPLE_THREADS - 1) / GRT_SAMPLE_THREADS;
    const int b0 = tid * per, b1 = min(GRT_V, b0 + per);
    double local = 0.0;
    for (int i = b0; i < b1; ++i) local += (double)probs[i];
    __shared__ double sc[GRT_SAMPLE_THREADS];
    sc[tid] = local;
    __syncthreads();
    if (tid == 0) {
      double acc = 0.0;
      for (int t = 0; t < GRT_SAMPLE_THREADS; ++t) {
        const double v = sc[t];
        sc[t] = acc;
        acc += v;
      }
      s_tok = GRT_V - 1;
    }
    __syncthreads();
    double acc = sc[tid];
    int found = -1;
    for (int i = b0; i < b1; ++i) {
      acc += (double)probs[i];
      if (u < acc) {
        found = i;
        break;
      }
    }
    if (found >= 0) atomicMin(&s_tok, found);
    __syncthreads();
  } else {
    // integer-CDF top-k / top-p (oracle.c:oc_sample_topkp)
#if GRT_TOPKP_SMEM
    // the logits are read ONCE (all loads of a thread in flight together), the
    // weights computed from registers into dynamic shared memory
    GRT_STAMP(0);
#if GRT_TOPKP_SMEM == 2
    // the draw's uniform (Philox over the step index) is known now: computed
    // while the logits load is in flight
    double u_draw;
    {
      u32 c[4] = {(u32)step, (u32)((u64)step >> 32), 0u, 0x53616D70u};
      const u64 seed = ctrl->seed;
      philox4x32_10(c, (u32)seed, (u32)(seed >> 32));
      u_draw = (double)((((u64)c[1] << 32) | (u64)c[0]) >> 11) * 0x1.0p-53;
    }
#endif
    constexpr int NV4 = GRT_V / 4;
    constexpr int PER = NV4 > 0 ? (NV4 + GRT_SAMPLE_THREADS - 1) / GRT_SAMPLE_THREADS : 1;
    float4 lv[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j4 = tid + k * GRT_SAMPLE_THREADS;
      lv[k] = j4 < NV4 ? reinterpret_cast<const float4*>(logits)[j4] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < PER; ++k) m = fmaxf(m, fmaxf(fmaxf(lv[k].x, lv[k].y), fmaxf(lv[k].z, lv[k].w)));
    for (int i = 4 * NV4 + tid; i < GRT_V; i += GRT_SAMPLE_THREADS) m = fmaxf(m, logits[i]);
    m = block_max_f(m, redf);
    extern __shared__ u32 wsm[];  // [GRT_V] weights, computed once (every pass below reads them)
    GRT_STAMP(1);
#if GRT_TOPKP_SMEM == 2
    // The first select's pass-0 histogram (digit = w >> 21; digit 0 summed per
    // thread, added once per warp) and the total weight are accumulated while
    // the weights are computed: the top-k count histogram when top-k is active,
    // else the top-p weight histogram -- one pass over the vocabulary fewer.
    __shared__ u32 rs_hist[2 * RS_B];
    const int top_k = ctrl->top_k;
    const float top_p = ctrl->top_p;
    const bool pre_k = top_k > 0 && top_k < GRT_V;
    const bool pre_p = !pre_k && top_p > 0.0f && top_p < 1.0f;
    for (int b = tid; b < 2 * RS_B; b += GRT_SAMPLE_THREADS) rs_hist[b] = 0;
    __syncthreads();
    u64 W_all = 0;
    u32 z_lo = 0, z_hi = 0;
    auto put = [&](int i, u32 w) {
      wsm[i] = w;
      W_all += w;
      if (pre_k || pre_p) {
        const int b = (int)(w >> 21);
        if (b == 0) {
          z_lo += pre_k ? 1u : (w & 0xFFFFu);
          z_hi += pre_k ? 0u : (w >> 16);
        } else if (pre_k) {
          atomicAdd(&rs_hist[b], 1u);
        } else {
          atomicAdd(&rs_hist[b], w & 0xFFFFu);
          atomicAdd(&rs_hist[RS_B + b], w >> 16);
        }
      }
    };
#else
    auto put = [&](int i, u32 w) { wsm[i] = w; };
#endif
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j4 = tid + k * GRT_SAMPLE_THREADS;
      if (j4 >= NV4) continue;
      put(4 * j4, (u32)topkp_weight_v(lv[k].x, m, temperature));
      put(4 * j4 + 1, (u32)topkp_weight_v(lv[k].y, m, temperature));
      put(4 * j4 + 2, (u32)topkp_weight_v(lv[k].z, m, temperature));
      put(4 * j4 + 3, (u32)topkp_weight_v(lv[k].w, m, temperature));
    }
    for (int i = 4 * NV4 + tid; i < GRT_V; i += GRT_SAMPLE_THREADS) put(i, (u32)topkp_weight(logits, i, m, temperature));
#if GRT_TOPKP_SMEM == 2
    for (int o = 16; o > 0; o >>= 1) {
      z_lo += __shfl_xor_sync(0xffffffffu, z_lo, o);
      z_hi += __shfl_xor_sync(0xffffffffu, z_hi, o);
    }
    if ((tid & 31) == 0) {
      if (z_lo) atomicAdd(&rs_hist[0], z_lo);
      if (z_hi) atomicAdd(&rs_hist[RS_B], z_hi);
    }
#endif
    __syncthreads();
    GRT_STAMP(2);
#define GRT_W(i) ((u64)wsm[i])
#define GRT_GE(w, i, floor) rs_ge((u32)(w), (i), (floor))
#else
    float m = -INFINITY;
    for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) m = fmaxf(m, logits[i]);
    m = block_max_f(m, redf);
#define GRT_W(i) topkp_weight(logits, (i), m, temperature)
#define GRT_GE(w, i, floor) (topkp_key((w), (i)) >= (floor))
#endif
#if GRT_TOPKP_SMEM == 2
    unsigned short* cand = (unsigned short*)(wsm + GRT_V);
    // (1) top-k threshold key: the top_k-th largest key
    u64 kth = 0;
    if (pre_k) kth = radix_select_compact(wsm, cand, 0, false, (u64)top_k, rs_hist, true);
    GRT_STAMP(3);
    // (2) top-p threshold key among keys >= kth
    u64 W = 0;
    if (kth == 0) {
      W = W_all;  // every key counts
    } else {
      for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) {
        const u64 w = GRT_W(i);
        if (GRT_GE(w, i, kth)) W += w;
      }
    }
    W = block_sum_u64(W, redu);
    u64 kappa = kth;
    GRT_STAMP(4);
    if (top_p > 0.0f && top_p < 1.0f) {
      u64 thresh = (u64)((double)top_p * (double)W);
      if (thresh < 1) thresh = 1;
      const u64 kp = radix_select_compact(wsm, cand, kth, true, thresh, rs_hist, pre_p);
      kappa = kp > kth ? kp : kth;
    }
    GRT_STAMP(5);
#else
    const int top_k = ctrl->top_k;
    const float top_p = ctrl->top_p;
    // (1) top-k threshold key
    u64 kth = 0;
    if (top_k > 0 && top_k < GRT_V) {
      u64 prefix = 0, mask = 0, need = (u64)top_k;
      for (int shift = 40; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += GRT_SAMPLE_THREADS) hist[b] = 0;
        __syncthreads();
        u64 zero = 0;  // digit 0 (tiny weights: most of the vocabulary) summed locally, one atomic per warp
        for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) {
          const u64 key = topkp_key(GRT_W(i), i);
          if ((key & mask) == prefix) {
            const int b = (int)((key >> shift) & 255);
            if (b == 0) zero += 1ull;
            else atomicAdd(&hist[b], 1ull);
          }
        }
        for (int o = 16; o > 0; o >>= 1) zero += __shfl_xor_sync(0xffffffffu, zero, o);
        if ((tid & 31) == 0 && zero) atomicAdd(&hist[0], zero);
        __syncthreads();
        radix_pick(hist, shift, prefix, mask, need);
      }
      kth = prefix;
    }
    // (2) top-p threshold key among keys >= kth
    u64 W = 0;
    for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) {
      const u64 w = GRT_W(i);
      if (topkp_key(w, i) >= kth) W += w;
    }
    W = block_sum_u64(W, redu);
    u64 kappa = kth;
    if (top_p > 0.0f && top_p < 1.0f) {
      u64 thresh = (u64)((double)top_p * (double)W);
      if (thresh < 1) thresh = 1;
      u64 prefix = 0, mask = 0, need = thresh;
      for (int shift = 40; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += GRT_SAMPLE_THREADS) hist[b] = 0;
        __syncthreads();
        u64 zero = 0;
        for (int i = tid; i < GRT_V; i += GRT_SAMPLE_THREADS) {
          const u64 w = GRT_W(i);
          const u64 key = topkp_key(w, i);
          if (key >= kth && (key & mask) == prefix) {
            const int b = (int)((key >> shift) & 255);
            if (b == 0) zero += w;
            else atomicAdd(&hist[b], w);
          }
        }
        for (int o = 16; o > 0; o >>= 1) zero += __shfl_xor_sync(0xffffffffu, zero, o);
        if ((tid & 31) == 0 && zero) atomicAdd(&hist[0], zero);
        __syncthreads();
        radix_pick(hist, shift, prefix, mask, need);
      }
      kappa = prefix > kth ? prefix : kth;
    }
#endif
#if GRT_TOPKP_SMEM == 2
    // (3) draw and inverse CDF in index order over the kept set: warp w owns the
    // contiguous index block [w*VB, (w+1)*VB) and its lanes read consecutive
    // indices (no bank conflicts); warp totals are scanned in warp order, the
    // warp holding the draw walks its block 32 indices at a time (integer
    // prefix sums: the serial walk's result exactly)
    {
      constexpr int NW = GRT_SAMPLE_THREADS / 32;
      constexpr int VB = ((GRT_V + NW - 1) / NW + 31) / 32 * 32;
      __shared__ u64 wtot[NW];
      __shared__ u64 s_S2;
      const int lane = tid & 31, wp = tid >> 5;
      const int i0 = wp * VB, i1 = min(GRT_V, i0 + VB);
      u64 t = 0;
      for (int i = i0 + lane; i < i1; i += 32) {
        const u64 w = GRT_W(i);
        if (GRT_GE(w, i, kappa)) t += w;
      }
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) wtot[wp] = t;
      if (tid == 0) s_tok = 0x7fffffff;
      __syncthreads();
      GRT_STAMP(7);
      if (wp == 0) {
        const u64 v = wtot[lane];
        u64 incl = v;
        for (int o = 1; o < 32; o <<= 1) {
          const u64 n2 = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += n2;
        }
        wtot[lane] = incl - v;  // exclusive
        if (lane == 31) s_S2 = incl;
      }
      __syncthreads();
      GRT_STAMP(8);
      const u64 S = s_S2;
      u64 r = (u64)(u_draw * (double)S);
      if (r >= S) r = S - 1;
      u64 acc = wtot[wp];
      if (S > 0 && acc <= r && r < acc + t) {  // this warp's block holds the draw
        // lane c sums chunk c = indices [i0 + 32c, i0 + 32c + 32) (rotated reads:
        // no bank conflicts), a scan over the 32 chunk sums finds the chunk, a
        // scan inside it the index -- the serial walk's token exactly
        static_assert(VB <= 32 * 32, "one chunk per lane");
        const int cb = i0 + 32 * lane;
        u64 cs = 0;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const int i = cb + ((k + lane) & 31);
          if (i < i1) {
            const u64 w = GRT_W(i);
            if (GRT_GE(w, i, kappa)) cs += w;
          }
        }
        u64 cincl = cs;
        for (int o = 1; o < 32; o <<= 1) {
          const u64 n2 = __shfl_up_sync(0xffffffffu, cincl, o);
          if (lane >= o) cincl += n2;
        }
        const unsigned hc = __ballot_sync(0xffffffffu, acc + cincl > r);
        const int ch = __ffs(hc) - 1;  // r < acc + t: some chunk reaches it
        acc += __shfl_sync(0xffffffffu, cincl - cs, ch);
        const int base = i0 + 32 * ch, i = base + lane;
        u64 w = 0;
        if (i < i1) {
          w = GRT_W(i);
          if (!GRT_GE(w, i, kappa)) w = 0;
        }
        u64 incl = w;
        for (int o = 1; o < 32; o <<= 1) {
          const u64 n2 = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += n2;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, w > 0 && acc + incl > r);
        if (lane == 0 && hit) s_tok = base + __ffs(hit) - 1;
      }
      __syncthreads();
    }
#else
    // (3) draw and inverse CDF in index order over the kept set
    const int per = (GRT_V + GRT_SAMPLE_THREADS - 1) / GRT_SAMPLE_THREADS;
    const int b0 = tid * per, b1 = min(GRT_V, b0 + per);
    u64 local = 0;
    for (int i = b0; i < b1; ++i) {
      const u64 w = GRT_W(i);
      if (topkp_key(w, i) >= kappa) local += w;
    }
    // exclusive prefix of the per-thread sums in thread order (parallel scan;
    // integer, so identical to the serial walk)
    __shared__ u64 sc[GRT_SAMPLE_THREADS];
    __shared__ u64 wsum[32];
    __shared__ u64 s_S;
    {
      const int lane = tid & 31, wp = tid >> 5;
      u64 v = local;
      for (int o = 1; o < 32; o <<= 1) {
        const u64 n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
      }
      if (lane == 31) wsum[wp] = v;
      __syncthreads();
      if (wp == 0) {
        u64 t = lane < (GRT_SAMPLE_THREADS >> 5) ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const u64 n = __shfl_up_sync(0xffffffffu, t, o);
          if (lane >= o) t += n;
        }
        wsum[lane] = t;
        if (lane == 31) s_S = t;
      }
      if (tid == 0) s_tok = 0x7fffffff;
      __syncthreads();
      sc[tid] = v - local + (wp > 0 ? wsum[wp - 1] : 0);
    }
    __syncthreads();
    const u64 S = s_S;
    u32 c[4] = {(u32)step, (u32)((u64)step >> 32), 0u, 0x53616D70u};
    const u64 seed = ctrl->seed;
    philox4x32_10(c, (u32)seed, (u32)(seed >> 32));
    const u64 bits = (((u64)c[1] << 32) | (u64)c[0]) >> 11;
    const double u = (double)bits * 0x1.0p-53;
    u64 r = (u64)(u * (double)S);
    if (r >= S) r = S - 1;
    u64 acc = sc[tid];
    if (S > 0 && acc <= r && r < acc + local) {
      for (int i = b0; i < b1; ++i) {
        const u64 w = GRT_W(i);
        if (topkp_key(w, i) < kappa) continue;
        acc += w;
        if (acc > r) {
          s_tok = i;
          break;
        }
      }
    }
    __syncthreads();
#endif
  }

  GRT_STAMP(6);
  if (tid == 0) {
    const int tok = s_tok;
    ctrl->tokens[pos] = tok;
    if (step < ctrl->max_gen) {
      ctrl->out_tokens[step] = tok;
      ctrl->out_stamps[2 * step] = s_t0;
      ctrl->out_stamps[2 * step + 1] = grt_globaltimer();
    }
    if (fence) __threadfence_system();
  }
  return s_tok;
}

extern "C" __global__ void __launch_bounds__(GRT_SAMPLE_THREADS) grt_sample(GrtCtrl* ctrl, const float* logits) {
  grt_launch_dependents();
  grt_griddep_wait();
  sample_impl(ctrl, logits);
}

// The fused dynamic block of one step (pipeline.cpp:87-93, submit_fused_block):
// sample_token from the previous pass's logits, then extend_position + slot
// append for the token just produced -- one launch instead of two.
extern "C" __global__ void __launch_bounds__(GRT_SAMPLE_THREADS)
    grt_sample_preprocess(GrtCtrl* ctrl, const float* logits, const void* emb, const void* pos_table, float* x) {
  grt_launch_dependents();
  grt_griddep_wait();
  const int pos = ctrl->seq_len;
  const int tok = sample_impl(ctrl, logits, false);  // block-uniform
  if (tok >= 0 && tok < GRT_V && pos < GRT_MAXSEQ) {
    // the token is known here: no re-read of seq_len / tokens[pos]
    gather_row(ctrl, pos, tok, emb, pos_table, x);
  } else {
    __syncthreads();  // tokens[seq_len] (given or sampled) visible block-wide
    preprocess_impl(ctrl, emb, pos_table, x);
  }
  if (threadIdx.x == 0) __threadfence_system();  // host-mapped token + stamps
}
