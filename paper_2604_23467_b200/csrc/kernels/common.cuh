// common.cuh -- sm_100a device helpers shared by the decode kernels:
// mbarrier + cp.async.bulk (TMA engine) staging, PDL grid-dependency control,
// bf16 packing, warp reductions.  Inline PTX only; no CUTLASS/CuTe.
#pragma once

#include <cuda_bf16.h>
#include <cstdint>

#include "kernels.h"

namespace grt {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- Programmatic Dependent Launch -------------------------------------------
// Every kernel on the step path is launched with programmatic stream
// serialization.  It lets the NEXT kernel launch immediately and only blocks on
// our completion at its own griddep_wait(), so weight prefetch (which does not
// depend on the previous kernel) overlaps the previous kernel's tail.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarrier -------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Orders this thread's prior generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) writes into the same buffer (WAR on a ring slot).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// L2 policy for weights: streamed exactly once per token, so evict first and
// keep the KV cache / activations resident in the 126 MB L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// cp.async.bulk global -> shared (TMA engine, SASS UBLKCP), completion counted
// on an mbarrier in bytes.  dst/src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Bulk L2 prefetch (TMA engine, fire and forget): pulls [src, src+bytes) into L2
// without occupying shared memory.  src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// one stamp per CTA (thread 0), only when tracing is on
constexpr int OP_TRACE_STRIDE = 8;
__device__ __forceinline__ void op_stamp(unsigned long long* tr, int i) {
  if (tr && threadIdx.x == 0) {
    const int cta = blockIdx.x + blockIdx.y * gridDim.x;
    tr[cta * OP_TRACE_STRIDE + i] = gtimer();
  }
}

// ---- numerics -----------------------------------------------------------------
// Sum of squares of a float4 with an explicit FMA chain: one contraction
// pattern for every kernel that must agree bit for bit (prefill RMSNorm).
__device__ __forceinline__ float sumsq4(float4 a) {
  return __fmaf_rn(a.w, a.w, __fmaf_rn(a.z, a.z, __fmaf_rn(a.y, a.y, __fmul_rn(a.x, a.x))));
}

// Row of position j of `head` in a layer's K or V cache (KvPaging, kernels.h).
__device__ __forceinline__ int64_t kv_row(const KvPaging& g, int head, int max_seq, int j) {
  if (g.page == 0) return static_cast<int64_t>(head) * max_seq + j;
  const int pi = j / g.page;
  return (static_cast<int64_t>(__ldg(g.table + pi)) * g.n_heads + head) * g.page + (j - pi * g.page);
}

// L2 prefetch of rows [0, n) of one head's K or V cache: one bulk request per
// contiguous run of <= 64 KB (a page, or the whole head when contiguous).
__device__ __forceinline__ void kv_prefetch_l2(const void* cache, const KvPaging& g, int head, int max_seq, int dh,
                                               int eb, int n) {
  const uint8_t* b = static_cast<const uint8_t*>(cache);
  const int run = g.page == 0 ? n : g.page;
  for (int j = 0; j < n; j += run) {
    const uint8_t* base = b + kv_row(g, head, max_seq, j) * dh * eb;
    const uint64_t bytes = static_cast<uint64_t>(min(run, n - j)) * dh * eb;
    for (uint64_t o = 0; o < bytes; o += 65536)
      prefetch_l2_bulk(base + o, static_cast<uint32_t>(bytes - o < 65536 ? bytes - o : 65536));
  }
}

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__device__ __forceinline__ T load_elem(const T* p, int64_t i) {
  return p[i];
}
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ void store_cast(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_cast(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

}  // namespace grt
