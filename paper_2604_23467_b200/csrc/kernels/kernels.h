// kernels.h -- host-side declarations of the sm_100a decode kernels.
//
// Plain CUDA runtime types only (no torch).  Each launcher enqueues one kernel
// on `stream`, optionally with Programmatic Dependent Launch so the kernel's
// weight prefetch overlaps the previous kernel (see common.cuh).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "../jit/ctrl.h"

namespace grt {

enum class Dt : int { F32 = 0, BF16 = 1 };

// KV cache addressing.  page == 0: contiguous rows per head, row(head, j) =
// head*max_seq + j (the reference KvCache layout, kv_cache.hpp:15-43).
// page > 0: paged pool [n_pages][n_heads][page][dh] (vLLM-style); position j
// lives in page table[j / page] at offset j % page.  Row r starts at r*dh.
struct KvPaging {
  int page = 0;
  int n_heads = 0;
  const int* table = nullptr;
};

enum NormKind : int { NORM_NONE = 0, NORM_LN = 1, NORM_RMS = 2 };

// Epilogues of the fused GEMV.  Rows are processed in adjacent PAIRS (2p, 2p+1)
// of the device weight layout; the pairing is what lets RoPE (rotate-half) and
// SwiGLU (gate,up) finish inside the GEMV.
enum EpiKind : int {
  EPI_STORE = 0,     // out[r] = v                                  (LM head, plain GEMV)
  EPI_RESID = 1,     // out[r] += v   (residual add, kernels.cpp:162-174) (Wo, W2/down)
  EPI_QKV = 2,       // q -> q_out, k/v -> KV row seq_len-1 (kernels.cpp:188-203)
  EPI_QKV_ROPE = 3,  // as EPI_QKV with rotate-half RoPE on q,k (LLaMA)
  EPI_SWIGLU = 4,    // act[p] = silu(gate_p) * up_p                 (LLaMA gate/up)
  EPI_RELU = 5,      // act[r] = max(v, 0)  (make_relu, kernels.cpp:176-186) (ref W1)
};

struct GemvParams {
  const void* w = nullptr;  // [n_rows, k] row-major device layout (transposed reference [k,n])
  int n_rows = 0;
  int k = 0;
  int rowb = 0;             // bytes of one row chunk slot in shared memory (set by the launcher)
  int ch = 0, nch = 0;      // k-chunk elements and chunks per row (set by the launcher)
  int chmax = 0;            // max chunk elements (0 = default 2048 bf16): stage size per task
  int stages = 0;           // ring slots per warp (set by the launcher from the smem budget)
  int pre_stages = 0;       // slots filled before the dependency wait (0 = all; set by the launcher)
  int l2_pre = 0;           // tasks per warp beyond the ring prefetched into L2 before the wait (launcher)
  int rms_defer = 1;        // RMSNorm: apply 1/rms to the dot products (epilogue) instead of to x
  const float* x = nullptr; // input activation [k] fp32
  const float* gamma = nullptr;
  const float* beta = nullptr;
  float eps = 1e-5f;
  float* out = nullptr;     // STORE / RESID / SWIGLU / RELU target
  // QKV epilogue
  float* q_out = nullptr;
  void* k_cache = nullptr;  // this layer's K [h][max_seq][dh]
  void* v_cache = nullptr;
  const int* seq_len = nullptr;  // device-resident live length; row written = seq_len-1
  const float* rope_cos = nullptr;  // [max_seq][dh/2]
  const float* rope_sin = nullptr;
  int n_heads = 0, head_dim = 0, max_seq = 0, d_model = 0;
  int kv_bf16 = 0;
  KvPaging kvp;
  int* err = nullptr;       // device error word (WrongLength / CacheFull flags)
  unsigned long long* trace = nullptr;  // optional [cta][4] %globaltimer stamps (profiling)
};

struct AttnParams {
  const float* q = nullptr;      // [h*dh], post-RoPE
  const void* k_cache = nullptr; // [h][max_seq][dh]
  const void* v_cache = nullptr;
  float* out = nullptr;          // [h*dh]
  float* part = nullptr;         // [h][nsplit][dh+2] split partials
  int* counters = nullptr;       // [h] arrival counters (self-resetting)
  const int* seq_len = nullptr;  // device live length (nullptr -> len_fixed)
  int len_fixed = 0;
  int n_heads = 0, head_dim = 0, max_seq = 0;
  int span_cap = 0;              // max positions per split CTA (smem sizing)
  float scale = 1.0f;
  int* err = nullptr;
  unsigned long long* trace = nullptr;  // optional [cta][4] %globaltimer stamps (profiling)
  int rounds = 1;                // passes per CTA (set by the launcher)
  KvPaging kvp;
  int trigger = 0;               // when the successor may launch: 0 start, 1 after KV loads, 2 at exit
  int prefetch = 0;              // round 0's rows of earlier steps loaded before the dependency wait
  int smem_rounds = 0;           // rounds 1..smem_rounds staged into shared memory before the wait (launcher)
  int max_len = 0;               // the bucket's last length: longer live lengths flag DEVERR_WRONG_LENGTH (launcher)
};
// Per-op trace stamps (8 slots per CTA): 0 CTA start, 1 dependency released
// (griddepcontrol.wait), 2 operands ready (activation loaded / KV rows loaded),
// 3 CTA done, 4 first weight stage landed, 5 streaming loop done.
constexpr int OP_TRACE_CTAS = 1024;  // stamp slots per kernel in a traced plan

// Device error flags (bit set by kernels, read by the host after a run).
enum DevErr : int {
  DEVERR_WRONG_LENGTH = 1,  // live seq_len outside the graph bucket
  DEVERR_CACHE_FULL = 2,
  DEVERR_TOKEN_RANGE = 4,
  DEVERR_TIMEOUT = 8,       // persistent pass watchdog (a CTA never arrived)
};

int num_sms(int device);

// Fused (norm) + GEMV + epilogue.  grid_ctas <= 0 picks one CTA per SM.
cudaError_t launch_gemv(Dt wdt, int norm, int epi, GemvParams p, cudaStream_t s, bool pdl, int grid_ctas);
size_t gemv_smem_bytes(Dt wdt, int k);
cudaError_t gemv_prepare(int device);  // raises the dynamic smem limit once per process

// Two consecutive decode GEMVs in one launch (gemv_pair.cu): a = residual GEMV
// (Wo: NORM_NONE, EPI_RESID), b = the RMS-normed gate/up GEMV on its output
// (EPI_SWIGLU), grid-wide barrier in between (one CTA per SM); bf16 weights.
struct GemvPairParams {
  GemvParams a, b;
  int* bar = nullptr;  // [2] arrive/depart counters, zero-initialised, self-resetting
  int* err = nullptr;
  int stages = 0, rowb = 0, xs_floats = 0;  // set by the launcher
};
cudaError_t launch_gemv_pair(int epi_b, GemvPairParams p, cudaStream_t s, bool pdl);

cudaError_t gemv_pair_prepare();

// Split-K flash-decode over the KV cache for live lengths up to max_len (the
// graph bucket's end): one thread-block cluster per head, partials merged over
// distributed shared memory.  Writes out[h*dh].
cudaError_t launch_attention(Dt kvdt, AttnParams p, int max_len, cudaStream_t s, bool pdl);
int attention_nsplit(int max_len, int n_heads, int sms);  // split partial buffer sizing (AttnParams::part)
int attention_splits(int max_len, int head_dim);         // cluster size of attn_decode_kernel for a bucket
cudaError_t attention_prepare();

// ---- batched prefill (prefill_gemm.cu, prefill.cu) ------------------------------
enum PgEpi : int {
  PG_EPI_STORE = 0,     // out[n][m] = v
  PG_EPI_RESID = 1,     // out[n][m] += v          (Wo, down: residual stream X)
  PG_EPI_SWIGLU = 2,    // out_bf16[n][m/2] = silu(gate) * up   (rows 2j, 2j+1)
  PG_EPI_QKV = 3,       // q -> q_out[n], k/v -> KV rows start_pos + n
  PG_EPI_QKV_ROPE = 4,  // as QKV with rotate-half RoPE at position start_pos + n
  PG_EPI_RELU = 5,      // out_bf16[n][m] = max(v, 0)  (reference arch W1, make_relu kernels.cpp:176-186)
};
struct PrefillGemmParams {
  int M = 0, K = 0, P = 0;  // Y[P, M] = X[P, K] . W[M, K]^T  (bf16 operands, fp32 accumulate)
  int ntile = 0, n_ntiles = 0, ksplit = 1, stages = 0, kbox = 1;  // set by the launcher
  // stream-K tail (set by the launcher; ksplit == 1 only): tiles [tail_first,
  // m_tiles*n_ntiles) -- the last, partial wave -- are split tail_ks ways in K
  // so their units fill the SMs; their partials go through a reduce kernel
  int tail_first = 0, tail_ks = 0;
  int box3d = 0;      // set by the launcher: both maps are 3D ({64, rows, K/64}): one TMA box per stage and operand
  int epi_stage = 0;  // set by the launcher: QKV epilogue through per-warp shared-memory staging
  int epi = PG_EPI_STORE;
  float* out = nullptr;
  void* out_bf16 = nullptr;
  float* q_out = nullptr;  // [P][d_model]
  void* k_cache = nullptr;
  void* v_cache = nullptr;
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  int head_dim = 0, max_seq = 0, d_model = 0, start_pos = 0, kv_bf16 = 0;
  KvPaging kvp;
  int defer_reduce = 0;    // PG_EPI_RESID + split K: leave the partials for launch_prefill_resid_norm
  int wide_split = 0;      // allow split K for P > 256 (partials through the reduce kernel)
  float* part = nullptr;   // split-K scratch, prefill_gemm_part_floats()
  int* counters = nullptr; // [m_tiles], zero-initialised, self-resetting
};
// tcgen05/TMEM GEMM; w: bf16 [M, K] row-major (the device weight layout), x:
// bf16 [P, K] row-major (P <= 512), both K % 64 == 0.
cudaError_t launch_prefill_gemm(const void* w, const void* x, PrefillGemmParams p, cudaStream_t s, bool pdl);
// same; writes the chosen tiling (ntile, n_ntiles, ksplit) back into *p
cudaError_t launch_prefill_gemm_ex(const void* w, const void* x, PrefillGemmParams* p, cudaStream_t s, bool pdl);
// Deferred split-K reduce of a residual GEMM fused with the RMSNorm that reads
// its output: X[n] += sum_s partial_s[n] (split order), Xn[n] = bf16(rmsnorm(X[n])
// * gamma) -- one launch instead of the reduce kernel + prefill_rmsnorm.
cudaError_t launch_prefill_resid_norm(const PrefillGemmParams& p, const float* gamma, float eps, void* Xn,
                                      cudaStream_t s);
cudaError_t prefill_gemm_prepare();
int prefill_gemm_ksplit(int M, int K, int sms);
size_t prefill_gemm_part_floats(int M, int K, int P, int sms);
constexpr int PREFILL_CHUNK = 512;  // tokens per batched pass (two 256-token TMEM accumulators)
cudaError_t launch_prefill_embed(Dt wdt, const int* tokens, int start, int P, const void* emb, const void* pos, int d,
                                 float* X, int vocab, int* err, cudaStream_t s);  // pos: nullptr for LLaMA
cudaError_t launch_prefill_layernorm(const float* X, int P, const float* gamma, const float* beta, float eps, int d,
                                     void* Xn, cudaStream_t s);
cudaError_t launch_prefill_rmsnorm(const float* X, int P, const float* gamma, float eps, int d, void* Xn,
                                   cudaStream_t s);
cudaError_t launch_prefill_attention(Dt kvdt, const float* Q, const void* k, const void* v, int start, int P, int d,
                                     int n_heads, int dh, int max_seq, float scale, void* out, cudaStream_t s,
                                     KvPaging kvp = KvPaging{});
cudaError_t launch_prefill_handoff(const float* X_last, int d, float* x, int* seq_len, int len, cudaStream_t s);

// ---- tensor-parallel exchange, in-process emulation (tp_emu.cu) ----------------
constexpr int TP_MAX = 8;
struct TpPtrs {
  float* p[TP_MAX];
};
cudaError_t launch_emu_allreduce(const TpPtrs& bufs, int T, size_t n, cudaStream_t s);
cudaError_t launch_emu_allgather(const TpPtrs& in, const TpPtrs& out, int T, size_t n, cudaStream_t s);

// Weight materialisation: writes a logical reference-layout tensor into its
// device layout.  `src` (host-copied, fp32 or bf16 on device) or Philox init.
struct MapDesc {
  int64_t rows = 0, cols = 0;   // logical reference shape ([k,n] for matrices, [V,d] tables)
  int transpose = 0;            // 1: matrix, physical row = f(j), col = p
  int64_t ld = 0;               // physical row length (k) when transposed
  int64_t row_base = 0;         // first physical row of this tensor's block
  int row_stride = 1;           // 2 for interleaved gate/up
  int row_offset = 0;           // 0 gate, 1 up
  int rope_pair = 0;            // permute j within heads: (i, i+half) -> (2i, 2i+1)
  int head_dim = 0;
  int dst_dtype = 0;            // Dt
  // Tensor-parallel shard window of the logical tensor: logical rows [p0, p1)
  // (row-parallel: input dims) x columns [j0, j1) (column-parallel: outputs).
  // Values are drawn at their LOGICAL index, so a shard holds exactly the
  // entries of the full model; physical positions are window-relative.
  // p1 == 0 / j1 == 0 mean "to the end".
  int64_t p0 = 0, p1 = 0, j0 = 0, j1 = 0;
};
cudaError_t launch_map_init(const MapDesc& d, void* dst, uint64_t seed, uint32_t tensor_id, cudaStream_t s);
// src holds the logical tensor [rows, cols] row-major, or [cols, rows] when src_out_in
// (src_dtype: 0 f32, 1 bf16, 2 f16)
cudaError_t launch_map_copy(const MapDesc& d, void* dst, const void* src, int src_dtype, bool src_out_in,
                            cudaStream_t s);
cudaError_t launch_map_read(const MapDesc& d, const void* dst, float* out_ref_layout, cudaStream_t s);

// ---- device-resident decode loop (loop.cu) ----
enum LoopStatus : int { LOOP_EOS = 1, LOOP_NO_BUCKET = 2 };
struct LoopCtl {
  int remaining;  // decode steps still to run
  int bucket;     // KV positions per graph key
  int key_lo;     // bucket key of switch body 0
  int n_keys;     // switch bodies
  int eos;        // stop token (-1 = none)
  int iters;      // steps executed (device count)
  int status;     // LoopStatus bits
  int pad;
};
cudaError_t launch_loop_ctl(const GrtCtrl* ctrl, LoopCtl* lc, cudaGraphConditionalHandle h_while,
                            cudaGraphConditionalHandle h_switch, cudaStream_t s);

}  // namespace grt
