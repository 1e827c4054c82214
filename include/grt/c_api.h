/*
 * grt/c_api.h -- C ABI of the B200-native graphrt decode path.
 *
 * Every entry point replaces one piece of the reference's C++ runtime/operator
 * API (reference = /root/reference/proj/core, namespace graphrt).  Plain C types,
 * opaque handles, caller-owned host buffers, no exceptions: every call returns a
 * grt_status whose numbering is the reference Errc list (error.hpp:10-39) in
 * declaration order, followed by the device-side codes.
 *
 * Threading: one host thread per session (the reference is single-threaded,
 * SPEC.md:217); sessions on different devices may run concurrently.  The library
 * runs its own capture thread internally (asynchronous graph capture).
 */
#ifndef GRT_C_API_H
#define GRT_C_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRT_ABI_VERSION 2

/* Replaces graphrt::Errc (error.hpp:10-39) + Error exceptions. */
typedef enum grt_status {
  GRT_OK = 0,
  GRT_ShapeMismatch = 1,
  GRT_TokenOutOfRange = 2,
  GRT_EmptyCache = 3,
  GRT_CacheFull = 4,
  GRT_InvalidConfig = 5,
  GRT_LengthOutOfRange = 6,
  GRT_PromptTooLong = 7,
  GRT_EmptyPrompt = 8,
  GRT_CaptureInProgress = 9,
  GRT_CaptureViolation = 10,
  GRT_ForeignBuffer = 11,
  GRT_SessionClosed = 12,
  GRT_EmptyCapture = 13,
  GRT_ReplayShapeError = 14,
  GRT_WrongLength = 15,
  GRT_KeyMismatch = 16,
  GRT_WarmupExceedsCapacity = 17,
  GRT_StaticInFusedBlock = 18,
  GRT_DeviceStopped = 19,
  GRT_UnknownEvent = 20,
  GRT_EmptySamples = 21,
  GRT_IoError = 22,
  /* device-side failures (no reference counterpart) */
  GRT_CudaError = 100,
  GRT_NvrtcError = 101,
  GRT_NcclError = 102,
  GRT_IpcError = 103,
  GRT_Unsupported = 104,
  GRT_NoDevice = 105
} grt_status;

typedef enum grt_arch { GRT_ARCH_REF = 0, GRT_ARCH_LLAMA = 1 } grt_arch;
typedef enum grt_dtype { GRT_F32 = 0, GRT_BF16 = 1, GRT_F16 = 2 /* host/checkpoint data only */ } grt_dtype;
typedef enum grt_init { GRT_INIT_MT19937 = 0, GRT_INIT_PHILOX = 1, GRT_INIT_NONE = 2 } grt_init;

/* Replaces graphrt::RunMode (pipeline.hpp:18-24) -- same order. */
typedef enum grt_run_mode {
  GRT_MODE_EAGER = 0,
  GRT_MODE_HYBRID = 1,
  GRT_MODE_GRAPH_ONLY = 2,
  GRT_MODE_ABLATE_ASYNC = 3,
  GRT_MODE_ABLATE_FUSED = 4,
  GRT_MODE_ABLATE_BOTH = 5,
  /* extension: the whole decode is ONE graph launch -- a
   * conditional WHILE node over [dynamic block, bucket SWITCH of static passes] */
  GRT_MODE_DEVICE_LOOP = 6
} grt_run_mode;

/* Replaces graphrt::EvictionPolicy (graph_cache.hpp:13). */
typedef enum grt_eviction { GRT_EVICT_LEAST_USED = 0, GRT_EVICT_LRU = 1 } grt_eviction;

/* Replaces graphrt::StepPath (pipeline.hpp:43). */
typedef enum grt_step_path {
  GRT_PATH_REPLAYED = 0,
  GRT_PATH_EAGER_FALLBACK = 1,
  GRT_PATH_BATCHED = 2,        /* extension: prompt served by the batched (tcgen05) prefill, launched eagerly */
  GRT_PATH_BATCHED_REPLAYED = 3 /* extension: the batched prefill replayed as one graph (per prompt length) */
} grt_step_path;

/* Replaces graphrt::SampleStrategy (kernels.hpp:105-115), extended with top-k/top-p. */
typedef enum grt_sample_kind {
  GRT_SAMPLE_GREEDY = 0,
  GRT_SAMPLE_TEMPERATURE = 1, /* reference-compatible: mt19937_64 uniform01, inverse CDF */
  GRT_SAMPLE_TOPKP = 2        /* integer-CDF top-k/top-p, Philox4x32-10 draws */
} grt_sample_kind;

/* Replaces graphrt::ModelConfig (model.hpp:17-29), extended for LLaMA/bf16/TP. */
typedef struct grt_model_config {
  int32_t arch;        /* grt_arch */
  int32_t n_layers;
  int32_t d_model;
  int32_t n_heads;
  int32_t vocab_size;
  int32_t max_seq_len;
  int32_t d_ff;        /* 0 => 4*d_model (model.hpp:26) */
  float norm_eps;      /* ln_eps (model.hpp:23) */
  uint64_t seed;       /* weight init seed (model.hpp:24) */
  int32_t init;        /* grt_init */
  int32_t weight_dtype;/* grt_dtype */
  int32_t kv_dtype;    /* grt_dtype */
  float rope_theta;
  int32_t device;      /* CUDA ordinal */
  int32_t tp_size;     /* 1 = single GPU */
  int32_t tp_rank;
  int32_t kv_page_size; /* 0 = contiguous KV [h][max_seq][dh] per layer (kv_cache.hpp:15-43);
                           > 0 = paged pool [n_pages][h][page][dh] addressed through a block table */
} grt_model_config;

/* Replaces graphrt::CacheConfig (pipeline.hpp:122-128), plus the bucket width. */
typedef struct grt_cache_config {
  uint64_t capacity;
  int32_t warmup_lo;
  int32_t warmup_hi;
  int32_t prefill_uses_graphs;
  int32_t policy;      /* grt_eviction */
  int32_t bucket_size; /* KV positions per graph key; 1 = the reference's exact-length keys */
  int32_t batched_prefill; /* 1 = one batched prefill pass (TTFT path); 0 = token-by-token like the reference */
  int32_t pass_impl;   /* 1 = the per-op kernel graph, 4 kernels per layer (the only supported value) */
  int32_t prefill_fuse_norm; /* 1 (default): a split-K residual GEMM of the batched prefill hands its partials
                                to the next RMSNorm launch (bit-identical to 0: separate reduce + norm) */
} grt_cache_config;

typedef struct grt_sample_params {
  int32_t kind;        /* grt_sample_kind */
  float temperature;
  int32_t top_k;       /* 0 = off */
  float top_p;         /* >= 1 = off */
  uint64_t seed;       /* sampler_seed (pipeline.hpp:138) */
} grt_sample_params;

/* Replaces graphrt::GenerationRequest (pipeline.hpp:133-141). */
typedef struct grt_generation_request {
  int32_t mode;        /* grt_run_mode */
  const int32_t* prompt;
  int32_t prompt_len;
  int32_t gen_len;
  grt_sample_params sampling;
  int32_t stop_on_eos; /* GRT_MODE_DEVICE_LOOP: nonzero = stop after sampling eos_token (zero-init: off) */
  int32_t eos_token;
} grt_generation_request;

/* Replaces graphrt::Counters (virtual_device.hpp:41-49) with real counts. */
typedef struct grt_counters {
  uint64_t dispatches;       /* host submissions (kernel launches + graph launches) */
  uint64_t kernel_launches;  /* kernels launched directly by the host */
  uint64_t fused_blocks;     /* dynamic blocks launched outside a graph */
  uint64_t graph_replays;    /* cudaGraphLaunch calls */
  uint64_t captures;         /* graphs captured + instantiated */
  uint64_t events_recorded;
  uint64_t events_waited;
  uint64_t graph_kernel_nodes; /* kernels executed inside replayed graphs */
} grt_counters;

/* Replaces graphrt::CacheStats (graph_cache.hpp:18-24). */
typedef struct grt_cache_stats {
  uint64_t hits, misses, inserts, evictions, releases;
} grt_cache_stats;

/* Replaces graphrt::GenerationResult (pipeline.hpp:143-159).  Array fields are
 * caller-owned buffers of the stated length (NULL = not requested). */
typedef struct grt_generation_result {
  int32_t* tokens;          /* [gen_len] */
  double* per_token_us;     /* [gen_len]; [0] measured from prefill completion */
  int32_t* prefill_paths;   /* [prompt_len] grt_step_path (or [1] for a batched prefill) */
  int32_t* decode_paths;    /* [gen_len] */
  double ttft_us;           /* request entry -> first token visible on the host */
  double total_us;          /* request entry -> everything retired */
  double prefill_us;        /* device time of the prefill (first pass start -> last pass end) */
  grt_counters counters;
  grt_cache_stats cache_delta;
  int32_t captures_completed;
  uint64_t cache_released;
  double* host_token_us;    /* [gen_len] host time (us from request entry) each token became visible */
} grt_generation_result;

typedef struct grt_model grt_model;
typedef struct grt_session grt_session;

/* ---- library ---------------------------------------------------------------- */
const char* grt_status_name(grt_status s);     /* errc_name (error.cpp:5-31) */
const char* grt_last_error(void);              /* thread-local message of the last failure */
int32_t grt_abi_version(void);
grt_status grt_device_count(int32_t* n);
/* Compiles the NVRTC dynamic-op module for a shape without loading it (no GPU needed). */
grt_status grt_jit_compile_check(int32_t d_model, int32_t vocab, int32_t max_seq, int32_t weight_bf16, int32_t arch_ref,
                                 uint64_t* cubin_bytes);
void grt_model_config_default(grt_model_config* c); /* ModelConfig{} defaults */
void grt_cache_config_default(grt_cache_config* c); /* CacheConfig{} defaults */

/* ---- model (replaces graphrt::Model, model.hpp:58-132) --------------------- */
grt_status grt_model_create(const grt_model_config* cfg, grt_model** out);   /* Model::Model */
grt_status grt_model_destroy(grt_model* m);
/* Overwrites one weight tensor from host memory given in the REFERENCE layout
 * ([k,n] for matrices, model.hpp:33-45); name e.g. "layers.3.wq", "head". */
grt_status grt_model_upload(grt_model* m, const char* tensor, const void* host, size_t bytes,
                            int32_t host_dtype);
/* Copies one weight tensor back in the reference layout as fp32. */
grt_status grt_model_download(grt_model* m, const char* tensor, float* host, size_t numel);
/* Loads weights from a safetensors checkpoint: one file, or a directory whose
 * *.safetensors shards are read in name order.  Tensor names are graphrt's own
 * (reference [k,n] layout, as grt_model_upload) or HuggingFace LLaMA names
 * (model.layers.N.self_attn.q_proj.weight, ... [out,in] layout); dtypes BF16, F16,
 * F32.  strict != 0: every model tensor must be present and no tensor unknown.
 * No reference counterpart: the reference only draws seeded weights
 * (init_model, model.cpp:30-76); SURVEY §8f rank 2. */
grt_status grt_model_load_safetensors(grt_model* m, const char* path, int32_t strict, int32_t* n_loaded);
/* Header-only inspection (no GPU): NUL-separated names into `names`, dtype
 * (grt_dtype or -1), rank and up to 2 dims per tensor; *n = tensor count. */
grt_status grt_safetensors_list(const char* path, char* names, int32_t names_len, int32_t* dtypes, int64_t* shapes,
                                int32_t cap, int32_t* n);
/* HuggingFace LLaMA tensor name -> graphrt name ("" if not a model weight);
 * *out_in = 1 when the checkpoint stores it [out,in]. */
grt_status grt_hf_tensor_name(const char* hf_name, char* out, int32_t out_len, int32_t* out_in);
/* Paged KV cache (kv_page_size > 0): the block table maps
 * logical page i (positions [i*page, (i+1)*page)) to a physical page of every
 * layer's pool.  `table` must hold n_pages distinct ids in [0, n_pages); the
 * default is the identity.  Takes effect for the next pass (the table lives in
 * device memory and every KV read/write goes through it). */
grt_status grt_model_kv_pages(grt_model* m, int32_t* page_size, int32_t* n_pages);
grt_status grt_model_set_kv_block_table(grt_model* m, const int32_t* table, int32_t n);
grt_status grt_model_weight_bytes(grt_model* m, uint64_t* bytes);            /* HBM bytes of weights */
grt_status grt_model_decode_bytes(grt_model* m, int32_t length, uint64_t* bytes); /* algorithmic bytes/pass */

/* ---- session (replaces graphrt::Session, pipeline.hpp:165-189) ------------- */
grt_status grt_session_create(grt_model* m, const grt_cache_config* cc, grt_session** out);
grt_status grt_session_destroy(grt_session* s);
grt_status grt_generate(grt_session* s, const grt_generation_request* req,
                        grt_generation_result* res);                           /* Session::run */
grt_status grt_cache_stats_get(grt_session* s, grt_cache_stats* st, uint64_t* size);
/* Times each kernel of the static plan for bucket `key` in isolation: `iters`
 * back-to-back launches bracketed by CUDA events on the session's compute
 * stream.  Fills up to `cap` entries of avg_ms / bytes (algorithmic HBM bytes)
 * and names (NUL-separated into `names`, `names_len` bytes); *n = plan size. */
grt_status grt_profile_plan(grt_session* s, int32_t key, int32_t iters, double* avg_ms, int64_t* bytes,
                            char* names, int32_t names_len, int32_t cap, int32_t* n);
/* Profiling: replays bucket `key`'s static plan once as a graph with per-CTA
 * %globaltimer stamps: out[kernel * stride + cta * 8 + e] (ns), e = start,
 * dependency released, operands ready, done, first weight stage, loop done. */
grt_status grt_trace_pass(grt_session* s, int32_t key, uint64_t* out, int64_t cap, int32_t* grid, int32_t* stride);
grt_status grt_session_counters(grt_session* s, grt_counters* c);

/* ---- step-level API (Model::step_math / prefill_math / reset, model.cpp:168-183) */
grt_status grt_reset(grt_session* s);
grt_status grt_step(grt_session* s, int32_t token);                 /* extend_position + slot append + plan(cur_len) */
grt_status grt_prefill(grt_session* s, const int32_t* ids, int32_t n); /* prefill_math */
grt_status grt_cur_len(grt_session* s, int32_t* len);
grt_status grt_get_logits(grt_session* s, float* out, int32_t n);   /* model.logits() */
grt_status grt_get_kv_row(grt_session* s, int32_t layer, int32_t slot, int32_t row, float* out); /* [h*dh] */
grt_status grt_sample(grt_session* s, const grt_sample_params* p, int32_t* token); /* make_sample_op */
grt_status grt_sampler_reset(grt_session* s, uint64_t seed);        /* SamplerRng::reset */

/* ---- explicit capture (replaces graphrt::CaptureEngine::begin_capture /
 * CaptureSession::record / end_capture and validate_replay,
 * exec_graph.hpp:73-141, exec_graph.cpp:49-103).  A capture is Open until
 * end_capture (Closed) or the first violation (Aborted: nothing kept, the key
 * released).  Errors: CaptureInProgress (key already open), CaptureViolation
 * (a host-valued op, or a dynamic op into a static-only graph), ForeignBuffer
 * (a binding outside the model arena), EmptyCapture, SessionClosed (use after
 * close/abort).  The graph lands in the session's cache under the step key. */
typedef struct grt_capture grt_capture;
typedef enum grt_capture_state { GRT_CAPTURE_OPEN = 0, GRT_CAPTURE_CLOSED = 1, GRT_CAPTURE_ABORTED = 2 } grt_capture_state;
typedef enum grt_capture_op {
  GRT_OP_PLAN = 0,              /* plan(plan_key)[index]: a static kernel */
  GRT_OP_SAMPLE_PREPROCESS = 1, /* the fused dynamic block (NVRTC sampler + extend_position + slot append) */
  GRT_OP_PREPROCESS = 2,        /* extend_position + slot append alone (NVRTC) */
  GRT_OP_HOST_TOKEN = 3         /* the step API's host->device token upload (needs a host value) */
} grt_capture_op;
/* fused != 0: a hybrid step graph (dynamic device ops allowed); 0: static-only */
grt_status grt_capture_begin(grt_session* s, int32_t key, int32_t fused, grt_capture** out);
grt_status grt_capture_record(grt_capture* c, int32_t op, int32_t plan_key, int32_t index);
/* records an op that binds caller memory [ptr, ptr+bytes) (a device memset) */
grt_status grt_capture_record_external(grt_capture* c, void* ptr, uint64_t bytes);
grt_status grt_capture_end(grt_capture* c, int32_t* kernel_count, uint64_t* epoch);
grt_status grt_capture_state_get(grt_capture* c, int32_t* state, int32_t* recorded);
void grt_capture_destroy(grt_capture* c);  /* also after its session: destroying a session closes its
                                             captures (calls then return SessionClosed) */
/* number of static kernels in plan(key) (Model::plan, model.cpp:118-154) */
grt_status grt_plan_size(grt_session* s, int32_t key, int32_t* n);
/* One step through the cached graph of `key` with `token` at position cur_len.
 * validate != 0: validate_replay first (host WrongLength unless key_of(cur_len+1)
 * == key); validate == 0: launch anyway -- a live length beyond the bucket trips
 * the device-side check (WrongLength). */
grt_status grt_session_replay(grt_session* s, int32_t key, int32_t fused, int32_t token, int32_t validate);
/* arena of the model: bytes reserved, bytes used, sub-allocations (never grows per capture) */
grt_status grt_model_arena_info(grt_model* m, uint64_t* capacity, uint64_t* used, uint64_t* allocations);
/* tensor-parallel state: group size, rank, and whether the residual stream's
 * allreduce buffer lives in an NCCL symmetric window (ncclCommWindowRegister) */
grt_status grt_model_tp_info(grt_model* m, int32_t* tp_size, int32_t* tp_rank, int32_t* symmetric);

/* ---- graph cache policy (replaces graphrt::GraphCache, graph_cache.hpp:29-81) ---
 * The session owns its own cache of cudaGraphExec_t; this standalone handle runs
 * the identical policy code on placeholder graphs (no GPU), for policy tests. */
typedef struct grt_graph_cache grt_graph_cache;
grt_status grt_graph_cache_create(uint64_t capacity, int32_t policy, grt_graph_cache** out);
grt_status grt_graph_cache_destroy(grt_graph_cache* c);
grt_status grt_graph_cache_lookup(grt_graph_cache* c, int32_t key, int32_t* hit);
/* graph_key != key reproduces KeyMismatch; *evicted = INT32_MIN when nothing was evicted. */
grt_status grt_graph_cache_insert(grt_graph_cache* c, int32_t key, int32_t graph_key, int32_t* evicted);
grt_status grt_graph_cache_warmup(grt_graph_cache* c, int32_t lo, int32_t hi, int32_t* captured);
grt_status grt_graph_cache_begin_session(grt_graph_cache* c);
grt_status grt_graph_cache_release_inactive(grt_graph_cache* c, uint64_t* dropped);
grt_status grt_graph_cache_query(grt_graph_cache* c, int32_t key, int32_t* contains, uint64_t* use_count,
                                 uint64_t* size, grt_cache_stats* stats);

/* ---- tensor parallelism ----------------------------------------
 * One process per GPU: rank 0 calls grt_tp_unique_id and shares the bytes with
 * the other ranks (e.g. torch.distributed broadcast); every rank creates its
 * model with tp_size/tp_rank set, then grt_model_attach_nccl before creating
 * its session.  The allreduce (after Wo and down) and the logits allgather are
 * NCCL collectives enqueued on the step stream, i.e. captured into the bucket
 * graphs.  No reference interface exists for this (the reference is
 * single-device). */
#define GRT_TP_UNIQUE_ID_BYTES 128
grt_status grt_tp_unique_id(uint8_t* out, int32_t len);
grt_status grt_model_attach_nccl(grt_model* m, const uint8_t* unique_id, int32_t len);
/* Single-device validation of the sharded model: tp_size ranks in one process
 * stepped in lockstep, collectives emulated in-process (rank-order sums). */
typedef struct grt_tp_emu grt_tp_emu;
grt_status grt_tp_emu_create(const grt_model_config* cfg, grt_tp_emu** out); /* cfg->tp_size ranks */
grt_status grt_tp_emu_destroy(grt_tp_emu* e);
grt_status grt_tp_emu_reset(grt_tp_emu* e);
grt_status grt_tp_emu_step(grt_tp_emu* e, int32_t token);
grt_status grt_tp_emu_logits(grt_tp_emu* e, float* out, int32_t n);
/* T ranks as T host threads with an in-process communicator: batched prefill
 * of prompt[0, n_prompt), then single steps; rank 0's logits (vocab_size). */
grt_status grt_tp_emu_threaded(const grt_model_config* cfg, const int32_t* prompt, int32_t n_prompt,
                               const int32_t* steps, int32_t n_steps, float* logits);

/* ---- two-process split (the paper's IPC, PAPER.md "two processes") ------------
 * Process B (graph generator) owns the model and replays the static pass;
 * process A (context generator) runs the NVRTC dynamic ops -- sampler and
 * preprocess -- directly on B's device memory, opened through
 * cudaIpcOpenMemHandle.  Steps are ordered by two interprocess CUDA events; a
 * host doorbell in POSIX shared memory only sequences the event record/wait
 * calls (no data crosses the host).  Replaces the in-process Channel
 * (pipeline.cpp:56-78). */
typedef struct grt_ipc_desc {
  uint8_t arena[64];      /* cudaIpcMemHandle_t of B's arena */
  uint8_t ev_ctx[64];     /* cudaIpcEventHandle_t: A records after its dynamic ops */
  uint8_t ev_static[64];  /* cudaIpcEventHandle_t: B records after the static pass */
  uint64_t off_ctrl, off_tokens, off_uniforms, off_scratch, off_emb, off_pos, off_x, off_logits;
  int32_t d_model, vocab, max_seq, weight_bf16, arch_ref, device, bucket_size, max_gen;
} grt_ipc_desc;
typedef struct grt_ipc_server grt_ipc_server;
typedef struct grt_ipc_client grt_ipc_client;
grt_status grt_ipc_server_create(grt_session* s, const char* shm_name, grt_ipc_desc* desc, grt_ipc_server** out);
/* Serves n_passes static passes (prompt + generated tokens), blocking. */
grt_status grt_ipc_server_serve(grt_ipc_server* sv, int32_t n_passes);
grt_status grt_ipc_server_destroy(grt_ipc_server* sv);
grt_status grt_ipc_client_create(const grt_ipc_desc* desc, const char* shm_name, grt_ipc_client** out);
/* Runs prompt_len + gen_len passes against a serving process B; tokens[gen_len],
 * per_token_us[gen_len] (device %globaltimer gaps, may be NULL). */
grt_status grt_ipc_client_generate(grt_ipc_client* c, const int32_t* prompt, int32_t prompt_len, int32_t gen_len,
                                   const grt_sample_params* sampling, int32_t* tokens, double* per_token_us);
grt_status grt_ipc_client_destroy(grt_ipc_client* c);

/* ---- op-level API on device pointers (kernel parity tests) ----------------- */
/* out[n] = W[n,k] . x[k] with W in the device ([n,k], row-major) layout. */
grt_status grt_op_gemv(const void* w, int32_t w_dtype, const float* x, float* out, int32_t n, int32_t k,
                       void* stream);
/* Single-query attention over positions [0,len) of K/V laid out [h, max_seq, dh].
 * q, k, v and out must be 16-byte aligned (vector loads; else GRT_InvalidConfig). */
grt_status grt_op_attention(const float* q, const void* k, const void* v, int32_t kv_dtype, float* out,
                            int32_t n_heads, int32_t head_dim, int32_t max_seq, int32_t len, float scale,
                            void* stream);
/* Batched-prefill projection on the tensor cores (tcgen05/TMEM): out[p, m] =
 * x[p, :] . W[m, :] for W bf16 [m_rows, k] and x bf16 [n_tok, k] (row-major,
 * k % 64 == 0, n_tok <= 512); out fp32 [n_tok, m_rows]. */
grt_status grt_op_prefill_gemm(const void* w, const void* x, float* out, int32_t m_rows, int32_t k, int32_t n_tok,
                               void* stream);
/* Samples from device logits (16-byte aligned, else GRT_InvalidConfig); writes
 * the token to *token_dev (device int32). */
grt_status grt_op_sample(const float* logits, int32_t vocab, const grt_sample_params* p, uint64_t step,
                         double uniform, int32_t* token_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GRT_C_API_H */
