// runtime.hpp -- B200-native host runtime behind the C ABI (include/grt/c_api.h).
//
// Class names and semantics mirror the reference runtime (graphrt):
//   Errc / Error              error.hpp:10-54
//   ModelConfig / Model       model.hpp:17-132
//   OpClass / KernelSpec / KernelInvocation   kernels.hpp:14-45
//   Workspace -> Arena        exec_graph.hpp:20-40   (one device allocation)
//   ExecGraph / CaptureEngine / CaptureSession  exec_graph.hpp:45-141 (cudaGraphExec_t)
//   GraphCache                graph_cache.hpp:29-81  (same eviction policy)
//   VirtualDevice -> CudaDevice  virtual_device.hpp:125-192 (real streams/events)
//   RunMode / ModePolicy / Channel / ContextGenerator / GraphGenerator / Session
//                             pipeline.hpp:18-189
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../jit/ctrl.h"
#include "../kernels/kernels.h"
#include "grt/c_api.h"

namespace grt {

// ---------------------------------------------------------------------------
// errors (error.hpp:10-54): codes are grt_status values.
using Errc = grt_status;

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

[[noreturn]] void raise(Errc code, const std::string& what);
const char* errc_name(Errc c) noexcept;
void cuda_check(cudaError_t e, const char* what);
void cu_check(CUresult e, const char* what);
const char* cu_error_string(CUresult e);

// ---------------------------------------------------------------------------
// config (model.hpp:17-29)
struct ModelConfig {
  int arch = GRT_ARCH_REF;
  int n_layers = 4;
  int d_model = 64;
  int n_heads = 4;
  int vocab_size = 256;
  int max_seq_len = 600;
  int d_ff_ = 0;
  float norm_eps = 1e-5f;
  uint64_t seed = 1234;
  int init = GRT_INIT_MT19937;
  int weight_dtype = GRT_F32;
  int kv_dtype = GRT_F32;
  float rope_theta = 10000.0f;
  int device = 0;
  int tp_size = 1;
  int tp_rank = 0;
  int kv_page_size = 0;  // 0 = contiguous KV

  int d_ff() const noexcept { return d_ff_ > 0 ? d_ff_ : 4 * d_model; }
  int head_dim() const noexcept { return d_model / n_heads; }
  bool llama() const noexcept { return arch == GRT_ARCH_LLAMA; }
  void validate() const;  // raises InvalidConfig
  static ModelConfig from_c(const grt_model_config& c);
};

// ---------------------------------------------------------------------------
// arena: the Workspace of the reference (exec_graph.hpp:20-40) on the device.
// Allocated once; never grows per capture.  contains() is the ForeignBuffer check.
class Arena {
 public:
  Arena() = default;
  ~Arena();
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  void reserve(size_t bytes);
  void* alloc(size_t bytes, size_t align = 256);
  bool contains(const void* p, size_t n) const;
  // memory outside the arena that bindings may use (the symmetric exchange buffer)
  void allow(const void* p, size_t n) { extra_.push_back({static_cast<const char*>(p), n}); }
  size_t used() const { return used_; }
  size_t capacity() const { return cap_; }
  size_t allocations() const { return count_; }
  char* base() const { return base_; }

 private:
  char* base_ = nullptr;
  size_t cap_ = 0, used_ = 0, count_ = 0;
  std::vector<std::pair<const char*, size_t>> extra_;
};

// ---------------------------------------------------------------------------
// operator API (kernels.hpp:14-45)
// Static: a plan kernel (graph-capturable).  Dynamic: a context op (sampler,
// preprocess) -- NVRTC code that reads token, position and RNG draw from device
// memory, so it is capturable too, but only into a FUSED step graph (hybrid);
// a static-only graph (graph_only / ablate_fused / the IPC split) rejects it,
// as CaptureSession::record rejects every dynamic op (exec_graph.cpp:56-70).
// Host: needs a host value at launch (the step API's token upload) -- never
// capturable (CaptureViolation).
enum class OpClass { Static, Dynamic, Host };

struct DevRange {
  const void* ptr;
  size_t bytes;
};

struct KernelSpec {
  std::string name;
  OpClass op_class = OpClass::Static;
  int64_t flops = 0;
  int64_t bytes = 0;  // algorithmic HBM bytes (roofline accounting)
};

// One kernel instance.  `launch` enqueues it on a stream: it binds device
// buffers (never host values), so it is equally valid eagerly or under capture.
// Tensor-parallel collective on the step path: an in-graph NCCL
// allreduce / allgather for one-rank-per-GPU sessions, or the in-process
// emulation used to validate the sharding on a single GPU.
class TpComm {
 public:
  virtual ~TpComm() = default;
  virtual cudaError_t allreduce_sum(float* buf, size_t n, cudaStream_t s) = 0;                   // in place
  virtual cudaError_t allgather(const float* in, float* out, size_t n_per_rank, cudaStream_t s) = 0;  // rank order
  // Device memory registered with the communicator for symmetric collectives
  // (NCCL: ncclMemAlloc + ncclCommWindowRegister); nullptr when unsupported.
  virtual void* alloc_symmetric(size_t /*bytes*/) { return nullptr; }
  virtual void free_symmetric(void* /*p*/) {}
};
enum CollectiveKind : int { COLL_NONE = 0, COLL_ALLREDUCE = 1, COLL_ALLGATHER = 2 };

struct KernelInvocation {
  KernelSpec spec;
  std::vector<DevRange> bindings;
  std::function<cudaError_t(cudaStream_t)> launch;
  // collectives (TP): `launch` calls the attached TpComm; the fields let an
  // emulation driver run the same exchange across in-process ranks
  int collective = COLL_NONE;
  float* coll_in = nullptr;
  float* coll_out = nullptr;
  size_t coll_n = 0;
};

// ---------------------------------------------------------------------------
// NVRTC-compiled dynamic kernels
class JitModule {
 public:
  JitModule(const std::string& defines_key, const std::vector<std::string>& opts, int device);
  ~JitModule();
  CUfunction fn(const char* name) const;
  double compile_ms() const { return compile_ms_; }

 private:
  CUmodule mod_ = nullptr;
  double compile_ms_ = 0;
  int vocab_ = 0;  // -DGRT_V of this specialisation
  mutable std::vector<CUfunction> fns_;  // handed out by fn() (dynamic-smem registry entries)
};
std::string jit_compile(const std::vector<std::string>& opts);  // NVRTC -> sm_100a cubin (no GPU needed)
std::shared_ptr<JitModule> jit_get(const std::vector<std::string>& opts, int device);
cudaError_t launch_jit(CUfunction f, dim3 grid, dim3 block, void** args, cudaStream_t s, bool pdl);

// ---------------------------------------------------------------------------
// model (model.hpp:58-132)
struct LogicalTensor {
  std::string name;
  int64_t rows = 0, cols = 0;
  int dtype = GRT_F32;
  void* dev = nullptr;  // base of the physical buffer holding it
  MapDesc map;
  uint32_t id = 0;      // draw-order index (Philox tensor id)
};

struct LayerBuffers {
  void* w_qkv = nullptr;  // [3d, d]
  void* w_o = nullptr;    // [d, d]
  void* w_up = nullptr;   // ref: W1 [ff, d]; llama: gate/up interleaved [2ff, d]
  void* w_down = nullptr; // [d, ff]
  float *ln1_g = nullptr, *ln1_b = nullptr, *ln2_g = nullptr, *ln2_b = nullptr;
  void* k = nullptr;      // [h][max_seq][dh]
  void* v = nullptr;
};

class Model {
 public:
  explicit Model(const ModelConfig& cfg);
  ~Model();

  const ModelConfig& config() const noexcept { return cfg_; }
  Arena& arena() noexcept { return arena_; }
  int device() const noexcept { return cfg_.device; }

  // Static plan for one bucket key (lengths ((key-1)*B, key*B]).  Memoized;
  // the returned reference is stable for the model's lifetime.  Raises
  // LengthOutOfRange outside [1, max_key].
  // impl 1 (the only one): 4 kernels per layer + LM head (gemv.cu, attention.cu,
  // gemv_pair.cu); a persistent single-kernel pass was measured slower and removed.
  const std::vector<KernelInvocation>& plan(int key, int bucket_size, int impl = 1);
  int max_key(int bucket_size) const { return (cfg_.max_seq_len + bucket_size - 1) / bucket_size; }
  static int key_of(int length, int bucket_size) { return (length + bucket_size - 1) / bucket_size; }

  // Dynamic ops (DYNAMIC, NVRTC kernels; every runtime value read from ctrl).
  KernelInvocation make_preprocess_op();   // extend_position + slot append
  KernelInvocation make_sample_op();       // sample_token
  KernelInvocation make_sample_preprocess_op();  // both, one launch (the fused dynamic block of a step graph)

  // Weight I/O in the reference layout.
  // out_in: `host` holds a matrix as [n, k] (nn.Linear / checkpoint layout)
  // instead of the reference's [k, n]
  void upload(const std::string& name, const void* host, size_t bytes, int host_dtype, bool out_in = false);
  void download(const std::string& name, float* host, size_t numel);
  const LogicalTensor& tensor(const std::string& name) const;
  bool has_tensor(const std::string& name) const;
  const std::vector<LogicalTensor>& tensors() const { return tensors_; }
  uint64_t weight_bytes() const { return weight_bytes_; }
  uint64_t decode_bytes(int length) const;  // algorithmic bytes of one pass at `length`

  // device state
  GrtCtrl* ctrl_dev() const { return ctrl_; }
  LoopCtl* loop_ctl_dev() const { return loop_ctl_; }
  int* tokens_dev() const { return tokens_; }
  double* uniforms_dev() const { return uniforms_; }
  float* logits_dev() const { return logits_; }
  float* scratch_dev() const { return scratch_; }
  float* x_dev() const { return x_; }
  const LayerBuffers& layer(int l) const { return layers_[l]; }
  volatile int* host_tokens() const { return h_out_tokens_; }
  volatile unsigned long long* host_stamps() const { return h_out_stamps_; }
  int max_gen() const { return max_gen_; }
  int kv_elem_bytes() const { return cfg_.kv_dtype == GRT_BF16 ? 2 : 4; }
  const KvPaging& kv_paging() const { return kvp_; }
  int kv_pages() const { return kv_pages_; }
  size_t kv_layer_elems() const { return kv_layer_elems_; }  // elements of one layer's K (or V) cache
  void set_kv_block_table(const int* table, int n);
  int64_t kv_row_host(int head, int pos) const;  // host view of kv_row (common.cuh)
  const std::set<const void*>& buffer_set() const { return buffers_; }

  // Batched prefill (LLaMA arch, bf16 weights): tokens_dev()[0, p) pass through
  // each layer together -- tcgen05 GEMMs for the projections, one causal
  // attention launch -- in chunks of PREFILL_CHUNK tokens; leaves the device in
  // the state p token-by-token passes would (KV rows [0, p), seq_len = p,
  // residual/logits of the last token).  Enqueued on `s`, no host sync.
  bool supports_batched_prefill() const;
  void prefill_batched(int p, cudaStream_t s, bool fuse_norm = true);

  // Tensor parallelism (tp_size > 1): this model holds rank tp_rank's shard --
  // QKV/gate/up/head column-parallel (heads, d_ff and vocab split), Wo/down
  // row-parallel, KV cache by head.  Collectives go through `comm`, which the
  // caller owns and must attach before any plan is built.
  int tp_size() const { return cfg_.tp_size; }
  int tp_rank() const { return cfg_.tp_rank; }
  // Collectives are planned whenever a communicator is attached -- including a
  // 1-rank group (tp_size 1), where they are identities: the NCCL capture path
  // exercised on one GPU.  Plans built before attaching are dropped.
  void attach_comm(TpComm* c);
  bool symmetric_exchange() const { return x_sym_ != nullptr; }
  TpComm* comm() const { return comm_; }
  float* logits_local_dev() const { return logits_local_; }
  const void* emb_dev() const { return emb_; }
  const void* pos_dev() const { return pos_ ? pos_ : emb_; }
  void reset_pass_sync() {  // after a grid-barrier watchdog expiry
    cudaMemset(pair_bar_, 0, static_cast<size_t>(cfg_.n_layers) * 4 * 4);
    cudaMemset(&ctrl_->err, 0, sizeof(int));
    cudaDeviceSynchronize();
  }

 private:
  void declare_tensors();
  void init_weights();
  std::vector<KernelInvocation> build_plan(int key, int bucket_size, int impl);
  unsigned long long* op_trace_ = nullptr;
  // set only while building a traced per-op plan
  void attention_split(int key, int bucket_size, int* nsplit, int* span_cap) const;

 public:
  // Profiling: the per-op plan captured as a graph and replayed once with
  // per-CTA %globaltimer stamps, [n_kernels][OP_TRACE_CTAS*8] (start,
  // released, operands ready, done, first stage, loop done).
  std::vector<uint64_t> trace_pass(int key, int bucket_size, cudaStream_t s, int* grid, int* stride, int impl = 1);

 private:
  void* arena_buf(size_t bytes, const char* what);

  ModelConfig cfg_;
  Arena arena_;
  std::vector<LogicalTensor> tensors_;
  std::vector<LayerBuffers> layers_;
  void *emb_ = nullptr, *pos_ = nullptr, *head_ = nullptr;
  float *lnf_g_ = nullptr, *lnf_b_ = nullptr;
  float *x_ = nullptr, *q_ = nullptr, *attn_ = nullptr, *act_ = nullptr, *logits_ = nullptr;
  float *attn_part_ = nullptr, *rope_cos_ = nullptr, *rope_sin_ = nullptr, *scratch_ = nullptr;
  int* attn_counters_ = nullptr;
  // batched-prefill workspace (allocated only when supported)
  float *pf_X_ = nullptr, *pf_Q_ = nullptr, *pf_part_ = nullptr;
  void *pf_Xn_ = nullptr, *pf_A_ = nullptr, *pf_act_ = nullptr;
  int* pf_cnt_ = nullptr;
  int* pair_bar_ = nullptr;
  float* x_sym_ = nullptr;     // the residual stream in communicator-registered memory (TP)
  KvPaging kvp_;
  int kv_pages_ = 0;
  size_t kv_layer_elems_ = 0;
  int* kv_table_ = nullptr;          // device [kv_pages_] block table
  std::vector<int> kv_table_host_;  // [h][<=4][dh+4] partials of the fused attention phase  // [2 * n_layers][2] barrier counters of the fused GEMV pairs
  // tensor-parallel shard dims: heads, attention width, d_ff, vocab per rank
  int hl_ = 0, dq_ = 0, ffl_ = 0, vl_ = 0;
  float* logits_local_ = nullptr;  // [vl_] before the allgather (== logits_ when tp_size == 1)
  TpComm* comm_ = nullptr;
  GrtCtrl* ctrl_ = nullptr;
  LoopCtl* loop_ctl_ = nullptr;
  int* tokens_ = nullptr;
  double* uniforms_ = nullptr;
  int max_gen_ = 0;
  int max_nsplit_ = 1;
  volatile int* h_out_tokens_ = nullptr;
  volatile unsigned long long* h_out_stamps_ = nullptr;
  uint64_t weight_bytes_ = 0;
  std::shared_ptr<JitModule> jit_;
  CUfunction f_pre_ = nullptr, f_sample_ = nullptr, f_sample_pre_ = nullptr;
  std::mutex plan_mu_;
  std::map<std::pair<int, int>, std::vector<KernelInvocation>> plans_;
  std::set<const void*> buffers_;
};

// ---------------------------------------------------------------------------
// capture / replay (exec_graph.hpp:45-141)
// ---------------------------------------------------------------------------
// checkpoints (checkpoint.cpp)
struct StTensor {
  std::string name, dtype_name;
  int dtype = -1;  // grt_dtype, -1 = unsupported
  std::vector<int64_t> shape;
  uint64_t begin = 0, end = 0;  // offsets into the data block
};
class SafetensorsFile {
 public:
  explicit SafetensorsFile(const std::string& path);  // raises IoError
  ~SafetensorsFile();
  SafetensorsFile(const SafetensorsFile&) = delete;
  SafetensorsFile& operator=(const SafetensorsFile&) = delete;
  const std::vector<StTensor>& tensors() const { return tensors_; }
  const void* data(const StTensor& t) const;

 private:
  std::string path_;
  int fd_ = -1;
  void* map_ = nullptr;
  size_t size_ = 0;
  uint64_t data_off_ = 0;
  std::vector<StTensor> tensors_;
};
std::string hf_to_grt_name(const std::string& hf, bool* out_in);
int load_safetensors(Model& m, const std::string& path, bool strict);

class ExecGraph {
 public:
  ExecGraph(int key, cudaGraphExec_t exec, size_t kernels, int64_t flops, uint64_t epoch, int device);
  ~ExecGraph();
  int length_key() const noexcept { return key_; }
  size_t kernel_count() const noexcept { return kernels_; }
  int64_t total_flops() const noexcept { return flops_; }
  uint64_t capture_epoch() const noexcept { return epoch_; }
  cudaGraphExec_t exec() const noexcept { return exec_; }
  void launch(cudaStream_t s) const;
  // Records an event after the latest launch; destruction waits for it, so an
  // evicted graph is only destroyed after its last replay retired.
  void mark_launched(cudaStream_t s);

 private:
  int key_;
  cudaGraphExec_t exec_;
  size_t kernels_;
  int64_t flops_;
  uint64_t epoch_;
  int device_;
  cudaEvent_t last_ = nullptr;
};
using ExecGraphPtr = std::shared_ptr<ExecGraph>;

class CaptureEngine {
 public:
  CaptureEngine(const Arena& arena, int device) : arena_(&arena), device_(device) {}
  // exec_graph.cpp:49-55 begin_capture: one open capture per key
  void open_key(int key);
  void close_key(int key);
  // capture + instantiate a validated list under an already-open key
  ExecGraphPtr instantiate(int key, const std::vector<const KernelInvocation*>& kernels, cudaStream_t stream);
  // the per-kernel checks of CaptureSession::record (exec_graph.cpp:56-77)
  void check(const KernelInvocation& k, bool allow_dynamic) const;
  // Captures `kernels` on `stream` (cudaStreamCaptureModeThreadLocal) and
  // instantiates them.  Raises CaptureViolation / ForeignBuffer / EmptyCapture /
  // CaptureInProgress like CaptureSession::record / end_capture.
  ExecGraphPtr capture(int key, const std::vector<const KernelInvocation*>& kernels, cudaStream_t stream);
  // captures whatever `fn` enqueues on `stream` (an internal, arena-only
  // sequence such as the batched prefill) under `key`
  ExecGraphPtr capture_fn(int key, const std::function<void(cudaStream_t)>& fn, cudaStream_t stream);
  // same checks, recorded into an existing (conditional body) graph
  void record_into(cudaGraph_t body, const std::vector<const KernelInvocation*>& kernels, cudaStream_t stream);
  void validate(const std::vector<const KernelInvocation*>& kernels) const;
  bool binding_allowed(const DevRange& r) const { return arena_->contains(r.ptr, r.bytes); }

 private:
  const Arena* arena_;
  int device_;
  std::mutex mu_;
  std::set<int> open_keys_;
  uint64_t epoch_ = 0;
};

// CaptureSession (exec_graph.hpp:73-103): Open -> record()* -> end_capture()
// -> Closed; any violation aborts it (Aborted, nothing recorded kept) and
// releases the key.  A closed or aborted session raises SessionClosed.
class CaptureSession {
 public:
  enum State { Open = 0, Closed = 1, Aborted = 2 };
  CaptureSession(CaptureEngine& engine, int key, bool allow_dynamic);
  ~CaptureSession();
  CaptureSession(const CaptureSession&) = delete;
  CaptureSession& operator=(const CaptureSession&) = delete;
  void record(const KernelInvocation* k);
  ExecGraphPtr end_capture(cudaStream_t stream);
  State state() const { return state_; }
  size_t recorded() const { return kernels_.size(); }
  int key() const { return key_; }

 private:
  void abort();
  CaptureEngine* engine_;
  int key_;
  bool allow_dynamic_;
  State state_ = Open;
  std::vector<const KernelInvocation*> kernels_;
};

// graph_cache.hpp:29-81, ported with the same policy and statistics.
enum class EvictionPolicy { LeastUsed = GRT_EVICT_LEAST_USED, LeastRecentlyUsed = GRT_EVICT_LRU };

class GraphCache {
 public:
  explicit GraphCache(size_t capacity, EvictionPolicy policy = EvictionPolicy::LeastUsed);
  std::optional<ExecGraphPtr> lookup(int key);
  std::optional<int> insert(int key, ExecGraphPtr graph);
  int precapture_warmup(int lo, int hi, const std::function<ExecGraphPtr(int)>& capture_fn);
  void begin_session();
  size_t release_inactive();
  size_t size() const noexcept { return entries_.size(); }
  size_t capacity() const noexcept { return capacity_; }
  bool contains(int key) const { return entries_.count(key) != 0; }
  uint64_t use_count(int key) const;
  const grt_cache_stats& stats() const noexcept { return stats_; }
  // graphs dropped by eviction/release, kept alive until their last launch retires
  std::vector<ExecGraphPtr> take_dropped();

 private:
  struct Entry {
    ExecGraphPtr graph;
    uint64_t use_count = 0, insert_seq = 0, last_use_seq = 0;
    bool active = false;
  };
  int pick_victim() const;
  size_t capacity_;
  EvictionPolicy policy_;
  std::map<int, Entry> entries_;
  uint64_t seq_ = 0;
  bool in_session_ = false;
  grt_cache_stats stats_{};
  std::vector<ExecGraphPtr> dropped_;
};

// ---------------------------------------------------------------------------
// pipeline (pipeline.hpp)
enum class RunMode { Eager = 0, Hybrid = 1, GraphOnly = 2, AblateAsync = 3, AblateFused = 4, AblateBoth = 5, DeviceLoop = 6 };
const char* mode_name(RunMode m) noexcept;

struct ModePolicy {
  bool use_cache = false;
  bool capture_on_miss = false;
  bool async_capture = true;  // Capture stream + capture thread (false = inline, serialised)
  bool fuse_dynamic = false;  // dynamic ops inside the step graph
};
ModePolicy policy_for(RunMode m) noexcept;

enum class StepPath {
  Replayed = GRT_PATH_REPLAYED,
  EagerFallback = GRT_PATH_EAGER_FALLBACK,
  Batched = GRT_PATH_BATCHED,
  BatchedReplayed = GRT_PATH_BATCHED_REPLAYED
};

struct StepRequest {
  int step_index = 0;
  int length_key = 0;  // bucket key
  bool fused = false;
};
struct StepResponse {
  int step_index = 0;
  StepPath path = StepPath::EagerFallback;
};

// Single-slot rendezvous with strict alternation (pipeline.cpp:56-78).
class Channel {
 public:
  void send_request(const StepRequest& r);
  StepRequest take_request();
  void send_response(const StepResponse& r);
  StepResponse take_response();

 private:
  enum class State { Idle, Requested, Serving, Responded };
  State state_ = State::Idle;
  StepRequest req_;
  StepResponse resp_;
};

struct CacheConfig {
  size_t capacity = 600;
  int warmup_lo = 1;
  int warmup_hi = 50;
  bool prefill_uses_graphs = true;
  EvictionPolicy policy = EvictionPolicy::LeastUsed;
  int bucket_size = 64;
  bool batched_prefill = false;
  int pass_impl = 1;  // 1: the per-op kernel graph (the only supported value)
  bool prefill_fuse_norm = true;  // split-K residual partials reduced inside the next RMSNorm launch
  static CacheConfig from_c(const grt_cache_config& c);
};

// Two real streams (Replay = compute, Capture = side stream) plus the
// background capture thread (virtual_device.hpp:125-192 with real CUDA).
class CudaDevice {
 public:
  explicit CudaDevice(int device);
  ~CudaDevice();
  cudaStream_t replay() const { return s_rep_; }
  cudaStream_t capture_stream() const { return s_cap_; }
  int device() const { return device_; }
  grt_counters& counters() { return counters_; }
  void submit_kernel(const KernelInvocation& inv);              // eager launch on Replay
  void submit_fused_block(const std::vector<KernelInvocation>& block);  // dynamic-only
  void submit_replay(const ExecGraphPtr& g);
  // Background capture: job runs on the capture thread, result harvested later.
  void submit_capture(int key, std::function<ExecGraphPtr(cudaStream_t)> job);
  std::vector<std::pair<int, ExecGraphPtr>> take_ready_captures();
  bool capture_pending(int key);
  void drain_captures();  // waits for the capture thread to go idle
  void sync_all();

 private:
  void capture_loop();
  int device_;
  cudaStream_t s_rep_ = nullptr, s_cap_ = nullptr;
  grt_counters counters_{};
  std::thread worker_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::pair<int, std::function<ExecGraphPtr(cudaStream_t)>>> jobs_;
  std::vector<std::pair<int, ExecGraphPtr>> ready_;
  std::set<int> pending_;
  std::string worker_error_;
  Errc worker_code_ = GRT_OK;
  bool busy_ = false;
  bool stop_ = false;
};

struct GenerationRequest {
  RunMode mode = RunMode::Hybrid;
  std::vector<int> prompt;
  int gen_len = 1;
  grt_sample_params sampling{GRT_SAMPLE_GREEDY, 1.0f, 0, 1.0f, 7};
  int eos_token = -1;  // DeviceLoop only
};

struct GenerationResult {
  std::vector<int> tokens;
  double ttft_us = 0, total_us = 0, prefill_us = 0;
  std::vector<double> per_token_us;
  grt_counters counters{};
  grt_cache_stats cache_delta{};
  std::vector<StepPath> prefill_paths, decode_paths;
  int captures_completed = 0;
  size_t cache_released = 0;
  std::vector<double> host_token_us;  // host time each token became visible (us from entry)
};

struct KernelProfile {
  std::string name;
  double avg_ms = 0;
  int64_t bytes = 0;
};

class Session {
 public:
  Session(Model& model, const CacheConfig& cc);
  ~Session();
  GenerationResult run(const GenerationRequest& req);
  std::vector<KernelProfile> profile_plan(int key, int iters);

  // step-level API (Model::step_math / prefill_math / reset / sample)
  void reset();
  void step(int token);
  void prefill(const std::vector<int>& ids);
  int cur_len() const { return cur_len_; }
  void logits(float* out, int n);
  void kv_row(int layer, int slot, int row, float* out);
  int sample(const grt_sample_params& p);
  void sampler_reset(uint64_t seed) {
    sampler_.seed(seed);
    n_sampled_ = 0;
  }

  // The static pass alone (no fused dynamic ops) for `key`, from the cache or
  // captured now; used by the two-process split, where the dynamic ops run in
  // the other process.
  ExecGraphPtr static_graph(int key);

  // Explicit capture (exec_graph.hpp:73-103 CaptureSession over this session's
  // engine): the graph lands in the session's cache under the step key.
  enum CaptureOp { OP_PLAN = 0, OP_SAMPLE_PREPROCESS = 1, OP_PREPROCESS = 2, OP_HOST_TOKEN = 3 };
  std::unique_ptr<CaptureSession> begin_capture(int key, bool fused);
  const KernelInvocation* capture_op(int kind, int plan_key, int index);
  ExecGraphPtr end_capture(CaptureSession& cs, bool fused);
  // validate_replay (exec_graph.cpp:91-103) + one replay of the cached graph for
  // `key` as step cur_len+1 with `token`; validate=false skips the host check so
  // the device-side length check is what trips
  void replay(int key, bool fused, int token, bool validate);

  GraphCache& cache() { return *cache_; }
  CudaDevice& device() { return *dev_; }
  const CacheConfig& cache_config() const { return cc_; }

 private:
  void validate(const GenerationRequest& req) const;
  void write_ctrl(int seq_len, int prompt_len, const grt_sample_params& sp, int max_gen);
  StepResponse serve(const StepRequest& req, bool allow_cache, const ModePolicy& pol);
  int harvest();
  std::vector<const KernelInvocation*> step_kernels(int key, bool fused);
  ExecGraphPtr capture_now(int key, bool fused, cudaStream_t s);
  int cache_key(int key, bool fused) const { return fused ? key : -key; }
  // prefill graphs live in the same cache under keys kPrefillKeyBase + prompt length
  static constexpr int kPrefillKeyBase = 1 << 24;
  StepPath serve_prefill(int p, const ModePolicy& pol);
  void check_device_errors();

  Model* model_;
  CacheConfig cc_;
  std::unique_ptr<CudaDevice> dev_;
  std::unique_ptr<CaptureEngine> engine_;
  std::unique_ptr<GraphCache> cache_;
  KernelInvocation pre_op_, sample_op_, sample_pre_op_;
  KernelInvocation host_token_op_;  // step API: tokens[cur_len] = step_token_ (OpClass::Host)
  int step_token_ = 0;
  std::mt19937_64 sampler_{7};
  int cur_len_ = 0;
  int n_sampled_ = 0;  // step-level sampler draws since sampler_reset (Philox counter / uniform index)
  int captures_completed_ = 0;
  GrtCtrl* h_ctrl_ = nullptr;  // pinned staging for ctrl writes
  // device-resident decode loop (loop.cu): one WHILE-node graph over every bucket
  struct DeviceLoop {
    cudaGraphExec_t exec = nullptr;
    int key_lo = 0, n_keys = 0;
    size_t kernels = 0, kernels_per_step = 0;
    double build_ms = 0;
  } loop_;
  LoopCtl* h_loop_ = nullptr;  // pinned staging
  void build_device_loop();

 public:
  int device_loop_keys() const { return loop_.n_keys; }
  double device_loop_build_ms() const { return loop_.build_ms; }
};

// ---------------------------------------------------------------------------
// tensor parallelism (tp.cpp)

// One rank per GPU: NCCL communicator over NVLink/NVSwitch; the collectives
// are enqueued on the step stream, so they are captured into the bucket graphs
// like every kernel (in the same order on every rank).
class NcclComm : public TpComm {
 public:
  NcclComm(const void* unique_id, int nranks, int rank, int device);
  ~NcclComm() override;
  cudaError_t allreduce_sum(float* buf, size_t n, cudaStream_t s) override;
  cudaError_t allgather(const float* in, float* out, size_t n_per_rank, cudaStream_t s) override;
  void* alloc_symmetric(size_t bytes) override;
  void free_symmetric(void* p) override;

 private:
  void* comm_ = nullptr;  // ncclComm_t
  std::vector<std::pair<void*, void*>> windows_;  // (buffer, ncclWindow_t)
};
std::vector<uint8_t> nccl_unique_id();

// T ranks of a tensor-parallel model in ONE process on one device, stepped in
// lockstep on one stream: every kernel of every rank in plan order, each
// collective replaced by the in-process exchange (tp_emu.cu).  Validates the
// sharding (column/row/vocab splits, head-sharded KV, rank-0 residual rule)
// against the tp_size == 1 model on a single GPU.
class TpEmu {
 public:
  explicit TpEmu(const ModelConfig& cfg);
  ~TpEmu();
  void reset();
  void step(int token);
  void logits(float* out, int n);
  int tp_size() const { return static_cast<int>(ranks_.size()); }

 private:
  std::vector<std::unique_ptr<Model>> ranks_;
  std::vector<KernelInvocation> pre_;
  cudaStream_t s_ = nullptr;
  int cur_len_ = 0;
  GrtCtrl* h_ctrl_ = nullptr;
};
// T ranks as T host threads (own Model/Session/stream each) with an in-process
// communicator: batched prefill of `prompt` then step(t) for t in `steps`;
// rank 0's logits out.  Validates the eager TP paths on one device.
void tp_emu_threaded(const ModelConfig& cfg, const std::vector<int>& prompt, const std::vector<int>& steps,
                     float* logits_out);

// ---------------------------------------------------------------------------
// two-process split (ipc.cpp)
grt_ipc_server* ipc_server_create(Session& s, Model& m, const char* shm_name, grt_ipc_desc* d);
void ipc_server_serve(grt_ipc_server* sv, int n_passes);
grt_ipc_client* ipc_client_create(const grt_ipc_desc* d, const char* shm_name);
void ipc_client_generate(grt_ipc_client* c, const int* prompt, int p, int n, const grt_sample_params& sp, int* tokens,
                         double* per_token_us);

}  // namespace grt

void grt_ipc_server_free(grt_ipc_server* sv);
void grt_ipc_client_free(grt_ipc_client* c);
