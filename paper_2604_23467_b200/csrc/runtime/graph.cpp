// graph.cpp -- ExecGraph / CaptureEngine / GraphCache.
//
// ExecGraph wraps a cudaGraphExec_t (exec_graph.hpp:45-69): replay = ONE
// cudaGraphLaunch for the whole step.  CaptureEngine keeps the reference's
// capture contract (exec_graph.cpp:49-89): only capturable ops, only buffers
// inside the model arena (ForeignBuffer), no empty captures, one open capture
// per key.  GraphCache is graph_cache.cpp:10-125 with the same policy.
#include <limits>

#include "runtime.hpp"

namespace grt {

// ---------------------------------------------------------------------------
// ExecGraph

ExecGraph::ExecGraph(int key, cudaGraphExec_t exec, size_t kernels, int64_t flops, uint64_t epoch, int device)
    : key_(key), exec_(exec), kernels_(kernels), flops_(flops), epoch_(epoch), device_(device) {}

ExecGraph::~ExecGraph() {
  if (device_ < 0) return;  // host-only placeholder (cache policy tests)
  cudaSetDevice(device_);
  if (last_) {
    cudaEventSynchronize(last_);  // deferred destroy: wait for the last replay
    cudaEventDestroy(last_);
  }
  if (exec_) cudaGraphExecDestroy(exec_);
}

void ExecGraph::launch(cudaStream_t s) const { cuda_check(cudaGraphLaunch(exec_, s), "cudaGraphLaunch"); }

void ExecGraph::mark_launched(cudaStream_t s) {
  if (!last_) cuda_check(cudaEventCreateWithFlags(&last_, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventRecord(last_, s), "cudaEventRecord");
}

// ---------------------------------------------------------------------------
// CaptureEngine

void CaptureEngine::open_key(int key) {
  std::lock_guard<std::mutex> lk(mu_);
  if (open_keys_.count(key)) raise(GRT_CaptureInProgress, "capture already open for key " + std::to_string(key));
  open_keys_.insert(key);
}

void CaptureEngine::close_key(int key) {
  std::lock_guard<std::mutex> lk(mu_);
  open_keys_.erase(key);
}

ExecGraphPtr CaptureEngine::capture(int key, const std::vector<const KernelInvocation*>& kernels, cudaStream_t stream) {
  open_key(key);
  struct Close {
    CaptureEngine* e;
    int key;
    ~Close() { e->close_key(key); }
  } close{this, key};
  validate(kernels);
  return instantiate(key, kernels, stream);
}

ExecGraphPtr CaptureEngine::instantiate(int key, const std::vector<const KernelInvocation*>& kernels,
                                        cudaStream_t stream) {
  int64_t flops = 0;
  for (const KernelInvocation* k : kernels) flops += k->spec.flops;
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  cudaError_t launch_err = cudaSuccess;
  std::string failed;
  for (const KernelInvocation* k : kernels) {
    launch_err = k->launch(stream);
    if (launch_err != cudaSuccess) {
      failed = k->spec.name;
      break;
    }
  }
  cudaGraph_t graph = nullptr;
  cudaError_t end_err = cudaStreamEndCapture(stream, &graph);
  if (launch_err != cudaSuccess || end_err != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    raise(GRT_CudaError, "capture of key " + std::to_string(key) + " failed at '" + failed +
                             "': " + cudaGetErrorString(launch_err != cudaSuccess ? launch_err : end_err));
  }
  cudaGraphExec_t exec = nullptr;
  cudaError_t ie = cudaGraphInstantiateWithFlags(&exec, graph, 0);
  cudaGraphDestroy(graph);
  cuda_check(ie, "cudaGraphInstantiate");
  // upload now (off the critical path) so the first replay does not pay it
  cuda_check(cudaGraphUpload(exec, stream), "cudaGraphUpload");
  uint64_t epoch;
  {
    std::lock_guard<std::mutex> lk(mu_);
    epoch = ++epoch_;
  }
  return std::make_shared<ExecGraph>(key, exec, kernels.size(), flops, epoch, device_);
}

ExecGraphPtr CaptureEngine::capture_fn(int key, const std::function<void(cudaStream_t)>& fn, cudaStream_t stream) {
  open_key(key);
  struct Close {
    CaptureEngine* e;
    int key;
    ~Close() { e->close_key(key); }
  } close{this, key};
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  std::string what;
  try {
    fn(stream);
  } catch (const std::exception& e) {
    what = e.what();
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t end_err = cudaStreamEndCapture(stream, &graph);
  if (!what.empty() || end_err != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    raise(GRT_CudaError, "capture of key " + std::to_string(key) + " failed: " +
                             (what.empty() ? std::string(cudaGetErrorString(end_err)) : what));
  }
  size_t n_nodes = 0;
  cudaGraphGetNodes(graph, nullptr, &n_nodes);
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiateWithFlags(&exec, graph, 0);
  cudaGraphDestroy(graph);
  cuda_check(ie, "cudaGraphInstantiate");
  cuda_check(cudaGraphUpload(exec, stream), "cudaGraphUpload");
  if (n_nodes == 0) {
    cudaGraphExecDestroy(exec);
    raise(GRT_EmptyCapture, "capture recorded zero kernels");
  }
  uint64_t epoch;
  {
    std::lock_guard<std::mutex> lk(mu_);
    epoch = ++epoch_;
  }
  return std::make_shared<ExecGraph>(key, exec, n_nodes, 0, epoch, device_);
}

void CaptureEngine::check(const KernelInvocation& k, bool allow_dynamic) const {
  if (!k.launch || k.spec.op_class == OpClass::Host)
    raise(GRT_CaptureViolation, "kernel '" + k.spec.name + "' needs host values at launch (not capturable)");
  if (k.spec.op_class == OpClass::Dynamic && !allow_dynamic)
    raise(GRT_CaptureViolation, "dynamic kernel '" + k.spec.name + "' recorded into a static-only graph");
  for (const DevRange& r : k.bindings)
    if (!binding_allowed(r))
      raise(GRT_ForeignBuffer, "kernel '" + k.spec.name + "' binds a buffer outside the model arena");
}

void CaptureEngine::validate(const std::vector<const KernelInvocation*>& kernels) const {
  if (kernels.empty()) raise(GRT_EmptyCapture, "capture recorded zero kernels");
  for (const KernelInvocation* k : kernels) check(*k, true);
}

// ---------------------------------------------------------------------------
// CaptureSession (exec_graph.cpp:49-103)

CaptureSession::CaptureSession(CaptureEngine& engine, int key, bool allow_dynamic)
    : engine_(&engine), key_(key), allow_dynamic_(allow_dynamic) {
  engine_->open_key(key);  // CaptureInProgress when the key is already open
}

CaptureSession::~CaptureSession() {
  if (state_ == Open) engine_->close_key(key_);
}

void CaptureSession::abort() {
  kernels_.clear();  // no partial graphs
  if (state_ == Open) engine_->close_key(key_);
  state_ = Aborted;
}

void CaptureSession::record(const KernelInvocation* k) {
  if (state_ != Open) raise(GRT_SessionClosed, "capture session is not open");
  try {
    engine_->check(*k, allow_dynamic_);
  } catch (...) {
    abort();
    throw;
  }
  kernels_.push_back(k);
}

ExecGraphPtr CaptureSession::end_capture(cudaStream_t stream) {
  if (state_ != Open) raise(GRT_SessionClosed, "capture session is not open");
  if (kernels_.empty()) {
    abort();
    raise(GRT_EmptyCapture, "capture recorded zero kernels");
  }
  ExecGraphPtr g;
  try {
    g = engine_->instantiate(key_, kernels_, stream);
  } catch (...) {
    abort();
    throw;
  }
  engine_->close_key(key_);
  state_ = Closed;
  return g;
}

void CaptureEngine::record_into(cudaGraph_t body, const std::vector<const KernelInvocation*>& kernels,
                                cudaStream_t stream) {
  validate(kernels);
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal),
             "cudaStreamBeginCaptureToGraph");
  cudaError_t launch_err = cudaSuccess;
  std::string failed;
  for (const KernelInvocation* k : kernels) {
    launch_err = k->launch(stream);
    if (launch_err != cudaSuccess) {
      failed = k->spec.name;
      break;
    }
  }
  cudaGraph_t g = nullptr;
  const cudaError_t end_err = cudaStreamEndCapture(stream, &g);
  if (launch_err != cudaSuccess || end_err != cudaSuccess) {
    cudaGetLastError();
    raise(GRT_CudaError, "capture into a conditional body failed at '" + failed +
                             "': " + cudaGetErrorString(launch_err != cudaSuccess ? launch_err : end_err));
  }
}

// ---------------------------------------------------------------------------
// GraphCache (graph_cache.cpp:10-125)

GraphCache::GraphCache(size_t capacity, EvictionPolicy policy) : capacity_(capacity), policy_(policy) {
  if (capacity == 0) raise(GRT_InvalidConfig, "cache capacity must be positive");
}

std::optional<ExecGraphPtr> GraphCache::lookup(int key) {
  auto it = entries_.find(key);
  if (it == entries_.end()) {
    ++stats_.misses;
    return std::nullopt;
  }
  ++stats_.hits;
  Entry& e = it->second;
  ++e.use_count;
  e.last_use_seq = ++seq_;
  if (in_session_) e.active = true;
  return e.graph;
}

std::optional<int> GraphCache::insert(int key, ExecGraphPtr graph) {
  if (!graph) raise(GRT_InvalidConfig, "insert: null graph");
  if (graph->length_key() != key)
    raise(GRT_KeyMismatch, "insert: graph built for key " + std::to_string(graph->length_key()) + " filed under key " +
                               std::to_string(key));
  std::optional<int> evicted;
  auto it = entries_.find(key);
  if (it != entries_.end()) {
    Entry& e = it->second;
    dropped_.push_back(std::move(e.graph));
    e.graph = std::move(graph);
    e.use_count = 0;
    e.insert_seq = ++seq_;
    e.last_use_seq = e.insert_seq;
    if (in_session_) e.active = true;
    ++stats_.inserts;
    return evicted;
  }
  if (entries_.size() == capacity_) {
    const int victim = pick_victim();
    dropped_.push_back(std::move(entries_[victim].graph));
    entries_.erase(victim);
    ++stats_.evictions;
    evicted = victim;
  }
  Entry e;
  e.graph = std::move(graph);
  e.insert_seq = ++seq_;
  e.last_use_seq = e.insert_seq;
  if (in_session_) e.active = true;
  entries_.emplace(key, std::move(e));
  ++stats_.inserts;
  return evicted;
}

int GraphCache::pick_victim() const {
  int victim = entries_.begin()->first;
  uint64_t best_p = std::numeric_limits<uint64_t>::max(), best_s = std::numeric_limits<uint64_t>::max();
  for (const auto& [key, e] : entries_) {
    const uint64_t primary = policy_ == EvictionPolicy::LeastUsed ? e.use_count : e.last_use_seq;
    const uint64_t secondary = e.insert_seq;
    if (primary < best_p || (primary == best_p && secondary < best_s)) {
      best_p = primary;
      best_s = secondary;
      victim = key;
    }
  }
  return victim;
}

int GraphCache::precapture_warmup(int lo, int hi, const std::function<ExecGraphPtr(int)>& capture_fn) {
  if (hi < lo) return 0;
  const size_t span = static_cast<size_t>(hi - lo + 1);
  if (span > capacity_)
    raise(GRT_WarmupExceedsCapacity, "warm-up range [" + std::to_string(lo) + ", " + std::to_string(hi) + "] holds " +
                                         std::to_string(span) + " graphs but capacity is " + std::to_string(capacity_));
  int captured = 0;
  for (int key = lo; key <= hi; ++key) {
    if (contains(key)) continue;
    insert(key, capture_fn(key));
    ++captured;
  }
  return captured;
}

void GraphCache::begin_session() {
  in_session_ = true;
  for (auto& [key, e] : entries_) e.active = false;
}

size_t GraphCache::release_inactive() {
  size_t dropped = 0;
  for (auto it = entries_.begin(); it != entries_.end();) {
    if (!it->second.active) {
      dropped_.push_back(std::move(it->second.graph));
      it = entries_.erase(it);
      ++dropped;
    } else {
      ++it;
    }
  }
  stats_.releases += dropped;
  return dropped;
}

uint64_t GraphCache::use_count(int key) const {
  auto it = entries_.find(key);
  if (it == entries_.end()) raise(GRT_EmptyCache, "use_count: no entry for key " + std::to_string(key));
  return it->second.use_count;
}

std::vector<ExecGraphPtr> GraphCache::take_dropped() {
  std::vector<ExecGraphPtr> out;
  out.swap(dropped_);
  return out;
}

}  // namespace grt
