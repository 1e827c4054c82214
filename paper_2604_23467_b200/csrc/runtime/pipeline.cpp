// pipeline.cpp -- CudaDevice, Channel, Session::run.
//
// Session::run keeps the reference's generation loop (pipeline.cpp:183-259):
// prefill passes at keys 1..p, then decode steps that sample, extend, and run
// the pass at key p+i; cleanup drains captures, harvests, releases inactive
// graphs.  What changes on the B200:
//   * the sampled token never comes back to the host inside the loop: it is
//     written to device memory (token history) and to host-mapped memory, so
//     the host keeps submitting without blocking (the reference syncs per
//     token, pipeline.cpp:102-109);
//   * in fused modes one decode step is ONE cudaGraphLaunch of
//     [sample, extend_position, static pass] -- zero host kernel launches;
//   * a miss runs the step with direct launches on the Replay stream while a
//     background thread captures the bucket's graph on the Capture stream
//     (cudaStreamCaptureModeThreadLocal) and instantiates it; the result is
//     harvested at the next step boundary (pipeline.cpp:118-126).
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>

#include "runtime.hpp"

namespace grt {

namespace {
double now_us() {
  using namespace std::chrono;
  return duration<double, std::micro>(steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// ---------------------------------------------------------------------------
// modes (pipeline.cpp:10-51)

const char* mode_name(RunMode m) noexcept {
  switch (m) {
    case RunMode::Eager: return "eager";
    case RunMode::Hybrid: return "hybrid";
    case RunMode::GraphOnly: return "graph_only";
    case RunMode::AblateAsync: return "ablate_async";
    case RunMode::AblateFused: return "ablate_fused";
    case RunMode::AblateBoth: return "ablate_both";
    case RunMode::DeviceLoop: return "device_loop";
  }
  return "?";
}

ModePolicy policy_for(RunMode m) noexcept {
  switch (m) {
    case RunMode::Eager: return {false, false, true, false};
    case RunMode::Hybrid: return {true, true, true, true};
    case RunMode::GraphOnly: return {true, false, true, true};
    case RunMode::AblateAsync: return {true, true, false, true};
    case RunMode::AblateFused: return {true, true, true, false};
    case RunMode::AblateBoth: return {true, true, false, false};
    case RunMode::DeviceLoop: return {true, false, true, true};
  }
  return {};
}

// ---------------------------------------------------------------------------
// Channel (pipeline.cpp:56-78)

void Channel::send_request(const StepRequest& r) {
  if (state_ != State::Idle) raise(GRT_SessionClosed, "channel: request out of turn");
  req_ = r;
  state_ = State::Requested;
}
StepRequest Channel::take_request() {
  if (state_ != State::Requested) raise(GRT_SessionClosed, "channel: no request pending");
  state_ = State::Serving;
  return req_;
}
void Channel::send_response(const StepResponse& r) {
  if (state_ != State::Serving) raise(GRT_SessionClosed, "channel: response out of turn");
  resp_ = r;
  state_ = State::Responded;
}
StepResponse Channel::take_response() {
  if (state_ != State::Responded) raise(GRT_SessionClosed, "channel: no response pending");
  state_ = State::Idle;
  return resp_;
}

CacheConfig CacheConfig::from_c(const grt_cache_config& c) {
  CacheConfig cc;
  cc.capacity = c.capacity;
  cc.warmup_lo = c.warmup_lo;
  cc.warmup_hi = c.warmup_hi;
  cc.prefill_uses_graphs = c.prefill_uses_graphs != 0;
  cc.policy = c.policy == GRT_EVICT_LRU ? EvictionPolicy::LeastRecentlyUsed : EvictionPolicy::LeastUsed;
  cc.bucket_size = c.bucket_size;
  cc.batched_prefill = c.batched_prefill != 0;
  cc.pass_impl = c.pass_impl;
  cc.prefill_fuse_norm = c.prefill_fuse_norm != 0;
  return cc;
}

// ---------------------------------------------------------------------------
// CudaDevice

CudaDevice::CudaDevice(int device) : device_(device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&s_rep_, cudaStreamNonBlocking), "cudaStreamCreate(replay)");
  cuda_check(cudaStreamCreateWithFlags(&s_cap_, cudaStreamNonBlocking), "cudaStreamCreate(capture)");
  worker_ = std::thread([this] { capture_loop(); });
}

CudaDevice::~CudaDevice() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  if (worker_.joinable()) worker_.join();
  cudaSetDevice(device_);
  cudaStreamSynchronize(s_rep_);
  cudaStreamSynchronize(s_cap_);
  ready_.clear();
  cudaStreamDestroy(s_rep_);
  cudaStreamDestroy(s_cap_);
}

void CudaDevice::capture_loop() {
  cudaSetDevice(device_);
  cudaFree(nullptr);
  for (;;) {
    std::pair<int, std::function<ExecGraphPtr(cudaStream_t)>> job;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [this] { return stop_ || !jobs_.empty(); });
      if (stop_ && jobs_.empty()) return;
      job = std::move(jobs_.front());
      jobs_.pop_front();
      busy_ = true;
    }
    ExecGraphPtr g;
    std::string err;
    Errc code = GRT_OK;
    try {
      g = job.second(s_cap_);
    } catch (const Error& e) {
      err = e.what();
      code = e.code();
    } catch (const std::exception& e) {
      err = e.what();
      code = GRT_CudaError;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (g) ready_.emplace_back(job.first, std::move(g));
      if (code != GRT_OK && worker_code_ == GRT_OK) {
        worker_code_ = code;
        worker_error_ = err;
      }
      pending_.erase(job.first);
      busy_ = false;
    }
    cv_.notify_all();
  }
}

void CudaDevice::submit_kernel(const KernelInvocation& inv) {
  cuda_check(inv.launch(s_rep_), inv.spec.name.c_str());
  ++counters_.dispatches;
  ++counters_.kernel_launches;
}

void CudaDevice::submit_fused_block(const std::vector<KernelInvocation>& block) {
  if (block.empty()) return;
  for (const KernelInvocation& inv : block)
    if (inv.spec.op_class != OpClass::Dynamic)
      raise(GRT_StaticInFusedBlock, "fused block member '" + inv.spec.name + "' is static; capture it instead");
  for (const KernelInvocation& inv : block) {
    cuda_check(inv.launch(s_rep_), inv.spec.name.c_str());
    ++counters_.kernel_launches;
    ++counters_.dispatches;
  }
  ++counters_.fused_blocks;
}

void CudaDevice::submit_replay(const ExecGraphPtr& g) {
  if (!g) raise(GRT_InvalidConfig, "submit_replay: null graph");
  g->launch(s_rep_);
  ++counters_.dispatches;
  ++counters_.graph_replays;
  counters_.graph_kernel_nodes += g->kernel_count();
}

void CudaDevice::submit_capture(int key, std::function<ExecGraphPtr(cudaStream_t)> job) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    pending_.insert(key);
    jobs_.emplace_back(key, std::move(job));
  }
  ++counters_.captures;
  cv_.notify_all();
}

std::vector<std::pair<int, ExecGraphPtr>> CudaDevice::take_ready_captures() {
  std::lock_guard<std::mutex> lk(mu_);
  if (worker_code_ != GRT_OK) {
    Errc c = worker_code_;
    std::string m = worker_error_;
    worker_code_ = GRT_OK;
    raise(c, "async capture failed: " + m);
  }
  std::vector<std::pair<int, ExecGraphPtr>> out;
  out.swap(ready_);
  return out;
}

bool CudaDevice::capture_pending(int key) {
  std::lock_guard<std::mutex> lk(mu_);
  return pending_.count(key) != 0;
}

void CudaDevice::drain_captures() {
  std::unique_lock<std::mutex> lk(mu_);
  cv_.wait(lk, [this] { return jobs_.empty() && !busy_; });
}

void CudaDevice::sync_all() {
  cuda_check(cudaStreamSynchronize(s_rep_), "sync replay");
  cuda_check(cudaStreamSynchronize(s_cap_), "sync capture");
}

// ---------------------------------------------------------------------------
// Session

Session::Session(Model& model, const CacheConfig& cc) : model_(&model), cc_(cc) {
  if (model.tp_size() > 1 && !model.comm())
    raise(GRT_InvalidConfig, "tensor-parallel model has no communicator (grt_model_attach_nccl)");
  // with a communicator the plans hold in-graph NCCL collectives; captures run
  // on the submitting thread (one NCCL communicator must not be driven from two
  // host threads), so every rank captures and launches in the same order
  if (cc_.bucket_size < 1) raise(GRT_InvalidConfig, "bucket_size must be >= 1");
  cuda_check(cudaSetDevice(model.device()), "cudaSetDevice");
  dev_ = std::make_unique<CudaDevice>(model.device());
  engine_ = std::make_unique<CaptureEngine>(model.arena(), model.device());
  cache_ = std::make_unique<GraphCache>(cc_.capacity, cc_.policy);
  pre_op_ = model.make_preprocess_op();
  sample_op_ = model.make_sample_op();
  sample_pre_op_ = model.make_sample_preprocess_op();
  host_token_op_.spec.name = "host_token_upload";
  host_token_op_.spec.op_class = OpClass::Host;
  host_token_op_.bindings = {{model.tokens_dev(), static_cast<size_t>(model.config().max_seq_len) * sizeof(int)}};
  host_token_op_.launch = [this](cudaStream_t s) {
    return cudaMemcpyAsync(model_->tokens_dev() + cur_len_, &step_token_, sizeof(int), cudaMemcpyHostToDevice, s);
  };
  void* hc = nullptr;
  cuda_check(cudaHostAlloc(&hc, sizeof(GrtCtrl), cudaHostAllocDefault), "cudaHostAlloc ctrl");
  h_ctrl_ = static_cast<GrtCtrl*>(hc);
  std::memset(h_ctrl_, 0, sizeof(GrtCtrl));
  write_ctrl(0, INT_MAX, grt_sample_params{GRT_SAMPLE_GREEDY, 1.0f, 0, 1.0f, 7}, model.max_gen());
  cuda_check(cudaStreamSynchronize(dev_->replay()), "session init");

  // Warm-up (graph_cache.cpp:90-106): offline pre-capture of the fused step
  // graphs for keys [warmup_lo, warmup_hi] (clamped to the model's key range).
  const int hi = std::min(cc_.warmup_hi, model.max_key(cc_.bucket_size));
  cache_->precapture_warmup(cc_.warmup_lo, hi, [this](int key) {
    return engine_->capture(cache_key(key, true), step_kernels(key, true), dev_->capture_stream());
  });
}

Session::~Session() {
  if (dev_) {
    try {
      dev_->drain_captures();
    } catch (...) {
    }
    cudaStreamSynchronize(dev_->replay());
  }
  if (loop_.exec) cudaGraphExecDestroy(loop_.exec);
  cache_.reset();
  dev_.reset();
  if (h_ctrl_) cudaFreeHost(h_ctrl_);
  if (h_loop_) cudaFreeHost(h_loop_);
}

// The device-resident decode loop (loop.cu): one graph
//   WHILE(h_while) { sample+preprocess -> loop_ctl -> SWITCH(h_switch) { pass(key_lo) .. pass(key_hi) } }
// built once per session over every bucket key of the model.  The static
// passes are the same plans the bucket graphs replay (same kernels, PDL
// edges), recorded into the switch bodies with cudaStreamBeginCaptureToGraph.
void Session::build_device_loop() {
  if (loop_.exec) return;
  const double t0 = now_us();
  const int B = cc_.bucket_size;
  loop_.key_lo = 1;
  loop_.n_keys = model_->max_key(B);
  cudaStream_t s = dev_->capture_stream();
  cuda_check(cudaSetDevice(model_->device()), "cudaSetDevice");
  cudaGraph_t g = nullptr;
  cuda_check(cudaGraphCreate(&g, 0), "cudaGraphCreate");
  struct Guard {
    cudaGraph_t g;
    ~Guard() { cudaGraphDestroy(g); }
  } guard{g};
  cudaGraphConditionalHandle h_while;
  cuda_check(cudaGraphConditionalHandleCreate(&h_while, g, 1, cudaGraphCondAssignDefault), "while handle");
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = h_while;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  cuda_check(cudaGraphAddNode(&wn, g, nullptr, 0, &wp), "while node");
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphConditionalHandle h_switch;
  cuda_check(cudaGraphConditionalHandleCreate(&h_switch, body, 0, cudaGraphCondAssignDefault), "switch handle");

  // [dynamic block, loop_ctl]
  KernelInvocation ctl;
  ctl.spec.name = "loop_ctl";
  ctl.spec.op_class = OpClass::Dynamic;
  ctl.bindings = {{model_->ctrl_dev(), sizeof(GrtCtrl)}, {model_->loop_ctl_dev(), sizeof(LoopCtl)}};
  {
    const GrtCtrl* c = model_->ctrl_dev();
    LoopCtl* lc = model_->loop_ctl_dev();
    ctl.launch = [c, lc, h_while, h_switch](cudaStream_t st) { return launch_loop_ctl(c, lc, h_while, h_switch, st); };
  }
  engine_->record_into(body, {&sample_pre_op_, &ctl}, s);
  size_t nn = 0;
  cuda_check(cudaGraphGetNodes(body, nullptr, &nn), "body nodes");
  std::vector<cudaGraphNode_t> nodes(nn);
  cuda_check(cudaGraphGetNodes(body, nodes.data(), &nn), "body nodes");
  cudaGraphNode_t sink = nullptr;
  for (cudaGraphNode_t n : nodes) {
    size_t nd = 0;
    cuda_check(cudaGraphNodeGetDependentNodes(n, nullptr, &nd), "dependents");
    if (nd == 0) sink = n;
  }
  if (!sink) raise(GRT_CudaError, "device loop: no sink node in the loop body");

  cudaGraphNodeParams sp = {};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = h_switch;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  sp.conditional.size = static_cast<unsigned>(loop_.n_keys);
  cudaGraphNode_t sn;
  cuda_check(cudaGraphAddNode(&sn, body, &sink, 1, &sp), "switch node");
  size_t kernels = 2;
  for (int i = 0; i < loop_.n_keys; ++i) {
    const auto& plan = model_->plan(loop_.key_lo + i, B, cc_.pass_impl);
    std::vector<const KernelInvocation*> ks;
    for (const auto& k : plan) ks.push_back(&k);
    engine_->record_into(sp.conditional.phGraph_out[i], ks, s);
    kernels += ks.size();
    if (i == 0) loop_.kernels_per_step = 2 + ks.size();
  }
  cuda_check(cudaGraphInstantiateWithFlags(&loop_.exec, g, 0), "device loop instantiate");
  cuda_check(cudaGraphUpload(loop_.exec, s), "device loop upload");
  cuda_check(cudaStreamSynchronize(s), "device loop upload");
  loop_.kernels = kernels;
  ++dev_->counters().captures;
  if (!h_loop_) {
    void* hl = nullptr;
    cuda_check(cudaHostAlloc(&hl, sizeof(LoopCtl), cudaHostAllocDefault), "cudaHostAlloc loop");
    h_loop_ = static_cast<LoopCtl*>(hl);
  }
  loop_.build_ms = (now_us() - t0) / 1000.0;
}

void Session::write_ctrl(int seq_len, int prompt_len, const grt_sample_params& sp, int max_gen) {
  cuda_check(cudaStreamSynchronize(dev_->replay()), "ctrl staging");
  GrtCtrl& c = *h_ctrl_;
  c.seq_len = seq_len;
  c.prompt_len = prompt_len;
  c.err = 0;
  c.sample_kind = sp.kind;
  c.temperature = sp.temperature;
  c.top_k = sp.top_k;
  c.top_p = sp.top_p;
  c.max_gen = std::min(max_gen, model_->max_gen());
  c.seed = sp.seed;
  c.tokens = model_->tokens_dev();
  c.uniforms = model_->uniforms_dev();
  c.scratch = model_->scratch_dev();
  int* dt = nullptr;
  unsigned long long* ds = nullptr;
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dt), const_cast<int*>(model_->host_tokens()), 0),
             "mapped tokens");
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ds),
                                      const_cast<unsigned long long*>(model_->host_stamps()), 0),
             "mapped stamps");
  c.out_tokens = dt;
  c.out_stamps = ds;
  cuda_check(cudaMemcpyAsync(model_->ctrl_dev(), h_ctrl_, sizeof(GrtCtrl), cudaMemcpyHostToDevice, dev_->replay()),
             "ctrl upload");
}

std::vector<const KernelInvocation*> Session::step_kernels(int key, bool fused) {
  const auto& plan = model_->plan(key, cc_.bucket_size, cc_.pass_impl);
  std::vector<const KernelInvocation*> ks;
  ks.reserve(plan.size() + 2);
  if (fused) ks.push_back(&sample_pre_op_);  // the dynamic block, one launch
  for (const auto& k : plan) ks.push_back(&k);
  return ks;
}

ExecGraphPtr Session::capture_now(int key, bool fused, cudaStream_t s) {
  return engine_->capture(cache_key(key, fused), step_kernels(key, fused), s);
}

int Session::harvest() {
  int landed = 0;
  for (auto& [key, g] : dev_->take_ready_captures()) {
    cache_->insert(key, std::move(g));
    ++landed;
  }
  captures_completed_ += landed;
  return landed;
}

// GraphGenerator::serve (pipeline.cpp:128-152)
StepResponse Session::serve(const StepRequest& req, bool allow_cache, const ModePolicy& pol) {
  harvest();
  const int key = req.length_key;
  const bool use_cache = pol.use_cache && allow_cache;
  const bool fused = pol.fuse_dynamic;
  const int ck = cache_key(key, fused);
  if (use_cache) {
    if (auto hit = cache_->lookup(ck)) {
      if (!fused) dev_->submit_fused_block({sample_op_, pre_op_});
      dev_->submit_replay(*hit);
      (*hit)->mark_launched(dev_->replay());
      return {req.step_index, StepPath::Replayed};
    }
  }
  // eager fallback: dynamic block, then every static kernel launched directly
  dev_->submit_fused_block({sample_op_, pre_op_});
  for (const KernelInvocation& inv : model_->plan(key, cc_.bucket_size, cc_.pass_impl)) dev_->submit_kernel(inv);
  if (use_cache && pol.capture_on_miss && !cache_->contains(ck)) {
    ++dev_->counters().events_recorded;  // ordering point, as record_event/wait_event in the reference
    ++dev_->counters().events_waited;
    if (pol.async_capture && !model_->comm()) {
      if (!dev_->capture_pending(ck))
        dev_->submit_capture(ck, [this, key, fused](cudaStream_t s) { return capture_now(key, fused, s); });
    } else {
      // ablate_async: capture serialised on the submitting thread
      ++dev_->counters().captures;
      cache_->insert(ck, capture_now(key, fused, dev_->capture_stream()));
      ++captures_completed_;
    }
  }
  return {req.step_index, StepPath::EagerFallback};
}

// The batched prefill through the graph cache (the reference serves every
// prefill pass through it, pipeline.cpp:207-214, prefill_uses_graphs): keyed
// by the exact prompt length (the GEMM tilings, split-K choices and chunking
// are functions of it); a miss runs the ~10 launches per layer eagerly and
// captures the sequence (asynchronously on the capture thread in hybrid mode,
// inline for ablate_async and under tensor parallelism), so the next prompt of
// this length is ONE cudaGraphLaunch.
StepPath Session::serve_prefill(int p, const ModePolicy& pol) {
  harvest();
  const bool use_cache = pol.use_cache && cc_.prefill_uses_graphs;
  const int ck = kPrefillKeyBase + p;
  if (use_cache) {
    if (auto hit = cache_->lookup(ck)) {
      dev_->submit_replay(*hit);
      (*hit)->mark_launched(dev_->replay());
      return StepPath::BatchedReplayed;
    }
  }
  model_->prefill_batched(p, dev_->replay(), cc_.prefill_fuse_norm);
  ++dev_->counters().dispatches;
  if (use_cache && pol.capture_on_miss && !cache_->contains(ck)) {
    auto job = [this, p, ck](cudaStream_t cs) {
      return engine_->capture_fn(ck, [this, p](cudaStream_t st) { model_->prefill_batched(p, st, cc_.prefill_fuse_norm); }, cs);
    };
    if (pol.async_capture && !model_->comm()) {
      if (!dev_->capture_pending(ck)) dev_->submit_capture(ck, job);
    } else {
      ++dev_->counters().captures;
      cache_->insert(ck, job(dev_->capture_stream()));
      ++captures_completed_;
    }
  }
  return StepPath::Batched;
}

ExecGraphPtr Session::static_graph(int key) {
  const int ck = cache_key(key, false);
  if (auto hit = cache_->lookup(ck)) return *hit;
  ExecGraphPtr g = capture_now(key, false, dev_->capture_stream());
  cache_->insert(ck, g);
  return g;
}

void Session::validate(const GenerationRequest& req) const {
  // Session::validate (pipeline.cpp:172-181)
  if (req.prompt.empty()) raise(GRT_EmptyPrompt, "run: prompt is empty");
  if (req.gen_len < 1) raise(GRT_InvalidConfig, "run: gen_len must be >= 1");
  const int total = static_cast<int>(req.prompt.size()) + req.gen_len;
  if (total > model_->config().max_seq_len)
    raise(GRT_PromptTooLong, "run: prompt + gen_len = " + std::to_string(total) + " exceeds max_seq_len " +
                                 std::to_string(model_->config().max_seq_len));
  for (int t : req.prompt)
    if (t < 0 || t >= model_->config().vocab_size) raise(GRT_TokenOutOfRange, "token id " + std::to_string(t));
  const auto& sp = req.sampling;
  if (sp.kind < GRT_SAMPLE_GREEDY || sp.kind > GRT_SAMPLE_TOPKP) raise(GRT_InvalidConfig, "unknown sample kind");
  if (sp.kind == GRT_SAMPLE_TOPKP && model_->config().vocab_size > 65535)
    raise(GRT_InvalidConfig, "top-k/top-p sampler needs vocab_size <= 65535");
}

void Session::check_device_errors() {
  int err = 0;
  cuda_check(cudaMemcpy(&err, &model_->ctrl_dev()->err, sizeof(int), cudaMemcpyDeviceToHost), "read err");
  if (err & DEVERR_TIMEOUT) {
    model_->reset_pass_sync();
    raise(GRT_CudaError, "device: persistent pass watchdog expired (a CTA never arrived)");
  }
  if (err & DEVERR_WRONG_LENGTH) raise(GRT_WrongLength, "device: live length outside the graph bucket");
  if (err & DEVERR_CACHE_FULL) raise(GRT_CacheFull, "device: kv cache at max_seq");
  if (err & DEVERR_TOKEN_RANGE) raise(GRT_TokenOutOfRange, "device: token id out of range");
}

GenerationResult Session::run(const GenerationRequest& req) {
  validate(req);
  if (req.mode == RunMode::DeviceLoop) build_device_loop();  // once per session, before the clock starts
  const ModePolicy pol = policy_for(req.mode);
  const int p = static_cast<int>(req.prompt.size());
  const int n = req.gen_len;
  const int B = cc_.bucket_size;
  cudaStream_t s = dev_->replay();
  cuda_check(cudaSetDevice(model_->device()), "cudaSetDevice");

  // leftovers from a previous run
  dev_->drain_captures();
  harvest();
  captures_completed_ = 0;
  dev_->counters() = grt_counters{};
  const grt_cache_stats before = cache_->stats();
  cache_->begin_session();

  // reset: tokens[0..p) = prompt; reference-compatible draws for temperature
  // sampling (one uniform01 per sampled token, kernels.cpp:282, in step order)
  volatile int* ht = model_->host_tokens();
  for (int i = 0; i < n; ++i) ht[i] = -1;
  std::vector<int> prompt(req.prompt);
  cuda_check(cudaMemcpy(model_->tokens_dev(), prompt.data(), p * sizeof(int), cudaMemcpyHostToDevice), "prompt");
  if (req.sampling.kind == GRT_SAMPLE_TEMPERATURE) {
    std::mt19937_64 eng(req.sampling.seed);
    std::vector<double> u(n);
    for (int i = 0; i < n; ++i) u[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
    cuda_check(cudaMemcpy(model_->uniforms_dev(), u.data(), n * sizeof(double), cudaMemcpyHostToDevice), "uniforms");
  }
  write_ctrl(0, p, req.sampling, n);
  cuda_check(cudaStreamSynchronize(s), "run setup");
  cur_len_ = 0;

  cudaEvent_t ev0, ev1;
  cuda_check(cudaEventCreate(&ev0), "event");
  cuda_check(cudaEventCreate(&ev1), "event");
  GenerationResult res;
  res.prefill_paths.reserve(p);
  res.decode_paths.reserve(n);
  Channel channel;

  const double t0 = now_us();
  cuda_check(cudaEventRecord(ev0, s), "event");
  if (cc_.batched_prefill && model_->supports_batched_prefill()) {
    // all p prompt tokens through each layer at once (tcgen05 GEMMs); leaves
    // the device exactly where p single-token passes would -- one graph replay
    // when this prompt length was captured before
    res.prefill_paths.assign(p, serve_prefill(p, pol));
  } else {
    for (int j = 1; j <= p; ++j) {
      channel.send_request({j, Model::key_of(j, B), pol.fuse_dynamic});
      channel.send_response(serve(channel.take_request(), cc_.prefill_uses_graphs, pol));
      res.prefill_paths.push_back(channel.take_response().path);
    }
  }
  cuda_check(cudaEventRecord(ev1, s), "event");

  // Tokens become visible in host-mapped memory as the device produces them;
  // the host stamps each arrival (the consumer-side latency) without ever
  // blocking the stream.
  res.host_token_us.assign(n, 0.0);
  int visible = 0;
  auto poll = [&](int upto) {  // stamp arrivals; block until tokens [0, upto) are visible
    const double deadline = now_us() + 300e6;
    for (;;) {
      while (visible < n && ht[visible] >= 0) res.host_token_us[visible++] = now_us() - t0;
      if (visible >= upto) return;
      const cudaError_t q = cudaStreamQuery(s);
      if (q != cudaSuccess && q != cudaErrorNotReady) cuda_check(q, "decode");
      if (q == cudaSuccess) {  // drained: anything still missing was never produced
        while (visible < n && ht[visible] >= 0) res.host_token_us[visible++] = now_us() - t0;
        return;
      }
      if (now_us() > deadline) raise(GRT_CudaError, "timed out waiting for sampled tokens");
    }
  };
  if (req.mode == RunMode::DeviceLoop) {
    // every decode step in ONE graph launch; bucket choice and stop on the device
    LoopCtl& lc = *h_loop_;
    lc = LoopCtl{};
    lc.remaining = n;
    lc.bucket = B;
    lc.key_lo = loop_.key_lo;
    lc.n_keys = loop_.n_keys;
    lc.eos = req.eos_token;
    cuda_check(cudaMemcpyAsync(model_->loop_ctl_dev(), h_loop_, sizeof(LoopCtl), cudaMemcpyHostToDevice, s),
               "loop ctl");
    cuda_check(cudaGraphLaunch(loop_.exec, s), "device loop launch");
    ++dev_->counters().dispatches;
    ++dev_->counters().graph_replays;
    res.decode_paths.assign(n, StepPath::Replayed);
    poll(1);
  } else {
    for (int i = 1; i <= n; ++i) {
      channel.send_request({i, Model::key_of(p + i, B), pol.fuse_dynamic});
      channel.send_response(serve(channel.take_request(), true, pol));
      res.decode_paths.push_back(channel.take_response().path);
      poll(i >= 2 ? 1 : 0);  // once step 2 is queued, wait for the first token (TTFT)
    }
  }
  poll(n);
  res.ttft_us = n > 0 ? res.host_token_us[0] : 0.0;

  // cleanup (pipeline.cpp:236-258)
  cuda_check(cudaStreamSynchronize(s), "decode");
  res.total_us = now_us() - t0;
  dev_->drain_captures();
  harvest();
  res.cache_released = cache_->release_inactive();
  cache_->take_dropped();  // destroyed here (each waits for its last replay)
  res.captures_completed = captures_completed_;
  float prefill_ms = 0.0f;
  cudaEventElapsedTime(&prefill_ms, ev0, ev1);
  res.prefill_us = prefill_ms * 1000.0;
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  check_device_errors();

  volatile unsigned long long* st = model_->host_stamps();
  res.tokens.resize(n);
  res.per_token_us.resize(n);
  for (int i = 0; i < n; ++i) {
    res.tokens[i] = ht[i];
    if (ht[i] < 0) {  // never produced (device loop stopped at the end-of-sequence token)
      res.per_token_us[i] = 0.0;
      continue;
    }
    const double end_i = static_cast<double>(st[2 * i + 1]);
    const double prev = i == 0 ? static_cast<double>(st[0]) : static_cast<double>(st[2 * i - 1]);
    res.per_token_us[i] = (end_i - prev) / 1000.0;
  }
  res.counters = dev_->counters();
  const grt_cache_stats after = cache_->stats();
  res.cache_delta.hits = after.hits - before.hits;
  res.cache_delta.misses = after.misses - before.misses;
  res.cache_delta.inserts = after.inserts - before.inserts;
  res.cache_delta.evictions = after.evictions - before.evictions;
  res.cache_delta.releases = after.releases - before.releases;
  cur_len_ = p + n;
  if (req.mode == RunMode::DeviceLoop) {
    LoopCtl lc;
    cuda_check(cudaMemcpy(&lc, model_->loop_ctl_dev(), sizeof(LoopCtl), cudaMemcpyDeviceToHost), "loop ctl");
    if (lc.status & LOOP_NO_BUCKET) raise(GRT_WrongLength, "device loop: live length outside every bucket");
    cuda_check(cudaMemcpy(&cur_len_, &model_->ctrl_dev()->seq_len, sizeof(int), cudaMemcpyDeviceToHost), "seq_len");
    res.counters.graph_kernel_nodes = static_cast<uint64_t>(lc.iters) * loop_.kernels_per_step;
  }
  return res;
}

// ---------------------------------------------------------------------------
// step-level API (model.cpp:168-183)

void Session::reset() {
  write_ctrl(0, INT_MAX, grt_sample_params{GRT_SAMPLE_GREEDY, 1.0f, 0, 1.0f, 7}, model_->max_gen());
  cuda_check(cudaStreamSynchronize(dev_->replay()), "reset");
  cur_len_ = 0;
}

void Session::step(int token) {
  const ModelConfig& c = model_->config();
  if (token < 0 || token >= c.vocab_size) raise(GRT_TokenOutOfRange, "token id " + std::to_string(token));
  if (cur_len_ >= c.max_seq_len) {
    if (!c.llama()) raise(GRT_ShapeMismatch, "position " + std::to_string(cur_len_) + " outside position table");
    raise(GRT_CacheFull, "kv cache at max_seq");
  }
  cudaStream_t s = dev_->replay();
  step_token_ = token;
  cuda_check(host_token_op_.launch(s), "token");
  dev_->submit_kernel(pre_op_);
  for (const KernelInvocation& inv :
       model_->plan(Model::key_of(cur_len_ + 1, cc_.bucket_size), cc_.bucket_size, cc_.pass_impl))
    dev_->submit_kernel(inv);
  cuda_check(cudaStreamSynchronize(s), "step");
  ++cur_len_;
  check_device_errors();
}

std::unique_ptr<CaptureSession> Session::begin_capture(int key, bool fused) {
  if (key < 1 || key > model_->max_key(cc_.bucket_size))
    raise(GRT_LengthOutOfRange, "capture key " + std::to_string(key) + " outside [1, max key]");
  return std::make_unique<CaptureSession>(*engine_, cache_key(key, fused), fused);
}

const KernelInvocation* Session::capture_op(int kind, int plan_key, int index) {
  switch (kind) {
    case OP_PLAN: {
      const auto& plan = model_->plan(plan_key, cc_.bucket_size, cc_.pass_impl);  // LengthOutOfRange
      if (index < 0 || index >= static_cast<int>(plan.size()))
        raise(GRT_InvalidConfig, "plan op index " + std::to_string(index) + " outside the plan");
      return &plan[index];
    }
    case OP_SAMPLE_PREPROCESS: return &sample_pre_op_;
    case OP_PREPROCESS: return &pre_op_;
    case OP_HOST_TOKEN: return &host_token_op_;
  }
  raise(GRT_InvalidConfig, "unknown capture op kind " + std::to_string(kind));
}

ExecGraphPtr Session::end_capture(CaptureSession& cs, bool fused) {
  ExecGraphPtr g = cs.end_capture(dev_->capture_stream());
  cuda_check(cudaStreamSynchronize(dev_->capture_stream()), "capture");
  cache_->insert(cs.key(), g);
  ++dev_->counters().captures;
  return g;
}

void Session::replay(int key, bool fused, int token, bool validate) {
  const ModelConfig& c = model_->config();
  if (token < 0 || token >= c.vocab_size) raise(GRT_TokenOutOfRange, "token id " + std::to_string(token));
  if (cur_len_ >= c.max_seq_len) raise(GRT_CacheFull, "kv cache at max_seq");
  auto hit = cache_->lookup(cache_key(key, fused));
  if (!hit) raise(GRT_InvalidConfig, "no cached graph for key " + std::to_string(key));
  if (validate && Model::key_of(cur_len_ + 1, cc_.bucket_size) != key)  // validate_replay: cur_len == length key
    raise(GRT_WrongLength, "replay of key " + std::to_string(key) + " at length " + std::to_string(cur_len_ + 1));
  cudaStream_t s = dev_->replay();
  step_token_ = token;
  cuda_check(host_token_op_.launch(s), "token");
  if (!fused) dev_->submit_kernel(pre_op_);  // static-only graph: the dynamic op runs outside it
  dev_->submit_replay(*hit);
  (*hit)->mark_launched(s);
  cuda_check(cudaStreamSynchronize(s), "replay");
  ++cur_len_;
  check_device_errors();
}

void Session::prefill(const std::vector<int>& ids) {
  if (ids.empty()) raise(GRT_EmptyPrompt, "prefill: prompt is empty");
  if (static_cast<int>(ids.size()) > model_->config().max_seq_len)
    raise(GRT_PromptTooLong, "prefill: prompt length " + std::to_string(ids.size()) + " exceeds max_seq_len");
  if (cc_.batched_prefill && cur_len_ == 0 && model_->supports_batched_prefill()) {
    for (int t : ids)
      if (t < 0 || t >= model_->config().vocab_size) raise(GRT_TokenOutOfRange, "token id " + std::to_string(t));
    cudaStream_t s = dev_->replay();
    cuda_check(cudaMemcpyAsync(model_->tokens_dev(), ids.data(), ids.size() * sizeof(int), cudaMemcpyHostToDevice, s),
               "prompt");
    model_->prefill_batched(static_cast<int>(ids.size()), s, cc_.prefill_fuse_norm);
    cuda_check(cudaStreamSynchronize(s), "prefill");
    cur_len_ = static_cast<int>(ids.size());
    check_device_errors();
    return;
  }
  for (int t : ids) step(t);
}

void Session::logits(float* out, int n) {
  if (n != model_->config().vocab_size) raise(GRT_ShapeMismatch, "logits buffer must hold vocab_size floats");
  cuda_check(cudaStreamSynchronize(dev_->replay()), "sync");
  cuda_check(cudaMemcpy(out, model_->logits_dev(), n * sizeof(float), cudaMemcpyDeviceToHost), "logits");
}

void Session::kv_row(int layer, int slot, int row, float* out) {
  const ModelConfig& c = model_->config();
  if (layer < 0 || layer >= c.n_layers || slot < 0 || slot > 1 || row < 0 || row >= c.max_seq_len)
    raise(GRT_ShapeMismatch, "kv_row out of range");
  const int h = c.n_heads, dh = c.head_dim();
  const LayerBuffers& L = model_->layer(layer);
  const char* base = static_cast<const char*>(slot == 0 ? L.k : L.v);
  const size_t eb = model_->kv_elem_bytes();
  std::vector<char> buf(static_cast<size_t>(dh) * eb);
  for (int hh = 0; hh < h; ++hh) {
    cuda_check(cudaMemcpy(buf.data(), base + static_cast<size_t>(model_->kv_row_host(hh, row)) * dh * eb, dh * eb,
                          cudaMemcpyDeviceToHost),
               "kv row");
    for (int e = 0; e < dh; ++e) {
      float v;
      if (eb == 2) {
        uint32_t u = static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(buf.data())[e]) << 16;
        std::memcpy(&v, &u, 4);
      } else {
        v = reinterpret_cast<const float*>(buf.data())[e];
      }
      out[hh * dh + e] = v;
    }
  }
}

std::vector<KernelProfile> Session::profile_plan(int key, int iters) {
  if (iters < 1) raise(GRT_InvalidConfig, "iters must be >= 1");
  const auto& plan = model_->plan(key, cc_.bucket_size, cc_.pass_impl);
  cudaStream_t s = dev_->replay();
  // a valid live length inside the bucket for the attention kernels
  const int len = std::min(key * cc_.bucket_size, model_->config().max_seq_len);
  write_ctrl(len, INT_MAX, grt_sample_params{GRT_SAMPLE_GREEDY, 1.0f, 0, 1.0f, 7}, model_->max_gen());
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  std::vector<KernelProfile> out;
  for (const KernelInvocation& inv : plan) {
    cuda_check(inv.launch(s), inv.spec.name.c_str());  // warm
    cuda_check(cudaEventRecord(e0, s), "event");
    for (int i = 0; i < iters; ++i) cuda_check(inv.launch(s), inv.spec.name.c_str());
    cuda_check(cudaEventRecord(e1, s), "event");
    cuda_check(cudaEventSynchronize(e1), "event");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    KernelProfile kp;
    kp.name = inv.spec.name;
    kp.avg_ms = ms / iters;
    kp.bytes = inv.spec.bytes;
    out.push_back(kp);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  write_ctrl(cur_len_, INT_MAX, grt_sample_params{GRT_SAMPLE_GREEDY, 1.0f, 0, 1.0f, 7}, model_->max_gen());
  cuda_check(cudaStreamSynchronize(s), "profile");
  return out;
}

int Session::sample(const grt_sample_params& sp) {
  if (sp.kind == GRT_SAMPLE_TOPKP && model_->config().vocab_size > 65535)
    raise(GRT_InvalidConfig, "top-k/top-p sampler needs vocab_size <= 65535");
  cudaStream_t s = dev_->replay();
  // The kernel's step index is seq_len - prompt_len; choose prompt_len so the
  // step is the number of draws since sampler_reset (SamplerRng semantics).
  const int idx = n_sampled_ % model_->max_gen();
  if (sp.kind == GRT_SAMPLE_TEMPERATURE) {
    const double u = static_cast<double>(sampler_() >> 11) * 0x1.0p-53;  // uniform01 (prng.hpp:15-17)
    cuda_check(cudaMemcpy(model_->uniforms_dev() + idx, &u, sizeof(double), cudaMemcpyHostToDevice), "uniform");
  }
  write_ctrl(cur_len_, cur_len_ - idx, sp, model_->max_gen());
  ++n_sampled_;
  dev_->submit_kernel(sample_op_);
  cuda_check(cudaStreamSynchronize(s), "sample");
  int tok = -1;
  cuda_check(cudaMemcpy(&tok, model_->tokens_dev() + cur_len_, sizeof(int), cudaMemcpyDeviceToHost), "token");
  // restore the step-API control state (sampler off)
  write_ctrl(cur_len_, INT_MAX, sp, model_->max_gen());
  cuda_check(cudaStreamSynchronize(s), "sample");
  return tok;
}

}  // namespace grt
