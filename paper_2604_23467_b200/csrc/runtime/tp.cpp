// tp.cpp -- tensor-parallel plumbing: the NCCL communicator whose
// allreduce / allgather are captured inside the bucket graphs, and TpEmu, the
// single-device lockstep driver that validates the sharded model.
#include <dlfcn.h>
#include <nccl.h>

#include <climits>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <type_traits>

#include "runtime.hpp"

namespace grt {

namespace {
// NCCL is resolved at run time (dlopen by soname) and only when tensor
// parallelism is used: if PyTorch is already loaded this binds to ITS NCCL, and
// loading this library first never pins a different libnccl.so.2 into the
// process.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (NCCL >= 2.27): symmetric memory windows
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommWindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n, auto& fp) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, n));
      if (!fp && err.empty()) err = std::string("libnccl.so.2 lacks ") + n;
    };
    sym("ncclGetUniqueId", api.GetUniqueId);
    sym("ncclCommInitRank", api.CommInitRank);
    sym("ncclCommDestroy", api.CommDestroy);
    sym("ncclAllReduce", api.AllReduce);
    sym("ncclAllGather", api.AllGather);
    sym("ncclGetErrorString", api.GetErrorString);
    // optional: absent in older NCCL builds (then the exchange buffer stays in the arena)
    api.MemAlloc = reinterpret_cast<decltype(api.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
    api.MemFree = reinterpret_cast<decltype(api.MemFree)>(dlsym(h, "ncclMemFree"));
    api.CommWindowRegister = reinterpret_cast<decltype(api.CommWindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
    api.CommWindowDeregister =
        reinterpret_cast<decltype(api.CommWindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
  });
  if (!err.empty()) raise(GRT_NcclError, err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) raise(GRT_NcclError, std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

std::vector<uint8_t> nccl_unique_id() {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::vector<uint8_t> out(sizeof(id.internal));
  std::memcpy(out.data(), id.internal, sizeof(id.internal));
  return out;
}

NcclComm::NcclComm(const void* unique_id, int nranks, int rank, int device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  ncclUniqueId id;
  std::memcpy(id.internal, unique_id, sizeof(id.internal));
  ncclComm_t c = nullptr;
  nccl_check(nccl().CommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  comm_ = c;
}

NcclComm::~NcclComm() {
  while (!windows_.empty()) free_symmetric(windows_.back().first);
  if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

cudaError_t NcclComm::allreduce_sum(float* buf, size_t n, cudaStream_t s) {
  return nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm_), s) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}

// Symmetric exchange buffer: ncclMemAlloc'd and registered as a symmetric
// window (collective over the communicator: every rank calls it, same size).
void* NcclComm::alloc_symmetric(size_t bytes) {
  const NcclApi& a = nccl();
  if (!a.MemAlloc || !a.MemFree || !a.CommWindowRegister || !a.CommWindowDeregister) return nullptr;
  void* p = nullptr;
  if (a.MemAlloc(&p, bytes) != ncclSuccess || !p) return nullptr;
  ncclWindow_t win = nullptr;
  if (a.CommWindowRegister(static_cast<ncclComm_t>(comm_), p, bytes, &win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
    a.MemFree(p);
    return nullptr;
  }
  windows_.push_back({p, win});
  return p;
}

void NcclComm::free_symmetric(void* p) {
  const NcclApi& a = nccl();
  for (size_t i = 0; i < windows_.size(); ++i)
    if (windows_[i].first == p) {
      a.CommWindowDeregister(static_cast<ncclComm_t>(comm_), static_cast<ncclWindow_t>(windows_[i].second));
      a.MemFree(p);
      windows_.erase(windows_.begin() + static_cast<std::ptrdiff_t>(i));
      return;
    }
}

cudaError_t NcclComm::allgather(const float* in, float* out, size_t n_per_rank, cudaStream_t s) {
  return nccl().AllGather(in, out, n_per_rank, ncclFloat32, static_cast<ncclComm_t>(comm_), s) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}

// ---------------------------------------------------------------------------

namespace {
constexpr int kEmuBucket = 64;

void write_step_ctrl(Model& m, GrtCtrl* h, int seq_len, cudaStream_t s) {
  std::memset(h, 0, sizeof(GrtCtrl));
  h->seq_len = seq_len;
  h->prompt_len = INT_MAX;  // step API: the sampler stays off
  h->sample_kind = GRT_SAMPLE_GREEDY;
  h->temperature = 1.0f;
  h->top_p = 1.0f;
  h->max_gen = m.max_gen();
  h->seed = 7;
  h->tokens = m.tokens_dev();
  h->uniforms = m.uniforms_dev();
  h->scratch = m.scratch_dev();
  int* dt = nullptr;
  unsigned long long* ds = nullptr;
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dt), const_cast<int*>(m.host_tokens()), 0), "mapped");
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ds), const_cast<unsigned long long*>(m.host_stamps()), 0),
             "mapped");
  h->out_tokens = dt;
  h->out_stamps = ds;
  cuda_check(cudaMemcpyAsync(m.ctrl_dev(), h, sizeof(GrtCtrl), cudaMemcpyHostToDevice, s), "ctrl upload");
  cuda_check(cudaStreamSynchronize(s), "ctrl upload");
}
}  // namespace

TpEmu::TpEmu(const ModelConfig& cfg) {
  if (cfg.tp_size < 1 || cfg.tp_size > TP_MAX) raise(GRT_InvalidConfig, "tp_size must be in [1, 8]");
  for (int r = 0; r < cfg.tp_size; ++r) {
    ModelConfig c = cfg;
    c.tp_rank = r;
    ranks_.push_back(std::make_unique<Model>(c));
  }
  cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
  void* hc = nullptr;
  cuda_check(cudaHostAlloc(&hc, sizeof(GrtCtrl), cudaHostAllocDefault), "cudaHostAlloc");
  h_ctrl_ = static_cast<GrtCtrl*>(hc);
  for (auto& m : ranks_) pre_.push_back(m->make_preprocess_op());
  reset();
}

TpEmu::~TpEmu() {
  if (s_) {
    cudaStreamSynchronize(s_);
    cudaStreamDestroy(s_);
  }
  if (h_ctrl_) cudaFreeHost(h_ctrl_);
}

void TpEmu::reset() {
  for (auto& m : ranks_) write_step_ctrl(*m, h_ctrl_, 0, s_);
  cur_len_ = 0;
}

void TpEmu::step(int token) {
  const ModelConfig& c = ranks_[0]->config();
  if (token < 0 || token >= c.vocab_size) raise(GRT_TokenOutOfRange, "token id " + std::to_string(token));
  if (cur_len_ >= c.max_seq_len) raise(GRT_CacheFull, "kv cache at max_seq");
  const int T = tp_size();
  for (int r = 0; r < T; ++r) {
    cuda_check(cudaMemcpyAsync(ranks_[r]->tokens_dev() + cur_len_, &token, sizeof(int), cudaMemcpyHostToDevice, s_),
               "token");
    cuda_check(pre_[r].launch(s_), "preprocess");
  }
  const int key = Model::key_of(cur_len_ + 1, kEmuBucket);
  std::vector<const std::vector<KernelInvocation>*> plans;
  for (auto& m : ranks_) plans.push_back(&m->plan(key, kEmuBucket, 1));
  const size_t n = plans[0]->size();
  for (size_t i = 0; i < n; ++i) {
    const KernelInvocation& k0 = (*plans[0])[i];
    if (k0.collective == COLL_NONE) {
      for (int r = 0; r < T; ++r) cuda_check((*plans[r])[i].launch(s_), (*plans[r])[i].spec.name.c_str());
      continue;
    }
    TpPtrs in{}, out{};
    for (int r = 0; r < T; ++r) {
      in.p[r] = (*plans[r])[i].coll_in;
      out.p[r] = (*plans[r])[i].coll_out;
    }
    if (k0.collective == COLL_ALLREDUCE)
      cuda_check(launch_emu_allreduce(in, T, k0.coll_n, s_), "emulated allreduce");
    else
      cuda_check(launch_emu_allgather(in, out, T, k0.coll_n, s_), "emulated allgather");
  }
  cuda_check(cudaStreamSynchronize(s_), "tp step");
  ++cur_len_;
  for (auto& m : ranks_) {
    int err = 0;
    cuda_check(cudaMemcpy(&err, &m->ctrl_dev()->err, sizeof(int), cudaMemcpyDeviceToHost), "err");
    if (err & DEVERR_WRONG_LENGTH) raise(GRT_WrongLength, "device: live length outside the graph bucket");
    if (err) raise(GRT_CudaError, "device error flags " + std::to_string(err));
  }
}

void TpEmu::logits(float* out, int n) {
  if (n != ranks_[0]->config().vocab_size) raise(GRT_ShapeMismatch, "logits buffer must hold vocab_size floats");
  cuda_check(cudaMemcpy(out, ranks_[0]->logits_dev(), n * sizeof(float), cudaMemcpyDeviceToHost), "logits");
}

// ---------------------------------------------------------------------------
// Threaded emulation: T ranks = T host threads on one device, each with its own
// Model, Session and stream, exchanging through EmuComm.  Exercises the EAGER
// tensor-parallel paths end to end -- batched prefill (allreduce of the [P, d]
// residual after Wo and down, logits allgather) and single steps -- exactly as
// the NCCL ranks run them (graphs are not captured here: a captured host
// rendezvous would not replay).

namespace {
struct EmuGroup {
  int T = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  TpPtrs in{}, out{};
  size_t n = 0;
  std::vector<cudaEvent_t> ready;
  cudaEvent_t done = nullptr;
};

class EmuComm : public TpComm {
 public:
  EmuComm(EmuGroup* g, int rank) : g_(g), rank_(rank) {}
  cudaError_t allreduce_sum(float* buf, size_t n, cudaStream_t s) override { return run(true, buf, buf, n, s); }
  cudaError_t allgather(const float* in, float* out, size_t n, cudaStream_t s) override {
    return run(false, const_cast<float*>(in), out, n, s);
  }

 private:
  cudaError_t run(bool reduce, float* in, float* out, size_t n, cudaStream_t s) {
    cudaError_t e = cudaEventRecord(g_->ready[rank_], s);
    if (e != cudaSuccess) return e;
    std::unique_lock<std::mutex> lk(g_->mu);
    g_->in.p[rank_] = in;
    g_->out.p[rank_] = out;
    g_->n = n;
    const uint64_t my_gen = g_->gen;
    if (++g_->arrived == g_->T) {  // last rank in: run the exchange on its stream
      for (int r = 0; r < g_->T; ++r) cudaStreamWaitEvent(s, g_->ready[r], 0);
      e = reduce ? launch_emu_allreduce(g_->in, g_->T, n, s) : launch_emu_allgather(g_->in, g_->out, g_->T, n, s);
      if (e == cudaSuccess) e = cudaEventRecord(g_->done, s);
      g_->arrived = 0;
      ++g_->gen;
      g_->cv.notify_all();
      return e;
    }
    g_->cv.wait(lk, [&] { return g_->gen != my_gen; });
    return cudaStreamWaitEvent(s, g_->done, 0);
  }
  EmuGroup* g_;
  int rank_;
};
}  // namespace

void tp_emu_threaded(const ModelConfig& cfg, const std::vector<int>& prompt, const std::vector<int>& steps,
                     float* logits_out) {
  const int T = cfg.tp_size;
  if (T < 2 || T > TP_MAX) raise(GRT_InvalidConfig, "tp_size must be in [2, 8]");
  EmuGroup grp;
  grp.T = T;
  grp.ready.resize(T);
  cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
  for (int r = 0; r < T; ++r) cuda_check(cudaEventCreateWithFlags(&grp.ready[r], cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&grp.done, cudaEventDisableTiming), "event");
  std::vector<std::unique_ptr<Model>> models(T);
  std::vector<std::unique_ptr<EmuComm>> comms(T);
  for (int r = 0; r < T; ++r) {
    ModelConfig c = cfg;
    c.tp_rank = r;
    models[r] = std::make_unique<Model>(c);
    comms[r] = std::make_unique<EmuComm>(&grp, r);
    models[r]->attach_comm(comms[r].get());
  }
  std::vector<std::string> errors(T);
  std::vector<std::thread> th;
  for (int r = 0; r < T; ++r)
    th.emplace_back([&, r] {
      try {
        cudaSetDevice(cfg.device);
        CacheConfig cc;
        cc.warmup_hi = 0;
        cc.batched_prefill = true;
        Session s(*models[r], cc);
        s.prefill(prompt);
        for (int t : steps) s.step(t);
        if (r == 0) s.logits(logits_out, cfg.vocab_size);
      } catch (const std::exception& e) {
        errors[r] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : grp.ready) cudaEventDestroy(e);
  cudaEventDestroy(grp.done);
  for (int r = 0; r < T; ++r)
    if (!errors[r].empty()) raise(GRT_CudaError, "rank " + std::to_string(r) + ": " + errors[r]);
}

}  // namespace grt
