// ipc.cpp -- the paper's two-process split (context generator A / graph
// generator B, PAPER.md) rebuilt on cudaIpc memory + event handles.
//
// Reference: the in-process Channel (pipeline.cpp:56-78) alternates a
// ContextGenerator (dynamic ops: extend_position + kv_append before a pass,
// sample_token after it, pipeline.cpp:87-109) with a GraphGenerator (static
// pass, pipeline.cpp:118-152).  Here they are two OS processes on one GPU:
//   * B owns the model arena and its bucket graphs (static pass only);
//   * A opens B's arena with cudaIpcOpenMemHandle and launches the NVRTC
//     dynamic kernels on B's buffers (ctrl block, token history, embedding, x,
//     logits) -- no activation, logit or token ever crosses the host;
//   * per pass i: A [waits ev_static(i-1)] sample + preprocess, records ev_ctx;
//     B waits ev_ctx, replays the bucket graph, records ev_static.  Both events
//     are cudaEventInterprocess.  A host doorbell (two counters in POSIX shared
//     memory) only orders each cudaStreamWaitEvent after the matching record.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <climits>
#include <cstring>
#include <random>
#include <thread>

#include "runtime.hpp"

namespace {

struct Bell {
  std::atomic<int64_t> ctx;     // passes whose dynamic ops A has enqueued (+ recorded ev_ctx)
  std::atomic<int64_t> stat;    // passes whose static graph B has enqueued (+ recorded ev_static)
  std::atomic<int32_t> abort_;
};

Bell* map_bell(const char* name, bool create) {
  const int fd = shm_open(name, create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) grt::raise(GRT_IpcError, std::string("shm_open ") + name);
  if (create && ftruncate(fd, sizeof(Bell)) != 0) {
    close(fd);
    grt::raise(GRT_IpcError, "ftruncate doorbell");
  }
  void* p = mmap(nullptr, sizeof(Bell), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) grt::raise(GRT_IpcError, "mmap doorbell");
  Bell* b = static_cast<Bell*>(p);
  if (create) {
    new (&b->ctx) std::atomic<int64_t>(0);
    new (&b->stat) std::atomic<int64_t>(0);
    new (&b->abort_) std::atomic<int32_t>(0);
  }
  return b;
}

void wait_at_least(std::atomic<int64_t>& c, int64_t v, const std::atomic<int32_t>& abort_) {
  const auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  while (c.load(std::memory_order_acquire) < v) {
    if (abort_.load(std::memory_order_relaxed)) grt::raise(GRT_IpcError, "peer process aborted");
    if (++spins > 1000) std::this_thread::yield();
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
      grt::raise(GRT_IpcError, "timed out waiting for the peer process");
  }
}

}  // namespace

struct grt_ipc_server {
  grt::Session* s = nullptr;
  grt::Model* m = nullptr;
  Bell* bell = nullptr;
  std::string shm;
  cudaEvent_t ev_ctx = nullptr, ev_static = nullptr;
  cudaStream_t stream = nullptr;
  int64_t passes = 0;  // passes served so far (doorbell counters are monotonic across runs)
};

struct grt_ipc_client {
  grt_ipc_desc d{};
  Bell* bell = nullptr;
  char* arena = nullptr;
  cudaEvent_t ev_ctx = nullptr, ev_static = nullptr;
  cudaStream_t stream = nullptr;
  std::shared_ptr<grt::JitModule> jit;
  CUfunction f_pre = nullptr, f_sample = nullptr;
  GrtCtrl* h_ctrl = nullptr;
  volatile int* h_tokens = nullptr;
  volatile unsigned long long* h_stamps = nullptr;
  int64_t passes = 0;  // passes driven so far (matches the server's count)
};

namespace grt {

grt_ipc_server* ipc_server_create(Session& s, Model& m, const char* shm_name, grt_ipc_desc* d) {
  if (m.tp_size() > 1) raise(GRT_Unsupported, "the two-process split is single-GPU");
  auto sv = std::make_unique<grt_ipc_server>();
  sv->s = &s;
  sv->m = &m;
  sv->shm = shm_name;
  sv->bell = map_bell(shm_name, true);
  cuda_check(cudaSetDevice(m.device()), "cudaSetDevice");
  const unsigned flags = cudaEventInterprocess | cudaEventDisableTiming;
  cuda_check(cudaEventCreateWithFlags(&sv->ev_ctx, flags), "ipc event");
  cuda_check(cudaEventCreateWithFlags(&sv->ev_static, flags), "ipc event");
  sv->stream = s.device().replay();
  std::memset(d, 0, sizeof(*d));
  cudaIpcMemHandle_t mh;
  cuda_check(cudaIpcGetMemHandle(&mh, m.arena().base()), "cudaIpcGetMemHandle");
  std::memcpy(d->arena, &mh, sizeof(mh));
  cudaIpcEventHandle_t eh;
  cuda_check(cudaIpcGetEventHandle(&eh, sv->ev_ctx), "cudaIpcGetEventHandle");
  std::memcpy(d->ev_ctx, &eh, sizeof(eh));
  cuda_check(cudaIpcGetEventHandle(&eh, sv->ev_static), "cudaIpcGetEventHandle");
  std::memcpy(d->ev_static, &eh, sizeof(eh));
  const char* base = m.arena().base();
  auto off = [&](const void* p) { return static_cast<uint64_t>(static_cast<const char*>(p) - base); };
  d->off_ctrl = off(m.ctrl_dev());
  d->off_tokens = off(m.tokens_dev());
  d->off_uniforms = off(m.uniforms_dev());
  d->off_scratch = off(m.scratch_dev());
  d->off_emb = off(m.emb_dev());
  d->off_pos = off(m.pos_dev());
  d->off_x = off(m.x_dev());
  d->off_logits = off(m.logits_dev());
  const ModelConfig& c = m.config();
  d->d_model = c.d_model;
  d->vocab = c.vocab_size;
  d->max_seq = c.max_seq_len;
  d->weight_bf16 = c.weight_dtype == GRT_BF16;
  d->arch_ref = c.llama() ? 0 : 1;
  d->device = c.device;
  d->bucket_size = s.cache_config().bucket_size;
  d->max_gen = m.max_gen();
  return sv.release();
}

void ipc_server_serve(grt_ipc_server* sv, int n) {
  Bell& b = *sv->bell;
  const int B = sv->s->cache_config().bucket_size;
  // the graphs this run needs, captured before the first pass
  std::vector<ExecGraphPtr> graphs;
  for (int key = 1; key <= Model::key_of(n, B); ++key) graphs.push_back(sv->s->static_graph(key));
  cuda_check(cudaStreamSynchronize(sv->s->device().capture_stream()), "captures");
  // The counters never reset: a run's pass i is number base+i+1 on both sides,
  // so a run can never consume the previous run's doorbell or events.
  const int64_t base = sv->passes;
  try {
    for (int i = 0; i < n; ++i) {
      wait_at_least(b.ctx, base + i + 1, b.abort_);
      cuda_check(cudaStreamWaitEvent(sv->stream, sv->ev_ctx, 0), "wait ev_ctx");
      graphs[Model::key_of(i + 1, B) - 1]->launch(sv->stream);
      cuda_check(cudaEventRecord(sv->ev_static, sv->stream), "record ev_static");
      b.stat.store(base + i + 1, std::memory_order_release);
    }
    sv->passes = base + n;
    cuda_check(cudaStreamSynchronize(sv->stream), "serve");
  } catch (...) {
    b.abort_.store(1);
    throw;
  }
}

grt_ipc_client* ipc_client_create(const grt_ipc_desc* d, const char* shm_name) {
  auto c = std::make_unique<grt_ipc_client>();
  c->d = *d;
  cuda_check(cudaSetDevice(d->device), "cudaSetDevice");
  c->bell = map_bell(shm_name, false);
  cudaIpcMemHandle_t mh;
  std::memcpy(&mh, d->arena, sizeof(mh));
  void* p = nullptr;
  cuda_check(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  c->arena = static_cast<char*>(p);
  cudaIpcEventHandle_t eh;
  std::memcpy(&eh, d->ev_ctx, sizeof(eh));
  cuda_check(cudaIpcOpenEventHandle(&c->ev_ctx, eh), "cudaIpcOpenEventHandle");
  std::memcpy(&eh, d->ev_static, sizeof(eh));
  cuda_check(cudaIpcOpenEventHandle(&c->ev_static, eh), "cudaIpcOpenEventHandle");
  cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
  // the same NVRTC specialisation the server's model uses (jit.cpp)
  c->jit = jit_get({"-DGRT_D=" + std::to_string(d->d_model), "-DGRT_V=" + std::to_string(d->vocab),
                    "-DGRT_MAXSEQ=" + std::to_string(d->max_seq),
                    std::string("-DGRT_WBF16=") + (d->weight_bf16 ? "1" : "0"),
                    std::string("-DGRT_ARCH_REF=") + (d->arch_ref ? "1" : "0")},
                   d->device);
  c->f_pre = c->jit->fn("grt_preprocess");
  c->f_sample = c->jit->fn("grt_sample");
  void* h = nullptr;
  cuda_check(cudaHostAlloc(&h, sizeof(GrtCtrl), cudaHostAllocDefault), "cudaHostAlloc");
  c->h_ctrl = static_cast<GrtCtrl*>(h);
  cuda_check(cudaHostAlloc(&h, d->max_gen * sizeof(int), cudaHostAllocMapped), "cudaHostAlloc");
  c->h_tokens = static_cast<volatile int*>(h);
  cuda_check(cudaHostAlloc(&h, 2 * d->max_gen * sizeof(unsigned long long), cudaHostAllocMapped), "cudaHostAlloc");
  c->h_stamps = static_cast<volatile unsigned long long*>(h);
  return c.release();
}

void ipc_client_generate(grt_ipc_client* c, const int* prompt, int p, int n, const grt_sample_params& sp, int* tokens,
                         double* per_token_us) {
  const grt_ipc_desc& d = c->d;
  if (p < 1 || n < 1 || p + n > d.max_seq || n > d.max_gen) raise(GRT_InvalidConfig, "ipc generate: bad lengths");
  Bell& b = *c->bell;
  char* A = c->arena;
  int* tokens_dev = reinterpret_cast<int*>(A + d.off_tokens);
  GrtCtrl* ctrl_dev = reinterpret_cast<GrtCtrl*>(A + d.off_ctrl);
  cuda_check(cudaMemcpyAsync(tokens_dev, prompt, p * sizeof(int), cudaMemcpyHostToDevice, c->stream), "prompt");
  if (sp.kind == GRT_SAMPLE_TEMPERATURE) {  // reference draw order (kernels.cpp:282)
    std::mt19937_64 eng(sp.seed);
    std::vector<double> u(n);
    for (int i = 0; i < n; ++i) u[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
    cuda_check(cudaMemcpyAsync(A + d.off_uniforms, u.data(), n * sizeof(double), cudaMemcpyHostToDevice, c->stream),
               "uniforms");
  }
  for (int i = 0; i < n; ++i) c->h_tokens[i] = -1;
  GrtCtrl& h = *c->h_ctrl;
  std::memset(&h, 0, sizeof(h));
  h.seq_len = 0;
  h.prompt_len = p;
  h.sample_kind = sp.kind;
  h.temperature = sp.temperature;
  h.top_k = sp.top_k;
  h.top_p = sp.top_p;
  h.max_gen = n;
  h.seed = sp.seed;
  h.tokens = tokens_dev;  // addresses valid in THIS process (IPC mapping)
  h.uniforms = reinterpret_cast<const double*>(A + d.off_uniforms);
  h.scratch = reinterpret_cast<float*>(A + d.off_scratch);
  int* dt = nullptr;
  unsigned long long* ds = nullptr;
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dt), const_cast<int*>(c->h_tokens), 0), "mapped");
  cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ds), const_cast<unsigned long long*>(c->h_stamps), 0),
             "mapped");
  h.out_tokens = dt;
  h.out_stamps = ds;
  cuda_check(cudaMemcpyAsync(ctrl_dev, &h, sizeof(GrtCtrl), cudaMemcpyHostToDevice, c->stream), "ctrl");
  cuda_check(cudaStreamSynchronize(c->stream), "ipc setup");

  const void* emb = A + d.off_emb;
  const void* pos = A + d.off_pos;
  float* x = reinterpret_cast<float*>(A + d.off_x);
  const float* logits = reinterpret_cast<const float*>(A + d.off_logits);
  const int pre_threads = std::min(1024, (d.d_model + 31) / 32 * 32);
  const int64_t base = c->passes;
  try {
    for (int i = 0; i < p + n; ++i) {
      if (i > 0) {
        wait_at_least(b.stat, base + i, b.abort_);
        cuda_check(cudaStreamWaitEvent(c->stream, c->ev_static, 0), "wait ev_static");
      }
      {  // sample_token (no-op during the prompt), then extend_position + slot append
        GrtCtrl* a0 = ctrl_dev;
        const float* a1 = logits;
        void* args[] = {&a0, &a1};
        cuda_check(launch_jit(c->f_sample, dim3(1), dim3(1024), args, c->stream, false), "ipc sample");
      }
      {
        GrtCtrl* a0 = ctrl_dev;
        const void* a1 = emb;
        const void* a2 = pos;
        float* a3 = x;
        void* args[] = {&a0, &a1, &a2, &a3};
        cuda_check(launch_jit(c->f_pre, dim3(1), dim3(pre_threads), args, c->stream, false), "ipc preprocess");
      }
      cuda_check(cudaEventRecord(c->ev_ctx, c->stream), "record ev_ctx");
      b.ctx.store(base + i + 1, std::memory_order_release);
    }
    wait_at_least(b.stat, base + p + n, b.abort_);
    // the last pass must retire before this call returns: the next run rewrites
    // the control block the pass reads
    cuda_check(cudaStreamWaitEvent(c->stream, c->ev_static, 0), "wait ev_static");
    c->passes = base + p + n;
    cuda_check(cudaStreamSynchronize(c->stream), "ipc generate");
  } catch (...) {
    b.abort_.store(1);
    throw;
  }
  int err = 0;
  cuda_check(cudaMemcpy(&err, &ctrl_dev->err, sizeof(int), cudaMemcpyDeviceToHost), "err");
  if (err) raise(GRT_CudaError, "device error flags " + std::to_string(err));
  for (int i = 0; i < n; ++i) {
    tokens[i] = c->h_tokens[i];
    if (per_token_us) {
      const double e = static_cast<double>(c->h_stamps[2 * i + 1]);
      const double s0 = i == 0 ? static_cast<double>(c->h_stamps[0]) : static_cast<double>(c->h_stamps[2 * i - 1]);
      per_token_us[i] = (e - s0) / 1000.0;
    }
  }
}

}  // namespace grt

void grt_ipc_server_free(grt_ipc_server* sv) {
  if (!sv) return;
  if (sv->ev_ctx) cudaEventDestroy(sv->ev_ctx);
  if (sv->ev_static) cudaEventDestroy(sv->ev_static);
  if (sv->bell) munmap(sv->bell, sizeof(Bell));
  if (!sv->shm.empty()) shm_unlink(sv->shm.c_str());
  delete sv;
}

void grt_ipc_client_free(grt_ipc_client* c) {
  if (!c) return;
  if (c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  if (c->ev_ctx) cudaEventDestroy(c->ev_ctx);
  if (c->ev_static) cudaEventDestroy(c->ev_static);
  if (c->arena) cudaIpcCloseMemHandle(c->arena);
  if (c->h_ctrl) cudaFreeHost(c->h_ctrl);
  if (c->h_tokens) cudaFreeHost(const_cast<int*>(c->h_tokens));
  if (c->h_stamps) cudaFreeHost(const_cast<unsigned long long*>(c->h_stamps));
  if (c->bell) munmap(c->bell, sizeof(Bell));
  delete c;
}
