// c_api.cpp -- extern "C" boundary (include/grt/c_api.h).  No exception crosses
// it: every graphrt::Error becomes its grt_status and a thread-local message.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>
#include <string>

#include "runtime.hpp"

struct grt_model {
  std::unique_ptr<grt::NcclComm> comm;  // destroyed after the model's sessions (declared first)
  std::unique_ptr<grt::Model> m;
};
struct grt_tp_emu {
  std::unique_ptr<grt::TpEmu> e;
};
struct grt_capture;
struct grt_session {
  grt_model* owner;
  std::unique_ptr<grt::Session> s;
  std::set<grt_capture*> captures;  // live capture handles (orphaned when the session goes first)
  ~grt_session();
};
struct grt_capture {
  grt_session* owner;  // nullptr once the session was destroyed
  bool fused;
  std::unique_ptr<grt::CaptureSession> cs;
  std::vector<std::unique_ptr<grt::KernelInvocation>> external;  // caller-bound ops (kept alive)
};
grt_session::~grt_session() {
  for (grt_capture* c : captures) {  // close them while the engine still exists
    c->cs.reset();
    c->owner = nullptr;
  }
}

namespace {
thread_local std::string g_last_error;

template <typename F>
grt_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return GRT_OK;
  } catch (const grt::Error& e) {
    g_last_error = e.what();
    return e.code();
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return GRT_InvalidConfig;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GRT_CudaError;
  }
}

grt::RunMode to_mode(int32_t m) {
  if (m < 0 || m > 6) grt::raise(GRT_InvalidConfig, "unknown mode " + std::to_string(m));
  return static_cast<grt::RunMode>(m);
}
}  // namespace

extern "C" {

const char* grt_status_name(grt_status s) { return grt::errc_name(s); }
const char* grt_last_error(void) { return g_last_error.c_str(); }
int32_t grt_abi_version(void) { return GRT_ABI_VERSION; }

grt_status grt_jit_compile_check(int32_t d_model, int32_t vocab, int32_t max_seq, int32_t weight_bf16, int32_t arch_ref,
                                 uint64_t* cubin_bytes) {
  return guard([&] {
    const std::string cubin = grt::jit_compile({"-DGRT_D=" + std::to_string(d_model), "-DGRT_V=" + std::to_string(vocab),
                                                "-DGRT_MAXSEQ=" + std::to_string(max_seq),
                                                "-DGRT_WBF16=" + std::to_string(weight_bf16 ? 1 : 0),
                                                "-DGRT_ARCH_REF=" + std::to_string(arch_ref ? 1 : 0)});
    if (cubin_bytes) *cubin_bytes = cubin.size();
  });
}

grt_status grt_device_count(int32_t* n) {
  return guard([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *n = c;
  });
}

void grt_model_config_default(grt_model_config* c) {
  std::memset(c, 0, sizeof(*c));
  grt::ModelConfig d;
  c->arch = d.arch;
  c->n_layers = d.n_layers;
  c->d_model = d.d_model;
  c->n_heads = d.n_heads;
  c->vocab_size = d.vocab_size;
  c->max_seq_len = d.max_seq_len;
  c->d_ff = 0;
  c->norm_eps = d.norm_eps;
  c->seed = d.seed;
  c->init = d.init;
  c->weight_dtype = d.weight_dtype;
  c->kv_dtype = d.kv_dtype;
  c->rope_theta = d.rope_theta;
  c->device = 0;
  c->tp_size = 1;
  c->tp_rank = 0;
  c->kv_page_size = 0;
}

void grt_cache_config_default(grt_cache_config* c) {
  std::memset(c, 0, sizeof(*c));
  grt::CacheConfig d;
  c->capacity = d.capacity;
  c->warmup_lo = d.warmup_lo;
  c->warmup_hi = d.warmup_hi;
  c->prefill_uses_graphs = d.prefill_uses_graphs ? 1 : 0;
  c->policy = GRT_EVICT_LEAST_USED;
  c->bucket_size = d.bucket_size;
  c->batched_prefill = d.batched_prefill ? 1 : 0;
  c->pass_impl = d.pass_impl;
  c->prefill_fuse_norm = d.prefill_fuse_norm ? 1 : 0;
}

grt_status grt_model_create(const grt_model_config* cfg, grt_model** out) {
  return guard([&] {
    if (!cfg || !out) grt::raise(GRT_InvalidConfig, "null argument");
    auto h = std::make_unique<grt_model>();
    h->m = std::make_unique<grt::Model>(grt::ModelConfig::from_c(*cfg));
    *out = h.release();
  });
}

grt_status grt_tp_unique_id(uint8_t* out, int32_t len) {
  return guard([&] {
    const std::vector<uint8_t> id = grt::nccl_unique_id();
    if (!out || len < static_cast<int32_t>(id.size())) grt::raise(GRT_InvalidConfig, "unique id buffer too small");
    std::memcpy(out, id.data(), id.size());
  });
}

grt_status grt_model_attach_nccl(grt_model* m, const uint8_t* unique_id, int32_t len) {
  return guard([&] {
    if (!m || !unique_id || len < GRT_TP_UNIQUE_ID_BYTES) grt::raise(GRT_InvalidConfig, "bad arguments");
    const grt::ModelConfig& c = m->m->config();
    m->comm = std::make_unique<grt::NcclComm>(unique_id, c.tp_size, c.tp_rank, c.device);
    m->m->attach_comm(m->comm.get());
  });
}

grt_status grt_tp_emu_create(const grt_model_config* cfg, grt_tp_emu** out) {
  return guard([&] {
    if (!cfg || !out) grt::raise(GRT_InvalidConfig, "null argument");
    auto h = std::make_unique<grt_tp_emu>();
    h->e = std::make_unique<grt::TpEmu>(grt::ModelConfig::from_c(*cfg));
    *out = h.release();
  });
}
grt_status grt_tp_emu_destroy(grt_tp_emu* e) {
  return guard([&] { delete e; });
}
grt_status grt_tp_emu_reset(grt_tp_emu* e) {
  return guard([&] { e->e->reset(); });
}
grt_status grt_tp_emu_step(grt_tp_emu* e, int32_t token) {
  return guard([&] { e->e->step(token); });
}
grt_status grt_tp_emu_logits(grt_tp_emu* e, float* out, int32_t n) {
  return guard([&] { e->e->logits(out, n); });
}

grt_status grt_ipc_server_create(grt_session* s, const char* shm_name, grt_ipc_desc* desc, grt_ipc_server** out) {
  return guard([&] {
    if (!s || !shm_name || !desc || !out) grt::raise(GRT_InvalidConfig, "null argument");
    *out = grt::ipc_server_create(*s->s, *s->owner->m, shm_name, desc);
  });
}
grt_status grt_ipc_server_serve(grt_ipc_server* sv, int32_t n_passes) {
  return guard([&] { grt::ipc_server_serve(sv, n_passes); });
}
grt_status grt_ipc_server_destroy(grt_ipc_server* sv) {
  return guard([&] { grt_ipc_server_free(sv); });
}
grt_status grt_ipc_client_create(const grt_ipc_desc* desc, const char* shm_name, grt_ipc_client** out) {
  return guard([&] {
    if (!desc || !shm_name || !out) grt::raise(GRT_InvalidConfig, "null argument");
    *out = grt::ipc_client_create(desc, shm_name);
  });
}
grt_status grt_ipc_client_generate(grt_ipc_client* c, const int32_t* prompt, int32_t prompt_len, int32_t gen_len,
                                   const grt_sample_params* sampling, int32_t* tokens, double* per_token_us) {
  return guard([&] {
    if (!c || !prompt || !sampling || !tokens) grt::raise(GRT_InvalidConfig, "null argument");
    grt::ipc_client_generate(c, prompt, prompt_len, gen_len, *sampling, tokens, per_token_us);
  });
}
grt_status grt_ipc_client_destroy(grt_ipc_client* c) {
  return guard([&] { grt_ipc_client_free(c); });
}

grt_status grt_tp_emu_threaded(const grt_model_config* cfg, const int32_t* prompt, int32_t n_prompt,
                               const int32_t* steps, int32_t n_steps, float* logits) {
  return guard([&] {
    if (!cfg || !prompt || n_prompt < 1 || !logits || (n_steps > 0 && !steps))
      grt::raise(GRT_InvalidConfig, "bad arguments");
    grt::tp_emu_threaded(grt::ModelConfig::from_c(*cfg), std::vector<int>(prompt, prompt + n_prompt),
                         std::vector<int>(steps, steps + std::max(0, n_steps)), logits);
  });
}

grt_status grt_model_destroy(grt_model* m) {
  return guard([&] { delete m; });
}

grt_status grt_model_upload(grt_model* m, const char* tensor, const void* host, size_t bytes, int32_t host_dtype) {
  return guard([&] { m->m->upload(tensor, host, bytes, host_dtype); });
}

grt_status grt_model_download(grt_model* m, const char* tensor, float* host, size_t numel) {
  return guard([&] { m->m->download(tensor, host, numel); });
}

grt_status grt_model_load_safetensors(grt_model* m, const char* path, int32_t strict, int32_t* n_loaded) {
  return guard([&] {
    const int n = grt::load_safetensors(*m->m, path, strict != 0);
    if (n_loaded) *n_loaded = n;
  });
}

grt_status grt_safetensors_list(const char* path, char* names, int32_t names_len, int32_t* dtypes, int64_t* shapes,
                                int32_t cap, int32_t* n) {
  return guard([&] {
    grt::SafetensorsFile f(path);
    const auto& ts = f.tensors();
    *n = static_cast<int32_t>(ts.size());
    size_t off = 0;
    for (size_t i = 0; i < ts.size() && static_cast<int32_t>(i) < cap; ++i) {
      if (dtypes) dtypes[i] = ts[i].dtype;
      if (shapes) {
        shapes[3 * i] = static_cast<int64_t>(ts[i].shape.size());
        shapes[3 * i + 1] = ts[i].shape.size() > 0 ? ts[i].shape[0] : 0;
        shapes[3 * i + 2] = ts[i].shape.size() > 1 ? ts[i].shape[1] : 0;
      }
      if (names && off + ts[i].name.size() + 1 <= static_cast<size_t>(names_len)) {
        memcpy(names + off, ts[i].name.c_str(), ts[i].name.size() + 1);
        off += ts[i].name.size() + 1;
      }
    }
  });
}

grt_status grt_hf_tensor_name(const char* hf_name, char* out, int32_t out_len, int32_t* out_in) {
  return guard([&] {
    bool oi = false;
    const std::string s = grt::hf_to_grt_name(hf_name, &oi);
    if (static_cast<int32_t>(s.size()) + 1 > out_len) grt::raise(GRT_InvalidConfig, "output buffer too small");
    memcpy(out, s.c_str(), s.size() + 1);
    if (out_in) *out_in = oi ? 1 : 0;
  });
}

grt_status grt_model_kv_pages(grt_model* m, int32_t* page_size, int32_t* n_pages) {
  return guard([&] {
    if (page_size) *page_size = m->m->kv_paging().page;
    if (n_pages) *n_pages = m->m->kv_pages();
  });
}

grt_status grt_model_set_kv_block_table(grt_model* m, const int32_t* table, int32_t n) {
  return guard([&] { m->m->set_kv_block_table(table, n); });
}

grt_status grt_model_weight_bytes(grt_model* m, uint64_t* bytes) {
  return guard([&] { *bytes = m->m->weight_bytes(); });
}

grt_status grt_model_decode_bytes(grt_model* m, int32_t length, uint64_t* bytes) {
  return guard([&] { *bytes = m->m->decode_bytes(length); });
}

grt_status grt_session_create(grt_model* m, const grt_cache_config* cc, grt_session** out) {
  return guard([&] {
    if (!m || !out) grt::raise(GRT_InvalidConfig, "null argument");
    grt_cache_config def;
    grt_cache_config_default(&def);
    auto h = std::make_unique<grt_session>();
    h->owner = m;
    h->s = std::make_unique<grt::Session>(*m->m, grt::CacheConfig::from_c(cc ? *cc : def));
    *out = h.release();
  });
}

grt_status grt_session_destroy(grt_session* s) {
  return guard([&] { delete s; });
}

grt_status grt_generate(grt_session* s, const grt_generation_request* req, grt_generation_result* res) {
  return guard([&] {
    if (!s || !req || !res) grt::raise(GRT_InvalidConfig, "null argument");
    grt::GenerationRequest r;
    r.mode = to_mode(req->mode);
    if (req->prompt_len > 0 && !req->prompt) grt::raise(GRT_InvalidConfig, "null prompt");
    r.prompt.assign(req->prompt, req->prompt + std::max(0, req->prompt_len));
    r.gen_len = req->gen_len;
    r.sampling = req->sampling;
    r.eos_token = req->stop_on_eos ? req->eos_token : -1;
    grt::GenerationResult out = s->s->run(r);
    if (res->tokens) std::memcpy(res->tokens, out.tokens.data(), out.tokens.size() * sizeof(int32_t));
    if (res->per_token_us) std::memcpy(res->per_token_us, out.per_token_us.data(), out.per_token_us.size() * sizeof(double));
    if (res->prefill_paths)
      for (size_t i = 0; i < out.prefill_paths.size(); ++i) res->prefill_paths[i] = static_cast<int32_t>(out.prefill_paths[i]);
    if (res->decode_paths)
      for (size_t i = 0; i < out.decode_paths.size(); ++i) res->decode_paths[i] = static_cast<int32_t>(out.decode_paths[i]);
    res->ttft_us = out.ttft_us;
    res->total_us = out.total_us;
    res->prefill_us = out.prefill_us;
    res->counters = out.counters;
    res->cache_delta = out.cache_delta;
    res->captures_completed = out.captures_completed;
    res->cache_released = out.cache_released;
    if (res->host_token_us)
      std::memcpy(res->host_token_us, out.host_token_us.data(), out.host_token_us.size() * sizeof(double));
  });
}

grt_status grt_trace_pass(grt_session* s, int32_t key, uint64_t* out, int64_t cap, int32_t* grid, int32_t* stride) {
  return guard([&] {
    int gr = 0, st = 0;
    s->s->device().sync_all();
    auto v = s->owner->m->trace_pass(key, s->s->cache_config().bucket_size, s->s->device().replay(), &gr, &st,
                                     s->s->cache_config().pass_impl);
    *grid = gr;
    *stride = st;
    for (int64_t i = 0; i < cap && i < static_cast<int64_t>(v.size()); ++i) out[i] = v[i];
  });
}

grt_status grt_profile_plan(grt_session* s, int32_t key, int32_t iters, double* avg_ms, int64_t* bytes, char* names,
                            int32_t names_len, int32_t cap, int32_t* n) {
  return guard([&] {
    auto prof = s->s->profile_plan(key, iters);
    if (n) *n = static_cast<int32_t>(prof.size());
    int32_t off = 0;
    for (int32_t i = 0; i < static_cast<int32_t>(prof.size()) && i < cap; ++i) {
      if (avg_ms) avg_ms[i] = prof[i].avg_ms;
      if (bytes) bytes[i] = prof[i].bytes;
      if (names && off + static_cast<int32_t>(prof[i].name.size()) + 1 <= names_len) {
        std::memcpy(names + off, prof[i].name.c_str(), prof[i].name.size() + 1);
        off += static_cast<int32_t>(prof[i].name.size()) + 1;
      }
    }
  });
}

grt_status grt_cache_stats_get(grt_session* s, grt_cache_stats* st, uint64_t* size) {
  return guard([&] {
    if (st) *st = s->s->cache().stats();
    if (size) *size = s->s->cache().size();
  });
}

grt_status grt_capture_begin(grt_session* s, int32_t key, int32_t fused, grt_capture** out) {
  return guard([&] {
    auto c = std::make_unique<grt_capture>();
    c->owner = s;
    c->fused = fused != 0;
    c->cs = s->s->begin_capture(key, c->fused);
    s->captures.insert(c.get());
    *out = c.release();
  });
}

namespace {
void live(const grt_capture* c) {
  if (!c || !c->owner || !c->cs) grt::raise(GRT_SessionClosed, "capture: its session was destroyed");
}
}  // namespace

grt_status grt_capture_record(grt_capture* c, int32_t op, int32_t plan_key, int32_t index) {
  return guard([&] {
    live(c);
    const grt::KernelInvocation* k = c->owner->s->capture_op(op, plan_key, index);
    c->cs->record(k);
  });
}

grt_status grt_capture_record_external(grt_capture* c, void* ptr, uint64_t bytes) {
  return guard([&] {
    live(c);
    auto k = std::make_unique<grt::KernelInvocation>();
    k->spec.name = "external_memset";
    k->bindings = {{ptr, static_cast<size_t>(bytes)}};
    k->launch = [ptr, bytes](cudaStream_t st) { return cudaMemsetAsync(ptr, 0, bytes, st); };
    c->cs->record(k.get());
    c->external.push_back(std::move(k));
  });
}

grt_status grt_capture_end(grt_capture* c, int32_t* kernel_count, uint64_t* epoch) {
  return guard([&] {
    live(c);
    grt::ExecGraphPtr g = c->owner->s->end_capture(*c->cs, c->fused);
    if (kernel_count) *kernel_count = static_cast<int32_t>(g->kernel_count());
    if (epoch) *epoch = g->capture_epoch();
  });
}

grt_status grt_capture_state_get(grt_capture* c, int32_t* state, int32_t* recorded) {
  return guard([&] {
    live(c);
    if (state) *state = static_cast<int32_t>(c->cs->state());
    if (recorded) *recorded = static_cast<int32_t>(c->cs->recorded());
  });
}

void grt_capture_destroy(grt_capture* c) {
  if (!c) return;
  if (c->owner) c->owner->captures.erase(c);
  delete c;
}

grt_status grt_plan_size(grt_session* s, int32_t key, int32_t* n) {
  return guard([&] {
    const grt::CacheConfig& cc = s->s->cache_config();
    *n = static_cast<int32_t>(s->owner->m->plan(key, cc.bucket_size, cc.pass_impl).size());
  });
}

grt_status grt_session_replay(grt_session* s, int32_t key, int32_t fused, int32_t token, int32_t validate) {
  return guard([&] { s->s->replay(key, fused != 0, token, validate != 0); });
}

grt_status grt_model_arena_info(grt_model* m, uint64_t* capacity, uint64_t* used, uint64_t* allocations) {
  return guard([&] {
    const grt::Arena& a = m->m->arena();
    if (capacity) *capacity = a.capacity();
    if (used) *used = a.used();
    if (allocations) *allocations = a.allocations();
  });
}

grt_status grt_model_tp_info(grt_model* m, int32_t* tp_size, int32_t* tp_rank, int32_t* symmetric) {
  return guard([&] {
    const grt::ModelConfig& c = m->m->config();
    if (tp_size) *tp_size = c.tp_size;
    if (tp_rank) *tp_rank = c.tp_rank;
    if (symmetric) *symmetric = m->m->symmetric_exchange() ? 1 : 0;
  });
}

grt_status grt_session_counters(grt_session* s, grt_counters* c) {
  return guard([&] { *c = s->s->device().counters(); });
}

grt_status grt_reset(grt_session* s) {
  return guard([&] { s->s->reset(); });
}

grt_status grt_step(grt_session* s, int32_t token) {
  return guard([&] { s->s->step(token); });
}

grt_status grt_prefill(grt_session* s, const int32_t* ids, int32_t n) {
  return guard([&] {
    std::vector<int> v;
    if (n > 0) v.assign(ids, ids + n);
    s->s->prefill(v);
  });
}

grt_status grt_cur_len(grt_session* s, int32_t* len) {
  return guard([&] { *len = s->s->cur_len(); });
}

grt_status grt_get_logits(grt_session* s, float* out, int32_t n) {
  return guard([&] { s->s->logits(out, n); });
}

grt_status grt_get_kv_row(grt_session* s, int32_t layer, int32_t slot, int32_t row, float* out) {
  return guard([&] { s->s->kv_row(layer, slot, row, out); });
}

grt_status grt_sample(grt_session* s, const grt_sample_params* p, int32_t* token) {
  return guard([&] { *token = s->s->sample(*p); });
}

grt_status grt_sampler_reset(grt_session* s, uint64_t seed) {
  return guard([&] { s->s->sampler_reset(seed); });
}

// ---- standalone graph cache (policy port, host only) -----------------------

struct grt_graph_cache {
  std::unique_ptr<grt::GraphCache> c;
};

grt_status grt_graph_cache_create(uint64_t capacity, int32_t policy, grt_graph_cache** out) {
  return guard([&] {
    auto h = std::make_unique<grt_graph_cache>();
    h->c = std::make_unique<grt::GraphCache>(
        capacity, policy == GRT_EVICT_LRU ? grt::EvictionPolicy::LeastRecentlyUsed : grt::EvictionPolicy::LeastUsed);
    *out = h.release();
  });
}

grt_status grt_graph_cache_destroy(grt_graph_cache* c) {
  return guard([&] { delete c; });
}

grt_status grt_graph_cache_lookup(grt_graph_cache* c, int32_t key, int32_t* hit) {
  return guard([&] { *hit = c->c->lookup(key).has_value() ? 1 : 0; });
}

grt_status grt_graph_cache_insert(grt_graph_cache* c, int32_t key, int32_t graph_key, int32_t* evicted) {
  return guard([&] {
    auto g = std::make_shared<grt::ExecGraph>(graph_key, nullptr, 1, 0, 0, -1);
    auto v = c->c->insert(key, std::move(g));
    *evicted = v ? *v : INT32_MIN;
    c->c->take_dropped();
  });
}

grt_status grt_graph_cache_warmup(grt_graph_cache* c, int32_t lo, int32_t hi, int32_t* captured) {
  return guard([&] {
    *captured = c->c->precapture_warmup(
        lo, hi, [](int key) { return std::make_shared<grt::ExecGraph>(key, nullptr, 1, 0, 0, -1); });
  });
}

grt_status grt_graph_cache_begin_session(grt_graph_cache* c) {
  return guard([&] { c->c->begin_session(); });
}

grt_status grt_graph_cache_release_inactive(grt_graph_cache* c, uint64_t* dropped) {
  return guard([&] {
    *dropped = c->c->release_inactive();
    c->c->take_dropped();
  });
}

grt_status grt_graph_cache_query(grt_graph_cache* c, int32_t key, int32_t* contains, uint64_t* use_count,
                                 uint64_t* size, grt_cache_stats* st) {
  return guard([&] {
    if (contains) *contains = c->c->contains(key) ? 1 : 0;
    if (use_count) *use_count = c->c->contains(key) ? c->c->use_count(key) : 0;
    if (size) *size = c->c->size();
    if (st) *st = c->c->stats();
  });
}

// ---- op-level entry points ------------------------------------------------

grt_status grt_op_gemv(const void* w, int32_t w_dtype, const float* x, float* out, int32_t n, int32_t k, void* stream) {
  return guard([&] {
    grt::GemvParams p;
    p.w = w;
    p.n_rows = n;
    p.k = k;
    p.x = x;
    p.out = out;
    int dev = 0;
    grt::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    grt::cuda_check(grt::gemv_prepare(dev), "gemv_prepare");
    grt::cuda_check(grt::launch_gemv(w_dtype == GRT_BF16 ? grt::Dt::BF16 : grt::Dt::F32, grt::NORM_NONE,
                                     grt::EPI_STORE, p, static_cast<cudaStream_t>(stream), false, 0),
                    "launch_gemv");
  });
}

grt_status grt_op_prefill_gemm(const void* w, const void* x, float* out, int32_t m_rows, int32_t k, int32_t n_tok,
                               void* stream) {
  return guard([&] {
    int dev = 0;
    grt::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    grt::cuda_check(grt::prefill_gemm_prepare(), "prefill_gemm_prepare");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    grt::PrefillGemmParams p;
    p.M = m_rows;
    p.K = k;
    p.P = n_tok;
    p.epi = grt::PG_EPI_STORE;
    p.out = out;
    const size_t nf = grt::prefill_gemm_part_floats(m_rows, k, n_tok, grt::num_sms(dev));
    if (nf) {
      grt::cuda_check(cudaMalloc(&p.part, nf * sizeof(float)), "cudaMalloc");
      grt::cuda_check(cudaMalloc(&p.counters, 4096 * sizeof(int)), "cudaMalloc");
      grt::cuda_check(cudaMemsetAsync(p.counters, 0, 4096 * sizeof(int), st), "cudaMemset");
    }
    const cudaError_t e = grt::launch_prefill_gemm(w, x, p, st, false);
    const cudaError_t e2 = cudaStreamSynchronize(st);
    if (p.part) cudaFree(p.part);
    if (p.counters) cudaFree(p.counters);
    grt::cuda_check(e, "launch_prefill_gemm");
    grt::cuda_check(e2, "prefill_gemm");
  });
}

grt_status grt_op_attention(const float* q, const void* k, const void* v, int32_t kv_dtype, float* out, int32_t n_heads,
                            int32_t head_dim, int32_t max_seq, int32_t len, float scale, void* stream) {
  return guard([&] {
    // the kernel loads q and the K/V rows with 16-byte vector loads
    if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
         reinterpret_cast<uintptr_t>(out)) & 15)
      grt::raise(GRT_InvalidConfig, "op_attention: q, k, v and out must be 16-byte aligned");
    int dev = 0;
    grt::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    grt::cuda_check(grt::attention_prepare(), "attention_prepare");
    grt::AttnParams a;
    a.q = q;
    a.k_cache = k;
    a.v_cache = v;
    a.out = out;
    a.len_fixed = len;
    a.n_heads = n_heads;
    a.head_dim = head_dim;
    a.max_seq = max_seq;
    a.scale = scale;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    grt::cuda_check(grt::launch_attention(kv_dtype == GRT_BF16 ? grt::Dt::BF16 : grt::Dt::F32, a, len, st, false),
                    "launch_attention");
    grt::cuda_check(cudaStreamSynchronize(st), "attention");
  });
}

grt_status grt_op_sample(const float* logits, int32_t vocab, const grt_sample_params* p, uint64_t step, double uniform,
                         int32_t* token_dev, void* stream) {
  return guard([&] {
    if (!p || vocab < 1 || step > (1u << 20)) grt::raise(GRT_InvalidConfig, "grt_op_sample: bad arguments");
    if (reinterpret_cast<uintptr_t>(logits) & 15)  // float4 loads of the logits
      grt::raise(GRT_InvalidConfig, "grt_op_sample: logits must be 16-byte aligned");
    int dev = 0;
    grt::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    auto jit = grt::jit_get({"-DGRT_D=8", "-DGRT_V=" + std::to_string(vocab), "-DGRT_MAXSEQ=1", "-DGRT_WBF16=0",
                             "-DGRT_ARCH_REF=0"},
                            dev);
    {  // keep the last few op-level modules alive (jit_get caches weakly): no NVRTC compile per call
      static std::mutex mu;
      static std::vector<std::shared_ptr<grt::JitModule>> keep;
      std::lock_guard<std::mutex> lk(mu);
      if (std::find(keep.begin(), keep.end(), jit) == keep.end()) {
        keep.push_back(jit);
        if (keep.size() > 8) keep.erase(keep.begin());
      }
    }
    CUfunction f = jit->fn("grt_sample");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // scratch: ctrl | tokens[step+1] | uniforms[step+1] | probs[vocab]
    const size_t n = static_cast<size_t>(step) + 1;
    char* buf = nullptr;
    const size_t bytes = 256 + n * 4 + 256 + n * 8 + static_cast<size_t>(vocab) * 4 + 256;
    grt::cuda_check(cudaMalloc(&buf, bytes), "cudaMalloc");
    GrtCtrl* ctrl = reinterpret_cast<GrtCtrl*>(buf);
    int* tokens = reinterpret_cast<int*>(buf + 256);
    double* uniforms = reinterpret_cast<double*>(buf + 256 + (n * 4 + 255) / 256 * 256);
    float* scratch = reinterpret_cast<float*>(reinterpret_cast<char*>(uniforms) + (n * 8 + 255) / 256 * 256);
    GrtCtrl h{};
    h.seq_len = static_cast<int>(step);
    h.prompt_len = 0;
    h.sample_kind = p->kind;
    h.temperature = p->temperature;
    h.top_k = p->top_k;
    h.top_p = p->top_p;
    h.max_gen = 0;  // no host-mapped outputs
    h.seed = p->seed;
    h.tokens = tokens;
    h.uniforms = uniforms;
    h.scratch = scratch;
    grt::cuda_check(cudaMemcpyAsync(ctrl, &h, sizeof(h), cudaMemcpyHostToDevice, st), "ctrl");
    grt::cuda_check(cudaMemcpyAsync(uniforms + step, &uniform, sizeof(double), cudaMemcpyHostToDevice, st), "u");
    void* args[] = {&ctrl, &logits};
    grt::cuda_check(grt::launch_jit(f, dim3(1), dim3(1024), args, st, false), "launch sample");
    grt::cuda_check(cudaMemcpyAsync(token_dev, tokens + step, sizeof(int), cudaMemcpyDeviceToDevice, st), "token");
    grt::cuda_check(cudaStreamSynchronize(st), "sample");
    cudaFree(buf);
  });
}

}  // extern "C"
