// model.cpp -- Model: device arena, weights, KV cache, static plans, dynamic ops.
//
// Mirrors graphrt::Model (model.hpp:58-132, model.cpp:30-183).  The reference's
// 14 kernels per layer (model.hpp:74-83) become 5 fused sm_100a kernels:
//   qkv   = ln1 + wq/wk/wv + (RoPE) + kv_write_k/v         (gemv.cu, EPI_QKV*)
//   attn  = attention over [0, seq_len)                     (attention.cu)
//   wo    = wo + residual_add                               (gemv.cu, EPI_RESID)
//   up    = ln2 + w1 + relu  |  rms + gate/up + SwiGLU      (gemv.cu, EPI_RELU/SWIGLU)
//   down  = w2 + residual_add                               (gemv.cu, EPI_RESID)
// plus ln_f + head (EPI_STORE).  Every length-dependent value is read from the
// device control block, so a plan is keyed by a BUCKET of lengths, not one.
#include <cmath>
#include <cstring>
#include <random>

#include "runtime.hpp"

namespace grt {

// ---------------------------------------------------------------------------
// errors

const char* errc_name(Errc c) noexcept {
  switch (c) {
    case GRT_OK: return "Ok";
    case GRT_ShapeMismatch: return "ShapeMismatch";
    case GRT_TokenOutOfRange: return "TokenOutOfRange";
    case GRT_EmptyCache: return "EmptyCache";
    case GRT_CacheFull: return "CacheFull";
    case GRT_InvalidConfig: return "InvalidConfig";
    case GRT_LengthOutOfRange: return "LengthOutOfRange";
    case GRT_PromptTooLong: return "PromptTooLong";
    case GRT_EmptyPrompt: return "EmptyPrompt";
    case GRT_CaptureInProgress: return "CaptureInProgress";
    case GRT_CaptureViolation: return "CaptureViolation";
    case GRT_ForeignBuffer: return "ForeignBuffer";
    case GRT_SessionClosed: return "SessionClosed";
    case GRT_EmptyCapture: return "EmptyCapture";
    case GRT_ReplayShapeError: return "ReplayShapeError";
    case GRT_WrongLength: return "WrongLength";
    case GRT_KeyMismatch: return "KeyMismatch";
    case GRT_WarmupExceedsCapacity: return "WarmupExceedsCapacity";
    case GRT_StaticInFusedBlock: return "StaticInFusedBlock";
    case GRT_DeviceStopped: return "DeviceStopped";
    case GRT_UnknownEvent: return "UnknownEvent";
    case GRT_EmptySamples: return "EmptySamples";
    case GRT_IoError: return "IoError";
    case GRT_CudaError: return "CudaError";
    case GRT_NvrtcError: return "NvrtcError";
    case GRT_NcclError: return "NcclError";
    case GRT_IpcError: return "IpcError";
    case GRT_Unsupported: return "Unsupported";
    case GRT_NoDevice: return "NoDevice";
  }
  return "UnknownError";
}

void raise(Errc code, const std::string& what) { throw Error(code, std::string(errc_name(code)) + ": " + what); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) raise(GRT_NoDevice, std::string(what) + ": " + cudaGetErrorString(e));
    raise(GRT_CudaError, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void cu_check(CUresult e, const char* what) {
  if (e != CUDA_SUCCESS) {
    raise(GRT_CudaError, std::string(what) + ": " + cu_error_string(e));
  }
}

// ---------------------------------------------------------------------------
// config

void ModelConfig::validate() const {
  // ModelConfig::validate (model.cpp:10-18)
  if (n_layers < 1) raise(GRT_InvalidConfig, "n_layers must be >= 1");
  if (d_model < 1) raise(GRT_InvalidConfig, "d_model must be >= 1");
  if (n_heads < 1) raise(GRT_InvalidConfig, "n_heads must be >= 1");
  if (d_model % n_heads != 0) raise(GRT_InvalidConfig, "d_model must be divisible by n_heads");
  if (vocab_size < 1) raise(GRT_InvalidConfig, "vocab_size must be >= 1");
  if (max_seq_len < 1) raise(GRT_InvalidConfig, "max_seq_len must be >= 1");
  if (!(norm_eps > 0.0f)) raise(GRT_InvalidConfig, "ln_eps must be positive");
  // device-layout requirements (16-byte bulk copies, 4-wide attention lanes)
  if (d_model % 8 != 0) raise(GRT_InvalidConfig, "d_model must be a multiple of 8 (16-byte rows)");
  if (d_ff() % 8 != 0) raise(GRT_InvalidConfig, "d_ff must be a multiple of 8");
  const int dh = head_dim();
  if (dh % 4 != 0 || dh > 128 || ((dh / 4) & (dh / 4 - 1)) != 0)
    raise(GRT_InvalidConfig, "head_dim must be 4*2^k <= 128");
  if (arch != GRT_ARCH_REF && arch != GRT_ARCH_LLAMA) raise(GRT_InvalidConfig, "unknown arch");
  if (weight_dtype != GRT_F32 && weight_dtype != GRT_BF16) raise(GRT_InvalidConfig, "weight_dtype");
  if (kv_dtype != GRT_F32 && kv_dtype != GRT_BF16) raise(GRT_InvalidConfig, "kv_dtype");
  if (init != GRT_INIT_MT19937 && init != GRT_INIT_PHILOX && init != GRT_INIT_NONE) raise(GRT_InvalidConfig, "init");
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) raise(GRT_InvalidConfig, "tp_rank must be in [0, tp_size)");
  if (kv_page_size < 0 || kv_page_size > max_seq_len) raise(GRT_InvalidConfig, "kv_page_size must be in [0, max_seq_len]");
  if (tp_size > 1) {
    if (arch != GRT_ARCH_LLAMA) raise(GRT_Unsupported, "tensor parallelism is implemented for the LLaMA arch");
    if (n_heads % tp_size != 0) raise(GRT_InvalidConfig, "n_heads must be divisible by tp_size");
    if (d_ff() % tp_size != 0 || (d_ff() / tp_size) % 8 != 0)
      raise(GRT_InvalidConfig, "d_ff / tp_size must be a multiple of 8");
    if (vocab_size % tp_size != 0) raise(GRT_InvalidConfig, "vocab_size must be divisible by tp_size");
    if ((d_model / tp_size) % 8 != 0) raise(GRT_InvalidConfig, "d_model / tp_size must be a multiple of 8");
  }
}

ModelConfig ModelConfig::from_c(const grt_model_config& c) {
  ModelConfig m;
  m.arch = c.arch;
  m.n_layers = c.n_layers;
  m.d_model = c.d_model;
  m.n_heads = c.n_heads;
  m.vocab_size = c.vocab_size;
  m.max_seq_len = c.max_seq_len;
  m.d_ff_ = c.d_ff;
  m.norm_eps = c.norm_eps;
  m.seed = c.seed;
  m.init = c.init;
  m.weight_dtype = c.weight_dtype;
  m.kv_dtype = c.kv_dtype;
  m.rope_theta = c.rope_theta;
  m.device = c.device;
  m.tp_size = c.tp_size < 1 ? 1 : c.tp_size;
  m.tp_rank = c.tp_rank;
  m.kv_page_size = c.kv_page_size;
  return m;
}

// ---------------------------------------------------------------------------
// arena

Arena::~Arena() {
  if (base_) cudaFree(base_);
}

void Arena::reserve(size_t bytes) {
  if (base_) raise(GRT_InvalidConfig, "arena already reserved");
  cuda_check(cudaMalloc(&base_, bytes), "cudaMalloc(arena)");
  cuda_check(cudaMemset(base_, 0, bytes), "cudaMemset(arena)");
  cap_ = bytes;
}

void* Arena::alloc(size_t bytes, size_t align) {
  size_t off = (used_ + align - 1) / align * align;
  if (off + bytes > cap_) raise(GRT_InvalidConfig, "arena overflow");
  used_ = off + bytes;
  ++count_;
  return base_ + off;
}

bool Arena::contains(const void* p, size_t n) const {
  const char* c = static_cast<const char*>(p);
  if (base_ && c >= base_ && c + n <= base_ + cap_) return true;
  for (const auto& [b, len] : extra_)
    if (c >= b && c + n <= b + len) return true;
  return false;
}

// Collectives are planned whenever a communicator is attached (a 1-rank group
// included).  The residual stream x -- the buffer every per-layer allreduce
// reduces in place -- moves into memory registered with the communicator when
// it supports that (NCCL symmetric windows: the low-latency symmetric
// allreduce kernels); plans built before are dropped.
void Model::attach_comm(TpComm* c) {
  comm_ = c;
  plans_.clear();
  if (!c || x_sym_) return;
  const size_t bytes = static_cast<size_t>(cfg_.d_model) * 4;
  void* sym = c->alloc_symmetric(bytes);
  if (!sym) return;
  cuda_check(cudaMemcpy(sym, x_, bytes, cudaMemcpyDeviceToDevice), "x -> symmetric buffer");
  x_sym_ = static_cast<float*>(sym);
  x_ = x_sym_;
  arena_.allow(x_sym_, bytes);
}

// ---------------------------------------------------------------------------
// model

namespace {

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// prng.hpp:15-17, :33-35 (std::mt19937_64's sequence is fixed by the standard)
inline double uniform01(std::mt19937_64& eng) { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
inline float uniform_symmetric(std::mt19937_64& eng, float limit) {
  return static_cast<float>((2.0 * uniform01(eng) - 1.0) * limit);
}

}  // namespace

void* Model::arena_buf(size_t bytes, const char* what) {
  void* p = arena_.alloc(bytes);
  buffers_.insert(p);
  (void)what;
  return p;
}

// Declares every logical tensor in the reference draw order (model.hpp:47-51);
// the LLaMA arch drops pos_table and the betas and replaces w1/w2 by
// w_gate/w_up/w_down (same order as oracle.c:declare_tensors).
void Model::declare_tensors() {
  const int64_t d = cfg_.d_model, ff = cfg_.d_ff(), V = cfg_.vocab_size;
  const int wdt = cfg_.weight_dtype;
  auto add = [&](const std::string& name, int64_t rows, int64_t cols, int dtype, void* dev, MapDesc m) {
    LogicalTensor t;
    t.name = name;
    t.rows = rows;
    t.cols = cols;
    t.dtype = dtype;
    t.dev = dev;
    m.rows = rows;
    m.cols = cols;
    m.dst_dtype = dtype;
    m.head_dim = cfg_.head_dim();
    t.map = m;
    t.id = static_cast<uint32_t>(tensors_.size());
    tensors_.push_back(t);
  };
  auto mat = [&](int64_t ld, int64_t row_base, int stride, int offset, int rope) {
    MapDesc m;
    m.transpose = 1;
    m.ld = ld;
    m.row_base = row_base;
    m.row_stride = stride;
    m.row_offset = offset;
    m.rope_pair = rope;
    return m;
  };
  // tensor-parallel windows: column-parallel keeps outputs [r*w, (r+1)*w),
  // row-parallel keeps inputs [r*w, (r+1)*w) (ld = w)
  const int64_t r = cfg_.tp_rank;
  auto cols = [&](MapDesc m, int64_t w) {
    m.j0 = r * w;
    m.j1 = (r + 1) * w;
    return m;
  };
  auto rows = [&](MapDesc m, int64_t w) {
    m.p0 = r * w;
    m.p1 = (r + 1) * w;
    return m;
  };
  const int64_t dq = dq_, ffl = ffl_, Vl = vl_;
  MapDesc plain;
  add("embedding", V, d, wdt, emb_, plain);
  if (!cfg_.llama()) add("pos_table", cfg_.max_seq_len, d, wdt, pos_, plain);
  const int rope = cfg_.llama() ? 1 : 0;
  for (int l = 0; l < cfg_.n_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    LayerBuffers& L = layers_[l];
    add(p + "wq", d, d, wdt, L.w_qkv, cols(mat(d, 0, 1, 0, rope), dq));
    add(p + "wk", d, d, wdt, L.w_qkv, cols(mat(d, dq, 1, 0, rope), dq));
    add(p + "wv", d, d, wdt, L.w_qkv, cols(mat(d, 2 * dq, 1, 0, 0), dq));
    add(p + "wo", d, d, wdt, L.w_o, rows(mat(dq, 0, 1, 0, 0), dq));
    if (!cfg_.llama()) {
      add(p + "w1", d, ff, wdt, L.w_up, mat(d, 0, 1, 0, 0));
      add(p + "w2", ff, d, wdt, L.w_down, mat(ff, 0, 1, 0, 0));
      add(p + "ln1_gamma", 1, d, GRT_F32, L.ln1_g, plain);
      add(p + "ln1_beta", 1, d, GRT_F32, L.ln1_b, plain);
      add(p + "ln2_gamma", 1, d, GRT_F32, L.ln2_g, plain);
      add(p + "ln2_beta", 1, d, GRT_F32, L.ln2_b, plain);
    } else {
      add(p + "w_gate", d, ff, wdt, L.w_up, cols(mat(d, 0, 2, 0, 0), ffl));
      add(p + "w_up", d, ff, wdt, L.w_up, cols(mat(d, 0, 2, 1, 0), ffl));
      add(p + "w_down", ff, d, wdt, L.w_down, rows(mat(ffl, 0, 1, 0, 0), ffl));
      add(p + "ln1_gamma", 1, d, GRT_F32, L.ln1_g, plain);
      add(p + "ln2_gamma", 1, d, GRT_F32, L.ln2_g, plain);
    }
  }
  add("lnf_gamma", 1, d, GRT_F32, lnf_g_, plain);
  if (!cfg_.llama()) add("lnf_beta", 1, d, GRT_F32, lnf_b_, plain);
  add("head", d, V, wdt, head_, cols(mat(d, 0, 1, 0, 0), Vl));
}

Model::Model(const ModelConfig& cfg) : cfg_(cfg) {
  cfg_.validate();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    cudaGetLastError();
    raise(GRT_NoDevice, "no CUDA device visible");
  }
  if (cfg_.device < 0 || cfg_.device >= ndev) raise(GRT_InvalidConfig, "device ordinal out of range");
  cuda_check(cudaSetDevice(cfg_.device), "cudaSetDevice");
  cuda_check(gemv_prepare(cfg_.device), "gemv_prepare");
  cuda_check(attention_prepare(), "attention_prepare");
  cuda_check(prefill_gemm_prepare(), "prefill_gemm_prepare");
  cuda_check(gemv_pair_prepare(), "gemv_pair_prepare");

  const int64_t d = cfg_.d_model, ff = cfg_.d_ff(), V = cfg_.vocab_size, S = cfg_.max_seq_len;
  const int64_t h = cfg_.n_heads, dh = cfg_.head_dim();
  const size_t wb = cfg_.weight_dtype == GRT_BF16 ? 2 : 4;
  const size_t kvb = kv_elem_bytes();
  const int sms = num_sms(cfg_.device);
  max_nsplit_ = attention_nsplit(static_cast<int>(S), static_cast<int>(h), sms);
  max_gen_ = static_cast<int>(S);
  const int64_t up_rows = cfg_.llama() ? 2 * ff : ff;
  // this rank's shard (the whole model when tp_size == 1)
  const int64_t T = cfg_.tp_size;
  hl_ = static_cast<int>(h / T);
  dq_ = static_cast<int>(d / T);
  ffl_ = static_cast<int>(ff / T);
  vl_ = static_cast<int>(V / T);
  const int64_t dq = dq_, ffl = ffl_, Vl = vl_, hl = hl_;
  const int64_t upl = cfg_.llama() ? 2 * ffl : ffl;
  // KV cache per layer: contiguous [hl][S][dh], or a pool of ceil(S/page) pages [hl][page][dh]
  const int PS = cfg_.kv_page_size;
  kv_pages_ = PS > 0 ? (S + PS - 1) / PS : 0;
  kv_layer_elems_ = PS > 0 ? static_cast<size_t>(kv_pages_) * hl * PS * dh : static_cast<size_t>(hl) * S * dh;

  // size the arena: weights, KV, workspace, control
  size_t need = 0;
  auto acc = [&](size_t b) { need += round_up(b, 256) + 256; };
  acc(V * d * wb);
  if (!cfg_.llama()) acc(S * d * wb);
  for (int l = 0; l < cfg_.n_layers; ++l) {
    acc(3 * dq * d * wb);
    acc(d * dq * wb);
    acc(upl * d * wb);
    acc(d * ffl * wb);
    for (int i = 0; i < 4; ++i) acc(d * 4);
    acc(kv_layer_elems_ * kvb);
    acc(kv_layer_elems_ * kvb);
  }
  acc(static_cast<size_t>(std::max(kv_pages_, 1)) * 4);  // KV block table
  acc(d * 4);
  acc(d * 4);
  acc(Vl * d * wb);
  acc(Vl * 4);              // local logits (tp)
  acc(d * 4);               // x
  acc(d * 4);               // q
  acc(d * 4);               // attn
  acc(up_rows * 4);         // act
  acc(V * 4);               // logits
  acc(V * 4);               // sampler scratch
  acc(h * max_nsplit_ * (dh + 2) * 4);
  acc(h * 4);
  acc(cfg_.n_layers * 4 * 4);  // fused-pair barrier counters
  acc(S * (dh / 2) * 4 * 2);
  acc(sizeof(GrtCtrl));
  acc(sizeof(LoopCtl));
  acc(S * 4);
  acc(max_gen_ * 8);
  const bool pf = supports_batched_prefill();
  size_t pf_part = 0;
  if (pf) {
    const int64_t C = PREFILL_CHUNK;
    const int64_t kmax = std::max(d, ff);
    pf_part = std::max({prefill_gemm_part_floats(static_cast<int>(3 * dq), static_cast<int>(d), PREFILL_CHUNK, sms),
                        prefill_gemm_part_floats(static_cast<int>(d), static_cast<int>(dq), PREFILL_CHUNK, sms),
                        prefill_gemm_part_floats(static_cast<int>(upl), static_cast<int>(d), PREFILL_CHUNK, sms),
                        prefill_gemm_part_floats(static_cast<int>(d), static_cast<int>(ffl), PREFILL_CHUNK, sms)});
    acc(C * d * 4);          // X
    acc(C * d * 4);          // Q
    acc(C * kmax * 2);       // Xn (bf16)
    acc(C * d * 2);          // attention out (bf16)
    acc(C * ff * 2);         // SwiGLU act (bf16)
    acc(std::max<size_t>(pf_part, 1) * 4);
    acc(4096 * 4);           // split-K tile counters
  }
  arena_.reserve(need);

  layers_.resize(cfg_.n_layers);
  emb_ = arena_buf(V * d * wb, "embedding");
  if (!cfg_.llama()) pos_ = arena_buf(S * d * wb, "pos_table");
  for (int l = 0; l < cfg_.n_layers; ++l) {
    LayerBuffers& L = layers_[l];
    L.w_qkv = arena_buf(3 * dq * d * wb, "w_qkv");
    L.w_o = arena_buf(d * dq * wb, "w_o");
    L.w_up = arena_buf(upl * d * wb, "w_up");
    L.w_down = arena_buf(d * ffl * wb, "w_down");
    L.ln1_g = static_cast<float*>(arena_buf(d * 4, "ln1_g"));
    L.ln1_b = static_cast<float*>(arena_buf(d * 4, "ln1_b"));
    L.ln2_g = static_cast<float*>(arena_buf(d * 4, "ln2_g"));
    L.ln2_b = static_cast<float*>(arena_buf(d * 4, "ln2_b"));
    L.k = arena_buf(kv_layer_elems_ * kvb, "k");
    L.v = arena_buf(kv_layer_elems_ * kvb, "v");
  }
  lnf_g_ = static_cast<float*>(arena_buf(d * 4, "lnf_g"));
  lnf_b_ = static_cast<float*>(arena_buf(d * 4, "lnf_b"));
  head_ = arena_buf(Vl * d * wb, "head");
  x_ = static_cast<float*>(arena_buf(d * 4, "x"));
  q_ = static_cast<float*>(arena_buf(d * 4, "q"));
  attn_ = static_cast<float*>(arena_buf(d * 4, "attn"));
  act_ = static_cast<float*>(arena_buf(up_rows * 4, "act"));
  logits_ = static_cast<float*>(arena_buf(V * 4, "logits"));
  logits_local_ = T > 1 ? static_cast<float*>(arena_buf(Vl * 4, "logits_local")) : logits_;
  scratch_ = static_cast<float*>(arena_buf(V * 4, "scratch"));
  attn_part_ = static_cast<float*>(arena_buf(h * max_nsplit_ * (dh + 2) * 4, "attn_part"));
  attn_counters_ = static_cast<int*>(arena_buf(h * 4, "attn_counters"));
  pair_bar_ = static_cast<int*>(arena_buf(cfg_.n_layers * 4 * 4, "pair_barriers"));
  kv_table_ = static_cast<int*>(arena_buf(static_cast<size_t>(std::max(kv_pages_, 1)) * 4, "kv_block_table"));
  kvp_.page = PS;
  kvp_.n_heads = static_cast<int>(hl);
  kvp_.table = kv_table_;
  kv_table_host_.resize(std::max(kv_pages_, 1));
  for (int i = 0; i < static_cast<int>(kv_table_host_.size()); ++i) kv_table_host_[i] = PS > 0 ? i : 0;
  cuda_check(cudaMemcpy(kv_table_, kv_table_host_.data(), kv_table_host_.size() * 4, cudaMemcpyHostToDevice),
             "kv block table");
  if (pf) {
    const int64_t C = PREFILL_CHUNK;
    pf_X_ = static_cast<float*>(arena_buf(C * d * 4, "prefill_x"));
    pf_Q_ = static_cast<float*>(arena_buf(C * d * 4, "prefill_q"));
    pf_Xn_ = arena_buf(C * std::max(d, ff) * 2, "prefill_xn");
    pf_A_ = arena_buf(C * d * 2, "prefill_attn");
    pf_act_ = arena_buf(C * ff * 2, "prefill_act");
    pf_part_ = static_cast<float*>(arena_buf(std::max<size_t>(pf_part, 1) * 4, "prefill_splitk"));
    pf_cnt_ = static_cast<int*>(arena_buf(4096 * 4, "prefill_counters"));
  }

  rope_cos_ = static_cast<float*>(arena_buf(S * (dh / 2) * 4, "rope_cos"));
  rope_sin_ = static_cast<float*>(arena_buf(S * (dh / 2) * 4, "rope_sin"));
  ctrl_ = static_cast<GrtCtrl*>(arena_buf(sizeof(GrtCtrl), "ctrl"));
  loop_ctl_ = static_cast<LoopCtl*>(arena_buf(sizeof(LoopCtl), "loop_ctl"));
  tokens_ = static_cast<int*>(arena_buf((S + 1) * 4, "tokens"));  // +1: a token sampled at a full cache (pos == S)
  uniforms_ = static_cast<double*>(arena_buf(max_gen_ * 8, "uniforms"));

  (void)up_rows;
  weight_bytes_ = (V * d + (cfg_.llama() ? 0 : S * d) + Vl * d) * wb +
                  static_cast<uint64_t>(cfg_.n_layers) * ((3 * dq * d + d * dq + upl * d + d * ffl) * wb) +
                  static_cast<uint64_t>(cfg_.n_layers) * 4 * d * 4 + 2 * d * 4;

  declare_tensors();
  init_weights();

  // RoPE table: cos/sin of pos * theta^(-2i/dh) in double, rounded to fp32
  // (identical to oracle.c:oc_rope_table).
  {
    const int64_t half = dh / 2;
    std::vector<float> c(S * half), s(S * half);
    for (int64_t p = 0; p < S; ++p)
      for (int64_t i = 0; i < half; ++i) {
        const double inv_freq = std::pow(static_cast<double>(cfg_.rope_theta), -(2.0 * i) / static_cast<double>(dh));
        const double ang = static_cast<double>(p) * inv_freq;
        c[p * half + i] = static_cast<float>(std::cos(ang));
        s[p * half + i] = static_cast<float>(std::sin(ang));
      }
    cuda_check(cudaMemcpy(rope_cos_, c.data(), c.size() * 4, cudaMemcpyHostToDevice), "rope cos");
    cuda_check(cudaMemcpy(rope_sin_, s.data(), s.size() * 4, cudaMemcpyHostToDevice), "rope sin");
  }

  // host-mapped outputs: sampled tokens + timestamps (zero-copy, no per-step sync)
  void* ht = nullptr;
  void* hs = nullptr;
  cuda_check(cudaHostAlloc(&ht, max_gen_ * sizeof(int), cudaHostAllocMapped), "cudaHostAlloc tokens");
  cuda_check(cudaHostAlloc(&hs, 2 * max_gen_ * sizeof(unsigned long long), cudaHostAllocMapped), "cudaHostAlloc stamps");
  h_out_tokens_ = static_cast<volatile int*>(ht);
  h_out_stamps_ = static_cast<volatile unsigned long long*>(hs);

  // NVRTC: specialise the dynamic ops on this model's shape.
  std::vector<std::string> opts = {
      "-DGRT_D=" + std::to_string(d),
      "-DGRT_V=" + std::to_string(V),
      "-DGRT_MAXSEQ=" + std::to_string(S),
      std::string("-DGRT_WBF16=") + (cfg_.weight_dtype == GRT_BF16 ? "1" : "0"),
      std::string("-DGRT_ARCH_REF=") + (cfg_.llama() ? "0" : "1"),
  };
  jit_ = jit_get(opts, cfg_.device);
  f_pre_ = jit_->fn("grt_preprocess");
  f_sample_ = jit_->fn("grt_sample");
  f_sample_pre_ = jit_->fn("grt_sample_preprocess");
  cuda_check(cudaDeviceSynchronize(), "model init");
}

Model::~Model() {
  cudaSetDevice(cfg_.device);
  cudaDeviceSynchronize();
  if (x_sym_ && comm_) comm_->free_symmetric(x_sym_);  // the communicator outlives the model (c_api.cpp)
  if (h_out_tokens_) cudaFreeHost(const_cast<int*>(h_out_tokens_));
  if (h_out_stamps_) cudaFreeHost(const_cast<unsigned long long*>(h_out_stamps_));
}

// init_model (model.cpp:30-76): U[-0.1, 0.1] for every tensor.
void Model::init_weights() {
  if (cfg_.init == GRT_INIT_NONE) return;
  if (cfg_.init == GRT_INIT_PHILOX) {
    for (const LogicalTensor& t : tensors_)
      cuda_check(launch_map_init(t.map, t.dev, cfg_.seed, t.id, nullptr), "philox init");
    cuda_check(cudaDeviceSynchronize(), "philox init");
    return;
  }
  // mt19937_64 stream in draw order, generated on the host (serial by nature).
  std::mt19937_64 eng(cfg_.seed);
  size_t max_n = 0;
  for (const LogicalTensor& t : tensors_) max_n = std::max<size_t>(max_n, t.rows * t.cols);
  float* staging = nullptr;
  cuda_check(cudaMalloc(&staging, max_n * 4), "cudaMalloc staging");
  std::vector<float> buf;
  for (const LogicalTensor& t : tensors_) {
    const size_t n = t.rows * t.cols;
    buf.resize(n);
    for (size_t i = 0; i < n; ++i) buf[i] = uniform_symmetric(eng, 0.1f);
    cuda_check(cudaMemcpy(staging, buf.data(), n * 4, cudaMemcpyHostToDevice), "upload");
    cuda_check(launch_map_copy(t.map, t.dev, staging, static_cast<int>(Dt::F32), false, nullptr), "map copy");
  }
  cuda_check(cudaDeviceSynchronize(), "mt19937 init");
  cudaFree(staging);
}

const LogicalTensor& Model::tensor(const std::string& name) const {
  for (const LogicalTensor& t : tensors_)
    if (t.name == name) return t;
  raise(GRT_ShapeMismatch, "unknown tensor '" + name + "'");
}

void Model::set_kv_block_table(const int* table, int n) {
  if (kvp_.page == 0) raise(GRT_InvalidConfig, "set_kv_block_table: the KV cache is contiguous (kv_page_size 0)");
  if (n != kv_pages_) raise(GRT_ShapeMismatch, "set_kv_block_table: expected " + std::to_string(kv_pages_) + " entries");
  std::vector<char> seen(kv_pages_, 0);
  for (int i = 0; i < n; ++i) {
    if (table[i] < 0 || table[i] >= kv_pages_ || seen[table[i]])
      raise(GRT_InvalidConfig, "set_kv_block_table: entries must be distinct page ids in [0, n_pages)");
    seen[table[i]] = 1;
  }
  kv_table_host_.assign(table, table + n);
  cuda_check(cudaSetDevice(cfg_.device), "cudaSetDevice");
  cuda_check(cudaDeviceSynchronize(), "kv block table");  // no pass in flight reads the old table
  cuda_check(cudaMemcpy(kv_table_, table, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice), "kv block table");
}

int64_t Model::kv_row_host(int head, int pos) const {
  if (kvp_.page == 0) return static_cast<int64_t>(head) * cfg_.max_seq_len + pos;
  const int pi = pos / kvp_.page;
  return (static_cast<int64_t>(kv_table_host_[pi]) * kvp_.n_heads + head) * kvp_.page + (pos - pi * kvp_.page);
}

bool Model::has_tensor(const std::string& name) const {
  for (const LogicalTensor& t : tensors_)
    if (t.name == name) return true;
  return false;
}

void Model::upload(const std::string& name, const void* host, size_t bytes, int host_dtype, bool out_in) {
  const LogicalTensor& t = tensor(name);
  const size_t n = t.rows * t.cols;
  if (host_dtype != GRT_F32 && host_dtype != GRT_BF16 && host_dtype != GRT_F16)
    raise(GRT_InvalidConfig, "upload '" + name + "': unknown host dtype");
  const size_t eb = host_dtype == GRT_F32 ? 4 : 2;
  if (bytes != n * eb) raise(GRT_ShapeMismatch, "upload '" + name + "': byte count mismatch");
  cuda_check(cudaSetDevice(cfg_.device), "cudaSetDevice");
  void* staging = nullptr;
  cuda_check(cudaMalloc(&staging, bytes), "cudaMalloc staging");
  cuda_check(cudaMemcpy(staging, host, bytes, cudaMemcpyHostToDevice), "upload");
  cuda_check(launch_map_copy(t.map, t.dev, staging, host_dtype, out_in && t.rows > 1, nullptr), "map copy");
  cuda_check(cudaDeviceSynchronize(), "upload");
  cudaFree(staging);
}

void Model::download(const std::string& name, float* host, size_t numel) {
  const LogicalTensor& t = tensor(name);
  const size_t n = t.rows * t.cols;
  if (numel != n) raise(GRT_ShapeMismatch, "download '" + name + "': numel mismatch");
  cuda_check(cudaSetDevice(cfg_.device), "cudaSetDevice");
  float* staging = nullptr;
  cuda_check(cudaMalloc(&staging, n * 4), "cudaMalloc staging");
  cuda_check(cudaMemset(staging, 0, n * 4), "cudaMemset staging");  // outside this rank's shard: 0
  cuda_check(launch_map_read(t.map, t.dev, staging, nullptr), "map read");
  cuda_check(cudaMemcpy(host, staging, n * 4, cudaMemcpyDeviceToHost), "download");
  cudaFree(staging);
}

uint64_t Model::decode_bytes(int length) const {
  const uint64_t d = cfg_.d_model, L = cfg_.n_layers;
  const uint64_t wb = cfg_.weight_dtype == GRT_BF16 ? 2 : 4;
  const uint64_t kvb = kv_elem_bytes();
  // weights streamed once (minus the embedding/pos tables: one row each)
  const uint64_t V = cfg_.vocab_size;
  uint64_t b = weight_bytes_ - (V * d + (cfg_.llama() ? 0 : cfg_.max_seq_len * d)) * wb;
  b += d * wb * (cfg_.llama() ? 1 : 2);            // embedding (+pos) row
  const uint64_t dq = static_cast<uint64_t>(dq_);  // this rank's heads
  b += L * 2 * static_cast<uint64_t>(length) * dq * kvb;  // K,V read over [0, length)
  b += L * 2 * dq * kvb;                                   // K,V row write
  return b;
}

// ---------------------------------------------------------------------------
// batched prefill

// Both architectures: LLaMA (RMSNorm, RoPE, SwiGLU) and the reference's own
// (LayerNorm with beta, learned position table, ReLU MLP); bf16 weights (the
// tcgen05 GEMM operands are the stored weights).
bool Model::supports_batched_prefill() const {
  const int dh = cfg_.head_dim();
  return cfg_.weight_dtype == GRT_BF16 && cfg_.d_model % 8 == 0 && cfg_.d_ff() % 8 == 0 &&
         (dh == 16 || dh == 32 || dh == 64 || dh == 128);
}

void Model::prefill_batched(int p, cudaStream_t s, bool fuse_norm) {
  if (!supports_batched_prefill()) raise(GRT_Unsupported, "batched prefill needs bf16 weights");
  if (p < 1 || p > cfg_.max_seq_len) raise(GRT_PromptTooLong, "batched prefill length out of range");
  const int d = cfg_.d_model, dh = cfg_.head_dim(), S = cfg_.max_seq_len;
  const int T = cfg_.tp_size, dq = dq_, ffl = ffl_, hl = hl_;  // this rank's shard
  if (T > 1 && !comm_) raise(GRT_InvalidConfig, "tensor-parallel prefill needs an attached communicator");
  const int resid_epi = (T == 1 || cfg_.tp_rank == 0) ? PG_EPI_RESID : PG_EPI_STORE;
  const Dt kvdt = cfg_.kv_dtype == GRT_BF16 ? Dt::BF16 : Dt::F32;
  const float scale = 1.0f / std::sqrt(static_cast<float>(dh));  // model.cpp:119
  const bool llama = cfg_.llama();
  int last_P = 0;
  for (int start = 0; start < p; start += PREFILL_CHUNK) {
    const int P = std::min(PREFILL_CHUNK, p - start);
    last_P = P;
    cuda_check(launch_prefill_embed(Dt::BF16, tokens_, start, P, emb_, llama ? nullptr : pos_, d, pf_X_,
                                    cfg_.vocab_size, &ctrl_->err, s),
               "prefill embed");
    // Single GPU: a residual GEMM that splits K leaves its partials to the next
    // RMSNorm launch (reduce + residual + norm in one kernel, bit-identical).
    const bool fuse_rn = !comm_ && fuse_norm && llama;
    auto norm = [&](const float* g, const float* b, const char* what) {
      if (llama)
        cuda_check(launch_prefill_rmsnorm(pf_X_, P, g, cfg_.norm_eps, d, pf_Xn_, s), what);
      else
        cuda_check(launch_prefill_layernorm(pf_X_, P, g, b, cfg_.norm_eps, d, pf_Xn_, s), what);
    };
    PrefillGemmParams prev_down;  // previous layer's down GEMM, if its reduce was deferred
    for (int l = 0; l < cfg_.n_layers; ++l) {
      const LayerBuffers& L = layers_[l];
      if (prev_down.defer_reduce && prev_down.ksplit > 1)
        cuda_check(launch_prefill_resid_norm(prev_down, L.ln1_g, cfg_.norm_eps, pf_Xn_, s), "prefill resid+rmsnorm1");
      else
        norm(L.ln1_g, L.ln1_b, "prefill norm1");
      PrefillGemmParams q;
      q.M = 3 * dq;
      q.K = d;
      q.P = P;
      q.epi = llama ? PG_EPI_QKV_ROPE : PG_EPI_QKV;
      q.q_out = pf_Q_;
      q.k_cache = L.k;
      q.kvp = kvp_;
      q.v_cache = L.v;
      q.rope_cos = rope_cos_;
      q.rope_sin = rope_sin_;
      q.head_dim = dh;
      q.max_seq = S;
      q.d_model = dq;
      q.start_pos = start;
      q.kv_bf16 = kvdt == Dt::BF16;
      q.part = pf_part_;
      q.counters = pf_cnt_;
      cuda_check(launch_prefill_gemm(L.w_qkv, pf_Xn_, q, s, true), "prefill qkv");
      cuda_check(launch_prefill_attention(kvdt, pf_Q_, L.k, L.v, start, P, dq, hl, dh, S, scale, pf_A_, s, kvp_),
                 "prefill attention");
      PrefillGemmParams o;
      o.M = d;
      o.K = dq;
      o.P = P;
      o.epi = resid_epi;
      o.out = pf_X_;
      o.part = pf_part_;
      o.counters = pf_cnt_;
      o.defer_reduce = fuse_rn ? 1 : 0;
      cuda_check(launch_prefill_gemm_ex(L.w_o, pf_A_, &o, s, true), "prefill wo");
      if (comm_) cuda_check(comm_->allreduce_sum(pf_X_, static_cast<size_t>(P) * d, s), "prefill allreduce wo");
      if (o.defer_reduce && o.ksplit > 1)
        cuda_check(launch_prefill_resid_norm(o, L.ln2_g, cfg_.norm_eps, pf_Xn_, s), "prefill resid+rmsnorm2");
      else
        norm(L.ln2_g, L.ln2_b, "prefill norm2");
      PrefillGemmParams u;  // gate/up + SwiGLU (LLaMA) | W1 + ReLU (reference arch)
      u.M = llama ? 2 * ffl : ffl;
      u.K = d;
      u.P = P;
      u.epi = llama ? PG_EPI_SWIGLU : PG_EPI_RELU;
      u.out_bf16 = pf_act_;
      u.part = pf_part_;
      u.counters = pf_cnt_;
      cuda_check(launch_prefill_gemm(L.w_up, pf_Xn_, u, s, true), "prefill gate_up");
      PrefillGemmParams w2;
      w2.M = d;
      w2.K = ffl;
      w2.P = P;
      w2.epi = resid_epi;
      w2.out = pf_X_;
      w2.part = pf_part_;
      w2.counters = pf_cnt_;
      w2.defer_reduce = fuse_rn && l + 1 < cfg_.n_layers ? 1 : 0;  // the last layer's output goes to the hand-off
      cuda_check(launch_prefill_gemm_ex(L.w_down, pf_act_, &w2, s, true), "prefill down");
      prev_down = w2;
      if (comm_) cuda_check(comm_->allreduce_sum(pf_X_, static_cast<size_t>(P) * d, s), "prefill allreduce down");
    }
  }
  // hand off to the decode state: last token's residual row, seq_len = p; then
  // ln_f + LM head for that row only (the only logits the sampler consumes)
  cuda_check(launch_prefill_handoff(pf_X_ + static_cast<int64_t>(last_P - 1) * d, d, x_, &ctrl_->seq_len, p, s),
             "prefill handoff");
  GemvParams hp;
  hp.w = head_;
  hp.n_rows = vl_;
  hp.k = d;
  hp.x = x_;
  hp.gamma = lnf_g_;
  hp.beta = lnf_b_;
  hp.eps = cfg_.norm_eps;
  hp.out = logits_local_;
  cuda_check(launch_gemv(Dt::BF16, llama ? NORM_RMS : NORM_LN, EPI_STORE, hp, s, false, 0), "prefill head");
  if (comm_) cuda_check(comm_->allgather(logits_local_, logits_, static_cast<size_t>(vl_), s), "prefill allgather");
}

// ---------------------------------------------------------------------------
// plans

void Model::attention_split(int key, int B, int* nsplit, int* span_cap) const {
  const int max_len = std::min(key * B, cfg_.max_seq_len);
  const int ns = std::min(max_nsplit_, attention_nsplit(max_len, cfg_.n_heads, num_sms(cfg_.device)));
  *nsplit = ns;
  *span_cap = ((max_len + ns - 1) / ns + 3) / 4 * 4;
}

std::vector<uint64_t> Model::trace_pass(int key, int B, cudaStream_t s, int* grid, int* stride, int impl) {
  if (impl == 1) {
    const int n_k = 5 * cfg_.n_layers + 1;
    const size_t n = static_cast<size_t>(n_k) * OP_TRACE_CTAS * 8;
    unsigned long long* buf = nullptr;
    cuda_check(cudaMalloc(&buf, n * 8), "cudaMalloc trace");
    op_trace_ = buf;
    std::vector<KernelInvocation> plan;
    try {
      plan = build_plan(key, B, 1);
    } catch (...) {
      op_trace_ = nullptr;
      cudaFree(buf);
      throw;
    }
    op_trace_ = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "trace capture");
    for (const KernelInvocation& inv : plan) cuda_check(inv.launch(s), inv.spec.name.c_str());
    cuda_check(cudaStreamEndCapture(s, &g), "trace capture");
    cuda_check(cudaGraphInstantiate(&ge, g, 0), "trace instantiate");
    cuda_check(cudaGraphLaunch(ge, s), "trace launch");  // warm
    cuda_check(cudaMemsetAsync(buf, 0, n * 8, s), "memset trace");
    cuda_check(cudaGraphLaunch(ge, s), "trace launch");
    cuda_check(cudaStreamSynchronize(s), "trace");
    std::vector<uint64_t> out(n);
    cuda_check(cudaMemcpy(out.data(), buf, n * 8, cudaMemcpyDeviceToHost), "trace copy");
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(buf);
    *grid = n_k;
    *stride = OP_TRACE_CTAS * 8;
    return out;
  }
  raise(GRT_InvalidConfig, "trace_pass: only the per-op plan (pass_impl 1) is traced");
}

// The fused pair launch (gemv_pair.cu) covers Wo + gate/up only.  Measured and
// rejected: down + next QKV as a pair (the down GEMV's 44 KB
// activation row leaves two ring stages), decode attention as phase 0 of the
// pair launch (an extra grid barrier + partial merge cost more than the kernel
// boundary they remove), and a persistent whole-pass kernel.
std::vector<KernelInvocation> Model::build_plan(int key, int B, int impl) {
  const int d = cfg_.d_model, ff = cfg_.d_ff(), V = cfg_.vocab_size, S = cfg_.max_seq_len;
  const int h = cfg_.n_heads, dh = cfg_.head_dim();
  const Dt wdt = cfg_.weight_dtype == GRT_BF16 ? Dt::BF16 : Dt::F32;
  const Dt kvdt = cfg_.kv_dtype == GRT_BF16 ? Dt::BF16 : Dt::F32;
  const size_t wb = wdt == Dt::BF16 ? 2 : 4;
  const size_t kvb = kv_elem_bytes();
  const int max_len = std::min(key * B, S);
  int nsplit = 1, span_cap = 4;
  attention_split(key, B, &nsplit, &span_cap);
  const bool llama = cfg_.llama();
  const int norm = llama ? NORM_RMS : NORM_LN;
  int* seq_len = &ctrl_->seq_len;
  int* err = &ctrl_->err;

  std::vector<KernelInvocation> plan;
  auto next_trace = [&]() -> unsigned long long* {
    return op_trace_ ? op_trace_ + plan.size() * OP_TRACE_CTAS * 8 : nullptr;
  };
  auto emit_gemv = [&](const std::string& name, int epi, int nrm, GemvParams p, size_t w_bytes) {
    p.trace = next_trace();
    KernelInvocation inv;
    inv.spec.name = name;
    inv.spec.op_class = OpClass::Static;
    inv.spec.flops = 2LL * p.n_rows * p.k;
    inv.spec.bytes = static_cast<int64_t>(w_bytes);
    inv.bindings = {{p.w, w_bytes}, {p.x, static_cast<size_t>(p.k) * 4}};
    if (p.out) inv.bindings.push_back({p.out, 4});
    inv.launch = [wdt, epi, nrm, p](cudaStream_t s) { return launch_gemv(wdt, nrm, epi, p, s, true, 0); };
    plan.push_back(std::move(inv));
  };
  // A residual GEMV (Wo, down) is held back and, when the next GEMV is the
  // RMS-normed one that consumes its output (gate/up, next layer's QKV, LM
  // head), both run as ONE launch with a grid barrier (gemv_pair.cu): the
  // weight ring streams across the boundary.  Single GPU, LLaMA, bf16 only.
  struct Pending {
    std::string name;
    GemvParams p;
    size_t bytes = 0;
    bool set = false;
  } pending;
  // collectives: every tensor-parallel plan, and a 1-rank group with a communicator
  const bool coll = comm_ != nullptr || cfg_.tp_size > 1;
  const bool fuse = !coll && llama && wdt == Dt::BF16 && !op_trace_;
  int n_pairs_emitted = 0;
  auto flush = [&]() {
    if (pending.set) emit_gemv(pending.name, EPI_RESID, NORM_NONE, pending.p, pending.bytes);
    pending.set = false;
  };
  auto gemv = [&](const char* name, int epi, int nrm, GemvParams p, size_t w_bytes) {
    if (fuse && epi == EPI_RESID && nrm == NORM_NONE) {
      flush();
      pending = Pending{name, p, w_bytes, true};
      return;
    }
    if (fuse && pending.set && nrm == NORM_RMS && epi == EPI_SWIGLU) {
      GemvPairParams pp;  // Wo + gate/up (k = 4096 both): 2048-element chunks (8 KB stages)
      pp.a = pending.p;
      pp.b = p;
      pp.bar = pair_bar_ + 2 * n_pairs_emitted++;
      pp.err = err;
      KernelInvocation inv;
      inv.spec.name = pending.name + "+" + name;
      inv.spec.op_class = OpClass::Static;
      inv.spec.flops = 2LL * pending.p.n_rows * pending.p.k + 2LL * p.n_rows * p.k;
      inv.spec.bytes = static_cast<int64_t>(pending.bytes + w_bytes);
      inv.bindings = {{pending.p.w, pending.bytes}, {p.w, w_bytes}, {pp.bar, 8},
                      {pending.p.x, static_cast<size_t>(pending.p.k) * 4}, {p.x, static_cast<size_t>(p.k) * 4}};
      inv.launch = [epi, pp](cudaStream_t s) { return launch_gemv_pair(epi, pp, s, true); };
      plan.push_back(std::move(inv));
      pending.set = false;
      return;
    }
    flush();
    emit_gemv(name, epi, nrm, p, w_bytes);
  };
  // Tensor parallelism: this rank's shard has hl heads (dq = hl*dh
  // attention dims), ffl d_ff columns and vl vocab rows.  Row-parallel Wo/down
  // produce partial residual updates: rank 0 adds its partial to x, the other
  // ranks overwrite x with theirs, and an in-place allreduce (sum) leaves
  // x + sum_r partial_r on every rank.  The LM head is vocab-parallel; an
  // allgather assembles the full logits (rank order) for the sampler.
  const int T = cfg_.tp_size, hl = hl_, dq = dq_, ffl = ffl_, vl = vl_;
  const int resid_epi = (T == 1 || cfg_.tp_rank == 0) ? EPI_RESID : EPI_STORE;
  TpComm** commp = &comm_;
  auto allreduce_x = [&](const char* name) {
    flush();
    KernelInvocation inv;
    inv.spec.name = name;
    inv.spec.op_class = OpClass::Static;
    inv.spec.bytes = static_cast<int64_t>(d) * 4;
    inv.bindings = {{x_, static_cast<size_t>(d) * 4}};
    inv.collective = COLL_ALLREDUCE;
    inv.coll_in = x_;
    inv.coll_out = x_;
    inv.coll_n = static_cast<size_t>(d);
    float* x = x_;
    inv.launch = [commp, x, d](cudaStream_t s) {
      if (!*commp) return cudaErrorInvalidValue;  // no communicator attached
      return (*commp)->allreduce_sum(x, static_cast<size_t>(d), s);
    };
    plan.push_back(std::move(inv));
  };
  for (int l = 0; l < cfg_.n_layers; ++l) {
    const LayerBuffers& L = layers_[l];
    {  // ln1 + q,k,v + (RoPE) + kv_write   (column-parallel: this rank's heads)
      GemvParams p;
      p.w = L.w_qkv;
      p.n_rows = 3 * dq;
      p.k = d;
      p.x = x_;
      p.gamma = L.ln1_g;
      p.beta = L.ln1_b;
      p.eps = cfg_.norm_eps;
      p.q_out = q_;
      p.k_cache = L.k;
      p.v_cache = L.v;
      p.seq_len = seq_len;
      p.rope_cos = rope_cos_;
      p.rope_sin = rope_sin_;
      p.n_heads = hl;
      p.head_dim = dh;
      p.max_seq = S;
      p.d_model = dq;  // q | k | v sections of the shard are dq rows each
      p.kv_bf16 = kvdt == Dt::BF16;
      p.kvp = kvp_;
      p.err = err;
      gemv("qkv", llama ? EPI_QKV_ROPE : EPI_QKV, norm, p, 3ull * dq * d * wb);
    }
    flush();
    {  // attention over [0, seq_len) for this rank's heads
      AttnParams a;
      a.q = q_;
      a.k_cache = L.k;
      a.v_cache = L.v;
      a.out = attn_;
      a.part = attn_part_;
      a.counters = attn_counters_;
      a.seq_len = seq_len;
      a.n_heads = hl;
      a.head_dim = dh;
      a.max_seq = S;
      a.span_cap = span_cap;
      a.scale = 1.0f / std::sqrt(static_cast<float>(dh));  // model.cpp:119
      a.err = err;
      a.kvp = kvp_;
      a.trace = next_trace();
      KernelInvocation inv;
      inv.spec.name = "attention";
      inv.spec.flops = static_cast<int64_t>(hl) * max_len * (4 * dh + 5);  // kernels.hpp:51
      inv.spec.bytes = 2LL * max_len * dq * kvb;
      inv.bindings = {{L.k, kv_layer_elems_ * kvb}, {L.v, kv_layer_elems_ * kvb},
                      {q_, static_cast<size_t>(dq) * 4}, {attn_, static_cast<size_t>(dq) * 4}};
      inv.launch = [kvdt, a, max_len](cudaStream_t s) { return launch_attention(kvdt, a, max_len, s, true); };
      plan.push_back(std::move(inv));
    }
    {  // wo + residual (row-parallel under TP)
      GemvParams p;
      p.w = L.w_o;
      p.n_rows = d;
      p.k = dq;
      p.x = attn_;
      p.out = x_;
      gemv("wo_residual", resid_epi, NORM_NONE, p, 1ull * d * dq * wb);
      if (coll) allreduce_x("allreduce_wo");
    }
    {  // ln2 + w1 + relu  |  rms + gate/up + SwiGLU   (column-parallel)
      GemvParams p;
      p.w = L.w_up;
      p.n_rows = llama ? 2 * ffl : ffl;
      p.k = d;
      p.x = x_;
      p.gamma = L.ln2_g;
      p.beta = L.ln2_b;
      p.eps = cfg_.norm_eps;
      p.out = act_;
      gemv(llama ? "gate_up_swiglu" : "w1_relu", llama ? EPI_SWIGLU : EPI_RELU, norm, p,
           static_cast<size_t>(p.n_rows) * d * wb);
    }
    {  // w2/down + residual (row-parallel)
      GemvParams p;
      p.w = L.w_down;
      p.n_rows = d;
      p.k = ffl;
      p.x = act_;
      p.out = x_;
      p.chmax = 3072;  // k = 11008 in 4 chunks of 2752 (11 KB stages): measured fastest
      gemv("down_residual", resid_epi, NORM_NONE, p, 1ull * d * ffl * wb);
      if (coll) allreduce_x("allreduce_down");
    }
  }
  {  // ln_f + head (vocab-parallel)
    GemvParams p;
    p.w = head_;
    p.n_rows = vl;
    p.k = d;
    p.x = x_;
    p.gamma = lnf_g_;
    p.beta = lnf_b_;
    p.eps = cfg_.norm_eps;
    p.out = logits_local_;
    gemv("lnf_head", EPI_STORE, norm, p, 1ull * vl * d * wb);
  }
  flush();
  if (coll) {
    KernelInvocation inv;
    inv.spec.name = "allgather_logits";
    inv.spec.op_class = OpClass::Static;
    inv.spec.bytes = static_cast<int64_t>(V) * 4;
    inv.bindings = {{logits_local_, static_cast<size_t>(vl) * 4}, {logits_, static_cast<size_t>(V) * 4}};
    inv.collective = COLL_ALLGATHER;
    inv.coll_in = logits_local_;
    inv.coll_out = logits_;
    inv.coll_n = static_cast<size_t>(vl);
    float* in = logits_local_;
    float* out = logits_;
    inv.launch = [commp, in, out, vl](cudaStream_t s) {
      if (!*commp) return cudaErrorInvalidValue;
      return (*commp)->allgather(in, out, static_cast<size_t>(vl), s);
    };
    plan.push_back(std::move(inv));
  }
  (void)ff;
  return plan;
}

const std::vector<KernelInvocation>& Model::plan(int key, int B, int impl) {
  if (B < 1) raise(GRT_InvalidConfig, "bucket_size must be >= 1");
  // pass_impl 0 (one persistent kernel for the whole pass) was measured slower
  // than the per-op graph and removed
  if (impl != 1) raise(GRT_Unsupported, "pass_impl must be 1 (the per-op kernel graph)");
  if (key < 1 || key > max_key(B))
    raise(GRT_LengthOutOfRange, "plan key " + std::to_string(key) + " outside [1, " + std::to_string(max_key(B)) + "]");
  std::lock_guard<std::mutex> lk(plan_mu_);
  const auto mk = std::make_pair(key, B * 4 + impl);
  auto it = plans_.find(mk);
  if (it == plans_.end()) it = plans_.emplace(mk, build_plan(key, B, impl)).first;
  return it->second;
}

KernelInvocation Model::make_preprocess_op() {
  KernelInvocation inv;
  inv.spec.name = "extend_position+slot_append";
  inv.spec.op_class = OpClass::Dynamic;
  inv.spec.flops = 2LL * cfg_.d_model;
  const size_t wb = cfg_.weight_dtype == GRT_BF16 ? 2 : 4;
  inv.spec.bytes = static_cast<int64_t>(cfg_.d_model) * (wb * (cfg_.llama() ? 1 : 2) + 4);
  inv.bindings = {{ctrl_, sizeof(GrtCtrl)}, {x_, static_cast<size_t>(cfg_.d_model) * 4}};
  CUfunction f = f_pre_;
  GrtCtrl* ctrl = ctrl_;
  const void* emb = emb_;
  const void* pos = pos_ ? pos_ : emb_;
  float* x = x_;
  const int threads = std::min(1024, (cfg_.d_model + 31) / 32 * 32);
  inv.launch = [f, ctrl, emb, pos, x, threads](cudaStream_t s) {
    GrtCtrl* a0 = ctrl;
    const void* a1 = emb;
    const void* a2 = pos;
    float* a3 = x;
    void* args[] = {&a0, &a1, &a2, &a3};
    return launch_jit(f, dim3(1), dim3(threads), args, s, true);
  };
  return inv;
}

KernelInvocation Model::make_sample_preprocess_op() {
  KernelInvocation inv;
  inv.spec.name = "sample_token+extend_position";
  inv.spec.op_class = OpClass::Dynamic;
  inv.spec.flops = cfg_.vocab_size + 2LL * cfg_.d_model;
  inv.spec.bytes = static_cast<int64_t>(cfg_.vocab_size) * 4 + static_cast<int64_t>(cfg_.d_model) * 6;
  inv.bindings = {{ctrl_, sizeof(GrtCtrl)},
                  {logits_, static_cast<size_t>(cfg_.vocab_size) * 4},
                  {x_, static_cast<size_t>(cfg_.d_model) * 4}};
  CUfunction f = f_sample_pre_;
  GrtCtrl* ctrl = ctrl_;
  const float* logits = logits_;
  const void* emb = emb_;
  const void* pos = pos_ ? pos_ : emb_;
  float* x = x_;
  inv.launch = [f, ctrl, logits, emb, pos, x](cudaStream_t s) {
    GrtCtrl* a0 = ctrl;
    const float* a1 = logits;
    const void* a2 = emb;
    const void* a3 = pos;
    float* a4 = x;
    void* args[] = {&a0, &a1, &a2, &a3, &a4};
    return launch_jit(f, dim3(1), dim3(1024), args, s, true);
  };
  return inv;
}

KernelInvocation Model::make_sample_op() {
  KernelInvocation inv;
  inv.spec.name = "sample_token";
  inv.spec.op_class = OpClass::Dynamic;
  inv.spec.flops = cfg_.vocab_size;
  inv.spec.bytes = static_cast<int64_t>(cfg_.vocab_size) * 4;
  inv.bindings = {{ctrl_, sizeof(GrtCtrl)}, {logits_, static_cast<size_t>(cfg_.vocab_size) * 4}};
  CUfunction f = f_sample_;
  GrtCtrl* ctrl = ctrl_;
  const float* logits = logits_;
  inv.launch = [f, ctrl, logits](cudaStream_t s) {
    GrtCtrl* a0 = ctrl;
    const float* a1 = logits;
    void* args[] = {&a0, &a1};
    return launch_jit(f, dim3(1), dim3(1024), args, s, true);
  };
  return inv;
}

}  // namespace grt
