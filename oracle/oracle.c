/*
 * oracle.c -- CPU restatement of the reference graphrt decode path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -ffp-contract=off so
 * every multiply and add rounds separately, exactly like the reference build
 * (x86-64 baseline, no FMA).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* mt19937_64 (std::mt19937_64, parameters fixed by the C++ standard).        */
/* prng.hpp:9-13 relies on the standard-pinned output sequence.               */

#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void oc_mt64_seed(oc_mt64* e, uint64_t seed) {
  e->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    e->mt[i] = 6364136223846793005ULL * (e->mt[i - 1] ^ (e->mt[i - 1] >> 62)) + (uint64_t)i;
  e->mti = MT_NN;
}

uint64_t oc_mt64_next(oc_mt64* e) {
  static const uint64_t mag01[2] = {0ULL, MT_MATRIX_A};
  uint64_t x;
  if (e->mti >= MT_NN) {
    int i;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (e->mt[i] & MT_UM) | (e->mt[i + 1] & MT_LM);
      e->mt[i] = e->mt[i + MT_MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < MT_NN - 1; ++i) {
      x = (e->mt[i] & MT_UM) | (e->mt[i + 1] & MT_LM);
      e->mt[i] = e->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (e->mt[MT_NN - 1] & MT_UM) | (e->mt[0] & MT_LM);
    e->mt[MT_NN - 1] = e->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    e->mti = 0;
  }
  x = e->mt[e->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* prng.hpp:15-17 */
double oc_uniform01(oc_mt64* e) { return (double)(oc_mt64_next(e) >> 11) * 0x1.0p-53; }

/* prng.hpp:33-35: static_cast<float>((2.0 * uniform01(eng) - 1.0) * limit) */
float oc_uniform_symmetric(oc_mt64* e, float limit) {
  return (float)((2.0 * oc_uniform01(e) - 1.0) * (double)limit);
}

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon et al. 2011).  Counter-based: value(seed, id, index). */

static inline void philox_mulhilo(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

void oc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    philox_mulhilo(0xD2511F53u, c0, &hi0, &lo0);
    philox_mulhilo(0xCD9E8D57u, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* Weight init, counter-based variant.  Counter = (index lo, index hi, tensor id,
 * 'grtI'), key = seed.  53 random bits -> the same (2u-1)*limit map as
 * uniform_symmetric (prng.hpp:33-35). */
float oc_philox_weight(uint64_t seed, uint32_t tensor_id, uint64_t index, float limit) {
  uint32_t ctr[4] = {(uint32_t)index, (uint32_t)(index >> 32), tensor_id, 0x67724954u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  oc_philox4x32_10(ctr, key, o);
  uint64_t bits = (((uint64_t)o[1] << 32) | (uint64_t)o[0]) >> 11;
  double u = (double)bits * 0x1.0p-53;
  return (float)((2.0 * u - 1.0) * (double)limit);
}

/* ------------------------------------------------------------------------- */
/* bf16 + shared sampler math                                                 */

uint16_t oc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return (uint16_t)((u >> 16) | 0x40u);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb; /* round to nearest even */
  return (uint16_t)(u >> 16);
}

float oc_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

float oc_round_bf16(float f) { return oc_bf16_to_f32(oc_f32_to_bf16(f)); }

/* Deterministic exp for z <= 0, identical on host and device: Cody-Waite range
 * reduction + degree-6 polynomial, every step an explicit fmaf or a single
 * rounded op (device twin: csrc/jit/sampler_math.cuh). */
float oc_grt_expf(float z) {
  if (!(z > -30.0f)) return 0.0f; /* e^-30 < 2^-43: below the 2^-31 weight quantum */
  if (z > 0.0f) z = 0.0f;
  float n = rintf(z * 1.44269504088896341f);
  float r = fmaf(n, -0.693145751953125f, z);
  r = fmaf(n, -1.428606765330187e-06f, r);
  float p = 1.3981999507e-3f;
  p = fmaf(p, r, 8.3334519073e-3f);
  p = fmaf(p, r, 4.1665795894e-2f);
  p = fmaf(p, r, 1.6666665459e-1f);
  p = fmaf(p, r, 5.0000001201e-1f);
  float r2 = r * r;
  float y = fmaf(p, r2, r);
  y = y + 1.0f;
  return ldexpf(y, (int)n);
}

/* ------------------------------------------------------------------------- */
/* Model                                                                      */

typedef struct oc_tensor {
  char name[48];
  int64_t rows, cols; /* reference layout: matrices [k, n]; vectors rows=1 */
  int dtype;          /* storage dtype */
  float* f;           /* when dtype == OC_F32 */
  uint16_t* h;        /* when dtype == OC_BF16 */
} oc_tensor;

typedef struct oc_layer {
  oc_tensor *ln1_g, *ln1_b, *wq, *wk, *wv, *wo, *ln2_g, *ln2_b, *w1, *w2;
  oc_tensor *wg, *wu, *wd; /* llama */
} oc_layer;

struct oc_model {
  oc_config cfg;
  int d_ff, head_dim;
  int n_tensors;
  oc_tensor* tensors;
  oc_tensor *embedding, *pos_table, *lnf_g, *lnf_b, *head;
  oc_layer* layers;
  float* kv; /* [L][2][max_seq][h*dh] (reference per-layer layout [max_seq,h,dh]) */
  int cur_len;
  /* workspace (model.cpp:83-93) */
  float *x, *ln_out, *q, *k, *v, *attn_out, *o, *mlp, *up, *logits, *probs;
  float *rope_cos, *rope_sin;
};

void oc_config_default(oc_config* c) {
  memset(c, 0, sizeof(*c));
  c->arch = OC_ARCH_REF;
  c->n_layers = 4;
  c->d_model = 64;
  c->n_heads = 4;
  c->vocab_size = 256;
  c->max_seq_len = 600;
  c->d_ff = 0;
  c->norm_eps = 1e-5f;
  c->seed = 1234;
  c->init = OC_INIT_MT19937;
  c->weight_dtype = OC_F32;
  c->kv_dtype = OC_F32;
  c->rope_theta = 10000.0f;
  c->n_threads = 1;
}

/* ModelConfig::validate (model.cpp:10-18) */
int oc_config_validate(const oc_config* c) {
  if (c->n_layers < 1 || c->d_model < 1 || c->n_heads < 1) return OC_InvalidConfig;
  if (c->d_model % c->n_heads != 0) return OC_InvalidConfig;
  if (c->vocab_size < 1 || c->max_seq_len < 1) return OC_InvalidConfig;
  if (!(c->norm_eps > 0.0f)) return OC_InvalidConfig;
  if (c->d_ff < 0) return OC_InvalidConfig;
  if (c->arch != OC_ARCH_REF && c->arch != OC_ARCH_LLAMA) return OC_InvalidConfig;
  if (c->arch == OC_ARCH_LLAMA && ((c->d_model / c->n_heads) % 2) != 0) return OC_InvalidConfig;
  return OC_OK;
}

static oc_tensor* add_tensor(oc_model* m, const char* name, int64_t rows, int64_t cols, int dtype) {
  oc_tensor* t = &m->tensors[m->n_tensors++];
  snprintf(t->name, sizeof(t->name), "%s", name);
  t->rows = rows;
  t->cols = cols;
  t->dtype = dtype;
  size_t n = (size_t)(rows * cols);
  if (dtype == OC_F32)
    t->f = (float*)calloc(n, sizeof(float));
  else
    t->h = (uint16_t*)calloc(n, sizeof(uint16_t));
  return t;
}

static inline float tget(const oc_tensor* t, int64_t i) {
  return t->dtype == OC_F32 ? t->f[i] : oc_bf16_to_f32(t->h[i]);
}

static inline void tset(oc_tensor* t, int64_t i, float v) {
  if (t->dtype == OC_F32)
    t->f[i] = v;
  else
    t->h[i] = oc_f32_to_bf16(v);
}

/* Declares every tensor in the reference draw order (model.hpp:47-51); the
 * LLaMA arch replaces pos_table/beta/w1/w2 by nothing/nothing/w_gate,w_up,w_down. */
static void declare_tensors(oc_model* m) {
  const oc_config* c = &m->cfg;
  const int64_t d = c->d_model, ff = m->d_ff, V = c->vocab_size;
  const int wdt = c->weight_dtype;
  char nm[48];
  m->tensors = (oc_tensor*)calloc((size_t)(16 * c->n_layers + 8), sizeof(oc_tensor));
  m->layers = (oc_layer*)calloc((size_t)c->n_layers, sizeof(oc_layer));
  m->embedding = add_tensor(m, "embedding", V, d, wdt);
  if (c->arch == OC_ARCH_REF) m->pos_table = add_tensor(m, "pos_table", c->max_seq_len, d, wdt);
  for (int l = 0; l < c->n_layers; ++l) {
    oc_layer* L = &m->layers[l];
#define T(field, nmx, r, cc, dt) \
  snprintf(nm, sizeof(nm), "layers.%d." nmx, l); \
  L->field = add_tensor(m, nm, r, cc, dt)
    T(wq, "wq", d, d, wdt);
    T(wk, "wk", d, d, wdt);
    T(wv, "wv", d, d, wdt);
    T(wo, "wo", d, d, wdt);
    if (c->arch == OC_ARCH_REF) {
      T(w1, "w1", d, ff, wdt);
      T(w2, "w2", ff, d, wdt);
      T(ln1_g, "ln1_gamma", 1, d, OC_F32);
      T(ln1_b, "ln1_beta", 1, d, OC_F32);
      T(ln2_g, "ln2_gamma", 1, d, OC_F32);
      T(ln2_b, "ln2_beta", 1, d, OC_F32);
    } else {
      T(wg, "w_gate", d, ff, wdt);
      T(wu, "w_up", d, ff, wdt);
      T(wd, "w_down", ff, d, wdt);
      T(ln1_g, "ln1_gamma", 1, d, OC_F32);
      T(ln2_g, "ln2_gamma", 1, d, OC_F32);
    }
#undef T
  }
  m->lnf_g = add_tensor(m, "lnf_gamma", 1, d, OC_F32);
  if (c->arch == OC_ARCH_REF) m->lnf_b = add_tensor(m, "lnf_beta", 1, d, OC_F32);
  m->head = add_tensor(m, "head", d, V, wdt);
}

/* init_model (model.cpp:30-76): every tensor U[-0.1,0.1], one stream, fixed order. */
static void init_weights(oc_model* m) {
  const oc_config* c = &m->cfg;
  if (c->init == OC_INIT_MT19937) {
    oc_mt64 eng;
    oc_mt64_seed(&eng, c->seed);
    for (int t = 0; t < m->n_tensors; ++t) {
      oc_tensor* T = &m->tensors[t];
      const int64_t n = T->rows * T->cols;
      for (int64_t i = 0; i < n; ++i) tset(T, i, oc_uniform_symmetric(&eng, 0.1f));
    }
  } else {
    for (int t = 0; t < m->n_tensors; ++t) {
      oc_tensor* T = &m->tensors[t];
      const int64_t n = T->rows * T->cols;
#pragma omp parallel for schedule(static) if (n > 65536)
      for (int64_t i = 0; i < n; ++i) tset(T, i, oc_philox_weight(c->seed, (uint32_t)t, (uint64_t)i, 0.1f));
    }
  }
}

void oc_rope_table(int max_seq, int head_dim, float theta, float* cos_out, float* sin_out) {
  const int half = head_dim / 2;
  for (int p = 0; p < max_seq; ++p)
    for (int i = 0; i < half; ++i) {
      double inv_freq = pow((double)theta, -(2.0 * (double)i) / (double)head_dim);
      double ang = (double)p * inv_freq;
      cos_out[(size_t)p * half + i] = (float)cos(ang);
      sin_out[(size_t)p * half + i] = (float)sin(ang);
    }
}

int oc_create(const oc_config* cfg, oc_model** out) {
  int rc = oc_config_validate(cfg);
  if (rc) return rc;
  oc_model* m = (oc_model*)calloc(1, sizeof(oc_model));
  m->cfg = *cfg;
  m->d_ff = cfg->d_ff > 0 ? cfg->d_ff : 4 * cfg->d_model;
  m->head_dim = cfg->d_model / cfg->n_heads;
#ifdef _OPENMP
  /* the OpenMP team size is process-global: set it on every create (0 = all
     cores), so an earlier 1-thread model does not leave later ones serial */
  omp_set_num_threads(cfg->n_threads > 0 ? cfg->n_threads : omp_get_num_procs());
#endif
  declare_tensors(m);
  init_weights(m);
  const size_t d = (size_t)cfg->d_model;
  m->kv = (float*)calloc((size_t)cfg->n_layers * 2 * (size_t)cfg->max_seq_len * d, sizeof(float));
  m->x = (float*)calloc(d, 4);
  m->ln_out = (float*)calloc(d, 4);
  m->q = (float*)calloc(d, 4);
  m->k = (float*)calloc(d, 4);
  m->v = (float*)calloc(d, 4);
  m->attn_out = (float*)calloc(d, 4);
  m->o = (float*)calloc(d, 4);
  m->mlp = (float*)calloc((size_t)m->d_ff, 4);
  m->up = (float*)calloc((size_t)m->d_ff, 4);
  m->logits = (float*)calloc((size_t)cfg->vocab_size, 4);
  m->probs = (float*)calloc((size_t)cfg->max_seq_len, 4);
  if (cfg->arch == OC_ARCH_LLAMA) {
    size_t n = (size_t)cfg->max_seq_len * (size_t)(m->head_dim / 2);
    m->rope_cos = (float*)calloc(n, 4);
    m->rope_sin = (float*)calloc(n, 4);
    oc_rope_table(cfg->max_seq_len, m->head_dim, cfg->rope_theta, m->rope_cos, m->rope_sin);
  }
  m->cur_len = 0;
  *out = m;
  return OC_OK;
}

void oc_destroy(oc_model* m) {
  if (!m) return;
  for (int t = 0; t < m->n_tensors; ++t) {
    free(m->tensors[t].f);
    free(m->tensors[t].h);
  }
  free(m->tensors);
  free(m->layers);
  free(m->kv);
  free(m->x);
  free(m->ln_out);
  free(m->q);
  free(m->k);
  free(m->v);
  free(m->attn_out);
  free(m->o);
  free(m->mlp);
  free(m->up);
  free(m->logits);
  free(m->probs);
  free(m->rope_cos);
  free(m->rope_sin);
  free(m);
}

void oc_reset(oc_model* m) { m->cur_len = 0; } /* KvCache::reset (kv_cache.hpp:28) */
int oc_cur_len(const oc_model* m) { return m->cur_len; }
const float* oc_logits(const oc_model* m) { return m->logits; }
const float* oc_x(const oc_model* m) { return m->x; }

/* ---- kernels ---- */

/* make_matmul (kernels.cpp:38-48) for m=1: out[j] = sum_p a[p]*b[p*n+j], ascending p,
 * separate multiply and add.  Columns are split across threads; per-element
 * accumulation order is unchanged, so the result is bit-identical to 1 thread. */
static void matmul_1xk(const float* a, const oc_tensor* b, float* out) {
  const int64_t k = b->rows, n = b->cols;
  const int64_t CB = 512;
  const int64_t nblk = (n + CB - 1) / CB;
#pragma omp parallel for schedule(static) if (k * n > (1 << 20))
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t j0 = blk * CB, j1 = (j0 + CB < n) ? j0 + CB : n;
    float* orow = out + j0;
    for (int64_t j = 0; j < j1 - j0; ++j) orow[j] = 0.0f;
    if (b->dtype == OC_F32) {
      for (int64_t p = 0; p < k; ++p) {
        const float av = a[p];
        const float* brow = b->f + p * n + j0;
        for (int64_t j = 0; j < j1 - j0; ++j) orow[j] += av * brow[j];
      }
    } else {
      for (int64_t p = 0; p < k; ++p) {
        const float av = a[p];
        const uint16_t* brow = b->h + p * n + j0;
        for (int64_t j = 0; j < j1 - j0; ++j) orow[j] += av * oc_bf16_to_f32(brow[j]);
      }
    }
  }
}

/* make_layernorm (kernels.cpp:66-83), one row. */
static void layernorm(const float* row, const oc_tensor* g, const oc_tensor* b, float eps, float* out, int64_t d) {
  float mean = 0.0f;
  for (int64_t j = 0; j < d; ++j) mean += row[j];
  mean /= (float)d;
  float var = 0.0f;
  for (int64_t j = 0; j < d; ++j) {
    const float c = row[j] - mean;
    var += c * c;
  }
  var /= (float)d;
  const float inv_std = 1.0f / sqrtf(var + eps);
  for (int64_t j = 0; j < d; ++j) out[j] = (row[j] - mean) * inv_std * g->f[j] + b->f[j];
}

/* RMSNorm: the layernorm loop without the mean and beta (LLaMA extension). */
static void rmsnorm(const float* row, const oc_tensor* g, float eps, float* out, int64_t d) {
  float ms = 0.0f;
  for (int64_t j = 0; j < d; ++j) ms += row[j] * row[j];
  ms /= (float)d;
  const float inv = 1.0f / sqrtf(ms + eps);
  for (int64_t j = 0; j < d; ++j) out[j] = row[j] * inv * g->f[j];
}

static inline float* kv_layer(oc_model* m, int layer, int slot) {
  const size_t d = (size_t)m->cfg.d_model;
  return m->kv + (((size_t)layer * 2 + (size_t)slot) * (size_t)m->cfg.max_seq_len) * d;
}

/* make_kv_write (kernels.cpp:188-203): copy into row `row`; bf16 KV rounds on store. */
static void kv_write(oc_model* m, int layer, int slot, int row, const float* src) {
  const int64_t d = m->cfg.d_model;
  float* dst = kv_layer(m, layer, slot) + (int64_t)row * d;
  if (m->cfg.kv_dtype == OC_F32)
    memcpy(dst, src, (size_t)d * 4);
  else
    for (int64_t i = 0; i < d; ++i) dst[i] = oc_round_bf16(src[i]);
}

/* make_attention (kernels.cpp:108-136). */
static void attention(oc_model* m, int layer, int length, float scale) {
  const int64_t h = m->cfg.n_heads, dh = m->head_dim;
  const float* pk = kv_layer(m, layer, 0);
  const float* pv = kv_layer(m, layer, 1);
  float* probs = m->probs;
  for (int64_t head = 0; head < h; ++head) {
    const float* qh = m->q + head * dh;
    float max_s = -INFINITY;
    for (int64_t j = 0; j < length; ++j) {
      const float* krow = pk + (j * h + head) * dh;
      float s = 0.0f;
      for (int64_t d = 0; d < dh; ++d) s += qh[d] * krow[d];
      s *= scale;
      probs[j] = s;
      max_s = s > max_s ? s : max_s; /* std::max(max_s, s) */
    }
    float denom = 0.0f;
    for (int64_t j = 0; j < length; ++j) {
      const float e = expf(probs[j] - max_s);
      probs[j] = e;
      denom += e;
    }
    float* oh = m->attn_out + head * dh;
    for (int64_t d = 0; d < dh; ++d) oh[d] = 0.0f;
    for (int64_t j = 0; j < length; ++j) {
      const float p = probs[j] / denom;
      const float* vrow = pv + (j * h + head) * dh;
      for (int64_t d = 0; d < dh; ++d) oh[d] += p * vrow[d];
    }
  }
}

/* RoPE rotate-half at position pos on a [h, dh] vector (LLaMA extension). */
static void rope(oc_model* m, float* vec, int pos) {
  const int64_t h = m->cfg.n_heads, dh = m->head_dim, half = dh / 2;
  const float* cs = m->rope_cos + (size_t)pos * (size_t)half;
  const float* sn = m->rope_sin + (size_t)pos * (size_t)half;
  for (int64_t head = 0; head < h; ++head) {
    float* v = vec + head * dh;
    for (int64_t i = 0; i < half; ++i) {
      const float a = v[i], b = v[i + half];
      v[i] = a * cs[i] - b * sn[i];
      v[i + half] = b * cs[i] + a * sn[i];
    }
  }
}

/* The static pass for `length` (build_plan, model.cpp:118-143). */
static void run_plan(oc_model* m, int length) {
  const oc_config* c = &m->cfg;
  const int64_t d = c->d_model, ff = m->d_ff;
  const float scale = 1.0f / sqrtf((float)m->head_dim);
  const int row = length - 1;
  for (int l = 0; l < c->n_layers; ++l) {
    oc_layer* L = &m->layers[l];
    if (c->arch == OC_ARCH_REF)
      layernorm(m->x, L->ln1_g, L->ln1_b, c->norm_eps, m->ln_out, d);
    else
      rmsnorm(m->x, L->ln1_g, c->norm_eps, m->ln_out, d);
    matmul_1xk(m->ln_out, L->wq, m->q);
    matmul_1xk(m->ln_out, L->wk, m->k);
    matmul_1xk(m->ln_out, L->wv, m->v);
    if (c->arch == OC_ARCH_LLAMA) {
      rope(m, m->q, row);
      rope(m, m->k, row);
    }
    kv_write(m, l, 0, row, m->k);
    kv_write(m, l, 1, row, m->v);
    attention(m, l, length, scale);
    matmul_1xk(m->attn_out, L->wo, m->o);
    for (int64_t i = 0; i < d; ++i) m->x[i] += m->o[i];
    if (c->arch == OC_ARCH_REF) {
      layernorm(m->x, L->ln2_g, L->ln2_b, c->norm_eps, m->ln_out, d);
      matmul_1xk(m->ln_out, L->w1, m->mlp);
      for (int64_t i = 0; i < ff; ++i) m->mlp[i] = m->mlp[i] > 0.0f ? m->mlp[i] : 0.0f;
      matmul_1xk(m->mlp, L->w2, m->o);
    } else {
      rmsnorm(m->x, L->ln2_g, c->norm_eps, m->ln_out, d);
      matmul_1xk(m->ln_out, L->wg, m->mlp);
      matmul_1xk(m->ln_out, L->wu, m->up);
      for (int64_t i = 0; i < ff; ++i) {
        const float g = m->mlp[i];
        const float s = g / (1.0f + expf(-g));
        m->mlp[i] = s * m->up[i];
      }
      matmul_1xk(m->mlp, L->wd, m->o);
    }
    for (int64_t i = 0; i < d; ++i) m->x[i] += m->o[i];
  }
  if (c->arch == OC_ARCH_REF)
    layernorm(m->x, m->lnf_g, m->lnf_b, c->norm_eps, m->ln_out, d);
  else
    rmsnorm(m->x, m->lnf_g, c->norm_eps, m->ln_out, d);
  matmul_1xk(m->ln_out, m->head, m->logits);
}

/* step_math (model.cpp:168-174): extend_position, slot append, plan(cur_len). */
int oc_step(oc_model* m, int token) {
  const oc_config* c = &m->cfg;
  const int64_t d = c->d_model;
  const int position = m->cur_len;
  if (token < 0 || token >= c->vocab_size) return OC_TokenOutOfRange;
  if (c->arch == OC_ARCH_REF && position >= c->max_seq_len) return OC_ShapeMismatch;
  if (m->cur_len >= c->max_seq_len) return OC_CacheFull;
  /* make_extend_position (kernels.cpp:255-257): x = emb[token] + pos[position] */
  for (int64_t j = 0; j < d; ++j) {
    float e = tget(m->embedding, (int64_t)token * d + j);
    if (c->arch == OC_ARCH_REF) e = e + tget(m->pos_table, (int64_t)position * d + j);
    m->x[j] = e;
  }
  /* slot append of the zero rows (model.cpp:160-162, kernels.cpp:225-234) */
  const int row = m->cur_len;
  m->cur_len++;
  for (int l = 0; l < c->n_layers; ++l) {
    memset(kv_layer(m, l, 0) + (int64_t)row * d, 0, (size_t)d * 4);
    memset(kv_layer(m, l, 1) + (int64_t)row * d, 0, (size_t)d * 4);
  }
  run_plan(m, m->cur_len);
  return OC_OK;
}

/* prefill_math (model.cpp:176-183) */
int oc_prefill(oc_model* m, const int* toks, int n) {
  if (n <= 0) return OC_EmptyPrompt;
  if (n > m->cfg.max_seq_len) return OC_PromptTooLong;
  for (int i = 0; i < n; ++i) {
    int rc = oc_step(m, toks[i]);
    if (rc) return rc;
  }
  return OC_OK;
}

int oc_kv_row(const oc_model* m, int layer, int slot, int row, float* out) {
  if (layer < 0 || layer >= m->cfg.n_layers || slot < 0 || slot > 1 || row < 0 || row >= m->cfg.max_seq_len)
    return OC_ShapeMismatch;
  const size_t d = (size_t)m->cfg.d_model;
  memcpy(out, kv_layer((oc_model*)m, layer, slot) + (size_t)row * d, d * 4);
  return OC_OK;
}

static const oc_tensor* find_tensor(const oc_model* m, const char* name) {
  for (int t = 0; t < m->n_tensors; ++t)
    if (strcmp(m->tensors[t].name, name) == 0) return &m->tensors[t];
  return NULL;
}

int64_t oc_weight_numel(const oc_model* m, const char* name) {
  const oc_tensor* t = find_tensor(m, name);
  return t ? t->rows * t->cols : -1;
}

int oc_weight_copy(const oc_model* m, const char* name, float* out, int64_t numel) {
  const oc_tensor* t = find_tensor(m, name);
  if (!t || numel != t->rows * t->cols) return OC_ShapeMismatch;
  for (int64_t i = 0; i < numel; ++i) out[i] = tget(t, i);
  return OC_OK;
}

/* ------------------------------------------------------------------------- */
/* Samplers                                                                   */

/* run_sampler greedy (kernels.cpp:265-270): strict >, lowest index wins ties. */
int oc_sample_greedy(const float* logits, int vocab) {
  int best = 0;
  for (int i = 1; i < vocab; ++i)
    if (logits[i] > logits[best]) best = i;
  return best;
}

/* run_sampler temperature (kernels.cpp:271-288). */
int oc_sample_temperature(const float* logits, int vocab, double temperature, oc_mt64* rng) {
  const float t = (float)temperature;
  float max_l = logits[0];
  for (int i = 1; i < vocab; ++i) max_l = logits[i] > max_l ? logits[i] : max_l; /* std::max */
  float* probs = (float*)malloc((size_t)vocab * 4);
  float denom = 0.0f;
  for (int i = 0; i < vocab; ++i) {
    const float e = expf((logits[i] - max_l) / t);
    probs[i] = e;
    denom += e;
  }
  const double u = oc_uniform01(rng) * denom;
  double acc = 0.0;
  int tok = vocab - 1;
  for (int i = 0; i < vocab; ++i) {
    acc += probs[i];
    if (u < acc) {
      tok = i;
      break;
    }
  }
  free(probs);
  return tok;
}

/* Integer-CDF top-k / top-p sampler (extension; the reference only has greedy
 * and temperature).  Bit-exact between this file and the NVRTC kernel because
 * every reduction is over integers:
 *   1. m = max logits; z_i = (l_i - m) / T (fp32 div); e_i = grt_expf(z_i)
 *   2. w_i = (uint64)(e_i * 2^31)                        (exact scaling, truncation; < 2^32)
 *   3. rank key K_i = w_i << 16 | (0xFFFF - i)           (larger weight first, then lower index)
 *   4. top-k (k in [1,V], 0 = off): keep the k largest keys
 *   5. top-p (p in (0,1), >=1 = off): W = sum kept w; thresh = max(1, (uint64)(p * (double)W));
 *      walk kept keys in descending order, keep the shortest prefix whose weight sum >= thresh
 *   6. S = sum kept w; u = 53-bit Philox(seed, step) draw; r = min(S-1, (uint64)(u * (double)S))
 *   7. token = smallest index i (ascending) among kept with inclusive prefix weight > r.
 * Temperature <= 0 means greedy.  If S == 0 (cannot happen: w_max = 2^31) -> argmax. */
typedef struct {
  uint64_t key;
  int idx;
} oc_kent;

static int cmp_key_desc(const void* a, const void* b) {
  uint64_t ka = ((const oc_kent*)a)->key, kb = ((const oc_kent*)b)->key;
  return ka < kb ? 1 : (ka > kb ? -1 : 0);
}

uint64_t oc_sampler_draw53(uint64_t seed, uint64_t step) {
  uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), 0u, 0x53616D70u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  oc_philox4x32_10(ctr, key, o);
  return (((uint64_t)o[1] << 32) | (uint64_t)o[0]) >> 11;
}

int oc_sample_topkp(const float* logits, int vocab, float temperature, int top_k, float top_p,
                    uint64_t seed, uint64_t step) {
  if (!(temperature > 0.0f)) return oc_sample_greedy(logits, vocab);
  float m = logits[0];
  for (int i = 1; i < vocab; ++i) m = logits[i] > m ? logits[i] : m;
  uint64_t* w = (uint64_t*)malloc((size_t)vocab * 8);
  unsigned char* kept = (unsigned char*)calloc((size_t)vocab, 1);
  oc_kent* ents = (oc_kent*)malloc((size_t)vocab * sizeof(oc_kent));
  for (int i = 0; i < vocab; ++i) {
    const float z = (logits[i] - m) / temperature;
    const float e = oc_grt_expf(z);
    w[i] = (uint64_t)(e * 2147483648.0f);
    ents[i].key = (w[i] << 16) | (uint64_t)(0xFFFF - i);
    ents[i].idx = i;
  }
  qsort(ents, (size_t)vocab, sizeof(oc_kent), cmp_key_desc);
  int nk = (top_k > 0 && top_k < vocab) ? top_k : vocab;
  uint64_t W = 0;
  for (int r = 0; r < nk; ++r) W += w[ents[r].idx];
  if (top_p > 0.0f && top_p < 1.0f) {
    uint64_t thresh = (uint64_t)((double)top_p * (double)W);
    if (thresh < 1) thresh = 1;
    uint64_t acc = 0;
    int r = 0;
    for (; r < nk; ++r) {
      acc += w[ents[r].idx];
      if (acc >= thresh) break;
    }
    nk = (r < nk) ? r + 1 : nk;
  }
  uint64_t S = 0;
  for (int r = 0; r < nk; ++r) {
    kept[ents[r].idx] = 1;
    S += w[ents[r].idx];
  }
  int tok = ents[0].idx;
  if (S > 0) {
    const double u = (double)oc_sampler_draw53(seed, step) * 0x1.0p-53;
    uint64_t r = (uint64_t)(u * (double)S);
    if (r >= S) r = S - 1;
    uint64_t acc = 0;
    for (int i = 0; i < vocab; ++i) {
      if (!kept[i]) continue;
      acc += w[i];
      if (acc > r) {
        tok = i;
        break;
      }
    }
  }
  free(w);
  free(kept);
  free(ents);
  return tok;
}

/* ------------------------------------------------------------------------- */
/* bench helpers                                                              */

/* make_prompt (bench.cpp:34-39) */
void oc_make_prompt(uint64_t base_seed, int prompt_len, int vocab_size, int* out) {
  oc_mt64 eng;
  oc_mt64_seed(&eng, base_seed * 1000003ULL + (uint64_t)prompt_len);
  for (int i = 0; i < prompt_len; ++i) out[i] = (int)(oc_mt64_next(&eng) % (uint64_t)vocab_size);
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* percentile (bench.cpp:41-49): nearest rank ceil(p/100*n). Returns NaN on bad input. */
double oc_percentile(const double* samples, int n, double p) {
  if (n <= 0 || !(p > 0.0) || p > 100.0) return NAN;
  double* s = (double*)malloc((size_t)n * sizeof(double));
  memcpy(s, samples, (size_t)n * sizeof(double));
  qsort(s, (size_t)n, sizeof(double), cmp_double);
  size_t rank = (size_t)ceil(p / 100.0 * (double)n);
  if (rank == 0) rank = 1;
  double v = s[rank - 1];
  free(s);
  return v;
}
