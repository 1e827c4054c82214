// ctrl.h -- the device-resident control block shared by the host runtime, the
// static kernels and the NVRTC-compiled dynamic kernels.
//
// This is what makes one captured graph replay across steps: every value the
// reference bakes into a kernel closure (token id, position, cache length, RNG
// draw -- kernels.hpp:14-19) lives here in device memory instead.
// Plain C so NVRTC can compile it without any include path.
#ifndef GRT_CTRL_H
#define GRT_CTRL_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct GrtCtrl {
  int seq_len;       /* live KV length (KvCache::cur_len, kv_cache.hpp:26) */
  int prompt_len;    /* sampler is a no-op while seq_len < prompt_len (prefill) */
  int err;           /* DevErr bits */
  int sample_kind;   /* grt_sample_kind */
  float temperature;
  int top_k;
  float top_p;
  int max_gen;       /* capacity of out_tokens / uniforms */
  unsigned long long seed;
  int* tokens;                    /* [max_seq] token history: prompt, then sampled */
  const double* uniforms;         /* [max_gen] reference-compatible uniform01 draws */
  float* scratch;                 /* [vocab] sampler scratch */
  volatile int* out_tokens;       /* host-mapped [max_gen] */
  volatile unsigned long long* out_stamps; /* host-mapped [2*max_gen]: start,end per step (ns) */
} GrtCtrl;

#ifdef __cplusplus
}
#endif
#endif
