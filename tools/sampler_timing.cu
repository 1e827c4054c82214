// sampler_timing.cu -- phase timing probe of the NVRTC sampler (not part of the
// product): dynamic_ops.cu compiled offline for V=32000 with GRT_STAMP recording
// clock64() of thread 0 at the phase boundaries of the integer-CDF top-k/top-p
// path (1 max, 2 weights, 3 top-k select, 4 W sum, 5 top-p select, 6 draw).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -Ipaper_2604_23467_b200/csrc/jit \
//        -DGRT_D=4096 -DGRT_V=32000 -DGRT_MAXSEQ=2048 -DGRT_WBF16=1 -DGRT_ARCH_REF=0 \
//        -o tools/sampler_timing tools/sampler_timing.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <random>
#include <vector>

__device__ long long g_stamps[16];
#define GRT_STAMP(i)                                  \
  do {                                                \
    if (threadIdx.x == 0) g_stamps[i] = clock64();    \
  } while (0)
#include "dynamic_ops.cu"

int main() {
  const int V = GRT_V;
  std::vector<float> lg(V);
  std::mt19937 rng(7);
  std::normal_distribution<float> nd(0.f, 3.f);
  float *dl, *scratch;
  int* tokens;
  double* uni;
  GrtCtrl* ctrl;
  cudaMalloc(&dl, V * 4);
  cudaMalloc(&scratch, V * 4);
  cudaMalloc(&tokens, 64 * 4);
  cudaMalloc(&uni, 64 * 8);
  cudaMalloc(&ctrl, sizeof(GrtCtrl));
  cudaFuncSetAttribute(grt_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, V * 6);
  struct Case {
    const char* name;
    int k;
    float p, scale;
  } cases[] = {{"top-p 0.9 (logits sd 3)", 0, 0.9f, 3.f}, {"top-p 0.9 (logits sd 0.3)", 0, 0.9f, 0.3f},
               {"top-k 50", 50, 1.0f, 3.f}, {"top-k 50 + top-p 0.9", 50, 0.9f, 3.f}};
  for (auto& c : cases) {
    for (int i = 0; i < V; ++i) lg[i] = nd(rng) * c.scale / 3.f;
    cudaMemcpy(dl, lg.data(), V * 4, cudaMemcpyHostToDevice);
    GrtCtrl h{};
    h.seq_len = 1;
    h.prompt_len = 0;
    h.sample_kind = 2;
    h.temperature = 0.8f;
    h.top_k = c.k;
    h.top_p = c.p;
    h.max_gen = 0;
    h.seed = 7;
    h.tokens = tokens;
    h.uniforms = uni;
    h.scratch = scratch;
    cudaMemcpy(ctrl, &h, sizeof(h), cudaMemcpyHostToDevice);
    long long st[16];
    double acc[16] = {0};
    const int reps = 20;
    for (int r = 0; r < reps + 1; ++r) {
      long long zero[16] = {0};
      cudaMemcpyToSymbol(g_stamps, zero, sizeof(zero));
      grt_sample<<<1, 1024, V * 6>>>(ctrl, dl);
      cudaDeviceSynchronize();
      cudaMemcpyFromSymbol(st, g_stamps, sizeof(st));
      if (r == 0) continue;
      long long prev = st[0];
      for (int i = 1; i <= 6; ++i) {
        if (st[i] == 0) continue;
        acc[i] += (st[i] - prev) / 1.965e3;  // us at 1965 MHz
        prev = st[i];
      }
      // draw internals: 5 -> 7 (warp totals), 7 -> 8 (scan), 8 -> 6 (draw + walk)
      if (st[7] && st[8]) {
        acc[12 + 0] += (st[7] - st[5]) / 1.965e3;
        acc[12 + 1] += (st[8] - st[7]) / 1.965e3;
        acc[12 + 2] += (st[6] - st[8]) / 1.965e3;
      }
      // select passes (the last select run): 9..13 end of pass 0..4
      for (int i = 9; i <= 11; ++i)
        if (st[i]) acc[i - 9 + 7] += (st[i] - (i == 9 ? 0 : st[i - 1])) / 1.965e3 * (i == 9 ? 0 : 1);
    }
    printf("%-28s", c.name);
    const char* nm[] = {"", "max", "weights", "top-k sel", "W sum", "top-p sel", "draw"};
    for (int i = 1; i <= 6; ++i) printf("  %s %.2f", nm[i], acc[i] / reps);
    printf("  us\n     draw: totals %.2f scan %.2f walk %.2f;  select pass1 %.2f pass2 %.2f\n", acc[12] / reps,
           acc[13] / reps, acc[14] / reps, acc[8] / reps, acc[9] / reps);
  }
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
