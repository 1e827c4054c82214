// loop.cu -- the device-resident decode loop.
//
// The whole decode of a request is ONE cudaGraphLaunch: a conditional WHILE
// node whose body is
//     [sample + extend_position (NVRTC)] -> [loop_ctl] -> SWITCH(bucket) { static pass of bucket k }
// loop_ctl runs after the dynamic block has bumped the device seq_len: it picks
// the bucket graph for the new length (the host-side GraphGenerator::serve
// decision, pipeline.cpp:128-152, moved on the device), counts the step down
// and clears the WHILE condition after the last step -- or right away on an
// end-of-sequence token or a device error, in which case the switch selects no
// body and the pass is skipped.  No host work happens between tokens.
#include <cuda_runtime.h>

#include "../jit/ctrl.h"
#include "kernels.h"

namespace grt {

__global__ void loop_ctl_kernel(const GrtCtrl* ctrl, LoopCtl* lc, cudaGraphConditionalHandle h_while,
                                cudaGraphConditionalHandle h_switch) {
  const int len = ctrl->seq_len;
  const int key = (len + lc->bucket - 1) / lc->bucket;
  int idx = key - lc->key_lo;
  const int rem = lc->remaining - 1;
  const bool eos = lc->eos >= 0 && len >= 1 && ctrl->tokens[len - 1] == lc->eos;
  bool stop = ctrl->err != 0 || eos;
  if (idx < 0 || idx >= lc->n_keys) {
    stop = true;
    atomicOr(&lc->status, LOOP_NO_BUCKET);
  }
  if (eos) atomicOr(&lc->status, LOOP_EOS);
  lc->remaining = rem;
  lc->iters += 1;
  cudaGraphSetConditional(h_switch, stop ? static_cast<unsigned>(lc->n_keys) : static_cast<unsigned>(idx));
  cudaGraphSetConditional(h_while, (!stop && rem > 0) ? 1u : 0u);
}

cudaError_t launch_loop_ctl(const GrtCtrl* ctrl, LoopCtl* lc, cudaGraphConditionalHandle h_while,
                            cudaGraphConditionalHandle h_switch, cudaStream_t s) {
  loop_ctl_kernel<<<1, 1, 0, s>>>(ctrl, lc, h_while, h_switch);
  return cudaGetLastError();
}

}  // namespace grt
