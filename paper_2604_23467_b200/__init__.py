"""B200-native hybrid JIT / CUDA-Graph batch-1 decode path (arXiv 2604.23467).

The product is libgraphrt_b200.so: a C++ runtime that mirrors the reference
graphrt API (Session / GraphCache / CaptureEngine / RunMode) over hand-written
sm_100a kernels and NVRTC-compiled dynamic ops, exported through the C ABI in
include/grt/c_api.h.  graphrt.py is the ctypes view of that ABI.
"""
from .graphrt import (ALL_MODES, ARCH_LLAMA, ARCH_REF, BF16, F32, INIT_MT19937, INIT_NONE, INIT_PHILOX,  # noqa: F401
                      CacheConfig, Errc, Error, EvictionPolicy, GenerationRequest, GenerationResult, Model,
                      ModelConfig, RunMode, SampleStrategy, Session, StepPath, mode_from_name, mode_name,
                      run_inference)
