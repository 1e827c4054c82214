// jit.cpp -- NVRTC path for the dynamic ops (the paper's JIT context generator).
//
// The reference runs its dynamic ops as host closures (kernels.cpp:205-308);
// the paper JIT-compiles them (TorchScript).  Here they are CUDA C++ compiled
// at runtime by NVRTC straight to an sm_100a cubin, specialised on the model
// shape, loaded with the driver API and launched with cuLaunchKernelEx
// (capturable, PDL-enabled).  Compiled modules are cached per (options, device).
#include <nvrtc.h>

#include <chrono>
#include <mutex>

#include "runtime.hpp"

namespace grt {

#include "jit_sources.inc"  // kDynamicOpsSrc, kCtrlHeaderSrc (generated from csrc/jit/ by build.py)

namespace {

void nvrtc_check(nvrtcResult r, const char* what, nvrtcProgram* prog = nullptr) {
  if (r == NVRTC_SUCCESS) return;
  std::string msg = std::string(what) + ": " + nvrtcGetErrorString(r);
  if (prog) {
    size_t n = 0;
    nvrtcGetProgramLogSize(*prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(*prog, log.data());
    msg += "\n" + log;
  }
  raise(GRT_NvrtcError, msg);
}

std::mutex g_jit_mu;
std::map<std::string, std::weak_ptr<JitModule>> g_jit_cache;

// The driver API is resolved at run time through cudaGetDriverEntryPoint, so
// the library loads (and its C ABI can be inspected) on hosts without
// libcuda.so.1; the product path still fails loudly there (NoDevice).
struct DriverApi {
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*LaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
};

template <typename F>
void resolve(const char* name, F*& fp) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
    cudaGetLastError();
    raise(GRT_NoDevice, std::string("driver entry point unavailable: ") + name);
  }
  fp = reinterpret_cast<F*>(p);
}

const DriverApi& drv() {
  static std::once_flag once;
  static DriverApi api;
  static std::string err;
  std::call_once(once, [] {
    try {
      resolve("cuModuleLoadData", api.ModuleLoadData);
      resolve("cuModuleUnload", api.ModuleUnload);
      resolve("cuModuleGetFunction", api.ModuleGetFunction);
      resolve("cuLaunchKernelEx", api.LaunchKernelEx);
      resolve("cuGetErrorString", api.GetErrorString);
      resolve("cuFuncSetAttribute", api.FuncSetAttribute);
    } catch (const Error& e) {
      err = e.what();
    }
  });
  if (!err.empty()) raise(GRT_NoDevice, err);
  return api;
}

}  // namespace

const char* cu_error_string(CUresult e) {
  const char* s = nullptr;
  try {
    drv().GetErrorString(e, &s);
  } catch (...) {
  }
  return s ? s : "unknown driver error";
}

std::string jit_compile(const std::vector<std::string>& opts) {
  nvrtcProgram prog;
  const char* headers[] = {kCtrlHeaderSrc};
  const char* names[] = {"ctrl.h"};
  nvrtc_check(nvrtcCreateProgram(&prog, kDynamicOpsSrc, "dynamic_ops.cu", 1, headers, names), "nvrtcCreateProgram");
  std::vector<std::string> all = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "-lineinfo"};
  all.insert(all.end(), opts.begin(), opts.end());
  std::vector<const char*> copts;
  for (const auto& o : all) copts.push_back(o.c_str());
  nvrtcResult r = nvrtcCompileProgram(prog, static_cast<int>(copts.size()), copts.data());
  if (r != NVRTC_SUCCESS) nvrtc_check(r, "nvrtcCompileProgram", &prog);
  size_t n = 0;
  nvrtc_check(nvrtcGetCUBINSize(prog, &n), "nvrtcGetCUBINSize");
  std::string cubin(n, '\0');
  nvrtc_check(nvrtcGetCUBIN(prog, cubin.data()), "nvrtcGetCUBIN");
  nvrtcDestroyProgram(&prog);
  return cubin;
}

// Dynamic shared memory of the NVRTC sampler kernels (top-k/top-p weights cache,
// dynamic_ops.cu GRT_TOPKP_SMEM): registered per CUfunction by JitModule::fn,
// applied by launch_jit.
static std::mutex g_dyn_mu;
static std::map<CUfunction, unsigned> g_dyn_smem;
constexpr int kSampleSmemMax = 196608;  // GRT_SAMPLE_SMEM_MAX in dynamic_ops.cu

JitModule::JitModule(const std::string& /*key*/, const std::vector<std::string>& opts, int device) {
  for (const auto& o : opts)
    if (o.rfind("-DGRT_V=", 0) == 0) vocab_ = atoi(o.c_str() + 8);
  const auto t0 = std::chrono::steady_clock::now();
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaFree(nullptr), "context init");
  const std::string cubin = jit_compile(opts);
  cu_check(drv().ModuleLoadData(&mod_, cubin.data()), "cuModuleLoadData");
  compile_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

JitModule::~JitModule() {
  {
    std::lock_guard<std::mutex> lk(g_dyn_mu);
    for (CUfunction f : fns_) g_dyn_smem.erase(f);
  }
  if (mod_) drv().ModuleUnload(mod_);
}

CUfunction JitModule::fn(const char* name) const {
  CUfunction f = nullptr;
  cu_check(drv().ModuleGetFunction(&f, mod_, name), name);
  // same L1/shared carveout as the GEMVs: PDL successors can co-reside without
  // an SM reconfiguration
  cu_check(drv().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 100), name);
  unsigned bytes = 0;
  if (std::string(name).rfind("grt_sample", 0) == 0 && vocab_ > 0 && vocab_ * 4 <= kSampleSmemMax) {
    // weights (u32) + the radix select's u16 candidate list when both fit (GRT_TOPKP_SMEM 2)
    bytes = static_cast<unsigned>(vocab_) * (vocab_ * 6 <= kSampleSmemMax && vocab_ <= 32768 ? 6 : 4);
    cu_check(drv().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, static_cast<int>(bytes)), name);
  }
  // every function is (re)registered: a handle of an unloaded module may be reused
  std::lock_guard<std::mutex> lk(g_dyn_mu);
  g_dyn_smem[f] = bytes;
  fns_.push_back(f);
  return f;
}

std::shared_ptr<JitModule> jit_get(const std::vector<std::string>& opts, int device) {
  std::string key = std::to_string(device);
  for (const auto& o : opts) key += " " + o;
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto it = g_jit_cache.find(key);
  if (it != g_jit_cache.end()) {
    if (auto sp = it->second.lock()) return sp;
  }
  auto sp = std::make_shared<JitModule>(key, opts, device);
  g_jit_cache[key] = sp;
  return sp;
}

cudaError_t launch_jit(CUfunction f, dim3 grid, dim3 block, void** args, cudaStream_t s, bool pdl) {
  CUlaunchConfig cfg = {};
  cfg.gridDimX = grid.x;
  cfg.gridDimY = grid.y;
  cfg.gridDimZ = grid.z;
  cfg.blockDimX = block.x;
  cfg.blockDimY = block.y;
  cfg.blockDimZ = block.z;
  {
    std::lock_guard<std::mutex> lk(g_dyn_mu);
    auto it = g_dyn_smem.find(f);
    cfg.sharedMemBytes = it == g_dyn_smem.end() ? 0 : it->second;
  }
  cfg.hStream = reinterpret_cast<CUstream>(s);
  CUlaunchAttribute attr[1];
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CUresult r = drv().LaunchKernelEx(&cfg, f, args, nullptr);
  if (r == CUDA_ERROR_INVALID_VALUE) return cudaErrorInvalidValue;
  if (r != CUDA_SUCCESS) return cudaErrorLaunchFailure;
  return cudaSuccess;
}

}  // namespace grt
