"""Python mirror of the reference graphrt runtime API over the C ABI.

Names, fields and error behaviour follow the reference (/root/reference/proj/core):
ModelConfig (model.hpp:17-29), CacheConfig (pipeline.hpp:122-128), RunMode
(pipeline.hpp:18-24), SampleStrategy (kernels.hpp:105-115), GenerationRequest /
GenerationResult (pipeline.hpp:133-159), Session / run_inference
(pipeline.hpp:165-189), Errc + Error (error.hpp:10-54).  Everything executes in
libgraphrt_b200.so (C++ runtime + sm_100a kernels); this module only marshals
arguments.  There is no CPU fallback: without the library or a GPU, calls fail.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GRT_LIB_PATH") or os.path.join(_HERE, "libgraphrt_b200.so")  # override: A/B of builds


class Errc(enum.IntEnum):
    """graphrt::Errc (error.hpp:10-39), same order; device codes appended."""
    Ok = 0
    ShapeMismatch = 1
    TokenOutOfRange = 2
    EmptyCache = 3
    CacheFull = 4
    InvalidConfig = 5
    LengthOutOfRange = 6
    PromptTooLong = 7
    EmptyPrompt = 8
    CaptureInProgress = 9
    CaptureViolation = 10
    ForeignBuffer = 11
    SessionClosed = 12
    EmptyCapture = 13
    ReplayShapeError = 14
    WrongLength = 15
    KeyMismatch = 16
    WarmupExceedsCapacity = 17
    StaticInFusedBlock = 18
    DeviceStopped = 19
    UnknownEvent = 20
    EmptySamples = 21
    IoError = 22
    CudaError = 100
    NvrtcError = 101
    NcclError = 102
    IpcError = 103
    Unsupported = 104
    NoDevice = 105


class Error(RuntimeError):
    """graphrt::Error: carries the Errc code (tests assert on the code)."""

    def __init__(self, code: int, what: str):
        super().__init__(what)
        self.code = Errc(code)


class RunMode(enum.IntEnum):
    Eager = 0
    Hybrid = 1
    GraphOnly = 2
    AblateAsync = 3
    AblateFused = 4
    AblateBoth = 5
    DeviceLoop = 6  # extension: the whole decode as one graph launch (WHILE + SWITCH nodes)


_MODE_NAMES = {RunMode.Eager: "eager", RunMode.Hybrid: "hybrid", RunMode.GraphOnly: "graph_only",
               RunMode.AblateAsync: "ablate_async", RunMode.AblateFused: "ablate_fused",
               RunMode.AblateBoth: "ablate_both", RunMode.DeviceLoop: "device_loop"}
ALL_MODES = list(RunMode)


def mode_name(m: RunMode) -> str:
    return _MODE_NAMES[RunMode(m)]


def mode_from_name(name: str) -> RunMode:
    for m, n in _MODE_NAMES.items():
        if n == name:
            return m
    raise Error(Errc.InvalidConfig, f"unknown mode '{name}'")


class StepPath(enum.IntEnum):
    Replayed = 0
    EagerFallback = 1
    Batched = 2  # prompt served by the batched (tcgen05) prefill, launched eagerly
    BatchedReplayed = 3  # the batched prefill replayed as one CUDA graph (per prompt length)


class EvictionPolicy(enum.IntEnum):
    LeastUsed = 0
    LeastRecentlyUsed = 1


ARCH_REF, ARCH_LLAMA = 0, 1
F32, BF16, F16 = 0, 1, 2
INIT_MT19937, INIT_PHILOX, INIT_NONE = 0, 1, 2


# ---------------------------------------------------------------------------
# C structs (include/grt/c_api.h)

class _ModelConfig(C.Structure):
    _fields_ = [("arch", C.c_int32), ("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("vocab_size", C.c_int32), ("max_seq_len", C.c_int32), ("d_ff", C.c_int32),
                ("norm_eps", C.c_float), ("seed", C.c_uint64), ("init", C.c_int32),
                ("weight_dtype", C.c_int32), ("kv_dtype", C.c_int32), ("rope_theta", C.c_float),
                ("device", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32),
                ("kv_page_size", C.c_int32)]


class _CacheConfig(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("warmup_lo", C.c_int32), ("warmup_hi", C.c_int32),
                ("prefill_uses_graphs", C.c_int32), ("policy", C.c_int32), ("bucket_size", C.c_int32),
                ("batched_prefill", C.c_int32), ("pass_impl", C.c_int32), ("prefill_fuse_norm", C.c_int32)]


class _SampleParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("temperature", C.c_float), ("top_k", C.c_int32), ("top_p", C.c_float),
                ("seed", C.c_uint64)]


class _Request(C.Structure):
    _fields_ = [("mode", C.c_int32), ("prompt", C.POINTER(C.c_int32)), ("prompt_len", C.c_int32),
                ("gen_len", C.c_int32), ("sampling", _SampleParams), ("stop_on_eos", C.c_int32),
                ("eos_token", C.c_int32)]


class _Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("dispatches", "kernel_launches", "fused_blocks", "graph_replays",
                                           "captures", "events_recorded", "events_waited",
                                           "graph_kernel_nodes")]


class _CacheStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("hits", "misses", "inserts", "evictions", "releases")]


class _Result(C.Structure):
    _fields_ = [("tokens", C.POINTER(C.c_int32)), ("per_token_us", C.POINTER(C.c_double)),
                ("prefill_paths", C.POINTER(C.c_int32)), ("decode_paths", C.POINTER(C.c_int32)),
                ("ttft_us", C.c_double), ("total_us", C.c_double), ("prefill_us", C.c_double),
                ("counters", _Counters), ("cache_delta", _CacheStats), ("captures_completed", C.c_int32),
                ("cache_released", C.c_uint64), ("host_token_us", C.POINTER(C.c_double))]


# Every symbol include/grt/c_api.h declares (tests check the library exports them all).
EXPORTS = [
    "grt_status_name", "grt_last_error", "grt_abi_version", "grt_device_count", "grt_jit_compile_check",
    "grt_model_config_default", "grt_cache_config_default", "grt_model_create", "grt_model_destroy",
    "grt_model_upload", "grt_model_download", "grt_model_weight_bytes", "grt_model_decode_bytes",
    "grt_model_load_safetensors", "grt_safetensors_list", "grt_hf_tensor_name",
    "grt_model_kv_pages", "grt_model_set_kv_block_table",
    "grt_session_create", "grt_session_destroy", "grt_generate", "grt_cache_stats_get", "grt_session_counters",
    "grt_reset", "grt_step", "grt_prefill", "grt_cur_len", "grt_get_logits", "grt_get_kv_row", "grt_sample",
    "grt_sampler_reset", "grt_op_gemv", "grt_op_attention", "grt_op_sample", "grt_op_prefill_gemm",
    "grt_graph_cache_create", "grt_graph_cache_destroy", "grt_graph_cache_lookup", "grt_graph_cache_insert",
    "grt_graph_cache_warmup", "grt_graph_cache_begin_session", "grt_graph_cache_release_inactive",
    "grt_graph_cache_query", "grt_profile_plan", "grt_trace_pass",
    "grt_tp_unique_id", "grt_model_attach_nccl", "grt_tp_emu_create", "grt_tp_emu_destroy", "grt_tp_emu_reset",
    "grt_tp_emu_step", "grt_tp_emu_logits", "grt_tp_emu_threaded",
    "grt_ipc_server_create", "grt_ipc_server_serve", "grt_ipc_server_destroy", "grt_ipc_client_create",
    "grt_ipc_client_generate", "grt_ipc_client_destroy",
    "grt_capture_begin", "grt_capture_record", "grt_capture_record_external", "grt_capture_end",
    "grt_capture_state_get", "grt_capture_destroy", "grt_plan_size", "grt_session_replay", "grt_model_arena_info",
    "grt_model_tp_info",
]

_lib = None


def lib():
    """Loads libgraphrt_b200.so; fails loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback for the decode path)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.grt_status_name.restype = C.c_char_p
        L.grt_status_name.argtypes = [C.c_int]
        L.grt_last_error.restype = C.c_char_p
        L.grt_abi_version.restype = C.c_int32
        L.grt_device_count.argtypes = [C.POINTER(C.c_int32)]
        L.grt_jit_compile_check.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_uint64)]
        L.grt_model_config_default.argtypes = [C.POINTER(_ModelConfig)]
        L.grt_model_config_default.restype = None
        L.grt_cache_config_default.argtypes = [C.POINTER(_CacheConfig)]
        L.grt_cache_config_default.restype = None
        L.grt_model_create.argtypes = [C.POINTER(_ModelConfig), C.POINTER(vp)]
        L.grt_model_destroy.argtypes = [vp]
        L.grt_model_upload.argtypes = [vp, C.c_char_p, vp, C.c_size_t, C.c_int32]
        L.grt_model_download.argtypes = [vp, C.c_char_p, C.POINTER(C.c_float), C.c_size_t]
        L.grt_model_weight_bytes.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.grt_model_kv_pages.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.grt_model_set_kv_block_table.argtypes = [vp, C.POINTER(C.c_int32), C.c_int32]
        L.grt_model_load_safetensors.argtypes = [vp, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_safetensors_list.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32)]
        L.grt_hf_tensor_name.argtypes = [C.c_char_p, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_model_decode_bytes.argtypes = [vp, C.c_int32, C.POINTER(C.c_uint64)]
        L.grt_session_create.argtypes = [vp, C.POINTER(_CacheConfig), C.POINTER(vp)]
        L.grt_tp_unique_id.argtypes = [C.c_char_p, C.c_int32]
        L.grt_ipc_server_create.argtypes = [vp, C.c_char_p, C.c_char_p, C.POINTER(vp)]
        L.grt_ipc_server_serve.argtypes = [vp, C.c_int32]
        L.grt_ipc_server_destroy.argtypes = [vp]
        L.grt_ipc_client_create.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(vp)]
        L.grt_ipc_client_generate.argtypes = [vp, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                              C.POINTER(_SampleParams), C.POINTER(C.c_int32),
                                              C.POINTER(C.c_double)]
        L.grt_ipc_client_destroy.argtypes = [vp]
        L.grt_model_attach_nccl.argtypes = [vp, C.c_char_p, C.c_int32]
        L.grt_tp_emu_create.argtypes = [C.POINTER(_ModelConfig), C.POINTER(vp)]
        L.grt_tp_emu_destroy.argtypes = [vp]
        L.grt_tp_emu_reset.argtypes = [vp]
        L.grt_tp_emu_step.argtypes = [vp, C.c_int32]
        L.grt_tp_emu_logits.argtypes = [vp, C.POINTER(C.c_float), C.c_int32]
        L.grt_tp_emu_threaded.argtypes = [C.POINTER(_ModelConfig), C.POINTER(C.c_int32), C.c_int32,
                                          C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_float)]
        L.grt_session_destroy.argtypes = [vp]
        L.grt_generate.argtypes = [vp, C.POINTER(_Request), C.POINTER(_Result)]
        L.grt_cache_stats_get.argtypes = [vp, C.POINTER(_CacheStats), C.POINTER(C.c_uint64)]
        L.grt_session_counters.argtypes = [vp, C.POINTER(_Counters)]
        L.grt_reset.argtypes = [vp]
        L.grt_step.argtypes = [vp, C.c_int32]
        L.grt_prefill.argtypes = [vp, C.POINTER(C.c_int32), C.c_int32]
        L.grt_cur_len.argtypes = [vp, C.POINTER(C.c_int32)]
        L.grt_get_logits.argtypes = [vp, C.POINTER(C.c_float), C.c_int32]
        L.grt_get_kv_row.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_float)]
        L.grt_sample.argtypes = [vp, C.POINTER(_SampleParams), C.POINTER(C.c_int32)]
        L.grt_sampler_reset.argtypes = [vp, C.c_uint64]
        L.grt_op_gemv.argtypes = [vp, C.c_int32, vp, vp, C.c_int32, C.c_int32, vp]
        L.grt_op_prefill_gemm.argtypes = [vp, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp]
        L.grt_op_attention.argtypes = [vp, vp, vp, C.c_int32, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_float, vp]
        L.grt_op_sample.argtypes = [vp, C.c_int32, C.POINTER(_SampleParams), C.c_uint64, C.c_double, vp, vp]
        L.grt_profile_plan.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                       C.c_char_p, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_trace_pass.argtypes = [vp, C.c_int32, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]
        L.grt_capture_begin.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.grt_capture_record.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32]
        L.grt_capture_record_external.argtypes = [vp, vp, C.c_uint64]
        L.grt_capture_end.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]
        L.grt_capture_state_get.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.grt_capture_destroy.argtypes = [vp]
        L.grt_capture_destroy.restype = None
        L.grt_plan_size.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_model_tp_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.grt_session_replay.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.grt_model_arena_info.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.grt_graph_cache_create.argtypes = [C.c_uint64, C.c_int32, C.POINTER(vp)]
        L.grt_graph_cache_destroy.argtypes = [vp]
        L.grt_graph_cache_lookup.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_graph_cache_insert.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_graph_cache_warmup.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
        L.grt_graph_cache_begin_session.argtypes = [vp]
        L.grt_graph_cache_release_inactive.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.grt_graph_cache_query.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                            C.POINTER(C.c_uint64), C.POINTER(_CacheStats)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().grt_last_error().decode(errors="replace")
        raise Error(rc, msg or Errc(rc).name)


# ---------------------------------------------------------------------------
# configs (model.hpp:17-29, pipeline.hpp:122-128)

@dataclass
class ModelConfig:
    n_layers: int = 4
    d_model: int = 64
    n_heads: int = 4
    vocab_size: int = 256
    max_seq_len: int = 600
    ln_eps: float = 1e-5
    seed: int = 1234
    # extensions (SURVEY §5 "Config / flags")
    arch: int = ARCH_REF
    d_ff_: int = 0
    init: int = INIT_MT19937
    weight_dtype: int = F32
    kv_dtype: int = F32
    rope_theta: float = 10000.0
    device: int = 0
    tp_size: int = 1   # tensor parallel ranks; this model holds rank tp_rank's shard
    tp_rank: int = 0
    kv_page_size: int = 0  # 0 = contiguous KV; > 0 = paged pool + block table

    def d_ff(self) -> int:
        return self.d_ff_ if self.d_ff_ > 0 else 4 * self.d_model

    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def _c(self) -> _ModelConfig:
        c = _ModelConfig()
        c.arch, c.n_layers, c.d_model, c.n_heads = self.arch, self.n_layers, self.d_model, self.n_heads
        c.vocab_size, c.max_seq_len, c.d_ff = self.vocab_size, self.max_seq_len, self.d_ff_
        c.norm_eps, c.seed, c.init = self.ln_eps, self.seed, self.init
        c.weight_dtype, c.kv_dtype, c.rope_theta = self.weight_dtype, self.kv_dtype, self.rope_theta
        c.device, c.tp_size, c.tp_rank = self.device, self.tp_size, self.tp_rank
        c.kv_page_size = self.kv_page_size
        return c

    @staticmethod
    def llama2_7b(**kw) -> "ModelConfig":
        """LLaMA-2 7B dims (SURVEY §8 '7B'), random init, bf16."""
        base = dict(arch=ARCH_LLAMA, n_layers=32, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=640,
                    d_ff_=11008, init=INIT_PHILOX, weight_dtype=BF16, kv_dtype=BF16, seed=1234)
        base.update(kw)
        return ModelConfig(**base)


@dataclass
class CacheConfig:
    capacity: int = 600
    warmup_lo: int = 1
    warmup_hi: int = 50
    prefill_uses_graphs: bool = True
    policy: EvictionPolicy = EvictionPolicy.LeastUsed
    bucket_size: int = 64
    batched_prefill: bool = False
    pass_impl: int = 1  # 1: the per-op kernel graph (the only supported value)
    prefill_fuse_norm: bool = True  # split-K residual partials reduced inside the next RMSNorm launch

    def _c(self) -> _CacheConfig:
        c = _CacheConfig()
        c.capacity, c.warmup_lo, c.warmup_hi = self.capacity, self.warmup_lo, self.warmup_hi
        c.prefill_uses_graphs = 1 if self.prefill_uses_graphs else 0
        c.policy, c.bucket_size = int(self.policy), self.bucket_size
        c.batched_prefill = 1 if self.batched_prefill else 0
        c.pass_impl = int(self.pass_impl)
        c.prefill_fuse_norm = 1 if self.prefill_fuse_norm else 0
        return c


@dataclass
class SampleStrategy:
    """kernels.hpp:105-115, plus the Philox top-k/top-p extension."""
    kind: int = 0  # 0 greedy, 1 temperature (reference-compatible), 2 top-k/top-p
    temperature: float = 1.0
    top_k: int = 0
    top_p: float = 1.0

    @staticmethod
    def greedy() -> "SampleStrategy":
        return SampleStrategy()

    @staticmethod
    def with_temperature(t: float) -> "SampleStrategy":
        return SampleStrategy(1, float(t))

    @staticmethod
    def top_kp(temperature: float, top_k: int = 0, top_p: float = 1.0) -> "SampleStrategy":
        return SampleStrategy(2, float(temperature), int(top_k), float(top_p))

    def _c(self, seed: int) -> _SampleParams:
        return _SampleParams(self.kind, self.temperature, self.top_k, self.top_p, seed)


@dataclass
class GenerationRequest:
    mode: RunMode = RunMode.Hybrid
    prompt: List[int] = field(default_factory=list)
    gen_len: int = 1
    strategy: SampleStrategy = field(default_factory=SampleStrategy.greedy)
    sampler_seed: int = 7
    eos_token: int = -1  # RunMode.DeviceLoop: stop after sampling this id


@dataclass
class Counters:
    dispatches: int = 0
    kernel_launches: int = 0
    fused_blocks: int = 0
    graph_replays: int = 0
    captures: int = 0
    events_recorded: int = 0
    events_waited: int = 0
    graph_kernel_nodes: int = 0


@dataclass
class CacheStats:
    hits: int = 0
    misses: int = 0
    inserts: int = 0
    evictions: int = 0
    releases: int = 0


@dataclass
class GenerationResult:
    tokens: List[int]
    ttft_us: float
    per_token_us: List[float]
    total_us: float
    prefill_us: float
    counters: Counters
    cache_delta: CacheStats
    prefill_paths: List[StepPath]
    decode_paths: List[StepPath]
    captures_completed: int
    cache_released: int
    host_token_us: List[float] = field(default_factory=list)


# ---------------------------------------------------------------------------

class Model:
    """graphrt::Model: weights + KV cache + workspace in one device arena."""

    def __init__(self, cfg: ModelConfig):
        self.cfg = cfg
        h = C.c_void_p()
        c = cfg._c()
        _check(lib().grt_model_create(C.byref(c), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().grt_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tp_info(self):
        """-> (tp_size, tp_rank, symmetric): symmetric = the allreduce buffer is an NCCL symmetric window."""
        a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().grt_model_tp_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, bool(c.value)

    def arena_info(self):
        """-> (capacity, used, allocations) of the model's single device arena."""
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().grt_model_arena_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def upload(self, name: str, array) -> None:
        """Overwrites a weight from a host array in the REFERENCE layout ([k,n])."""
        import numpy as np
        a = np.ascontiguousarray(array)
        if a.dtype == np.float32:
            dt = F32
        elif a.dtype == np.uint16:  # raw bf16 bits
            dt = BF16
        else:
            a = a.astype(np.float32)
            dt = F32
        _check(lib().grt_model_upload(self._h, name.encode(), a.ctypes.data, a.nbytes, dt))

    def download(self, name: str, numel: int):
        import numpy as np
        out = np.zeros(numel, np.float32)
        _check(lib().grt_model_download(self._h, name.encode(), out.ctypes.data_as(C.POINTER(C.c_float)), numel))
        return out

    def load_safetensors(self, path: str, strict: bool = True) -> int:
        """Loads a safetensors checkpoint (file or directory of shards); graphrt or
        HuggingFace LLaMA tensor names.  Returns the number of tensors loaded."""
        n = C.c_int32()
        _check(lib().grt_model_load_safetensors(self._h, str(path).encode(), 1 if strict else 0, C.byref(n)))
        return n.value

    def kv_pages(self):
        """(page_size, n_pages) of the paged KV pool; (0, 0) when contiguous."""
        ps, n = C.c_int32(), C.c_int32()
        _check(lib().grt_model_kv_pages(self._h, C.byref(ps), C.byref(n)))
        return ps.value, n.value

    def set_kv_block_table(self, table) -> None:
        """Logical page i -> physical page table[i] (a permutation of range(n_pages))."""
        arr = (C.c_int32 * max(1, len(table)))(*[int(t) for t in table])
        _check(lib().grt_model_set_kv_block_table(self._h, arr, len(table)))

    def attach_nccl(self, unique_id: bytes) -> None:
        """Joins this rank's model to the NCCL tensor-parallel group (all ranks call it)."""
        _check(lib().grt_model_attach_nccl(self._h, bytes(unique_id), len(unique_id)))

    def weight_bytes(self) -> int:
        v = C.c_uint64()
        _check(lib().grt_model_weight_bytes(self._h, C.byref(v)))
        return v.value

    def decode_bytes(self, length: int) -> int:
        v = C.c_uint64()
        _check(lib().grt_model_decode_bytes(self._h, length, C.byref(v)))
        return v.value


IPC_DESC_BYTES = 3 * 64 + 8 * 8 + 8 * 4  # sizeof(grt_ipc_desc)


class IpcServer:
    """Process B of the two-process split: serves static passes of `session`."""

    def __init__(self, session: "Session", shm_name: str):
        self.desc = C.create_string_buffer(IPC_DESC_BYTES)
        h = C.c_void_p()
        _check(lib().grt_ipc_server_create(session._h, shm_name.encode(), self.desc, C.byref(h)))
        self._h = h
        self.session = session

    def descriptor(self) -> bytes:
        return self.desc.raw

    def serve(self, n_passes: int):
        _check(lib().grt_ipc_server_serve(self._h, int(n_passes)))

    def close(self):
        if getattr(self, "_h", None):
            lib().grt_ipc_server_destroy(self._h)
            self._h = None


class IpcClient:
    """Process A of the two-process split: NVRTC dynamic ops on B's memory."""

    def __init__(self, descriptor: bytes, shm_name: str):
        h = C.c_void_p()
        self._desc = C.create_string_buffer(bytes(descriptor), IPC_DESC_BYTES)
        _check(lib().grt_ipc_client_create(self._desc, shm_name.encode(), C.byref(h)))
        self._h = h

    def generate(self, prompt, gen_len: int, strategy: "SampleStrategy" = None, seed: int = 7):
        import numpy as np
        strategy = strategy or SampleStrategy.greedy()
        pr = (C.c_int32 * len(prompt))(*prompt)
        toks = (C.c_int32 * gen_len)()
        us = (C.c_double * gen_len)()
        sp = strategy._c(seed)
        _check(lib().grt_ipc_client_generate(self._h, pr, len(prompt), gen_len, C.byref(sp), toks, us))
        return list(toks), np.ctypeslib.as_array(us).copy()

    def close(self):
        if getattr(self, "_h", None):
            lib().grt_ipc_client_destroy(self._h)
            self._h = None


def tp_unique_id() -> bytes:
    """NCCL unique id for a tensor-parallel group (rank 0 creates, every rank attaches)."""
    buf = C.create_string_buffer(128)
    _check(lib().grt_tp_unique_id(buf, 128))
    return buf.raw


def tp_emu_threaded(cfg: "ModelConfig", prompt, steps=()):
    """cfg.tp_size ranks as host threads (own model/session/stream) with an
    in-process communicator: batched prefill + single steps; rank 0's logits."""
    import numpy as np
    c = cfg._c()
    pr = (C.c_int32 * len(prompt))(*prompt)
    st = (C.c_int32 * max(1, len(steps)))(*steps)
    out = np.zeros(cfg.vocab_size, np.float32)
    _check(lib().grt_tp_emu_threaded(C.byref(c), pr, len(prompt), st, len(steps),
                                     out.ctypes.data_as(C.POINTER(C.c_float))))
    return out


class TPEmu:
    """Single-device validation of a tensor-parallel model: cfg.tp_size ranks in
    one process, stepped in lockstep with the collectives emulated in-process."""

    def __init__(self, cfg: "ModelConfig"):
        h = C.c_void_p()
        c = cfg._c()
        _check(lib().grt_tp_emu_create(C.byref(c), C.byref(h)))
        self._h = h
        self.vocab = cfg.vocab_size

    def reset(self):
        _check(lib().grt_tp_emu_reset(self._h))

    def step(self, token: int):
        _check(lib().grt_tp_emu_step(self._h, int(token)))

    def prefill(self, tokens):
        for t in tokens:
            self.step(t)

    def logits(self):
        import numpy as np
        out = np.zeros(self.vocab, np.float32)
        _check(lib().grt_tp_emu_logits(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), self.vocab))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().grt_tp_emu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """graphrt::Session (pipeline.hpp:165-189): a model plus its graph cache."""

    def __init__(self, model_cfg, cache_cfg: Optional[CacheConfig] = None):
        self.model = model_cfg if isinstance(model_cfg, Model) else Model(model_cfg)
        self.cache_cfg = cache_cfg or CacheConfig()
        h = C.c_void_p()
        cc = self.cache_cfg._c()
        _check(lib().grt_session_create(self.model._h, C.byref(cc), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().grt_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # Session::run (pipeline.cpp:183-259)
    def run(self, req: GenerationRequest) -> GenerationResult:
        p = len(req.prompt)
        n = max(req.gen_len, 0)
        prompt = (C.c_int32 * max(p, 1))(*req.prompt) if p else (C.c_int32 * 1)()
        r = _Request(int(req.mode), C.cast(prompt, C.POINTER(C.c_int32)), p, req.gen_len,
                     req.strategy._c(req.sampler_seed), 1 if req.eos_token >= 0 else 0,
                     max(int(req.eos_token), 0))
        toks = (C.c_int32 * max(n, 1))()
        gaps = (C.c_double * max(n, 1))()
        pp = (C.c_int32 * max(p, 1))()
        dp = (C.c_int32 * max(n, 1))()
        res = _Result()
        res.tokens = C.cast(toks, C.POINTER(C.c_int32))
        res.per_token_us = C.cast(gaps, C.POINTER(C.c_double))
        res.prefill_paths = C.cast(pp, C.POINTER(C.c_int32))
        res.decode_paths = C.cast(dp, C.POINTER(C.c_int32))
        hts = (C.c_double * max(n, 1))()
        res.host_token_us = C.cast(hts, C.POINTER(C.c_double))
        _check(lib().grt_generate(self._h, C.byref(r), C.byref(res)))
        cn = Counters(*[getattr(res.counters, f) for f, _ in _Counters._fields_])
        cd = CacheStats(*[getattr(res.cache_delta, f) for f, _ in _CacheStats._fields_])
        return GenerationResult(list(toks)[:n], res.ttft_us, list(gaps)[:n], res.total_us, res.prefill_us, cn, cd,
                                [StepPath(x) for x in list(pp)[:p]], [StepPath(x) for x in list(dp)[:n]],
                                res.captures_completed, res.cache_released, list(hts)[:n])

    def cache_stats(self):
        st = _CacheStats()
        size = C.c_uint64()
        _check(lib().grt_cache_stats_get(self._h, C.byref(st), C.byref(size)))
        return CacheStats(*[getattr(st, f) for f, _ in _CacheStats._fields_]), size.value

    def profile_plan(self, key: int, iters: int = 20):
        """Per-kernel average time (ms) and algorithmic bytes of bucket `key`'s plan."""
        cap = 4096
        ms = (C.c_double * cap)()
        by = (C.c_int64 * cap)()
        names = C.create_string_buffer(1 << 16)
        n = C.c_int32()
        _check(lib().grt_profile_plan(self._h, key, iters, ms, by, names, len(names), cap, C.byref(n)))
        nm = names.raw.split(b"\0")
        return [(nm[i].decode(), ms[i], by[i]) for i in range(min(n.value, cap))]

    def trace_pass(self, key: int):
        """Per-CTA %globaltimer stamps of one replay of the static plan: array
        [kernels, OP_TRACE_CTAS * 8] (ns)."""
        import numpy as np
        cap = (5 * self.model.cfg.n_layers + 1) * 8192
        buf = (C.c_uint64 * cap)()
        gr, st = C.c_int32(), C.c_int32()
        _check(lib().grt_trace_pass(self._h, key, buf, cap, C.byref(gr), C.byref(st)))
        return np.ctypeslib.as_array(buf)[: gr.value * st.value].reshape(gr.value, st.value).copy()

    # step-level API (Model::step_math / prefill_math / reset, model.cpp:168-183)
    def reset(self):
        _check(lib().grt_reset(self._h))

    def step(self, token: int):
        _check(lib().grt_step(self._h, int(token)))

    def prefill(self, ids: Sequence[int]):
        arr = (C.c_int32 * max(len(ids), 1))(*ids)
        _check(lib().grt_prefill(self._h, arr, len(ids)))

    @property
    def cur_len(self) -> int:
        v = C.c_int32()
        _check(lib().grt_cur_len(self._h, C.byref(v)))
        return v.value

    def logits(self):
        import numpy as np
        out = np.zeros(self.model.cfg.vocab_size, np.float32)
        _check(lib().grt_get_logits(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), out.size))
        return out

    def kv_row(self, layer: int, slot: int, row: int):
        import numpy as np
        out = np.zeros(self.model.cfg.d_model, np.float32)
        _check(lib().grt_get_kv_row(self._h, layer, slot, row, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def sample(self, strategy: SampleStrategy, seed: int = 0) -> int:
        p = strategy._c(seed)
        t = C.c_int32()
        _check(lib().grt_sample(self._h, C.byref(p), C.byref(t)))
        return t.value

    def sampler_reset(self, seed: int):
        _check(lib().grt_sampler_reset(self._h, seed))

    # explicit capture / replay (exec_graph.hpp:73-141)
    def plan_size(self, key: int) -> int:
        n = C.c_int32()
        _check(lib().grt_plan_size(self._h, int(key), C.byref(n)))
        return n.value

    def begin_capture(self, key: int, fused: bool = False) -> "CaptureSession":
        h = C.c_void_p()
        _check(lib().grt_capture_begin(self._h, int(key), 1 if fused else 0, C.byref(h)))
        return CaptureSession(self, h)

    def replay(self, key: int, token: int, fused: bool = True, validate: bool = True):
        _check(lib().grt_session_replay(self._h, int(key), 1 if fused else 0, int(token), 1 if validate else 0))


class CaptureState(enum.IntEnum):
    Open = 0
    Closed = 1
    Aborted = 2


class CaptureOp(enum.IntEnum):
    Plan = 0
    SamplePreprocess = 1
    Preprocess = 2
    HostToken = 3


class CaptureSession:
    """graphrt::CaptureSession (exec_graph.hpp:73-103) over a Session's engine."""

    def __init__(self, sess: "Session", h):
        self.sess, self._h = sess, h

    def record(self, op: CaptureOp, plan_key: int = 0, index: int = 0):
        _check(lib().grt_capture_record(self._h, int(op), int(plan_key), int(index)))

    def record_plan(self, plan_key: int, index: int):
        self.record(CaptureOp.Plan, plan_key, index)

    def record_external(self, ptr: int, nbytes: int):
        _check(lib().grt_capture_record_external(self._h, C.c_void_p(ptr), nbytes))

    def end_capture(self):
        """-> (kernel_count, capture_epoch)"""
        n, ep = C.c_int32(), C.c_uint64()
        _check(lib().grt_capture_end(self._h, C.byref(n), C.byref(ep)))
        return n.value, ep.value

    @property
    def state(self) -> CaptureState:
        st, rec = C.c_int32(), C.c_int32()
        _check(lib().grt_capture_state_get(self._h, C.byref(st), C.byref(rec)))
        return CaptureState(st.value)

    @property
    def recorded(self) -> int:
        st, rec = C.c_int32(), C.c_int32()
        _check(lib().grt_capture_state_get(self._h, C.byref(st), C.byref(rec)))
        return rec.value

    def close(self):
        if getattr(self, "_h", None):
            lib().grt_capture_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GraphCache:
    """graphrt::GraphCache (graph_cache.hpp:29-81) on placeholder graphs: the
    same C++ policy object each Session uses for its cudaGraphExec_t entries."""

    def __init__(self, capacity: int, policy: EvictionPolicy = EvictionPolicy.LeastUsed):
        h = C.c_void_p()
        _check(lib().grt_graph_cache_create(capacity, int(policy), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().grt_graph_cache_destroy(self._h)
            self._h = None

    def lookup(self, key: int) -> bool:
        v = C.c_int32()
        _check(lib().grt_graph_cache_lookup(self._h, key, C.byref(v)))
        return bool(v.value)

    def insert(self, key: int, graph_key: Optional[int] = None) -> Optional[int]:
        v = C.c_int32()
        _check(lib().grt_graph_cache_insert(self._h, key, key if graph_key is None else graph_key, C.byref(v)))
        return None if v.value == -2 ** 31 else v.value

    def precapture_warmup(self, lo: int, hi: int) -> int:
        v = C.c_int32()
        _check(lib().grt_graph_cache_warmup(self._h, lo, hi, C.byref(v)))
        return v.value

    def begin_session(self):
        _check(lib().grt_graph_cache_begin_session(self._h))

    def release_inactive(self) -> int:
        v = C.c_uint64()
        _check(lib().grt_graph_cache_release_inactive(self._h, C.byref(v)))
        return v.value

    def _query(self, key=0):
        cont, use, size, st = C.c_int32(), C.c_uint64(), C.c_uint64(), _CacheStats()
        _check(lib().grt_graph_cache_query(self._h, key, C.byref(cont), C.byref(use), C.byref(size), C.byref(st)))
        return bool(cont.value), use.value, size.value, CacheStats(*[getattr(st, f) for f, _ in _CacheStats._fields_])

    def contains(self, key: int) -> bool:
        return self._query(key)[0]

    def use_count(self, key: int) -> int:
        if not self.contains(key):
            raise Error(Errc.EmptyCache, f"use_count: no entry for key {key}")
        return self._query(key)[1]

    def size(self) -> int:
        return self._query()[2]

    def stats(self) -> CacheStats:
        return self._query()[3]


def run_inference(model_cfg: ModelConfig, cache_cfg: CacheConfig, req: GenerationRequest) -> GenerationResult:
    """run_inference (pipeline.hpp:186-189): build a session, run once."""
    s = Session(model_cfg, cache_cfg)
    try:
        return s.run(req)
    finally:
        s.close()


# ---------------------------------------------------------------------------
# op-level entry points on device pointers (kernel parity tests)

def op_gemv(w_ptr: int, w_dtype: int, x_ptr: int, out_ptr: int, n: int, k: int, stream: int = 0):
    _check(lib().grt_op_gemv(w_ptr, w_dtype, x_ptr, out_ptr, n, k, stream or None))


def op_prefill_gemm(w_ptr: int, x_ptr: int, out_ptr: int, m_rows: int, k: int, n_tok: int, stream: int = 0):
    """tcgen05 prefill GEMM: out[n_tok, m_rows] = x[n_tok, k] . W[m_rows, k]^T (bf16 in, fp32 out)."""
    _check(lib().grt_op_prefill_gemm(w_ptr, x_ptr, out_ptr, m_rows, k, n_tok, stream or None))


def op_attention(q_ptr, k_ptr, v_ptr, kv_dtype, out_ptr, n_heads, head_dim, max_seq, length, scale, stream=0):
    _check(lib().grt_op_attention(q_ptr, k_ptr, v_ptr, kv_dtype, out_ptr, n_heads, head_dim, max_seq, length,
                                  scale, stream or None))


def op_sample(logits_ptr: int, vocab: int, strategy: SampleStrategy, seed: int, step: int, uniform: float,
              token_ptr: int, stream: int = 0):
    p = strategy._c(seed)
    _check(lib().grt_op_sample(logits_ptr, vocab, C.byref(p), step, uniform, token_ptr, stream or None))


def jit_compile_check(d_model: int, vocab: int, max_seq: int, weight_bf16: bool, arch_ref: bool) -> int:
    n = C.c_uint64()
    _check(lib().grt_jit_compile_check(d_model, vocab, max_seq, int(weight_bf16), int(arch_ref), C.byref(n)))
    return n.value


def device_count() -> int:
    n = C.c_int32()
    _check(lib().grt_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
# checkpoints

def safetensors_list(path: str):
    """[(name, grt dtype or -1, shape tuple)] from a safetensors header (no GPU)."""
    n = C.c_int32()
    _check(lib().grt_safetensors_list(str(path).encode(), None, 0, None, None, 0, C.byref(n)))
    cap = n.value
    names = C.create_string_buffer(max(1, 512 * cap))
    dts = (C.c_int32 * max(1, cap))()
    shp = (C.c_int64 * max(1, 3 * cap))()
    _check(lib().grt_safetensors_list(str(path).encode(), names, len(names), dts, shp, cap, C.byref(n)))
    out, raw = [], names.raw.split(b"\0")
    for i in range(cap):
        rank = shp[3 * i]
        out.append((raw[i].decode(), dts[i], tuple(shp[3 * i + 1: 3 * i + 1 + rank])))
    return out


def hf_tensor_name(hf_name: str):
    """HuggingFace LLaMA name -> (graphrt name or "", stored [out,in])."""
    buf = C.create_string_buffer(256)
    oi = C.c_int32()
    _check(lib().grt_hf_tensor_name(hf_name.encode(), buf, len(buf), C.byref(oi)))
    return buf.value.decode(), bool(oi.value)


def write_safetensors(path: str, tensors, metadata=None) -> None:
    """Minimal safetensors writer (numpy): {name: array}; uint16 arrays are raw
    bf16 bits, float16/float32 as themselves.  Test and tooling helper."""
    import numpy as np
    hdr, blobs, off = {}, [], 0
    for name, a in tensors.items():
        a = np.ascontiguousarray(a)
        dt = {np.dtype(np.uint16): "BF16", np.dtype(np.float16): "F16", np.dtype(np.float32): "F32"}[a.dtype]
        b = a.tobytes()
        hdr[name] = {"dtype": dt, "shape": list(a.shape), "data_offsets": [off, off + len(b)]}
        blobs.append(b)
        off += len(b)
    if metadata:
        hdr["__metadata__"] = metadata
    import json as _json
    h = _json.dumps(hdr).encode()
    h += b" " * ((8 - len(h) % 8) % 8)
    with open(path, "wb") as f:
        f.write(len(h).to_bytes(8, "little"))
        f.write(h)
        for b in blobs:
            f.write(b)

