"""ctypes view of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this
module.  It is the checker: the CUDA product path never routes through it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REFDUMP = os.path.join(HERE, "_ref", "refdump")

ARCH_REF, ARCH_LLAMA = 0, 1
INIT_MT19937, INIT_PHILOX = 0, 1
F32, BF16 = 0, 1


class OcConfig(C.Structure):
    _fields_ = [
        ("arch", C.c_int),
        ("n_layers", C.c_int),
        ("d_model", C.c_int),
        ("n_heads", C.c_int),
        ("vocab_size", C.c_int),
        ("max_seq_len", C.c_int),
        ("d_ff", C.c_int),
        ("norm_eps", C.c_float),
        ("seed", C.c_uint64),
        ("init", C.c_int),
        ("weight_dtype", C.c_int),
        ("kv_dtype", C.c_int),
        ("rope_theta", C.c_float),
        ("n_threads", C.c_int),
    ]


class OcMt64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int)]


_lib = None


def build():
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.oc_config_default.argtypes = [C.POINTER(OcConfig)]
        L.oc_create.argtypes = [C.POINTER(OcConfig), C.POINTER(C.c_void_p)]
        L.oc_create.restype = C.c_int
        L.oc_destroy.argtypes = [C.c_void_p]
        L.oc_reset.argtypes = [C.c_void_p]
        L.oc_cur_len.argtypes = [C.c_void_p]
        L.oc_step.argtypes = [C.c_void_p, C.c_int]
        L.oc_prefill.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int]
        L.oc_logits.argtypes = [C.c_void_p]
        L.oc_logits.restype = C.POINTER(C.c_float)
        L.oc_x.argtypes = [C.c_void_p]
        L.oc_x.restype = C.POINTER(C.c_float)
        L.oc_kv_row.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.oc_weight_numel.argtypes = [C.c_void_p, C.c_char_p]
        L.oc_weight_numel.restype = C.c_int64
        L.oc_weight_copy.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_float), C.c_int64]
        L.oc_sample_greedy.argtypes = [C.POINTER(C.c_float), C.c_int]
        L.oc_sample_temperature.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_double, C.POINTER(OcMt64)]
        L.oc_sample_topkp.argtypes = [C.POINTER(C.c_float), C.c_int, C.c_float, C.c_int, C.c_float,
                                      C.c_uint64, C.c_uint64]
        L.oc_sampler_draw53.argtypes = [C.c_uint64, C.c_uint64]
        L.oc_sampler_draw53.restype = C.c_uint64
        L.oc_mt64_seed.argtypes = [C.POINTER(OcMt64), C.c_uint64]
        L.oc_mt64_next.argtypes = [C.POINTER(OcMt64)]
        L.oc_mt64_next.restype = C.c_uint64
        L.oc_uniform01.argtypes = [C.POINTER(OcMt64)]
        L.oc_uniform01.restype = C.c_double
        L.oc_philox_weight.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float]
        L.oc_philox_weight.restype = C.c_float
        L.oc_grt_expf.argtypes = [C.c_float]
        L.oc_grt_expf.restype = C.c_float
        L.oc_round_bf16.argtypes = [C.c_float]
        L.oc_round_bf16.restype = C.c_float
        L.oc_make_prompt.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.oc_percentile.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_double]
        L.oc_percentile.restype = C.c_double
        L.oc_rope_table.argtypes = [C.c_int, C.c_int, C.c_float, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        _lib = L
    return _lib


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def config(**kw) -> OcConfig:
    c = OcConfig()
    lib().oc_config_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class OracleModel:
    """Model::step_math / prefill_math restated (model.cpp:168-183)."""

    def __init__(self, **kw):
        self.cfg = config(**kw)
        h = C.c_void_p()
        rc = lib().oc_create(C.byref(self.cfg), C.byref(h))
        if rc:
            raise ValueError(f"oc_create failed rc={rc}")
        self.h = h
        self.vocab = self.cfg.vocab_size

    def __del__(self):
        if getattr(self, "h", None):
            lib().oc_destroy(self.h)
            self.h = None

    def reset(self):
        lib().oc_reset(self.h)

    @property
    def cur_len(self):
        return lib().oc_cur_len(self.h)

    def step(self, tok: int) -> int:
        return lib().oc_step(self.h, int(tok))

    def prefill(self, toks) -> int:
        arr = (C.c_int * len(toks))(*toks)
        return lib().oc_prefill(self.h, arr, len(toks))

    def logits(self) -> np.ndarray:
        return np.ctypeslib.as_array(lib().oc_logits(self.h), shape=(self.vocab,)).copy()

    def x(self) -> np.ndarray:
        return np.ctypeslib.as_array(lib().oc_x(self.h), shape=(self.cfg.d_model,)).copy()

    def kv_row(self, layer, slot, row) -> np.ndarray:
        out = np.zeros(self.cfg.d_model, np.float32)
        rc = lib().oc_kv_row(self.h, layer, slot, row, _fp(out))
        if rc:
            raise ValueError(rc)
        return out

    def weight(self, name: str) -> np.ndarray:
        n = lib().oc_weight_numel(self.h, name.encode())
        if n < 0:
            raise KeyError(name)
        out = np.zeros(n, np.float32)
        lib().oc_weight_copy(self.h, name.encode(), _fp(out), n)
        return out

    def generate_greedy(self, prompt, gen):
        """prefill_math, then sample/step like pipeline_test.cpp:140-158."""
        rc = self.prefill(prompt)
        if rc:
            raise ValueError(rc)
        toks, logits = [], []
        for i in range(gen):
            lg = self.logits()
            logits.append(lg)
            t = sample_greedy(lg)
            toks.append(t)
            if i + 1 < gen:
                rc = self.step(t)
                if rc:
                    raise ValueError(rc)
        return toks, np.stack(logits)


def sample_greedy(logits) -> int:
    a = np.ascontiguousarray(logits, np.float32)
    return lib().oc_sample_greedy(_fp(a), a.size)


class MtRng:
    def __init__(self, seed):
        self.s = OcMt64()
        lib().oc_mt64_seed(C.byref(self.s), seed)

    def next(self):
        return lib().oc_mt64_next(C.byref(self.s))

    def uniform01(self):
        return lib().oc_uniform01(C.byref(self.s))


def sample_temperature(logits, t, rng: MtRng) -> int:
    a = np.ascontiguousarray(logits, np.float32)
    return lib().oc_sample_temperature(_fp(a), a.size, t, C.byref(rng.s))


def sample_topkp(logits, temperature, top_k, top_p, seed, step) -> int:
    a = np.ascontiguousarray(logits, np.float32)
    return lib().oc_sample_topkp(_fp(a), a.size, temperature, top_k, top_p, seed, step)


def make_prompt(base_seed, n, vocab):
    out = (C.c_int * n)()
    lib().oc_make_prompt(base_seed, n, vocab, out)
    return list(out)


def percentile(samples, p):
    a = np.ascontiguousarray(samples, np.float64)
    return lib().oc_percentile(a.ctypes.data_as(C.POINTER(C.c_double)), a.size, p)


def rope_table(max_seq, head_dim, theta):
    half = head_dim // 2
    c = np.zeros(max_seq * half, np.float32)
    s = np.zeros(max_seq * half, np.float32)
    lib().oc_rope_table(max_seq, head_dim, theta, _fp(c), _fp(s))
    return c.reshape(max_seq, half), s.reshape(max_seq, half)


def refdump(*args) -> dict:
    """Run the reference library (oracle/_ref/refdump) and parse its JSON."""
    import json
    if not os.path.exists(REFDUMP):
        raise FileNotFoundError(REFDUMP)
    out = subprocess.run([REFDUMP] + [str(a) for a in args], check=True, capture_output=True, text=True)
    return json.loads(out.stdout)
