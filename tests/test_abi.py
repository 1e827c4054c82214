"""The C-ABI boundary: the library builds for sm_100a, loads without a GPU,
exports every entry point include/grt/c_api.h declares, and fails loudly
(NoDevice) instead of falling back to the CPU."""
import os
import re
import subprocess

import pytest

from paper_2604_23467_b200 import graphrt as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "grt", "c_api.h")).read()
    return sorted(set(re.findall(r"^\s*(?:grt_status|void|const char\*|int32_t)\s+(grt_[a-z0-9_]+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", g.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (grt_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(g.EXPORTS) == syms  # the ctypes view binds exactly the declared ABI


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", g.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", g.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # cp.async.bulk (TMA engine) weight staging
    assert "SYNCS.PHASECHK" in sass  # mbarrier waits


def test_status_names_follow_reference_errc_order():
    L = g.lib()
    # error.hpp:10-39 declaration order
    names = ["Ok", "ShapeMismatch", "TokenOutOfRange", "EmptyCache", "CacheFull", "InvalidConfig",
             "LengthOutOfRange", "PromptTooLong", "EmptyPrompt", "CaptureInProgress", "CaptureViolation",
             "ForeignBuffer", "SessionClosed", "EmptyCapture", "ReplayShapeError", "WrongLength", "KeyMismatch",
             "WarmupExceedsCapacity", "StaticInFusedBlock", "DeviceStopped", "UnknownEvent", "EmptySamples",
             "IoError"]
    for i, n in enumerate(names):
        assert L.grt_status_name(i).decode() == n
        assert g.Errc(i).name == n
    assert L.grt_abi_version() == 2


@pytest.mark.parametrize("shape", [(64, 256, 600, 0, 1), (16, 32, 24, 0, 1), (4096, 32000, 640, 1, 0),
                                   (128, 1000, 160, 1, 0)])
def test_nvrtc_dynamic_ops_compile_for_sm100a(shape):
    """The JIT context path (preprocess + sampler) compiles for every shape."""
    assert g.jit_compile_check(*shape) > 10000


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(g.Error) as e:
        g.Model(g.ModelConfig())
    assert e.value.code == g.Errc.NoDevice


def test_mode_names_round_trip():
    # pipeline_test.cpp:87-91
    for m in g.ALL_MODES:
        assert g.mode_from_name(g.mode_name(m)) == m
    assert g.mode_name(g.RunMode.Hybrid) == "hybrid"
    with pytest.raises(g.Error) as e:
        g.mode_from_name("turbo")
    assert e.value.code == g.Errc.InvalidConfig


def test_header_is_plain_c_and_links(tmp_path):
    """include/grt/c_api.h is a C99 header (no C++ or torch types) and a C program
    links against the shared library and calls the GPU-free entry points."""
    src = tmp_path / "probe.c"
    src.write_text(
        '#include <stdio.h>\n#include "grt/c_api.h"\n'
        "int main(void) {\n"
        "  grt_model_config c; grt_cache_config cc; grt_generation_request r = {0};\n"
        "  grt_model_config_default(&c); grt_cache_config_default(&cc); (void)r;\n"
        "  int32_t out_in = 0; char name[64];\n"
        '  if (grt_hf_tensor_name("lm_head.weight", name, 64, &out_in) != GRT_OK) return 2;\n'
        '  printf("%d %s %s %d %d\\n", grt_abi_version(), grt_status_name(GRT_CacheFull), name, out_in,\n'
        "         c.kv_page_size);\n"
        "  return 0;\n}\n")
    exe = tmp_path / "probe"
    libdir = os.path.dirname(g.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L" + libdir, "-lgraphrt_b200", "-Wl,-rpath," + libdir], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out == [str(g.lib().grt_abi_version()), "CacheFull", "head", "1", "0"]
