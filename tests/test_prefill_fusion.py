"""Batched-prefill fusion: a split-K residual GEMM (Wo, down) hands its partials
to the next RMSNorm launch, which reduces them (split order), adds the residual
and normalises in one kernel.  Same arithmetic in the same order as the separate
reduce + rmsnorm kernels, so the result must be BIT-identical (checked with the
fusion switched off through GRT_PREFILL_FUSE_NORM=0 in a child process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/oracle")
import pyoracle as po
from paper_2604_23467_b200 import graphrt as g
cfg = g.ModelConfig.llama2_7b(n_layers=3, max_seq_len=256)
s = g.Session(cfg, g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True))
out = []
for P in (10, 37, 100):
    s.reset()
    s.prefill(po.make_prompt(42, P, 32000))
    out.append(s.logits())
    out.append(s.kv_row(2, 1, P - 1))
    s.step(5)
    out.append(s.logits())
np.save(sys.argv[2], np.concatenate(out))
"""


def _run(tmp_path, fuse):
    path = str(tmp_path / f"fuse{fuse}.npy")
    env = dict(os.environ, GRT_PREFILL_FUSE_NORM=str(fuse))
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, path], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_fused_resid_norm_is_bit_identical(tmp_path):
    a = _run(tmp_path, 0)
    b = _run(tmp_path, 1)
    assert a.shape == b.shape and np.isfinite(a).all()
    assert np.array_equal(a, b)
