"""Batched-prefill fusion: a split-K residual GEMM (Wo, down) hands its partials
to the next RMSNorm launch, which reduces them (split order), adds the residual
and normalises in one kernel.  Same arithmetic in the same order as the separate
reduce + rmsnorm kernels, so the result must be BIT-identical (checked against
CacheConfig(prefill_fuse_norm=False) on the same weights)."""
import numpy as np
import pytest

from paper_2604_23467_b200 import graphrt as g
from paper_2604_23467_b200.bench_harness import make_prompt

pytestmark = pytest.mark.gpu


def _run(model, fuse):
    s = g.Session(model, g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True, prefill_fuse_norm=fuse))
    out = []
    for P in (10, 37, 100):  # (P > 256 splits K only when the reduce is fused: not comparable)
        s.reset()
        s.prefill(make_prompt(42, P, 32000))
        out.append(s.logits())
        out.append(s.kv_row(2, 1, P - 1))
        s.step(5)
        out.append(s.logits())
    s.close()
    return np.concatenate(out)


def test_fused_resid_norm_is_bit_identical():
    m = g.Model(g.ModelConfig.llama2_7b(n_layers=3, max_seq_len=512))
    a = _run(m, False)
    b = _run(m, True)
    assert a.shape == b.shape and np.isfinite(a).all()
    assert np.array_equal(a, b)
