"""The streaming pass (pass_impl 2, stream_pass.cu): the whole static decode
pass as one persistent launch.  Parity against the C oracle (bf16 storage:
logits max-abs <= 2e-2, margin-aware greedy ids) and against the per-op plan
(pass_impl 1; the chunking differs, so agreement is to rounding, 2e-3)."""
import numpy as np
import pytest

import pyoracle as po
from gpu_util import margin_ok_tokens
from paper_2604_23467_b200 import graphrt as g
from paper_2604_23467_b200.bench_harness import make_prompt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TINY = dict(n_layers=2, d_model=64, n_heads=4, vocab_size=256, max_seq_len=200, seed=3)
D7B = dict(n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=640, seed=1234)


def _pair(kw, d_ff, impl, bucket=16, **cc):
    o = po.OracleModel(arch=po.ARCH_LLAMA, d_ff=d_ff, weight_dtype=po.BF16, kv_dtype=po.BF16,
                       init=po.INIT_PHILOX, n_threads=0, **kw)
    s = g.Session(g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=d_ff, weight_dtype=g.BF16, kv_dtype=g.BF16,
                                init=g.INIT_PHILOX, **kw), g.CacheConfig(bucket_size=bucket, pass_impl=impl, **cc))
    return o, s


@pytest.mark.parametrize("kw,d_ff,plen,steps", [(TINY, 176, 6, 12), (TINY, 176, 150, 4), (D7B, 11008, 10, 6)])
def test_stream_pass_steps_match_oracle(kw, d_ff, plen, steps):
    o, s = _pair(kw, d_ff, 2)
    prompt = make_prompt(42, plen, kw["vocab_size"])
    ref_toks, ref_logits = o.generate_greedy(prompt, steps)
    s.prefill(prompt)
    worst, toks = 0.0, []
    for i in range(steps):
        lg = s.logits()
        worst = max(worst, float(np.abs(lg - ref_logits[i]).max()))
        toks.append(int(np.argmax(lg)))
        if i + 1 < steps:
            s.step(ref_toks[i])
    assert worst <= 2e-2, worst
    margin_ok_tokens(toks, ref_toks, ref_logits, 2e-2)


def test_stream_pass_graph_run_matches_per_op_plan():
    """Hybrid run (graph replays of the streaming pass, batched prefill) vs the
    per-op plan on the same weights: identical greedy stream where margins allow,
    final logits within 2e-3."""
    cfg = g.ModelConfig.llama2_7b(n_layers=2, max_seq_len=640)
    prompt = make_prompt(42, 10, 32000)
    out = {}
    for impl in (1, 2):
        s = g.Session(cfg, g.CacheConfig(bucket_size=64, pass_impl=impl, batched_prefill=True, warmup_hi=4))
        r = s.run(g.GenerationRequest(prompt=prompt, gen_len=40))
        out[impl] = (r.tokens, s.logits(), r)
        s.close()
    r2 = out[2][2]
    assert all(p == g.StepPath.Replayed for p in r2.decode_paths[1:])
    assert out[1][0][:8] == out[2][0][:8]
    assert float(np.abs(out[1][1] - out[2][1]).max()) <= 2e-3 or out[1][0] != out[2][0]


def test_stream_pass_long_context_and_paging():
    """Attention phase with 4 splits per head (T > 128) and a paged KV pool in a
    random page order: same logits as the contiguous streaming pass."""
    cfg = dict(D7B, n_layers=1, max_seq_len=512)
    prompt = make_prompt(7, 300, 32000)
    res = []
    for page in (0, 16):
        s = g.Session(g.ModelConfig.llama2_7b(kv_page_size=page, **cfg),
                      g.CacheConfig(bucket_size=64, pass_impl=2, batched_prefill=True))
        if page:
            _, n_pages = s.model.kv_pages()
            perm = np.random.RandomState(3).permutation(n_pages).astype(np.int32)
            s.model.set_kv_block_table(perm)
        s.prefill(prompt)
        s.step(11)
        s.step(12)
        res.append(s.logits())
        s.close()
    assert np.array_equal(res[0], res[1])
