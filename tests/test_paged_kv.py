"""Paged KV cache (the reference cache is contiguous,
kv_cache.hpp:10-14).  With kv_page_size > 0 every layer's K/V is a pool of
[n_pages][h][page][dh] addressed through a device block table; every kernel
that reads or writes the cache (QKV epilogue, decode attention, batched-prefill
GEMM epilogue and flash attention, the L2 prefetch) goes through it.  The arithmetic is unchanged, so a paged model with
ANY page permutation must reproduce the contiguous model bit for bit."""

import numpy as np
import pytest

import pyoracle as po
from paper_2604_23467_b200 import graphrt as g


def test_paged_config_validation_without_gpu():
    with pytest.raises(g.Error) as e:  # validated before any device work
        g.Model(g.ModelConfig(kv_page_size=-1))
    assert e.value.code in (g.Errc.InvalidConfig, g.Errc.NoDevice)


@pytest.mark.gpu
def test_tiny_ref_paged_reproduces_reference(golden):
    gd = golden("tiny_ref_greedy.json")
    m = g.Model(g.ModelConfig(kv_page_size=8))
    ps, n = m.kv_pages()
    assert (ps, n) == (8, 75)
    m.set_kv_block_table(list(reversed(range(n))))
    s = g.Session(m, g.CacheConfig(bucket_size=16))
    r = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=gd["prompt"], gen_len=32))
    assert r.tokens == gd["tokens"]
    r = s.run(g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=gd["prompt"], gen_len=32))
    assert r.tokens == gd["tokens"]
    # step API: logits within the fp32 tolerance of the reference fixture
    s.reset()
    s.prefill(gd["prompt"])
    assert float(np.abs(s.logits() - np.asarray(gd["logits"][0], np.float32)).max()) <= 1e-4


def _llama(page, **kw):
    base = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=256,
                d_ff_=11008, weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX, seed=7, kv_page_size=page)
    base.update(kw)
    return g.Model(g.ModelConfig(**base))


@pytest.mark.gpu
@pytest.mark.parametrize("page,batched", [(16, True), (64, True), (16, False)])
def test_llama_7b_dims_paged_bit_identical_to_contiguous(page, batched):
    rng = np.random.default_rng(page)
    mp = _llama(page)
    _, n = mp.kv_pages()
    mp.set_kv_block_table(rng.permutation(n).tolist())
    sp = g.Session(mp, g.CacheConfig(bucket_size=32, warmup_hi=0, batched_prefill=batched))
    sc = g.Session(_llama(0), g.CacheConfig(bucket_size=32, warmup_hi=0, batched_prefill=batched))
    prompt = po.make_prompt(42, 150, 32000)  # > 128: the tcgen05 prefill attention reads through the page table
    sp.prefill(prompt)
    sc.prefill(prompt)
    assert np.array_equal(sp.logits(), sc.logits())
    for t in (11, 12, 13):
        sp.step(t)
        sc.step(t)
        assert np.array_equal(sp.logits(), sc.logits())
    for row in (0, 33, 152):
        assert np.array_equal(sp.kv_row(1, 0, row), sc.kv_row(1, 0, row))
        assert np.array_equal(sp.kv_row(0, 1, row), sc.kv_row(0, 1, row))
    a = sp.run(g.GenerationRequest(prompt=prompt, gen_len=24))
    b = sc.run(g.GenerationRequest(prompt=prompt, gen_len=24))
    assert a.tokens == b.tokens


@pytest.mark.gpu
def test_paged_errors():
    m = _llama(0, n_layers=1, max_seq_len=64)
    with pytest.raises(g.Error) as e:
        m.set_kv_block_table([0])
    assert e.value.code == g.Errc.InvalidConfig
    m = _llama(16, n_layers=1, max_seq_len=64)
    assert m.kv_pages() == (16, 4)
    for bad in ([0, 1, 2], [0, 1, 2, 2], [0, 1, 2, 4]):
        with pytest.raises(g.Error):
            m.set_kv_block_table(bad)
    with pytest.raises(g.Error) as e:
        g.Session(m, g.CacheConfig(bucket_size=16, pass_impl=0))
    assert e.value.code == g.Errc.Unsupported


@pytest.mark.gpu
def test_paged_tensor_parallel_shards_match_single_gpu():
    """TP ranks (host threads, head-sharded KV pools with their own identity
    block tables) with paging vs the contiguous tp_size=1 model."""
    kw = dict(arch=g.ARCH_LLAMA, init=g.INIT_PHILOX, weight_dtype=g.BF16, kv_dtype=g.BF16, n_layers=2,
              d_model=128, n_heads=4, vocab_size=512, max_seq_len=256, d_ff_=320, seed=5)
    prompt = po.make_prompt(42, 40, 512)
    ref = g.Session(g.ModelConfig(**kw), g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True))
    ref.prefill(prompt)
    for t in (3, 9):
        ref.step(t)
    got = g.tp_emu_threaded(g.ModelConfig(tp_size=2, kv_page_size=16, **kw), prompt, (3, 9))
    assert float(np.abs(ref.logits() - got).max()) <= 2e-3
