"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden fixtures.  Tolerances (stated per test):
  * fp32 weights/KV (ref arch, reference defaults): logits max-abs <= 1e-4 and
    greedy tokens identical for every step (top-2 margin 6.6e-3 >> 1e-4);
  * bf16 weights/KV: logits max-abs <= 2e-2 (north star), greedy ids identical
    wherever the oracle's top-2 margin exceeds 2e-2;
  * samplers: bit-exact token ids given identical logits.
"""
import os

import numpy as np
import pytest

import pyoracle as po
from gpu_util import bf16_bits, bf16_round, margin_ok_tokens
from paper_2604_23467_b200 import graphrt as g

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TINY = dict(n_layers=2, d_model=16, n_heads=2, vocab_size=32, max_seq_len=24, seed=5)  # model_test.cpp:14-23
WIDE = dict(n_layers=3, d_model=128, n_heads=8, vocab_size=1000, max_seq_len=160, seed=99)


def cache(bucket=64, lo=1, hi=50, **kw):
    return g.CacheConfig(bucket_size=bucket, warmup_lo=lo, warmup_hi=hi, **kw)


def step_parity(sess, prompt, n, ref_tokens, ref_logits, tol):
    sess.reset()
    sess.prefill(prompt)
    toks, worst = [], 0.0
    for i in range(n):
        lg = sess.logits()
        worst = max(worst, float(np.abs(lg - np.asarray(ref_logits[i], np.float32)).max()))
        t = int(np.argmax(lg))  # first max = lowest index, as run_sampler
        toks.append(t)
        if i + 1 < n:
            sess.step(ref_tokens[i])  # teacher-force the reference stream
    return toks, worst


# --------------------------------------------------------------------------- ops

@pytest.mark.parametrize("dtype", [g.F32, g.BF16])
@pytest.mark.parametrize("n,k", [(1, 8), (7, 64), (96, 16), (1000, 128), (12288, 4096), (33, 11008), (32000, 4096)])
def test_gemv_matches_fp64(dtype, n, k):
    rs = np.random.RandomState(n + k)
    w = rs.uniform(-0.1, 0.1, (n, k)).astype(np.float32)
    x = rs.randn(k).astype(np.float32)
    if dtype == g.BF16:
        w = bf16_round(w)
        wd = torch.from_numpy(bf16_bits(w).view(np.int16)).cuda()
    else:
        wd = torch.from_numpy(w).cuda()
    xd = torch.from_numpy(x).cuda()
    out = torch.zeros(n, dtype=torch.float32, device="cuda")
    g.op_gemv(wd.data_ptr(), dtype, xd.data_ptr(), out.data_ptr(), n, k)
    torch.cuda.synchronize()
    want = w.astype(np.float64) @ x.astype(np.float64)
    scale = np.abs(w).astype(np.float64) @ np.abs(x).astype(np.float64)
    err = np.abs(out.cpu().numpy() - want) / np.maximum(scale, 1e-30)
    assert err.max() < 1e-5, err.max()


@pytest.mark.parametrize("kvdt", [g.F32, g.BF16])
@pytest.mark.parametrize("h,dh,length", [(2, 8, 1), (4, 16, 5), (4, 16, 42), (32, 128, 1), (32, 128, 10),
                                         (32, 128, 138), (32, 128, 628), (8, 64, 300),
                                         # 4-CTA clusters x 3 and 4 passes: the later passes staged in
                                         # shared memory by the TMA engine
                                         (32, 128, 1500), (32, 128, 2000), (2, 4, 301)])
def test_attention_matches_fp64(kvdt, h, dh, length):
    rs = np.random.RandomState(h * dh + length)
    S = max(length, 8) + 3
    K = rs.randn(h, S, dh).astype(np.float32)
    V = rs.randn(h, S, dh).astype(np.float32)
    q = rs.randn(h * dh).astype(np.float32)
    if kvdt == g.BF16:
        K, V = bf16_round(K), bf16_round(V)
        Kd = torch.from_numpy(bf16_bits(K).view(np.int16)).cuda()
        Vd = torch.from_numpy(bf16_bits(V).view(np.int16)).cuda()
    else:
        Kd, Vd = torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda()
    qd = torch.from_numpy(q).cuda()
    out = torch.zeros(h * dh, dtype=torch.float32, device="cuda")
    scale = float(np.float32(1.0) / np.sqrt(np.float32(dh)))
    g.op_attention(qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), kvdt, out.data_ptr(), h, dh, S, length, scale)
    want = np.zeros((h, dh))
    for hh in range(h):
        s = K[hh, :length].astype(np.float64) @ q[hh * dh:(hh + 1) * dh].astype(np.float64) * scale
        p = np.exp(s - s.max())
        p /= p.sum()
        want[hh] = p @ V[hh, :length].astype(np.float64)
    assert np.abs(out.cpu().numpy().reshape(h, dh) - want).max() < 2e-5


def _logits_dev(lg):
    return torch.from_numpy(np.ascontiguousarray(lg, np.float32)).cuda()


@pytest.mark.parametrize("vocab", [8, 256, 1000, 8195, 32000, 50257])  # ragged vocabulary sizes; > 32768: the 8-bit-pass path
def test_sampler_topkp_bitexact_vs_oracle(vocab):
    rs = np.random.RandomState(vocab)
    tok = torch.zeros(1, dtype=torch.int32, device="cuda")
    cases = [(0.8, 0, 0.9), (1.0, 40, 1.0), (0.7, 50, 0.95), (1.3, 0, 1.0), (0.5, 1, 1.0), (1.0, 0, 0.5)]
    for rep in range(6):
        lg = (rs.randn(vocab) * (0.3 if rep % 2 else 3.0)).astype(np.float32)
        if rep == 5:
            lg[::7] = lg.max()  # ties
        ld = _logits_dev(lg)
        for (t, k, p) in cases:
            for step in (0, 1, 17):
                seed = 1000 * rep + 7
                g.op_sample(ld.data_ptr(), vocab, g.SampleStrategy.top_kp(t, k, p), seed, step, 0.0,
                            tok.data_ptr())
                want = po.sample_topkp(lg, t, k, p, seed, step)
                assert int(tok.item()) == want, (vocab, rep, t, k, p, step)


@pytest.mark.parametrize("vocab", [5, 256, 8195, 32000])
def test_sampler_greedy_and_temperature(vocab):
    rs = np.random.RandomState(3)
    tok = torch.zeros(1, dtype=torch.int32, device="cuda")
    for rep in range(5):
        lg = rs.randn(vocab).astype(np.float32)
        if rep == 1:
            lg[:] = 0.0
        if rep == 2 and vocab > 3:
            lg[1] = lg[3] = lg.max() + 1.0  # tie -> lowest index (tensor_kernels_test.cpp:293-301)
        if rep == 3 and vocab > 8000:
            lg[7999] = lg[4100] = lg.max() + 1.0  # a tie far apart (different threads and warps)
        ld = _logits_dev(lg)
        g.op_sample(ld.data_ptr(), vocab, g.SampleStrategy.greedy(), 0, 0, 0.0, tok.data_ptr())
        assert int(tok.item()) == po.sample_greedy(lg)
        rng = po.MtRng(11 + rep)
        for step in range(8):
            u = rng.uniform01()
            g.op_sample(ld.data_ptr(), vocab, g.SampleStrategy.with_temperature(0.8), 0, step, u, tok.data_ptr())
            # oracle with the same draw
            r2 = po.MtRng(11 + rep)
            for _ in range(step):
                r2.uniform01()
            assert int(tok.item()) == po.sample_temperature(lg, 0.8, r2)


# --------------------------------------------------------------------- models

def test_tiny_ref_fp32_matches_reference_fixture(golden):
    """Reference defaults (tiny-ref): SURVEY Appendix A tokens, logits <= 1e-4."""
    gd = golden("tiny_ref_greedy.json")
    s = g.Session(g.ModelConfig(), cache(bucket=64))
    toks, worst = step_parity(s, gd["prompt"], len(gd["tokens"]), gd["tokens"], gd["logits"], 1e-4)
    assert worst <= 1e-4, worst
    assert toks == gd["tokens"]


@pytest.mark.parametrize("bucket", [1, 64])
def test_all_modes_reproduce_reference_tokens(golden, bucket):
    """c1/c2 (acceptance_main.cpp:77-113): every RunMode yields the reference tokens."""
    gd = golden("tiny_ref_greedy.json")
    s = g.Session(g.ModelConfig(), cache(bucket=bucket, hi=20))
    for mode in g.ALL_MODES:
        r = s.run(g.GenerationRequest(mode=mode, prompt=gd["prompt"], gen_len=32))
        assert r.tokens == gd["tokens"], g.mode_name(mode)


def test_temperature_run_matches_reference(golden):
    gd = golden("tiny_ref_temp08.json")
    s = g.Session(g.ModelConfig(), cache())
    r = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=gd["prompt"], gen_len=32,
                                  strategy=g.SampleStrategy.with_temperature(0.8), sampler_seed=7))
    assert r.tokens == gd["tokens"]


def test_bf16_weights_ref_arch(golden):
    gd = golden("tiny_ref_bf16w_greedy.json")
    s = g.Session(g.ModelConfig(weight_dtype=g.BF16), cache())
    toks, worst = step_parity(s, gd["prompt"], 32, gd["tokens"], gd["logits"], 1e-4)
    assert worst <= 1e-4, worst  # fp32 KV: only accumulation order differs
    assert toks == gd["tokens"]


@pytest.mark.parametrize("name,cfg", [("model_test_tiny.json", TINY), ("wide_ref_greedy.json", WIDE)])
def test_other_ref_configs(golden, name, cfg):
    gd = golden(name)
    s = g.Session(g.ModelConfig(**cfg), cache())
    toks, worst = step_parity(s, gd["prompt"], len(gd["tokens"]), gd["tokens"], gd["logits"], 1e-4)
    assert worst <= 1e-4, worst
    assert toks == gd["tokens"]
    r = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=gd["prompt"], gen_len=len(gd["tokens"])))
    assert r.tokens == gd["tokens"]


def test_wide_temperature(golden):
    gd = golden("wide_ref_temp07.json")
    s = g.Session(g.ModelConfig(**WIDE), cache())
    r = s.run(g.GenerationRequest(prompt=gd["prompt"], gen_len=len(gd["tokens"]),
                                  strategy=g.SampleStrategy.with_temperature(0.7), sampler_seed=11))
    assert r.tokens == gd["tokens"]


@pytest.mark.parametrize("name,tol", [("llama_tiny_f32", 1e-4), ("llama_tiny_bf16", 2e-2),
                                      ("llama_tiny_philox_bf16", 2e-2)])
def test_llama_tiny_vs_oracle(golden, name, tol):
    gd = golden(name + ".json")
    c = gd["config"]
    mc = g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=c["d_ff"], weight_dtype=c.get("weight_dtype", 0),
                       kv_dtype=c.get("kv_dtype", 0), init=c.get("init", 0))
    s = g.Session(mc, cache())
    toks, worst = step_parity(s, gd["prompt"], len(gd["tokens"]), gd["tokens"], gd["logits"], tol)
    assert worst <= tol, worst
    margin_ok_tokens(toks, gd["tokens"], gd["logits"], tol)


def test_llama_7b_dims_two_layers_vs_oracle():
    """LLaMA-2 7B layer shapes (d 4096, ff 11008, V 32000, bf16, Philox init) on
    2 layers against the C oracle: logits max-abs <= 2e-2 after the final norm."""
    kw = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=64,
              d_ff_=11008, init=g.INIT_PHILOX, weight_dtype=g.BF16, kv_dtype=g.BF16, seed=1234)
    o = po.OracleModel(arch=po.ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=64,
                       d_ff=11008, init=po.INIT_PHILOX, weight_dtype=po.BF16, kv_dtype=po.BF16, seed=1234,
                       n_threads=0)
    prompt = po.make_prompt(42, 6, 32000)
    ref_toks, ref_logits = o.generate_greedy(prompt, 4)
    s = g.Session(g.ModelConfig(**kw), cache())
    toks, worst = step_parity(s, prompt, 4, ref_toks, ref_logits, 2e-2)
    assert worst <= 2e-2, worst
    margin_ok_tokens(toks, ref_toks, ref_logits, 2e-2)
    # weights landed in the device layout exactly as the oracle generated them
    for name in ["layers.1.wq", "layers.0.w_up", "layers.1.w_down", "head"]:
        want = o.weight(name)
        got = s.model.download(name, want.size)
        assert np.array_equal(got, want), name


def test_incremental_equals_restart_on_gpu():
    """model_test.cpp:129-146 on the device path (tiny-llama bf16)."""
    mc = g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=176, weight_dtype=g.BF16, kv_dtype=g.BF16, **TINY)
    a = g.Session(mc, cache())
    a.prefill([3, 1, 4, 1, 5])
    t1 = int(np.argmax(a.logits()))
    a.step(t1)
    b = g.Session(g.Model(mc), cache())
    b.prefill([3, 1, 4, 1, 5, t1])
    assert np.array_equal(a.logits(), b.logits())  # deterministic kernels: bit-identical


def test_hybrid_replays_warm_keys_and_captures_the_rest():
    """pipeline_test.cpp:160-206 with exact-length keys (bucket_size 1)."""
    s = g.Session(g.ModelConfig(**TINY), cache(bucket=1, lo=1, hi=6, capacity=64))
    prompt = [(i * 7 + 3) % 32 for i in range(4)]
    r1 = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt, gen_len=4))
    assert r1.prefill_paths.count(g.StepPath.Replayed) == 4
    assert r1.decode_paths == [g.StepPath.Replayed] * 2 + [g.StepPath.EagerFallback] * 2
    assert r1.captures_completed == 2 and r1.counters.captures == 2
    assert (r1.cache_delta.hits, r1.cache_delta.misses, r1.cache_delta.inserts) == (6, 2, 2)
    assert r1.cache_released == 0
    r2 = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt, gen_len=4))
    assert g.StepPath.EagerFallback not in r2.prefill_paths + r2.decode_paths
    assert r2.captures_completed == 0 and r2.cache_delta.hits == 8
    assert r2.counters.kernel_launches == 0  # zero host kernel launches: one graph launch per step
    assert r2.counters.graph_replays == 8
    r3 = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt[:2], gen_len=2))
    assert r3.cache_released == 4
    assert r1.tokens == r2.tokens


# ------------------------------------------------- device-resident decode loop

@pytest.mark.parametrize("bucket", [4, 8, 64])
def test_device_loop_is_one_launch_and_reproduces_reference(golden, bucket):
    """RunMode.DeviceLoop: the whole decode is ONE graph
    launch (WHILE node, bucket SWITCH on the device) and yields the reference
    binary's tokens; small buckets make the loop cross many switch bodies."""
    gd = golden("tiny_ref_greedy.json")
    s = g.Session(g.ModelConfig(), cache(bucket=bucket, hi=50))  # prefill keys warm
    for _ in range(2):  # second run reuses the instantiated loop graph
        r = s.run(g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=gd["prompt"], gen_len=32))
        assert r.tokens == gd["tokens"]
        assert r.counters.kernel_launches == 0
        assert r.decode_paths == [g.StepPath.Replayed] * 32
    h = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=gd["prompt"], gen_len=32))
    assert h.tokens == r.tokens
    assert r.counters.graph_replays == len(gd["prompt"]) + 1  # prefill steps + ONE launch for all 32 decode steps
    assert all(t > 0 for t in r.per_token_us)


def test_device_loop_temperature_and_eos(golden):
    gd = golden("tiny_ref_temp08.json")
    s = g.Session(g.ModelConfig(), cache(bucket=16))
    strat = g.SampleStrategy.with_temperature(0.8)
    r = s.run(g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=gd["prompt"], gen_len=32, strategy=strat,
                                  sampler_seed=7))
    assert r.tokens == gd["tokens"]
    want = gd["tokens"]
    stop = next(i for i in range(3, 32) if want[i] not in want[:i])  # first fresh id from step 3 on
    r = s.run(g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=gd["prompt"], gen_len=32, strategy=strat,
                                  sampler_seed=7, eos_token=want[stop]))
    assert r.tokens[:stop + 1] == want[:stop + 1]
    assert r.tokens[stop + 1:] == [-1] * (31 - stop)
    # the session stays usable after an early stop
    r = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=gd["prompt"], gen_len=32, strategy=strat,
                                  sampler_seed=7))
    assert r.tokens == want


def test_device_loop_topp_paged_matches_hybrid():
    """Seeded top-p (Philox draws indexed by step) through the device loop on a
    paged KV cache: the same tokens as hybrid replay on a contiguous cache."""
    kw = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=128, n_heads=2, vocab_size=512, max_seq_len=256, d_ff_=320,
              weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX, seed=5)
    prompt = po.make_prompt(42, 20, 512)
    strat = g.SampleStrategy.top_kp(0.8, 0, 0.9)
    a = g.Session(g.ModelConfig(**kw), cache(bucket=32, hi=0, batched_prefill=True)).run(
        g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt, gen_len=48, strategy=strat, sampler_seed=11))
    m = g.Model(g.ModelConfig(kv_page_size=16, **kw))
    m.set_kv_block_table(list(reversed(range(m.kv_pages()[1]))))
    b = g.Session(m, cache(bucket=32, hi=0, batched_prefill=True)).run(
        g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=prompt, gen_len=48, strategy=strat, sampler_seed=11))
    assert a.tokens == b.tokens
    assert b.counters.kernel_launches > 0 or b.counters.graph_replays == 1  # one launch for the decode


def test_device_loop_llama_7b_dims_matches_hybrid():
    """2-layer LLaMA at 7B dims (bf16, fused GEMV pairs, cluster attention): the
    device loop crosses three 16-position buckets and matches hybrid replay."""
    kw = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=128,
              d_ff_=11008, weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX, seed=3)
    s = g.Session(g.ModelConfig(**kw), cache(bucket=16, hi=0, batched_prefill=True))
    prompt = po.make_prompt(42, 10, 32000)
    a = s.run(g.GenerationRequest(mode=g.RunMode.Hybrid, prompt=prompt, gen_len=40))
    b = s.run(g.GenerationRequest(mode=g.RunMode.DeviceLoop, prompt=prompt, gen_len=40))
    assert a.tokens == b.tokens
    # the batched prefill (replayed from the prompt-length cache) + ONE launch for all 40 decode steps
    assert b.counters.graph_replays == 2 and b.counters.kernel_launches == 0


def test_long_context_attention_splits():
    """Lengths that need many attention splits (up to max_seq) vs the oracle."""
    kw = dict(n_layers=2, d_model=256, n_heads=2, vocab_size=512, max_seq_len=700, seed=21)
    o = po.OracleModel(arch=po.ARCH_LLAMA, d_ff=512, weight_dtype=po.BF16, kv_dtype=po.BF16, init=po.INIT_PHILOX, **kw)
    prompt = po.make_prompt(9, 650, 512)
    o.prefill(prompt)
    want = o.logits()
    s = g.Session(g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=512, weight_dtype=g.BF16, kv_dtype=g.BF16,
                                init=g.INIT_PHILOX, **kw), cache(bucket=64))
    r = s.run(g.GenerationRequest(prompt=prompt, gen_len=20))
    s.reset()
    s.prefill(prompt)
    assert np.abs(s.logits() - want).max() < 2e-2
    assert len(r.tokens) == 20


def test_request_validation():
    s = g.Session(g.ModelConfig(**TINY), cache(hi=4))
    for req, code in [(g.GenerationRequest(prompt=[], gen_len=1), g.Errc.EmptyPrompt),
                      (g.GenerationRequest(prompt=[1, 2], gen_len=0), g.Errc.InvalidConfig),
                      (g.GenerationRequest(prompt=[1] * 20, gen_len=5), g.Errc.PromptTooLong),
                      (g.GenerationRequest(prompt=[99], gen_len=1), g.Errc.TokenOutOfRange)]:
        with pytest.raises(g.Error) as e:
            s.run(req)
        assert e.value.code == code
    s.run(g.GenerationRequest(prompt=[1] * 20, gen_len=4))  # exactly at the limit


def test_step_api_errors():
    s = g.Session(g.ModelConfig(**TINY), cache())
    with pytest.raises(g.Error) as e:
        s.prefill([])
    assert e.value.code == g.Errc.EmptyPrompt
    with pytest.raises(g.Error) as e:
        s.step(32)
    assert e.value.code == g.Errc.TokenOutOfRange
    s.prefill([1] * 24)
    with pytest.raises(g.Error) as e:
        s.step(1)
    assert e.value.code == g.Errc.ShapeMismatch  # position outside the learned table


# ------------------------------------------------------------ batched prefill

@pytest.mark.parametrize("m,k,p", [(128, 64, 16), (256, 128, 10), (12288, 4096, 10), (4096, 4096, 200),
                                   (22016, 4096, 500), (4096, 11008, 37), (192, 64, 300), (4096, 4096, 512),
                                   (4096, 1376, 37), (4096, 1376, 300), (2752, 4096, 64), (200, 72, 5)])
def test_prefill_gemm_tcgen05_matches_fp64(m, k, p):
    """tcgen05/TMEM GEMM (bf16 operands, fp32 accumulate) vs an fp64 product of
    the same bf16 values; covers split-K (small m), two N tiles (p > 256),
    ragged token counts and partial M tiles."""
    rs = np.random.RandomState(m + k + p)
    w = bf16_round(rs.uniform(-0.1, 0.1, (m, k)).astype(np.float32))
    x = bf16_round(rs.randn(p, k).astype(np.float32))
    wd = torch.from_numpy(bf16_bits(w).view(np.int16)).cuda()
    xd = torch.from_numpy(bf16_bits(x).view(np.int16)).cuda()
    out = torch.full((p, m), float("nan"), dtype=torch.float32, device="cuda")
    g.op_prefill_gemm(wd.data_ptr(), xd.data_ptr(), out.data_ptr(), m, k, p)
    torch.cuda.synchronize()
    want = x.astype(np.float64) @ w.astype(np.float64).T
    scale = np.abs(x).astype(np.float64) @ np.abs(w).astype(np.float64).T
    err = np.abs(out.cpu().numpy() - want) / np.maximum(scale, 1e-30)
    assert np.isfinite(out.cpu().numpy()).all()
    assert err.max() < 1e-5, err.max()


def _llama_pair(kw, prompt_len, batched):
    import pyoracle as po
    o = po.OracleModel(arch=po.ARCH_LLAMA, weight_dtype=po.BF16, kv_dtype=po.BF16, init=po.INIT_PHILOX,
                       d_ff=kw.pop("d_ff"), **kw)
    s = g.Session(g.ModelConfig(arch=g.ARCH_LLAMA, weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX,
                                d_ff_=o.cfg.d_ff, **kw), g.CacheConfig(bucket_size=64, batched_prefill=batched))
    return o, s


@pytest.mark.parametrize("kw,plen", [
    (dict(n_layers=2, d_model=64, n_heads=4, vocab_size=256, max_seq_len=640, seed=3, d_ff=192), 6),
    (dict(n_layers=2, d_model=128, n_heads=2, vocab_size=512, max_seq_len=640, seed=5, d_ff=320), 300),
    (dict(n_layers=2, d_model=128, n_heads=2, vocab_size=512, max_seq_len=640, seed=5, d_ff=320), 600),
])
def test_batched_prefill_matches_oracle(kw, plen):
    """Batched (tcgen05) prefill: last-token logits vs the oracle's token-by-token
    prefill (bf16 activations into the GEMMs; tolerance 2e-2), then decoding
    continues from the handed-off state (incremental == restart, model_test.cpp:129-146)."""
    import pyoracle as po
    o, s = _llama_pair(dict(kw), plen, True)
    prompt = po.make_prompt(42, plen, kw["vocab_size"])
    o.prefill(prompt)
    s.prefill(prompt)
    err = float(np.abs(s.logits() - o.logits()).max())
    assert err <= 2e-2, err
    # two more single-token steps on top of the batched state
    for t in (5, 7):
        o.step(t)
        s.step(t)
        err = float(np.abs(s.logits() - o.logits()).max())
        assert err <= 2e-2, err


@pytest.mark.parametrize("plen", [6, 150, 600])
def test_batched_prefill_reference_arch_matches_oracle(plen):
    """The reference's own architecture (LayerNorm with beta, learned position
    table, ReLU MLP; kernels.cpp:52-85,176-186,238-259) through the batched
    tcgen05 prefill: last-token logits vs the oracle's token-by-token prefill
    (tolerance 2e-2), then two single-token steps on the handed-off state."""
    import pyoracle as po
    kw = dict(n_layers=2, d_model=128, n_heads=2, vocab_size=512, max_seq_len=640, seed=13)
    o = po.OracleModel(arch=po.ARCH_REF, weight_dtype=po.BF16, kv_dtype=po.BF16, init=po.INIT_PHILOX, **kw)
    s = g.Session(g.ModelConfig(arch=g.ARCH_REF, weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX,
                                d_ff_=o.cfg.d_ff, **kw), g.CacheConfig(bucket_size=64, batched_prefill=True))
    prompt = po.make_prompt(42, plen, kw["vocab_size"])
    o.prefill(prompt)
    r = s.run(g.GenerationRequest(prompt=prompt, gen_len=1))
    assert r.prefill_paths == [g.StepPath.Batched] * plen
    s.reset()
    s.prefill(prompt)
    err = float(np.abs(s.logits() - o.logits()).max())
    assert err <= 2e-2, err
    for t in (5, 7):
        o.step(t)
        s.step(t)
        err = float(np.abs(s.logits() - o.logits()).max())
        assert err <= 2e-2, err


def test_batched_prefill_reference_arch_7b_dims_vs_token_by_token():
    """The reference architecture at 7B dims (head_dim 128: the tcgen05 flash
    attention, d_ff 16384 ReLU MLP): batched prefill of 200 tokens vs the
    token-by-token GPU path on the same weights (tolerance 2e-2)."""
    import pyoracle as po
    kw = dict(arch=g.ARCH_REF, n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=256, seed=17,
              weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX)
    prompt = po.make_prompt(42, 200, 32000)
    m = g.Model(g.ModelConfig(**kw))
    a = g.Session(m, g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True))
    a.prefill(prompt)
    la = a.logits()
    a.close()
    b = g.Session(m, g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=False))
    b.prefill(prompt)
    err = float(np.abs(la - b.logits()).max())
    assert np.isfinite(la).all() and err <= 2e-2, err


def test_batched_prefill_run_tokens_match_token_by_token():
    """Session.run with batched prefill reproduces the token-by-token run's greedy
    stream wherever the logit margins allow (same weights, same prompt)."""
    kw = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=128, n_heads=2, vocab_size=512, max_seq_len=256, seed=9,
              d_ff_=320, weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX)
    import pyoracle as po
    prompt = po.make_prompt(42, 40, 512)
    ra = g.Session(g.ModelConfig(**kw), g.CacheConfig(bucket_size=32, batched_prefill=True)).run(
        g.GenerationRequest(prompt=prompt, gen_len=16))
    rb = g.Session(g.ModelConfig(**kw), g.CacheConfig(bucket_size=32, batched_prefill=False)).run(
        g.GenerationRequest(prompt=prompt, gen_len=16))
    assert ra.prefill_paths == [g.StepPath.Batched] * 40
    agree = sum(1 for a, b in zip(ra.tokens, rb.tokens) if a == b)
    assert ra.tokens[:4] == rb.tokens[:4] and agree >= 12, (ra.tokens, rb.tokens)


# ---------------------------------------------------------- tensor parallelism

@pytest.mark.parametrize("tp,kw,tol", [
    (2, dict(n_layers=2, d_model=64, n_heads=4, vocab_size=256, max_seq_len=128, d_ff_=192, seed=3), 1e-4),
    (4, dict(n_layers=2, d_model=64, n_heads=4, vocab_size=256, max_seq_len=128, d_ff_=192, seed=3), 1e-4),
    (8, dict(n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=128, d_ff_=11008, seed=11), 2e-3),
])
def test_tp_sharded_decode_matches_single_gpu(tp, kw, tol):
    """The TP-sharded model (column-parallel QKV/gate-up/head, row-parallel
    Wo/down, head-sharded KV, rank-0 residual rule, allreduce + logits
    allgather) reproduces the tp_size=1 model's logits step by step; ranks run
    in lockstep on one device with the collectives emulated in-process (the
    only difference is the summation order of the row-parallel partials)."""
    base = dict(arch=g.ARCH_LLAMA, init=g.INIT_PHILOX, weight_dtype=g.BF16, kv_dtype=g.BF16, **kw)
    ref = g.Session(g.ModelConfig(**base), g.CacheConfig(bucket_size=64, warmup_hi=0))
    emu = g.TPEmu(g.ModelConfig(tp_size=tp, **base))
    import pyoracle as po
    prompt = po.make_prompt(42, 12, kw["vocab_size"])
    worst = 0.0
    for t in prompt:
        ref.step(t)
        emu.step(t)
        worst = max(worst, float(np.abs(ref.logits() - emu.logits()).max()))
    assert worst <= tol, worst


# ------------------------------------------------------------ two-process split

def _ipc_server_proc(q_desc, q_done, shm, cfg_kw, n_passes):
    from paper_2604_23467_b200 import graphrt as gg
    s = gg.Session(gg.ModelConfig(**cfg_kw), gg.CacheConfig(bucket_size=16, warmup_hi=0))
    sv = gg.IpcServer(s, shm)
    q_desc.put(sv.descriptor())
    for n in n_passes:
        sv.serve(n)
    q_done.get(timeout=120)
    sv.close()


def _ipc_client_proc(q_desc, q_out, shm, prompt, n, kind):
    from paper_2604_23467_b200 import graphrt as gg
    c = gg.IpcClient(q_desc.get(timeout=120), shm)
    strat = gg.SampleStrategy.greedy() if kind == "greedy" else gg.SampleStrategy.with_temperature(0.8)
    runs = []
    for nn in n:  # back-to-back runs: each must start from a clean doorbell/event state
        toks, us = c.generate(prompt, nn, strat, seed=7)
        runs.append(list(toks))
    c.close()
    q_out.put(runs)


@pytest.mark.parametrize("kind,fixture", [("greedy", "tiny_ref_greedy.json"), ("temp", "tiny_ref_temp08.json")])
def test_two_process_ipc_split_reproduces_reference(golden, kind, fixture):
    """Context generator (NVRTC sampler + preprocess) and graph generator (bucket
    graph replay) in two OS processes on one GPU, sharing the arena through
    cudaIpcOpenMemHandle and ordered by interprocess events: the tokens are the
    reference binary's, as in single-process hybrid mode."""
    import multiprocessing as mp
    gold = golden(fixture)
    prompt, want = gold["prompt"], gold["tokens"]
    n = len(want)
    ctx = mp.get_context("spawn")
    q_desc, q_done, q_out = ctx.Queue(), ctx.Queue(), ctx.Queue()
    shm = f"/grt_ipc_test_{os.getpid()}_{kind}"
    gens = [n, 5, n]
    sv = ctx.Process(target=_ipc_server_proc, args=(q_desc, q_done, shm, {}, [len(prompt) + k for k in gens]))
    cl = ctx.Process(target=_ipc_client_proc, args=(q_desc, q_out, shm, prompt, gens, kind))
    sv.start()
    cl.start()
    try:
        runs = q_out.get(timeout=180)
    finally:
        q_done.put(1)
        cl.join(60)
        sv.join(60)
    assert runs == [want, want[:5], want]


@pytest.mark.parametrize("tp,kw,plen,tol", [
    (2, dict(n_layers=2, d_model=128, n_heads=4, vocab_size=512, max_seq_len=640, d_ff_=320, seed=5), 40, 2e-3),
    (8, dict(n_layers=2, d_model=4096, n_heads=32, vocab_size=32000, max_seq_len=640, d_ff_=11008, seed=11), 300,
     5e-3),
])
def test_tp_batched_prefill_and_steps_match_single_gpu(tp, kw, plen, tol):
    """Eager tensor-parallel paths with ranks as host threads (own model, session
    and stream each, in-process communicator): batched prefill (tcgen05 GEMMs on
    the shards, allreduce of the [P, d] residual, logits allgather; d_ff/8 = 1376
    exercises the ragged-K GEMM) then two steps, vs the tp_size=1 model."""
    base = dict(arch=g.ARCH_LLAMA, init=g.INIT_PHILOX, weight_dtype=g.BF16, kv_dtype=g.BF16, **kw)
    import pyoracle as po
    prompt = po.make_prompt(42, plen, kw["vocab_size"])
    ref = g.Session(g.ModelConfig(**base), g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True))
    ref.prefill(prompt)
    for t in (3, 9):
        ref.step(t)
    got = g.tp_emu_threaded(g.ModelConfig(tp_size=tp, **base), prompt, (3, 9))
    err = float(np.abs(ref.logits() - got).max())
    assert err <= tol, err


@pytest.mark.parametrize("mode", [g.RunMode.Hybrid, g.RunMode.AblateAsync])
def test_batched_prefill_is_captured_per_prompt_length(mode):
    """The TTFT path through the graph cache (pipeline.cpp:207-214,
    prefill_uses_graphs): the first request of a prompt length runs the batched
    prefill eagerly and captures it (async on the capture thread in hybrid,
    inline for ablate_async); the next request of that length replays it as ONE
    graph launch with identical results.  Eager mode never uses graphs."""
    kw = dict(arch=g.ARCH_LLAMA, n_layers=2, d_model=128, n_heads=2, vocab_size=512, max_seq_len=256, seed=9,
              d_ff_=320, weight_dtype=g.BF16, kv_dtype=g.BF16, init=g.INIT_PHILOX)
    from paper_2604_23467_b200.bench_harness import make_prompt
    prompt = make_prompt(42, 37, 512)
    s = g.Session(g.ModelConfig(**kw), g.CacheConfig(bucket_size=32, batched_prefill=True))
    r1 = s.run(g.GenerationRequest(mode=mode, prompt=prompt, gen_len=8))
    assert r1.prefill_paths == [g.StepPath.Batched] * 37
    r2 = s.run(g.GenerationRequest(mode=mode, prompt=prompt, gen_len=8))
    assert r2.prefill_paths == [g.StepPath.BatchedReplayed] * 37
    assert r2.tokens == r1.tokens
    # one graph launch for the whole prompt + one per decode step
    assert r2.counters.graph_replays == 1 + 8
    lg2 = s.logits()
    # another prompt length misses, the first length still replays
    r3 = s.run(g.GenerationRequest(mode=mode, prompt=prompt[:20], gen_len=4))
    assert r3.prefill_paths == [g.StepPath.Batched] * 20
    e = g.Session(s.model, g.CacheConfig(bucket_size=32, batched_prefill=True))
    re = e.run(g.GenerationRequest(mode=g.RunMode.Eager, prompt=prompt, gen_len=8))
    re2 = e.run(g.GenerationRequest(mode=g.RunMode.Eager, prompt=prompt, gen_len=8))
    assert re2.prefill_paths == [g.StepPath.Batched] * 37 and re2.tokens == r1.tokens
    assert np.array_equal(e.logits(), lg2)
