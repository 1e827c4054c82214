"""Pins the C restatement (oracle/) against the reference's own outputs.

The fixtures in tests/golden/ were produced by the unmodified reference library
(tests/golden/make_golden.py); these CPU tests prove the oracle reproduces them
bit for bit before any GPU result is compared against the oracle.
"""
import numpy as np
import pytest

import pyoracle as po


def test_tiny_ref_greedy_matches_reference_bitexact(golden):
    g = golden("tiny_ref_greedy.json")
    # SURVEY Appendix A tokens, produced by the reference binary.
    assert g["prompt"] == [7, 226, 123, 48, 233, 161, 21, 56, 125, 232]
    assert g["tokens"][:8] == [159, 201, 180, 226, 32, 134, 32, 199]
    m = po.OracleModel()
    toks, lg = m.generate_greedy(g["prompt"], len(g["tokens"]))
    assert toks == g["tokens"]
    assert np.array_equal(lg, np.array(g["logits"], np.float32))


def test_tiny_ref_temperature_matches_reference(golden):
    g = golden("tiny_ref_temp08.json")
    m = po.OracleModel()
    assert m.prefill(g["prompt"]) == 0
    rng = po.MtRng(g["sampler_seed"])
    toks = []
    for i, want_logits in enumerate(g["logits"]):
        lg = m.logits()
        assert np.array_equal(lg, np.array(want_logits, np.float32))
        t = po.sample_temperature(lg, g["temperature"], rng)
        toks.append(t)
        m.step(t)
    assert toks == g["tokens"]


def test_bf16_rounded_weights_match_reference(golden):
    g = golden("tiny_ref_bf16w_greedy.json")
    m = po.OracleModel(weight_dtype=po.BF16)
    toks, lg = m.generate_greedy(g["prompt"], len(g["tokens"]))
    assert toks == g["tokens"]
    assert np.array_equal(lg, np.array(g["logits"], np.float32))


def test_model_test_tiny_config(golden):
    g = golden("model_test_tiny.json")
    m = po.OracleModel(n_layers=2, d_model=16, n_heads=2, vocab_size=32, max_seq_len=24, seed=5)
    toks, lg = m.generate_greedy(g["prompt"], len(g["tokens"]))
    assert toks == g["tokens"]
    assert np.array_equal(lg, np.array(g["logits"], np.float32))


def test_wide_config(golden):
    g = golden("wide_ref_greedy.json")
    m = po.OracleModel(n_layers=3, d_model=128, n_heads=8, vocab_size=1000, max_seq_len=160, seed=99,
                       n_threads=4)
    toks, lg = m.generate_greedy(g["prompt"], len(g["tokens"]))
    assert toks == g["tokens"]
    assert np.array_equal(lg, np.array(g["logits"], np.float32))


def test_wide_temperature(golden):
    g = golden("wide_ref_temp07.json")
    m = po.OracleModel(n_layers=3, d_model=128, n_heads=8, vocab_size=1000, max_seq_len=160, seed=99)
    m.prefill(g["prompt"])
    rng = po.MtRng(g["sampler_seed"])
    toks = []
    for _ in g["tokens"]:
        t = po.sample_temperature(m.logits(), g["temperature"], rng)
        toks.append(t)
        m.step(t)
    assert toks == g["tokens"]


def test_all_reference_modes_agree_with_math_path(golden):
    modes = golden("tiny_ref_modes.json")
    toks = {k: v["tokens"] for k, v in modes.items()}
    assert len(set(map(tuple, toks.values()))) == 1
    prompt = modes["eager"]["prompt"]
    m = po.OracleModel()
    mine, _ = m.generate_greedy(prompt, len(toks["eager"]))
    assert mine == toks["eager"]
    # c3 dispatch shape from the reference: hybrid = 2/prefill + 3/decode.
    assert modes["hybrid"]["dispatches"] == 2 * len(prompt) + 3 * 24


def test_kats(golden):
    k = golden("kat.json")
    rng = po.MtRng(1234)
    assert [str(rng.next()) for _ in range(8)] == k["mt19937_64_seed1234_first8"]
    assert po.make_prompt(42, 10, 256) == k["make_prompt_42_10_256"]
    assert po.make_prompt(42, 10, 32000) == k["make_prompt_42_10_32000"]
    for samples, p, want in k["percentile_cases"]:
        assert po.percentile(samples, p) == want


@pytest.mark.parametrize("name", ["llama_tiny_f32", "llama_tiny_bf16", "llama_tiny_philox_bf16"])
def test_llama_oracle_frozen(golden, name):
    g = golden(name + ".json")
    m = po.OracleModel(**g["config"])
    toks, lg = m.generate_greedy(g["prompt"], len(g["tokens"]))
    assert toks == g["tokens"]
    assert np.array_equal(lg, np.array(g["logits"], np.float32))


def test_incremental_equals_restart():
    """model_test.cpp:129-146: a decode step equals prefilling the extended prompt."""
    for kw in [{}, dict(arch=po.ARCH_LLAMA, d_ff=176, weight_dtype=po.BF16, kv_dtype=po.BF16)]:
        a = po.OracleModel(n_layers=2, d_model=16, n_heads=2, vocab_size=32, max_seq_len=24, seed=5, **kw)
        prompt = [3, 1, 4, 1, 5]
        a.prefill(prompt)
        t1 = po.sample_greedy(a.logits())
        a.step(t1)
        b = po.OracleModel(n_layers=2, d_model=16, n_heads=2, vocab_size=32, max_seq_len=24, seed=5, **kw)
        b.prefill(prompt + [t1])
        assert np.array_equal(a.logits(), b.logits())


def test_error_codes():
    m = po.OracleModel(n_layers=2, d_model=16, n_heads=2, vocab_size=32, max_seq_len=24, seed=5)
    assert m.prefill([]) == 8           # EmptyPrompt
    assert m.prefill([1] * 25) == 7     # PromptTooLong
    assert m.step(32) == 2              # TokenOutOfRange
    assert m.prefill([1] * 24) == 0
    assert m.step(1) == 1               # position outside the learned table: ShapeMismatch
    ml = po.OracleModel(arch=po.ARCH_LLAMA, n_layers=1, d_model=16, n_heads=2, vocab_size=32,
                        max_seq_len=4, d_ff=32)
    assert ml.prefill([1] * 4) == 0
    assert ml.step(1) == 4              # CacheFull


def test_greedy_tie_break_and_temperature_uniformity():
    # tensor_kernels_test.cpp:293-314
    assert po.sample_greedy(np.array([0.5, 2.0, -1.0, 2.0, 1.0], np.float32)) == 1
    assert po.sample_greedy(np.zeros(5, np.float32)) == 0
    rng = po.MtRng(123)
    z = np.zeros(8, np.float32)
    hist = np.bincount([po.sample_temperature(z, 1.0, rng) for _ in range(40000)], minlength=8)
    assert np.all(np.abs(hist / 40000 - 1 / 8) < 0.01)


def test_topkp_sampler_properties():
    rs = np.random.RandomState(0)
    lg = rs.randn(1000).astype(np.float32)
    # top_k = 1 is greedy
    for s in range(20):
        assert po.sample_topkp(lg, 0.8, 1, 1.0, 7, s) == po.sample_greedy(lg)
    # tokens stay inside the top-k set
    topk = set(np.argsort(-lg, kind="stable")[:10].tolist())
    for s in range(200):
        assert po.sample_topkp(lg, 1.0, 10, 1.0, 3, s) in topk
    # deterministic given (seed, step)
    a = [po.sample_topkp(lg, 0.9, 0, 0.9, 5, s) for s in range(50)]
    b = [po.sample_topkp(lg, 0.9, 0, 0.9, 5, s) for s in range(50)]
    assert a == b
    # temperature <= 0 is greedy
    assert po.sample_topkp(lg, 0.0, 0, 1.0, 1, 1) == po.sample_greedy(lg)


def test_grt_expf_accuracy():
    for z in np.linspace(-29.9, 0, 2001).astype(np.float32):
        e = po.lib().oc_grt_expf(float(z))
        assert abs(e - np.exp(np.float64(z))) <= 4e-7 * np.exp(np.float64(z)) + 1e-30
