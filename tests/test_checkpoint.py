"""Safetensors checkpoint loader (no reference counterpart --
the reference only draws seeded weights, init_model model.cpp:30-76).

CPU: header parsing, HuggingFace name mapping, loud failures on corrupt files.
GPU: a HuggingFace-named LLaMA checkpoint ([out,in] nn.Linear layout, bf16/f16)
of the oracle's weights loads into a model created with init=NONE and then
reproduces the oracle's logits (same tolerance as the Philox-initialised model,
tests/test_gpu_parity.py); a graphrt-named dump round-trips bit for bit.
"""
import os

import numpy as np
import pytest

from gpu_util import bf16_bits
from paper_2604_23467_b200 import graphrt as g

LLAMA_KW = dict(n_layers=2, d_model=64, n_heads=4, vocab_size=256, max_seq_len=64, seed=3)
D_FF = 176


def hf_names(n_layers):
    names = ["model.embed_tokens.weight", "model.norm.weight", "lm_head.weight"]
    for l in range(n_layers):
        p = f"model.layers.{l}."
        names += [p + s for s in ("self_attn.q_proj.weight", "self_attn.k_proj.weight", "self_attn.v_proj.weight",
                                  "self_attn.o_proj.weight", "mlp.gate_proj.weight", "mlp.up_proj.weight",
                                  "mlp.down_proj.weight", "input_layernorm.weight",
                                  "post_attention_layernorm.weight")]
    return names


# ------------------------------------------------------------------- CPU only

def test_hf_name_mapping():
    assert g.hf_tensor_name("model.embed_tokens.weight") == ("embedding", False)
    assert g.hf_tensor_name("lm_head.weight") == ("head", True)
    assert g.hf_tensor_name("model.norm.weight") == ("lnf_gamma", False)
    assert g.hf_tensor_name("model.layers.31.self_attn.q_proj.weight") == ("layers.31.wq", True)
    assert g.hf_tensor_name("model.layers.0.mlp.down_proj.weight") == ("layers.0.w_down", True)
    assert g.hf_tensor_name("model.layers.7.post_attention_layernorm.weight") == ("layers.7.ln2_gamma", False)
    assert g.hf_tensor_name("model.layers.0.self_attn.rotary_emb.inv_freq")[0] == ""
    assert g.hf_tensor_name("model.layers.x.mlp.up_proj.weight")[0] == ""
    assert len({g.hf_tensor_name(n)[0] for n in hf_names(4)}) == 3 + 9 * 4


def test_safetensors_header_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    t = {"a.weight": rng.standard_normal((3, 5)).astype(np.float32),
         "b": rng.standard_normal(7).astype(np.float16),
         "c.bf16": bf16_bits(rng.standard_normal((4, 2)).astype(np.float32))}
    path = tmp_path / "x.safetensors"
    g.write_safetensors(str(path), t, metadata={"format": "pt"})
    got = g.safetensors_list(str(path))
    assert got == [("a.weight", g.F32, (3, 5)), ("b", g.F16, (7,)), ("c.bf16", g.BF16, (4, 2))]


@pytest.mark.parametrize("corrupt", ["short", "hdr_len", "bad_json", "offsets"])
def test_corrupt_checkpoints_fail_loudly(tmp_path, corrupt):
    path = tmp_path / "bad.safetensors"
    g.write_safetensors(str(path), {"w": np.ones((2, 2), np.float32)})
    raw = bytearray(path.read_bytes())
    if corrupt == "short":
        raw = raw[:5]
    elif corrupt == "hdr_len":
        raw[0:8] = (1 << 40).to_bytes(8, "little")
    elif corrupt == "bad_json":
        raw[8] = ord("[")
    else:  # data block shorter than the offsets claim
        raw = raw[:-4]
    path.write_bytes(bytes(raw))
    with pytest.raises(g.Error) as e:
        g.safetensors_list(str(path))
    assert e.value.code == g.Errc.IoError
    with pytest.raises(g.Error) as e:
        g.safetensors_list(str(tmp_path / "missing.safetensors"))
    assert e.value.code == g.Errc.IoError


# ------------------------------------------------------------------------ GPU

def _oracle():
    import pyoracle as po
    return po.OracleModel(arch=po.ARCH_LLAMA, d_ff=D_FF, weight_dtype=po.BF16, kv_dtype=po.BF16,
                          init=po.INIT_PHILOX, **LLAMA_KW)


def _hf_checkpoint(o, fmt):
    """The oracle's (bf16-valued) weights under HuggingFace names/layouts."""
    d, V, ff = LLAMA_KW["d_model"], LLAMA_KW["vocab_size"], D_FF

    def enc(a, norm=False):
        a = np.asarray(a, np.float32)
        if norm and fmt != "f16":  # norm gains are fp32 in the arena
            return a
        return bf16_bits(a) if fmt == "bf16" else a.astype(np.float16) if fmt == "f16" else a

    t = {"model.embed_tokens.weight": enc(o.weight("embedding").reshape(V, d)),
         "model.norm.weight": enc(o.weight("lnf_gamma"), True),
         "lm_head.weight": enc(o.weight("head").reshape(d, V).T)}
    for l in range(LLAMA_KW["n_layers"]):
        p, q = f"model.layers.{l}.", f"layers.{l}."
        for hf, ours, k, n in (("self_attn.q_proj", "wq", d, d), ("self_attn.k_proj", "wk", d, d),
                               ("self_attn.v_proj", "wv", d, d), ("self_attn.o_proj", "wo", d, d),
                               ("mlp.gate_proj", "w_gate", d, ff), ("mlp.up_proj", "w_up", d, ff),
                               ("mlp.down_proj", "w_down", ff, d)):
            t[p + hf + ".weight"] = enc(o.weight(q + ours).reshape(k, n).T)
        t[p + "input_layernorm.weight"] = enc(o.weight(q + "ln1_gamma"), True)
        t[p + "post_attention_layernorm.weight"] = enc(o.weight(q + "ln2_gamma"), True)
    t["model.layers.0.self_attn.rotary_emb.inv_freq"] = np.ones(8, np.float32)  # ignored, as in HF dumps
    return t


def _empty_model():
    return g.Model(g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=D_FF, weight_dtype=g.BF16, kv_dtype=g.BF16,
                                 init=g.INIT_NONE, **LLAMA_KW))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt,sharded", [("bf16", False), ("bf16", True), ("f32", False)])
def test_hf_checkpoint_reproduces_oracle(tmp_path, fmt, sharded):
    import pyoracle as po
    o = _oracle()
    t = _hf_checkpoint(o, fmt)
    if sharded:  # HF-style directory of shards
        names = sorted(t)
        g.write_safetensors(str(tmp_path / "model-00001-of-00002.safetensors"), {n: t[n] for n in names[::2]})
        g.write_safetensors(str(tmp_path / "model-00002-of-00002.safetensors"), {n: t[n] for n in names[1::2]})
        path = str(tmp_path)
    else:
        path = str(tmp_path / "model.safetensors")
        g.write_safetensors(path, t)
    m = _empty_model()
    assert m.load_safetensors(path) == 3 + 9 * LLAMA_KW["n_layers"]
    s = g.Session(m, g.CacheConfig(bucket_size=16))
    prompt = po.make_prompt(42, 6, LLAMA_KW["vocab_size"])
    o.prefill(prompt)
    s.prefill(prompt)
    err = float(np.abs(s.logits() - o.logits()).max())
    assert err <= 2e-2, err
    # identical to the Philox-initialised model bit for bit (same bf16 weights)
    ref = g.Session(g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=D_FF, weight_dtype=g.BF16, kv_dtype=g.BF16,
                                  init=g.INIT_PHILOX, **LLAMA_KW), g.CacheConfig(bucket_size=16))
    ref.prefill(prompt)
    assert np.array_equal(ref.logits(), s.logits())


@pytest.mark.gpu
def test_f16_checkpoint_loads_within_rounding(tmp_path):
    o = _oracle()
    path = str(tmp_path / "m.safetensors")
    g.write_safetensors(path, _hf_checkpoint(o, "f16"))
    m = _empty_model()
    m.load_safetensors(path)
    w = m.download("layers.1.w_down", D_FF * LLAMA_KW["d_model"])
    ref = o.weight("layers.1.w_down")
    assert np.abs(w - ref).max() <= 2 ** -9 * np.abs(ref).max()  # f16 -> bf16 double rounding


@pytest.mark.gpu
def test_graphrt_named_dump_round_trips(tmp_path):
    src = g.Model(g.ModelConfig(arch=g.ARCH_LLAMA, d_ff_=D_FF, weight_dtype=g.BF16, kv_dtype=g.BF16,
                                init=g.INIT_PHILOX, **LLAMA_KW))
    o = _oracle()
    names = ["embedding", "lnf_gamma", "head"] + [f"layers.{l}.{n}" for l in range(LLAMA_KW["n_layers"])
                                                   for n in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down",
                                                             "ln1_gamma", "ln2_gamma")]
    d, V, ff = LLAMA_KW["d_model"], LLAMA_KW["vocab_size"], D_FF
    shape = {"embedding": (V, d), "head": (d, V), "wq": (d, d), "wk": (d, d), "wv": (d, d), "wo": (d, d),
             "w_gate": (d, ff), "w_up": (d, ff), "w_down": (ff, d)}
    t = {}
    for n in names:
        a = src.download(n, o.weight(n).size)
        t[n] = a if "gamma" in n else bf16_bits(a).reshape(shape[n.split(".")[-1]])  # reference [k,n] layout
    path = str(tmp_path / "dump.safetensors")
    g.write_safetensors(path, t)
    m = _empty_model()
    assert m.load_safetensors(path) == len(names)
    for n in names:
        assert np.array_equal(m.download(n, o.weight(n).size), src.download(n, o.weight(n).size)), n


@pytest.mark.gpu
def test_strict_loading_errors(tmp_path):
    o = _oracle()
    t = _hf_checkpoint(o, "bf16")
    del t["model.layers.1.mlp.up_proj.weight"]
    path = str(tmp_path / "partial.safetensors")
    g.write_safetensors(path, t)
    with pytest.raises(g.Error) as e:
        _empty_model().load_safetensors(path)
    assert e.value.code == g.Errc.ShapeMismatch and "layers.1.w_up" in str(e.value)
    assert _empty_model().load_safetensors(path, strict=False) == 3 + 9 * 2 - 1
    # wrong shape (a transposed [in,out] matrix under an HF name)
    t = _hf_checkpoint(o, "bf16")
    t["model.layers.0.mlp.gate_proj.weight"] = np.ascontiguousarray(t["model.layers.0.mlp.gate_proj.weight"].T)
    g.write_safetensors(path, t)
    with pytest.raises(g.Error) as e:
        _empty_model().load_safetensors(path)
    assert e.value.code == g.Errc.ShapeMismatch
    # a layer the configuration does not have
    t = _hf_checkpoint(o, "bf16")
    t["model.layers.5.input_layernorm.weight"] = t["model.norm.weight"]
    g.write_safetensors(path, t)
    with pytest.raises(g.Error) as e:
        _empty_model().load_safetensors(path)
    assert e.value.code == g.Errc.ShapeMismatch
