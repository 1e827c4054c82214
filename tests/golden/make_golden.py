"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE LIBRARY.

Run in the build container (needs /root/reference, which the GPU box does not
have):  python tests/golden/make_golden.py

Every fixture except the llama_* ones is the output of the unmodified reference
(graphrt core compiled from /root/reference/proj/core/src by oracle/Makefile,
driven through its public API by oracle/refdump.cpp).  The llama_* fixtures come
from the C restatement itself (the reference cannot express RMSNorm/RoPE/SwiGLU,
SURVEY §0 F3); they freeze the oracle's LLaMA output so drift is caught.
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402

subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def strip(obj):
    if isinstance(obj, dict):
        return {k: strip(v) for k, v in obj.items() if k not in ("init_ms", "prefill_ms", "pass_ms")}
    return obj


def save(name, obj):
    obj = strip(obj)
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print("wrote", name)


def ref(*args):
    return po.refdump(*args)


# 1. Reference defaults (tiny-ref), SURVEY Appendix A.
save("tiny_ref_greedy.json", ref("--gen", 32))
save("tiny_ref_temp08.json", ref("--gen", 32, "--temperature", 0.8, "--sampler-seed", 7))
save("tiny_ref_bf16w_greedy.json", ref("--gen", 32, "--round-bf16"))
# 2. model_test.cpp tiny() config (L2 d16 h2 V32 S24 seed 5).
tiny = ["--layers", 2, "--d", 16, "--heads", 2, "--vocab", 32, "--max-seq", 24, "--seed", 5]
save("model_test_tiny.json", ref(*tiny, "--prompt", "3,1,4,1,5", "--gen", 12))
# 3. A wider config (more heads, larger vocab, longer context).
wide = ["--layers", 3, "--d", 128, "--heads", 8, "--vocab", 1000, "--max-seq", 160, "--seed", 99]
save("wide_ref_greedy.json", ref(*wide, "--prompt-len", 37, "--prompt-seed", 5, "--gen", 20))
save("wide_ref_temp07.json", ref(*wide, "--prompt-len", 9, "--prompt-seed", 6, "--gen", 20,
                                 "--temperature", 0.7, "--sampler-seed", 11, "--dump-logits", 0))
# 4. Every RunMode through Session::run (tokens must agree, pipeline_test.cpp:108-123).
modes = {}
for m in ["eager", "hybrid", "graph_only", "ablate_async", "ablate_fused", "ablate_both"]:
    modes[m] = ref("--mode", m, "--gen", 24, "--prompt-len", 13, "--prompt-seed", 3)
save("tiny_ref_modes.json", modes)
# 5. Known-answer values of the PRNG / prompt / percentile helpers.
rng = po.MtRng(1234)
kat = {
    "mt19937_64_seed1234_first8": [str(rng.next()) for _ in range(8)],
    "make_prompt_42_10_256": po.make_prompt(42, 10, 256),
    "make_prompt_42_10_32000": po.make_prompt(42, 10, 32000),
    "percentile_cases": [[[5.0, 1.0, 3.0, 2.0, 4.0], 50.0, po.percentile([5, 1, 3, 2, 4], 50)],
                         [[5.0, 1.0, 3.0, 2.0, 4.0], 99.0, po.percentile([5, 1, 3, 2, 4], 99)],
                         [[7.0], 1.0, po.percentile([7], 1)]],
}
save("kat.json", kat)
# 6. LLaMA-arch fixtures from the restatement (no reference exists).
for name, kw in {
    "llama_tiny_f32": dict(arch=po.ARCH_LLAMA, d_ff=176),
    "llama_tiny_bf16": dict(arch=po.ARCH_LLAMA, d_ff=176, weight_dtype=po.BF16, kv_dtype=po.BF16),
    "llama_tiny_philox_bf16": dict(arch=po.ARCH_LLAMA, d_ff=176, weight_dtype=po.BF16, kv_dtype=po.BF16,
                                   init=po.INIT_PHILOX),
}.items():
    m = po.OracleModel(**kw)
    prompt = po.make_prompt(42, 10, 256)
    toks, lg = m.generate_greedy(prompt, 16)
    save(name + ".json", {"config": kw, "prompt": prompt, "tokens": toks,
                          "logits": [[float("%.9g" % v) for v in row] for row in lg.tolist()]})
