"""Per-token device gaps of one 7B greedy run (P=10, 136 steps): where the p99 comes from."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2604_23467_b200 import graphrt as g  # noqa: E402
import pyoracle as po  # noqa: E402

mode = g.mode_from_name(sys.argv[1] if len(sys.argv) > 1 else "hybrid")
s = g.Session(g.ModelConfig.llama2_7b(max_seq_len=640), g.CacheConfig(bucket_size=64, warmup_hi=20, batched_prefill=True))
req = g.GenerationRequest(mode=mode, prompt=po.make_prompt(42, 10, 32000), gen_len=136)
s.run(req)
r = s.run(req)
us = r.per_token_us
order = sorted(range(len(us)), key=lambda i: -us[i])
print("slowest steps (index, length, us):", [(i, 10 + i + 1, round(us[i], 1)) for i in order[:10]])
print("median us:", sorted(us)[len(us) // 2])
print("by step:", [round(u) for u in us])
