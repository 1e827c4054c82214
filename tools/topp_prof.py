"""A warm 7B top-p run (P=10, 24 steps) for an ncu launch list of the sampler."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "topp"
s = g.Session(g.ModelConfig.llama2_7b(n_layers=2, max_seq_len=128), g.CacheConfig(bucket_size=64, warmup_hi=2, batched_prefill=True))
strat = g.SampleStrategy.top_kp(0.8, 0, 0.9) if kind == "topp" else (
    g.SampleStrategy.top_kp(0.8, 50, 1.0) if kind == "topk" else g.SampleStrategy.greedy())
req = g.GenerationRequest(prompt=list(range(1, 11)), gen_len=24, strategy=strat, sampler_seed=7)
s.run(req)
r = s.run(req)
print(kind, "p50 us", sorted(r.per_token_us)[12])
