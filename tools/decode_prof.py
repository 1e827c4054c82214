"""Eager decode steps of LLaMA-2-7B dims (step API: the plan's kernels launched
directly, no graph capture thread) for ncu captures of single kernels.
usage: python tools/decode_prof.py P [layers] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402
from paper_2604_23467_b200.bench_harness import make_prompt  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 10
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4
s = g.Session(g.ModelConfig.llama2_7b(n_layers=L, max_seq_len=640),
              g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True))
s.prefill(make_prompt(42, P, 32000))
for t in range(n):
    s.step(100 + t)
print("ok", s.cur_len)
