"""Phase timeline of the streaming pass (pass_impl 2, LLaMA-2 7B) from per-CTA
%globaltimer stamps: per phase (averaged over layers) the time from the last
CTA finishing the previous phase to the last CTA finishing this one, and the
spread of finish times across CTAs."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = g.ModelConfig.llama2_7b(n_layers=layers, max_seq_len=640)
s = g.Session(cfg, g.CacheConfig(bucket_size=64, warmup_hi=0, pass_impl=2))
s.run(g.GenerationRequest(prompt=list(range(1, 11)), gen_len=70))  # seq_len = 80
key = (80 + 63) // 64
names = ["qkv", "attn_partial", "attn_merge", "wo", "up", "down"]
for rep in range(3):
    tr = s.trace_pass(key).astype(np.int64)
L = layers
t_start, t_wait, t_end = tr[:, 0].min(), tr[:, 1].max(), tr[:, 2 + 8 * L].max()
out = {"total_us": (t_end - t_start) / 1e3, "wait_us": (t_wait - t_start) / 1e3}
prev = tr[:, 1]
acc = {n: [] for n in names}
spread = {n: [] for n in names}
for l in range(L):
    for i, n in enumerate(names):
        cur = tr[:, 2 + 8 * l + i]
        acc[n].append((cur.max() - prev.max()) / 1e3)
        spread[n].append((cur.max() - cur.min()) / 1e3)
        prev = cur
for n in names:
    out[n + "_us"] = round(float(np.mean(acc[n])), 3)
    out[n + "_spread_us"] = round(float(np.mean(spread[n])), 3)
out["head_us"] = (t_end - prev.max()) / 1e3
out["per_layer_us"] = round(sum(out[n + "_us"] for n in names), 3)
print(json.dumps(out, indent=1))
