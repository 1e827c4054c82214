"""Phase timeline of the persistent decode pass (LLaMA-2 7B) from per-CTA
%globaltimer stamps (grt_trace_pass).  Prints, averaged over layers, for each
phase: barrier latency (last arrival of the previous phase -> first CTA
released), release skew, and work time (release -> last CTA done)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = g.ModelConfig.llama2_7b(n_layers=layers, max_seq_len=640)
s = g.Session(cfg, g.CacheConfig(bucket_size=64, warmup_hi=0))
s.run(g.GenerationRequest(prompt=list(range(1, 11)), gen_len=70))  # seq_len = 80
key = (80 + 63) // 64
res = []
for rep in range(3):
    tr = s.trace_pass(key).astype(np.int64)
    L = layers
    t0 = tr[:, L * 10 + 2].min()
    ph = {"qkv": (0, 1), "attn": (2, 3), "wo": (4, 5), "up": (6, 7), "down": (8, 9)}
    out = {}
    prev_end = None
    for name, (a, b) in ph.items():
        st = tr[:, [l * 10 + a for l in range(L)]]
        en = tr[:, [l * 10 + b for l in range(L)]]
        work = en.max(0) - st.max(0)
        skew = st.max(0) - st.min(0)
        out[name] = {"work_us": float(work.mean() / 1e3), "release_skew_us": float(skew.mean() / 1e3),
                     "end_spread_us": float((en.max(0) - en.min(0)).mean() / 1e3)}
    # barrier latency: previous phase's last end -> this phase's first start
    order = ["qkv", "attn", "wo", "up", "down"]
    for i, name in enumerate(order):
        a = ph[name][0]
        pb = ph[order[i - 1]][1]
        lat = []
        for l in range(L):
            if i == 0 and l == 0:
                continue
            pl = l if i > 0 else l - 1
            lat.append(tr[:, l * 10 + a].min() - tr[:, pl * 10 + pb].max())
        out[name]["barrier_us"] = float(np.mean(lat) / 1e3)
    total = (tr[:, L * 10 + 1].max() - t0) / 1e3
    out["total_us"] = float(total)
    out["head_us"] = float((tr[:, L * 10 + 1].max() - tr[:, L * 10 + 0].min()) / 1e3)
    res.append(out)
print(json.dumps(res[-1], indent=1))
ready = tr[:, L * 10 + 3].sum()
waited = tr[:, L * 10 + 4].sum()
print(json.dumps({"stages_ready_on_arrival": int(ready), "stages_waited": int(waited),
                  "ready_frac": float(ready / max(1, ready + waited))}))
