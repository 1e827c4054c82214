"""One batched prefill of LLaMA-2-7B dims (n_layers from argv) at prompt length P,
for ncu launch lists / captures of the prefill kernels.
usage: python tools/prefill_prof.py P [layers] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 500
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = g.ModelConfig.llama2_7b(n_layers=L, max_seq_len=640)
s = g.Session(cfg, g.CacheConfig(bucket_size=64, warmup_hi=0, batched_prefill=True))
prompt = [(i * 7919 + 17) % 32000 for i in range(P)]
for r in range(reps):
    s.reset()
    t0 = time.time()
    s.prefill(prompt)
    print(f"prefill P={P} layers={L}: {1e3 * (time.time() - t0):.2f} ms (host wall, incl. sync)")
