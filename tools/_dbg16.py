import sys, numpy as np, collections
sys.path.insert(0, '.')
from paper_2604_23467_b200 import graphrt as g
cfg = g.ModelConfig.llama2_7b(n_layers=2, max_seq_len=64)
s = g.Session(cfg, g.CacheConfig(bucket_size=64, warmup_hi=0))
bad = 0
for it in range(12):
    s.reset()
    for j in range(9):
        try:
            s.step(1 + j)
        except Exception as e:
            bad += 1
            print("iter", it, "len", j + 1, e)
print("step-api bad", bad)
try:
    r = s.run(g.GenerationRequest(prompt=[1, 2, 3], gen_len=40))
    print("run ok", r.tokens[:5])
except Exception as e:
    print("run:", e)
