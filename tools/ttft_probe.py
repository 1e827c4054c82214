"""TTFT of repeated identical requests (LLaMA-2 7B, P from argv): batched prefill
launched eagerly vs replayed from the prompt-length graph cache."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402
from paper_2604_23467_b200.bench_harness import make_prompt  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = g.Model(g.ModelConfig.llama2_7b(max_seq_len=640))
prompt = make_prompt(42, P, 32000)
for graphs in (False, True):
    s = g.Session(m, g.CacheConfig(bucket_size=64, warmup_hi=10, capacity=4096, batched_prefill=True,
                                   prefill_uses_graphs=graphs))
    rows = []
    for i in range(8):
        r = s.run(g.GenerationRequest(prompt=prompt, gen_len=16))
        rows.append((round(r.ttft_us / 1e3, 3), round(r.prefill_us / 1e3, 3), r.prefill_paths[0].name))
    print("graphs" if graphs else "eager ", rows)
    s.close()
