"""Timeline of the per-op decode plan (pass_impl=1) captured as a CUDA graph, from
per-CTA %globaltimer stamps: for each kernel kind, averaged over layers,
  dep   = first CTA released (griddepcontrol.wait) - previous kernel's last CTA done
  ready = last CTA's operands ready - first release
  body  = last CTA done - first release
  tail  = last CTA done - median CTA done
  eff   = this kernel's last done - previous kernel's last done
  early = previous kernel's last done - median CTA start (how long CTAs were resident before it ended)
usage: python tools/op_trace.py [layers] [seq_len]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_23467_b200 import graphrt as g  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
T = int(sys.argv[2]) if len(sys.argv) > 2 else 80
cfg = g.ModelConfig.llama2_7b(n_layers=layers, max_seq_len=640)
s = g.Session(cfg, g.CacheConfig(bucket_size=64, warmup_hi=0, pass_impl=1))
s.run(g.GenerationRequest(prompt=list(range(1, 11)), gen_len=T - 10))
key = (T + 63) // 64
names = ["qkv", "attn", "wo", "gate_up", "down"] * layers + ["head"]
for rep in range(2):
    tr = s.trace_pass(key).astype(np.int64).reshape(len(names), -1, 8)
    rows = {}
    prev_end = None
    t0 = None
    for i, nm in enumerate(names):
        st = tr[i]
        st = st[st[:, 0] > 0]
        if t0 is None:
            t0 = st[:, 0].min()
        rel = st[:, 1].min()
        done = st[:, 3][st[:, 3] > 0]
        rdy = st[:, 2][st[:, 2] > 0]
        end = done.max()
        r = rows.setdefault(nm, {k: [] for k in ("dep", "ready", "body", "tail", "eff", "ctas", "start_spread", "early",
                                                 "first", "loop", "epi")})
        if (st[:, 4] > 0).any():
            r["first"].append(np.median(st[:, 4] - st[:, 1]))  # first stage landed, relative to release
            r["loop"].append(np.median(st[:, 5] - st[:, 2]))   # streaming loop after operands ready
            r["epi"].append(np.median(st[:, 3] - st[:, 5]))    # deferred epilogue + CTA sync
        if prev_end is not None:
            r["dep"].append(rel - prev_end)
            r["early"].append(prev_end - np.median(st[:, 0]))
            r["eff"].append(end - prev_end)
        r["ready"].append(rdy.max() - rel)
        r["body"].append(end - rel)
        r["tail"].append(end - np.median(done))
        r["ctas"].append(len(st))
        r["start_spread"].append(st[:, 0].max() - st[:, 0].min())
        prev_end = end
    total = prev_end - t0
    print(f"rep {rep}: graph span {total / 1e3:.1f} us ({total / 1e3 / layers:.2f} us/layer)")
    for nm, r in rows.items():
        f = {k: (np.mean(v) / 1e3 if v else float('nan')) for k, v in r.items() if k != "ctas"}
        print(f"  {nm:8s} ctas={int(np.mean(r['ctas'])):4d} dep={f['dep']:6.2f} ready={f['ready']:6.2f} "
              f"body={f['body']:6.2f} tail={f['tail']:6.2f} eff={f['eff']:6.2f} start_spread={f['start_spread']:6.2f} "
              f"early={f['early']:6.2f} first={f['first']:6.2f} loop={f['loop']:6.2f} epi={f['epi']:6.2f} us")
# per-CTA operand latency distribution of the attention kernels (last rep)
i_att = [i for i, n in enumerate(names) if n == "attn"]
lat = []
for i in i_att:
    st = tr[i]
    st = st[(st[:, 0] > 0) & (st[:, 2] > 0)]
    lat.append(st[:, 2] - st[:, 1])
lat = np.concatenate(lat) / 1e3
print("attn ready-released per CTA us: p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(lat, [10, 50, 90, 100])))
# attention phases (median over CTAs, relative to release): scores, CTA merge done, cluster barrier, rank-0 merge, exit
ph = {k: [] for k in ("scores", "cta_merge", "cluster1", "merged", "exit")}
for i in i_att:
    st = tr[i]
    st = st[(st[:, 0] > 0) & (st[:, 3] > 0)]
    r = st[:, 1]
    for k, c in zip(ph, (2, 4, 5, 6, 3)):
        v = st[:, c]
        ok = v > 0
        if ok.any():
            ph[k].append(np.median(v[ok] - r[ok]))
print("attn phases (median us after release): " + " ".join(f"{k}={np.mean(v) / 1e3:.2f}" for k, v in ph.items() if v))
