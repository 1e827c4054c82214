"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel
count / mean / share over the last N launches.  usage: launch_summary.py FILE [N]"""
import collections
import csv
import sys

path = sys.argv[1]
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lines = [l for l in open(path) if not l.startswith("==")]
rows = list(csv.DictReader(lines))
vals = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    vals.append((r["Kernel Name"], v))
if n_last:
    vals = vals[-n_last:]
agg = collections.defaultdict(list)
for n, v in vals:
    agg[n.split("(")[0][:70]].append(v)
tot = sum(v for _, v in vals)
print(f"{len(vals)} launches, total {tot:.1f} us")
for n, vs in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{n:70s} n={len(vs):5d} mean={sum(vs) / len(vs):9.2f} us  share={sum(vs) / tot:.3f}")
