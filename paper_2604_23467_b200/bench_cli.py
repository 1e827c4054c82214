"""graphrt_bench equivalent (tools/bench_main.cpp:14-98): the latency sweep from
a config file and/or flags, CSV out, summary tables on stdout.

    python -m paper_2604_23467_b200.bench_cli [--config FILE] [--csv OUT]
        [--modes eager,hybrid,...] [--prompt-lens 10,50] [--gen-lens 10,50]
        [--trials N] [--seed S] [--strategy greedy|temperature] [--temperature T]
        [--model-preset tiny-ref|llama2-7b] [--set section.key=value ...]

Precedence as the reference: defaults < --config < flags.
"""
from __future__ import annotations

import argparse
import sys

from . import bench_harness as bh
from . import graphrt as g


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="graphrt_bench")
    ap.add_argument("--config")
    ap.add_argument("--csv")
    ap.add_argument("--modes")
    ap.add_argument("--prompt-lens")
    ap.add_argument("--gen-lens")
    ap.add_argument("--trials", type=int)
    ap.add_argument("--seed", type=int)
    ap.add_argument("--strategy", choices=["greedy", "temperature"])
    ap.add_argument("--temperature", type=float)
    ap.add_argument("--model-preset", choices=["tiny-ref", "llama2-7b"], default="tiny-ref")
    ap.add_argument("--set", action="append", default=[], help="extra section.key=value (after --config)")
    a = ap.parse_args(argv)
    cfg = bh.BenchConfig()
    if a.model_preset == "llama2-7b":
        cfg.model = g.ModelConfig.llama2_7b()
        cfg.cache = g.CacheConfig(bucket_size=64, batched_prefill=True)
    kv = bh.parse_config_file(a.config) if a.config else {}
    flags = {"bench.modes": a.modes, "bench.prompt_lens": a.prompt_lens, "bench.gen_lens": a.gen_lens,
             "bench.trials": a.trials, "bench.seed": a.seed, "bench.strategy": a.strategy,
             "bench.temperature": a.temperature}
    kv.update({k: str(v) for k, v in flags.items() if v is not None})
    kv.update(bh.parse_config_text("\n".join(a.set)))
    try:
        ignored = bh.apply_config(cfg, kv)
        if ignored:
            print("ignored (virtual-clock keys, real hardware here): " + ", ".join(sorted(ignored)), file=sys.stderr)
        res = bh.run_bench(cfg, progress=sys.stderr)
    except g.Error as e:
        print(f"graphrt_bench: {e}", file=sys.stderr)
        return 1
    for s in res.skipped_cells:
        print("skipped " + s, file=sys.stderr)
    if a.csv:
        bh.write_csv_file(a.csv, res.rows)
    bh.format_summary(sys.stdout, res.summaries)
    return 0


if __name__ == "__main__":
    sys.exit(main())
