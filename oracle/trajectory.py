"""Oracle trajectory for bench.py's parity stamp -- TEST INFRASTRUCTURE ONLY.

    python oracle/trajectory.py OUT.npz --layers 32 --max-seq 64 --prompt 1,2,3 --tokens 4,5

Runs the C restatement (oracle.c; model.cpp:168-183 prefill_math / step_math at
the LLaMA-2-7B dims, bf16 weights and KV, Philox init, seed 1234) in its own
process, so the checker is never mapped into the measured process: prefill of
the prompt, then one step per teacher-forced token.  Writes the logits after the
prefill and after every step, plus wall-clock timings (init, per pass) and the
thread count, to OUT.npz.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import pyoracle as po  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--max-seq", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--prompt", required=True)
    ap.add_argument("--tokens", default="")
    args = ap.parse_args()
    prompt = [int(x) for x in args.prompt.split(",") if x]
    toks = [int(x) for x in args.tokens.split(",") if x]
    t0 = time.perf_counter()
    o = po.OracleModel(arch=po.ARCH_LLAMA, n_layers=args.layers, d_model=4096, n_heads=32, vocab_size=32000,
                       max_seq_len=args.max_seq, d_ff=11008, init=po.INIT_PHILOX, weight_dtype=po.BF16,
                       kv_dtype=po.BF16, seed=args.seed, n_threads=0)
    init_s = time.perf_counter() - t0
    t1 = time.perf_counter()
    rc = o.prefill(prompt)
    if rc:
        raise SystemExit(f"oracle prefill failed rc={rc}")
    prefill_s = time.perf_counter() - t1
    logits = [o.logits()]
    step_s = []
    for t in toks:
        t1 = time.perf_counter()
        rc = o.step(t)
        step_s.append(time.perf_counter() - t1)
        if rc:
            raise SystemExit(f"oracle step failed rc={rc}")
        logits.append(o.logits())
    np.savez(args.out, logits=np.stack(logits), init_s=init_s, prefill_s=prefill_s, step_s=np.asarray(step_s),
             threads=os.cpu_count() or 1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
