"""Helpers for the -m gpu parity tests (device memory via torch: plumbing only)."""
import numpy as np


def margin_ok_tokens(gpu_tokens, ref_tokens, ref_logits, tol):
    """Greedy ids must match wherever the reference top-2 margin exceeds tol;
    comparison stops at the first divergence allowed by a sub-tolerance margin
    (after it the two streams condition on different tokens)."""
    for i, (a, b) in enumerate(zip(gpu_tokens, ref_tokens)):
        lg = np.asarray(ref_logits[i], np.float64)
        top2 = np.sort(lg)[-2:]
        margin = top2[1] - top2[0]
        if a != b:
            assert margin <= tol, f"step {i}: gpu {a} vs ref {b} with margin {margin:.3g} > {tol}"
            return i
    return len(gpu_tokens)


def bf16_bits(a):
    """fp32 -> bf16 bit patterns (RNE), as uint16."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_round(a):
    return (bf16_bits(a).astype(np.uint32) << 16).view(np.float32)
