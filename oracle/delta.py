"""fp-free CPU oracle of the bf16 delta-sparsity scan (NEXT 3 of SURVEY.md §8(f)) — TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:446 / :463-468: "the trainer needs to ship only a tiny fraction of its weights" — a
bit-exact comparison of consecutive bf16 snapshots (sparsity 0.989-0.993); SPEC.md:297-313 fixes
the operation: compute_delta returns exactly the indices whose 16-bit words differ, in increasing
order, with the new words; apply_delta(prev, compute_delta(prev, next)) = next bit for bit.
Elements are opaque 16-bit words (SPEC.md design decision): no numeric interpretation."""

from __future__ import annotations

import numpy as np


def compute_delta(prev, nxt):
    """(indices u32[k] increasing, words u16[k], sparsity) — an explicit element-wise loop."""
    a = np.ascontiguousarray(prev).view(np.uint16)
    b = np.ascontiguousarray(nxt).view(np.uint16)
    if a.shape != b.shape:
        raise ValueError("length-mismatch")
    idx, words = [], []
    for i in range(a.size):
        if a[i] != b[i]:
            idx.append(i)
            words.append(b[i])
    n = a.size
    sparsity = 1.0 - len(idx) / n if n else 1.0
    return np.array(idx, dtype=np.uint32), np.array(words, dtype=np.uint16), sparsity


def apply_delta(base, idx, words):
    """base with words[j] written at idx[j]."""
    out = np.array(np.ascontiguousarray(base).view(np.uint16), copy=True)
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= out.size):
        raise ValueError("index-out-of-range")
    out[idx] = np.asarray(words, dtype=np.uint16)
    return out
