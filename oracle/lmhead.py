"""CPU fp64 oracle of the fused LM-head log-prob (NEXT 4 of SURVEY.md §8(f), forward half) —
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md §8(f) NEXT 4: "Fused LM-head GEMM + loss (tcgen05, logits never materialised) ...
it takes hidden states and W" (BASELINE.json north_star: the logits of the policy's LM head are
the input of the loss today).  The logits are x = h W^T (one row of hidden states h [d] against
every vocabulary row of the LM-head weight W [V, d]); the log-prob is then c3 of SURVEY.md §8(c)
applied to x (token_logprob).  The oracle is that definition written out: an fp64 matrix product
of the exactly decoded bf16 inputs (a library primitive as one step), then c3.
"""

from __future__ import annotations

import numpy as np

from .policy_loss import decode_bf16, token_logprob


def lmhead_logits(hidden_bits, weight_bits) -> np.ndarray:
    """x = h W^T in fp64 from bf16 bit patterns: hidden [N, d], weight [V, d] (uint16)."""
    h = decode_bf16(np.asarray(hidden_bits, dtype=np.uint16))
    w = decode_bf16(np.asarray(weight_bits, dtype=np.uint16))
    if h.ndim != 2 or w.ndim != 2 or h.shape[1] != w.shape[1]:
        raise ValueError("hidden [N, d] and weight [V, d] must share d")
    return h @ w.T


def lmhead_logprob(hidden_bits, weight_bits, targets, inv_temperature: float = 1.0):
    """(logp, lse) fp64 of c3 on x = h W^T (NEXT 4)."""
    return token_logprob(lmhead_logits(hidden_bits, weight_bits), targets, inv_temperature)
