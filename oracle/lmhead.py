"""CPU fp64 oracle of the fused LM-head loss (NEXT 4 of SURVEY.md §8(f): forward log-prob and the
backward through the LM head) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

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


def lmhead_loss_backward(hidden_bits, weight_bits, targets, scale, inv_temperature: float = 1.0):
    """(dh, dW) fp64 of the LM-head loss backward (NEXT 4 backward half).

    The trainer step's gradient w.r.t. the logits is c7 of SURVEY.md §8(c):
        G[t, v] = s_t (p_{t,v} - [v == y_t]),   p_t = softmax(x_t * inv_T),   x = h W^T
    (s_t already carries inv_T, as the scale of rl_policy_loss_fwd_bwd / rl_policy_loss_from_logp;
    rows with y_t outside [0, V) or s_t = 0 give G[t] = 0).  The chain rule through x = h W^T is
        dh = G W        ([N, V] x [V, d])
        dW = G^T h      ([V, N] x [N, d])
    Written out: fp64 logits from the exactly decoded bf16 inputs (library matmul as one step),
    the softmax, G, then the two products (library matmuls)."""
    h = decode_bf16(np.asarray(hidden_bits, dtype=np.uint16))
    w = decode_bf16(np.asarray(weight_bits, dtype=np.uint16))
    x = (h @ w.T) * float(inv_temperature)
    n, V = x.shape
    y = np.asarray(targets, dtype=np.int64)
    s = np.asarray(scale, dtype=np.float64)
    m = x.max(axis=1, keepdims=True)
    e = np.exp(x - m)
    p = e / e.sum(axis=1, keepdims=True)
    G = s[:, None] * p
    ok = (y >= 0) & (y < V)
    G[np.nonzero(ok)[0], y[ok]] -= s[ok]
    G[~ok] = 0.0
    return G @ w, G.T @ h, G
