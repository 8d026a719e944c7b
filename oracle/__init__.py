"""CPU fp64 oracle for the AstraFlow (arXiv 2605.15565) trainer policy-loss hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.
The product path (``paper_2605_15565_b200``) never imports it and has no CPU
fallback; the two share no code (SURVEY.md §8(c) "Implementation rules").

Everything here is plain, slow and written to be checked by eye against the
definitions in DESIGN.md §3 (which restate SURVEY.md §8(c) c1–c9):

* ``group_advantage``   – c1, GRPO group-relative advantages ("group-level reward
  normalization"; 8 rollouts per prompt), zero-variance
  predicate, optional batch-level normalisation.
* ``seq_bookkeeping``   – c2, token->sequence map, staleness mask ("max staleness 8",
  PAPER.md:776; SPEC.md:142 worked example), active-token counts.
* ``token_logprob``     – c3, log-softmax over V then gather (BASELINE.json north_star).
* ``policy_loss_fwd_bwd`` – c4–c7, clipped importance-ratio surrogate against the
  behaviour log-probs, token-mean weighting and dL/dlogits = scale·(softmax − onehot).
* ``vocab_shard_stats`` / ``vocab_combine`` – c8, vocab-parallel log-softmax combine.
* NEXT rows: ``policy_loss_fwd_bwd``'s ref_logp / prox_logp / want_entropy
  (k3 KL, decoupled ratio, entropy — readings N1-N3) and ``m2po_mask`` (M2PO second-moment
  masking, reading M1).
* ``lmhead_logprob`` / ``lmhead_loss_backward`` – NEXT 4: c3 on x = h W^T from the LM head's
  hidden states and weight (the logits never given), and the backward dh = G W, dW = G^T h with
  G = s (softmax - onehot) (c7 through the LM head).

Parity status of every function is listed in DESIGN.md §4 ("pins").
"""

from .policy_loss import (  # noqa: F401
    STD_UNBIASED, STD_BIASED, STD_NONE,
    AGG_TOKEN_MEAN, AGG_SEQ_MEAN_TOKEN_MEAN, AGG_SUM,
    LossParams,
    decode_bf16,
    m2po_mask,
    group_advantage,
    seq_bookkeeping,
    token_logprob,
    policy_loss_fwd_bwd,
    vocab_shard_stats,
    vocab_combine,
)
from . import delta  # noqa: F401,E402
from .lmhead import lmhead_logits, lmhead_logprob, lmhead_loss_backward  # noqa: F401,E402
