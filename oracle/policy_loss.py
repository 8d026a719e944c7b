"""fp64 CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Definitions follow SURVEY.md §8(c) steps c1–c9 and the readings Z1–Z24 listed in
DESIGN.md §3.  The paper gives no formula for any of this path (it is a
systems paper; its only equation is the autoscaler), so the
definition is the north_star's (BASELINE.json) plus the paper's named settings:
GRPO group normalisation, PPO-style clipped surrogate
("4 PPO mini-batches"), rollout temperature 1.0,
max staleness 8, zero-advantage predicate.

Scalar steps that must be bit-exact (c1 advantages, c2 bookkeeping) are explicit
left-to-right Python loops over Python floats (IEEE binary64; CPython never
contracts a*b+c into an FMA).  Row math (c3–c7) uses NumPy in fp64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

STD_UNBIASED, STD_BIASED, STD_NONE = 0, 1, 2
AGG_TOKEN_MEAN, AGG_SEQ_MEAN_TOKEN_MEAN, AGG_SUM = 0, 1, 2
STALE_HIST_BINS = 16


def decode_bf16(bits: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float64, exact (bits<<16 is the fp32 pattern)."""
    b = np.ascontiguousarray(bits).view(np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


# ----------------------------------------------------------------------------- c1
def group_advantage(rewards: Sequence[float], cu_groups: Sequence[int],
                    std_mode: int = STD_UNBIASED, eps: float = 1e-6,
                    batch_norm: bool = False, bn_eps: float = 1e-6,
                    seq_weight: Optional[Sequence[int]] = None):
    """c1: GRPO group-relative advantages ("group-level reward
    normalization", :580 GRPO; groups of 8 rollouts, :574).

    For group g with members i = cu[g] .. cu[g+1]-1 (index order):
      zero_var[g] = all r_i == r_first (exact equality; singleton -> true,
      SPEC.md:232); then A_i = +0.0.
      else  mu = (((r0 + r1) + r2) ... ) / n
            d_i = r_i - mu
            q   = ((d0*d0 + d1*d1) + ...)
            sigma = sqrt(q/(n-1)) [unbiased] | sqrt(q/n) [biased]
            A_i = d_i / (sigma + eps)      [STD_NONE: A_i = d_i]
    Optional batch-level normalisation ("batch-level advantage
    normalization"; reading Z6): token-weighted with weights L_i = seq_weight[i]:
      W = sum L_i; mu_B = (sum L_i*A_i)/W; v_B = (sum L_i*((A_i-mu_B)*(A_i-mu_B)))/W
      A_i <- (A_i - mu_B)/(sqrt(v_B) + bn_eps)      (skipped when W == 0)
    Output: float32(A_i) (round to nearest even) and zero_var as uint8.
    Raises ValueError on an empty group ("empty group -> invalid-argument").
    """
    r = [float(x) for x in rewards]
    cu = [int(x) for x in cu_groups]
    n_groups = len(cu) - 1
    if n_groups < 0 or cu[0] != 0 or cu[-1] != len(r):
        raise ValueError("cu_groups must start at 0 and end at n_seq")
    adv = [0.0] * len(r)
    zero_var = [0] * n_groups
    for g in range(n_groups):
        lo, hi = cu[g], cu[g + 1]
        n = hi - lo
        if n <= 0:
            raise ValueError(f"empty group {g}")
        first = r[lo]
        allequal = True
        for i in range(lo, hi):
            if not (r[i] == first):
                allequal = False
        if allequal:
            zero_var[g] = 1
            for i in range(lo, hi):
                adv[i] = 0.0
            continue
        acc = 0.0
        for i in range(lo, hi):
            acc = acc + r[i]
        mu = acc / n
        q = 0.0
        for i in range(lo, hi):
            d = r[i] - mu
            q = q + d * d
        if std_mode == STD_UNBIASED:
            sigma = math.sqrt(q / (n - 1))
        elif std_mode == STD_BIASED:
            sigma = math.sqrt(q / n)
        elif std_mode == STD_NONE:
            sigma = None
        else:
            raise ValueError("bad std_mode")
        for i in range(lo, hi):
            d = r[i] - mu
            adv[i] = d if sigma is None else d / (sigma + eps)
    if batch_norm:
        if seq_weight is None:
            raise ValueError("batch_norm needs seq_weight (active tokens per sequence)")
        L = [int(x) for x in seq_weight]
        W = 0
        for x in L:
            W += x
        if W > 0:
            s = 0.0
            for i in range(len(r)):
                s = s + float(L[i]) * adv[i]
            mu_b = s / float(W)
            v = 0.0
            for i in range(len(r)):
                e = adv[i] - mu_b
                v = v + float(L[i]) * (e * e)
            v_b = v / float(W)
            den = math.sqrt(v_b) + bn_eps
            for i in range(len(r)):
                adv[i] = (adv[i] - mu_b) / den
    return np.array(adv, dtype=np.float64).astype(np.float32), np.array(zero_var, dtype=np.uint8)


# ----------------------------------------------------------------------------- c2
def seq_bookkeeping(cu_seqlens: Sequence[int], loss_mask, targets, vocab: int,
                    seq_version=None, trainer_version: int = 0, max_staleness: int = -1):
    """c2: token->sequence map, staleness mask, active-token counts.

    staleness_i = trainer_version - seq_version[i] (0 when no versions given);
    a sequence is usable iff 0 <= staleness_i and (max_staleness < 0 or
    staleness_i <= max_staleness)  ("max staleness 8"; SPEC.md:142:
    20 - 11 = 9 > 8 -> discarded).  staleness_i < 0 is a counted error (neg_staleness).
    valid_t = loss_mask_t != 0  and 0 <= y_t < V  and usable(seq(t)).
    Counts: active_tokens = sum valid; stale_masked = tokens with mask and in-range
    target dropped only because staleness > max_staleness; neg_staleness = sequences;
    bad_targets = tokens with y_t >= V (any mask).  stale_hist[b] = sequences with
    staleness min(s, 15) = b (negative staleness not binned).
    """
    cu = [int(x) for x in cu_seqlens]
    n_seq = len(cu) - 1
    n_tok = cu[-1]
    mask = [int(x) for x in loss_mask]
    y = [int(x) for x in targets]
    if len(mask) != n_tok or len(y) != n_tok:
        raise ValueError("length mismatch")
    token_seq = [0] * n_tok
    for i in range(n_seq):
        for t in range(cu[i], cu[i + 1]):
            token_seq[t] = i
    stale = [0] * n_seq
    if seq_version is not None:
        for i in range(n_seq):
            stale[i] = int(trainer_version) - int(seq_version[i])
    usable = [True] * n_seq
    neg = 0
    hist = [0] * STALE_HIST_BINS
    for i in range(n_seq):
        if stale[i] < 0:
            usable[i] = False
            neg += 1
            continue
        hist[min(stale[i], STALE_HIST_BINS - 1)] += 1
        if max_staleness >= 0 and stale[i] > max_staleness:
            usable[i] = False
    valid = [0] * n_tok
    seq_active = [0] * n_seq
    active = stale_masked = bad = 0
    for t in range(n_tok):
        in_range = 0 <= y[t] < vocab
        if y[t] >= vocab:
            bad += 1
        i = token_seq[t]
        if mask[t] != 0 and in_range:
            if usable[i]:
                valid[t] = 1
                seq_active[i] += 1
                active += 1
            elif stale[i] >= 0:
                stale_masked += 1
    return dict(
        token_seq=np.array(token_seq, dtype=np.int32),
        valid=np.array(valid, dtype=np.uint8),
        seq_active=np.array(seq_active, dtype=np.int32),
        seq_staleness=np.array(stale, dtype=np.int32),
        stale_hist=np.array(hist, dtype=np.int64),
        active_tokens=active, stale_masked=stale_masked,
        neg_staleness=neg, bad_targets=bad,
    )


# ----------------------------------------------------------------------------- c3
def token_logprob(logits: np.ndarray, targets, inv_temperature: float = 1.0):
    """c3: z = x*inv_T; M = max_v z; S = sum_v exp(z - M); lse = M + ln S;
    logp = z_y - lse for 0 <= y < V; logp = 0 for y < 0 (ignored); NaN for y >= V.
    Returns (logp, lse) in fp64.  ``logits`` is [N, V] float (decode bf16 first)."""
    x = np.asarray(logits, dtype=np.float64)
    n, V = x.shape
    y = np.asarray(targets, dtype=np.int64)
    z = x * float(inv_temperature)
    M = np.max(z, axis=1) if V > 0 else np.full(n, -np.inf)
    with np.errstate(invalid="ignore", over="ignore"):
        S = np.sum(np.exp(z - M[:, None]), axis=1)
        lse = M + np.log(S)
    logp = np.zeros(n, dtype=np.float64)
    for t in range(n):
        if 0 <= y[t] < V:
            logp[t] = z[t, y[t]] - lse[t]
        elif y[t] >= V:
            logp[t] = np.nan
    return logp, lse


# ----------------------------------------------------------------------------- c4-c7
@dataclass
class LossParams:
    """Knobs of the clipped surrogate (SURVEY.md §8(b) rl_loss_params; readings Z8-Z16)."""
    clip_eps_low: float = 0.2
    clip_eps_high: float = 0.2
    inv_temperature: float = 1.0
    log_ratio_clamp: float = 20.0
    agg: int = AGG_TOKEN_MEAN
    global_active_tokens: float = 0.0
    global_num_seqs: int = 0
    trainer_version: int = 0
    max_staleness: int = -1
    grad_scale: float = 1.0
    kl_coef: float = 0.0   # NEXT 2: beta of the k3 KL term vs ref_logp (1e-3); reading N1


def policy_loss_fwd_bwd(logits: np.ndarray, targets, old_logp, loss_mask, token_seq,
                        seq_adv, seq_version, seq_active, p: LossParams,
                        clip_override=None, want_dlogits: bool = True,
                        ref_logp=None, prox_logp=None, want_entropy: bool = False):
    """c4–c7 for the token rows given (any subset of a batch; the global
    normalisers come from ``p``).

    Per token t with sequence i = token_seq[t] and A = seq_adv[i]:
      valid_t  (c2 rule, with p.trainer_version / p.max_staleness)
      logp_t   (c3)
      D = logp - old;  Dc = min(max(D, -c), c);  clamp_active = Dc != D;  r = exp(Dc)
      u = r*A;  k = min(max(r, 1-eps_l), 1+eps_h)*A;  L_t = -min(u, k)
      clipped_t = 2 if A > 0 and r > 1+eps_h; 1 if A < 0 and r < 1-eps_l; else 0
      w_t = 1/N_active_global | 1/(S_global*L_i) | 1          (p.agg)
      s_t = w*A*r*inv_T*grad_scale if valid and clipped == 0 and not clamp_active else 0
      dlogits[t, v] = s_t * (exp(z_v - lse) - [v == y_t])      (rows with valid=0 are 0)
      loss = fsum_t valid_t * w_t * L_t
    ``clip_override`` (optional int array) replaces the clipped_t decision — used only
    inside the tie band of reading Z23, where either decision is correct.

    NEXT 2 extensions (the paper names the KL coefficient, and
    the staleness-aware setting, but no formulas — readings N1-N3):
      prox_logp (decoupled ratio, N2): r = exp(clamp(logp - prox)) is the clipped ratio and the
        surrogate is weighted by the behaviour correction rho = exp(clamp(prox - old)), no
        gradient through rho:  L_t = -rho * min(r A, clip(r) A).  prox_logp=None -> rho = 1,
        r vs old (the standard surrogate).
      ref_logp + p.kl_coef (k3 KL penalty, N1): Dk = clamp(ref - logp); KL_t = exp(Dk) - Dk - 1;
        L_t += kl_coef * KL_t;  dKL/dlogp = 1 - exp(Dk) (0 when the clamp is active).
      s_t = w * (rho A r [unclipped, unclamped] - kl_coef (1 - exp(Dk)) [KL unclamped]) inv_T grad_scale
      want_entropy (N3): H_t = lse_t - sum_v p_v z_v for valid tokens (reported, no gradient);
        stats entropy_sum = fsum valid H_t;  kl_sum = fsum valid w KL_t.
    """
    x = np.asarray(logits, dtype=np.float64)
    n, V = x.shape
    y = np.asarray(targets, dtype=np.int64)
    old = np.asarray(old_logp, dtype=np.float64)
    mask = np.asarray(loss_mask)
    tseq = np.asarray(token_seq, dtype=np.int64)
    adv = np.asarray(seq_adv, dtype=np.float64)
    ver = None if seq_version is None else np.asarray(seq_version, dtype=np.int64)
    L_seq = None if seq_active is None else np.asarray(seq_active, dtype=np.int64)
    invT = float(p.inv_temperature)
    c = float(p.log_ratio_clamp)
    lo_b, hi_b = 1.0 - float(p.clip_eps_low), 1.0 + float(p.clip_eps_high)

    prox = None if prox_logp is None else np.asarray(prox_logp, dtype=np.float64)
    ref = None if ref_logp is None else np.asarray(ref_logp, dtype=np.float64)
    beta = float(p.kl_coef)
    if beta != 0.0 and ref is None:
        raise ValueError("kl_coef != 0 needs ref_logp")
    logp, lse = token_logprob(x, y, invT)
    dl = np.zeros((n, V), dtype=np.float64) if want_dlogits else None
    entropy = np.zeros(n, dtype=np.float64)
    kl_terms, ent_terms = [], []
    loss_terms = []
    valid = np.zeros(n, dtype=np.uint8)
    clipped = np.zeros(n, dtype=np.uint8)
    scale = np.zeros(n, dtype=np.float64)
    ratio = np.zeros(n, dtype=np.float64)
    wl = np.zeros(n, dtype=np.float64)   # per-token w_t * L_t (0 for invalid tokens)
    st = dict(active_tokens=0, ratio_sum=0.0, clipped_low=0, clipped_high=0, clamped=0,
              stale_masked=0, bad_targets=0, neg_staleness=0, weight_sum=0.0)
    ratio_terms, weight_terms = [], []
    for t in range(n):
        i = int(tseq[t])
        stale = (p.trainer_version - int(ver[i])) if ver is not None else 0
        usable = stale >= 0 and (p.max_staleness < 0 or stale <= p.max_staleness)
        in_range = 0 <= y[t] < V
        if y[t] >= V:
            st["bad_targets"] += 1
        if stale < 0:
            st["neg_staleness"] += 1   # counted per token here (per-sequence in c2)
        if not (mask[t] != 0 and in_range):
            continue
        if not usable:
            if stale >= 0:
                st["stale_masked"] += 1
            continue
        valid[t] = 1
        A = float(adv[i])
        base = old[t] if prox is None else prox[t]          # the clipped ratio's denominator
        rho = 1.0
        if prox is not None:
            rho = math.exp(min(max(prox[t] - old[t], -c), c))  # behaviour correction, no gradient
        D = logp[t] - base
        Dc = min(max(D, -c), c)
        clamp_active = Dc != D
        r = math.exp(Dc)
        u = r * A
        k = min(max(r, lo_b), hi_b) * A
        L = -rho * min(u, k)
        kl, dkl = 0.0, 0.0
        if beta != 0.0:
            Dk = ref[t] - logp[t]
            Dkc = min(max(Dk, -c), c)
            kl = math.exp(Dkc) - Dkc - 1.0
            dkl = (1.0 - math.exp(Dkc)) if Dkc == Dk else 0.0
            L += beta * kl
        if A > 0 and r > hi_b:
            cl = 2
        elif A < 0 and r < lo_b:
            cl = 1
        else:
            cl = 0
        if clip_override is not None:
            cl = int(clip_override[t])
        if p.agg == AGG_TOKEN_MEAN:
            w = 1.0 / p.global_active_tokens if p.global_active_tokens > 0 else 0.0
        elif p.agg == AGG_SEQ_MEAN_TOKEN_MEAN:
            Li = int(L_seq[i])
            w = 1.0 / (float(p.global_num_seqs) * Li) if (Li > 0 and p.global_num_seqs > 0) else 0.0
        elif p.agg == AGG_SUM:
            w = 1.0
        else:
            raise ValueError("bad agg")
        g = (rho * A * r) if (cl == 0 and not clamp_active) else 0.0   # -dL_sur/dlogp
        g -= beta * dkl                                                  # -dL_kl/dlogp
        s = w * g * invT * float(p.grad_scale)
        clipped[t] = cl
        scale[t] = s
        ratio[t] = r
        loss_terms.append(w * L)
        wl[t] = w * L
        ratio_terms.append(r)
        weight_terms.append(w)
        kl_terms.append(w * kl)
        if want_entropy:
            prob = np.exp(x[t] * invT - lse[t])
            entropy[t] = lse[t] - float(np.sum(prob * (x[t] * invT)))
            ent_terms.append(entropy[t])
        st["active_tokens"] += 1
        st["clipped_low"] += cl == 1
        st["clipped_high"] += cl == 2
        st["clamped"] += bool(clamp_active)
        if want_dlogits and s != 0.0:
            prob = np.exp(x[t] * invT - lse[t])
            row = s * prob
            row[y[t]] -= s
            dl[t] = row
    st["ratio_sum"] = math.fsum(ratio_terms)
    st["weight_sum"] = math.fsum(weight_terms)
    st["kl_sum"] = math.fsum(kl_terms)
    st["entropy_sum"] = math.fsum(ent_terms)
    loss = math.fsum(loss_terms)
    return dict(loss=loss, dlogits=dl, logp=logp, lse=lse, valid=valid, clipped=clipped,
                scale=scale, ratio=ratio, token_loss=wl, stats=st, entropy=entropy)


# ----------------------------------------------------------------------------- c8
def vocab_shard_stats(logits_shard: np.ndarray, targets, vocab_offset: int,
                      inv_temperature: float = 1.0):
    """c8, per shard r covering global columns [o, o + V_r):
    m_r = max z, s_r = sum exp(z - m_r), xy_r = z_y if o <= y < o + V_r else 0 (owned flag).
    An empty shard gives (m=-inf, s=0)."""
    x = np.asarray(logits_shard, dtype=np.float64) * float(inv_temperature)
    n, Vr = x.shape
    y = np.asarray(targets, dtype=np.int64)
    if Vr == 0:
        return np.full(n, -np.inf), np.zeros(n), np.zeros(n), np.zeros(n, dtype=bool)
    m = np.max(x, axis=1)
    with np.errstate(invalid="ignore"):
        s = np.sum(np.exp(x - m[:, None]), axis=1)
    owned = (y >= vocab_offset) & (y < vocab_offset + Vr)
    xy = np.zeros(n)
    for t in range(n):
        if owned[t]:
            xy[t] = x[t, y[t] - vocab_offset]
    return m, s, xy, owned


def vocab_combine(ms, ss, xys):
    """c8 combine: M = max_r m_r; S = sum_r s_r * exp(m_r - M); lse = M + ln S;
    z_y = sum of the (single) owned target logit.  Returns (lse, z_y)."""
    m = np.stack(ms)
    s = np.stack(ss)
    M = np.max(m, axis=0)
    with np.errstate(invalid="ignore"):
        S = np.sum(s * np.exp(m - M[None, :]), axis=0)
    return M + np.log(S), np.sum(np.stack(xys), axis=0)


# ----------------------------------------------------------------------------- NEXT 1: M2PO
def m2po_mask(logp, old_logp, valid, tau: float):
    """M2PO second-moment trust masking (reading M1; "M2PO ... with
    m²-threshold 0.01" — the paper gives no formula, so this follows the M2PO definition it cites):

      delta_t = logp_t - old_t,  m_t = delta_t^2           for valid tokens (fp32, the kernel's
                                                            precision: the mask is a decision)
      order the valid tokens by m descending, ties by token index ascending;
      k* = the smallest k >= 0 such that the mean of m over the remaining n_valid - k tokens is
           <= tau (sums in fp64, left to right over the sorted order); k* = n_valid if none
      mask_t = 1 for the kept valid tokens, 0 for masked and invalid tokens.

    Returns (mask u8[N], k_star, m2_before, m2_after) with m2 = mean of m over the tokens kept."""
    lp = np.asarray(logp, dtype=np.float32)
    old = np.asarray(old_logp, dtype=np.float32)
    val = np.asarray(valid) != 0
    n = len(lp)
    d = (lp - old).astype(np.float32)
    m = (d * d).astype(np.float32)
    idx = [t for t in range(n) if val[t]]
    idx.sort(key=lambda t: (-float(m[t]), t))
    nv = len(idx)
    # suffix sums S_k = sum of m over sorted positions k..nv-1 (fp64, sequential from the end)
    suffix = [0.0] * (nv + 1)
    for i in range(nv - 1, -1, -1):
        suffix[i] = suffix[i + 1] + float(m[idx[i]])
    k_star = nv
    for k in range(nv):
        if suffix[k] / (nv - k) <= tau:
            k_star = k
            break
    mask = np.zeros(n, dtype=np.uint8)
    for i in range(k_star, nv):
        mask[idx[i]] = 1
    m2_before = suffix[0] / nv if nv else 0.0
    m2_after = suffix[k_star] / (nv - k_star) if nv > k_star else 0.0
    return mask, k_star, m2_before, m2_after
