"""Seeded parity cases shared by the GPU tests: inputs come from synth/ (generators) and,
for the behaviour log-probs, from the ORACLE's log-probs plus synth's seeded drift (never
from the CUDA path).  Expected values come only from oracle/."""
from __future__ import annotations

import math

import numpy as np

import oracle
import synth


def small_case(n_prompts=2, group=4, seq_len=64, vocab=1024, dtype="f32", seed=1, ld=None,
               mask_mode="prompt16", ignore_frac=0.05, staleness_max=0, max_staleness=-1,
               trainer_version=10, stale_outlier_frac=0.0, big_delta_frac=0.0,
               sigma_delta=0.05, force_zero_var_group=True):
    cfg = synth.SynthConfig("case", n_prompts, group, seq_len, vocab, dtype, seed, mask_mode,
                            ignore_frac=ignore_frac, force_zero_var_group=force_zero_var_group,
                            trainer_version=trainer_version, staleness_max=staleness_max,
                            stale_outlier_frac=stale_outlier_frac, sigma_delta=sigma_delta,
                            big_delta_frac=big_delta_frac, max_staleness=max_staleness)
    lay = synth.seq_layout(cfg)
    N = cfg.n_tokens
    ld = synth.pad_ld(vocab) if ld is None else ld
    x, y = synth.host_logits(vocab, np.arange(N), seed, dtype)
    if ld > vocab:
        pad = np.zeros((N, ld), dtype=x.dtype)
        pad[:, :vocab] = x
        xs = pad
    else:
        xs = x
    y = np.where(lay["ignore"] != 0, -100, y).astype(np.int32)
    x64 = oracle.decode_bf16(x) if dtype == "bf16" else x.astype(np.float64)
    ref_logp, _ = oracle.token_logprob(x64, y)
    tseq = np.repeat(np.arange(cfg.n_seq), seq_len).astype(np.int32)
    tstale = (trainer_version - lay["seq_version"])[tseq]
    old = synth.perturb_old_logp(np.where(y >= 0, ref_logp, 0.0), tstale, lay["big_delta"], cfg, seed)
    return dict(cfg=cfg, logits=xs, x64=x64, targets=y, old_logp=old, vocab=vocab, ld=ld,
                dtype=dtype, max_staleness=max_staleness, **lay)


def oracle_chain(case, params: oracle.LossParams, std_mode=oracle.STD_UNBIASED, eps=1e-6,
                 batch_norm=False, bn_eps=1e-6, rows=None, ref_logp=None, prox_logp=None,
                 want_entropy=False):
    """Advantages -> bookkeeping -> loss, all in the oracle (optionally on a row subset; the
    global normalisers always come from the full batch)."""
    bk = oracle.seq_bookkeeping(case["cu_seqlens"], case["loss_mask"], case["targets"],
                                case["vocab"], case["seq_version"], case["trainer_version"],
                                case["max_staleness"])
    adv, zv = oracle.group_advantage(case["rewards"], case["cu_groups"], std_mode, eps,
                                     batch_norm, bn_eps, bk["seq_active"])
    p = oracle.LossParams(**{**params.__dict__})
    p.global_active_tokens = bk["active_tokens"]
    p.trainer_version = case["trainer_version"]
    p.max_staleness = case["max_staleness"]
    if p.global_num_seqs == 0:
        p.global_num_seqs = len(case["rewards"])
    sel = np.arange(len(case["targets"])) if rows is None else np.asarray(rows)
    out = oracle.policy_loss_fwd_bwd(case["x64"][sel], case["targets"][sel], case["old_logp"][sel],
                                     case["loss_mask"][sel], bk["token_seq"][sel], adv,
                                     case["seq_version"], bk["seq_active"], p,
                                     ref_logp=None if ref_logp is None else np.asarray(ref_logp)[sel],
                                     prox_logp=None if prox_logp is None else np.asarray(prox_logp)[sel],
                                     want_entropy=want_entropy)
    return dict(bk=bk, adv=adv, zero_var=zv, loss=out, params=p, rows=sel)


def clip_band(ratio_ref, valid, eps_lo, eps_hi, width=1e-3):
    """Reading Z23: tokens whose reference log-ratio is within `width` of a clip boundary."""
    lr = np.log(np.where(valid != 0, np.maximum(ratio_ref, 1e-300), 1.0))
    return (valid != 0) & ((np.abs(lr - math.log(1 - eps_lo)) <= width) |
                           (np.abs(lr - math.log(1 + eps_hi)) <= width))
