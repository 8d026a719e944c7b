"""Pins of the fp64 CPU oracle (runs without a GPU).

Each test pins the oracle to something other than itself:
hand-worked examples (tests/golden/*.json, cited), closed forms, invariants,
an independent library route (torch CPU fp64 cross_entropy / autograd), finite
differences, and brute force.  Chosen so a dropped term, wrong sign, wrong index
or transposed operand in the oracle fails at least one of them.
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
from oracle import LossParams

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- c3 log-probs
def test_e1_worked_logprob():
    # V=3, x=[0, ln2, ln3], y=2 -> lse = ln 6, logp = -ln 2, p = [1/6,1/3,1/2]
    x = np.array([[0.0, math.log(2.0), math.log(3.0)]])
    logp, lse = oracle.token_logprob(x, [2])
    assert abs(lse[0] - math.log(6.0)) <= 2e-16 * 4
    assert abs(logp[0] + math.log(2.0)) <= 2e-16 * 4
    for y, pv in enumerate([1 / 6, 1 / 3, 1 / 2]):
        lp, _ = oracle.token_logprob(x, [y])
        assert abs(math.exp(lp[0]) - pv) < 1e-15


@pytest.mark.parametrize("V", [1, 7, 1024, 128256, 151936])
def test_constant_row_is_minus_log_v(V):
    # closed form: uniform logits give log(1/V) (BASELINE.json north_star)
    x = np.full((2, V), 3.25)
    logp, _ = oracle.token_logprob(x, [0, V - 1])
    assert np.allclose(logp, -math.log(V), atol=1e-12, rtol=0)


def test_logp_matches_torch_cross_entropy_fp64():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = rng.normal(size=(37, 53)) * 4
    y = rng.integers(0, 53, size=37)
    logp, _ = oracle.token_logprob(x, y)
    ref = -torch.nn.functional.cross_entropy(torch.tensor(x, dtype=torch.float64),
                                             torch.tensor(y), reduction="none").numpy()
    assert np.allclose(logp, ref, atol=1e-13, rtol=0)


def test_logp_shift_and_permutation_invariance():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(9, 31)) * 3
    y = rng.integers(0, 31, size=9)
    base, _ = oracle.token_logprob(x, y)
    shifted, _ = oracle.token_logprob(x + 123.5, y)
    assert np.allclose(base, shifted, atol=1e-12)
    perm = rng.permutation(31)
    inv = np.argsort(perm)
    permuted, _ = oracle.token_logprob(x[:, perm], inv[y])
    assert np.allclose(base, permuted, atol=1e-13)


def test_logp_ignore_and_bad_targets():
    x = np.zeros((3, 4))
    logp, _ = oracle.token_logprob(x, [-100, 4, 1])
    assert logp[0] == 0.0 and math.isnan(logp[1]) and abs(logp[2] + math.log(4)) < 1e-15


def test_temperature_scales_logits():
    rng = np.random.default_rng(2)
    x = rng.normal(size=(5, 11))
    y = rng.integers(0, 11, size=5)
    a, _ = oracle.token_logprob(x, y, inv_temperature=0.5)
    # closed form at T -> infinity (inv_T = 0): uniform -> -ln V
    b, _ = oracle.token_logprob(x, y, inv_temperature=0.0)
    c, _ = oracle.token_logprob(x * 0.5, y, inv_temperature=1.0)
    assert np.allclose(a, c, atol=1e-14)
    assert np.allclose(b, -math.log(11), atol=1e-14)


def test_all_neg_inf_row_gives_nan():
    x = np.full((1, 5), -np.inf)
    logp, _ = oracle.token_logprob(x, [2])
    assert math.isnan(logp[0])


def test_neg_inf_entries_are_probability_zero():
    x = np.array([[0.0, -np.inf, 0.0]])
    logp, _ = oracle.token_logprob(x, [0])
    assert abs(logp[0] + math.log(2)) < 1e-15


# ----------------------------------------------------------------------------- c1 advantages
def test_zero_advantage_spec_examples():
    g = _gold("spec_examples.json")
    for ex in g["zero_advantage"]:
        r = ex["rewards"]
        adv, zv = oracle.group_advantage(r, [0, len(r)])
        assert bool(zv[0]) == ex["zero"]
        if ex["zero"]:
            assert np.all(adv == 0) and not np.any(np.signbit(adv))


def test_zero_var_eight_tenths_is_exactly_zero():
    # eight copies of 0.1: sequential mean is 0.09999999999999999, d != 0 without the
    # special case (reading Z5); with it A must be exactly +0.0
    r = [0.1] * 8
    acc = 0.0
    for v in r:
        acc += v
    assert acc / 8 != 0.1          # the hazard the special case exists for
    adv, zv = oracle.group_advantage(r, [0, 8])
    assert zv[0] == 1 and np.all(adv == 0.0)


def test_empty_group_is_invalid():
    with pytest.raises(ValueError):
        oracle.group_advantage([1.0, 0.0], [0, 0, 2])


@pytest.mark.parametrize("k", range(0, 9))
def test_binary_closed_form_n8(k):
    # closed form for binary rewards: mean k/n, sum of squared deviations k(n-k)/n
    n, eps = 8, 1e-6
    r = [1.0] * k + [0.0] * (n - k)
    for mode, ddof in ((oracle.STD_UNBIASED, 1), (oracle.STD_BIASED, 0)):
        adv, zv = oracle.group_advantage(r, [0, n], std_mode=mode, eps=eps)
        if k in (0, n):
            assert zv[0] == 1 and np.all(adv == 0)
            continue
        sigma = math.sqrt(k * (n - k) / n / (n - ddof))
        ap, am = (1 - k / n) / (sigma + eps), (-k / n) / (sigma + eps)
        assert np.allclose(adv[:k], ap, rtol=2e-7) and np.allclose(adv[k:], am, rtol=2e-7)
    g = _gold("spec_examples.json")
    if str(k) in g["closed_form_binary_n8_unbiased_eps1e-6"]:
        ap, am = g["closed_form_binary_n8_unbiased_eps1e-6"][str(k)]
        adv, _ = oracle.group_advantage(r, [0, n])
        assert abs(adv[0] - ap) < 1e-6 and abs(adv[-1] - am) < 1e-6
    if str(k) in g["closed_form_binary_n8_biased_eps1e-6"]:
        ap, am = g["closed_form_binary_n8_biased_eps1e-6"][str(k)]
        adv, _ = oracle.group_advantage(r, [0, n], std_mode=oracle.STD_BIASED)
        assert abs(adv[0] - ap) < 1e-6 and abs(adv[-1] - am) < 1e-6


def test_pair_values():
    g = _gold("spec_examples.json")["pair_01"]
    a, _ = oracle.group_advantage([0.0, 1.0], [0, 2])
    assert a[1] == np.float32(g["unbiased"]) and a[0] == np.float32(-g["unbiased"])
    b, _ = oracle.group_advantage([0.0, 1.0], [0, 2], std_mode=oracle.STD_BIASED)
    assert b[1] == np.float32(g["biased"])


def test_std_none_is_mean_centering():
    a, _ = oracle.group_advantage([0.0, 1.0, 1.0, 1.0], [0, 4], std_mode=oracle.STD_NONE)
    assert np.allclose(a, [-0.75, 0.25, 0.25, 0.25])


def test_zero_predicate_brute_force_10000_groups():
    # agrees with brute-force pairwise equality on 10,000 random groups
    rng = random.Random(7)
    for _ in range(10000):
        n = rng.randint(1, 8)
        pool = [0.0, 1.0, 0.5, 0.1, 0.1 + 1e-17, 1e-300, -0.0]
        r = [rng.choice(pool) for _ in range(n)]
        brute = all(r[i] == r[j] for i in range(n) for j in range(n))
        _, zv = oracle.group_advantage(r, [0, n])
        assert bool(zv[0]) == brute


def test_advantages_sum_to_zero_and_affine_invariance():
    rng = np.random.default_rng(3)
    sizes = rng.integers(2, 17, size=50)
    cu = np.concatenate([[0], np.cumsum(sizes)])
    r = rng.normal(size=cu[-1])
    adv, _ = oracle.group_advantage(r, cu, eps=0.0)
    adv2, _ = oracle.group_advantage(3.5 * r - 2.0, cu, eps=0.0)
    for g in range(len(sizes)):
        seg = adv[cu[g]:cu[g + 1]].astype(np.float64)
        assert abs(seg.sum()) < 1e-5
        # unbiased std of standardized values is 1
        assert abs(np.std(seg, ddof=1) - 1.0) < 1e-5
    assert np.allclose(adv, adv2, atol=1e-5)


def test_advantages_permutation_equivariant_and_groups_independent():
    # SURVEY §8(c) group advantage: A_i depends only on r_i and its own group's moments, so
    # permuting members inside a group permutes A the same way, and changing another group's
    # rewards leaves this group's A untouched (a wrong segment index fails one of the two).
    rng = np.random.default_rng(11)
    sizes = rng.integers(2, 12, size=20)
    cu = np.concatenate([[0], np.cumsum(sizes)])
    r = rng.normal(size=cu[-1])
    adv, _ = oracle.group_advantage(r, cu, eps=1e-6)
    perm = np.arange(cu[-1])
    for g in range(len(sizes)):
        perm[cu[g]:cu[g + 1]] = cu[g] + rng.permutation(sizes[g])
    adv_p, _ = oracle.group_advantage(r[perm], cu, eps=1e-6)
    # summation order inside a group changes, so equal up to rounding of the moments
    assert np.allclose(np.asarray(adv_p), np.asarray(adv)[perm], rtol=0, atol=1e-6)
    r2 = r.copy()
    r2[cu[3]:cu[4]] = rng.normal(size=sizes[3]) * 10.0
    adv2, _ = oracle.group_advantage(r2, cu, eps=1e-6)
    keep = np.ones(cu[-1], bool)
    keep[cu[3]:cu[4]] = False
    assert np.array_equal(np.asarray(adv2)[keep], np.asarray(adv)[keep])


def test_batch_norm_token_weighted_moments():
    rng = np.random.default_rng(4)
    cu = np.arange(0, 65, 8)
    r = (rng.uniform(size=64) < 0.4).astype(np.float64)
    r[:8] = 1.0            # a zero-variance group (shifted by batch norm by design, Z6)
    L = rng.integers(0, 300, size=64)
    adv, zv = oracle.group_advantage(r, cu, batch_norm=True, bn_eps=0.0, seq_weight=L)
    a = adv.astype(np.float64)
    W = L.sum()
    mu = (L * a).sum() / W
    var = (L * (a - mu) ** 2).sum() / W
    assert abs(mu) < 1e-6 and abs(var - 1.0) < 1e-5
    assert zv[0] == 1 and adv[0] != 0.0


# ----------------------------------------------------------------------------- c2 bookkeeping
def test_staleness_spec_example():
    for ex in _gold("spec_examples.json")["staleness"]:
        bk = oracle.seq_bookkeeping([0, 3], [1, 1, 1], [0, 1, 2], 4, [ex["produced_at"]],
                                    ex["trainer_version"], ex["max_staleness"])
        assert (bk["active_tokens"] == 0) == ex["discarded"]
        assert bk["stale_masked"] == (3 if ex["discarded"] else 0)


def test_bookkeeping_brute_force():
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 20, size=30)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    N = int(cu[-1])
    mask = (rng.uniform(size=N) < 0.7).astype(np.uint8)
    V = 50
    y = rng.integers(-3, V + 3, size=N)
    ver = rng.integers(5, 14, size=30)
    bk = oracle.seq_bookkeeping(cu, mask, y, V, ver, 12, 4)
    seq = np.repeat(np.arange(30), lens)
    assert np.array_equal(bk["token_seq"], seq)
    stale = 12 - ver
    ok = (stale >= 0) & (stale <= 4)
    valid = (mask != 0) & (y >= 0) & (y < V) & ok[seq]
    assert np.array_equal(bk["valid"], valid.astype(np.uint8))
    assert np.array_equal(bk["seq_active"], np.bincount(seq[valid], minlength=30))
    assert bk["active_tokens"] == bk["seq_active"].sum() == valid.sum()
    assert bk["neg_staleness"] == (stale < 0).sum()
    assert bk["bad_targets"] == (y >= V).sum()
    assert bk["stale_masked"] == ((mask != 0) & (y >= 0) & (y < V) & (stale[seq] > 4)).sum()
    # staleness histogram: per sequence, bin min(s, 15); negative staleness not binned
    assert np.array_equal(bk["stale_hist"], np.bincount(np.minimum(stale[stale >= 0], 15), minlength=16))


def test_stale_hist_bins_and_clamp():
    # seven sequences with staleness -1, 0, 0, 3, 15, 16, 40 (trainer version 50): bins 0:2, 3:1, 15:3
    ver = [51, 50, 50, 47, 35, 34, 10]
    cu = np.arange(8) * 2
    bk = oracle.seq_bookkeeping(cu, np.ones(14, np.uint8), np.zeros(14, np.int64), 4, ver, 50, -1)
    expect = np.zeros(16, dtype=np.int64)
    expect[0], expect[3], expect[15] = 2, 1, 3
    assert np.array_equal(bk["stale_hist"], expect)
    assert bk["neg_staleness"] == 1 and bk["active_tokens"] == 12 and bk["stale_masked"] == 0


# ----------------------------------------------------------------------------- c4-c7 loss
def _e5():
    g = _gold("e5_policy_loss.json")
    x = np.array([[0.0 if k == 0 else math.log(k) for k in row] for row in g["logits_ln"]])
    y = np.array(g["targets"])
    logp, _ = oracle.token_logprob(x, y)
    old = logp - np.log(np.array(g["ratio"]))
    return g, x, y, old


def test_e5_worked_loss_and_gradient():
    g, x, y, old = _e5()
    p = LossParams(clip_eps_low=g["clip_eps"], clip_eps_high=g["clip_eps"], global_active_tokens=3)
    out = oracle.policy_loss_fwd_bwd(x, y, old, [1, 1, 1], [0, 1, 2], g["adv"], None, None, p)
    assert abs(out["loss"] - g["expected_loss"]) < 1e-14
    assert np.allclose(out["scale"], g["expected_scale"], atol=1e-14)
    assert list(out["clipped"]) == g["expected_clipped"]
    assert np.allclose(out["dlogits"], g["expected_dlogits"], atol=1e-14)


def test_e6_branches():
    for b in _gold("e5_policy_loss.json")["e6_branches"]:
        x = np.zeros((1, 4))
        logp, _ = oracle.token_logprob(x, [1])
        old = logp - math.log(b["r"])
        p = LossParams(agg=oracle.AGG_SUM)
        out = oracle.policy_loss_fwd_bwd(x, [1], old, [1], [0], [b["A"]], None, None, p)
        assert out["clipped"][0] == b["clipped"]
        assert abs(out["loss"] - b["L"]) < 1e-12
        assert (np.abs(out["dlogits"]).max() == 0) == b["grad_zero"]


def test_ratio_one_loss_is_minus_weighted_mean_adv():
    # E4 closed form: old = logp -> r = 1 -> L_t = -A -> loss = -(token-weighted mean of A)
    rng = np.random.default_rng(6)
    N, V, S = 40, 17, 5
    x = rng.normal(size=(N, V))
    y = rng.integers(0, V, size=N)
    logp, _ = oracle.token_logprob(x, y)
    tseq = np.sort(rng.integers(0, S, size=N))
    adv = rng.normal(size=S).astype(np.float32)
    mask = (rng.uniform(size=N) < 0.8).astype(np.uint8)
    p = LossParams(global_active_tokens=float(mask.sum()))
    out = oracle.policy_loss_fwd_bwd(x, y, logp, mask, tseq, adv, None, None, p)
    expect = -sum(float(adv[tseq[t]]) for t in range(N) if mask[t]) / mask.sum()
    assert abs(out["loss"] - expect) < 1e-12
    ones = np.ones(S, dtype=np.float32)
    out1 = oracle.policy_loss_fwd_bwd(x, y, logp, mask, tseq, ones, None, None, p)
    assert abs(out1["loss"] + 1.0) < 1e-15


def test_ratio_and_weight_sums_closed_forms():
    """stats ratio_sum / weight_sum against closed forms that do not involve the logits:
    old = logp - delta gives r_t = exp(clamp(delta_t)) for every valid token; weight_sum is 1 for
    TOKEN_MEAN with N_active = the valid count, (#sequences with L_i > 0) / S for
    SEQ_MEAN_TOKEN_MEAN, and the valid count for SUM; masked / stale / ignored tokens add nothing."""
    rng = np.random.default_rng(12)
    N, V, S = 60, 11, 6
    x = rng.normal(size=(N, V)) * 2
    y = rng.integers(0, V, size=N)
    y[::13] = -100
    logp, _ = oracle.token_logprob(x, y)
    delta = rng.normal(size=N) * 0.4
    delta[5], delta[6] = 30.0, -25.0          # beyond the log-ratio clamp c = 20
    old = logp - delta
    tseq = np.sort(rng.integers(0, S - 1, size=N))   # sequence S-1 has no tokens
    mask = (rng.uniform(size=N) < 0.75).astype(np.uint8)
    mask[5] = mask[6] = 1
    ver = np.full(S, 10)
    ver[2] = 5                                 # staleness 5 > max 3: masked
    valid = (mask != 0) & (y >= 0) & (tseq != 2)
    nv = int(valid.sum())
    L = np.bincount(tseq[valid], minlength=S)
    adv = rng.normal(size=S).astype(np.float32)
    r = np.exp(np.clip(delta, -20.0, 20.0))
    for agg, wsum in ((oracle.AGG_TOKEN_MEAN, 1.0), (oracle.AGG_SEQ_MEAN_TOKEN_MEAN, (L > 0).sum() / S),
                      (oracle.AGG_SUM, float(nv))):
        p = LossParams(agg=agg, global_active_tokens=float(nv), global_num_seqs=S, trainer_version=10,
                       max_staleness=3)
        out = oracle.policy_loss_fwd_bwd(x, y, old, mask, tseq, adv, ver, L, p)
        st = out["stats"]
        assert st["active_tokens"] == nv
        assert abs(st["ratio_sum"] - r[valid].sum()) <= 1e-12 * r[valid].sum()
        assert abs(st["weight_sum"] - wsum) <= 1e-12 * max(1.0, wsum)
        assert st["clamped"] == int(valid[5]) + int(valid[6])


def test_seq_mean_equals_token_mean_for_equal_lengths():
    rng = np.random.default_rng(8)
    S, T, V = 4, 6, 9
    x = rng.normal(size=(S * T, V))
    y = rng.integers(0, V, size=S * T)
    logp, _ = oracle.token_logprob(x, y)
    old = logp + rng.normal(size=S * T) * 0.3
    tseq = np.repeat(np.arange(S), T)
    adv = rng.normal(size=S).astype(np.float32)
    L = np.full(S, T)
    a = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(S * T), tseq, adv, None, L,
                                   LossParams(global_active_tokens=S * T))
    b = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(S * T), tseq, adv, None, L,
                                   LossParams(agg=oracle.AGG_SEQ_MEAN_TOKEN_MEAN, global_num_seqs=S))
    assert abs(a["loss"] - b["loss"]) < 1e-14
    assert np.allclose(a["dlogits"], b["dlogits"], atol=1e-16)


def _random_case(seed, N=12, V=13, S=3):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(N, V)) * 2
    y = rng.integers(0, V, size=N)
    logp, _ = oracle.token_logprob(x, y)
    old = logp + rng.normal(size=N) * 0.5
    tseq = np.sort(rng.integers(0, S, size=N))
    adv = rng.normal(size=S).astype(np.float32)
    return x, y, old, tseq, adv


def _loss_only(x, y, old, tseq, adv, p, clip_override):
    return oracle.policy_loss_fwd_bwd(x, y, old, np.ones(len(y)), tseq, adv, None, None, p,
                                      clip_override=clip_override, want_dlogits=False)["loss"]


@pytest.mark.parametrize("seed", range(6))
def test_gradient_finite_differences(seed):
    x, y, old, tseq, adv = _random_case(seed)
    p = LossParams(global_active_tokens=len(y), inv_temperature=0.7, grad_scale=1.0)
    out = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(len(y)), tseq, adv, None, None, p)
    # stay away from the clip kinks: skip tokens within 1e-4 of a clip boundary
    r = out["ratio"]
    near = (np.abs(r - 0.8) < 1e-4) | (np.abs(r - 1.2) < 1e-4)
    h = 1e-6
    num = np.zeros_like(x)
    for t in range(x.shape[0]):
        if near[t]:
            continue
        for v in range(x.shape[1]):
            xp = x.copy(); xp[t, v] += h
            xm = x.copy(); xm[t, v] -= h
            num[t, v] = (_loss_only(xp, y, old, tseq, adv, p, out["clipped"]) -
                         _loss_only(xm, y, old, tseq, adv, p, out["clipped"])) / (2 * h)
    ok = ~near
    assert np.allclose(num[ok], out["dlogits"][ok], atol=1e-8)


def test_gradient_matches_torch_autograd():
    torch = pytest.importorskip("torch")
    x, y, old, tseq, adv = _random_case(11, N=30, V=21, S=4)
    p = LossParams(global_active_tokens=30, clip_eps_low=0.2, clip_eps_high=0.28)
    out = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(30), tseq, adv, None, None, p)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    lp = torch.log_softmax(xt, dim=1).gather(1, torch.tensor(y)[:, None])[:, 0]
    r = torch.exp(lp - torch.tensor(old))
    A = torch.tensor(adv.astype(np.float64))[torch.tensor(tseq)]
    L = -torch.minimum(r * A, torch.clamp(r, 0.8, 1.28) * A)
    loss = L.sum() / 30
    loss.backward()
    assert abs(loss.item() - out["loss"]) < 1e-13
    assert np.allclose(xt.grad.numpy(), out["dlogits"], atol=1e-14)


def test_gradient_rows_sum_to_zero_and_masked_rows_zero():
    x, y, old, tseq, adv = _random_case(12, N=20, V=30)
    mask = np.ones(20, dtype=np.uint8); mask[[3, 7]] = 0
    y = y.copy(); y[5] = -100
    p = LossParams(global_active_tokens=17)
    out = oracle.policy_loss_fwd_bwd(x, y, old, mask, tseq, adv, None, None, p)
    assert np.all(np.abs(out["dlogits"].sum(axis=1)) < 1e-15 * 30)
    for t in (3, 5, 7):
        assert np.all(out["dlogits"][t] == 0)
    assert out["stats"]["active_tokens"] == 17 and out["logp"][5] == 0.0


def test_log_ratio_clamp_stops_gradient():
    x = np.zeros((2, 4))
    logp, _ = oracle.token_logprob(x, [0, 1])
    old = logp - np.array([25.0, 19.0])
    out = oracle.policy_loss_fwd_bwd(x, [0, 1], old, [1, 1], [0, 1], [-1.0, -1.0], None, None,
                                     LossParams(agg=oracle.AGG_SUM))
    assert abs(out["ratio"][0] - math.exp(20.0)) < 1e-6 * math.exp(20.0)
    assert out["stats"]["clamped"] == 1
    assert np.all(out["dlogits"][0] == 0) and np.any(out["dlogits"][1] != 0)


def test_staleness_masks_in_loss():
    x = np.zeros((4, 3))
    logp, _ = oracle.token_logprob(x, [0, 1, 2, 0])
    out = oracle.policy_loss_fwd_bwd(x, [0, 1, 2, 0], logp, [1, 1, 1, 1], [0, 0, 1, 2],
                                     [1.0, 1.0, 1.0], [20, 11, 21], None,
                                     LossParams(agg=oracle.AGG_SUM, trainer_version=20, max_staleness=8))
    assert list(out["valid"]) == [1, 1, 0, 0]
    assert out["stats"]["stale_masked"] == 1 and out["stats"]["neg_staleness"] == 1


def test_grad_scale_and_temperature_linear():
    x, y, old, tseq, adv = _random_case(13)
    a = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(12), tseq, adv, None, None,
                                   LossParams(global_active_tokens=12))
    b = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(12), tseq, adv, None, None,
                                   LossParams(global_active_tokens=12, grad_scale=3.0))
    assert np.allclose(3.0 * a["dlogits"], b["dlogits"], atol=1e-15)
    assert a["loss"] == b["loss"]


# ----------------------------------------------------------------------------- c8 vocab-parallel
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_vocab_split_combine_equals_unsplit(P):
    rng = np.random.default_rng(20 + P)
    V = 101
    x = rng.normal(size=(16, V)) * 5
    y = rng.integers(0, V, size=16)
    logp, lse = oracle.token_logprob(x, y)
    bounds = np.linspace(0, V, P + 1).astype(int)
    if P == 3:
        bounds = np.array([0, 0, 60, V])          # includes an empty shard
    ms, ss, xs = [], [], []
    for r in range(len(bounds) - 1):
        m, s, xy, _ = oracle.vocab_shard_stats(x[:, bounds[r]:bounds[r + 1]], y, bounds[r])
        ms.append(m); ss.append(s); xs.append(xy)
    lse2, zy = oracle.vocab_combine(ms, ss, xs)
    assert np.allclose(lse2, lse, atol=1e-12, rtol=0)
    assert np.allclose(zy - lse2, logp, atol=1e-12, rtol=0)


def test_parity_case_builder_runs_on_cpu():
    """The seeded case builder used by the GPU tests and smoke() (inputs only + oracle chain)."""
    from tests.cases import oracle_chain, small_case
    case = small_case()
    ref = oracle_chain(case, LossParams())
    assert ref["bk"]["active_tokens"] > 0 and ref["zero_var"][0] == 1
    assert np.isfinite(ref["loss"]["loss"])
    case = small_case(vocab=1003, ld=1008, dtype="bf16", staleness_max=8, stale_outlier_frac=0.3,
                      max_staleness=8, big_delta_frac=0.2)
    ref = oracle_chain(case, LossParams())
    assert ref["loss"]["stats"]["stale_masked"] > 0


# ----------------------------------------------------------------------------- NEXT 2 (N1-N3)
def _softmax(z):
    e = np.exp(z - z.max())
    return e / e.sum()


def test_k3_kl_is_unbiased_for_the_exact_kl():
    """N1 pin: the per-token k3 estimator KL_t = e^{ref-logp} - (ref-logp) - 1, averaged over
    targets drawn from pi (exact expectation over all V targets of one row), equals the closed-form
    KL(pi || pi_ref) = sum p log(p / p_ref) of the two distributions."""
    rng = np.random.default_rng(21)
    V = 7
    z, zr = rng.normal(size=V) * 1.5, rng.normal(size=V) * 1.5
    p, pr = _softmax(z), _softmax(zr)
    x = np.tile(z, (V, 1))
    y = np.arange(V)
    logp = np.log(p)
    ref = np.log(pr)
    out = oracle.policy_loss_fwd_bwd(x, y, logp, np.ones(V), np.zeros(V, dtype=int), [0.0], None, None,
                                     LossParams(agg=oracle.AGG_SUM, kl_coef=1.0), ref_logp=ref)
    per_token = out["token_loss"]   # A = 0: the surrogate is 0, L_t = KL_t (w = 1)
    assert abs(float(np.sum(p * per_token)) - float(np.sum(p * np.log(p / pr)))) < 1e-12
    assert np.all(per_token >= 0)
    assert abs(out["stats"]["kl_sum"] - float(np.sum(per_token))) < 1e-12


def test_kl_vanishes_at_the_reference_and_is_linear_in_beta():
    x, y, old, tseq, adv = _random_case(22)
    logp, _ = oracle.token_logprob(x, y)
    p0 = LossParams(global_active_tokens=len(y))
    base = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(len(y)), tseq, adv, None, None, p0)
    same = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(len(y)), tseq, adv, None, None,
                                      LossParams(global_active_tokens=len(y), kl_coef=0.5), ref_logp=logp)
    assert same["loss"] == base["loss"] and np.array_equal(same["dlogits"], base["dlogits"])
    ref = logp + np.random.default_rng(3).normal(size=len(y)) * 0.3
    b1 = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(len(y)), tseq, adv, None, None,
                                    LossParams(global_active_tokens=len(y), kl_coef=1e-3), ref_logp=ref)
    b2 = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(len(y)), tseq, adv, None, None,
                                    LossParams(global_active_tokens=len(y), kl_coef=2e-3), ref_logp=ref)
    assert abs((b2["loss"] - base["loss"]) - 2 * (b1["loss"] - base["loss"])) < 1e-14
    assert np.allclose(b2["dlogits"] - base["dlogits"], 2 * (b1["dlogits"] - base["dlogits"]), atol=1e-16)


def test_decoupled_ratio_reduces_to_the_standard_surrogate():
    """N2 pins: prox = old is the standard surrogate exactly; without clipping, rho * r =
    (pi_prox / pi_behav)(pi / pi_prox) = pi / pi_behav for ANY proximal policy, so loss and gradient
    equal the standard unclipped ones."""
    x, y, old, tseq, adv = _random_case(23)
    n = len(y)
    p = LossParams(global_active_tokens=n)
    std = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(n), tseq, adv, None, None, p)
    same = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(n), tseq, adv, None, None, p, prox_logp=old)
    assert same["loss"] == std["loss"] and np.array_equal(same["dlogits"], std["dlogits"])
    noclip = LossParams(global_active_tokens=n, clip_eps_low=1e9, clip_eps_high=1e9)
    prox = old + np.random.default_rng(4).normal(size=n) * 0.4
    a = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(n), tseq, adv, None, None, noclip)
    b = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(n), tseq, adv, None, None, noclip, prox_logp=prox)
    assert abs(a["loss"] - b["loss"]) < 1e-12
    assert np.allclose(a["dlogits"], b["dlogits"], atol=1e-14)


@pytest.mark.parametrize("seed", range(3))
def test_extended_objective_finite_differences(seed):
    """Gradient of the full objective (clipped decoupled surrogate + k3 KL) against central
    differences of the oracle's own loss."""
    x, y, old, tseq, adv = _random_case(30 + seed)
    n = len(y)
    rng = np.random.default_rng(40 + seed)
    logp, _ = oracle.token_logprob(x, y)
    prox = old + rng.normal(size=n) * 0.2
    ref = logp + rng.normal(size=n) * 0.5
    p = LossParams(global_active_tokens=n, kl_coef=0.3, inv_temperature=0.8)
    out = oracle.policy_loss_fwd_bwd(x, y, old, np.ones(n), tseq, adv, None, None, p, ref_logp=ref,
                                     prox_logp=prox)
    r = out["ratio"]
    near = (np.abs(r - 0.8) < 1e-4) | (np.abs(r - 1.2) < 1e-4)
    f = lambda xx: oracle.policy_loss_fwd_bwd(xx, y, old, np.ones(n), tseq, adv, None, None, p,
                                              clip_override=out["clipped"], want_dlogits=False,
                                              ref_logp=ref, prox_logp=prox)["loss"]
    h = 1e-6
    num = np.zeros_like(x)
    for t in range(n):
        if near[t]:
            continue
        for v in range(x.shape[1]):
            xp = x.copy(); xp[t, v] += h
            xm = x.copy(); xm[t, v] -= h
            num[t, v] = (f(xp) - f(xm)) / (2 * h)
    assert np.allclose(num[~near], out["dlogits"][~near], atol=1e-8)


def test_entropy_closed_forms_and_scipy():
    """N3 pins: a constant row has entropy ln V; random rows match scipy.stats.entropy of the
    softmax (natural log)."""
    scipy_stats = pytest.importorskip("scipy.stats")
    rng = np.random.default_rng(24)
    V = 50
    x = rng.normal(size=(6, V)) * 2
    x[0] = 3.0
    y = rng.integers(0, V, size=6)
    out = oracle.policy_loss_fwd_bwd(x, y, oracle.token_logprob(x, y)[0], np.ones(6), np.zeros(6, dtype=int),
                                     [1.0], None, None, LossParams(agg=oracle.AGG_SUM), want_entropy=True)
    assert abs(out["entropy"][0] - math.log(V)) < 1e-12
    for t in range(1, 6):
        assert abs(out["entropy"][t] - scipy_stats.entropy(_softmax(x[t]))) < 1e-12
    assert abs(out["stats"]["entropy_sum"] - math.fsum(out["entropy"])) < 1e-12


# ----------------------------------------------------------------------------- NEXT 1: M2PO (M1)
def test_m2po_mask_is_the_minimal_subset_by_brute_force():
    """M1 pin: over every subset of a tiny batch, the fewest tokens whose removal brings the kept
    mean of (logp - old)^2 to <= tau equals the oracle's k*, and its kept set satisfies the bound."""
    import itertools
    rng = np.random.default_rng(50)
    for trial in range(40):
        n = int(rng.integers(1, 11))
        lp = rng.normal(size=n).astype(np.float32)
        old = (lp + rng.normal(size=n) * rng.uniform(0.05, 1.0)).astype(np.float32)
        valid = (rng.random(n) < 0.85).astype(np.uint8)
        tau = float(rng.uniform(0.001, 0.5))
        mask, k, _, m2a = oracle.m2po_mask(lp, old, valid, tau)
        m = ((lp - old).astype(np.float32) ** 2).astype(np.float64)
        vidx = [t for t in range(n) if valid[t]]
        best = len(vidx)
        for r in range(len(vidx) + 1):                      # r = tokens removed
            ok = any(np.mean([m[t] for t in vidx if t not in drop]) <= tau
                     for drop in map(set, itertools.combinations(vidx, r)) if len(vidx) - r > 0)
            if ok:
                best = r
                break
        assert k == best, (trial, k, best)
        kept = [t for t in range(n) if mask[t]]
        assert all(valid[t] for t in kept) and len(kept) == len(vidx) - k
        if kept:
            assert np.mean([m[t] for t in kept]) <= tau and abs(m2a - np.mean([m[t] for t in kept])) < 1e-12


def test_m2po_limits():
    rng = np.random.default_rng(51)
    lp = rng.normal(size=50).astype(np.float32)
    old = (lp + rng.normal(size=50) * 0.3).astype(np.float32)
    valid = np.ones(50, dtype=np.uint8)
    mask, k, m2b, m2a = oracle.m2po_mask(lp, old, valid, 1e9)       # huge tau keeps everything
    assert k == 0 and mask.sum() == 50 and m2a == m2b
    mask, k, _, _ = oracle.m2po_mask(lp, lp, valid, 0.0)              # ratio 1: nothing to mask
    assert k == 0 and mask.sum() == 50
    mask, k, _, m2a = oracle.m2po_mask(lp, old, valid, 0.0)           # tau 0 keeps only m == 0 tokens
    assert k == 50 - int(np.sum(((lp - old).astype(np.float32) ** 2) == 0)) and m2a == 0.0
    # larger tau never masks more (monotone)
    ks = [oracle.m2po_mask(lp, old, valid, t)[1] for t in (0.01, 0.03, 0.1, 0.3)]
    assert ks == sorted(ks, reverse=True)


# ----------------------------------------------------------------------------- NEXT 3: delta scan
def test_delta_spec_examples():
    """identical snapshots -> empty, sparsity 1.0; [a,b,c,d] -> [a,x,c,d] ->
    [(1, x)], sparsity 0.75."""
    from oracle import delta
    a = np.array([1, 2, 3, 4], dtype=np.uint16)
    idx, w, s = delta.compute_delta(a, a)
    assert idx.size == 0 and s == 1.0
    b = a.copy(); b[1] = 0xBEEF
    idx, w, s = delta.compute_delta(a, b)
    assert list(idx) == [1] and list(w) == [0xBEEF] and s == 0.75


def test_delta_brute_force_round_trip_and_payload_bound():
    """Independent element-wise comparison (np.nonzero) on random pairs; apply(compute) = next;
    payload bound 6 (1 - s) N bytes."""
    from oracle import delta
    rng = np.random.default_rng(60)
    for n, frac in ((1000, 0.01), (1000, 0.5), (3, 1.0), (0, 0.0), (777, 0.0)):
        a = rng.integers(0, 1 << 16, size=n, dtype=np.uint16)
        b = a.copy()
        ch = rng.random(n) < frac
        b[ch] = b[ch] ^ rng.integers(1, 1 << 16, size=int(ch.sum()), dtype=np.uint16)
        idx, w, s = delta.compute_delta(a, b)
        assert np.array_equal(idx, np.nonzero(a != b)[0].astype(np.uint32)) and np.array_equal(w, b[idx])
        assert np.array_equal(delta.apply_delta(a, idx, w), b)
        assert 6 * idx.size <= 6 * (1 - s) * n + 1e-9
        assert np.all(np.diff(idx.astype(np.int64)) > 0)
    # bf16 bit patterns, not values: +0 and -0 differ, equal NaN payloads do not
    a = np.array([0x0000, 0x7FC0, 0x3F80], dtype=np.uint16)
    b = np.array([0x8000, 0x7FC0, 0x3F80], dtype=np.uint16)
    assert list(delta.compute_delta(a, b)[0]) == [0]


# ----------------------------------------------------------------------------- NEXT 4: LM head
def _bf16_bits(x):
    """fp64 values that are exactly bf16 -> their bit patterns (asserts exactness)."""
    f = np.asarray(x, dtype=np.float32)
    b = (f.view(np.uint32) >> 16).astype(np.uint16)
    assert np.array_equal((b.astype(np.uint32) << 16).view(np.float32), f)
    return b


def test_lmhead_closed_form():
    """h = e_0, W[:, 0] = a: x = a exactly, logp_y = a_y - ln sum_v e^{a_v} (pure-Python closed
    form) — a wrong operand order or a dropped row/column changes x."""
    a = [0.0, 1.0, 2.0, -3.5, 0.25]
    d = 4
    W = np.zeros((len(a), d))
    W[:, 0] = a
    W[:, 1] = 7.0       # multiplied by h[1] = 0: no contribution
    H = np.zeros((1, d))
    H[0, 0] = 1.0
    for y in range(len(a)):
        lp, lse = oracle.lmhead_logprob(_bf16_bits(H), _bf16_bits(W), [y])
        ref_lse = math.log(math.fsum(math.exp(v) for v in a))
        assert abs(lse[0] - ref_lse) < 1e-14 and abs(lp[0] - (a[y] - ref_lse)) < 1e-14


def test_lmhead_brute_force_rectangular():
    """N=3, d=5, V=4 (all different): x by explicit fsum dot products, log-softmax by fsum —
    a transposed weight (V x d vs d x V) or wrong row of h fails."""
    rng = np.random.default_rng(3)
    H = rng.integers(-8, 9, size=(3, 5)) / 4.0
    W = rng.integers(-8, 9, size=(4, 5)) / 8.0
    y = [0, 3, 1]
    lp, lse = oracle.lmhead_logprob(_bf16_bits(H), _bf16_bits(W), y, inv_temperature=0.5)
    for t in range(3):
        x = [0.5 * math.fsum(H[t, k] * W[v, k] for k in range(5)) for v in range(4)]
        m = max(x)
        ref = m + math.log(math.fsum(math.exp(v - m) for v in x))
        assert abs(lse[t] - ref) < 1e-13 and abs(lp[t] - (x[y[t]] - ref)) < 1e-13


def test_lmhead_invariants():
    """Equal weight rows -> logp = -ln V for any h; a common vector added to
    every weight row (x_v += h.c) and a permutation of the vocabulary rows with relabelled targets
    leave logp unchanged."""
    rng = np.random.default_rng(5)
    N, d, V = 6, 16, 37
    H = np.round(rng.normal(size=(N, d)) * 8) / 8
    W = np.round(rng.normal(size=(V, d)) * 8) / 8
    y = rng.integers(0, V, size=N)
    row = np.round(rng.normal(size=d) * 4) / 4
    lp_c, _ = oracle.lmhead_logprob(_bf16_bits(H), _bf16_bits(np.tile(row, (V, 1))), y)
    assert np.allclose(lp_c, -math.log(V), atol=1e-13, rtol=0)
    lp, _ = oracle.lmhead_logprob(_bf16_bits(H), _bf16_bits(W), y)
    c = np.round(rng.normal(size=d) * 2) / 2
    lp_s, _ = oracle.lmhead_logprob(_bf16_bits(H), _bf16_bits(W + c), y)
    assert np.allclose(lp_s, lp, atol=1e-11, rtol=0)
    perm = rng.permutation(V)
    inv = np.argsort(perm)
    lp_p, _ = oracle.lmhead_logprob(_bf16_bits(H), _bf16_bits(W[perm]), inv[y])
    assert np.allclose(lp_p, lp, atol=1e-13, rtol=0)


def test_lmhead_torch_route():
    """Independent library route: -cross_entropy(h @ W^T) in torch CPU fp64."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    N, d, V = 5, 64, 300
    hb = _bf16_bits(np.round(rng.normal(size=(N, d)) * 16) / 16)
    wb = _bf16_bits(np.round(rng.normal(size=(V, d)) * 16) / 64)
    y = rng.integers(0, V, size=N)
    lp, _ = oracle.lmhead_logprob(hb, wb, y)
    h = torch.from_numpy((hb.astype(np.uint32) << 16).view(np.float32).astype(np.float64))
    w = torch.from_numpy((wb.astype(np.uint32) << 16).view(np.float32).astype(np.float64))
    ref = -torch.nn.functional.cross_entropy(h @ w.T, torch.from_numpy(y), reduction="none")
    assert np.allclose(lp, ref.numpy(), atol=1e-12, rtol=0)


def _lm_objective_torch(H, W, y, s, invT):
    """F(h, W) = sum_t (s_t / invT) (-log softmax((h W^T) invT)[y_t]) in torch CPU fp64: its
    gradients are dh = G W and dW = G^T h with G = s (p - onehot) (independent autograd route)."""
    import torch
    x = (H @ W.T) * invT
    lp = torch.log_softmax(x, dim=1)
    ok = (y >= 0) & (y < W.shape[0])
    yy = torch.where(ok, y, torch.zeros_like(y))
    return -(torch.where(ok, s / invT, torch.zeros_like(s)) * lp.gather(1, yy[:, None])[:, 0]).sum()


def test_lmhead_backward_matches_torch_autograd():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(71)
    N, d, V = 7, 6, 11
    H = rng.integers(-16, 17, size=(N, d)) / 8.0
    W = rng.integers(-16, 17, size=(V, d)) / 16.0
    y = np.array([0, 10, 3, -100, 5, 11, 7])      # an ignored and an out-of-range target: G row 0
    s = rng.normal(size=N)
    for invT in (1.0, 0.7):
        dh, dW, G = oracle.lmhead_loss_backward(_bf16_bits(H), _bf16_bits(W), y, s, invT)
        Ht = torch.tensor(H, dtype=torch.float64, requires_grad=True)
        Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
        _lm_objective_torch(Ht, Wt, torch.tensor(y), torch.tensor(s), invT).backward()
        assert np.allclose(dh, Ht.grad.numpy(), atol=1e-12, rtol=1e-12)
        assert np.allclose(dW, Wt.grad.numpy(), atol=1e-12, rtol=1e-12)
        assert np.all(G[3] == 0) and np.all(G[5] == 0)
        assert np.allclose(G.sum(axis=1), 0.0, atol=1e-12)      # rows of softmax - onehot sum to 0


def test_lmhead_backward_finite_differences():
    """Central differences of F (pure NumPy, no autograd) at every entry of h and of W."""
    rng = np.random.default_rng(72)
    N, d, V = 4, 3, 5
    H = rng.integers(-8, 9, size=(N, d)) / 8.0
    W = rng.integers(-8, 9, size=(V, d)) / 8.0
    y = np.array([1, 4, 0, 2])
    s = np.array([0.5, -1.25, 2.0, 0.75])
    invT = 0.8

    def F(Hm, Wm):
        x = (Hm @ Wm.T) * invT
        m = x.max(axis=1, keepdims=True)
        lse = (m + np.log(np.exp(x - m).sum(axis=1, keepdims=True)))[:, 0]
        return float(np.sum((s / invT) * (lse - x[np.arange(N), y])))

    dh, dW, _ = oracle.lmhead_loss_backward(_bf16_bits(H), _bf16_bits(W), y, s, invT)
    eps = 1e-6
    for M, grad in ((H, dh), (W, dW)):
        for idx in np.ndindex(M.shape):
            Mp, Mm = M.copy(), M.copy()
            Mp[idx] += eps
            Mm[idx] -= eps
            fd = (F(Mp, W) - F(Mm, W)) / (2 * eps) if M is H else (F(H, Mp) - F(H, Mm)) / (2 * eps)
            assert abs(fd - grad[idx]) <= 1e-7, (idx, fd, grad[idx])
