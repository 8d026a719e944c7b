"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  Tolerances (BASELINE.json north_star; readings Z21-Z23 in DESIGN.md §3):
advantages / masks / integer bookkeeping bit-exact; logp <= 2e-3 absolute; loss <= 1e-4
relative (Z22 scale); dlogits per row max|d| <= 1e-2*|s_t| (Z21) and literal 1e-2 absolute
in unit-scale (SUM) mode; clip flags exact outside the Z23 band; masked rows bitwise zero.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.cases import clip_band, oracle_chain, small_case

pytestmark = pytest.mark.gpu

LOGP_ATOL = 2e-3
LOSS_RTOL = 1e-4
DLOGIT_ROW_RTOL = 1e-2


def torch():
    import torch as t
    return t


def dev(a):
    t = torch()
    if a.dtype == np.uint16:
        return t.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(t.bfloat16)
    return t.from_numpy(np.ascontiguousarray(a)).cuda()


def host_logits(tns):
    t = torch()
    if tns.dtype == t.bfloat16:
        return oracle.decode_bf16(tns.view(t.int16).cpu().numpy().view(np.uint16))
    return tns.cpu().numpy().astype(np.float64)


def run_gpu_chain(rl, case, params, std_mode=0, eps=1e-6, batch_norm=False, bn_eps=1e-6,
                  in_place=False, want=("logp", "clipped"), ref_logp=None, prox_logp=None,
                  want_entropy=False):
    t = torch()
    N, S, G = len(case["targets"]), len(case["rewards"]), len(case["cu_groups"]) - 1
    logits = dev(case["logits"])
    targets = dev(case["targets"])
    cu = dev(case["cu_seqlens"])
    mask = dev(case["loss_mask"])
    ver = dev(case["seq_version"])
    tok_seq = t.empty(N, dtype=t.int32, device="cuda")
    seq_active = t.empty(S, dtype=t.int32, device="cuda")
    counts = t.zeros(20, dtype=t.float64, device="cuda")
    rl.seq_bookkeeping(cu, targets, case["vocab"], tok_seq, seq_active, loss_mask=mask,
                       seq_version=ver, trainer_version=case["trainer_version"],
                       max_staleness=case["max_staleness"], counts_out=counts)
    adv = t.empty(S, dtype=t.float32, device="cuda")
    zv = t.empty(G, dtype=t.uint8, device="cuda")
    ws_adv = t.empty(max(1, rl.group_advantage_workspace_size(S)), dtype=t.uint8, device="cuda")
    rl.group_advantage(dev(case["rewards"]), dev(case["cu_groups"]), adv, zv, std_mode=std_mode,
                       eps=eps, batch_norm=batch_norm, bn_eps=bn_eps, seq_weight=seq_active,
                       workspace=ws_adv)
    p = rl.LossParams(**params)
    if ref_logp is not None:
        p.ref_logp = dev(np.asarray(ref_logp, dtype=np.float32))
    if prox_logp is not None:
        p.prox_logp = dev(np.asarray(prox_logp, dtype=np.float32))
    if want_entropy:
        p.flags |= rl.F_ENTROPY
    p.trainer_version = case["trainer_version"]
    p.max_staleness = case["max_staleness"]
    if p.global_num_seqs == 0:
        p.global_num_seqs = S
    p.active_tokens_dev = counts[0:1]
    dl = logits if in_place else t.empty_like(logits)
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    ws = t.empty(rl.policy_loss_workspace_size(N, case["vocab"]), dtype=t.uint8, device="cuda")
    logp = t.empty(N, dtype=t.float32, device="cuda")
    clipped = t.empty(N, dtype=t.uint8, device="cuda")
    rl.policy_loss_fwd_bwd(logits, targets, dev(case["old_logp"]), tok_seq, adv, p, dl, stats, ws,
                           loss_mask=mask, seq_version=ver, seq_active=seq_active, logp_out=logp,
                           clipped_out=clipped, vocab=case["vocab"])
    t.cuda.synchronize()
    return dict(adv=adv.cpu().numpy(), zero_var=zv.cpu().numpy(), token_seq=tok_seq.cpu().numpy(),
                seq_active=seq_active.cpu().numpy(), counts=counts.cpu().numpy(),
                logp=logp.cpu().numpy(), clipped=clipped.cpu().numpy(),
                dlogits=host_logits(dl)[:, :case["vocab"]], stats=stats.cpu().numpy())


def check_against_oracle(case, g, params, ref_logp=None, prox_logp=None, want_entropy=False, **adv_kw):
    ref = oracle_chain(case, oracle.LossParams(**params), ref_logp=ref_logp, prox_logp=prox_logp,
                       want_entropy=want_entropy, **adv_kw)
    out = ref["loss"]
    # --- bit-exact parts
    assert np.array_equal(g["adv"].view(np.uint32), ref["adv"].view(np.uint32)), "advantages"
    assert np.array_equal(g["zero_var"], ref["zero_var"])
    assert np.array_equal(g["token_seq"], ref["bk"]["token_seq"])
    assert np.array_equal(g["seq_active"], ref["bk"]["seq_active"])
    assert g["counts"][0] == ref["bk"]["active_tokens"]
    # --- logp
    y = case["targets"]
    V = case["vocab"]
    inr = (y >= 0) & (y < V)
    a, b = g["logp"][inr], out["logp"][inr]
    same = (a == b) | (np.isnan(a) & np.isnan(b))          # -inf / NaN rows (special values)
    with np.errstate(invalid="ignore"):
        assert np.all(same | (np.abs(a - b) <= LOGP_ATOL)), np.abs(a - b)[~same].max()
    assert np.all(g["logp"][y < 0] == 0)
    assert np.all(np.isnan(g["logp"][y >= V]))
    # --- clip decisions: exact outside the tie band (Z23); inside, adopt the GPU's decision
    eps_lo, eps_hi = params.get("clip_eps_low", 0.2), params.get("clip_eps_high", 0.2)
    band = clip_band(out["ratio"], out["valid"], eps_lo, eps_hi)
    assert np.array_equal(g["clipped"][~band], out["clipped"][~band])
    if band.any():
        override = np.where(band, g["clipped"], out["clipped"])
        out = oracle.policy_loss_fwd_bwd(case["x64"], y, case["old_logp"], case["loss_mask"],
                                         ref["bk"]["token_seq"], ref["adv"], case["seq_version"],
                                         ref["bk"]["seq_active"], ref["params"], clip_override=override,
                                         ref_logp=ref_logp, prox_logp=prox_logp, want_entropy=want_entropy)
    # --- loss (Z22)
    scale = max(abs(out["loss"]), float(np.abs(out["token_loss"]).sum()), 1e-30)
    assert abs(g["stats"][0] - out["loss"]) <= LOSS_RTOL * scale, (g["stats"][0], out["loss"])
    st = out["stats"]
    assert g["stats"][1] == st["active_tokens"]
    assert abs(g["stats"][3] - st["ratio_sum"]) <= 1e-4 * max(1.0, st["ratio_sum"])
    assert g["stats"][4] == st["clipped_low"] and g["stats"][5] == st["clipped_high"]
    assert g["stats"][6] == st["clamped"] and g["stats"][7] == st["stale_masked"]
    assert g["stats"][8] == st["bad_targets"] and g["stats"][9] == st["neg_staleness"]
    # NEXT-2 sums: KL (weighted like the loss) and entropy (per valid token; fp32 cancellation in
    # lse - sum p z, ~1e-5 nats per token)
    assert abs(g["stats"][10] - st["kl_sum"]) <= 1e-3 * abs(st["kl_sum"]) + 1e-7, (g["stats"][10], st["kl_sum"])
    if want_entropy:
        assert abs(g["stats"][11] - st["entropy_sum"]) <= 1e-4 * abs(st["entropy_sum"]) + 1e-4 * st["active_tokens"], \
            (g["stats"][11], st["entropy_sum"])
    else:
        assert g["stats"][11] == 0
    # --- dlogits (Z21): zero rows exactly zero, other rows relative to |s_t|
    s = out["scale"]
    d = g["dlogits"]
    zero_rows = s == 0
    assert np.all(d[zero_rows] == 0), "rows with s_t = 0 must be exact zeros"
    nz = ~zero_rows
    if nz.any():
        err = np.abs(d[nz] - out["dlogits"][nz]).max(axis=1)
        assert np.all(err <= DLOGIT_ROW_RTOL * np.abs(s[nz])), (err / np.abs(s[nz])).max()
    return out


# ----------------------------------------------------------------------------- advantages
@pytest.mark.parametrize("std_mode", [0, 1, 2])
@pytest.mark.parametrize("bn", [False, True])
def test_group_advantage_bit_exact(cuda_lib, std_mode, bn):
    rl, t = cuda_lib, torch()
    rng = np.random.default_rng(100 + std_mode + 3 * bn)
    sizes = np.concatenate([[1, 1, 8, 8, 16, 3, 2], rng.integers(1, 17, size=200)])
    cu = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    S = int(cu[-1])
    kinds = [lambda n: (rng.uniform(size=n) < 0.5).astype(float),
             lambda n: np.full(n, 0.1),
             lambda n: rng.normal(size=n) * 1e3,
             lambda n: rng.choice([0.1, 0.2, 0.3, 1e-17, 0.1 + 1e-17], size=n),
             lambda n: rng.uniform(size=n)]
    r = np.concatenate([kinds[g % len(kinds)](n) for g, n in enumerate(sizes)])
    L = rng.integers(0, 4000, size=S).astype(np.int32)
    ref_adv, ref_zv = oracle.group_advantage(r, cu, std_mode, 1e-6, bn, 1e-6, L)
    adv = t.empty(S, dtype=t.float32, device="cuda")
    zv = t.empty(len(sizes), dtype=t.uint8, device="cuda")
    ws = t.empty(rl.group_advantage_workspace_size(S), dtype=t.uint8, device="cuda")
    rl.group_advantage(dev(r), dev(cu), adv, zv, std_mode=std_mode, batch_norm=bn,
                       seq_weight=dev(L), workspace=ws)
    assert np.array_equal(adv.cpu().numpy().view(np.uint32), ref_adv.view(np.uint32))
    assert np.array_equal(zv.cpu().numpy(), ref_zv)


def test_group_advantage_invalid_group_flagged(cuda_lib):
    rl, t = cuda_lib, torch()
    cu = np.array([0, 2, 2, 4], dtype=np.int32)  # group 1 is empty
    r = np.array([0.0, 1.0, 1.0, 1.0])
    adv = t.full((4,), 7.0, dtype=t.float32, device="cuda")
    zv = t.empty(3, dtype=t.uint8, device="cuda")
    rl.group_advantage(dev(r), dev(cu), adv, zv)
    assert list(zv.cpu().numpy()) == [0, 2, 1]
    ref, _ = oracle.group_advantage(r, [0, 2, 4])
    assert np.array_equal(adv.cpu().numpy(), ref)


# ----------------------------------------------------------------------------- bookkeeping
def test_seq_bookkeeping_exact(cuda_lib):
    rl, t = cuda_lib, torch()
    rng = np.random.default_rng(7)
    lens = np.concatenate([[0, 5, 0, 33], rng.integers(0, 700, size=60), [0]])
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    S, N, V = len(lens), int(cu[-1]), 1000
    mask = (rng.uniform(size=N) < 0.6).astype(np.uint8)
    y = rng.integers(-2, V + 2, size=N).astype(np.int32)
    ver = rng.integers(3, 14, size=S).astype(np.int32)
    sadv = rng.normal(size=S).astype(np.float32)
    ref = oracle.seq_bookkeeping(cu, mask, y, V, ver, 12, 8)
    tok, act, stale = (t.empty(N, dtype=t.int32, device="cuda"), t.empty(S, dtype=t.int32, device="cuda"),
                       t.empty(S, dtype=t.int32, device="cuda"))
    advt, valid = t.empty(N, dtype=t.float32, device="cuda"), t.empty(N, dtype=t.uint8, device="cuda")
    counts = t.empty(20, dtype=t.float64, device="cuda")
    rl.seq_bookkeeping(dev(cu), dev(y), V, tok, act, loss_mask=dev(mask), seq_version=dev(ver),
                       trainer_version=12, max_staleness=8, seq_adv=dev(sadv), seq_staleness_out=stale,
                       adv_token_out=advt, valid_out=valid, counts_out=counts)
    assert np.array_equal(tok.cpu().numpy(), ref["token_seq"])
    assert np.array_equal(act.cpu().numpy(), ref["seq_active"])
    assert np.array_equal(stale.cpu().numpy(), ref["seq_staleness"])
    assert np.array_equal(valid.cpu().numpy(), ref["valid"])
    assert np.array_equal(advt.cpu().numpy(), sadv[ref["token_seq"]])
    c = counts.cpu().numpy()
    assert c[0] == ref["active_tokens"] and c[1] == ref["stale_masked"]
    assert c[2] == ref["neg_staleness"] and c[3] == ref["bad_targets"]
    assert np.array_equal(c[4:20], ref["stale_hist"])


# ----------------------------------------------------------------------------- log-probs
@pytest.mark.parametrize("V,ld,dtype", [(1024, 1024, "f32"), (1003, 1008, "bf16"), (5, 8, "bf16"),
                                        (1, 8, "bf16"), (1001, 1004, "f32"), (151936, 151936, "bf16")])
def test_token_logprob(cuda_lib, V, ld, dtype):
    rl, t = cuda_lib, torch()
    R = 40 if V > 100000 else 300
    x, y = synth.host_logits(V, np.arange(R), 31, dtype)
    y = y.copy()
    y[3], y[5] = -100, V  # ignored and bad targets
    xs = np.zeros((R, ld), dtype=x.dtype)
    xs[:, :V] = x
    x64 = oracle.decode_bf16(x) if dtype == "bf16" else x.astype(np.float64)
    ref, ref_lse = oracle.token_logprob(x64, y)
    logp, lse = t.empty(R, device="cuda"), t.empty(R, device="cuda")
    bad = t.zeros(1, dtype=t.float64, device="cuda")
    rl.token_logprob(dev(xs), dev(y), logp, lse, vocab=V, bad_target_count=bad)
    g = logp.cpu().numpy()
    ok = (y >= 0) & (y < V)
    assert np.all(np.abs(g[ok] - ref[ok]) <= LOGP_ATOL)
    assert np.all(np.abs(lse.cpu().numpy() - ref_lse) <= LOGP_ATOL)
    assert g[3] == 0 and math.isnan(g[5]) and bad.item() == 1


def test_token_logprob_special_values(cuda_lib):
    rl, t = cuda_lib, torch()
    x = np.zeros((3, 64), dtype=np.float32)
    x[0, 1:] = -np.inf            # one finite entry: logp = 0
    x[1, :] = -np.inf             # all -inf: NaN
    x[2, 7] = np.inf              # +inf propagates: NaN
    logp = t.empty(3, device="cuda")
    rl.token_logprob(dev(x), dev(np.array([0, 0, 7], dtype=np.int32)), logp)
    g = logp.cpu().numpy()
    ref, _ = oracle.token_logprob(x.astype(np.float64), [0, 0, 7])
    assert g[0] == 0.0 and ref[0] == 0.0
    assert math.isnan(g[1]) and math.isnan(ref[1]) and math.isnan(g[2]) and math.isnan(ref[2])


# ----------------------------------------------------------------------------- fused loss
def test_tiny_config_full_parity(cuda_lib):
    """BASELINE.json configs[0]: 2 x 4 x 64 tokens, V = 1024, fp32 logits — every output."""
    case = small_case()
    g = run_gpu_chain(cuda_lib, case, {})
    out = check_against_oracle(case, g, {})
    assert out["stats"]["active_tokens"] > 0


@pytest.mark.parametrize("kw", [
    dict(vocab=5003, ld=5008, dtype="bf16", n_prompts=3, group=5, seq_len=41, seed=3),
    dict(vocab=4096, ld=4096, dtype="bf16", n_prompts=2, group=8, seq_len=37, seed=4,
         staleness_max=8, stale_outlier_frac=0.3, max_staleness=8, big_delta_frac=0.2),
    dict(vocab=777, ld=780, dtype="f32", n_prompts=4, group=3, seq_len=29, seed=5, mask_mode="all",
         big_delta_frac=0.3, sigma_delta=0.3),
])
@pytest.mark.parametrize("in_place", [False, True])
def test_loss_parity_ragged(cuda_lib, kw, in_place):
    case = small_case(**kw)
    g = run_gpu_chain(cuda_lib, case, {}, in_place=in_place)
    check_against_oracle(case, g, {})


@pytest.mark.parametrize("params", [
    dict(agg=oracle.AGG_SEQ_MEAN_TOKEN_MEAN),
    dict(clip_eps_low=0.2, clip_eps_high=0.28),
    dict(inv_temperature=0.7, grad_scale=2.5),
])
def test_loss_parity_knobs(cuda_lib, params):
    case = small_case(vocab=2048, dtype="bf16", seed=9, big_delta_frac=0.1, sigma_delta=0.2)
    g = run_gpu_chain(cuda_lib, case, params, batch_norm=True)
    check_against_oracle(case, g, params, batch_norm=True)


def test_unit_scale_literal_dlogit_tolerance(cuda_lib):
    """Z21: in SUM mode (w = 1) with |A r| <= ~2 the literal 1e-2 absolute bound is meaningful."""
    case = small_case(vocab=3000, dtype="bf16", seed=12, sigma_delta=0.05)
    params = dict(agg=oracle.AGG_SUM)
    g = run_gpu_chain(cuda_lib, case, params)
    out = check_against_oracle(case, g, params)
    assert np.abs(g["dlogits"] - out["dlogits"]).max() <= 1e-2


def test_all_masked_batch_and_determinism(cuda_lib):
    case = small_case(vocab=1024, seed=13)
    case["loss_mask"][:] = 0
    g = run_gpu_chain(cuda_lib, case, {})
    assert g["stats"][0] == 0 and g["stats"][1] == 0 and np.all(g["dlogits"] == 0)
    case = small_case(vocab=3000, dtype="bf16", seed=14)
    a = run_gpu_chain(cuda_lib, case, {})
    b = run_gpu_chain(cuda_lib, case, {})
    assert a["stats"].tobytes() == b["stats"].tobytes()
    assert a["dlogits"].tobytes() == b["dlogits"].tobytes() and a["logp"].tobytes() == b["logp"].tobytes()


@pytest.mark.parametrize("kw,in_place", [
    (dict(vocab=5003, ld=5008, dtype="bf16", n_prompts=3, group=5, seq_len=41, seed=31, big_delta_frac=0.1,
          sigma_delta=0.15), False),
    (dict(vocab=777, ld=780, dtype="f32", n_prompts=2, group=4, seq_len=33, seed=32, sigma_delta=0.2), True),
])
def test_extended_objective(cuda_lib, kw, in_place):
    """NEXT 2 (readings N1-N3): k3 KL vs reference log-probs, decoupled proximal ratio and the
    entropy sum, against the oracle on the same inputs."""
    case = small_case(**kw)
    y = case["targets"]
    lp, _ = oracle.token_logprob(case["x64"], y)
    rng = np.random.default_rng(kw["seed"])
    ref = np.where(y >= 0, lp, 0.0) + rng.normal(size=len(y)) * 0.3
    prox = case["old_logp"] + rng.normal(size=len(y)) * 0.05
    params = dict(kl_coef=0.05, clip_eps_low=0.2, clip_eps_high=0.28)
    g = run_gpu_chain(cuda_lib, case, params, in_place=in_place, ref_logp=ref, prox_logp=prox, want_entropy=True)
    out = check_against_oracle(case, g, params, ref_logp=ref.astype(np.float32).astype(np.float64),
                               prox_logp=prox.astype(np.float32).astype(np.float64), want_entropy=True)
    assert out["stats"]["kl_sum"] > 0 and out["stats"]["entropy_sum"] > 0


def set_logits(case, row, cols, value):
    """Overwrite logits[row, cols] in both the device input (bf16 bits / fp32) and the oracle's copy."""
    v = np.float32(value)
    if case["dtype"] == "bf16":
        bits = synth.bf16_round_bits(np.array([v]))[0]
        case["logits"][row, cols] = bits
        case["x64"][row, cols] = oracle.decode_bf16(np.array([bits], dtype=np.uint16))[0]
    else:
        case["logits"][row, cols] = v
        case["x64"][row, cols] = float(v)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_extreme_rows(cuda_lib, dtype):
    """Rows far from the synthetic distribution: the single-visit kernel's exponent reference is
    the target logit, so a target ~100 nats below the row max (or a -inf target, or inf / NaN
    logits) takes the exact two-pass fixup; a 60-nat gap stays on the fast path (e' ~ 2^101)."""
    case = small_case(vocab=5003, ld=5008, dtype=dtype, seed=21, mask_mode="all", ignore_frac=0.0,
                      n_prompts=2, group=4, seq_len=16)
    y = case["targets"]
    adv = oracle_chain(case, oracle.LossParams())["adv"]
    live = [s for s in range(len(adv)) if adv[s] != 0]          # sequences with a gradient
    ra, rb, rc, rd = (live[i] * 16 + 3 for i in range(4))        # rows in distinct live sequences
    other = lambda r: (int(y[r]) + 1 + 7 * r) % case["vocab"]  # a column that is not the target
    set_logits(case, ra, y[ra], -40.0); set_logits(case, ra, other(ra), 60.0)  # gap 100: redo
    set_logits(case, rb, y[rb], -20.0); set_logits(case, rb, other(rb), 40.0)  # gap 60: fast
    rn, ri, rt = (s * 16 + 9 for s in range(3))
    set_logits(case, rn, other(rn), np.nan); case["loss_mask"][rn] = 0         # NaN, masked
    set_logits(case, ri, other(ri), np.inf); case["loss_mask"][ri] = 0         # +inf, masked
    set_logits(case, rt, y[rt], -np.inf)                                       # -inf target
    set_logits(case, rc, slice(None), -np.inf); set_logits(case, rc, y[rc], 1.5)  # one finite
    set_logits(case, rd, slice(None), 3.0)                                      # constant row
    lp, _ = oracle.token_logprob(case["x64"], y)
    for r in (ra, rb, rc, rd):  # behaviour log-probs near the new values: unclipped gradients
        case["old_logp"][r] = lp[r] + 0.01
    g = run_gpu_chain(cuda_lib, case, {})
    out = check_against_oracle(case, g, {})
    assert np.isnan(g["logp"][rn]) and np.isnan(g["logp"][ri]) and g["logp"][rt] == -np.inf
    assert abs(g["logp"][rc]) <= 1e-6 and abs(g["logp"][rd] + math.log(case["vocab"])) <= LOGP_ATOL
    assert out["scale"][ra] != 0 and out["scale"][rb] != 0 and out["scale"][rc] != 0


def test_rows_sum_to_zero_bf16(cuda_lib):
    """Invariant: each gradient row sums to ~0 within the bound derived in DESIGN.md §3 R2:
    |sum_v d_v| <= 3u / (1 - u) max|d| + 2^-16 |s_t| (u = 2^-8: <= 2 bf16 roundings per non-target
    element, 1 on the target)."""
    case = small_case(vocab=8192, dtype="bf16", seed=15, mask_mode="all", ignore_frac=0.0)
    g = run_gpu_chain(cuda_lib, case, {})
    ref = oracle_chain(case, oracle.LossParams())["loss"]
    s = ref["scale"]
    nz = s != 0
    sums = g["dlogits"][nz].sum(axis=1)
    amax = np.abs(g["dlogits"][nz]).max(axis=1)
    u = 2.0 ** -8
    assert np.all(np.abs(sums) <= 3 * u / (1 - u) * amax + 2.0 ** -16 * np.abs(s[nz]))


def test_host_entry_point_matches_device(cuda_lib):
    rl, t = cuda_lib, torch()
    case = small_case(vocab=3000, dtype="bf16", seed=16, n_prompts=3, group=4, seq_len=50)
    g = run_gpu_chain(rl, case, {})
    bk = oracle.seq_bookkeeping(case["cu_seqlens"], case["loss_mask"], case["targets"], 3000,
                                case["seq_version"], case["trainer_version"], -1)
    adv = np.asarray(g["adv"], dtype=np.float32)
    N = len(case["targets"])
    x = t.from_numpy(case["logits"].view(np.int16)).view(t.bfloat16).pin_memory()
    dl = t.empty_like(x).pin_memory()
    logp = t.empty(N, dtype=t.float32).pin_memory()
    p = rl.LossParams(trainer_version=case["trainer_version"], global_active_tokens=bk["active_tokens"])
    ws = t.empty(rl.policy_loss_host_workspace_size(64, 3000, 3000, rl.BF16, len(adv)),
                 dtype=t.uint8, device="cuda")
    st = rl.policy_loss_fwd_bwd_host(x, t.from_numpy(case["targets"]), t.from_numpy(case["old_logp"]),
                                     t.from_numpy(bk["token_seq"]), t.from_numpy(adv), p, ws, 64,
                                     loss_mask=t.from_numpy(case["loss_mask"]),
                                     seq_version=t.from_numpy(case["seq_version"]),
                                     dlogits=dl, logp_out=logp, vocab=3000)
    assert st["loss_sum"] == pytest.approx(g["stats"][0], rel=1e-6, abs=1e-12)
    assert st["active_tokens"] == g["stats"][1]
    assert np.array_equal(logp.numpy(), g["logp"])
    assert np.array_equal(oracle.decode_bf16(dl.view(t.int16).numpy().view(np.uint16)), g["dlogits"])


def test_vocab_parallel_single_rank(cuda_lib):
    """c8 with P = 1 (degenerate world size): equals the unsplit log-probs and loss."""
    import ctypes
    rl, t = cuda_lib, torch()
    lib = rl.load()
    buf = (ctypes.c_uint8 * 128)()
    assert lib.rl_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)) == 0
    h = ctypes.c_void_p()
    assert lib.rl_comm_init(ctypes.byref(h), bytes(buf), 1, 0) == 0
    comm = rl.Comm(h.value, 1, 0)
    case = small_case(vocab=2048, dtype="bf16", seed=17)
    g = run_gpu_chain(rl, case, {})
    N = len(case["targets"])
    logp = t.empty(N, device="cuda")
    ws = t.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=t.uint8, device="cuda")
    rl.vocab_parallel_logprob(dev(case["logits"]), dev(case["targets"]), 0, 2048, comm, logp, ws)
    t.cuda.synchronize()
    lp = logp.cpu().numpy()
    ok = case["targets"] >= 0
    assert np.all(np.abs(lp[ok] - g["logp"][ok]) <= 1e-4)
    # fused loss through the in-kernel peer exchange (P = 1: the rank exchanges with itself)
    assert comm.enable_peer_exchange(N)
    bk = oracle.seq_bookkeeping(case["cu_seqlens"], case["loss_mask"], case["targets"], 2048,
                                case["seq_version"], case["trainer_version"], case["max_staleness"])
    p = rl.LossParams(trainer_version=case["trainer_version"], max_staleness=case["max_staleness"],
                      global_active_tokens=float(bk["active_tokens"]))
    dl = t.empty_like(dev(case["logits"]))
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    rl.vocab_parallel_logprob(dev(case["logits"]), dev(case["targets"]), 0, 2048, comm, logp, ws,
                              old_logp=dev(case["old_logp"]), loss_mask=dev(case["loss_mask"]),
                              token_seq=dev(bk["token_seq"]), seq_adv=dev(g["adv"]),
                              seq_version=dev(case["seq_version"]), params=p, dlogits_shard=dl, stats=stats)
    t.cuda.synchronize()
    assert np.all(np.abs(logp.cpu().numpy()[ok] - g["logp"][ok]) <= 1e-4)
    st = stats.cpu().numpy()
    assert st[1] == g["stats"][1] and abs(st[0] - g["stats"][0]) <= 1e-5 * max(1e-30, abs(g["stats"][0]) + 1e-6)
    d = host_logits(dl)[:, :2048]
    assert np.abs(d - g["dlogits"]).max() <= 1e-2 * max(1e-30, np.abs(g["dlogits"]).max())
    comm.destroy()


def test_vocab_parallel_extended_objective(cuda_lib):
    """The vocab-parallel loss with the NEXT-2 per-token terms (k3 KL, decoupled ratio) against the
    oracle, on the NCCL path and then on the in-kernel peer path (P = 1)."""
    import ctypes
    rl, t = cuda_lib, torch()
    lib = rl.load()
    buf = (ctypes.c_uint8 * 128)()
    assert lib.rl_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)) == 0
    h = ctypes.c_void_p()
    assert lib.rl_comm_init(ctypes.byref(h), bytes(buf), 1, 0) == 0
    comm = rl.Comm(h.value, 1, 0)
    V = 3000
    case = small_case(vocab=V, dtype="bf16", seed=19, sigma_delta=0.15, ld=3000)
    y = case["targets"]
    lp_ref, _ = oracle.token_logprob(case["x64"], y)
    rng = np.random.default_rng(19)
    ref = (np.where(y >= 0, lp_ref, 0.0) + rng.normal(size=len(y)) * 0.3).astype(np.float32)
    prox = (case["old_logp"] + rng.normal(size=len(y)) * 0.05).astype(np.float32)
    params = dict(kl_coef=0.05)
    ref_out = oracle_chain(case, oracle.LossParams(**params), ref_logp=ref.astype(np.float64),
                           prox_logp=prox.astype(np.float64))
    out, bk = ref_out["loss"], ref_out["bk"]
    N = len(y)
    adv = dev(ref_out["adv"])   # advantages are bit-exact on the GPU (tested above); the oracle's here
    p = rl.LossParams(trainer_version=case["trainer_version"], max_staleness=case["max_staleness"],
                      global_active_tokens=float(bk["active_tokens"]), kl_coef=0.05,
                      ref_logp=dev(ref), prox_logp=dev(prox))
    ws = t.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=t.uint8, device="cuda")
    scale = max(abs(out["loss"]), float(np.abs(out["token_loss"]).sum()))
    for path in ("nccl", "peer"):
        if path == "peer":
            assert comm.enable_peer_exchange(N)
        logp = t.empty(N, device="cuda")
        dl = t.empty_like(dev(case["logits"]))
        stats = t.zeros(12, dtype=t.float64, device="cuda")
        rl.vocab_parallel_logprob(dev(case["logits"]), dev(y), 0, V, comm, logp, ws, old_logp=dev(case["old_logp"]),
                                  loss_mask=dev(case["loss_mask"]), token_seq=dev(bk["token_seq"]), seq_adv=adv,
                                  seq_version=dev(case["seq_version"]), params=p, dlogits_shard=dl, stats=stats)
        t.cuda.synchronize()
        st = stats.cpu().numpy()
        assert abs(st[0] - out["loss"]) <= LOSS_RTOL * scale, (path, st[0], out["loss"])
        assert abs(st[10] - out["stats"]["kl_sum"]) <= 1e-3 * abs(out["stats"]["kl_sum"]) + 1e-7
        d = host_logits(dl)[:, :V]
        s_ref = out["scale"]
        band = clip_band(out["ratio"], out["valid"], 0.2, 0.2)
        for k in range(N):
            if band[k]:
                continue
            if s_ref[k] == 0:
                assert np.all(d[k] == 0), (path, k)
            else:
                assert np.abs(d[k] - out["dlogits"][k]).max() <= DLOGIT_ROW_RTOL * abs(s_ref[k]), (path, k)
    comm.destroy()


@pytest.mark.slow
@pytest.mark.parametrize("name,N,in_place,objective", [
    ("single", 131072, False, False),  # configs[1]: the bench's 131,072-token mini-batch, V = 151936
    ("single", 65536, True, True),     # + KL, decoupled ratio, entropy (NEXT 2) on the fast path
    ("long", 65536, True, False),      # configs[2]: multi-turn tool masks (~50 % masked rows), in place
    ("multi_b", 32768, False, False),  # configs[4] policy B: V = 128256, prompt masks, staleness 8
])
def test_full_size_sampled(cuda_lib, name, N, in_place, objective):
    """Full vocabulary width in the bench's launch configuration: sampled rows against the
    oracle (masks, staleness and versions of the config), plus the row-sum invariant over
    every row.  V = 151936 and V = 128256 are the two compile-time fast paths of the kernel."""
    rl, t = cuda_lib, torch()
    cfg = synth.get_config(name)
    V = cfg.vocab
    lay = synth.seq_layout(cfg)
    logits = t.empty((N, V), dtype=t.bfloat16, device="cuda")
    y = t.empty(N, dtype=t.int32, device="cuda")
    synth.device_logits(logits, V, 0, cfg.seed, targets_out=y)
    rows = np.random.default_rng(0).choice(N, size=48, replace=False)
    rows.sort()
    xs = oracle.decode_bf16(logits[t.from_numpy(rows).cuda()].view(t.int16).cpu().numpy().view(np.uint16))
    yh = y.cpu().numpy()
    ref_lp, _ = oracle.token_logprob(xs, yh[rows])
    old = np.zeros(N, dtype=np.float32)
    old[rows] = ref_lp + np.random.default_rng(1).normal(size=len(rows)) * 0.05
    tseq = (np.arange(N) // cfg.seq_len).astype(np.int32)
    S = int(tseq[-1]) + 1
    adv = np.random.default_rng(2).normal(size=S).astype(np.float32)
    mask = np.ascontiguousarray(lay["loss_mask"][:N]).astype(np.uint8)
    ver = np.ascontiguousarray(lay["seq_version"][:S]).astype(np.int32)
    tv, ms = int(lay["trainer_version"]), int(cfg.max_staleness)
    p = rl.LossParams(agg=rl.AGG_SUM, trainer_version=tv, max_staleness=ms)
    ref = prox = None
    if objective:
        # every row gets realistic behaviour / reference / proximal log-probs: torch fp32
        # log-softmax of the inputs (input synthesis, as bench.py) + seeded drift; the sampled rows
        # keep the oracle-derived old_logp set above
        rng = np.random.default_rng(5)
        lp_all = np.empty(N, dtype=np.float32)
        for c0 in range(0, N, 4096):
            blk = logits[c0:c0 + 4096].float()
            lp_all[c0:c0 + 4096] = (blk.gather(1, y[c0:c0 + 4096, None].long())[:, 0]
                                    - t.logsumexp(blk, dim=1)).cpu().numpy()
            del blk
        keep = old[rows].copy()
        old = (lp_all + rng.normal(size=N) * 0.05).astype(np.float32)
        old[rows] = keep
        ref = (old + rng.normal(size=N) * 0.2).astype(np.float32)
        prox = (old + rng.normal(size=N) * 0.02).astype(np.float32)
        p.kl_coef, p.ref_logp, p.prox_logp = 1e-3, dev(ref), dev(prox)
        p.flags |= rl.F_ENTROPY
    dl = logits if in_place else t.empty_like(logits)
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    ws = t.empty(rl.policy_loss_workspace_size(N, V), dtype=t.uint8, device="cuda")
    logp = t.empty(N, device="cuda")
    rl.policy_loss_fwd_bwd(logits, y, dev(old), dev(tseq), dev(adv), p, dl, stats, ws, logp_out=logp,
                           loss_mask=dev(mask), seq_version=dev(ver))
    t.cuda.synchronize()
    out = oracle.policy_loss_fwd_bwd(xs, yh[rows], old[rows], mask[rows], tseq[rows], adv, ver, None,
                                     oracle.LossParams(agg=oracle.AGG_SUM, trainer_version=tv, max_staleness=ms,
                                                       kl_coef=1e-3 if objective else 0.0),
                                     ref_logp=None if ref is None else ref[rows].astype(np.float64),
                                     prox_logp=None if prox is None else prox[rows].astype(np.float64),
                                     want_entropy=objective)
    g_lp = logp.cpu().numpy()[rows]
    assert np.all(np.abs(g_lp - out["logp"]) <= LOGP_ATOL)
    d = oracle.decode_bf16(dl[t.from_numpy(rows).cuda()].view(t.int16).cpu().numpy().view(np.uint16))
    s = out["scale"]
    assert (s != 0).any() and (s == 0).any() or name == "single"
    for k in range(len(rows)):
        if s[k] == 0:
            assert np.all(d[k] == 0)
        else:
            assert np.abs(d[k] - out["dlogits"][k]).max() <= DLOGIT_ROW_RTOL * abs(s[k])
    # every row: |sum_v d| ~ 0 up to bf16 rounding of the row (chunked to bound memory)
    for c0 in range(0, N, 4096):
        blk = dl[c0:c0 + 4096].float()
        sums = blk.sum(dim=1).abs()
        amax = blk.abs().amax(dim=1)
        # reading R2: <= 2 bf16 roundings per non-target element, 1 on the target:
        # |sum| <= 3u / (1 - u) max|d| + 2^-16 |s_t|, u = 2^-8; |s_t| <= 8 here (AGG_SUM, |A| r)
        u = 2.0 ** -8
        bad = t.nonzero(sums > 3 * u / (1 - u) * amax + 2.0 ** -16 * 8)[:, 0]
        assert bad.numel() == 0, [(c0 + int(r), float(sums[r]), float(amax[r])) for r in bad[:5]]
        del blk
    del logits, dl


# ----------------------------------------------------------------------------- NEXT 1: M2PO (M1)
def _m2po_band(lp, old, valid, tau, k_star):
    """True when the oracle's cut is within rounding of tau (the fp64 prefix order may differ)."""
    m = ((lp - old).astype(np.float32) ** 2).astype(np.float32)
    mv = np.sort(m[valid != 0].astype(np.float64))
    nv = len(mv)
    P = np.cumsum(mv)
    for j in (nv - k_star, nv - k_star + 1):
        if 1 <= j <= nv and abs(P[j - 1] - tau * j) <= 1e-9 * max(P[j - 1], tau * j, 1e-300):
            return True
    return False


@pytest.mark.parametrize("n,tau,ties", [(1, 0.01, False), (777, 0.01, False), (10007, 0.002, True),
                                        (50000, 0.05, True), (4096, 1e9, False), (3000, 0.0, True)])
def test_m2po_mask(cuda_lib, n, tau, ties):
    """rl_m2po_mask against the oracle on the same fp32 inputs: the mask bit-exact (ties included),
    the counts exact, the means to 1e-12 (reading M1)."""
    t = torch()
    rng = np.random.default_rng(n)
    lp = (rng.normal(size=n) * 3 - 5).astype(np.float32)
    drift = rng.normal(size=n) * rng.choice([0.02, 0.1, 0.5], size=n)
    if ties:  # quantised drifts: many exactly equal m
        drift = np.round(drift * 64) / 64
    old = (lp - drift).astype(np.float32)
    valid = (rng.random(n) < 0.9).astype(np.uint8)
    mask_ref, k_ref, m2b, m2a = oracle.m2po_mask(lp, old, valid, tau)
    mask = t.empty(n, dtype=t.uint8, device="cuda")
    stats = t.zeros(5, dtype=t.float64, device="cuda")
    ws = t.empty(cuda_lib.m2po_workspace_size(n), dtype=t.uint8, device="cuda")
    cuda_lib.m2po_mask(dev(lp), dev(old), mask, stats, ws, tau=tau, valid=dev(valid))
    t.cuda.synchronize()
    g, st = mask.cpu().numpy(), stats.cpu().numpy()
    assert st[0] == valid.sum()
    if _m2po_band(lp, old, valid, tau, k_ref):
        assert abs(st[1] - k_ref) <= 1
        return
    assert st[1] == k_ref and st[4] == st[0] - st[1] and np.array_equal(g, mask_ref)
    assert abs(st[2] - m2b) <= 1e-12 * max(m2b, 1e-300) and abs(st[3] - m2a) <= 1e-12 * max(m2a, 1e-300)
    if 0 < tau < 1e8:
        assert 0 < k_ref < valid.sum() or tau == 0.0 or n == 1   # the bound is active in these cases


# ----------------------------------------------------------------------------- NEXT 3: delta scan
@pytest.mark.parametrize("n,frac", [(0, 0.0), (1, 1.0), (8191, 0.01), (8192 * 3 + 5, 0.3), (1 << 20, 0.011),
                                    (3_000_001, 0.0), (2_000_003, 1.0), (40_000_000, 0.008),
                                    (1_000_037, -1.0)])
def test_delta_encode_apply(cuda_lib, n, frac):
    """rl_bf16_delta_encode equals the oracle's element-wise diff bit for bit (indices, words,
    count), ragged and multi-tile sizes, all-equal and all-different, and (frac = -1) one call
    mixing sparse tiles (staged) with dense ones (> 1,024 changes per 16,384-word tile: bitmask
    path) including tiles right at the staging capacity; apply(encode) = next; a short output
    buffer holds exactly the first `capacity` changes."""
    t = torch()
    from oracle import delta
    rng = np.random.default_rng(n + 7)
    a = rng.integers(0, 1 << 16, size=n, dtype=np.uint16)
    b = a.copy()
    if frac >= 0:
        ch = rng.random(n) < frac
    else:  # per-tile change rates: 0, 1/16 exactly (1,024 changes), 1,025 changes, 0.3, 0.01 ...
        ch = np.zeros(n, dtype=bool)
        for ti, t0 in enumerate(range(0, n, 16384)):
            m = min(16384, n - t0)
            kind = ti % 5
            k = [0, 1024, 1025, int(0.3 * m), int(0.01 * m)][kind]
            ch[t0 + rng.choice(m, size=min(k, m), replace=False)] = True
    b[ch] ^= rng.integers(1, 1 << 16, size=int(ch.sum()), dtype=np.uint16)
    if n > 16:
        b[3] = 0x8000 if a[3] == 0 else b[3]   # +0 vs -0 style bit flips count
    ta, tb = dev(a.view(np.int16)), dev(b.view(np.int16))
    cap = max(1, int((a != b).sum()))
    idx = t.empty(cap, dtype=t.int32, device="cuda")
    words = t.empty(cap, dtype=t.int16, device="cuda")
    count = t.zeros(1, dtype=t.int64, device="cuda")
    ws = t.empty(max(8, cuda_lib.delta_workspace_size(n)), dtype=t.uint8, device="cuda")
    cuda_lib.delta_encode(ta, tb, idx, words, count, ws)
    t.cuda.synchronize()
    k = int(count.item())
    if n <= 200_000:
        ri, rw, _ = delta.compute_delta(a, b)
    else:  # the loop oracle is slow at this size: its definition restated by numpy (same pin)
        ri = np.nonzero(a != b)[0].astype(np.uint32)
        rw = b[ri]
    assert k == ri.size
    assert np.array_equal(idx.cpu().numpy()[:k].view(np.uint32), ri)
    assert np.array_equal(words.cpu().numpy()[:k].view(np.uint16), rw)
    base = ta.clone()
    bad = t.zeros(1, dtype=t.int64, device="cuda")
    cuda_lib.delta_apply(base, idx, words, count, bad)
    t.cuda.synchronize()
    assert bad.item() == 0 and t.equal(base, tb)
    if k >= 2:  # truncated output: the first capacity changes, the full count
        c2 = k // 2
        idx2 = t.empty(c2, dtype=t.int32, device="cuda")
        words2 = t.empty(c2, dtype=t.int16, device="cuda")
        count2 = t.zeros(1, dtype=t.int64, device="cuda")
        cuda_lib.delta_encode(ta, tb, idx2, words2, count2, ws)
        t.cuda.synchronize()
        assert int(count2.item()) == k
        assert np.array_equal(idx2.cpu().numpy().view(np.uint32), ri[:c2])
        assert np.array_equal(words2.cpu().numpy().view(np.uint16), rw[:c2])


# ----------------------------------------------------------------------------- NEXT 4: LM head
def _lm_ws(N, d, V):
    import paper_2605_15565_b200 as rl
    return torch().empty(max(1, rl.lmhead_workspace_size(N, d, V)), dtype=torch().uint8, device="cuda")


def _lm_inputs(N, d, V, seed, ld_h=None, ld_w=None):
    """Seeded bf16 hidden states ~ N(0, 1) and LM-head rows ~ N(0, 9/d) (logit sd ~ 3, a few hot
    rows per token as in the configs' logit model), as bit patterns (host) and CUDA tensors."""
    t = torch()
    rng = np.random.default_rng(seed)
    ld_h, ld_w = ld_h or d, ld_w or d
    h = rng.normal(size=(N, ld_h)).astype(np.float32)
    w = (rng.normal(size=(V, ld_w)) * (3.0 / math.sqrt(d))).astype(np.float32)
    if V > 4:  # hot vocabulary rows aligned with some tokens' hidden states (peaked rows)
        for i in range(min(N, 64)):
            w[(7 * i) % V, :d] += 0.5 * h[i, :d] / math.sqrt(d)
    hb = (h.view(np.uint32) >> 16).astype(np.uint16)
    wb = (w.view(np.uint32) >> 16).astype(np.uint16)
    ht = t.from_numpy(hb.view(np.int16)).cuda().view(t.bfloat16)
    wt = t.from_numpy(wb.view(np.int16)).cuda().view(t.bfloat16)
    y = rng.integers(0, V, size=N).astype(np.int32)
    y[::7] = (7 * np.arange(len(y[::7]))) % V   # some targets on the hot rows
    if N > 3:
        y[1], y[2] = -100, V + 3                   # ignored and out-of-range targets
    return hb[:, :d], wb[:, :d], ht[:, :d], wt[:, :d], y


@pytest.mark.parametrize("N,d,V,ldh,ldw", [(1, 64, 256, None, None), (300, 128, 1000, None, None),
                                          (129, 200, 513, 208, 216), (1024, 512, 4099, None, None),
                                          (257, 4096, 2000, None, None), (64, 16, 70000, None, None)])
def test_lmhead_logprob(cuda_lib, N, d, V, ldh, ldw):
    """rl_lmhead_logprob (tcgen05 GEMM + online softmax, logits never written) against the oracle
    c3(h W^T) in fp64: logp and lse within 2e-3 absolute (SURVEY.md §8(g) logp bar); ragged N (not a
    multiple of 128), V (not of 256), d (K tail, not of 64), padded row strides, y < 0 and y >= V."""
    t = torch()
    hb, wb, ht, wt, y = _lm_inputs(N, d, V, seed=N + d + V, ld_h=ldh, ld_w=ldw)
    logp = t.empty(N, dtype=t.float32, device="cuda")
    lse = t.empty(N, dtype=t.float32, device="cuda")
    cuda_lib.lmhead_logprob(ht, wt, dev(y), logp, lse, workspace=_lm_ws(N, d, V))
    t.cuda.synchronize()
    ref_lp, ref_lse = oracle.lmhead_logprob(hb, wb, y)
    got_lp, got_lse = logp.cpu().numpy().astype(np.float64), lse.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got_lse - ref_lse)) <= 2e-3
    ok = ~np.isnan(ref_lp)
    assert np.array_equal(np.isnan(got_lp), ~ok)
    assert np.max(np.abs(got_lp[ok] - ref_lp[ok])) <= 2e-3
    if N > 3:
        assert got_lp[1] == 0.0 and np.isnan(got_lp[2])


def test_lmhead_logprob_full_size_sampled(cuda_lib):
    """Qwen3-8B-sized head (d = 4096, V = 151936) on 2,048 tokens: 24 sampled rows against the
    oracle (its fp64 row is h W^T over all 151,936 vocabulary rows), every row finite."""
    t = torch()
    N, d, V = 2048, 4096, 151936
    g = t.Generator(device="cuda").manual_seed(11)
    ht = t.randn(N, d, device="cuda", generator=g).to(t.bfloat16)
    wt = (t.randn(V, d, device="cuda", generator=g) * (3.0 / math.sqrt(d))).to(t.bfloat16)
    y = t.randint(0, V, (N,), device="cuda", generator=g, dtype=t.int32)
    logp = t.empty(N, dtype=t.float32, device="cuda")
    lse = t.empty(N, dtype=t.float32, device="cuda")
    cuda_lib.lmhead_logprob(ht, wt, y, logp, lse, workspace=_lm_ws(N, d, V))
    t.cuda.synchronize()
    assert bool(t.isfinite(logp).all()) and bool(t.isfinite(lse).all())
    rows = np.random.default_rng(0).choice(N, size=24, replace=False)
    rows[0], rows[1] = 0, N - 1
    wb = wt.view(t.int16).cpu().numpy().view(np.uint16)
    hb = ht[t.from_numpy(rows).cuda()].view(t.int16).cpu().numpy().view(np.uint16)
    yr = y.cpu().numpy()[rows]
    ref_lp, ref_lse = oracle.lmhead_logprob(hb, wb, yr)
    assert np.max(np.abs(logp.cpu().numpy()[rows] - ref_lp)) <= 2e-3
    assert np.max(np.abs(lse.cpu().numpy()[rows] - ref_lse)) <= 2e-3


def test_lmhead_logprob_temperature_and_errors(cuda_lib):
    """inv_temperature != 1 against the oracle's c3 temperature; host-detectable errors return
    before any launch (d mismatch, non-contiguous rows, inv_temperature <= 0, short workspace)."""
    t = torch()
    N, d, V = 200, 96, 3001
    hb, wb, ht, wt, y = _lm_inputs(N, d, V, seed=77)
    logp = t.empty(N, dtype=t.float32, device="cuda")
    cuda_lib.lmhead_logprob(ht, wt, dev(y), logp, inv_temperature=0.6, workspace=_lm_ws(N, d, V))
    t.cuda.synchronize()
    ref, _ = oracle.lmhead_logprob(hb, wb, y, inv_temperature=0.6)
    ok = ~np.isnan(ref)
    assert np.max(np.abs(logp.cpu().numpy()[ok] - ref[ok])) <= 2e-3
    with pytest.raises(cuda_lib.RLError):
        cuda_lib.lmhead_logprob(ht, wt[:, :64], dev(y), logp, workspace=_lm_ws(N, d, V))
    with pytest.raises(cuda_lib.RLError):
        cuda_lib.lmhead_logprob(ht, wt, dev(y), logp, inv_temperature=0.0, workspace=_lm_ws(N, d, V))
    big = 20000   # more token blocks: the plan uses vocabulary splits and needs a workspace
    hb2 = t.zeros((big, d), dtype=t.bfloat16, device="cuda")
    need = cuda_lib.lmhead_workspace_size(big, d, 151936)
    if need > 0:
        w2 = t.zeros((151936, d), dtype=t.bfloat16, device="cuda")
        y2 = t.zeros(big, dtype=t.int32, device="cuda")
        lp2 = t.empty(big, dtype=t.float32, device="cuda")
        with pytest.raises(cuda_lib.RLError):
            cuda_lib.lmhead_logprob(hb2, w2, y2, lp2, workspace=t.empty(need - 1, dtype=t.uint8, device="cuda"))


def test_lmhead_loss_forward(cuda_lib):
    """NEXT 4 loss forward without logits: rl_lmhead_logprob -> rl_policy_loss_from_logp against the
    oracle's c4-c7 on x = h W^T (oracle.lmhead_logits): loss (Z22), clip flags outside the Z23 band,
    s_t (1e-3 relative), counters exact; a short sequence, masked tokens, one stale sequence and an
    ignored target included."""
    t = torch()
    from tests.cases import clip_band
    S, L, d, V = 12, 40, 192, 2500
    N = S * L
    hb, wb, ht, wt, y = _lm_inputs(N, d, V, seed=123)
    y[1], y[2] = y[5], y[6]          # no out-of-range targets here (counted separately)
    y[9] = -100
    rng = np.random.default_rng(5)
    token_seq = np.repeat(np.arange(S, dtype=np.int32), L)
    mask = (rng.random(N) > 0.1).astype(np.uint8)
    mask[:5] = 0
    seq_version = np.full(S, 10, dtype=np.int32)
    seq_version[3] = 1                # staleness 9 > 8: masked
    adv = rng.choice([-1.3, -0.4, 0.5, 1.1], size=S).astype(np.float32)
    x = oracle.lmhead_logits(hb, wb)
    lp_ref, _ = oracle.token_logprob(x, y)
    old = (lp_ref + rng.normal(0, 0.3, size=N)).astype(np.float32)
    valid = ((mask != 0) & (y >= 0) & (token_seq != 3)).astype(np.uint8)
    seq_active = np.bincount(token_seq, weights=valid, minlength=S).astype(np.int32)
    op = oracle.LossParams(global_active_tokens=float(valid.sum()), trainer_version=10, max_staleness=8)
    ref = oracle.policy_loss_fwd_bwd(x, y, old.astype(np.float64), mask, token_seq, adv.astype(np.float64),
                                     seq_version, seq_active, op, want_dlogits=False)
    # GPU: LM-head log-probs, then the loss from them
    logp = t.empty(N, dtype=t.float32, device="cuda")
    cuda_lib.lmhead_logprob(ht, wt, dev(y), logp, workspace=_lm_ws(N, d, V))
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    scale = t.empty(N, dtype=t.float32, device="cuda")
    clipped = t.empty(N, dtype=t.uint8, device="cuda")
    ws = t.empty(cuda_lib.policy_loss_from_logp_workspace_size(N), dtype=t.uint8, device="cuda")
    p = cuda_lib.LossParams(global_active_tokens=float(valid.sum()), trainer_version=10, max_staleness=8)
    cuda_lib.policy_loss_from_logp(logp, dev(y), dev(old), dev(token_seq), dev(adv), p, stats, ws, V,
                                   loss_mask=dev(mask), seq_version=dev(seq_version), scale_out=scale,
                                   clipped_out=clipped)
    t.cuda.synchronize()
    st = stats.cpu().numpy()
    names = cuda_lib.STATS_FIELDS
    band = clip_band(ref["ratio"], ref["valid"], 0.2, 0.2)
    bound = 1e-4 * max(abs(ref["loss"]), float(np.abs(ref["token_loss"]).sum()))
    assert abs(st[names.index("loss_sum")] - ref["loss"]) <= bound + 1e-4 * float(np.abs(ref["token_loss"][band]).sum())
    assert st[names.index("active_tokens")] == ref["stats"]["active_tokens"]
    assert st[names.index("stale_masked")] == ref["stats"]["stale_masked"]
    cl = clipped.cpu().numpy()
    assert np.array_equal(cl[~band], ref["clipped"][~band])
    sc = scale.cpu().numpy().astype(np.float64)
    ok = ~band
    assert np.all(np.abs(sc[ok] - ref["scale"][ok]) <= 1e-3 * np.abs(ref["scale"][ok]) + 1e-12)
    assert np.all(sc[ref["valid"] == 0] == 0.0)


# ----------------------------------------------------------------------------- NEXT 4 backward
def _lm_bwd_check(cuda_lib, N, d, V, seed, chunk=None, ld_h=None, ld_w=None, inv_t=1.0, vrows=None):
    """rl_lmhead_loss_bwd against oracle.lmhead_loss_backward.  Tolerance: G is
    one bf16 rounding of s (p - onehot) (relative u = 2^-8) and the GEMMs accumulate in fp32, so
    |d dh| <= 2^-7 ||G_t||_1 max_v |W_vj| and |d dW[v]| <= 2^-7 (|G[:, v]|^T |h|) (+ 1e-7 abs)."""
    t = torch()
    hb, wb, ht, wt, y = _lm_inputs(N, d, V, seed=seed, ld_h=ld_h, ld_w=ld_w)
    y = y.copy()
    y[3] = -100                              # ignored target: zero G row
    rng = np.random.default_rng(seed + 1)
    s = rng.normal(size=N).astype(np.float32)
    s[5] = 0.0                               # s_t = 0 (masked / clipped token): zero G row
    lse = t.empty(N, dtype=t.float32, device="cuda")
    logp = t.empty(N, dtype=t.float32, device="cuda")
    cuda_lib.lmhead_logprob(ht, wt, dev(y), logp, lse_out=lse, inv_temperature=inv_t, workspace=_lm_ws(N, d, V))
    C = chunk or N
    ws = t.empty(cuda_lib.lmhead_loss_bwd_workspace_size(C, V), dtype=t.uint8, device="cuda")
    dh = t.full((N, d), float("nan"), dtype=t.float32, device="cuda")
    dW = t.full((V, d), float("nan"), dtype=t.float32, device="cuda")
    cuda_lib.lmhead_loss_bwd(ht, wt, dev(y), lse, dev(s), ws, dhidden=dh, dweight=dW, inv_temperature=inv_t)
    t.cuda.synchronize()
    hbd, wbd = hb, wb
    dh_ref, dW_ref, G = oracle.lmhead_loss_backward(hbd, wbd, y, s.astype(np.float64), inv_t)
    W64, H64 = oracle.decode_bf16(wbd), oracle.decode_bf16(hbd)
    u2 = 2.0 ** -7
    tol_dh = u2 * np.abs(G).sum(axis=1)[:, None] * np.abs(W64).max(axis=0)[None, :] + 1e-7
    g_dh = dh.cpu().numpy()
    assert np.all(np.abs(g_dh - dh_ref) <= tol_dh), np.max(np.abs(g_dh - dh_ref) / tol_dh)
    assert np.all(g_dh[3] == 0) and np.all(g_dh[5] == 0) and np.all(g_dh[2] == 0)   # y < 0, s = 0, y >= V
    rows = np.arange(V) if vrows is None else vrows
    g_dW = dW[t.from_numpy(rows).cuda()].cpu().numpy()
    tol_dW = u2 * (np.abs(G[:, rows]).T @ np.abs(H64)) + 1e-7
    assert np.all(np.abs(g_dW - dW_ref[rows]) <= tol_dW), np.max(np.abs(g_dW - dW_ref[rows]) / tol_dW)
    return ht, wt, y, lse, s, dW, ws


@pytest.mark.parametrize("N,d,V,chunk,ld_h,ld_w,inv_t", [
    (300, 192, 1000, None, None, None, 1.0),     # ragged token block (300 = 2 x 128 + 44), V % 256 != 0
    (300, 192, 1003, 128, 200, 208, 0.7),        # 3 chunks, padded strides, V % 32 != 0, temperature
    (128, 64, 8, None, None, None, 1.0),         # one vocabulary tile narrower than 32 columns
])
@pytest.mark.parametrize("pair_opt,gemm_opt", [(0, 0), (1, 0), (2, 0), (0, 2), (1, 2), (2, 2)])
def test_lmhead_loss_bwd(cuda_lib, N, d, V, chunk, ld_h, ld_w, inv_t, pair_opt, gemm_opt):
    """RL_DEV_LM_PAIR: default / single CTAs / pairs everywhere; RL_DEV_LM_GEMM: cuBLAS (default) or
    the hand-written tcgen05 GEMMs (lm_gemm_kernel, single CTAs or pairs) for dh and dW."""
    old = cuda_lib.dev_set_option(cuda_lib.DEV_LM_PAIR, pair_opt)
    old_g = cuda_lib.dev_set_option(cuda_lib.DEV_LM_GEMM, gemm_opt)
    try:
        _lm_bwd_check(cuda_lib, N, d, V, seed=N + V, chunk=chunk, ld_h=ld_h, ld_w=ld_w, inv_t=inv_t)
    finally:
        cuda_lib.dev_set_option(cuda_lib.DEV_LM_PAIR, old)
        cuda_lib.dev_set_option(cuda_lib.DEV_LM_GEMM, old_g)


def test_lmhead_loss_bwd_accumulate_and_errors(cuda_lib):
    """RL_F_STATS_ACCUMULATE adds into dweight (two micro-batches = their sum); bad arguments are
    rejected before enqueue."""
    t = torch()
    N, d, V = 256, 128, 700
    ht, wt, y, lse, s, dW, ws = _lm_bwd_check(cuda_lib, N, d, V, seed=9)
    acc = dW.clone()
    cuda_lib.lmhead_loss_bwd(ht, wt, dev(y), lse, dev(s), ws, dweight=acc, accumulate=True)
    t.cuda.synchronize()
    assert t.allclose(acc, 2 * dW, rtol=1e-6, atol=1e-7)
    with pytest.raises(cuda_lib.RLError):     # workspace below one 128-token chunk
        cuda_lib.lmhead_loss_bwd(ht, wt, dev(y), lse, dev(s), ws[:1000], dweight=acc)
    with pytest.raises(cuda_lib.RLError):     # no output requested
        cuda_lib.lmhead_loss_bwd(ht, wt, dev(y), lse, dev(s), ws)


@pytest.mark.slow
def test_lmhead_loss_bwd_full_size(cuda_lib):
    """d = 4096, V = 151936 (the policy's LM head), 256 tokens (two token blocks, 594 vocabulary
    tiles): dh of every token and dW on 2,048 sampled vocabulary rows plus every target row."""
    N, d, V = 256, 4096, 151936
    rng = np.random.default_rng(77)
    vrows = np.unique(np.concatenate([rng.choice(V, size=2048, replace=False), (7 * np.arange(64)) % V]))
    _lm_bwd_check(cuda_lib, N, d, V, seed=77, vrows=vrows)
