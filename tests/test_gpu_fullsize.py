"""Full-size parity — SURVEY.md §8(g): C2-C5 "on >= 4096 sampled rows plus all per-token and
per-sequence scalars".

Every unsampled row is masked (loss_mask = 0), so the kernels' loss statistics cover exactly the
sampled rows, which the fp64 oracle recomputes block by block (its row math is row-separable; the
global normalisers are passed in).  The bookkeeping and the advantages run over the WHOLE batch on
both sides and are compared exactly; the log-prob of EVERY row is compared with a plain PyTorch
fp32 log-softmax.  Behaviour log-probs come from the oracle's log-probs plus synth's drift; rows
whose ratio would fall inside the clip tie band (reading Z23) get their drift nudged out of it, so
clip decisions compare exactly.

Also here: the vocab-parallel path at the production shard widths (P = 1 with the column widths of
P = 8 / 4 / 1 on the NCCL and the in-kernel peer paths, plus the C1 all-reduce call), reading R2's
worst case (a dominant NON-target column), and RL_F_SKIP_MASKED_READS at full width.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.cases import clip_band

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LOGP_ATOL = 2e-3
LOSS_RTOL = 1e-4
DLOGIT_ROW_RTOL = 1e-2
N_SAMPLED = 4096
BLOCK = 256


def torch():
    import torch as t
    return t


def dev(a):
    t = torch()
    if a.dtype == np.uint16:
        return t.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(t.bfloat16)
    return t.from_numpy(np.ascontiguousarray(a)).cuda()


def rows_bits(x, rows, V):
    """bf16 bit patterns of the given rows (first V columns), host uint16."""
    t = torch()
    return x[t.from_numpy(rows).cuda(), :V].view(t.int16).cpu().numpy().view(np.uint16)


def torch_logp_all(x, y, V):
    """Plain PyTorch fp32 log-softmax + gather over every row (independent of the library)."""
    t = torch()
    out = np.empty(x.shape[0], dtype=np.float32)
    for c0 in range(0, x.shape[0], 4096):
        blk = x[c0:c0 + 4096, :V].float()
        yy = y[c0:c0 + 4096].long()
        lp = blk.gather(1, yy.clamp(0, V - 1)[:, None])[:, 0] - t.logsumexp(blk, dim=1)
        out[c0:c0 + 4096] = t.where(yy >= 0, lp, t.zeros_like(lp)).cpu().numpy()
        del blk
    return out


def oracle_logp_rows(bits, y_rows):
    lp = np.empty(len(y_rows))
    for b0 in range(0, len(y_rows), BLOCK):
        lp[b0:b0 + BLOCK], _ = oracle.token_logprob(oracle.decode_bf16(bits[b0:b0 + BLOCK]), y_rows[b0:b0 + BLOCK])
    return lp


def nudge_out_of_band(old, lp_ref, valid, eps=0.2):
    """Move behaviour log-probs whose ratio sits within 1e-3 of a clip boundary by 5e-3 (input
    synthesis: the Z23 band then holds no token and clip flags compare exactly)."""
    r = np.exp(lp_ref - old.astype(np.float64))
    band = clip_band(r, valid, eps, eps)
    old = old.copy()
    old[band] += np.float32(5e-3)
    return old


def check_sampled(bits, rows, y, old, mask, tseq, adv, ver, seq_active, po, g_logp, g_dl_bits, g_stats,
                  g_clipped=None, ref=None, prox=None, want_entropy=False, extra_counts=(0, 0), read=None):
    """Oracle over the sampled rows, block by block, against the GPU outputs: logp (2e-3; rows the
    kernel was told not to read — `read` False — report 0), clip flags (exact), dlogits per row
    (Z21 plus the propagated log-prob error of s_t, reading Z21' in DESIGN.md §3; zero rows bitwise
    zero), and every statistic."""
    V = bits.shape[1]
    loss_terms, ratio_terms, weight_terms, kl_terms, ent_terms = [], [], [], [], []
    tl_abs = 0.0
    cnt = dict(active_tokens=0, clipped_low=0, clipped_high=0, clamped=0, stale_masked=0)
    worst = 0.0
    for b0 in range(0, len(rows), BLOCK):
        rb = rows[b0:b0 + BLOCK]
        xs = oracle.decode_bf16(bits[b0:b0 + BLOCK])
        out = oracle.policy_loss_fwd_bwd(xs, y[rb], old[rb], mask[rb], tseq[rb], adv, ver, seq_active, po,
                                         ref_logp=None if ref is None else ref[rb].astype(np.float64),
                                         prox_logp=None if prox is None else prox[rb].astype(np.float64),
                                         want_entropy=want_entropy)
        inr = (y[rb] >= 0) & (y[rb] < V)
        if read is not None:
            assert np.all(g_logp[rb][inr & ~read[rb]] == 0)
            inr &= read[rb]
        err_lp = np.abs(g_logp[rb][inr] - out["logp"][inr])
        assert np.all(err_lp <= LOGP_ATOL), err_lp.max()
        # Z21': |ds/dlogp| |dlogp| = w invT (|rho A r| + beta e^Dk) |dlogp| (0 unless the KL term is on)
        dlp = np.abs(np.where(inr, g_logp[rb] - out["logp"], 0.0))
        s_prop = np.zeros(len(rb))
        if ref is not None and po.kl_coef != 0.0:
            w = 1.0 / po.global_active_tokens if po.agg == oracle.AGG_TOKEN_MEAN else 1.0
            rho = np.exp(np.clip(prox[rb] - old[rb], -20, 20)) if prox is not None else 1.0
            ekl = np.exp(np.clip(ref[rb] - out["logp"], -20, 20))
            s_prop = w * po.inv_temperature * (np.abs(rho * adv[tseq[rb]] * out["ratio"]) + po.kl_coef * ekl) * dlp
        if g_clipped is not None:
            assert np.array_equal(g_clipped[rb], out["clipped"])
        d = oracle.decode_bf16(g_dl_bits[b0:b0 + BLOCK])
        s = out["scale"]
        for k in range(len(rb)):
            if s[k] == 0:
                assert np.all(d[k] == 0), ("row", int(rb[k]), "must be exact zeros")
            else:
                e = np.abs(d[k] - out["dlogits"][k]).max() / (abs(s[k]) + s_prop[k] / DLOGIT_ROW_RTOL)
                worst = max(worst, e)
                assert e <= DLOGIT_ROW_RTOL, ("row", int(rb[k]), e, s[k], s_prop[k])
        loss_terms.append(out["loss"])
        tl_abs += float(np.abs(out["token_loss"]).sum())
        st = out["stats"]
        for key in cnt:
            cnt[key] += st[key]
        ratio_terms.append(st["ratio_sum"])
        weight_terms.append(st["weight_sum"])
        kl_terms.append(st["kl_sum"])
        ent_terms.append(st["entropy_sum"])
    loss = math.fsum(loss_terms)
    assert abs(g_stats[0] - loss) <= LOSS_RTOL * max(abs(loss), tl_abs, 1e-30), (g_stats[0], loss)
    assert g_stats[1] == cnt["active_tokens"]
    wsum = math.fsum(weight_terms)
    assert abs(g_stats[2] - wsum) <= 1e-9 * max(1.0, wsum)
    rsum = math.fsum(ratio_terms)
    assert abs(g_stats[3] - rsum) <= 1e-4 * max(1.0, rsum), (g_stats[3], rsum)
    assert g_stats[4] == cnt["clipped_low"] and g_stats[5] == cnt["clipped_high"]
    assert g_stats[6] == cnt["clamped"] and g_stats[7] == cnt["stale_masked"]
    assert g_stats[8] == extra_counts[0] and g_stats[9] == extra_counts[1]
    kls = math.fsum(kl_terms)
    assert abs(g_stats[10] - kls) <= 1e-3 * abs(kls) + 1e-7
    if want_entropy:
        es = math.fsum(ent_terms)
        assert abs(g_stats[11] - es) <= 1e-4 * abs(es) + 1e-4 * cnt["active_tokens"], (g_stats[11], es)
    return worst


# ------------------------------------------------------------------------------- C2, C3, C5
@pytest.mark.parametrize("name,n_seq,in_place,objective,skip", [
    ("single", 64, False, False, False),   # configs[1]: 64 x 2048 = the bench's 131,072-token mini-batch
    ("single", 32, True, True, True),      # + KL / decoupled ratio / entropy, in place, SKIP_MASKED_READS
    ("long", 8, True, False, False),       # configs[2]: one GRPO group of 32,768-token agentic rows
    ("multi_a", 16, False, True, False),   # configs[4] policy A: prompt masks, staleness 0..10, max 8
    ("multi_b", 8, False, False, True),    # configs[4] policy B: V = 128256
])
def test_full_chain_sampled(cuda_lib, name, n_seq, in_place, objective, skip):
    rl, t = cuda_lib, torch()
    cfg = synth.get_config(name)
    V = cfg.vocab
    lay = synth.seq_layout(cfg)
    L = cfg.seq_len
    N = n_seq * L
    S, G = n_seq, n_seq // cfg.group
    cu = np.ascontiguousarray(lay["cu_seqlens"][:S + 1]).astype(np.int32)
    cu_groups = np.arange(G + 1, dtype=np.int32) * cfg.group
    rewards = np.ascontiguousarray(lay["rewards"][:S]).astype(np.float64)   # rl_group_advantage takes fp64
    ver = np.ascontiguousarray(lay["seq_version"][:S]).astype(np.int32)
    tv, ms = int(lay["trainer_version"]), int(cfg.max_staleness)
    x = t.empty((N, V), dtype=t.bfloat16, device="cuda")
    yd = t.empty(N, dtype=t.int32, device="cuda")
    synth.device_logits(x, V, 0, cfg.seed, targets_out=yd)
    y = yd.cpu().numpy()
    rows = np.sort(np.random.default_rng(cfg.seed).choice(N, size=N_SAMPLED, replace=False))
    mask = np.zeros(N, dtype=np.uint8)
    mask[rows] = np.asarray(lay["loss_mask"][:N])[rows]
    bits = rows_bits(x, rows, V)
    lp_all = torch_logp_all(x, yd, V)          # before an in-place call overwrites the logits
    # behaviour / reference / proximal log-probs of the sampled rows (oracle log-probs + drift)
    lp_ref = oracle_logp_rows(bits, y[rows])
    tstale = (tv - ver)[np.repeat(np.arange(S), L)]
    big = np.zeros(N, dtype=np.uint8)
    big[rows] = np.asarray(lay["big_delta"][:N])[rows]
    base = np.zeros(N)
    base[rows] = lp_ref
    old = synth.perturb_old_logp(base, tstale, big, cfg, cfg.seed)
    bk = oracle.seq_bookkeeping(cu, mask, y, V, ver, tv, ms)
    old[rows] = nudge_out_of_band(old[rows], lp_ref, bk["valid"][rows])
    ref = prox = None
    if objective:
        rng = np.random.default_rng(cfg.seed + 7)
        ref = (old + rng.normal(size=N) * 0.2).astype(np.float32)
        prox = (old + rng.normal(size=N) * 0.01).astype(np.float32)
    # ---- GPU chain: bookkeeping -> advantages -> fused loss (one launch config as bench.py)
    tok_seq = t.empty(N, dtype=t.int32, device="cuda")
    seq_active = t.empty(S, dtype=t.int32, device="cuda")
    counts = t.zeros(20, dtype=t.float64, device="cuda")
    rl.seq_bookkeeping(dev(cu), yd, V, tok_seq, seq_active, loss_mask=dev(mask), seq_version=dev(ver),
                       trainer_version=tv, max_staleness=ms, counts_out=counts)
    adv = t.empty(S, dtype=t.float32, device="cuda")
    zv = t.empty(G, dtype=t.uint8, device="cuda")
    ws_adv = t.empty(max(1, rl.group_advantage_workspace_size(S)), dtype=t.uint8, device="cuda")
    rl.group_advantage(dev(rewards), dev(cu_groups), adv, zv, seq_weight=seq_active, workspace=ws_adv)
    p = rl.LossParams(trainer_version=tv, max_staleness=ms, global_num_seqs=S, active_tokens_dev=counts[0:1])
    if objective:
        p.kl_coef, p.ref_logp, p.prox_logp = 1e-3, dev(ref), dev(prox)
        p.flags |= rl.F_ENTROPY
    if skip:
        p.flags |= rl.F_SKIP_MASKED_READS
    dl = x if in_place else t.empty_like(x)
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    ws = t.empty(rl.policy_loss_workspace_size(N, V), dtype=t.uint8, device="cuda")
    logp = t.empty(N, device="cuda")
    clipped = t.empty(N, dtype=t.uint8, device="cuda")
    rl.policy_loss_fwd_bwd(x, yd, dev(old), tok_seq, adv, p, dl, stats, ws, loss_mask=dev(mask),
                           seq_version=dev(ver), seq_active=seq_active, logp_out=logp, clipped_out=clipped)
    t.cuda.synchronize()
    # ---- per-sequence and integer scalars: exact
    adv_o, zv_o = oracle.group_advantage(rewards, cu_groups, seq_weight=bk["seq_active"])
    assert np.array_equal(adv.cpu().numpy().view(np.uint32), adv_o.view(np.uint32))
    assert np.array_equal(zv.cpu().numpy(), zv_o)
    assert np.array_equal(tok_seq.cpu().numpy(), bk["token_seq"])
    assert np.array_equal(seq_active.cpu().numpy(), bk["seq_active"])
    c = counts.cpu().numpy()
    assert c[0] == bk["active_tokens"] and c[1] == bk["stale_masked"]
    assert c[2] == bk["neg_staleness"] and c[3] == bk["bad_targets"]
    assert np.array_equal(c[4:20], bk["stale_hist"])
    # ---- every row's log-prob (plain PyTorch fp32 reference); skipped rows report 0
    g_lp = logp.cpu().numpy()
    read = (bk["valid"] != 0) if skip else np.ones(N, dtype=bool)
    assert np.all(np.abs(g_lp[read] - lp_all[read]) <= LOGP_ATOL), np.abs(g_lp[read] - lp_all[read]).max()
    if skip:
        assert np.all(g_lp[~read] == 0)
    # ---- sampled rows against the oracle
    po = oracle.LossParams(trainer_version=tv, max_staleness=ms, global_num_seqs=S,
                           global_active_tokens=float(bk["active_tokens"]), kl_coef=1e-3 if objective else 0.0)
    neg_tok = int(sum(cu[i + 1] - cu[i] for i in range(S) if bk["seq_staleness"][i] < 0))
    worst = check_sampled(bits, rows, y, old, mask, bk["token_seq"], adv_o.astype(np.float64), ver, bk["seq_active"],
                          po, g_lp, rows_bits(dl, rows, V), stats.cpu().numpy(), g_clipped=clipped.cpu().numpy(),
                          ref=ref, prox=prox, want_entropy=objective,
                          extra_counts=(bk["bad_targets"], neg_tok), read=read)
    print(f"{name}: worst dlogits row error / |s_t| = {worst:.3e}")
    # unsampled rows are masked: bitwise zero gradient (a sample of them)
    others = np.setdiff1d(np.arange(N), rows)[:: max(1, (N - N_SAMPLED) // 512)]
    assert not rows_bits(dl, others, V).any()
    del x, dl


# ------------------------------------------------------------------------------- R2 worst case
def test_r2_dominant_nontarget_column(cuda_lib):
    """Reading R2 at V = 151936: rows where a NON-target column carries p in [0.85, 0.999] (a
    confident model that sampled another token) — the largest gradient element is s p_h, the one
    the bf16 rounding chain bounds.  Every row must meet Z21 (max |d - d_ref| <= 1e-2 |s_t|), and
    the row sums meet the bound derived in DESIGN.md §3 R2."""
    rl, t = cuda_lib, torch()
    V, N = 151936, 2048
    bits, y, h = synth.dominant_logits(N, V, seed=23)
    x = dev(bits)
    lp_ref = oracle_logp_rows(bits, y)
    tseq = (np.arange(N) // 64).astype(np.int32)
    S = int(tseq[-1]) + 1
    adv = np.random.default_rng(23).uniform(0.5, 2.0, size=S).astype(np.float32)
    old = lp_ref.astype(np.float32)      # ratio 1: every row unclipped, s_t = A (AGG_SUM)
    p = rl.LossParams(agg=rl.AGG_SUM)
    dl = t.empty_like(x)
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    ws = t.empty(rl.policy_loss_workspace_size(N, V), dtype=t.uint8, device="cuda")
    logp = t.empty(N, device="cuda")
    rl.policy_loss_fwd_bwd(x, dev(y), dev(old), dev(tseq), dev(adv), p, dl, stats, ws, logp_out=logp)
    t.cuda.synchronize()
    po = oracle.LossParams(agg=oracle.AGG_SUM)
    gb = dl.view(t.int16).cpu().numpy().view(np.uint16)
    n_dom, worst, worst_sum = 0, 0.0, 0.0
    for b0 in range(0, N, BLOCK):
        xs = oracle.decode_bf16(bits[b0:b0 + BLOCK])
        sl = slice(b0, b0 + BLOCK)
        out = oracle.policy_loss_fwd_bwd(xs, y[sl], old[sl], np.ones(len(xs), np.uint8), tseq[sl],
                                         adv.astype(np.float64), None, None, po)
        d = oracle.decode_bf16(gb[sl])
        ph = np.exp(xs[np.arange(len(xs)), h[sl]] - out["lse"])
        for k in range(len(xs)):
            s = abs(out["scale"][k])
            e = np.abs(d[k] - out["dlogits"][k]).max() / s
            worst = max(worst, e)
            assert e <= DLOGIT_ROW_RTOL, (b0 + k, e, ph[k])
            if h[b0 + k] != y[b0 + k] and 0.85 <= ph[k] <= 0.999:
                n_dom += 1
            amax = np.abs(d[k]).max()
            excess = abs(d[k].sum()) - R2_ROWSUM * amax - R2_ABS * s
            worst_sum = max(worst_sum, abs(d[k].sum()) / amax)
            assert excess <= 0, (b0 + k, abs(d[k].sum()), amax, s)
    assert n_dom >= 600, n_dom
    print(f"R2: {n_dom} dominant non-target rows; worst row error / |s_t| = {worst:.3e}; "
          f"worst |row sum| / max|d| = {worst_sum:.3e}")


# derived in DESIGN.md §3 R2: non-target elements carry <= 2 bf16 roundings (e' cache, output), the
# target one, so |sum_v d_v| <= 3u / (1 - u) max|d| + R2_ABS |s_t| (u = 2^-8; the absolute term
# covers the fp32 row sum S' and p_y = 2^15 / S', relative error <= 2^-16)
U_BF16 = 2.0 ** -8
R2_ROWSUM = 3 * U_BF16 / (1 - U_BF16)
R2_ABS = 2.0 ** -16


# ------------------------------------------------------------------------------- C4 vocab-parallel
@pytest.mark.parametrize("W", [18992, 37984, 151936])
@pytest.mark.parametrize("path", ["nccl", "peer", "peer_ring", "peer_rs1", "peer_rs2", "peer_tmem"])
def test_vocab_parallel_production_widths(cuda_lib, W, path):
    """rl_vocab_parallel_logprob at P = 1 with the per-rank column width of P = 8 (18,992), P = 4
    (37,984) and the whole vocabulary: the kernels' multi-chunk slice geometry of configs[3], on the
    NCCL path and on the in-kernel peer path, with the KL and decoupled-ratio terms, then the C1
    all-reduce call (rl_comm_allreduce_f64, a sum over one rank)."""
    rl, t = cuda_lib, torch()
    N = 8192
    cfg = synth.get_config("vocabpar")
    x = t.empty((N, W), dtype=t.bfloat16, device="cuda")
    yd = t.empty(N, dtype=t.int32, device="cuda")
    synth.device_logits(x, W, 0, cfg.seed, targets_out=yd)
    y = yd.cpu().numpy()
    rows = np.sort(np.random.default_rng(W).choice(N, size=N_SAMPLED, replace=False))
    mask = np.zeros(N, dtype=np.uint8)
    mask[rows] = 1
    L = 1024
    S = N // L
    tseq = (np.arange(N) // L).astype(np.int32)
    ver = np.full(S, 10, dtype=np.int32)
    ver[1] = 9
    adv = np.random.default_rng(W + 1).normal(size=S).astype(np.float32)
    bits = rows_bits(x, rows, W)
    lp_ref = oracle_logp_rows(bits, y[rows])
    rng = np.random.default_rng(W + 2)
    old = np.zeros(N, dtype=np.float32)
    drift = rng.normal(size=len(rows)) * 0.05
    big = rng.uniform(size=len(rows)) < 0.02
    drift[big] = rng.uniform(0.3, 1.0, size=big.sum()) * np.sign(rng.normal(size=big.sum()))
    old[rows] = (lp_ref + drift).astype(np.float32)
    old[rows] = nudge_out_of_band(old[rows], lp_ref, np.ones(len(rows), np.uint8))
    ref = (old + rng.normal(size=N) * 0.2).astype(np.float32)
    prox = (old + rng.normal(size=N) * 0.01).astype(np.float32)
    n_act = float(len(rows))
    p = rl.LossParams(trainer_version=10, kl_coef=1e-3, ref_logp=dev(ref), prox_logp=dev(prox),
                      global_active_tokens=n_act)
    comm = rl.Comm.local()
    try:
        if path.startswith("peer"):
            assert comm.enable_peer_exchange(N)
            rl.dev_set_option(rl.DEV_VP_KERNEL, 1 if path == "peer_ring" else 2)
            if path in ("peer_rs1", "peer_rs2"):   # the multi-rank configurations: rows parked in smem
                rl.dev_set_option(rl.DEV_VC_ROWS, 2 if path == "peer_rs1" else 3)
            if path == "peer_tmem":   # rows parked in tensor memory
                rl.dev_set_option(rl.DEV_VC_TMEM, 2)
        else:
            rl.dev_set_option(rl.DEV_VP_PATH, 1)
        dl = t.empty_like(x)
        stats = t.zeros(12, dtype=t.float64, device="cuda")
        ws = t.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=t.uint8, device="cuda")
        logp = t.empty(N, device="cuda")
        lp_all = torch_logp_all(x, yd, W)
        for _ in range(2):   # twice: the second call runs on the other parity of the peer slots
            rl.vocab_parallel_logprob(x, yd, 0, W, comm, logp, ws, old_logp=dev(old), loss_mask=dev(mask),
                                      token_seq=dev(tseq), seq_adv=dev(adv), seq_version=dev(ver), params=p,
                                      dlogits_shard=dl, stats=stats)
        comm.allreduce_f64(stats)
        t.cuda.synchronize()
    finally:
        rl.dev_set_option(rl.DEV_VP_PATH, 0)
        rl.dev_set_option(rl.DEV_VP_KERNEL, 0)
        rl.dev_set_option(rl.DEV_VC_ROWS, 0)
        rl.dev_set_option(rl.DEV_VC_TMEM, 0)
        comm.destroy()
    g_lp = logp.cpu().numpy()
    assert np.all(np.abs(g_lp - lp_all) <= LOGP_ATOL), np.abs(g_lp - lp_all).max()
    po = oracle.LossParams(trainer_version=10, kl_coef=1e-3, global_active_tokens=n_act)
    check_sampled(bits, rows, y, old, mask, tseq, adv.astype(np.float64), ver, None, po, g_lp,
                  rows_bits(dl, rows, W), stats.cpu().numpy(), ref=ref, prox=prox)
    others = np.setdiff1d(np.arange(N), rows)[::8]
    assert not rows_bits(dl, others, W).any()


# ------------------------------------------------------------------------------- vocab-parallel edge cases
@pytest.mark.parametrize("N", [1, 7, 149, 1000])
@pytest.mark.parametrize("W", [8, 1000, 1004, 18992])
@pytest.mark.parametrize("path", ["peer", "peer_ring", "peer_rs1", "peer_tmem", "nccl"])
def test_vocab_parallel_edge_shapes(cuda_lib, N, W, path):
    """Few rows (fewer than the 148 CTAs: idle CTAs, one row per CTA), a single 16-B vector per row
    (W = 8), widths with and without whole vectors per consumer thread, on both peer kernels and the
    NCCL path: logp, loss and every dlogits row against the oracle."""
    rl, t = cuda_lib, torch()
    ld = (W + 7) // 8 * 8                     # row stride: 16-B aligned rows (W = 1004: 4 tail columns)
    x = t.empty((N, ld), dtype=t.bfloat16, device="cuda")
    yd = t.empty(N, dtype=t.int32, device="cuda")
    synth.device_logits(x, W, 0, W + N, targets_out=yd)
    y = yd.cpu().numpy()
    y[::5] = -100
    yd = dev(y)
    bits = rows_bits(x, np.arange(N), W)
    lp_ref = oracle_logp_rows(bits, y)
    rng = np.random.default_rng(N + W)
    old = np.where(y >= 0, lp_ref + rng.normal(size=N) * 0.1, 0.0).astype(np.float32)
    tseq = (np.arange(N) // 3).astype(np.int32)
    adv = rng.normal(size=int(tseq[-1]) + 1).astype(np.float32)
    mask = (rng.uniform(size=N) < 0.9).astype(np.uint8)
    comm = rl.Comm.local()
    try:
        if path.startswith("peer"):
            assert comm.enable_peer_exchange(N)
            rl.dev_set_option(rl.DEV_VP_KERNEL, 1 if path == "peer_ring" else 2)
            if path in ("peer_rs1", "peer_rs2"):   # the multi-rank configurations: rows parked in smem
                rl.dev_set_option(rl.DEV_VC_ROWS, 2 if path == "peer_rs1" else 3)
            if path == "peer_tmem":   # rows parked in tensor memory
                rl.dev_set_option(rl.DEV_VC_TMEM, 2)
        else:
            rl.dev_set_option(rl.DEV_VP_PATH, 1)
        dl = t.empty_like(x)
        stats = t.zeros(12, dtype=t.float64, device="cuda")
        ws = t.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=t.uint8, device="cuda")
        logp = t.empty(N, device="cuda")
        p = rl.LossParams(agg=rl.AGG_SUM)
        rl.vocab_parallel_logprob(x, yd, 0, W, comm, logp, ws, vocab_shard=W, old_logp=dev(old), loss_mask=dev(mask),
                                  token_seq=dev(tseq), seq_adv=dev(adv), params=p, dlogits_shard=dl, stats=stats)
        t.cuda.synchronize()
    finally:
        rl.dev_set_option(rl.DEV_VP_PATH, 0)
        rl.dev_set_option(rl.DEV_VP_KERNEL, 0)
        rl.dev_set_option(rl.DEV_VC_ROWS, 0)
        rl.dev_set_option(rl.DEV_VC_TMEM, 0)
        comm.destroy()
    out = oracle.policy_loss_fwd_bwd(oracle.decode_bf16(bits), y, old, mask, tseq, adv.astype(np.float64), None,
                                     None, oracle.LossParams(agg=oracle.AGG_SUM))
    g_lp = logp.cpu().numpy()
    ok = y >= 0
    assert np.all(np.abs(g_lp[ok] - out["logp"][ok]) <= LOGP_ATOL)
    st = stats.cpu().numpy()
    band = clip_band(out["ratio"], out["valid"], 0.2, 0.2)
    if not band.any():
        sc = max(abs(out["loss"]), float(np.abs(out["token_loss"]).sum()), 1e-30)
        assert abs(st[0] - out["loss"]) <= LOSS_RTOL * sc
        d = oracle.decode_bf16(rows_bits(dl, np.arange(N), W))
        for k in range(N):
            s = out["scale"][k]
            if s == 0:
                assert np.all(d[k] == 0), k
            else:
                assert np.abs(d[k] - out["dlogits"][k]).max() <= DLOGIT_ROW_RTOL * abs(s), k
    assert st[1] == out["stats"]["active_tokens"]


# ------------------------------------------------------------------------------- determinism
@pytest.mark.parametrize("kind,W", [("sv", 151936), ("peer", 37984), ("peer", 18992), ("peer_rs1", 18992),
                                    ("peer_tmem", 37984), ("peer_tmem", 18992), ("peer_ring", 37984), ("nccl", 37984)])
def test_repeated_calls_bitwise_identical(cuda_lib, kind, W):
    """Five back-to-back calls on the same inputs give bit-identical log-probs, statistics and
    dlogits (the reduction order is fixed, §8(a) a6).  Guards the TMA-ring consumer protocol: a warp
    releasing a ring slot before all its lanes read it (fixed in sm100::mbar_arrive_lane0) showed up
    as rare, slightly different row statistics between identical calls."""
    rl, t = cuda_lib, torch()
    N = 16384
    x = t.empty((N, W), dtype=t.bfloat16, device="cuda")
    yd = t.empty(N, dtype=t.int32, device="cuda")
    synth.device_logits(x, W, 0, 11, targets_out=yd)
    g = t.Generator(device="cuda").manual_seed(3)
    old = -t.rand(N, device="cuda", generator=g) * 4
    L = 512
    tseq = (t.arange(N, device="cuda") // L).to(t.int32)
    adv = t.randn(N // L, device="cuda", generator=g)
    p = rl.LossParams(global_active_tokens=float(N))
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    logp = t.empty(N, device="cuda")
    dl = t.empty_like(x)
    outs = []
    comm = None
    try:
        if kind == "sv":
            ws = t.empty(rl.policy_loss_workspace_size(N, W), dtype=t.uint8, device="cuda")
            call = lambda: rl.policy_loss_fwd_bwd(x, yd, old, tseq, adv, p, dl, stats, ws, logp_out=logp)
        else:
            comm = rl.Comm.local()
            if kind.startswith("peer"):
                assert comm.enable_peer_exchange(N)
                rl.dev_set_option(rl.DEV_VP_KERNEL, 1 if kind == "peer_ring" else 2)
                if kind == "peer_rs1":
                    rl.dev_set_option(rl.DEV_VC_ROWS, 2)
                if kind == "peer_tmem":
                    rl.dev_set_option(rl.DEV_VC_TMEM, 2)
            else:
                rl.dev_set_option(rl.DEV_VP_PATH, 1)
            ws = t.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=t.uint8, device="cuda")
            call = lambda: rl.vocab_parallel_logprob(x, yd, 0, W, comm, logp, ws, old_logp=old, token_seq=tseq,
                                                     seq_adv=adv, params=p, dlogits_shard=dl, stats=stats)
        for _ in range(5):
            stats.zero_()
            call()
            outs.append((logp.clone(), stats.clone(), dl.view(t.int16)[::7].clone()))
        t.cuda.synchronize()
    finally:
        rl.dev_set_option(rl.DEV_VP_PATH, 0)
        rl.dev_set_option(rl.DEV_VP_KERNEL, 0)
        rl.dev_set_option(rl.DEV_VC_ROWS, 0)
        rl.dev_set_option(rl.DEV_VC_TMEM, 0)
        if comm is not None:
            comm.destroy()
    for c in range(1, 5):
        for a, b, what in zip(outs[0], outs[c], ("logp", "stats", "dlogits")):
            diff = (a != b).nonzero()
            assert diff.numel() == 0, (kind, W, c, what, diff[:8].flatten().tolist())


# ------------------------------------------------------------------------------- padded vocabulary
@pytest.mark.parametrize("in_place", [False, True])
def test_padded_vocab_tail_columns(cuda_lib, in_place):
    """V = 151,665 (Qwen2.5's vocabulary, not a multiple of 8) in rows of ld = 151,936: the default
    kernel must take its generic instantiation (the exact-width ones assume whole 16-B vectors) and
    cover the 1 scalar tail column of every row — targets placed in the last 9 columns, sampled rows
    against the oracle, the pad columns beyond V left untouched."""
    rl, t = cuda_lib, torch()
    N, V, ld = 8192, 151665, 151936
    x = t.empty((N, ld), dtype=t.bfloat16, device="cuda")
    yd = t.empty(N, dtype=t.int32, device="cuda")
    synth.device_logits(x, V, 0, 21, targets_out=yd)
    x[:, V:] = 7.0                                 # pad columns: must stay as they are
    y = yd.cpu().numpy()
    y[::3] = V - 1 - (np.arange(len(y[::3])) % 9)  # targets in the tail (incl. the scalar column)
    y[::11] = -100
    yd = dev(y)
    rows = np.sort(np.random.default_rng(9).choice(N, size=N_SAMPLED, replace=False))
    mask = np.zeros(N, dtype=np.uint8)
    mask[rows] = 1
    L = 512
    tseq = (np.arange(N) // L).astype(np.int32)
    adv = np.random.default_rng(10).normal(size=N // L).astype(np.float32)
    bits = rows_bits(x, rows, V)
    lp_ref = oracle_logp_rows(bits, y[rows])
    rng = np.random.default_rng(12)
    old = np.zeros(N, dtype=np.float32)
    ok = y[rows] >= 0
    old[rows] = np.where(ok, lp_ref + rng.normal(size=len(rows)) * 0.05, 0.0).astype(np.float32)
    old[rows] = nudge_out_of_band(old[rows], lp_ref, ok.astype(np.uint8))
    n_act = float((mask[rows] != 0)[ok].sum())
    p = rl.LossParams(global_active_tokens=n_act)
    dl = x if in_place else t.full_like(x, 7.0)
    stats = t.zeros(12, dtype=t.float64, device="cuda")
    ws = t.empty(rl.policy_loss_workspace_size(N, V), dtype=t.uint8, device="cuda")
    logp = t.empty(N, device="cuda")
    clipped = t.empty(N, dtype=t.uint8, device="cuda")
    rl.policy_loss_fwd_bwd(x, yd, dev(old), dev(tseq), dev(adv), p, dl, stats, ws, loss_mask=dev(mask),
                           logp_out=logp, clipped_out=clipped, vocab=V)
    t.cuda.synchronize()
    g_lp = logp.cpu().numpy()
    po = oracle.LossParams(global_active_tokens=n_act)
    check_sampled(bits, rows, y, old, mask, tseq, adv.astype(np.float64), None, None, po, g_lp,
                  rows_bits(dl, rows, V), stats.cpu().numpy(), g_clipped=clipped.cpu().numpy())
    assert t.all(dl[:, V:] == 7.0), "pad columns beyond V were written"
