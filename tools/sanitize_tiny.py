"""One tiny call of every kernel family of librlpolicy.so, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_tiny.py [family ...]

Families: sv (single-visit cluster loss + its two-pass fixup), two_pass, sv_ext (NEXT-2 terms),
logprob, bookkeeping, advantage, vp_nccl (stats + all-gather + vp_finish_tma, P = 1), vp_peer
(vp_ring_kernel, P = 1 self exchange, two calls: both slot parities), m2po, delta, lmhead.
Shapes span several chunks / tiles and a ragged tail but stay small (sanitizers are ~100x slower).
Prints SANITIZE_OK <family> after each family completes (results are checked by the parity tests).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_15565_b200 as rl  # noqa: E402
import synth  # noqa: E402


def loss_inputs(N, V, dtype=torch.bfloat16, seed=1):
    x = torch.empty((N, V), dtype=dtype, device="cuda")
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    synth.device_logits(x, V, 0, seed, targets_out=y)
    y[::17] = -100
    old = torch.randn(N, device="cuda") * 0.5 - 3.0
    L = 64
    S = (N + L - 1) // L
    tseq = (torch.arange(N, device="cuda") // L).to(torch.int32)
    adv = torch.randn(S, device="cuda")
    mask = (torch.rand(N, device="cuda") < 0.8).to(torch.uint8)
    return x, y, old, tseq, adv, mask, S


def fam_sv(two_pass=False, ext=False):
    rl.dev_set_option(rl.DEV_LOSS_KERNEL, 1 if two_pass else 0)
    for V in (1000, 151936):   # ragged small V; the EXACT full-width instantiation
        N = 300 if V < 10000 else 40
        x, y, old, tseq, adv, mask, S = loss_inputs(N, V)
        p = rl.LossParams(global_active_tokens=float(N))
        if ext:
            p.kl_coef, p.ref_logp, p.prox_logp = 1e-3, old + 0.1, old - 0.05
            p.flags |= rl.F_ENTROPY
        dl = torch.empty_like(x)
        stats = torch.zeros(12, dtype=torch.float64, device="cuda")
        ws = torch.empty(rl.policy_loss_workspace_size(N, V), dtype=torch.uint8, device="cuda")
        logp = torch.empty(N, device="cuda")
        clipped = torch.empty(N, dtype=torch.uint8, device="cuda")
        rl.policy_loss_fwd_bwd(x, y, old, tseq, adv, p, dl, stats, ws, loss_mask=mask, logp_out=logp,
                               clipped_out=clipped)
        p.flags |= rl.F_SKIP_MASKED_READS
        rl.policy_loss_fwd_bwd(x, y, old, tseq, adv, p, x, stats, ws, loss_mask=mask, logp_out=logp)  # in place
    torch.cuda.synchronize()
    rl.dev_set_option(rl.DEV_LOSS_KERNEL, 0)


def fam_logprob():
    for V in (1000, 151936):
        N = 200
        x, y, *_ = loss_inputs(N, V)
        logp = torch.empty(N, device="cuda")
        lse = torch.empty(N, device="cuda")
        rl.token_logprob(x, y, logp, lse)
    torch.cuda.synchronize()


def fam_bookkeeping_advantage():
    N, V = 1000, 500
    cu = torch.tensor([0, 5, 5, 300, 1000], dtype=torch.int32, device="cuda")
    y = torch.randint(-2, V + 2, (N,), dtype=torch.int32, device="cuda")
    S = 4
    tok = torch.empty(N, dtype=torch.int32, device="cuda")
    act = torch.empty(S, dtype=torch.int32, device="cuda")
    counts = torch.zeros(20, dtype=torch.float64, device="cuda")
    rl.seq_bookkeeping(cu, y, V, tok, act, loss_mask=(torch.rand(N, device="cuda") < 0.5).to(torch.uint8),
                       seq_version=torch.tensor([3, 9, 10, 12], dtype=torch.int32, device="cuda"),
                       trainer_version=11, max_staleness=1, counts_out=counts)
    rewards = torch.rand(64, device="cuda", dtype=torch.float64)
    cug = torch.arange(0, 65, 8, dtype=torch.int32, device="cuda")
    adv = torch.empty(64, device="cuda")
    zv = torch.empty(8, dtype=torch.uint8, device="cuda")
    ws = torch.empty(max(1, rl.group_advantage_workspace_size(64)), dtype=torch.uint8, device="cuda")
    w = torch.randint(0, 100, (64,), dtype=torch.int32, device="cuda")
    rl.group_advantage(rewards, cug, adv, zv, batch_norm=True, seq_weight=w, workspace=ws)
    torch.cuda.synchronize()


def fam_vp(peer):
    comm = rl.Comm.local()
    rl.dev_set_option(rl.DEV_VP_PATH, 0 if peer else 1)
    for V in (1000, 18992):    # small; the P = 8 shard width (2 ring slots per slice)
        N = 400
        x, y, old, tseq, adv, mask, S = loss_inputs(N, V)
        if peer:
            assert comm.enable_peer_exchange(N)
        p = rl.LossParams(global_active_tokens=float(N), kl_coef=1e-3, ref_logp=old + 0.1)
        dl = torch.empty_like(x)
        stats = torch.zeros(12, dtype=torch.float64, device="cuda")
        ws = torch.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=torch.uint8, device="cuda")
        logp = torch.empty(N, device="cuda")
        for _ in range(2):
            rl.vocab_parallel_logprob(x, y, 0, V, comm, logp, ws, old_logp=old, loss_mask=mask, token_seq=tseq,
                                      seq_adv=adv, params=p, dlogits_shard=dl, stats=stats)
        rl.vocab_parallel_logprob(x, y, 0, V, comm, logp, ws)   # log-prob only
        comm.allreduce_f64(stats)
    torch.cuda.synchronize()
    rl.dev_set_option(rl.DEV_VP_PATH, 0)
    comm.destroy()


def fam_m2po():
    n = 5000
    logp = torch.randn(n, device="cuda") - 2
    old = logp + torch.randn(n, device="cuda") * 0.1
    mask = torch.empty(n, dtype=torch.uint8, device="cuda")
    st = torch.zeros(5, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.m2po_workspace_size(n), dtype=torch.uint8, device="cuda")
    rl.m2po_mask(logp, old, mask, st, ws, tau=0.002)
    torch.cuda.synchronize()


def fam_delta():
    n = 3 * 16384 + 77
    a = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device="cuda")
    b = a.clone()
    b[torch.randint(0, n, (n // 50,), device="cuda")] += 1
    cap = n
    idx = torch.empty(cap, dtype=torch.int32, device="cuda")
    words = torch.empty(cap, dtype=torch.int16, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(rl.delta_workspace_size(n), dtype=torch.uint8, device="cuda")
    rl.delta_encode(a, b, idx, words, cnt, ws)
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    rl.delta_apply(a, idx, words, cnt, bad)
    torch.cuda.synchronize()


def fam_lmhead():
    N, d, V = 300, 256, 1000
    h = (torch.randn(N, d, device="cuda") * 0.5).to(torch.bfloat16)
    W = (torch.randn(V, d, device="cuda") * 0.05).to(torch.bfloat16)
    y = torch.randint(0, V, (N,), dtype=torch.int32, device="cuda")
    logp = torch.empty(N, device="cuda")
    lse = torch.empty(N, device="cuda")
    ws = torch.empty(max(1, rl.lmhead_workspace_size(N, d, V)), dtype=torch.uint8, device="cuda")
    rl.lmhead_logprob(h, W, y, logp, lse, workspace=ws)
    torch.cuda.synchronize()


FAMILIES = {
    "sv": lambda: fam_sv(),
    "two_pass": lambda: fam_sv(two_pass=True),
    "sv_ext": lambda: fam_sv(ext=True),
    "logprob": fam_logprob,
    "bookkeeping": fam_bookkeeping_advantage,
    "vp_nccl": lambda: fam_vp(False),
    "vp_peer": lambda: fam_vp(True),
    "m2po": fam_m2po,
    "delta": fam_delta,
    "lmhead": fam_lmhead,
}

if __name__ == "__main__":
    rl.load()
    for name in (sys.argv[1:] or list(FAMILIES)):
        FAMILIES[name]()
        print("SANITIZE_OK", name, flush=True)
