"""Fused-loss cost of the NEXT-2 terms (development tool): one 131,072 x 151,936 bf16 call with
each option on its own.   python tools/objbench.py [clip kl prox entropy full]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2605_15565_b200 as rl
    import synth
    rl.load()
    N, V = 131072, 151936
    x = torch.empty((N, V), dtype=torch.bfloat16, device="cuda")
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    synth.device_logits(x, V, 0, 2, targets_out=y)
    dl = torch.empty_like(x)
    lp = torch.empty(N, device="cuda")
    rl.token_logprob(x, y, lp)
    old = lp + 0.02 * torch.randn(N, device="cuda")
    ref = old + 0.2 * torch.randn(N, device="cuda")
    prox = old + 0.02 * torch.randn(N, device="cuda")
    tseq = torch.zeros(N, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.policy_loss_workspace_size(N, V), dtype=torch.uint8, device="cuda")
    names = [a for a in sys.argv[1:] if not a.startswith("-")] or ["clip", "kl", "prox", "entropy", "full"]
    for name in names:
        p = rl.LossParams(agg=rl.AGG_SUM)
        if name in ("kl", "full"):
            p.kl_coef, p.ref_logp = 1e-3, ref
        if name in ("prox", "full"):
            p.prox_logp = prox
        if name in ("entropy", "full"):
            p.flags |= rl.F_ENTROPY
        f = lambda: rl.policy_loss_fwd_bwd(x, y, old, tseq, adv, p, dl, stats, ws, logp_out=lp)
        f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(int(os.environ.get("OBJ_REPS", "5"))):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{name:8s}: {min(ts):7.3f} ms  {2 * N * V * 2 / min(ts) / 1e6:7.1f} GB/s  (redo rows: "
              f"{int(ws[-(N + 255) // 256 * 256:][:N].sum().item()) if False else 'n/a'})")


if __name__ == "__main__":
    main()
