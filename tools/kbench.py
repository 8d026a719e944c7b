"""Kernel micro-benchmark (development tool): times the fused loss kernel variants, the
read-only log-prob kernel and a torch copy of the same bytes, each with CUDA events.

    python tools/kbench.py [--rows 131072] [--vocab 151936] [--reps 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=131072)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--two-pass", action="store_true", help="the exact two-pass kernel (development option)")
    args = ap.parse_args()
    import torch
    import paper_2605_15565_b200 as rl
    import synth
    rl.load()
    N, V = args.rows, args.vocab
    x = torch.empty((N, V), dtype=torch.bfloat16, device="cuda")
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    synth.device_logits(x, V, 0, 2, targets_out=y)
    dl = torch.empty_like(x)
    old = torch.zeros(N, dtype=torch.float32, device="cuda")
    tseq = torch.zeros(N, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, dtype=torch.float32, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.policy_loss_workspace_size(N, V), dtype=torch.uint8, device="cuda")
    logp = torch.empty(N, device="cuda")
    nbytes = N * V * 2

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return min(ts), sum(ts) / len(ts)

    t, avg = timeit(lambda: dl.copy_(x))
    print(f"torch copy      : {t:8.3f} ms  {2 * nbytes / t / 1e6:8.1f} GB/s (avg {avg:.3f})")
    t, avg = timeit(lambda: rl.token_logprob(x, y, logp))
    print(f"token_logprob   : {t:8.3f} ms  {nbytes / t / 1e6:8.1f} GB/s read (avg {avg:.3f})")
    p = rl.LossParams(agg=rl.AGG_SUM)
    kern = "two_pass" if args.two_pass else "sv"
    rl.dev_set_option(rl.DEV_LOSS_KERNEL, 1 if kern == "two_pass" else 0)
    t, avg = timeit(lambda: rl.policy_loss_fwd_bwd(x, y, old, tseq, adv, p, dl, stats, ws, logp_out=logp))
    print(f"loss ({kern:8s}): {t:8.3f} ms  {2 * nbytes / t / 1e6:8.1f} GB/s R+W (avg {avg:.3f})")
    t, avg = timeit(lambda: rl.policy_loss_fwd_bwd(x, y, old, tseq, adv, p, x, stats, ws, logp_out=logp))
    print(f"loss in-place   : {t:8.3f} ms  {2 * nbytes / t / 1e6:8.1f} GB/s R+W (avg {avg:.3f})")


if __name__ == "__main__":
    main()
