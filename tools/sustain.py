"""Sustained-load check (development tool): back-to-back fused-loss calls on distinct buffers, per-call
CUDA-event times in groups, with nvidia-smi SM clock / power samples.
    python tools/sustain.py [--calls 60] [--copy | --logprob]"""
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2605_15565_b200 as rl
    import synth
    calls = int(sys.argv[sys.argv.index("--calls") + 1]) if "--calls" in sys.argv else 60
    rl.load()
    N, V = 131072, 151936
    xs, ys = [], []
    for i in range(2):
        x = torch.empty((N, V), dtype=torch.bfloat16, device="cuda")
        y = torch.empty(N, dtype=torch.int32, device="cuda")
        synth.device_logits(x, V, 0, 2 + i, targets_out=y)
        xs.append(x)
        ys.append(y)
    dl = torch.empty(N * V, dtype=torch.bfloat16, device="cuda").view(N, V)
    old = torch.zeros(N, dtype=torch.float32, device="cuda")
    tseq = torch.zeros(N, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, dtype=torch.float32, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.policy_loss_workspace_size(N, V), dtype=torch.uint8, device="cuda")
    logp = torch.empty(N, device="cuda")
    p = rl.LossParams(agg=rl.AGG_SUM)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks.mem",
                                  "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True).stdout
            samples.append(out.strip())
            stop.wait(0.2)

    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    ev = []
    for i in range(calls):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if "--copy" in sys.argv:
            dl.copy_(xs[i % 2])
        elif "--logprob" in sys.argv:
            rl.token_logprob(xs[i % 2], ys[i % 2], logp)
        else:
            rl.policy_loss_fwd_bwd(xs[i % 2], ys[i % 2], old, tseq, adv, p, dl, stats, ws, logp_out=logp)
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ts = [a.elapsed_time(b) for a, b in ev]
    nbytes = (1 if "--logprob" in sys.argv else 2) * N * V * 2
    G = max(10, calls // 12)
    for g in range(0, calls, G):
        grp = ts[g:g + G]
        m = sum(grp) / len(grp)
        print(f"calls {g:3d}-{g + len(grp) - 1:3d}: avg {m:7.3f} ms  {nbytes / m / 1e6:7.1f} GB/s  min {min(grp):.3f}")
    print("smi (sm MHz, W, mem MHz):", samples[:: max(1, len(samples) // 16)])


if __name__ == "__main__":
    main()
