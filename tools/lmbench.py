"""Fused LM-head log-prob throughput (development tool, NEXT 4): rl_lmhead_logprob on N tokens of
a d = 4096, V = 151936 bf16 head (Qwen3-8B sized), TFLOP/s of the GEMM it contains (2 N V d).
    python tools/lmbench.py [--rows 16384] [--reps 5] [--bwd [--chunk C]]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2605_15565_b200 as rl
    N = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 16384
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    d, V = 4096, 151936
    rl.load()
    if "--single" in sys.argv:   # single-CTA kernels instead of cta_group::2 pairs (development A/B)
        rl.dev_set_option(rl.DEV_LM_PAIR, 1)
    if "--pairs" in sys.argv:    # pairs for the forward too
        rl.dev_set_option(rl.DEV_LM_PAIR, 2)
    if "--own-gemm" in sys.argv:  # the backward's dh / dW GEMMs on lm_gemm_kernel (tcgen05)
        rl.dev_set_option(rl.DEV_LM_GEMM, 2)

    g = torch.Generator(device="cuda").manual_seed(1)
    h = torch.randn(N, d, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda", generator=g) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    y = torch.randint(0, V, (N,), device="cuda", generator=g, dtype=torch.int32)
    lp = torch.empty(N, device="cuda")
    lse = torch.empty(N, device="cuda")
    ws = torch.empty(max(1, rl.lmhead_workspace_size(N, d, V)), dtype=torch.uint8, device="cuda")
    call = lambda: rl.lmhead_logprob(h, w, y, lp, lse, workspace=ws)
    call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    fl = 2.0 * N * V * d
    # the same GEMM through cuBLAS, logits materialised (the unfused baseline's first step)
    x = h[:2048] @ w.T
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        x = h[:2048] @ w.T
    b.record()
    torch.cuda.synchronize()
    tc = a.elapsed_time(b) / 3
    print(f"lmhead N={N} d={d} V={V}: min {min(ts):.3f} ms avg {sum(ts)/len(ts):.3f} ms "
          f"{fl / min(ts) / 1e9:.1f} TFLOP/s; cuBLAS h[:2048] @ W^T: {tc:.3f} ms "
          f"{2.0 * 2048 * V * d / tc / 1e9:.1f} TFLOP/s")
    if "--bwd" in sys.argv:  # NEXT 4 backward: G recompute (2NVd) + dh (2NVd) + dW (2NVd)
        C = int(sys.argv[sys.argv.index("--chunk") + 1]) if "--chunk" in sys.argv else min(N, 8192)
        s = torch.randn(N, device="cuda", generator=g) * 1e-4
        wsb = torch.empty(rl.lmhead_loss_bwd_workspace_size(C, V), dtype=torch.uint8, device="cuda")
        dh = torch.empty(N, d, device="cuda")
        dW = torch.empty(V, d, device="cuda")
        bwd = lambda: rl.lmhead_loss_bwd(h, w, y, lse, s, wsb, dhidden=dh, dweight=dW)
        bwd()
        torch.cuda.synchronize()
        tb = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            bwd()
            b.record()
            torch.cuda.synchronize()
            tb.append(a.elapsed_time(b))
        flb = 6.0 * N * V * d
        print(f"lmhead bwd N={N} chunk={C}: min {min(tb):.3f} ms avg {sum(tb)/len(tb):.3f} ms "
              f"{flb / min(tb) / 1e9:.1f} TFLOP/s (6 N V d)")


if __name__ == "__main__":
    main()
