"""Vocab-parallel call on ONE GPU with a shard of V/P columns (development tool): times
rl_vocab_parallel_logprob with the fused loss on a 1-rank comm, so the kernels can be profiled
in isolation (ncu) — the all-gather of a 1-rank comm is a copy.
    python tools/vpbench.py [--P 4] [--width W] [--rows 65536] [--reps 10] [--adv0 (s = 0: zero rows)] [--peer]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2605_15565_b200 as rl
    import synth
    P = int(sys.argv[sys.argv.index("--P") + 1]) if "--P" in sys.argv else 4
    N = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 65536
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 10
    lib = rl.load()
    V = 151936
    Vr = int(sys.argv[sys.argv.index("--width") + 1]) if "--width" in sys.argv else (V + P - 1) // P // 8 * 8
    x = torch.empty((N, Vr), dtype=torch.bfloat16, device="cuda")
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    synth.device_logits(x, Vr, 0, 4, targets_out=y)
    dl = torch.empty_like(x)
    comm = rl.Comm.local()
    logp = torch.empty(N, device="cuda")
    old = torch.zeros(N, device="cuda")
    tseq = torch.zeros(N, dtype=torch.int32, device="cuda")
    adv = torch.zeros(1, device="cuda") if "--adv0" in sys.argv else torch.ones(1, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=torch.uint8, device="cuda")
    p = rl.LossParams(agg=rl.AGG_SUM)
    if "--peer" in sys.argv:  # in-kernel exchange (vp_cache_kernel; --ring: vp_ring_kernel)
        assert comm.enable_peer_exchange(N)
        if "--ring" in sys.argv:
            rl.dev_set_option(rl.DEV_VP_KERNEL, 1)
        if "--groups" in sys.argv:
            rl.dev_set_option(rl.DEV_VC_GROUPS, int(sys.argv[sys.argv.index("--groups") + 1]))
        if "--pub" in sys.argv:  # record send mode (0 collector strong, 1 last warp weak, 2 collector weak)
            rl.dev_set_option(rl.DEV_VC_PUB, int(sys.argv[sys.argv.index("--pub") + 1]) + 1)
        if "--delay" in sys.argv:  # vp_ring_kernel rows between a slice's two reads
            rl.dev_set_option(rl.DEV_VR_DELAY, int(sys.argv[sys.argv.index("--delay") + 1]))
        if "--tmem" in sys.argv:  # parked rows in tensor memory
            rl.dev_set_option(rl.DEV_VC_TMEM, 2)
        if "--rs" in sys.argv:   # rows parked in shared memory
            rl.dev_set_option(rl.DEV_VC_ROWS, int(sys.argv[sys.argv.index("--rs") + 1]) + 1)
    else:
        rl.dev_set_option(rl.DEV_VP_PATH, 1)
    call = lambda: rl.vocab_parallel_logprob(x, y, 0, Vr, comm, logp, ws, vocab_shard=Vr, old_logp=old,
                                             token_seq=tseq, seq_adv=adv, params=p, dlogits_shard=dl, stats=stats)
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
    nbytes = 2 * N * Vr * 2
    print(f"vocab-parallel shard P={P} ({Vr} cols) x {N} rows: min {min(ts):.3f} ms avg {sum(ts)/len(ts):.3f} ms"
          f"  {nbytes / min(ts) / 1e6:.1f} GB/s algorithmic (R+W)")
    comm.destroy()


if __name__ == "__main__":
    main()
