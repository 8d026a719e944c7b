"""Vocab-parallel call on ONE GPU with a shard of V/P columns (development tool): times
rl_vocab_parallel_logprob with the fused loss on a 1-rank comm, so the kernels can be profiled
in isolation (ncu) — the all-gather of a 1-rank comm is a copy.
    python tools/vpbench.py [--P 4] [--rows 65536] [--reps 10] [--adv0 (s = 0: zero rows)] [--peer]"""
import ctypes
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
    Vr = (V + P - 1) // P // 8 * 8
    x = torch.empty((N, Vr), dtype=torch.bfloat16, device="cuda")
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    synth.device_logits(x, Vr, 0, 4, targets_out=y)
    dl = torch.empty_like(x)
    buf = (ctypes.c_uint8 * 128)()
    assert lib.rl_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)) == 0
    h = ctypes.c_void_p()
    assert lib.rl_comm_init(ctypes.byref(h), bytes(buf), 1, 0) == 0
    comm = rl.Comm(h.value, 1, 0)
    logp = torch.empty(N, device="cuda")
    old = torch.zeros(N, device="cuda")
    tseq = torch.zeros(N, dtype=torch.int32, device="cuda")
    adv = torch.zeros(1, device="cuda") if "--adv0" in sys.argv else torch.ones(1, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.vocab_parallel_workspace_size(N, 1), dtype=torch.uint8, device="cuda")
    p = rl.LossParams(agg=rl.AGG_SUM)
    if "--peer" in sys.argv:  # in-kernel exchange (RL_VP_FUSED=smem selects the first fused kernel)
        assert comm.enable_peer_exchange(N)
    call = lambda: rl.vocab_parallel_logprob(x, y, 0, Vr, comm, logp, ws, vocab_shard=Vr, old_logp=old,
                                             token_seq=tseq, seq_adv=adv, params=p, dlogits_shard=dl, stats=stats)
    call()
    torch.cuda.synchronize()
    tracing = os.environ.get("RL_TRACE") is not None and "--peer" in sys.argv
    if tracing:
        lib.rl_debug_trace_vp2.restype = ctypes.c_int
        lib.rl_debug_trace_vp2.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        assert lib.rl_debug_trace_vp2(None, 0, 1) == 0
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if tracing:  # per-CTA cycles of team 0 / the service lane, averaged over CTAs and calls
        buf = (ctypes.c_ulonglong * (256 * 4))()
        assert lib.rl_debug_trace_vp2(ctypes.cast(buf, ctypes.c_void_p), ctypes.sizeof(buf), 0) == 0
        import numpy as np
        tr = np.frombuffer(buf, dtype=np.uint64).reshape(256, 4)[:148].astype(np.float64) / reps
        mhz = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else 1965
        for i, name in enumerate(["team0 pass 1", "team0 wait scale", "team0 pass 2", "service wait peers"]):
            print(f"  {name:20s} {tr[:, i].mean() / (mhz * 1e3):8.3f} ms per call (cycles at {mhz} MHz)")
    nbytes = 2 * N * Vr * 2
    print(f"vocab-parallel shard P={P} ({Vr} cols) x {N} rows: min {min(ts):.3f} ms avg {sum(ts)/len(ts):.3f} ms"
          f"  {nbytes / min(ts) / 1e6:.1f} GB/s algorithmic (R+W)")
    comm.destroy()


if __name__ == "__main__":
    main()
