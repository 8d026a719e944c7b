"""vp_cache_kernel phase counters across P ranks (development; needs the trace build):
    python -m paper_2605_15565_b200.build --variant trace
    RL_LIB_PATH=paper_2605_15565_b200/librlpolicy_trace.so torchrun --nproc-per-node P tools/vptrace.py [--width-of W]
Each rank holds its shard of a 65,536-token row batch (V = 151936 split P ways, or the width of a
W-way split); prints, per rank, the per-row averages of the kernel's cycle counters (CTA mean)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2605_15565_b200 as rl
    import synth
    from paper_2605_15565_b200.parallel import shard_vocab
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = rl.load()
    lib.rl_debug_vc_trace.restype = ctypes.c_int
    lib.rl_debug_vc_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    comm = rl.Comm.from_torch() if world > 1 else rl.Comm.local()
    if "--pub" in sys.argv:
        rl.dev_set_option(6, int(sys.argv[sys.argv.index("--pub") + 1]) + 1)
    if "--rs" in sys.argv:
        rl.dev_set_option(5, int(sys.argv[sys.argv.index("--rs") + 1]) + 1)
    rl.dev_set_option(rl.DEV_VP_KERNEL, 2)   # the register-cache kernel (the only one with counters)
    V, N = 151936, 65536
    W = int(sys.argv[sys.argv.index("--width-of") + 1]) if "--width-of" in sys.argv else world
    sh = shard_vocab(V, W, rank % W)
    Vr = sh.size
    x = torch.empty((N, Vr), dtype=torch.bfloat16, device=dev)
    y = torch.empty(N, dtype=torch.int32, device=dev)
    synth.device_logits(x, Vr, 0, 4 + rank, targets_out=y)
    y = (y + sh.offset) if world > 1 else y
    assert comm.enable_peer_exchange(N)
    logp = torch.empty(N, device=dev)
    old = torch.zeros(N, device=dev)
    tseq = torch.zeros(N, dtype=torch.int32, device=dev)
    adv = torch.ones(1, device=dev)
    stats = torch.zeros(12, dtype=torch.float64, device=dev)
    dl = torch.empty_like(x)
    ws = torch.empty(rl.vocab_parallel_workspace_size(N, world), dtype=torch.uint8, device=dev)
    p = rl.LossParams(agg=rl.AGG_SUM)
    off, Vt = (sh.offset, V) if world > 1 else (0, Vr)
    call = lambda: rl.vocab_parallel_logprob(x, y, off, Vt, comm, logp, ws, vocab_shard=Vr, old_logp=old,
                                             token_seq=tseq, seq_adv=adv, params=p, dlogits_shard=dl, stats=stats)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    assert lib.rl_debug_vc_trace(None, 0, 1) == 0
    reps = 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        call()
    b.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (256 * 12))()
    assert lib.rl_debug_vc_trace(ctypes.cast(buf, ctypes.c_void_p), ctypes.sizeof(buf), 0) == 0
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(256, 12)[:148].astype(np.float64)
    rows_per_cta = N / 148 * reps
    ghz = 1.965
    names = ["consumer wait scale", "consumer wait data", "collector wait own record",
             "collector poll peers", "collector chain / row"]
    line = [f"[rank {rank}] {a.elapsed_time(b) / reps:.3f} ms/call, Vr={Vr}"]
    for i, nm in list(enumerate(names)) + [(8, "collector records -> scale")]:
        per = tr[:, i].mean() / (rows_per_cta if i < 2 else max(1.0, tr[:, 5].mean())) / (ghz * 1e3)
        line.append(f"{nm}: {per:.2f} us/row")
    print("; ".join(line), flush=True)
    if "--dump" in sys.argv:   # per-CTA counters of this rank (cross-rank straggler analysis)
        np.save(sys.argv[sys.argv.index("--dump") + 1] + f"_rank{rank}.npy", tr)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
