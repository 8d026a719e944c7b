"""Vocab-parallel peer path across ranks at a chosen shard width (development):
    torchrun --nproc-per-node P tools/vp_width_multi.py --width W [KEY=VALUE dev options ...]
Every rank holds W columns of a V = P*W vocabulary (65,536 rows); times 20 back-to-back fused-loss
calls with CUDA events and prints the max over ranks (e.g. the P = 8 shard width on 4 GPUs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2605_15565_b200 as rl
    import synth
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rl.load()
    opts = [a for a in sys.argv[1:] if "=" in a]
    for kv in opts:
        k, v = kv.split("=")
        rl.dev_set_option(int(k), int(v))
    W = int(sys.argv[sys.argv.index("--width") + 1])
    N, V = 65536, world * W
    comm = rl.Comm.from_torch()
    x = torch.empty((N, W), dtype=torch.bfloat16, device=dev)
    y = torch.empty(N, dtype=torch.int32, device=dev)
    synth.device_logits(x, W, 0, 7, targets_out=y)   # same rows and targets on every rank: the targets
    # fall in rank 0's columns (a consistent global id), as in a real split
    old = torch.zeros(N, device=dev)   # ratio = e^logp < 1 - eps with A = 1 > 0: unclipped, s != 0 on every row
    tseq = (torch.arange(N, device=dev) // 2048).to(torch.int32)
    adv = torch.ones(N // 2048, device=dev)
    p = rl.LossParams(agg=rl.AGG_SUM)
    dl = torch.empty_like(x)
    ws = torch.empty(rl.vocab_parallel_workspace_size(N, world), dtype=torch.uint8, device=dev)
    logp = torch.empty(N, device=dev)
    st = torch.zeros(12, dtype=torch.float64, device=dev)
    assert comm.enable_peer_exchange(N)
    call = lambda: rl.vocab_parallel_logprob(x, y, rank * W, V, comm, logp, ws, old_logp=old, token_seq=tseq,
                                             seq_adv=adv, params=p, dlogits_shard=dl, stats=st)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        call()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        gbs = 2 * N * W * 2 / (t.item() * 1e-3) / 1e9
        print(f"VP_WIDTH P={world} W={W} opts={opts}: {t.item():.3f} ms per call (max over ranks), "
              f"{gbs:.0f} GB/s per rank algorithmic", flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
