"""Back-to-back determinism of the vocab-parallel peer path across ranks (development):
    RL_LIB_PATH=... torchrun --nproc-per-node P tools/race_check.py [--vocab V] [KEY=VALUE ...]
Every rank holds its shard of the same seeded [4096, V] logits (V = 151936 by default); 8 calls with no collective in
between; prints, on rank 0, how many log-probs of calls 0..6 differ bitwise from call 7."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2605_15565_b200 as rl
    import synth
    from paper_2605_15565_b200.parallel import shard_vocab
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rl.load()
    for kv in [a for a in sys.argv[1:] if "=" in a]:
        k, v = kv.split("=")
        rl.dev_set_option(int(k), int(v))
    comm = rl.Comm.from_torch()
    V = int(sys.argv[sys.argv.index("--vocab") + 1]) if "--vocab" in sys.argv else 151936
    N = 4096
    xf = torch.empty((N, V), dtype=torch.bfloat16, device=dev)
    y = torch.empty(N, dtype=torch.int32, device=dev)
    synth.device_logits(xf, V, 0, 4, targets_out=y)
    sh = shard_vocab(V, world, rank)
    xs = xf[:, sh.offset:sh.offset + sh.size].contiguous()
    del xf
    old = torch.zeros(N, device=dev) - 3.0
    tseq = (torch.arange(N, device=dev) // 512).to(torch.int32)
    adv = torch.randn(N // 512, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
    p = rl.LossParams(agg=rl.AGG_SUM)
    dl = torch.empty_like(xs)
    ws = torch.empty(rl.vocab_parallel_workspace_size(N, world), dtype=torch.uint8, device=dev)
    logp = torch.empty(N, device=dev)
    assert comm.enable_peer_exchange(N)
    outs = []
    for _ in range(8):
        st = torch.zeros(12, dtype=torch.float64, device=dev)
        rl.vocab_parallel_logprob(xs, y, sh.offset, V, comm, logp, ws, old_logp=old, token_seq=tseq, seq_adv=adv,
                                  params=p, dlogits_shard=dl, stats=st)
        outs.append(logp.clone())
    torch.cuda.synchronize()
    bad = [int((o != outs[-1]).sum()) for o in outs[:-1]]
    if rank == 0:
        print(f"RACE_CHECK lib={os.path.basename(os.environ.get('RL_LIB_PATH', 'librlpolicy.so'))} "
              f"opts={[a for a in sys.argv[1:] if '=' in a]} differing rows per call: {bad}", flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
