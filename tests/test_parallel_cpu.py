"""Host logic of the N > 1 path on CPU (no GPU): sharding plans, and the shard algebra of the
two parallel modes exercised with a world_size-2 gloo process group — each rank computes its
shard with the oracle, the ranks exchange exactly what the GPU path exchanges (batch counts
before, loss statistics after; vocab-parallel (m, s, z_y) records), and the result must equal the
unsplit oracle."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2605_15565_b200.parallel import policy_group, shard_sequences, shard_vocab


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_sequences_partition(world):
    rng = np.random.default_rng(world)
    lens = rng.integers(0, 4000, size=64)
    cu = np.concatenate([[0], np.cumsum(lens)])
    shards = [shard_sequences(cu, world, r) for r in range(world)]
    assert shards[0].seq_begin == 0 and shards[-1].seq_end == 64
    for a, b in zip(shards, shards[1:]):
        assert a.seq_end == b.seq_begin and a.tok_end == b.tok_begin
    assert sum(s.n_tokens for s in shards) == cu[-1]
    ideal = cu[-1] / world
    assert max(abs(s.n_tokens - ideal) for s in shards) <= lens.max()


def test_shard_sequences_equal_lengths_even_split():
    cu = np.arange(65) * 32768          # config 2: 64 sequences x 32768
    for world in (2, 4, 8):
        assert {shard_sequences(cu, world, r).n_seq for r in range(world)} == {64 // world}


@pytest.mark.parametrize("V,world", [(151936, 8), (128256, 4), (1024, 3), (13, 2), (5, 8)])
def test_shard_vocab_partition(V, world):
    shards = [shard_vocab(V, world, r) for r in range(world)]
    assert shards[0].offset == 0
    assert sum(s.size for s in shards) == V
    for a, b in zip(shards, shards[1:]):
        assert a.offset + a.size == b.offset and (b.size == 0 or b.offset % 8 == 0)
    if V == 151936 and world == 8:
        assert all(s.size == 18992 for s in shards)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.cases import small_case
        case = small_case(n_prompts=3, group=4, seq_len=40, vocab=301, dtype="f32", seed=42,
                          staleness_max=3, max_staleness=2, big_delta_frac=0.2, sigma_delta=0.2)
        # ---------------- token parallel
        sh = shard_sequences(case["cu_seqlens"], world, rank)
        t0, t1, s0, s1 = sh.tok_begin, sh.tok_end, sh.seq_begin, sh.seq_end
        cu_local = np.asarray(case["cu_seqlens"][s0:s1 + 1]) - t0
        bk = oracle.seq_bookkeeping(cu_local, case["loss_mask"][t0:t1], case["targets"][t0:t1],
                                    case["vocab"], case["seq_version"][s0:s1], case["trainer_version"],
                                    case["max_staleness"])
        cnt = torch.tensor([float(bk["active_tokens"])], dtype=torch.float64)
        dist.all_reduce(cnt)                                   # rl_batch_counts all-reduce
        adv, _ = oracle.group_advantage(case["rewards"], case["cu_groups"])   # replicated
        p = oracle.LossParams(global_active_tokens=cnt.item(), trainer_version=case["trainer_version"],
                              max_staleness=case["max_staleness"])
        out = oracle.policy_loss_fwd_bwd(case["x64"][t0:t1], case["targets"][t0:t1],
                                         case["old_logp"][t0:t1], case["loss_mask"][t0:t1],
                                         bk["token_seq"] + s0, adv, case["seq_version"], None, p)
        st = torch.tensor([out["loss"], out["stats"]["active_tokens"], out["stats"]["ratio_sum"],
                           out["stats"]["clipped_low"], out["stats"]["clipped_high"]], dtype=torch.float64)
        dist.all_reduce(st)                                    # rl_loss_stats all-reduce
        # ---------------- vocab parallel
        vs = shard_vocab(case["vocab"], world, rank)
        m, s, xy, owned = oracle.vocab_shard_stats(case["x64"][:, vs.offset:vs.offset + vs.size],
                                                   case["targets"], vs.offset)
        rec = torch.tensor(np.stack([m, s, xy]), dtype=torch.float64)
        allrec = [torch.zeros_like(rec) for _ in range(world)]
        dist.all_gather(allrec, rec)                           # the vp record all-gather
        lse, zy = oracle.vocab_combine([r[0].numpy() for r in allrec], [r[1].numpy() for r in allrec],
                                       [r[2].numpy() for r in allrec])
        if rank == 0:
            q.put(dict(stats=st.numpy(), lse=lse, zy=zy))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_shard_algebra():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from tests.cases import oracle_chain, small_case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = small_case(n_prompts=3, group=4, seq_len=40, vocab=301, dtype="f32", seed=42,
                      staleness_max=3, max_staleness=2, big_delta_frac=0.2, sigma_delta=0.2)
    ref = oracle_chain(case, oracle.LossParams())["loss"]
    st = res["stats"]
    assert abs(st[0] - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
    assert st[1] == ref["stats"]["active_tokens"]
    assert abs(st[2] - ref["stats"]["ratio_sum"]) < 1e-9
    assert st[3] == ref["stats"]["clipped_low"] and st[4] == ref["stats"]["clipped_high"]
    logp, lse = oracle.token_logprob(case["x64"], case["targets"])
    ok = case["targets"] >= 0
    assert np.allclose(res["lse"], lse, atol=1e-12)
    assert np.allclose((res["zy"] - res["lse"])[ok], logp[ok], atol=1e-12)


@pytest.mark.parametrize("world,n_pol", [(8, 2), (4, 2), (5, 2), (3, 3), (1, 2), (7, 3)])
def test_policy_groups_partition(world, n_pol):
    gs = [policy_group(world, n_pol, r) for r in range(world)]
    for r, g in enumerate(gs):
        assert r in g.ranks and g.key == r - g.first
        same = lambda h: (h.policy, h.first, h.size) == (g.policy, g.first, g.size)  # noqa: E731
        assert all(same(policy_group(world, n_pol, q)) for q in g.ranks)
    if world >= n_pol:
        assert sorted({g.policy for g in gs}) == list(range(n_pol))
        sizes = [g.size for g in gs]
        assert max(sizes) - min(sizes) <= 1
    if (world, n_pol) == (8, 2):
        assert [g.policy for g in gs] == [0] * 4 + [1] * 4


MP_CASES = [dict(n_prompts=2, group=4, seq_len=48, vocab=96, dtype="f32", seed=51, staleness_max=8,
                 max_staleness=8, stale_outlier_frac=0.3, trainer_version=100, big_delta_frac=0.1),
            dict(n_prompts=2, group=4, seq_len=40, vocab=80, dtype="f32", seed=52, staleness_max=3,
                 max_staleness=8, trainer_version=57, sigma_delta=0.3)]


def _worker_policies(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.cases import small_case
        g = policy_group(world, 2, rank)
        # every rank creates every group (torch requires it); the rank uses its own (rl_comm_split)
        groups = [dist.new_group(list(policy_group(world, 2, r0).ranks))
                  for r0 in sorted({policy_group(world, 2, r).first for r in range(world)})]
        sub = groups[g.policy]
        case = small_case(**MP_CASES[g.policy])
        sh = shard_sequences(case["cu_seqlens"], g.size, g.key)
        t0, t1, s0, s1 = sh.tok_begin, sh.tok_end, sh.seq_begin, sh.seq_end
        bk = oracle.seq_bookkeeping(np.asarray(case["cu_seqlens"][s0:s1 + 1]) - t0, case["loss_mask"][t0:t1],
                                    case["targets"][t0:t1], case["vocab"], case["seq_version"][s0:s1],
                                    case["trainer_version"], case["max_staleness"])
        cnt = torch.tensor([float(bk["active_tokens"])], dtype=torch.float64)
        dist.all_reduce(cnt, group=sub)                        # within the policy's trainer group only
        adv, _ = oracle.group_advantage(case["rewards"], case["cu_groups"])
        p = oracle.LossParams(global_active_tokens=cnt.item(), trainer_version=case["trainer_version"],
                              max_staleness=case["max_staleness"])
        out = oracle.policy_loss_fwd_bwd(case["x64"][t0:t1], case["targets"][t0:t1], case["old_logp"][t0:t1],
                                         case["loss_mask"][t0:t1], bk["token_seq"] + s0, adv,
                                         case["seq_version"], None, p)
        st = torch.tensor([out["loss"], out["stats"]["active_tokens"], out["stats"]["stale_masked"],
                           out["stats"]["clipped_low"] + out["stats"]["clipped_high"]], dtype=torch.float64)
        dist.all_reduce(st, group=sub)
        if g.key == 0:
            q.put((g.policy, st.numpy()))
    finally:
        dist.destroy_process_group()


def test_world4_gloo_two_policy_groups():
    """configs[4] structure on CPU: 4 ranks split into 2 policy trainer groups of 2 (colour =
    policy); each group is token-parallel over its own policy's batch (different V, staleness
    mix) with its all-reduces inside the group; each group's result equals the unsplit oracle of
    that policy alone."""
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from tests.cases import oracle_chain, small_case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_policies, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for pol in (0, 1):
        case = small_case(**MP_CASES[pol])
        ref = oracle_chain(case, oracle.LossParams())["loss"]
        st = res[pol]
        assert abs(st[0] - ref["loss"]) <= 1e-12 * max(1.0, abs(ref["loss"]))
        assert st[1] == ref["stats"]["active_tokens"] and st[2] == ref["stats"]["stale_masked"]
        assert st[3] == ref["stats"]["clipped_low"] + ref["stats"]["clipped_high"]
    assert res[0][2] > 0     # policy A's staleness outliers are masked by max_staleness = 8
