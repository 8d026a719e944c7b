"""Multi-GPU parity check (one process per GPU; launched by tests/test_gpu_multi.py):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_check.py

token parallel: whole-sequence shards, rl_batch_counts all-reduced through rl_comm before the
loss, rl_loss_stats after it -> global loss / counts equal the unsplit oracle, each rank's dlogits
rows equal the oracle's rows.  vocab parallel: column shards, NCCL all-gather combine -> logp on
every rank and each dlogits shard equal the oracle (NCCL path and in-kernel peer path, at V = 5003
and at the production V = 151936 with back-to-back peer calls).  M2PO global mask.  comm split.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2605_15565_b200 as rl
    from paper_2605_15565_b200.parallel import shard_sequences, shard_vocab
    from tests.cases import oracle_chain, small_case

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rl.load()
    comm = rl.Comm.from_torch()

    def d(a):
        if a.dtype == np.uint16:
            return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(dev).view(torch.bfloat16)
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    case = small_case(n_prompts=4, group=4, seq_len=48, vocab=5003, ld=5008, dtype="bf16", seed=77,
                      staleness_max=3, max_staleness=2, big_delta_frac=0.1, sigma_delta=0.1)
    V, S = case["vocab"], len(case["rewards"])
    ref = oracle_chain(case, oracle.LossParams())
    out_ref = ref["loss"]
    fails = []

    # ------------------------------------------------------------------ token parallel
    sh = shard_sequences(case["cu_seqlens"], world, rank)
    t0, t1, s0, s1 = sh.tok_begin, sh.tok_end, sh.seq_begin, sh.seq_end
    n = t1 - t0
    adv = torch.empty(S, dtype=torch.float32, device=dev)
    rl.group_advantage(d(case["rewards"]), d(case["cu_groups"]), adv)       # replicated
    counts = torch.zeros(20, dtype=torch.float64, device=dev)
    tok = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    act = torch.empty(max(s1 - s0, 1), dtype=torch.int32, device=dev)
    cu_local = (np.asarray(case["cu_seqlens"][s0:s1 + 1]) - t0).astype(np.int32)
    rl.seq_bookkeeping(d(cu_local), d(case["targets"][t0:t1]), V, tok[:n], act[:s1 - s0],
                       loss_mask=d(case["loss_mask"][t0:t1]), seq_version=d(case["seq_version"][s0:s1]),
                       trainer_version=case["trainer_version"], max_staleness=case["max_staleness"],
                       counts_out=counts)
    comm.allreduce_f64(counts)                        # N_active over all ranks
    logits = d(case["logits"][t0:t1])
    dl = torch.empty_like(logits)
    stats = torch.zeros(12, dtype=torch.float64, device=dev)
    ws = torch.empty(rl.policy_loss_workspace_size(n, V), dtype=torch.uint8, device=dev)
    p = rl.LossParams(trainer_version=case["trainer_version"], max_staleness=case["max_staleness"],
                      active_tokens_dev=counts[0:1])
    rl.policy_loss_fwd_bwd(logits, d(case["targets"][t0:t1]), d(case["old_logp"][t0:t1]), tok[:n],
                           adv[s0:], p, dl, stats, ws, loss_mask=d(case["loss_mask"][t0:t1]),
                           seq_version=d(case["seq_version"][s0:s1]), vocab=V)
    comm.allreduce_f64(stats)
    torch.cuda.synchronize()
    st = stats.cpu().numpy()
    scale = max(abs(out_ref["loss"]), float(np.abs(out_ref["token_loss"]).sum()))
    if abs(st[0] - out_ref["loss"]) > 1e-4 * scale:
        fails.append(f"tp loss {st[0]} vs {out_ref['loss']}")
    if st[1] != out_ref["stats"]["active_tokens"] or counts[0].item() != ref["bk"]["active_tokens"]:
        fails.append(f"tp active {st[1]} vs {out_ref['stats']['active_tokens']}")
    g = oracle.decode_bf16(dl.view(torch.int16).cpu().numpy().view(np.uint16))[:, :V]
    s_ref = out_ref["scale"][t0:t1]
    for i in range(n):
        if s_ref[i] == 0:
            if np.any(g[i] != 0):
                fails.append(f"tp row {t0 + i} not zero")
        elif np.abs(g[i] - out_ref["dlogits"][t0 + i]).max() > 1e-2 * abs(s_ref[i]):
            fails.append(f"tp row {t0 + i} dlogits")

    # ------------------------------------------------------------------ vocab parallel
    # twice: the NCCL all-gather path, then the fused in-kernel peer-exchange path
    for mode in ("nccl", "peer"):
      if mode == "peer":
        if not comm.enable_peer_exchange(len(case["targets"])):
            fails.append("peer exchange unavailable")
            break
      vs = shard_vocab(V, world, rank)
      N = len(case["targets"])
      ld_s = max(8, (vs.size + 7) // 8 * 8)
      shard = np.zeros((N, ld_s), dtype=np.uint16)
      shard[:, :vs.size] = case["logits"][:, vs.offset:vs.offset + vs.size]
      shard_t = d(shard)
      dls = torch.empty_like(shard_t)
      logp = torch.empty(N, dtype=torch.float32, device=dev)
      lse = torch.empty(N, dtype=torch.float32, device=dev)
      stats_v = torch.zeros(12, dtype=torch.float64, device=dev)
      ws_v = torch.empty(rl.vocab_parallel_workspace_size(N, world), dtype=torch.uint8, device=dev)
      p_v = rl.LossParams(trainer_version=case["trainer_version"], max_staleness=case["max_staleness"],
                          global_active_tokens=float(ref["bk"]["active_tokens"]))
      tok_full = d(ref["bk"]["token_seq"])
      rl.vocab_parallel_logprob(shard_t, d(case["targets"]), vs.offset, V, comm, logp, ws_v, lse_out=lse,
                                vocab_shard=vs.size, old_logp=d(case["old_logp"]),
                                loss_mask=d(case["loss_mask"]), token_seq=tok_full, seq_adv=adv,
                                seq_version=d(case["seq_version"]), params=p_v, dlogits_shard=dls,
                                stats=stats_v)
      comm.allreduce_f64(stats_v)
      torch.cuda.synchronize()
      lp = logp.cpu().numpy()
      y = case["targets"]
      ok = (y >= 0) & (y < V)
      if np.abs(lp[ok] - out_ref["logp"][ok]).max() > 2e-3:
          fails.append(f"{mode} vp logp max err {np.abs(lp[ok] - out_ref['logp'][ok]).max()}")
      sv = stats_v.cpu().numpy()
      if abs(sv[0] - out_ref["loss"]) > 1e-4 * scale or sv[1] != out_ref["stats"]["active_tokens"]:
          fails.append(f"{mode} vp loss {sv[0]} vs {out_ref['loss']} active {sv[1]}")
      gv = oracle.decode_bf16(dls.view(torch.int16).cpu().numpy().view(np.uint16))[:, :vs.size]
      s_all = out_ref["scale"]
      for i in range(N):
          refrow = out_ref["dlogits"][i, vs.offset:vs.offset + vs.size]
          if s_all[i] == 0:
              if np.any(gv[i] != 0):
                  fails.append(f"{mode} vp row {i} not zero")
          elif vs.size and np.abs(gv[i] - refrow).max() > 1e-2 * abs(s_all[i]):
              fails.append(f"{mode} vp row {i} dlogits")

    # ------------------------------------------------------------------ vocab parallel, V = 151936
    # the production width: every rank holds its shard of the same seeded [N, 151936] logits (P = 2:
    # 75,968 columns -> vp_ring_kernel; P = 4 / 8: 37,984 / 18,992 -> vp_cache_kernel); three
    # back-to-back peer calls with NO collective in between (the exchange slots alternate by epoch
    # parity), each call's stats kept apart; the last call checked against the oracle on 256 rows
    import synth
    Vf, Nf = 151936, 4096
    xf = torch.empty((Nf, Vf), dtype=torch.bfloat16, device=dev)
    yf = torch.empty(Nf, dtype=torch.int32, device=dev)
    synth.device_logits(xf, Vf, 0, 4, targets_out=yf)
    vs = shard_vocab(Vf, world, rank)
    xs = xf[:, vs.offset:vs.offset + vs.size].contiguous()
    rows = np.sort(np.random.default_rng(5).choice(Nf, size=256, replace=False))
    bits_rows = xf[torch.from_numpy(rows).to(dev)].view(torch.int16).cpu().numpy().view(np.uint16)
    lp_ref_rows, _ = oracle.token_logprob(oracle.decode_bf16(bits_rows), yf.cpu().numpy()[rows])
    maskf = np.zeros(Nf, dtype=np.uint8)
    maskf[rows] = 1
    oldf = np.zeros(Nf, dtype=np.float32)
    oldf[rows] = (lp_ref_rows + np.random.default_rng(6).normal(size=256) * 0.05).astype(np.float32)
    tseqf = (np.arange(Nf) // 512).astype(np.int32)
    advf = np.random.default_rng(7).normal(size=Nf // 512).astype(np.float32)
    pf = rl.LossParams(agg=rl.AGG_SUM)
    dlf = torch.empty_like(xs)
    lpf = torch.empty(Nf, dtype=torch.float32, device=dev)
    wsf = torch.empty(rl.vocab_parallel_workspace_size(Nf, world), dtype=torch.uint8, device=dev)
    # RL_DEV_VP_KERNEL: the default kernel choice, then the register cache forced with each record
    # send mode (RL_DEV_VC_PUB: default, collector strong, last warp weak, collector weak)
    for vk, pub in ((0, 0), (2, 0), (2, 1), (2, 2), (2, 3)):
        rl.dev_set_option(rl.DEV_VC_PUB, pub)
        rl.dev_set_option(rl.DEV_VP_KERNEL, vk)
        if comm.enable_peer_exchange(Nf):
            st_calls = [torch.zeros(12, dtype=torch.float64, device=dev) for _ in range(3)]
            lp_calls = []
            for c in range(3):
                rl.vocab_parallel_logprob(xs, yf, vs.offset, Vf, comm, lpf, wsf, old_logp=d(oldf), loss_mask=d(maskf),
                                          token_seq=d(tseqf), seq_adv=d(advf), params=pf, dlogits_shard=dlf,
                                          stats=st_calls[c])
                lp_calls.append(lpf.clone())
            for c in range(3):
                comm.allreduce_f64(st_calls[c])
            torch.cuda.synchronize()
            sts = [c.cpu().numpy() for c in st_calls]
            if not (np.array_equal(sts[0], sts[1]) and np.array_equal(sts[1], sts[2])):
                lps = [c.cpu().numpy() for c in lp_calls]
                bad = [np.flatnonzero(lps[c] != lps[2]) for c in range(2)]
                fails.append(f"full-width vp (kernel option {vk}, pub {pub}): back-to-back calls differ: "
                             f"stats {sts[0][:4]} {sts[1][:4]} {sts[2][:4]}; logp rows differing from call 2: "
                             f"{[(len(b), b[:6].tolist(), lps[c][b[:3]].tolist(), lps[2][b[:3]].tolist()) for c, b in enumerate(bad)]}")
            yh = yf.cpu().numpy()
            outf = oracle.policy_loss_fwd_bwd(oracle.decode_bf16(bits_rows), yh[rows], oldf[rows], maskf[rows],
                                              tseqf[rows], advf.astype(np.float64), None, None,
                                              oracle.LossParams(agg=oracle.AGG_SUM))
            lpg = lpf.cpu().numpy()[rows]
            if np.abs(lpg - outf["logp"]).max() > 2e-3:
                fails.append(f"full-width vp ({vk}, {pub}) logp err {np.abs(lpg - outf['logp']).max()}")
            sc = max(abs(outf["loss"]), float(np.abs(outf["token_loss"]).sum()))
            if abs(sts[2][0] - outf["loss"]) > 1e-4 * sc or sts[2][1] != outf["stats"]["active_tokens"]:
                fails.append(f"full-width vp loss {sts[2][0]} vs {outf['loss']}")
            gs = oracle.decode_bf16(dlf[torch.from_numpy(rows).to(dev)].view(torch.int16).cpu().numpy().view(np.uint16))
            for k, i in enumerate(rows):
                refrow = outf["dlogits"][k, vs.offset:vs.offset + vs.size]
                s_k = outf["scale"][k]
                if s_k == 0:
                    if np.any(gs[k] != 0):
                        fails.append(f"full-width vp row {i} not zero")
                elif np.abs(gs[k] - refrow).max() > 1e-2 * abs(s_k):
                    fails.append(f"full-width vp row {i} dlogits err {np.abs(gs[k] - refrow).max() / abs(s_k)}")
        else:
            fails.append("full-width vp: peer exchange unavailable")
    rl.dev_set_option(rl.DEV_VP_KERNEL, 0)
    rl.dev_set_option(rl.DEV_VC_PUB, 0)
    del xf, xs, dlf

    # ------------------------------------------------------------------ M2PO global selection
    # every rank passes its own n tokens; the mask must equal the oracle's over the concatenation
    n_m = 5003
    rngs = [np.random.default_rng(900 + q) for q in range(world)]
    lps, olds, vals = [], [], []
    for q in range(world):
        lp_q = (rngs[q].normal(size=n_m) * 3 - 5).astype(np.float32)
        dr = np.round(rngs[q].normal(size=n_m) * rngs[q].choice([0.02, 0.3], size=n_m) * 64) / 64
        lps.append(lp_q)
        olds.append((lp_q - dr).astype(np.float32))
        vals.append((rngs[q].random(n_m) < 0.9).astype(np.uint8))
    mask_ref, k_ref, _, _ = oracle.m2po_mask(np.concatenate(lps), np.concatenate(olds), np.concatenate(vals), 0.01)
    mk = torch.empty(n_m, dtype=torch.uint8, device=dev)
    mst = torch.zeros(5, dtype=torch.float64, device=dev)
    mws = torch.empty(rl.m2po_workspace_size(n_m, world), dtype=torch.uint8, device=dev)
    rl.m2po_mask(d(lps[rank]), d(olds[rank]), mk, mst, mws, tau=0.01, valid=d(vals[rank]), comm=comm)
    torch.cuda.synchronize()
    if not np.array_equal(mk.cpu().numpy(), mask_ref[rank * n_m:(rank + 1) * n_m]) or mst[1].item() != k_ref:
        fails.append(f"m2po global mask (k {mst[1].item()} vs {k_ref})")

    # ------------------------------------------------------------------ comm split
    sub = comm.split(rank % 2, rank)
    one = torch.ones(1, dtype=torch.float64, device=dev)
    sub.allreduce_f64(one)
    torch.cuda.synchronize()
    if one.item() != sub.nranks or sub.nranks != len(range(rank % 2, world, 2)):
        fails.append(f"split group size {one.item()} vs {sub.nranks}")
    sub.destroy()

    flag = torch.tensor([len(fails)], dtype=torch.int32, device=dev)
    dist.all_reduce(flag)
    for f in fails[:10]:
        print(f"[rank {rank}] FAIL {f}", flush=True)
    comm.destroy()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_OK" if flag.item() == 0 else "MGPU_FAIL", flush=True)
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
