#!/usr/bin/env python
"""Benchmark of the policy-loss hot path (BASELINE.json metric:
"policy-loss fwd+bwd tokens/s @V=151936; % of HBM roofline; 1/2/4/8 GPUs").

One step = one pass of the whole hot path over one synthetic batch of BASELINE.json
configs[1] ("single-policy GRPO batch: 32 prompts x 8 responses x 2048 tokens, vocab 151936,
bf16 logits"), processed as the paper's 4 PPO mini-batches of 131,072 tokens:
  4 x rl_seq_bookkeeping  ->  rl_group_advantage (group + batch normalisation)
  ->  4 x rl_policy_loss_fwd_bwd (fused log-softmax / gather / ratio / clip / dlogits).
With N GPUs (torchrun) every rank processes its own batch of that shape (weak scaling, data
parallel): per mini-batch the active-token counts are all-reduced before the loss (so the
token-mean uses the global N_active) and the loss statistics after it, with the library's
NCCL communicator.

Inputs are resident in HBM before timing: a pool of 2 distinct mini-batch logits buffers
(39.8 GB each, far larger than the 126 MB L2, so no L2 flush is needed) and one dlogits
buffer; mini-batch j of a step reads pool buffer j % 2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--kernel two_pass]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "policy-loss fwd+bwd tokens/s @V=151936; % of HBM roofline; 1/2/4/8 GPUs"
WORKLOAD = "single-policy GRPO batch (BASELINE.json configs[1]): 32 prompts x 8 responses x 2048 tokens, V=151936, bf16 logits"
N_MINIBATCH = 4          # PAPER.md:574 "4 PPO mini-batches per iteration"
SIDE_BYTES = 17          # target 4 + old_logp 4 + mask 1 + logp out 4 + token_seq 4
OBJECTIVE = "clip"       # --objective
KERNEL = "sv"            # --kernel
SKIP_MASKED = False      # --skip-masked


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="sv", choices=["sv", "two_pass"],
                    help="rl_policy_loss_fwd_bwd kernel (two_pass: the development A/B option)")
    ap.add_argument("--vp-path", default="peer", choices=["peer", "nccl"],
                    help="vocabpar: in-kernel NVLink peer exchange (default) or the NCCL all-gather path")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="tiny: launch the chain directly, no CUDA graph")
    ap.add_argument("--skip-masked", action="store_true",
                    help="RL_F_SKIP_MASKED_READS: masked rows are not read (write-only zeros; logp 0 there)")
    ap.add_argument("--minibatch-tokens", type=int, default=131072)
    ap.add_argument("--vp-kernel", default="auto", choices=["auto", "cache", "ring"],
                    help="vocabpar peer path: the library's choice (auto), the register-cache kernel whenever the "
                         "shard fits it, or the L2 ring")
    ap.add_argument("--dev-opt", action="append", default=[], metavar="KEY=VALUE",
                    help="development option of the library (include/rl_policy_dev.h), repeatable; for A/B runs")
    ap.add_argument("--vc-rows", type=int, default=-1,
                    help="vocabpar peer path, vp_cache_kernel: rows parked in shared memory (-1 = default)")
    ap.add_argument("--vp-width-of", type=int, default=0,
                    help="vocabpar on ONE GPU: one rank's share of a P-way split (a [65536, V/P] shard as its own "
                         "vocabulary, exchange with itself) — the per-rank work of configs[3] at P")
    ap.add_argument("--resident", action="store_true",
                    help="single: the rank's whole 524,288-token batch as ONE resident in-place call (159 GB)")
    ap.add_argument("--objective", default="clip", choices=["clip", "full", "m2po"],
                    help="clip: the north_star's clipped surrogate (default); full: + decoupled proximal "
                         "ratio, k3 KL penalty (beta 1e-3, PAPER.md:572) and entropy (NEXT 2); m2po: "
                         "rl_token_logprob -> rl_m2po_mask (tau 0.01, PAPER.md:572) -> unclipped loss (NEXT 1)")
    ap.add_argument("--config", default="single", choices=["single", "tiny", "long", "vocabpar", "multi", "lmhead"],
                    help="BASELINE.json config (single = the headline metric's workload, the default)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(kernel)
    return None if e is None else e.get("dram_bytes_per_launch")


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- oracle legs
def _oracle_rows(args):
    import numpy as np
    import oracle
    x16, y, old, adv, reps = args
    x64 = oracle.decode_bf16(x16)
    n = len(y)
    for _ in range(reps):
        oracle.policy_loss_fwd_bwd(x64, y, old, np.ones(n, dtype=np.uint8), np.zeros(n, dtype=np.int32),
                                   adv, None, None, oracle.LossParams(global_active_tokens=131072.0))
    return n * reps


def time_oracle(sample_rows_bits, targets, old, n_rows_total, workers):
    """Time the fp64 oracle (as it stands) on `n_rows_total` rows split over `workers`
    processes; returns (tokens/s, seconds)."""
    import multiprocessing as mp
    import numpy as np
    R = len(targets)
    per = max(1, n_rows_total // R)
    chunks = np.array_split(np.arange(R), workers)
    adv = np.array([0.5], dtype=np.float32)
    jobs = [(sample_rows_bits[c], targets[c], old[c], adv, per) for c in chunks if len(c)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(len(jobs)) as pool:
        pool.map(_oracle_rows, [(j[0][:1], j[1][:1], j[2][:1], adv, 1) for j in jobs])  # warm
        t0 = time.perf_counter()
        done = sum(pool.map(_oracle_rows, jobs))
        dt = time.perf_counter() - t0
    return done / dt, dt, done


def run_reference(args):
    """--impl reference: the oracle timed on the host cores on bounded samples of the same
    workload (this tier's reference arm)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    cfg = synth.get_config("single")
    R = 64
    x, y = synth.host_logits(cfg.vocab, np.arange(R), cfg.seed, "bf16")
    lp, _ = oracle.token_logprob(oracle.decode_bf16(x), y)
    old = (lp + np.random.default_rng(0).normal(size=R) * 0.02).astype(np.float32)
    workers = host_cores()
    rows_per_step = 16 * workers
    tok, secs = 0, 0.0
    for i in range(args.warmup + args.steps):
        rate, dt, done = time_oracle(x, y, old, rows_per_step, workers)
        if i >= args.warmup:
            tok += done
            secs += dt
    value = tok / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": f"{rows_per_step} token rows per step"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": workers, "kind": "oracle",
                         "sample": f"{rows_per_step} rows x V=151936 fwd+bwd per step, {workers} processes"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def make_pool(torch, synth, dev, n_buf, MB, V, seed, rank, cfg_seed_row0=0):
    """`n_buf` distinct resident [MB, V] bf16 logits buffers (device generator), their sampled
    targets and behaviour log-probs (torch fp32 log-softmax + seeded drift: input synthesis)."""
    pool, pool_y, pool_old = [], [], []
    for b in range(n_buf):
        x = torch.empty((MB, V), dtype=torch.bfloat16, device=dev)
        y = torch.empty(MB, dtype=torch.int32, device=dev)
        synth.device_logits(x, V, row0=(rank * n_buf + b + cfg_seed_row0) * MB, seed=seed, targets_out=y)
        old = torch.empty(MB, dtype=torch.float32, device=dev)
        g = torch.Generator(device=dev)
        g.manual_seed(77 + b + 10 * rank)
        for c0 in range(0, MB, 4096):
            blk = x[c0:c0 + 4096].float()
            lp = blk.gather(1, y[c0:c0 + 4096, None].long())[:, 0] - torch.logsumexp(blk, dim=1)
            old[c0:c0 + 4096] = lp + 0.02 * torch.randn(lp.shape, generator=g, device=dev)
            del blk
        pool.append(x)
        pool_y.append(y)
        pool_old.append(old)
    return pool, pool_y, pool_old


class TokenParallelWorkload:
    """Configs single / long / multi: whole sequences per rank, each rank's share processed as
    mini-batch calls of MB tokens streaming through a pool of 2 resident logits buffers.
    One step: bookkeeping of every call (counts all-reduced over the policy's ranks) ->
    advantages (group + batch normalisation) -> fused loss of every call (stats all-reduced)."""

    def __init__(self, rl, torch, np, synth, dev, comm, cfg, seqs, MB, n_calls, rank, max_staleness,
                 n_pool=2, dlogits_buf=None, in_place=False):
        self.rl, self.torch, self.comm = rl, torch, comm
        V, T = cfg.vocab, cfg.seq_len
        self.V, self.MB, self.n_calls = V, MB, n_calls
        lay = synth.seq_layout(cfg)
        s0, s1 = seqs                     # this rank's sequences [s0, s1) of the policy batch
        self.trainer_version, self.max_staleness = lay["trainer_version"], max_staleness
        self.pool, self.pool_y, self.pool_old = make_pool(torch, synth, dev, n_pool, MB, V, cfg.seed, rank)
        self.full = OBJECTIVE == "full"
        if self.full:  # reference / proximal log-probs: behaviour log-probs + seeded drift (input synthesis)
            g = torch.Generator(device=dev)
            g.manual_seed(991 + rank)
            self.pool_ref = [o + 0.2 * torch.randn(o.shape, generator=g, device=dev) for o in self.pool_old]
            self.pool_prox = [o + 0.02 * torch.randn(o.shape, generator=g, device=dev) for o in self.pool_old]
        if in_place:                 # dlogits overwrite the (single) resident logits buffer
            self.dlogits = self.pool[0]
        elif dlogits_buf is not None:  # shared [MB * V_max] bf16 buffer viewed as [MB, V]
            self.dlogits = dlogits_buf[:MB * V].view(MB, V)
        else:
            self.dlogits = torch.empty((MB, V), dtype=torch.bfloat16, device=dev)
        S_all = cfg.n_seq
        G = S_all // cfg.group
        self.rewards = torch.from_numpy(lay["rewards"]).to(dev)
        self.cu_groups = torch.from_numpy(lay["cu_groups"]).to(dev)
        self.seq_version = torch.from_numpy(lay["seq_version"]).to(dev)
        self.adv = torch.empty(S_all, dtype=torch.float32, device=dev)
        self.zero_var = torch.empty(G, dtype=torch.uint8, device=dev)
        self.seq_active = torch.zeros(S_all, dtype=torch.int32, device=dev)
        self.ws_adv = torch.empty(rl.group_advantage_workspace_size(S_all), dtype=torch.uint8, device=dev)
        # the rank's step batch: n_calls mini-batches of MB tokens (MB/T sequences each) starting at
        # sequence s0; ONE bookkeeping call covers all of them (token_seq relative to s0), so the
        # batch counts come out of the library whole (no host-side sum) and are all-reduced
        tok0 = s0 * T
        self.s0, self.n_seq_rank = s0, n_calls * MB // T
        mask_all = lay["loss_mask"]
        self.cu_rank = torch.from_numpy((np.arange(self.n_seq_rank + 1) * T).astype(np.int32)).to(dev)
        self.mask_rank = torch.from_numpy(np.ascontiguousarray(mask_all[tok0:tok0 + n_calls * MB])).to(dev)
        self.y_rank = torch.cat([self.pool_y[c % len(self.pool_y)] for c in range(n_calls)])
        self.tok_rank = torch.empty(n_calls * MB, dtype=torch.int32, device=dev)
        self.calls = [dict(stats=torch.zeros(12, dtype=torch.float64, device=dev),
                           logp=torch.empty(MB, dtype=torch.float32, device=dev)) for _ in range(n_calls)]
        self.total_counts = torch.zeros(20, dtype=torch.float64, device=dev)
        self.ws = torch.empty(rl.policy_loss_workspace_size(MB, V), dtype=torch.uint8, device=dev)
        self.tokens_per_step = n_calls * MB
        self.bytes_per_token = 2 * V * 2 + SIDE_BYTES + (8 if self.full else 0)  # + ref, prox reads
        self.m2po = OBJECTIVE == "m2po"
        if self.m2po:  # the roofline stays the loss call's (the log-prob pass is a separate kernel)
            self.m2_logp = torch.empty(MB, dtype=torch.float32, device=dev)
            self.m2_mask = torch.empty(MB, dtype=torch.uint8, device=dev)
            self.m2_stats = torch.zeros(5, dtype=torch.float64, device=dev)
            self.m2_ws = torch.empty(rl.m2po_workspace_size(MB, comm.nranks if comm is not None else 1),
                                     dtype=torch.uint8, device=dev)
        self.launches = 0
        self.ev = []

    def step(self, record):
        rl, torch = self.rl, self.torch
        P = len(self.pool)
        s0, ns, MB = self.s0, self.n_seq_rank, self.MB
        rl.seq_bookkeeping(self.cu_rank, self.y_rank, self.V, self.tok_rank, self.seq_active[s0:s0 + ns],
                           loss_mask=self.mask_rank, seq_version=self.seq_version[s0:s0 + ns],
                           trainer_version=self.trainer_version, max_staleness=self.max_staleness,
                           counts_out=self.total_counts)
        self.launches += 2
        # N_active of the whole (policy) batch: the rank's counts, all-reduced over the policy's ranks
        if self.comm is not None:
            self.comm.allreduce_f64(self.total_counts)
        rl.group_advantage(self.rewards, self.cu_groups, self.adv, self.zero_var, batch_norm=True,
                           seq_weight=self.seq_active, workspace=self.ws_adv)
        self.launches += 1
        stream = torch.cuda.current_stream()
        for c, cl in enumerate(self.calls):
            p = rl.LossParams(trainer_version=self.trainer_version, max_staleness=self.max_staleness,
                              active_tokens_dev=self.total_counts[0:1])
            mask = self.mask_rank[c * MB:(c + 1) * MB]
            if self.m2po:  # NEXT 1: fresh log-probs -> global second-moment mask -> unclipped loss
                rl.token_logprob(self.pool[c % P], self.pool_y[c % P], self.m2_logp)
                rl.m2po_mask(self.m2_logp, self.pool_old[c % P], self.m2_mask, self.m2_stats, self.m2_ws,
                             tau=0.01, valid=mask, comm=self.comm)
                mask = self.m2_mask
                p.clip_eps_low = p.clip_eps_high = 1e30
                p.active_tokens_dev = self.m2_stats[4:5]
                self.launches += 9
            if self.full:
                p.kl_coef, p.ref_logp, p.prox_logp = 1e-3, self.pool_ref[c % P], self.pool_prox[c % P]
                p.flags |= rl.F_ENTROPY
            if SKIP_MASKED:
                p.flags |= rl.F_SKIP_MASKED_READS
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            rl.policy_loss_fwd_bwd(self.pool[c % P], self.pool_y[c % P], self.pool_old[c % P],
                                   self.tok_rank[c * MB:(c + 1) * MB], self.adv[s0:s0 + ns], p, self.dlogits,
                                   cl["stats"], self.ws, loss_mask=mask, seq_version=self.seq_version[s0:s0 + ns],
                                   logp_out=cl["logp"])
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                self.ev.append((e0, e1))
            # sv: loss_sv_kernel + two-pass fixup + stats reduce; cluster / two_pass: kernel + reduce
            self.launches += 3 if KERNEL == "sv" else 2
            if self.comm is not None:
                self.comm.allreduce_f64(cl["stats"])

    def kernel_ms(self):
        ms = [a.elapsed_time(b) for a, b in self.ev]
        return sum(ms) / len(ms)


class VocabParallelWorkload:
    """Config vocabpar (BASELINE.json configs[3]): 65,536 tokens, V split over the ranks; one step
    = rl_vocab_parallel_logprob with the fused loss on the rank's column shard."""

    def __init__(self, rl, torch, np, synth, dev, comm, cfg, world, rank, width_of=0):
        from paper_2605_15565_b200.parallel import shard_vocab
        self.rl, self.torch, self.comm = rl, torch, comm
        V = cfg.vocab
        N = cfg.n_tokens
        if width_of > 1 and world == 1:   # one rank's shard width as the whole (own) vocabulary
            V = shard_vocab(V, width_of, 0).size
        sh = shard_vocab(V, world, rank)
        self.off, self.Vr = sh.offset, sh.size
        ld = max(8, (self.Vr + 7) // 8 * 8)
        full = torch.empty((4096, V), dtype=torch.bfloat16, device=dev)
        self.shard = torch.empty((N, ld), dtype=torch.bfloat16, device=dev)
        self.y = torch.empty(N, dtype=torch.int32, device=dev)
        self.old = torch.empty(N, dtype=torch.float32, device=dev)
        g = torch.Generator(device=dev)
        g.manual_seed(99)
        for c0 in range(0, N, 4096):   # identical full rows on every rank, each keeps its columns
            synth.device_logits(full, V, row0=c0, seed=cfg.seed, targets_out=self.y[c0:c0 + 4096])
            self.shard[c0:c0 + 4096, :self.Vr].copy_(full[:, self.off:self.off + self.Vr])
            blk = full.float()
            lp = blk.gather(1, self.y[c0:c0 + 4096, None].long())[:, 0] - torch.logsumexp(blk, dim=1)
            self.old[c0:c0 + 4096] = lp + 0.02 * torch.randn(lp.shape, generator=g, device=dev)
        del full, blk
        lay = synth.seq_layout(cfg)
        self.lay = lay
        self.dl = torch.empty_like(self.shard)
        self.logp = torch.empty(N, dtype=torch.float32, device=dev)
        self.mask = torch.from_numpy(lay["loss_mask"]).to(dev)
        self.cu = torch.from_numpy(lay["cu_seqlens"]).to(dev)
        self.tok = torch.empty(N, dtype=torch.int32, device=dev)
        S = cfg.n_seq
        self.seq_active = torch.empty(S, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(20, dtype=torch.float64, device=dev)
        self.rewards = torch.from_numpy(lay["rewards"]).to(dev)
        self.cu_groups = torch.from_numpy(lay["cu_groups"]).to(dev)
        self.seq_version = torch.from_numpy(lay["seq_version"]).to(dev)
        self.adv = torch.empty(S, dtype=torch.float32, device=dev)
        self.ws_adv = torch.empty(rl.group_advantage_workspace_size(S), dtype=torch.uint8, device=dev)
        self.stats = torch.zeros(12, dtype=torch.float64, device=dev)
        self.ws = torch.empty(rl.vocab_parallel_workspace_size(N, world), dtype=torch.uint8, device=dev)
        self.V, self.N = V, N
        self.tokens_per_step = N
        # algorithmic bytes per token on this rank: read + write of the shard row + side data
        self.bytes_per_token = 2 * self.Vr * 2 + SIDE_BYTES
        self.launches = 0
        self.ev = []

    def step(self, record):
        rl, torch = self.rl, self.torch
        rl.seq_bookkeeping(self.cu, self.y, self.V, self.tok, self.seq_active, loss_mask=self.mask,
                           seq_version=self.seq_version, trainer_version=self.lay["trainer_version"],
                           counts_out=self.counts)
        rl.group_advantage(self.rewards, self.cu_groups, self.adv, batch_norm=True, seq_weight=self.seq_active,
                           workspace=self.ws_adv)
        p = rl.LossParams(trainer_version=self.lay["trainer_version"], active_tokens_dev=self.counts[0:1])
        stream = torch.cuda.current_stream()
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        rl.vocab_parallel_logprob(self.shard, self.y, self.off, self.V, self.comm, self.logp, self.ws,
                                  vocab_shard=self.Vr, old_logp=self.old, loss_mask=self.mask, token_seq=self.tok,
                                  seq_adv=self.adv, seq_version=self.seq_version, params=p,
                                  dlogits_shard=self.dl, stats=self.stats)
        if record:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            self.ev.append((e0, e1))
        self.comm.allreduce_f64(self.stats)
        self.launches += 2 + 1 + 3

    def kernel_ms(self):
        ms = [a.elapsed_time(b) for a, b in self.ev]
        return sum(ms) / len(ms)


CONFIG_WORKLOADS = {
    "single": "single-policy GRPO batch (BASELINE.json configs[1]): 32 prompts x 8 responses x 2048 tokens, "
              "V=151936, bf16 logits, per GPU",
    "long": "long agentic trajectories (BASELINE.json configs[2]): 8 prompts x 8 responses x 32768 tokens, "
            "multi-turn with tool output masked, V=151936, token-sharded over the GPUs",
    "vocabpar": "vocab-parallel (BASELINE.json configs[3]): 65,536 tokens, V=151936 split across the GPUs",
    "multi": "multi-policy step (BASELINE.json configs[4]): 2 policies (V 151936 / 128256), 128 x 8 x 4096 "
             "tokens, staleness <= 8, one GPU group per policy",
}


def main():
    global OBJECTIVE, KERNEL, SKIP_MASKED
    args = parse()
    OBJECTIVE, KERNEL, SKIP_MASKED = args.objective, args.kernel, args.skip_masked
    # the image sets NCCL_DEBUG=VERSION, whose only output is a banner NCCL prints on stdout: keep
    # stdout to the single JSON line (an explicit WARN / INFO setting is left alone)
    if os.environ.get("NCCL_DEBUG") == "VERSION":
        os.environ["NCCL_DEBUG"] = "NONE"
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "lmhead":
        return run_lmhead(args)
    if args.config == "tiny":
        return run_tiny(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_15565_b200 as rl
    import synth
    from paper_2605_15565_b200.parallel import policy_group, shard_sequences

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rl.load()
    if args.kernel == "two_pass":
        rl.dev_set_option(rl.DEV_LOSS_KERNEL, 1)
    if args.vp_path == "nccl":
        rl.dev_set_option(rl.DEV_VP_PATH, 1)
    if args.vp_kernel != "auto":
        rl.dev_set_option(rl.DEV_VP_KERNEL, 1 if args.vp_kernel == "ring" else 2)
    if args.vc_rows >= 0:
        rl.dev_set_option(rl.DEV_VC_ROWS, args.vc_rows + 1)
    for kv in args.dev_opt:
        k, v = kv.split("=")
        rl.dev_set_option(int(k), int(v))
    comm = None
    if world > 1 or args.config == "vocabpar":
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
            comm = rl.Comm.from_torch()
        else:
            comm = rl.Comm.local()
    MB = args.minibatch_tokens
    scaling = "weak"
    kern = args.kernel
    parallelism = f"dp{world} (token-parallel)"
    if args.config == "single":
        cfg = synth.get_config("single")
        cfg = synth.get_config("single", seed=cfg.seed + 1000 * rank)   # each rank its own batch (DP)
        n_calls = N_MINIBATCH
        S = n_calls * MB // cfg.seq_len
        if args.resident:   # C2 also timed as one resident batch with in-place dlogits
            need = n_calls * MB * cfg.vocab * 2 + (4 << 30)
            free = torch.cuda.mem_get_info(dev)[0]
            if free < need:
                raise SystemExit(f"--resident needs {need / 2**30:.1f} GiB free, {free / 2**30:.1f} GiB available")
            MB, n_calls = n_calls * MB, 1
            wl = TokenParallelWorkload(rl, torch, np, synth, dev, comm, cfg, (0, S), MB, 1, rank, -1, n_pool=1,
                                       in_place=True)
        else:
            wl = TokenParallelWorkload(rl, torch, np, synth, dev, comm, cfg, (0, S), MB, n_calls, rank, -1)
        # each rank's own batch: restrict advantages to its sequences
        wl.rewards, wl.cu_groups = wl.rewards[:S], wl.cu_groups[:S // cfg.group + 1]
        wl.adv, wl.zero_var = wl.adv[:S], wl.zero_var[:S // cfg.group]
        wl.seq_active = wl.seq_active[:S]
        kname = f"rl_policy_loss_fwd_bwd ({kern})"
    elif args.config == "long":
        cfg = synth.get_config("long")
        sh = shard_sequences(np.arange(cfg.n_seq + 1) * cfg.seq_len, world, rank)
        n_calls = sh.n_tokens // MB
        wl = TokenParallelWorkload(rl, torch, np, synth, dev, comm, cfg, (sh.seq_begin, sh.seq_end), MB, n_calls,
                                   rank, -1)
        scaling = "strong"
        kname = f"rl_policy_loss_fwd_bwd ({kern})"
    elif args.config == "multi":
        grp = policy_group(world, 2, rank)          # contiguous trainer group per policy (4 + 4 of 8)
        policy = grp.policy
        cfgs = [synth.get_config("multi_a"), synth.get_config("multi_b")]
        sub = comm.split(policy, grp.key) if comm is not None else None
        ranks_pp = grp.size
        prank = grp.key
        cfg = cfgs[policy]
        sh = shard_sequences(np.arange(cfg.n_seq + 1) * cfg.seq_len, ranks_pp, prank)
        n_calls = sh.n_tokens // MB
        if world == 1:   # one GPU: both policies' batches in turn (one logits buffer each, shared dlogits)
            shared = torch.empty(MB * max(c.vocab for c in cfgs), dtype=torch.bfloat16, device=dev)
            wl = [TokenParallelWorkload(rl, torch, np, synth, dev, None, c, (0, c.n_seq), MB,
                                        c.n_tokens // MB, rank, c.max_staleness, n_pool=1, dlogits_buf=shared)
                  for c in cfgs]
        else:
            wl = TokenParallelWorkload(rl, torch, np, synth, dev, sub, cfg, (sh.seq_begin, sh.seq_end), MB,
                                       n_calls, prank, cfg.max_staleness)
        scaling = "strong"
        parallelism = f"2 policy groups x {ranks_pp} GPU (token-parallel within a group)"
        kname = f"rl_policy_loss_fwd_bwd ({kern})"
    elif args.config == "vocabpar":
        cfg = synth.get_config("vocabpar")
        wl = VocabParallelWorkload(rl, torch, np, synth, dev, comm, cfg, world, rank, args.vp_width_of)
        fused_vp = args.vp_path == "peer" and comm.enable_peer_exchange(cfg.n_tokens)
        scaling = "strong"
        parallelism = (f"vocab-parallel over {world} GPU: " + (
            "one fused kernel per rank, per-row (max, sum-exp, target logit) exchanged by NVLink peer stores"
            if fused_vp else "vp_stats + NCCL all-gather + vp_finish"))
        if args.vp_width_of > 1 and world == 1:
            parallelism = (f"ONE GPU doing one rank's share of a {args.vp_width_of}-way vocabulary split "
                           f"({wl.Vr} columns as its own vocabulary, exchange with itself)")
        fits = wl.Vr % 8 == 0 and wl.Vr // 8 <= 11 * 448
        # the library's choice (vocab_parallel.cu): the register cache on one rank when the shard fits
        # it, the ring on more; --vp-kernel cache / ring force one
        use_cache = fits and (args.vp_kernel == "cache" or (args.vp_kernel == "auto" and world == 1))
        vk = "vp_cache_kernel" if use_cache else "vp_ring_kernel"
        kname = "rl_vocab_parallel_logprob (" + (f"{vk}, in-kernel peer exchange" if fused_vp
                                                 else "vp_stats + NCCL all-gather + vp_finish") + ")"
    else:
        raise SystemExit(f"unknown config {args.config}")
    wls = wl if isinstance(wl, list) else [wl]
    torch.cuda.synchronize()

    def step(record):
        for w in wls:
            w.step(record)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for w in wls:
        w.launches = 0
        w.ev = []
    stream = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    torch.cuda.nvtx.range_push("timed")   # ncu --nvtx --nvtx-include timed/: the timed launches only
    for i in range(args.steps):
        step(True)
        evs[i + 1].record(stream)    # step boundaries: the per-step distribution (no extra sync)
    torch.cuda.nvtx.range_pop()
    t0, t1 = evs[0], evs[-1]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t0.elapsed_time(t1)
    gpu_launches = sum(w.launches for w in wls)
    if world > 1:
        tt = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = tt.item()
    tokens_rank = sum(w.tokens_per_step for w in wls)
    tok_all = torch.tensor([float(tokens_rank)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tok_all)
    tokens_step = tok_all.item() if args.config != "vocabpar" else float(wls[0].tokens_per_step)
    value = tokens_step * args.steps / (elapsed_ms / 1e3)
    # per-step distribution (this rank's step boundaries; the headline is the max-over-ranks total)
    step_ms = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])
    step_stats = {"p10": float(np.percentile(step_ms, 10)), "p50": float(np.median(step_ms)),
                  "p90": float(np.percentile(step_ms, 90)), "min": float(step_ms.min()), "max": float(step_ms.max())}
    # loss-active tokens of the step (valid tokens: masks, ignored targets and staleness applied)
    # (total_counts is already summed over the workload's comm group: each rank adds its share)
    active_step = sum(float(w.total_counts[0].item()) / (w.comm.nranks if w.comm is not None else 1)
                      for w in wls if hasattr(w, "total_counts"))
    if world > 1:
        at = torch.tensor([active_step], dtype=torch.float64, device=dev)
        dist.all_reduce(at)
        active_step = at.item()
    active_rate = active_step * args.steps / (elapsed_ms / 1e3) if active_step else None

    # roofline of the dominant kernel: algorithmic bytes per launch / its average launch duration
    w0 = wls[0]
    launch_tokens = w0.MB if hasattr(w0, "MB") else w0.N
    if SKIP_MASKED and hasattr(w0, "total_counts"):   # masked rows are written, not read
        frac = float(w0.total_counts[0].item()) / max(1.0, float(w0.tokens_per_step) *
                                                      (w0.comm.nranks if w0.comm is not None else 1))
        w0.bytes_per_token = w0.V * 2 * (1 + frac) + SIDE_BYTES
    alg_bytes = launch_tokens * w0.bytes_per_token
    avg_ms = w0.kernel_ms()
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    peak, peak_src = measured_peak_hbm()
    traffic = ncu_traffic(kern) if args.config in ("single", "long", "multi") else None

    e2e, cpu = None, None
    if args.config == "single":
        if not args.no_e2e:
            S_mb = MB // 2048
            e2e = measure_e2e(rl, torch, dev, w0.pool[0], w0.pool_y[0], w0.pool_old[0], w0.tok_rank[:MB],
                              w0.adv[:S_mb], w0.mask_rank[:MB], w0.seq_version[:S_mb],
                              {"trainer_version": w0.trainer_version}, w0.V, args)
            if world > 1:
                tt = torch.tensor([e2e["seconds"]], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                e2e["value"] = world * e2e["tokens"] / tt.item()
            e2e = {k: e2e[k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step", "sample")}
        if rank == 0 and world == 1 and not args.no_cpu:
            x16 = w0.pool[0][:64].view(torch.int16).cpu().numpy().view(np.uint16)
            yy = w0.pool_y[0][:64].cpu().numpy()
            oo = w0.pool_old[0][:64].cpu().numpy()
            workers = host_cores()
            rate, secs, done = time_oracle(x16, yy, oo, 8192, workers)
            cpu = {"value": rate, "unit": "tokens/s", "cores": workers, "kind": "oracle",
                   "sample": f"{done} token rows (64 distinct rows of mini-batch 0) x V=151936 fwd+bwd "
                             f"in {secs:.1f} s wall over {workers} processes"}

    if rank == 0:
        workload = CONFIG_WORKLOADS[args.config]
        if args.resident:
            workload = "one resident in-place call over the whole 524,288-token batch: " + workload
        elif MB != 131072:
            workload = f"PROFILING ONLY ({MB}-token calls): " + workload
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload, "config": args.config, "tokens_per_step": tokens_step,
                       "tokens_per_rank_per_step": tokens_rank, "call_tokens": launch_tokens,
                       "vocab": w0.V, "parallelism": parallelism, "loss_kernel": kern,
                       "l2": "no flush: every loss call streams a distinct >= 2.5 GB logits buffer >> 126 MB L2",
                       "agg": "token_mean", "batch_norm": True, "skip_masked_reads": SKIP_MASKED,
                       "objective": {"full": "clipped decoupled surrogate + k3 KL (beta 1e-3) + entropy",
                                     "m2po": "M2PO: log-prob pass + second-moment mask (tau 0.01) + unclipped loss",
                                     }.get(args.objective, "clipped surrogate")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": kname, "algorithmic_bytes_per_launch": alg_bytes,
                         "bytes_per_token": w0.bytes_per_token, "avg_launch_ms": avg_ms,
                         "frac_of_8TBs": achieved / 8000.0},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk,
            "step_ms": step_stats, "active_tokens_per_s": active_rate,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()


def run_tiny(args):
    """configs[0] (BASELINE.json "tiny: 2 prompts x 4 responses x 64 tokens, vocab 1024, fp32 logits, 1
    GPU (CPU oracle in seconds)"): a step is the whole chain on the device — bookkeeping, group
    advantages (+ batch normalisation), the fused loss — over the 512 tokens; the full fp64 oracle
    chain on the same inputs is timed beside it on the host.  Launch-bound by construction (a 4 MB
    batch): reported for the record, not a roofline claim.  Replicas only (N > 1: rank 0 reports)."""
    import numpy as np
    import torch
    import paper_2605_15565_b200 as rl
    import synth
    local = int(os.environ.get("LOCAL_RANK", "0"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rl.load()
    cfg = synth.get_config("tiny")
    lay = synth.seq_layout(cfg)
    N, V, S, G = cfg.n_tokens, cfg.vocab, cfg.n_seq, cfg.n_seq // cfg.group
    x_h, y_h = synth.host_logits(cfg, np.arange(N), cfg.seed, "f32")
    y_h = np.where(lay["ignore"] != 0, -100, y_h).astype(np.int32)
    x = torch.from_numpy(x_h).to(dev)
    y = torch.from_numpy(y_h).to(dev)
    # behaviour log-probs: a setup rl_token_logprob pass + synth's seeded drift (untimed input synthesis)
    lp0 = torch.empty(N, device=dev)
    rl.token_logprob(x, y, lp0)
    tstale = (lay["trainer_version"] - lay["seq_version"])[np.repeat(np.arange(S), cfg.seq_len)]
    old_h = synth.perturb_old_logp(np.where(y_h >= 0, lp0.cpu().numpy(), 0.0), tstale, lay["big_delta"], cfg, cfg.seed)
    old = torch.from_numpy(old_h).to(dev)
    cu = torch.from_numpy(lay["cu_seqlens"].astype(np.int32)).to(dev)
    cug = torch.from_numpy(lay["cu_groups"].astype(np.int32)).to(dev)
    rew = torch.from_numpy(lay["rewards"].astype(np.float64)).to(dev)
    mask = torch.from_numpy(lay["loss_mask"]).to(dev)
    ver = torch.from_numpy(lay["seq_version"].astype(np.int32)).to(dev)
    tok = torch.empty(N, dtype=torch.int32, device=dev)
    act = torch.empty(S, dtype=torch.int32, device=dev)
    counts = torch.zeros(20, dtype=torch.float64, device=dev)
    adv = torch.empty(S, device=dev)
    zv = torch.empty(G, dtype=torch.uint8, device=dev)
    ws_a = torch.empty(rl.group_advantage_workspace_size(S), dtype=torch.uint8, device=dev)
    dl = torch.empty_like(x)
    stats = torch.zeros(12, dtype=torch.float64, device=dev)
    ws = torch.empty(rl.policy_loss_workspace_size(N, V, rl.F32), dtype=torch.uint8, device=dev)
    logp = torch.empty(N, device=dev)
    p = rl.LossParams(trainer_version=lay["trainer_version"], max_staleness=cfg.max_staleness,
                      active_tokens_dev=counts[0:1])

    def step():
        rl.seq_bookkeeping(cu, y, V, tok, act, loss_mask=mask, seq_version=ver, trainer_version=lay["trainer_version"],
                           max_staleness=cfg.max_staleness, counts_out=counts)
        rl.group_advantage(rew, cug, adv, zv, batch_norm=True, seq_weight=act, workspace=ws_a)
        rl.policy_loss_fwd_bwd(x, y, old, tok, adv, p, dl, stats, ws, loss_mask=mask, seq_version=ver, logp_out=logp)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # the 5-launch chain is launch-bound: capture it once as a CUDA graph and replay it per step
    # (the library enqueues on torch's current stream, so the capture sees every launch)
    graph = None
    if not args.no_graph:
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cs):
                step()
        torch.cuda.current_stream().wait_stream(cs)
        graph.replay()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for i in range(args.steps):
        run()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1])
    step_ms = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])
    # the oracle, as it stands, over the same 512 tokens (the whole chain), on this host
    import oracle
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        bk = oracle.seq_bookkeeping(lay["cu_seqlens"], lay["loss_mask"], y_h, V, lay["seq_version"],
                                    lay["trainer_version"], cfg.max_staleness)
        adv_o, _ = oracle.group_advantage(lay["rewards"], lay["cu_groups"], batch_norm=True,
                                          seq_weight=bk["seq_active"])
        oracle.policy_loss_fwd_bwd(x_h.astype(np.float64), y_h, old_h, lay["loss_mask"], bk["token_seq"], adv_o,
                                   lay["seq_version"], bk["seq_active"],
                                   oracle.LossParams(global_active_tokens=float(bk["active_tokens"]),
                                                     trainer_version=lay["trainer_version"],
                                                     max_staleness=cfg.max_staleness))
    osecs = (time.perf_counter() - t0) / reps
    if rank == 0:
        bpt = 2 * V * 4 + SIDE_BYTES
        per = float(np.median(step_ms))
        print(json.dumps({
            "metric": METRIC, "value": N * args.steps / (ms / 1e3), "unit": "tokens/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "tiny (BASELINE.json configs[0]): 2 prompts x 4 responses x 64 tokens, V=1024, "
                                   "fp32 logits, 1 GPU", "config": "tiny", "tokens_per_step": N,
                       "cuda_graph": graph is not None,
                       "l2": "not flushed: a 4 MB batch is L2-resident; launch-bound (reported for the record)"},
            "roofline": {"bound": "hbm", "achieved": N * bpt / (per / 1e3) / 1e9, "peak": measured_peak_hbm()[0],
                         "unit": "GB/s", "frac": N * bpt / (per / 1e3) / 1e9 / measured_peak_hbm()[0],
                         "traffic": None, "kernel": "whole chain (bookkeeping + advantages + loss, 5 launches)",
                         "note": "launch-bound: 4 MB per step"},
            "cpu_baseline": {"value": N / osecs, "unit": "tokens/s", "cores": 1, "kind": "oracle",
                             "sample": f"the full fp64 oracle chain over all {N} tokens: {osecs:.3f} s per pass"},
            "e2e": None, "gpu_launches": 5 * args.steps, "clocks": clk,
            "step_ms": {"p10": float(np.percentile(step_ms, 10)), "p50": per,
                        "p90": float(np.percentile(step_ms, 90))}}), flush=True)


def run_lmhead(args):
    """NEXT 4 (not the headline metric): the LM-head policy-loss training step without logits on
    one GPU — rl_lmhead_logprob (tcgen05 GEMM + online softmax) -> rl_policy_loss_from_logp (loss
    statistics and s_t) -> rl_lmhead_loss_bwd (tcgen05 logits recompute into G = s (p - onehot) per
    16,384-token chunk + cuBLAS dh = G W, dW += G^T h) over 65,536 tokens of a Qwen3-8B-sized head
    (d = 4096, V = 151936, bf16).  Tensor roofline: 8 N V d flops per step (2 forward + 2 recompute
    + 2 dh + 2 dW) against MEASURED_PEAKS.json's sustained bf16 figure (a long step).  Replicas only
    for N > 1 (independent token batches, no collective)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2605_15565_b200 as rl
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    rl.load()
    N, d, V, C = 65536, 4096, 151936, 16384
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    h = torch.randn(N, d, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(V, d, device=dev, generator=g) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    y = torch.randint(0, V, (N,), device=dev, generator=g, dtype=torch.int32)
    lp = torch.empty(N, device=dev)
    lse = torch.empty(N, device=dev)
    ws = torch.empty(max(1, rl.lmhead_workspace_size(N, d, V)), dtype=torch.uint8, device=dev)
    # the loss inputs: 256-token sequences, behaviour log-probs = a setup forward pass + drift
    L = 256
    S = N // L
    tseq = (torch.arange(N, device=dev) // L).to(torch.int32)
    adv = torch.randn(S, device=dev, generator=g)
    rl.lmhead_logprob(h, w, y, lp, lse, workspace=ws)
    old = lp + 0.02 * torch.randn(N, device=dev, generator=g)
    stats = torch.zeros(12, dtype=torch.float64, device=dev)
    scale = torch.empty(N, device=dev)
    ws_l = torch.empty(rl.policy_loss_from_logp_workspace_size(N), dtype=torch.uint8, device=dev)
    p = rl.LossParams(global_active_tokens=float(N))
    ws_b = torch.empty(rl.lmhead_loss_bwd_workspace_size(C, V), dtype=torch.uint8, device=dev)
    dh = torch.empty(N, d, device=dev)
    dW = torch.empty(V, d, device=dev)
    fwd_launches = 1 + (rl.lmhead_workspace_size(N, d, V) > 0)
    launches = fwd_launches + 2 + 3 * (N // C)   # fwd (+combine), loss + reduce, per chunk: grad kernel + 2 GEMMs

    def step():
        rl.lmhead_logprob(h, w, y, lp, lse, workspace=ws)
        rl.policy_loss_from_logp(lp, y, old, tseq, adv, p, stats, ws_l, V, scale_out=scale)
        rl.lmhead_loss_bwd(h, w, y, lse, scale, ws_b, dhidden=dh, dweight=dW)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    evs[0].record(stream)
    for i in range(args.steps):
        fe[i][0].record(stream)
        rl.lmhead_logprob(h, w, y, lp, lse, workspace=ws)
        fe[i][1].record(stream)
        rl.policy_loss_from_logp(lp, y, old, tseq, adv, p, stats, ws_l, V, scale_out=scale)
        rl.lmhead_loss_bwd(h, w, y, lse, scale, ws_b, dhidden=dh, dweight=dW)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1])
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
    per_step = ms / args.steps
    step_ms = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)])
    fwd_ms = float(np.mean([a.elapsed_time(b) for a, b in fe]))
    flops = 8.0 * N * V * d
    achieved = flops / (per_step / 1e3) / 1e12
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, src = 2250.0, "fallback (nominal dense bf16)"
    if os.path.exists(pk):
        with open(pk) as f:
            peak, src = float(json.load(f)["bf16_tflops_sustained"]), \
                "measured (MEASURED_PEAKS.json bf16_tflops_sustained: cuBLAS 8192^3 back to back for 4 s)"
    if rank == 0:
        print(json.dumps({
            "metric": "fused LM-head policy-loss step tokens/s (NEXT 4 fwd + bwd; d=4096, V=151936)",
            "value": world * N * args.steps / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "65,536 tokens x Qwen3-8B-sized LM head (d 4096, V 151936) per GPU per step: "
                                   "log-prob forward, loss, backward to dh and dW; logits never materialised",
                       "config": "lmhead", "tokens_per_step": world * N, "parallelism": f"replicas x{world}",
                       "bwd_chunk_tokens": C,
                       "l2": "no flush: every GEMM streams the 1.24 GB weight >> 126 MB L2"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": src,
                         "kernel": "the step: lmhead_kernel<logprob> + lmhead_kernel<grad> + cuBLAS dh / dW GEMMs",
                         "algorithmic_flops_per_launch": flops, "avg_launch_ms": per_step,
                         "forward_ms": fwd_ms, "forward_tflops": 2.0 * N * V * d / (fwd_ms / 1e3) / 1e12,
                         "backward_ms": per_step - fwd_ms,
                         "backward_tflops": 6.0 * N * V * d / ((per_step - fwd_ms) / 1e3) / 1e12},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches * args.steps, "clocks": clk,
            "step_ms": {"p10": float(np.percentile(step_ms, 10)), "p50": float(np.median(step_ms)),
                        "p90": float(np.percentile(step_ms, 90))}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(rl, torch, dev, x_dev, y_dev, old_dev, tok_dev, adv_dev, mask_dev, ver_dev, lay, V, args):
    """End-to-end through rl_policy_loss_fwd_bwd_host: every step copies its logits and side
    arrays from pinned host memory (H2D inside the timed region), runs the fused kernel and
    reads back the gradient dlogits (bf16, the same size as the logits), the per-token
    log-probs and the loss statistics (D2H) — the library overlaps the H2D of chunk c+1, the
    kernel on chunk c and the D2H of chunk c-1 (PCIe is full duplex)."""
    E = 32768                      # tokens per e2e step (9.96 GB of bf16 logits in, 9.96 GB of dlogits out)
    CH = 4096                      # staging chunk
    x = torch.empty((E, V), dtype=torch.bfloat16, pin_memory=True)
    x.copy_(x_dev[:E])
    dlh = torch.empty((E, V), dtype=torch.bfloat16, pin_memory=True)
    y, old, tok = y_dev[:E].cpu().pin_memory(), old_dev[:E].cpu().pin_memory(), tok_dev[:E].cpu().pin_memory()
    mask = mask_dev[:E].cpu().pin_memory()
    n_seq = E // 2048
    adv, ver = adv_dev[:n_seq].cpu(), ver_dev[:n_seq].cpu()
    logp = torch.empty(E, dtype=torch.float32, pin_memory=True)
    ws = torch.empty(rl.policy_loss_host_workspace_size(CH, V, V, rl.BF16, n_seq), dtype=torch.uint8, device=dev)
    p = rl.LossParams(trainer_version=lay["trainer_version"], global_active_tokens=float(E))
    torch.cuda.synchronize()
    steps, warm = max(3, min(args.steps, 5)), 2
    for i in range(warm + steps):
        if i == warm:
            t0 = time.perf_counter()
        rl.policy_loss_fwd_bwd_host(x, y, old, tok, adv, p, ws, CH, loss_mask=mask, seq_version=ver,
                                    logp_out=logp, dlogits=dlh)
    secs = time.perf_counter() - t0
    h2d = E * V * 2 + E * (4 + 4 + 4 + 1) + n_seq * 8
    d2h = E * V * 2 + E * 4 + 8 * 12
    return {"value": E * steps / secs, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "seconds": secs, "tokens": E * steps,
            "sample": f"{E} tokens per step through rl_policy_loss_fwd_bwd_host, {CH}-token chunks, "
                      "logits in and dlogits out through pinned host memory"}


if __name__ == "__main__":
    main()
