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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default=None, choices=[None, "cluster", "two_pass"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--minibatch-tokens", type=int, default=131072)
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
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.kernel:
        os.environ["RL_LOSS_KERNEL"] = args.kernel
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_15565_b200 as rl
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rl.load()
    comm = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
        comm = rl.Comm.from_torch()
    cfg = synth.get_config("single")
    V = cfg.vocab
    T = cfg.seq_len
    MB = args.minibatch_tokens
    N = N_MINIBATCH * MB                # 524,288 tokens per rank at the default MB
    assert MB % T == 0 and N <= cfg.n_tokens
    S_mb = MB // T
    S = N // T                          # 256 sequences per rank at the default MB
    G = S // cfg.group
    lay = synth.seq_layout(cfg, seed=cfg.seed + 1000 * rank)

    # --- resident inputs: 2 distinct mini-batch logits buffers + targets / old logp
    POOL = 2
    pool, pool_y, pool_old = [], [], []
    for b in range(POOL):
        x = torch.empty((MB, V), dtype=torch.bfloat16, device=dev)
        y = torch.empty(MB, dtype=torch.int32, device=dev)
        synth.device_logits(x, V, row0=(rank * POOL + b) * MB, seed=cfg.seed, targets_out=y)
        # behaviour log-probs: log-softmax via torch (input synthesis only) + seeded drift
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
    dlogits = torch.empty((MB, V), dtype=torch.bfloat16, device=dev)
    torch.cuda.synchronize()

    rewards = torch.from_numpy(lay["rewards"][:S]).to(dev)
    cu_groups = torch.from_numpy(lay["cu_groups"][:G + 1]).to(dev)
    seq_version = torch.from_numpy(lay["seq_version"][:S]).to(dev)
    mask = torch.from_numpy(lay["loss_mask"][:N]).to(dev)
    cu_mb = torch.from_numpy((np.arange(S_mb + 1) * T).astype(np.int32)).to(dev)
    token_seq = torch.empty((N_MINIBATCH, MB), dtype=torch.int32, device=dev)
    seq_active = torch.empty(S, dtype=torch.int32, device=dev)
    counts = torch.zeros((N_MINIBATCH, 20), dtype=torch.float64, device=dev)
    adv = torch.empty(S, dtype=torch.float32, device=dev)
    zero_var = torch.empty(G, dtype=torch.uint8, device=dev)
    ws_adv = torch.empty(rl.group_advantage_workspace_size(S), dtype=torch.uint8, device=dev)
    stats = torch.zeros((N_MINIBATCH, 10), dtype=torch.float64, device=dev)
    ws = torch.empty(rl.policy_loss_workspace_size(MB, V), dtype=torch.uint8, device=dev)
    logp = torch.empty((N_MINIBATCH, MB), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ev_loss = []          # (start, end) CUDA events around every loss launch in the timed region
    launches = [0]

    def step(record: bool):
        for j in range(N_MINIBATCH):
            rl.seq_bookkeeping(cu_mb, pool_y[j % POOL], V, token_seq[j], seq_active[j * S_mb:(j + 1) * S_mb],
                               loss_mask=mask[j * MB:(j + 1) * MB],
                               seq_version=seq_version[j * S_mb:(j + 1) * S_mb],
                               trainer_version=lay["trainer_version"], max_staleness=-1,
                               counts_out=counts[j])
            launches[0] += 2
            if comm is not None:
                comm.allreduce_f64(counts[j])
        rl.group_advantage(rewards, cu_groups, adv, zero_var, batch_norm=True, seq_weight=seq_active,
                           workspace=ws_adv)
        launches[0] += 1
        for j in range(N_MINIBATCH):
            p = rl.LossParams(trainer_version=lay["trainer_version"], active_tokens_dev=counts[j, 0:1])
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            rl.policy_loss_fwd_bwd(pool[j % POOL], pool_y[j % POOL], pool_old[j % POOL], token_seq[j],
                                   adv[j * S_mb:(j + 1) * S_mb], p, dlogits, stats[j], ws,
                                   loss_mask=mask[j * MB:(j + 1) * MB],
                                   seq_version=seq_version[j * S_mb:(j + 1) * S_mb],
                                   logp_out=logp[j])
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                ev_loss.append((e0, e1))
            launches[0] += 2
            if comm is not None:
                comm.allreduce_f64(stats[j])

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
    launches[0] = 0
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step(True)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t0.elapsed_time(t1)
    gpu_launches = launches[0]
    if world > 1:
        tt = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = tt.item()
    loss_ms = [a.elapsed_time(b) for a, b in ev_loss]
    avg_loss_ms = sum(loss_ms) / len(loss_ms)
    tokens_total = world * N * args.steps
    value = tokens_total / (elapsed_ms / 1e3)

    # --- roofline of the dominant kernel (fused loss): algorithmic bytes / launch duration
    bytes_per_token = 2 * V * 2 + SIDE_BYTES
    alg_bytes = MB * bytes_per_token
    achieved = alg_bytes / (avg_loss_ms / 1e3) / 1e9
    peak, peak_src = measured_peak_hbm()
    kern = os.environ.get("RL_LOSS_KERNEL", "cluster")
    traffic = ncu_traffic(kern)

    # --- e2e: the host-buffer C-ABI entry point, pinned host logits, H2D inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(rl, torch, dev, pool[0], pool_y[0], pool_old[0], token_seq[0], adv[:S_mb],
                          mask[:MB], seq_version[:S_mb], lay, V, args)
        if world > 1:
            tt = torch.tensor([e2e["seconds"]], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e["value"] = world * e2e["tokens"] / tt.item()
        e2e = {k: e2e[k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step", "sample")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        x16 = pool[0][:64].view(torch.int16).cpu().numpy().view(np.uint16)
        yy = pool_y[0][:64].cpu().numpy()
        oo = pool_old[0][:64].cpu().numpy()
        workers = host_cores()
        rate, secs, done = time_oracle(x16, yy, oo, 8192, workers)
        cpu = {"value": rate, "unit": "tokens/s", "cores": workers, "kind": "oracle",
               "sample": f"{done} token rows (64 distinct rows of mini-batch 0) x V=151936 fwd+bwd "
                         f"in {secs:.1f} s wall over {workers} processes"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD if MB == 131072 else f"PROFILING ONLY: {N} tokens/step",
                       "tokens_per_rank_per_step": N,
                       "minibatches_per_step": N_MINIBATCH, "minibatch_tokens": MB, "vocab": V,
                       "global_batch_tokens": world * N, "parallelism": f"dp{world} (token-parallel)",
                       "loss_kernel": kern, "l2": "no flush: each call streams a distinct 39.8 GB "
                       "buffer (pool of 2) >> 126 MB L2", "agg": "token_mean", "batch_norm": True},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": f"rl_policy_loss_fwd_bwd ({kern})",
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "bytes_per_token": bytes_per_token, "avg_launch_ms": avg_loss_ms,
                         "frac_of_8TBs": achieved / 8000.0},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
        dist.destroy_process_group()


def measure_e2e(rl, torch, dev, x_dev, y_dev, old_dev, tok_dev, adv_dev, mask_dev, ver_dev, lay, V, args):
    """End-to-end through rl_policy_loss_fwd_bwd_host: every step copies its logits and side
    arrays from pinned host memory (H2D inside the timed region), runs the fused kernel and
    reads back the loss statistics and per-token log-probs (D2H)."""
    E = 32768                      # tokens per e2e step (9.96 GB of bf16 logits)
    CH = 4096                      # staging chunk
    x = torch.empty((E, V), dtype=torch.bfloat16, pin_memory=True)
    x.copy_(x_dev[:E])
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
                                    logp_out=logp)
    secs = time.perf_counter() - t0
    h2d = E * V * 2 + E * (4 + 4 + 4 + 1) + n_seq * 8
    d2h = E * 4 + 80
    return {"value": E * steps / secs, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "seconds": secs, "tokens": E * steps,
            "sample": f"{E} tokens per step through rl_policy_loss_fwd_bwd_host, {CH}-token chunks"}


if __name__ == "__main__":
    main()
