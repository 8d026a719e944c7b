"""Seeded input recipes (SURVEY.md §8(d) "Synthetic inputs").

Configs mirror BASELINE.json ``configs`` (tiny, single, long, vocabpar, multi).
Per-sequence / per-token side arrays are generated on the host with NumPy
(O(tokens), cheap at every size).  Logits are generated either on the host
(``host_logits``, per-row counter-based Philox streams, any row subset) or on the
device (``device_logits``, torch CUDA RNG, chunked; used at full size where the
host cannot hold [N, V]).  Nothing here computes any part of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

__all__ = [
    "SynthConfig", "CONFIGS", "get_config", "seq_layout", "host_logits", "device_logits",
    "perturb_old_logp", "bf16_round_bits", "pad_ld", "dominant_logits",
]


@dataclass(frozen=True)
class SynthConfig:
    name: str
    n_prompts: int
    group: int
    seq_len: int
    vocab: int
    dtype: str                  # "f32" | "bf16"
    seed: int
    mask_mode: str              # "prompt16" | "all" | "multiturn" | "prompt_u"
    ignore_frac: float = 0.0    # fraction of targets set to -100 (ignored)
    force_zero_var_group: bool = False
    trainer_version: int = 10
    staleness_max: int = 0      # per-sequence staleness drawn U{0..staleness_max}
    stale_outlier_frac: float = 0.0   # fraction of sequences with staleness in {9, 10}
    sigma_delta: float = 0.02   # old-logp drift, scaled by (1 + staleness)
    big_delta_frac: float = 0.0  # fraction of tokens with |delta| ~ U[0.3, 1]
    max_staleness: int = -1     # the loss knob used with this config
    vocab_shards: int = 1
    extra: dict = field(default_factory=dict)

    @property
    def n_seq(self) -> int:
        return self.n_prompts * self.group

    @property
    def n_tokens(self) -> int:
        return self.n_seq * self.seq_len


CONFIGS = {
    # BASELINE.json configs[0]: 2 prompts x 4 responses x 64 tokens, V=1024, fp32
    "tiny": SynthConfig("tiny", 2, 4, 64, 1024, "f32", 1, "prompt16", ignore_frac=0.05,
                        force_zero_var_group=True, sigma_delta=0.05),
    # configs[1]: 32 x 8 x 2048, V=151936 bf16, 1 GPU
    "single": SynthConfig("single", 32, 8, 2048, 151936, "bf16", 2, "all",
                          staleness_max=1, sigma_delta=0.02),
    # configs[2]: 8 x 8 x 32768 multi-turn, tool output masked; token-sharded 2/4/8
    "long": SynthConfig("long", 8, 8, 32768, 151936, "bf16", 3, "multiturn",
                        staleness_max=1, sigma_delta=0.02),
    # configs[3]: 64K tokens, V split over 8 GPUs
    "vocabpar": SynthConfig("vocabpar", 8, 8, 1024, 151936, "bf16", 4, "all",
                            staleness_max=1, vocab_shards=8),
    # configs[4]: 2 policies (151936 / 128256), 128 x 8 x 4096, mixed staleness
    "multi_a": SynthConfig("multi_a", 64, 8, 4096, 151936, "bf16", 5, "prompt_u",
                           trainer_version=100, staleness_max=8, stale_outlier_frac=0.05,
                           big_delta_frac=0.01, max_staleness=8),
    "multi_b": SynthConfig("multi_b", 64, 8, 4096, 128256, "bf16", 6, "prompt_u",
                           trainer_version=57, staleness_max=8, stale_outlier_frac=0.05,
                           big_delta_frac=0.01, max_staleness=8),
}


def get_config(name: str, **overrides) -> SynthConfig:
    return replace(CONFIGS[name], **overrides) if overrides else CONFIGS[name]


def pad_ld(vocab: int, mult: int = 8) -> int:
    return (vocab + mult - 1) // mult * mult


# ----------------------------------------------------------------------------- side data
def seq_layout(cfg: SynthConfig, seed: Optional[int] = None):
    """Per-sequence and per-token side arrays for a whole config (host, NumPy).

    Returns dict: rewards f64[S] (Bernoulli(p_g), p_g ~ U(0,1); binary as in the
    paper's math workloads), cu_groups i32[G+1], cu_seqlens i32[S+1], loss_mask u8[N],
    ignore i8[N] (1 where the target is to be replaced by -100), seq_version i32[S],
    trainer_version, big_delta u8[N] (tokens that get an outlier behaviour drift).
    """
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed if seed is None else seed, 0xA5]))
    S, G, n = cfg.n_seq, cfg.n_prompts, cfg.group
    p_g = rng.uniform(0.0, 1.0, size=G)
    rewards = (rng.uniform(size=(G, n)) < p_g[:, None]).astype(np.float64)
    if cfg.force_zero_var_group:
        rewards[0, :] = 1.0
    rewards = rewards.reshape(S)
    cu_groups = (np.arange(G + 1) * n).astype(np.int32)
    cu_seqlens = (np.arange(S + 1, dtype=np.int64) * cfg.seq_len).astype(np.int32)
    N = cfg.n_tokens
    T = cfg.seq_len
    mask = np.ones(N, dtype=np.uint8)
    if cfg.mask_mode == "prompt16":
        m = mask.reshape(S, T)
        m[:, :16] = 0
    elif cfg.mask_mode == "prompt_u":
        m = mask.reshape(S, T)
        plen = rng.integers(256, 2001, size=S)          # prompts <= 2000 tokens
        for i in range(S):
            m[i, :min(plen[i], T)] = 0
    elif cfg.mask_mode == "multiturn":
        # prompt U[512,4096] masked, then alternating assistant spans
        # U[64,1024] (unmasked; per-turn max_new_tokens 512-1024) and
        # tool/env spans U[32,1024] (masked, "tool-output masked", BASELINE.json configs[2])
        m = mask.reshape(S, T)
        for i in range(S):
            pos = int(rng.integers(512, 4097))
            m[i, :pos] = 0
            assistant = True
            while pos < T:
                ln = int(rng.integers(64, 1025)) if assistant else int(rng.integers(32, 1025))
                if not assistant:
                    m[i, pos:pos + ln] = 0
                pos += ln
                assistant = not assistant
    elif cfg.mask_mode != "all":
        raise ValueError(cfg.mask_mode)
    ignore = (rng.uniform(size=N) < cfg.ignore_frac).astype(np.uint8) if cfg.ignore_frac > 0 \
        else np.zeros(N, dtype=np.uint8)
    stale = rng.integers(0, cfg.staleness_max + 1, size=S) if cfg.staleness_max > 0 \
        else np.zeros(S, dtype=np.int64)
    if cfg.stale_outlier_frac > 0:
        out = rng.uniform(size=S) < cfg.stale_outlier_frac
        stale = np.where(out, rng.integers(9, 11, size=S), stale)
    seq_version = (cfg.trainer_version - stale).astype(np.int32)
    big = (rng.uniform(size=N) < cfg.big_delta_frac).astype(np.uint8) if cfg.big_delta_frac > 0 \
        else np.zeros(N, dtype=np.uint8)
    return dict(rewards=rewards, cu_groups=cu_groups, cu_seqlens=cu_seqlens, loss_mask=mask,
                ignore=ignore, seq_version=seq_version, trainer_version=cfg.trainer_version,
                seq_staleness_drawn=stale.astype(np.int32), big_delta=big)


# ----------------------------------------------------------------------------- logits
def bf16_round_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round-to-nearest-even (NaN kept quiet)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    nan = np.isnan(x)
    out = rounded.astype(np.uint16)
    out[nan] = 0x7FC0
    return out


def _row_rng(seed: int, row: int) -> np.random.Generator:
    # counter-based: stream depends only on (seed, global row id)
    return np.random.Generator(np.random.Philox(key=np.array([seed, row], dtype=np.uint64)))


def host_logits(cfg_or_vocab, rows, seed: int, dtype: str = "f32"):
    """Logit model: x_v = sigma_t*g_v + sum_j D_j [v == h_j],
    g ~ N(0,1), sigma_t ~ U[1,3], k_t ~ U{1..4} hot columns, D_0 ~ U[6,20],
    D_j>0 ~ U[2,10]; bf16 rows are rounded RNE.  Targets are sampled exactly at
    T = 1 by Gumbel-max on the stored (rounded) values.

    Returns (logits, targets) with logits float32 [R, V] (dtype f32) or uint16 bf16
    bits [R, V] (dtype bf16).
    """
    V = cfg_or_vocab if isinstance(cfg_or_vocab, int) else cfg_or_vocab.vocab
    rows = np.asarray(rows, dtype=np.int64)
    R = len(rows)
    out = np.empty((R, V), dtype=np.float32 if dtype == "f32" else np.uint16)
    y = np.empty(R, dtype=np.int32)
    for k, row in enumerate(rows):
        g = _row_rng(seed, int(row))
        sigma = g.uniform(1.0, 3.0)
        x = (sigma * g.standard_normal(V)).astype(np.float32)
        nh = int(g.integers(1, 5))
        cols = g.integers(0, V, size=nh)
        for j in range(nh):
            x[cols[j]] += np.float32(g.uniform(6.0, 20.0) if j == 0 else g.uniform(2.0, 10.0))
        if dtype == "bf16":
            bits = bf16_round_bits(x)
            out[k] = bits
            xs = (bits.astype(np.uint32) << 16).view(np.float32)
        else:
            out[k] = x
            xs = x
        u = g.uniform(np.finfo(np.float64).tiny, 1.0, size=V)
        y[k] = int(np.argmax(xs.astype(np.float64) - np.log(-np.log(u))))
    return out, y


def device_logits(out, vocab: int, row0: int, seed: int, chunk: int = 2048, targets_out=None):
    """Fill a device tensor ``out`` [R, ld] (torch bf16 or f32, CUDA) with the logit
    model of ``host_logits`` using torch's CUDA Philox RNG, chunk by chunk; rows are
    global ids row0..row0+R-1 and each chunk's stream is keyed on (seed, global
    chunk index), so shards of one batch reproduce the unsharded batch as long as
    row0 is a multiple of ``chunk``.  Columns >= vocab (padding up to ld) are set to 0.
    Writes the Gumbel-max sampled targets into ``targets_out`` (int32 [R]) if given.
    """
    R, ld = out.shape
    return _device_fill(out, R, ld, vocab, row0, seed, chunk, targets_out)


def _device_fill(out, R, ld, V, row0, seed, chunk, targets_out):
    import torch
    dev = out.device
    assert row0 % chunk == 0, "row0 must be chunk-aligned for reproducible shards"
    for c0 in range(0, R, chunk):
        c1 = min(R, c0 + chunk)
        n = c1 - c0
        gen = torch.Generator(device=dev)
        gen.manual_seed((seed * 1_000_003 + (row0 + c0) // chunk) & 0x7FFFFFFFFFFFFFFF)
        sigma = torch.rand((n, 1), generator=gen, device=dev) * 2.0 + 1.0
        x = torch.randn((n, V), generator=gen, device=dev, dtype=torch.float32)
        x.mul_(sigma)
        nh = torch.randint(1, 5, (n,), generator=gen, device=dev)
        cols = torch.randint(0, V, (n, 4), generator=gen, device=dev)
        d0 = torch.rand((n, 1), generator=gen, device=dev) * 14.0 + 6.0
        dj = torch.rand((n, 3), generator=gen, device=dev) * 8.0 + 2.0
        d = torch.cat([d0, dj], dim=1) * (torch.arange(4, device=dev)[None, :] < nh[:, None])
        x.scatter_add_(1, cols, d)
        xs = x.to(out.dtype)
        out[c0:c1, :V].copy_(xs)
        if ld > V:
            out[c0:c1, V:].zero_()
        if targets_out is not None:
            u = torch.rand((n, V), generator=gen, device=dev, dtype=torch.float32)
            u.clamp_(min=1e-30).log_().neg_().log_().neg_()   # Gumbel(0,1)
            u.add_(xs.float())
            targets_out[c0:c1].copy_(torch.argmax(u, dim=1).to(torch.int32))
            del u
        del x, xs
    return out


def perturb_old_logp(logp_ref: np.ndarray, token_staleness: np.ndarray, big_delta: np.ndarray,
                     cfg: SynthConfig, seed: int) -> np.ndarray:
    """Behaviour log-probs = reference log-probs + drift delta_t ~ N(0, sigma^2),
    sigma = sigma_delta*(1 + staleness); plus |delta| ~ U[0.3, 1] (random sign) on
    the ``big_delta`` tokens so both clip branches fire."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x51]))
    n = len(logp_ref)
    sig = cfg.sigma_delta * (1.0 + np.asarray(token_staleness, dtype=np.float64))
    delta = rng.standard_normal(n) * sig
    bigv = rng.uniform(0.3, 1.0, size=n) * np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
    delta = np.where(np.asarray(big_delta) != 0, bigv, delta)
    return (np.asarray(logp_ref, dtype=np.float64) + delta).astype(np.float32)


def dominant_logits(n_rows: int, vocab: int, seed: int):
    """Rows built to stress the bf16 gradient path (reading R2): a N(0,1)
    background plus ONE dominant column h_t with D_t ~ U[14, 21] (over a ~152K-column N(0,1)
    background that makes its probability ~0.75-0.9995), and a target y_t drawn uniformly among
    the other columns — a confident model that sampled another token, so the row's largest
    gradient element is a non-target s p_h.  Every 4th row instead puts the dominant column at
    the target.  Returns (bf16 bits [n, V], targets int32 [n], dominant columns int32 [n])."""
    g = np.random.Generator(np.random.Philox(key=np.array([seed, 0xD0], dtype=np.uint64)))
    x = g.standard_normal((n_rows, vocab), dtype=np.float32)
    h = g.integers(0, vocab, size=n_rows)
    y = (h + g.integers(1, vocab, size=n_rows)) % vocab
    y = np.where(np.arange(n_rows) % 4 == 3, h, y)
    x[np.arange(n_rows), h] += g.uniform(14.0, 21.0, size=n_rows).astype(np.float32)
    return bf16_round_bits(x), y.astype(np.int32), h.astype(np.int32)
