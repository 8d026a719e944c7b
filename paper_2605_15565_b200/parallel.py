"""Host-side sharding plans for the two ways the path splits across GPUs (
SURVEY.md §8(e)).  Pure integer bookkeeping: no arithmetic of the method lives here.

* token / sequence parallel: whole sequences per rank, contiguous, balanced by token count;
  per-sequence arrays stay replicated, so every rank computes identical advantages and only the
  batch counts (before) and loss statistics (after) are all-reduced.
* vocab parallel: contiguous column ranges, every boundary a multiple of 8 columns so each
  shard row keeps 16-B aligned bf16 vectors.
* multi-policy (configs[4]): the world splits into one contiguous trainer group per policy
  (rl_comm_split colour = policy, key = rank in the group); each group is token-parallel on its own
  policy's batch and the groups never communicate.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

__all__ = ["SeqShard", "shard_sequences", "VocabShard", "shard_vocab", "PolicyGroup", "policy_group"]


@dataclass(frozen=True)
class SeqShard:
    seq_begin: int
    seq_end: int
    tok_begin: int
    tok_end: int

    @property
    def n_seq(self) -> int:
        return self.seq_end - self.seq_begin

    @property
    def n_tokens(self) -> int:
        return self.tok_end - self.tok_begin


def shard_sequences(cu_seqlens: Sequence[int], world: int, rank: int) -> SeqShard:
    """Contiguous whole-sequence shard of rank `rank`: sequence boundaries are chosen so each
    rank's token count is as close as possible to total/world (greedy on the prefix sums).
    Every sequence belongs to exactly one rank; ranks may be empty when world > n_seq."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    cu = [int(x) for x in cu_seqlens]
    n_seq, total = len(cu) - 1, cu[-1]
    # boundary b_r = the sequence index whose start is closest to r*total/world (monotone)
    bounds = [0]
    for r in range(1, world):
        target = r * total / world
        i = bounds[-1]
        while i < n_seq and abs(cu[i + 1] - target) <= abs(cu[i] - target):
            i += 1
        bounds.append(i)
    bounds.append(n_seq)
    s0, s1 = bounds[rank], bounds[rank + 1]
    return SeqShard(s0, s1, cu[s0], cu[s1])


@dataclass(frozen=True)
class VocabShard:
    offset: int
    size: int


def shard_vocab(vocab: int, world: int, rank: int, align: int = 8) -> VocabShard:
    """Columns [offset, offset + size) of rank `rank`; boundaries are multiples of `align`
    (the last shard takes the remainder)."""
    if world < 1 or not (0 <= rank < world) or vocab < 1:
        raise ValueError("bad vocab/world/rank")
    units = (vocab + align - 1) // align
    per = units // world
    extra = units % world
    u0 = rank * per + min(rank, extra)
    u1 = u0 + per + (1 if rank < extra else 0)
    lo, hi = min(vocab, u0 * align), min(vocab, u1 * align)
    return VocabShard(lo, hi - lo)


@dataclass(frozen=True)
class PolicyGroup:
    policy: int      # rl_comm_split colour
    key: int         # rank inside the policy's trainer group (rl_comm_split key)
    size: int        # ranks in the group
    first: int       # global rank of the group's rank 0

    @property
    def ranks(self) -> range:
        return range(self.first, self.first + self.size)


def policy_group(world: int, n_policies: int, rank: int) -> PolicyGroup:
    """Trainer group of global rank `rank` when `world` ranks serve `n_policies` policies:
    contiguous groups, the first world % n_policies groups one rank larger (4 + 4 for the
    paper's two policies on 8 GPUs).  With world < n_policies the single rank serves all
    policies in turn (group 0 of size 1)."""
    if world < 1 or n_policies < 1 or not (0 <= rank < world):
        raise ValueError("bad world/n_policies/rank")
    if world < n_policies:
        return PolicyGroup(0, rank, world, 0)
    per, extra = divmod(world, n_policies)
    first = 0
    for pol in range(n_policies):
        size = per + (1 if pol < extra else 0)
        if rank < first + size:
            return PolicyGroup(pol, rank - first, size, first)
        first += size
    raise AssertionError("unreachable")
