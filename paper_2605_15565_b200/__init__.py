"""B200-native trainer policy-loss hot path of AstraFlow (arXiv 2605.15565).

Thin ctypes binding over the C-ABI library ``librlpolicy.so`` (include/rl_policy.h).
Argument marshalling only: every step of the path runs in the library's sm_100a kernels.
There is no CPU fallback: if the library is missing or CUDA is unavailable, calls raise.

Functions keep the C names without the ``rl_`` prefix and take torch tensors:
``group_advantage``, ``seq_bookkeeping``, ``token_logprob``, ``policy_loss_fwd_bwd``,
``policy_loss_fwd_bwd_host``, ``vocab_parallel_logprob`` and the ``Comm`` wrapper.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

__all__ = [
    "load", "lib_path", "RLError", "LossParams", "STATS_FIELDS", "COUNTS_FIELDS",
    "STD_UNBIASED", "STD_BIASED", "STD_NONE", "AGG_TOKEN_MEAN", "AGG_SEQ_MEAN_TOKEN_MEAN",
    "AGG_SUM", "F_STATS_ACCUMULATE", "F_SKIP_MASKED_READS", "F_ENTROPY", "F32", "BF16",
    "group_advantage", "group_advantage_workspace_size", "seq_bookkeeping", "token_logprob",
    "policy_loss_fwd_bwd", "policy_loss_workspace_size", "policy_loss_fwd_bwd_host",
    "policy_loss_host_workspace_size", "vocab_parallel_logprob",
    "vocab_parallel_workspace_size", "m2po_mask", "m2po_workspace_size", "delta_encode", "delta_apply",
    "delta_workspace_size", "lmhead_logprob", "lmhead_workspace_size", "policy_loss_from_logp",
    "policy_loss_from_logp_workspace_size", "lmhead_loss_bwd", "lmhead_loss_bwd_workspace_size", "Comm",
    "EXPORTED_SYMBOLS",
]

F32, BF16 = 0, 1
STD_UNBIASED, STD_BIASED, STD_NONE = 0, 1, 2
AGG_TOKEN_MEAN, AGG_SEQ_MEAN_TOKEN_MEAN, AGG_SUM = 0, 1, 2
F_STATS_ACCUMULATE, F_SKIP_MASKED_READS, F_ENTROPY = 0x1, 0x2, 0x4
STALE_HIST_BINS = 16
STATS_FIELDS = ("loss_sum", "active_tokens", "weight_sum", "ratio_sum", "clipped_low",
                "clipped_high", "clamped", "stale_masked", "bad_targets", "neg_staleness",
                "kl_sum", "entropy_sum")
COUNTS_FIELDS = ("active_tokens", "stale_masked", "neg_staleness", "bad_targets")
N_COUNTS = len(COUNTS_FIELDS) + STALE_HIST_BINS

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

vp, i32, i64, f32, f64, u32, sz = (C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double,
                                   C.c_uint32, C.c_size_t)


class _Params(C.Structure):
    _fields_ = [("clip_eps_low", f32), ("clip_eps_high", f32), ("inv_temperature", f32),
                ("log_ratio_clamp", f32), ("grad_scale", f32), ("agg", i32),
                ("trainer_version", i32), ("max_staleness", i32), ("global_num_seqs", i32),
                ("flags", u32), ("global_active_tokens", f64), ("active_tokens_dev", vp),
                ("kl_coef", f32), ("ref_logp", vp), ("prox_logp", vp)]


# name -> (restype, argtypes)
_SIGS = {
    "rl_status_string": (C.c_char_p, [i32]),
    "rl_last_error": (C.c_char_p, []),
    "rl_abi_version": (i32, []),
    "rl_loss_params_default": (None, [vp]),
    "rl_group_advantage_workspace_size": (sz, [i32]),
    "rl_group_advantage": (i32, [vp, vp, i32, i32, i32, f64, i32, f64, vp, vp, sz, vp, vp, vp]),
    "rl_seq_bookkeeping": (i32, [vp, i32, i64, vp, vp, i64, vp, i32, i32, vp, vp, vp, vp, vp, vp,
                                 vp, vp]),
    "rl_token_logprob": (i32, [vp, i32, i64, i64, i64, vp, f32, vp, vp, vp, vp]),
    "rl_policy_loss_workspace_size": (sz, [i64, i64, i32]),
    "rl_policy_loss_fwd_bwd": (i32, [vp, i32, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                     vp, vp, vp, vp, sz, vp]),
    "rl_policy_loss_host_workspace_size": (sz, [i64, i64, i64, i32, i32]),
    "rl_policy_loss_fwd_bwd_host": (i32, [vp, i32, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, i32,
                                          vp, vp, vp, vp, i64, vp, sz, vp]),
    "rl_comm_unique_id": (i32, [vp]),
    "rl_comm_init": (i32, [vp, vp, i32, i32]),
    "rl_comm_split": (i32, [vp, i32, i32, vp]),
    "rl_comm_destroy": (i32, [vp]),
    "rl_comm_size": (i32, [vp, vp, vp]),
    "rl_comm_allreduce_f64": (i32, [vp, vp, sz, vp]),
    "rl_comm_enable_peer_exchange": (i32, [vp, i64]),
    "rl_vocab_parallel_workspace_size": (sz, [i64, i32]),
    "rl_vocab_parallel_logprob": (i32, [vp, i32, i64, i64, i64, i64, i64, vp, f32, vp, vp, vp, vp,
                                        vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
    "rl_m2po_workspace_size": (sz, [i64, i32]),
    "rl_m2po_mask": (i32, [vp, vp, vp, i64, f32, vp, vp, vp, vp, sz, vp]),
    "rl_bf16_delta_workspace_size": (sz, [i64]),
    "rl_bf16_delta_encode": (i32, [vp, vp, i64, vp, vp, i64, vp, vp, sz, vp]),
    "rl_bf16_delta_apply": (i32, [vp, i64, vp, vp, vp, i64, vp, vp]),
    "rl_lmhead_logprob": (i32, [vp, i64, vp, i64, i64, i64, i64, vp, f32, vp, vp, vp, sz, vp]),
    "rl_lmhead_workspace_size": (sz, [i64, i64, i64]),
    "rl_policy_loss_from_logp_workspace_size": (sz, [i64]),
    "rl_lmhead_loss_bwd_workspace_size": (sz, [i64, i64]),
    "rl_lmhead_loss_bwd": (i32, [vp, i64, vp, i64, i64, i64, i64, vp, vp, vp, f32, vp, i64, vp, i64, u32, vp, sz, vp]),
    "rl_policy_loss_from_logp": (i32, [vp, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


class RLError(RuntimeError):
    pass


def lib_path() -> str:
    # RL_LIB_PATH: development A/B of another build of the same library (tools/); default in-tree
    return os.environ.get("RL_LIB_PATH") or os.path.join(_HERE, "librlpolicy.so")


def load():
    """Load the in-tree librlpolicy.so (build it with ``python -m paper_2605_15565_b200.build``)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise RLError(f"{path} is missing: run `python -m paper_2605_15565_b200.build` "
                      "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib.rl_dev_set_option.restype = i32  # development hook (include/rl_policy_dev.h)
    lib.rl_dev_set_option.argtypes = [i32, i32]
    _LIB = lib
    return lib


# development options (include/rl_policy_dev.h): alternative kernels kept for A/B parity tests
DEV_LOSS_KERNEL, DEV_VP_PATH, DEV_LM_SPLITS, DEV_VP_KERNEL, DEV_VC_GROUPS, DEV_VC_ROWS, DEV_VC_PUB, DEV_LM_PAIR, \
    DEV_LM_GEMM, DEV_VR_DELAY, DEV_VC_TMEM = 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10


def dev_set_option(key: int, value: int) -> int:
    """Set a development option of the library; returns the previous value."""
    old = load().rl_dev_set_option(key, value)
    if old < 0:
        raise RLError(f"unknown development option {key}")
    return old


def _check(status: int, what: str):
    if status != 0:
        lib = load()
        raise RLError(f"{what}: {lib.rl_status_string(status).decode()} "
                      f"({lib.rl_last_error().decode()})")


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _dev(t, what):
    if t is not None and not t.is_cuda:
        raise RLError(f"{what} must be a CUDA tensor (no CPU fallback)")
    return _ptr(t)


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _dtype_code(t):
    import torch
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise RLError(f"unsupported logits dtype {t.dtype}")


@dataclass
class LossParams:
    """Mirror of rl_loss_params (include/rl_policy.h)."""
    clip_eps_low: float = 0.2
    clip_eps_high: float = 0.2
    inv_temperature: float = 1.0
    log_ratio_clamp: float = 20.0
    grad_scale: float = 1.0
    agg: int = AGG_TOKEN_MEAN
    trainer_version: int = 0
    max_staleness: int = -1
    global_num_seqs: int = 0
    flags: int = 0
    global_active_tokens: float = 0.0
    active_tokens_dev: object = None   # CUDA tensor (float64 scalar view) or int pointer
    kl_coef: float = 0.0               # beta of the k3 KL term (reading N1)
    ref_logp: object = None            # CUDA float32 [n_tokens] (required iff kl_coef != 0)
    prox_logp: object = None           # CUDA float32 [n_tokens] or None (decoupled ratio, N2)

    def _c(self) -> _Params:
        p = _Params()
        for f, _ in _Params._fields_:
            if f in ("active_tokens_dev", "ref_logp", "prox_logp"):
                v = getattr(self, f)
                if v is not None and hasattr(v, "is_cuda") and not v.is_cuda:
                    raise RLError(f"{f} must be a CUDA tensor")
                setattr(p, f, _ptr(v))
            else:
                setattr(p, f, getattr(self, f))
        return p


# ----------------------------------------------------------------------------- (1)
def group_advantage_workspace_size(n_seq: int) -> int:
    return load().rl_group_advantage_workspace_size(n_seq)


def group_advantage(rewards, cu_groups, adv_out, zero_var_out=None, std_mode=STD_UNBIASED,
                    eps=1e-6, batch_norm=False, bn_eps=1e-6, seq_weight=None, workspace=None,
                    stream=None):
    lib = load()
    if rewards.element_size() != 8 or cu_groups.element_size() != 4:
        raise RLError("rewards must be float64 and cu_groups int32 (rl_group_advantage)")
    n_groups = cu_groups.numel() - 1
    n_seq = rewards.numel()
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check(lib.rl_group_advantage(_dev(rewards, "rewards"), _dev(cu_groups, "cu_groups"), n_groups,
                                  n_seq, std_mode, eps, int(bool(batch_norm)), bn_eps,
                                  _dev(seq_weight, "seq_weight"), _dev(workspace, "workspace"),
                                  ws_bytes, _dev(adv_out, "adv_out"),
                                  _dev(zero_var_out, "zero_var_out"), _stream(stream)),
           "rl_group_advantage")


# ----------------------------------------------------------------------------- (2)
def seq_bookkeeping(cu_seqlens, targets, vocab, token_seq_out, seq_active_out, loss_mask=None,
                    seq_version=None, trainer_version=0, max_staleness=-1, seq_adv=None,
                    seq_staleness_out=None, adv_token_out=None, valid_out=None, counts_out=None,
                    stream=None):
    """counts_out: CUDA float64 tensor with >= 20 elements (rl_batch_counts)."""
    lib = load()
    if counts_out is not None and counts_out.numel() < N_COUNTS:
        raise RLError("counts_out needs 20 float64 elements")
    _check(lib.rl_seq_bookkeeping(_dev(cu_seqlens, "cu_seqlens"), cu_seqlens.numel() - 1,
                                  targets.numel(), _dev(loss_mask, "loss_mask"),
                                  _dev(targets, "targets"), vocab, _dev(seq_version, "seq_version"),
                                  trainer_version, max_staleness, _dev(seq_adv, "seq_adv"),
                                  _dev(token_seq_out, "token_seq_out"),
                                  _dev(seq_active_out, "seq_active_out"),
                                  _dev(seq_staleness_out, "seq_staleness_out"),
                                  _dev(adv_token_out, "adv_token_out"), _dev(valid_out, "valid_out"),
                                  _dev(counts_out, "counts_out"), _stream(stream)),
           "rl_seq_bookkeeping")


# ----------------------------------------------------------------------------- (3)
def token_logprob(logits, targets, logp_out, lse_out=None, vocab=None, inv_temperature=1.0,
                  bad_target_count=None, stream=None):
    lib = load()
    n, ld = logits.shape
    V = ld if vocab is None else vocab
    if logits.stride(1) != 1 or logits.stride(0) != ld:
        raise RLError("logits must be a contiguous [n_tokens, ld] tensor")
    _check(lib.rl_token_logprob(_dev(logits, "logits"), _dtype_code(logits), n, V, ld,
                                _dev(targets, "targets"), inv_temperature, _dev(logp_out, "logp_out"),
                                _dev(lse_out, "lse_out"), _dev(bad_target_count, "bad_target_count"),
                                _stream(stream)),
           "rl_token_logprob")


# ----------------------------------------------------------------------------- (4)
def policy_loss_workspace_size(n_tokens, vocab, dtype=BF16) -> int:
    return load().rl_policy_loss_workspace_size(n_tokens, vocab, dtype)


def policy_loss_fwd_bwd(logits, targets, old_logp, token_seq, seq_adv, params: LossParams,
                        dlogits, stats, workspace, loss_mask=None, seq_version=None,
                        seq_active=None, logp_out=None, clipped_out=None, vocab=None,
                        stream=None):
    """stats: CUDA float64 tensor with >= 12 elements (rl_loss_stats, STATS_FIELDS order).
    dlogits may be ``logits`` itself (in place)."""
    lib = load()
    n, ld = logits.shape
    V = ld if vocab is None else vocab
    if logits.stride(1) != 1 or logits.stride(0) != ld or dlogits.shape != logits.shape or \
            dlogits.stride() != logits.stride() or dlogits.dtype != logits.dtype:
        raise RLError("logits/dlogits must be contiguous [n_tokens, ld] tensors of one dtype")
    if stats.numel() < len(STATS_FIELDS):
        raise RLError(f"stats needs {len(STATS_FIELDS)} float64 elements")
    p = params._c()
    _check(lib.rl_policy_loss_fwd_bwd(
        _dev(logits, "logits"), _dtype_code(logits), n, V, ld, _dev(targets, "targets"),
        _dev(old_logp, "old_logp"), _dev(loss_mask, "loss_mask"), _dev(token_seq, "token_seq"),
        _dev(seq_adv, "seq_adv"), _dev(seq_version, "seq_version"), _dev(seq_active, "seq_active"),
        C.byref(p), _dev(dlogits, "dlogits"), _dev(logp_out, "logp_out"),
        _dev(clipped_out, "clipped_out"), _dev(stats, "stats"), _dev(workspace, "workspace"),
        workspace.numel() * workspace.element_size(), _stream(stream)),
        "rl_policy_loss_fwd_bwd")


def policy_loss_host_workspace_size(chunk_tokens, vocab, ld, dtype, n_seq) -> int:
    return load().rl_policy_loss_host_workspace_size(chunk_tokens, vocab, ld, dtype, n_seq)


def policy_loss_fwd_bwd_host(logits, targets, old_logp, token_seq, seq_adv, params: LossParams,
                             workspace, chunk_tokens, loss_mask=None, seq_version=None,
                             seq_active=None, dlogits=None, logp_out=None, vocab=None,
                             stats_out=None, stream=None):
    """All array arguments are CPU tensors (pinned for overlap); workspace is a CUDA tensor.
    Returns the rl_loss_stats as a dict (also written into ``stats_out`` if given)."""
    import torch
    lib = load()
    for name, t in (("logits", logits), ("targets", targets), ("old_logp", old_logp),
                    ("token_seq", token_seq), ("seq_adv", seq_adv)):
        if t.is_cuda:
            raise RLError(f"{name} must be a host tensor for the host-buffer entry point")
    n, ld = logits.shape
    V = ld if vocab is None else vocab
    st = stats_out if stats_out is not None else torch.zeros(len(STATS_FIELDS), dtype=torch.float64)
    p = params._c()
    _check(lib.rl_policy_loss_fwd_bwd_host(
        _ptr(logits), _dtype_code(logits), n, V, ld, _ptr(targets), _ptr(old_logp), _ptr(loss_mask),
        _ptr(token_seq), _ptr(seq_adv), _ptr(seq_version), _ptr(seq_active), seq_adv.numel(),
        C.byref(p), _ptr(dlogits), _ptr(logp_out), _ptr(st), chunk_tokens,
        _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(), _stream(stream)),
        "rl_policy_loss_fwd_bwd_host")
    return dict(zip(STATS_FIELDS, st.tolist()))


# ----------------------------------------------------------------------------- (5)
class Comm:
    """rl_comm (NCCL) bootstrapped over a torch.distributed process group."""

    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    @classmethod
    def from_torch(cls, group=None):
        import torch
        import torch.distributed as dist
        lib = load()
        rank, n = dist.get_rank(group), dist.get_world_size(group)
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib.rl_comm_unique_id(C.cast(buf, vp)), "rl_comm_unique_id")
        t = torch.tensor(bytearray(buf), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = bytes(t.cpu().tolist())
        h = vp()
        _check(lib.rl_comm_init(C.byref(h), raw, n, rank), "rl_comm_init")
        return cls(h.value, n, rank)

    @classmethod
    def local(cls):
        """A single-rank communicator (P = 1: the vocab-parallel path on one GPU, the all-reduce
        a no-op sum) without a torch process group."""
        lib = load()
        buf = (C.c_uint8 * 128)()
        _check(lib.rl_comm_unique_id(C.cast(buf, vp)), "rl_comm_unique_id")
        h = vp()
        _check(lib.rl_comm_init(C.byref(h), bytes(buf), 1, 0), "rl_comm_init")
        return cls(h.value, 1, 0)

    def split(self, color: int, key: int):
        lib = load()
        h = vp()
        _check(lib.rl_comm_split(self.handle, color, key, C.byref(h)), "rl_comm_split")
        if not h.value:
            return None
        n, r = i32(), i32()
        _check(lib.rl_comm_size(h.value, C.byref(n), C.byref(r)), "rl_comm_size")
        return Comm(h.value, n.value, r.value)

    def enable_peer_exchange(self, max_tokens: int) -> bool:
        """Collective: map every rank's exchange buffer (CUDA IPC over NVLink) so the fused
        vocab-parallel loss runs as one kernel per rank.  Returns False if P2P is unavailable."""
        st = load().rl_comm_enable_peer_exchange(self.handle, int(max_tokens))
        if st == 3:   # RL_ERR_UNSUPPORTED: keep the NCCL path
            return False
        _check(st, "rl_comm_enable_peer_exchange")
        return True

    def allreduce_f64(self, buf, stream=None):
        _check(load().rl_comm_allreduce_f64(self.handle, _dev(buf, "buf"), buf.numel(),
                                            _stream(stream)), "rl_comm_allreduce_f64")

    def destroy(self):
        if self.handle:
            _check(load().rl_comm_destroy(self.handle), "rl_comm_destroy")
            self.handle = None


def vocab_parallel_workspace_size(n_tokens, nranks) -> int:
    return load().rl_vocab_parallel_workspace_size(n_tokens, nranks)


def vocab_parallel_logprob(logits_shard, targets, vocab_offset, vocab_total, comm: Comm, logp_out,
                           workspace, lse_out=None, vocab_shard=None, inv_temperature=1.0,
                           old_logp=None, loss_mask=None, token_seq=None, seq_adv=None,
                           seq_version=None, seq_active=None, params: Optional[LossParams] = None,
                           dlogits_shard=None, stats=None, stream=None):
    lib = load()
    n, ld = logits_shard.shape
    Vr = ld if vocab_shard is None else vocab_shard
    p = params._c() if params is not None else None
    _check(lib.rl_vocab_parallel_logprob(
        _dev(logits_shard, "logits_shard"), _dtype_code(logits_shard), n, Vr, vocab_offset,
        vocab_total, ld, _dev(targets, "targets"), inv_temperature, comm.handle,
        _dev(logp_out, "logp_out"), _dev(lse_out, "lse_out"), _dev(old_logp, "old_logp"),
        _dev(loss_mask, "loss_mask"), _dev(token_seq, "token_seq"), _dev(seq_adv, "seq_adv"),
        _dev(seq_version, "seq_version"), _dev(seq_active, "seq_active"),
        C.byref(p) if p is not None else None, _dev(dlogits_shard, "dlogits_shard"),
        _dev(stats, "stats"), _dev(workspace, "workspace"),
        workspace.numel() * workspace.element_size(), _stream(stream)),
        "rl_vocab_parallel_logprob")


# ----------------------------------------------------------------------------- (6) M2PO
def m2po_workspace_size(n_tokens: int, nranks: int = 1) -> int:
    return load().rl_m2po_workspace_size(n_tokens, nranks)


def m2po_mask(logp, old_logp, mask_out, stats_out, workspace, tau=0.01, valid=None, comm=None, stream=None):
    """M2PO second-moment trust mask (reading M1): mask_out (CUDA uint8 [n]) gets 1 for the kept
    valid tokens; stats_out (CUDA float64 [5]) = (n_valid, n_masked, mean m before, after, n_kept).
    With ``comm`` the selection is global over its ranks (same n on every rank)."""
    lib = load()
    n = logp.numel()
    _check(lib.rl_m2po_mask(_dev(logp, "logp"), _dev(old_logp, "old_logp"), _dev(valid, "valid"), n, float(tau),
                            None if comm is None else comm.handle, _dev(mask_out, "mask_out"),
                            _dev(stats_out, "stats_out"), _dev(workspace, "workspace"),
                            workspace.numel() * workspace.element_size(), _stream(stream)), "rl_m2po_mask")


# ----------------------------------------------------------------------------- (7) delta scan
def delta_workspace_size(n_words: int) -> int:
    return load().rl_bf16_delta_workspace_size(n_words)


def delta_encode(prev, nxt, idx_out, word_out, count_out, workspace, stream=None):
    """Index-sorted (idx u32, word u16) of every position where the 16-bit words of ``prev`` and
    ``nxt`` (CUDA tensors of one 2-byte dtype, same numel) differ; count_out: CUDA uint64/int64 [1]."""
    lib = load()
    n = prev.numel()
    if nxt.numel() != n or prev.element_size() != 2 or nxt.element_size() != 2:
        raise RLError("prev/nxt must be 2-byte tensors of the same length")
    _check(lib.rl_bf16_delta_encode(_dev(prev, "prev"), _dev(nxt, "nxt"), n, _dev(idx_out, "idx_out"),
                                    _dev(word_out, "word_out"), idx_out.numel(), _dev(count_out, "count_out"),
                                    _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
                                    _stream(stream)), "rl_bf16_delta_encode")


def delta_apply(base, idx, words, count, bad_count, stream=None):
    """base[idx[j]] = words[j] for the first min(count, len(idx)) changes (in place)."""
    lib = load()
    _check(lib.rl_bf16_delta_apply(_dev(base, "base"), base.numel(), _dev(idx, "idx"), _dev(words, "words"),
                                   _dev(count, "count"), idx.numel(), _dev(bad_count, "bad_count"),
                                   _stream(stream)), "rl_bf16_delta_apply")


def lmhead_workspace_size(n_tokens, d, vocab):
    return int(load().rl_lmhead_workspace_size(int(n_tokens), int(d), int(vocab)))


def lmhead_logprob(hidden, weight, targets, logp_out, lse_out=None, inv_temperature=1.0, workspace=None,
                   stream=None):
    """Fused LM-head log-prob (NEXT 4, forward): logp_t = log_softmax((h W^T) * inv_T)[y_t] without
    materialising the logits.  hidden bf16 [N, d] and weight bf16 [V, d] (row strides may exceed d),
    targets int32 [N]; logp_out / lse_out float32 [N]; workspace: CUDA uint8 tensor of at least
    lmhead_workspace_size(N, d, V) bytes (None when that is 0)."""
    lib = load()
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise RLError("hidden [N, d] and weight [V, d] must share d")
    if hidden.element_size() != 2 or weight.element_size() != 2:
        raise RLError("hidden / weight must be bf16")
    if hidden.stride(1) != 1 or weight.stride(1) != 1:
        raise RLError("hidden / weight rows must be contiguous")
    n, d = hidden.shape
    _check(lib.rl_lmhead_logprob(_dev(hidden, "hidden"), hidden.stride(0), _dev(weight, "weight"), weight.stride(0),
                                 n, d, weight.shape[0], _dev(targets, "targets"), float(inv_temperature),
                                 _dev(logp_out, "logp_out"), _dev(lse_out, "lse_out") if lse_out is not None else None,
                                 _dev(workspace, "workspace") if workspace is not None else None,
                                 workspace.numel() * workspace.element_size() if workspace is not None else 0,
                                 _stream(stream)), "rl_lmhead_logprob")


def lmhead_loss_bwd_workspace_size(chunk_tokens, vocab):
    return int(load().rl_lmhead_loss_bwd_workspace_size(int(chunk_tokens), int(vocab)))


def lmhead_loss_bwd(hidden, weight, targets, lse, scale, workspace, dhidden=None, dweight=None,
                    inv_temperature=1.0, accumulate=False, stream=None):
    """NEXT 4 backward: dhidden = G W, dweight (+)= G^T h with G = s (softmax(h W^T inv_T) - onehot),
    the logits recomputed on the tensor cores, never stored (G is written per token chunk into
    ``workspace``).  hidden bf16 [N, d], weight bf16 [V, d]; dhidden / dweight float32 [N, d] / [V, d]."""
    lib = load()
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.shape[1] != weight.shape[1]:
        raise RLError("hidden [N, d] and weight [V, d] must share d")
    n, d = hidden.shape
    V = weight.shape[0]
    for t, nm, shp in ((dhidden, "dhidden", (n, d)), (dweight, "dweight", (V, d))):
        if t is not None and (t.dtype.itemsize != 4 or tuple(t.shape) != shp or t.stride(1) != 1):
            raise RLError(f"{nm} must be float32 {shp} with contiguous rows")
    _check(lib.rl_lmhead_loss_bwd(
        _dev(hidden, "hidden"), hidden.stride(0), _dev(weight, "weight"), weight.stride(0), n, d, V,
        _dev(targets, "targets"), _dev(lse, "lse"), _dev(scale, "scale"), float(inv_temperature),
        _dev(dhidden, "dhidden"), dhidden.stride(0) if dhidden is not None else d,
        _dev(dweight, "dweight"), dweight.stride(0) if dweight is not None else d,
        F_STATS_ACCUMULATE if accumulate else 0, _dev(workspace, "workspace"),
        workspace.numel() * workspace.element_size(), _stream(stream)), "rl_lmhead_loss_bwd")


def policy_loss_from_logp_workspace_size(n_tokens):
    return int(load().rl_policy_loss_from_logp_workspace_size(int(n_tokens)))


def policy_loss_from_logp(logp, targets, old_logp, token_seq, seq_adv, params: LossParams, stats, workspace,
                          vocab, loss_mask=None, seq_version=None, seq_active=None, scale_out=None,
                          clipped_out=None, stream=None):
    """c4–c7 from per-token log-probs (e.g. lmhead_logprob's): loss statistics into ``stats``
    (CUDA float64, STATS_FIELDS order) and the gradient scale s_t into ``scale_out``."""
    lib = load()
    if stats.numel() < len(STATS_FIELDS):
        raise RLError(f"stats needs {len(STATS_FIELDS)} float64 elements")
    p = params._c()
    _check(lib.rl_policy_loss_from_logp(
        _dev(logp, "logp"), logp.numel(), int(vocab), _dev(targets, "targets"), _dev(old_logp, "old_logp"),
        _dev(loss_mask, "loss_mask"), _dev(token_seq, "token_seq"), _dev(seq_adv, "seq_adv"),
        _dev(seq_version, "seq_version"), _dev(seq_active, "seq_active"), C.byref(p),
        _dev(scale_out, "scale_out"), _dev(clipped_out, "clipped_out"), _dev(stats, "stats"),
        _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(), _stream(stream)),
        "rl_policy_loss_from_logp")

