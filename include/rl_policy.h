/*
 * rl_policy.h — C ABI of the B200-native trainer policy-loss hot path of
 * AstraFlow (arXiv 2605.15565).
 *
 * The path (BASELINE.json north_star): per consumed rollout
 * (mini-)batch, (1) GRPO group-relative advantages over each prompt's response
 * group ("group-level reward normalization"; 8 rollouts per
 * prompt; GRPO), (2) sequence/version bookkeeping
 * ("max staleness 8"), (3) per-token log-probs of the
 * sampled tokens (log-softmax over V, then gather), (4) the token-level clipped
 * importance-ratio surrogate against the behaviour log-probs recorded with the
 * rollout's weight version (PPO; "4 PPO mini-batches")
 * and its fused backward dL/dlogits = scale*(softmax - onehot), (5) the
 * vocab-parallel variant with a cross-GPU combine of (max, sum-exp, target logit).
 * The exact definitions (and every reading where the paper is silent) are in
 * DESIGN.md §3; the fp64 CPU oracle in oracle/ implements them.
 *
 * Conventions (all entry points):
 *  - Pointers documented "device" must be CUDA device pointers on the current
 *    device; "host" pointers are read during the call only.  The caller owns every
 *    buffer; the library allocates nothing on the hot path (scratch comes from the
 *    caller's workspace, sized by the *_workspace_size functions).  The only
 *    library-owned object is rl_comm (an NCCL communicator).
 *  - Calls enqueue work on `stream` (a cudaStream_t; NULL = legacy default stream)
 *    and return without synchronising.  Outputs are valid after the stream syncs.
 *  - Errors: host-detectable problems (NULL required pointer, negative size, bad
 *    enum, ld < vocab, misalignment) return a non-OK status and enqueue NOTHING.
 *    A failed launch returns RL_ERR_CUDA; NCCL failures RL_ERR_NCCL.
 *    rl_last_error() gives a thread-local human-readable detail.
 *    Data errors found on the device never trap: they are counted in the stats /
 *    counts outputs (target >= vocab -> logp NaN and the token is masked; negative
 *    staleness -> the sequence is masked).
 *  - Logits rows are row-major [n_tokens, ld], ld >= vocab, with the row start
 *    16-byte aligned (base pointer 16-B aligned and ld % 8 == 0 for bf16,
 *    ld % 4 == 0 for f32).  Row t is the distribution that scored targets[t] (the
 *    next-token shift is the caller's job).  Columns [vocab, ld) are never read or
 *    written.
 *  - dlogits may alias logits exactly (same pointer, same ld) for in-place use;
 *    partial overlap is undefined.  Every row of dlogits is written (exact zeros
 *    for masked rows).
 *  - All calls are deterministic: same inputs -> bitwise-identical outputs.
 */
#ifndef RL_POLICY_H_
#define RL_POLICY_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RL_POLICY_ABI_VERSION 2

typedef void* rl_stream; /* cudaStream_t */

typedef enum {
  RL_OK = 0,
  RL_ERR_INVALID_ARGUMENT = 1, /* NULL required pointer, negative size, bad enum, ld < vocab */
  RL_ERR_ALIGNMENT = 2,        /* logits/dlogits not 16-B aligned, or ld not a multiple of 16 B */
  RL_ERR_UNSUPPORTED = 3,      /* dtype / device not supported (requires sm_100) */
  RL_ERR_WORKSPACE = 4,        /* workspace NULL or smaller than *_workspace_size() */
  RL_ERR_CUDA = 5,             /* a CUDA launch or runtime call failed */
  RL_ERR_NCCL = 6              /* an NCCL call failed */
} rl_status;

typedef enum { RL_F32 = 0, RL_BF16 = 1 } rl_dtype; /* logits and dlogits share the dtype */

/* Group std estimator (reading Z2/Z4): unbiased (n-1), biased (n), or none (mean-centering only). */
typedef enum { RL_STD_UNBIASED = 0, RL_STD_BIASED = 1, RL_STD_NONE = 2 } rl_std_mode;

/* Loss aggregation (reading Z8): global token mean, sequence-mean of token-means, or plain sum. */
typedef enum { RL_AGG_TOKEN_MEAN = 0, RL_AGG_SEQ_MEAN_TOKEN_MEAN = 1, RL_AGG_SUM = 2 } rl_loss_agg;

/* rl_loss_params.flags */
#define RL_F_STATS_ACCUMULATE 0x1u /* add into *stats instead of overwriting it */
#define RL_F_SKIP_MASKED_READS 0x2u /* masked rows: do not read logits (logp_out = 0), only write zeros */
#define RL_F_ENTROPY 0x4u /* also sum the per-token entropy H_t = lse - sum_v p_v z_v of valid tokens into
                             stats->entropy_sum (rl_policy_loss_fwd_bwd; reading N3) */

#define RL_STALE_HIST_BINS 16

/* Device-resident batch counts written by rl_seq_bookkeeping (all integer-valued doubles,
 * so they can be summed across ranks with one fp64 all-reduce). */
typedef struct {
  double active_tokens;   /* sum of valid_t */
  double stale_masked;    /* tokens (mask=1, 0<=y<V) dropped only because staleness > max_staleness */
  double neg_staleness;   /* SEQUENCES with trainer_version - seq_version < 0 (counted error) */
  double bad_targets;     /* tokens with y >= vocab (counted error) */
  double stale_hist[RL_STALE_HIST_BINS]; /* sequences by staleness min(s,15); negative not binned */
} rl_batch_counts;

/* Device-resident loss statistics written by rl_policy_loss_fwd_bwd (all doubles). */
typedef struct {
  double loss_sum;      /* sum_t valid_t * w_t * L_t  (= the loss for TOKEN_MEAN / SEQ_MEAN) */
  double active_tokens; /* sum_t valid_t */
  double weight_sum;    /* sum_t valid_t * w_t */
  double ratio_sum;     /* sum_t valid_t * r_t */
  double clipped_low;   /* valid tokens with A < 0 and r < 1 - eps_low  */
  double clipped_high;  /* valid tokens with A > 0 and r > 1 + eps_high */
  double clamped;       /* valid tokens whose log-ratio hit +-log_ratio_clamp */
  double stale_masked;  /* tokens (mask=1, 0<=y<V) dropped because staleness > max_staleness */
  double bad_targets;   /* tokens with y >= vocab */
  double neg_staleness; /* TOKENS whose sequence has negative staleness */
  double kl_sum;        /* sum_t valid_t * w_t * KL_t (k3 vs ref_logp; 0 unless kl_coef != 0), reading N1 */
  double entropy_sum;   /* sum_t valid_t * H_t (only with RL_F_ENTROPY), reading N3 */
} rl_loss_stats;
#define RL_LOSS_STATS_N 12

typedef struct {
  float clip_eps_low;    /* default 0.2 (reading Z9) */
  float clip_eps_high;   /* default 0.2 */
  float inv_temperature; /* default 1.0 (rollout temperature 1.0) */
  float log_ratio_clamp; /* default 20: r = exp(clamp(logp - old, -c, c)) (reading Z11) */
  float grad_scale;      /* extra multiplier on dlogits only, default 1 */
  int32_t agg;           /* rl_loss_agg, default RL_AGG_TOKEN_MEAN */
  int32_t trainer_version; /* current trainer weight version (staleness = this - seq_version) */
  int32_t max_staleness;   /* < 0 disables the staleness mask; 8 per PAPER.md:776 */
  int32_t global_num_seqs; /* S_global for RL_AGG_SEQ_MEAN_TOKEN_MEAN */
  uint32_t flags;          /* RL_F_* */
  double global_active_tokens;     /* N_active over ALL ranks/chunks of this (mini-)batch;
                                      used iff active_tokens_dev == NULL */
  const double* active_tokens_dev; /* device pointer to the same count (e.g. &counts->active_tokens
                                      after rl_comm_allreduce_f64); NULL -> use the host value */
  /* NEXT-2 terms (readings N1, N2), default off: */
  float kl_coef;                   /* beta: L_t += beta * KL_t, KL_t = e^{ref-logp} - (ref-logp) - 1 (k3);
                                      PAPER.md:572 "fixed KL penalty coefficient of 10^-3" */
  const float* ref_logp;           /* device [n_tokens] reference-policy log-probs; required iff kl_coef != 0 */
  const float* prox_logp;          /* device [n_tokens] proximal-policy log-probs or NULL: the clipped ratio is
                                      pi/pi_prox and the surrogate is weighted by pi_prox/pi_behav (old_logp),
                                      no gradient through that weight (decoupled ratio) */
} rl_loss_params;

/* ---------------------------------------------------------------- misc */
const char* rl_status_string(rl_status s);
const char* rl_last_error(void); /* thread-local detail of the last non-OK return ("" if none) */
int32_t rl_abi_version(void);    /* RL_POLICY_ABI_VERSION */
void rl_loss_params_default(rl_loss_params* p); /* fills the defaults above (host pointer) */

/* ---------------------------------------------------------------- (1) advantages
 * GRPO group-relative advantages, c1 of DESIGN.md §3 (PAPER.md:572 group-level reward
 * normalization; SPEC.md:56-64 zero-variance predicate; PAPER.md:572 batch-level
 * advantage normalisation as option).  Bit-exact to the fp64 definition:
 *   zero_var[g] = all rewards of g bitwise-equal (singletons included) -> A_i = +0
 *   else mu = sequential sum / n; q = sequential sum of (r_i-mu)^2;
 *        sigma = sqrt(q/(n-1)) | sqrt(q/n); A_i = (r_i - mu)/(sigma + eps) | (r_i - mu)
 *   optional batch norm (token-weighted by seq_weight[i]), then float32 RNE.
 * rewards   device f64 [n_seq], group-major (group g = sequences cu_groups[g]..cu_groups[g+1]-1)
 * cu_groups device i32 [n_groups+1], cu_groups[0] = 0, cu_groups[n_groups] = n_seq
 * seq_weight device i32 [n_seq] active tokens per sequence; required iff batch_norm != 0
 * workspace device, >= rl_group_advantage_workspace_size(n_seq) bytes; required iff batch_norm
 * adv_out   device f32 [n_seq]
 * zero_var_out device u8 [n_groups] or NULL: 1 = zero variance, 0 = not, 2 = INVALID group
 *           (empty or out of range — SPEC.md:60 invalid-argument; its members are left untouched)
 */
size_t rl_group_advantage_workspace_size(int32_t n_seq);
rl_status rl_group_advantage(const double* rewards, const int32_t* cu_groups, int32_t n_groups,
                             int32_t n_seq, int32_t std_mode, double eps, int32_t batch_norm,
                             double bn_eps, const int32_t* seq_weight, void* workspace,
                             size_t workspace_bytes, float* adv_out, uint8_t* zero_var_out,
                             rl_stream stream);

/* ---------------------------------------------------------------- (2) bookkeeping
 * Sequence / version bookkeeping, c2 of DESIGN.md §3 (PAPER.md:160 model version,
 * PAPER.md:776 max staleness, SPEC.md:142 worked example 20-11=9>8 -> masked).
 * cu_seqlens   device i32 [n_seq+1], cu_seqlens[0] = 0, cu_seqlens[n_seq] = n_tokens
 * loss_mask    device u8 [n_tokens] (NULL = all ones); targets device i32 [n_tokens]
 *              (y < 0 = ignored, y >= vocab = counted error)
 * seq_version  device i32 [n_seq] behaviour weight version, or NULL (staleness 0)
 * seq_adv      device f32 [n_seq] or NULL; if given, adv_token_out[t] = seq_adv[token_seq[t]]
 * Outputs (device): token_seq_out i32 [n_tokens] (required); seq_active_out i32 [n_seq]
 *   (required; valid tokens per sequence); seq_staleness_out i32 [n_seq] or NULL;
 *   adv_token_out f32 [n_tokens] or NULL; valid_out u8 [n_tokens] or NULL;
 *   counts_out rl_batch_counts or NULL (overwritten).
 */
rl_status rl_seq_bookkeeping(const int32_t* cu_seqlens, int32_t n_seq, int64_t n_tokens,
                             const uint8_t* loss_mask, const int32_t* targets, int64_t vocab,
                             const int32_t* seq_version, int32_t trainer_version,
                             int32_t max_staleness, const float* seq_adv,
                             int32_t* token_seq_out, int32_t* seq_active_out,
                             int32_t* seq_staleness_out, float* adv_token_out, uint8_t* valid_out,
                             rl_batch_counts* counts_out, rl_stream stream);

/* ---------------------------------------------------------------- (3) token log-probs
 * c3 of DESIGN.md §3 (north_star: log-softmax over the vocabulary then gather):
 *   z = x * inv_temperature; lse = max z + ln sum exp(z - max z); logp = z_y - lse.
 * Read-only single streaming pass over the logits (no grad; for behaviour/proximal/
 * reference recompute).  y < 0 -> logp 0; y >= vocab -> logp NaN and counted.
 * logits device [n_tokens, ld] of dtype; targets device i32 [n_tokens]
 * logp_out device f32 [n_tokens]; lse_out device f32 [n_tokens] or NULL
 * bad_target_count device f64 scalar or NULL (ADDED to, not overwritten)
 */
rl_status rl_token_logprob(const void* logits, int32_t dtype, int64_t n_tokens, int64_t vocab,
                           int64_t ld, const int32_t* targets, float inv_temperature,
                           float* logp_out, float* lse_out, double* bad_target_count,
                           rl_stream stream);

/* ---------------------------------------------------------------- (4) fused loss fwd+bwd
 * c3–c7 of DESIGN.md §3 in ONE streaming pass over the logits (logits read once from
 * HBM, dlogits written once):
 *   valid_t = mask_t && 0 <= y_t < V && 0 <= staleness(seq) (<= max_staleness if >= 0)
 *   r = exp(clamp(logp - old_logp, +-c)); L_t = -min(r A, clip(r, 1-eps_l, 1+eps_h) A)
 *   w_t = 1/N_active | 1/(S_global L_seq) | 1;  s_t = w A r inv_T grad_scale if unclipped
 *   and unclamped else 0;  dlogits[t,v] = s_t * (softmax(z_t)_v - [v == y_t])
 * logits   device [n_tokens, ld] (dtype); dlogits device [n_tokens, ld] (same dtype), may == logits
 * targets  device i32 [n_tokens]; old_logp device f32 [n_tokens] (behaviour log-probs)
 * loss_mask device u8 [n_tokens] or NULL (all ones)
 * token_seq device i32 [n_tokens] sequence index into the per-sequence arrays
 * seq_adv   device f32 [n_seq] (from rl_group_advantage); seq_version device i32 [n_seq] or NULL
 * seq_active device i32 [n_seq] (required for RL_AGG_SEQ_MEAN_TOKEN_MEAN, else may be NULL)
 * p         HOST pointer to the parameters (read during the call only)
 * logp_out  device f32 [n_tokens] or NULL; clipped_out device u8 [n_tokens] or NULL
 *           (0 none, 1 low, 2 high)
 * stats     device rl_loss_stats (overwritten, or added to with RL_F_STATS_ACCUMULATE)
 * workspace device, >= rl_policy_loss_workspace_size(n_tokens, vocab, dtype) bytes
 */
size_t rl_policy_loss_workspace_size(int64_t n_tokens, int64_t vocab, int32_t dtype);
rl_status rl_policy_loss_fwd_bwd(const void* logits, int32_t dtype, int64_t n_tokens,
                                 int64_t vocab, int64_t ld, const int32_t* targets,
                                 const float* old_logp, const uint8_t* loss_mask,
                                 const int32_t* token_seq, const float* seq_adv,
                                 const int32_t* seq_version, const int32_t* seq_active,
                                 const rl_loss_params* p, void* dlogits, float* logp_out,
                                 uint8_t* clipped_out, rl_loss_stats* stats, void* workspace,
                                 size_t workspace_bytes, rl_stream stream);

/* Same as rl_policy_loss_fwd_bwd but every array argument is a HOST pointer (pinned or
 * pageable); the library streams the rows through device staging buffers taken from the
 * caller's DEVICE workspace (>= rl_policy_loss_host_workspace_size()), overlapping the
 * host->device copy of chunk k+1, the kernel on chunk k and the device->host copy of
 * chunk k-1.  *stats_host is written (or accumulated) when the call returns; this call
 * synchronises `stream`.  dlogits_host may be NULL (gradient discarded). */
size_t rl_policy_loss_host_workspace_size(int64_t chunk_tokens, int64_t vocab, int64_t ld,
                                          int32_t dtype, int32_t n_seq);
rl_status rl_policy_loss_fwd_bwd_host(const void* logits_host, int32_t dtype, int64_t n_tokens,
                                      int64_t vocab, int64_t ld, const int32_t* targets_host,
                                      const float* old_logp_host, const uint8_t* loss_mask_host,
                                      const int32_t* token_seq_host, const float* seq_adv_host,
                                      const int32_t* seq_version_host,
                                      const int32_t* seq_active_host, int32_t n_seq,
                                      const rl_loss_params* p, void* dlogits_host,
                                      float* logp_out_host, rl_loss_stats* stats_host,
                                      int64_t chunk_tokens, void* workspace,
                                      size_t workspace_bytes, rl_stream stream);

/* ---------------------------------------------------------------- (5) multi-GPU
 * rl_comm wraps an NCCL communicator (NVLink 5 / NVSwitch).  Bootstrap: rank 0 calls
 * rl_comm_unique_id, the 128 bytes are broadcast by the caller (e.g. over the torch
 * process group), then every rank calls rl_comm_init on its current device.
 */
typedef struct rl_comm rl_comm;
rl_status rl_comm_unique_id(void* out_128_bytes_host);
rl_status rl_comm_init(rl_comm** out, const void* unique_id_host, int32_t nranks, int32_t rank);
rl_status rl_comm_split(rl_comm* parent, int32_t color, int32_t key, rl_comm** out); /* per-policy groups */
rl_status rl_comm_destroy(rl_comm* c);
rl_status rl_comm_size(const rl_comm* c, int32_t* nranks, int32_t* rank);
/* In-place sum all-reduce of n doubles (device) — used for rl_batch_counts (before the loss,
 * so every rank sees N_active_global) and rl_loss_stats (after). */
rl_status rl_comm_allreduce_f64(rl_comm* c, double* buf, size_t n, rl_stream stream);

/* Collective (every rank of `c`, same max_tokens): allocate this rank's peer-exchange buffer for
 * vocab-parallel calls of up to max_tokens rows and map every peer's buffer into this process
 * (CUDA IPC over NVLink / NVSwitch; handles exchanged with one NCCL all-gather).  Enabled only if
 * EVERY rank mapped every peer (an NCCL min-reduction of the per-rank result), so all ranks take
 * the same path.  Afterwards rl_vocab_parallel_logprob with the fused loss runs as ONE kernel per
 * rank that sends each row's shard record (log2-domain lse of the shard, target logit) to every
 * rank as two 8-byte words tagged with the call's epoch (slots double-buffered by epoch parity)
 * and polls the peers' records inside the kernel: vp_ring_kernel (slices re-read from L2: a ~14 us
 * exchange window that absorbs the cross-GPU lockstep jitter); on a single rank
 * vp_cache_kernel for bf16 shards of <= 4,928 whole 16-B vectors (row slices held in registers:
 * logits read once, one exp per element).  A rank that never publishes makes its peers
 * trap after 30 s (RL_ERR_CUDA) instead of hanging.  Returns RL_ERR_UNSUPPORTED (and leaves the
 * NCCL path in use on every rank) if a peer is not P2P-accessible; > 8 ranks are unsupported.
 * The buffers are released by rl_comm_destroy; calling it again re-maps (collective). */
rl_status rl_comm_enable_peer_exchange(rl_comm* c, int64_t max_tokens);

/* Vocab-parallel log-prob (+ optional fused loss/grad on the local shard), c8 of DESIGN.md §3.
 * Each rank holds the columns [vocab_offset, vocab_offset + vocab_shard) of every row.
 * With rl_comm_enable_peer_exchange and the fused loss requested: one kernel per rank (records
 *   exchanged through peer memory, see above: 2 HBM units per element).  Otherwise:
 * Phase 1 (kernel): per row (m_r, s_r, t_y-if-owned) over the local shard.
 * Phase 2 (NCCL all-gather over NVLink of the 3 floats per row).
 * Phase 3 (kernel): M = max m_r, S = sum s_r 2^(m_r - M), lse, logp (identical on all ranks);
 *   if old_logp != NULL also the loss terms (counted once, on the rank owning y) and the
 *   local dlogits shard s_t*(softmax - onehot) for the shard's columns.
 * targets are GLOBAL ids.  logp_out / lse_out device f32 [n_tokens] (all ranks).
 * Loss inputs as in rl_policy_loss_fwd_bwd; dlogits_shard may alias logits_shard.
 * stats: per-rank partial; sum over ranks with rl_comm_allreduce_f64 to get the batch loss.
 * workspace >= rl_vocab_parallel_workspace_size(n_tokens, nranks).
 */
size_t rl_vocab_parallel_workspace_size(int64_t n_tokens, int32_t nranks);
rl_status rl_vocab_parallel_logprob(const void* logits_shard, int32_t dtype, int64_t n_tokens,
                                    int64_t vocab_shard, int64_t vocab_offset,
                                    int64_t vocab_total, int64_t ld, const int32_t* targets,
                                    float inv_temperature, rl_comm* comm, float* logp_out,
                                    float* lse_out, const float* old_logp,
                                    const uint8_t* loss_mask, const int32_t* token_seq,
                                    const float* seq_adv, const int32_t* seq_version,
                                    const int32_t* seq_active, const rl_loss_params* p,
                                    void* dlogits_shard, rl_loss_stats* stats, void* workspace,
                                    size_t workspace_bytes, rl_stream stream);

/* ---------------------------------------------------------------- (6) M2PO mask (NEXT 1)
 * M2PO second-moment trust masking, reading M1 of DESIGN.md §3 ("M2PO ... with
 * m²-threshold 0.01"; the paper gives no formula).  For every token with valid != 0,
 * m_t = (logp_t - old_logp_t)^2 in fp32; the fewest largest-m tokens are masked so that the mean
 * m of the kept valid tokens is <= tau (ties of equal m: the lower token index is masked first).
 * With comm != NULL the selection is GLOBAL over the ranks of comm (global token index =
 * rank * n_tokens + t: every rank must pass the same n_tokens — pad with valid = 0) and every
 * rank derives the same cut; comm == NULL selects over this call's tokens.
 *   logp, old_logp  device float [n_tokens] (logp e.g. from rl_token_logprob)
 *   valid           device u8 [n_tokens] or NULL (= all valid)
 *   mask_out        device u8 [n_tokens]: 1 = kept valid token, 0 = masked or invalid.  Use it as
 *                   the loss_mask of rl_policy_loss_fwd_bwd (with clip_eps_* large: M2PO's
 *                   surrogate is unclipped) and &stats_out[4] as its active_tokens_dev
 *   stats_out       device double[5]: (n_valid, n_masked, mean m of the valid tokens,
 *                   mean m of the kept tokens, n_kept), over all ranks of comm
 *   workspace       device, >= rl_m2po_workspace_size(n_tokens, nranks) bytes
 * Errors: RL_ERR_INVALID_ARGUMENT (n_tokens < 0, tau < 0 or NaN, NULL arrays), RL_ERR_UNSUPPORTED
 * (n_tokens * nranks >= 2^31), RL_ERR_WORKSPACE, RL_ERR_NCCL.  Deterministic (radix sort, fixed
 * scan, order-free max). */
size_t rl_m2po_workspace_size(int64_t n_tokens, int32_t nranks);
rl_status rl_m2po_mask(const float* logp, const float* old_logp, const uint8_t* valid, int64_t n_tokens,
                       float tau, rl_comm* comm, uint8_t* mask_out, double* stats_out, void* workspace,
                       size_t workspace_bytes, rl_stream stream);

/* ---------------------------------------------------------------- (7) bf16 delta scan (NEXT 3)
 * Bit-exact diff of two weight snapshots of n_words 16-bit words (
 * "exactly the indices whose 16-bit words differ"), as index-sorted
 * (u32 index, u16 new word) pairs, and its inverse.  Words are opaque bit patterns (+0 != -0).
 * encode: prev, next  device, 16-B aligned, n_words in [0, 2^32) (larger models: per tensor)
 *         idx_out, word_out  device [capacity]: the first min(count, capacity) changes
 *         count_out  device u64: the number of changes (may exceed capacity: then only the
 *                    first `capacity` are written — the caller re-runs with a larger buffer)
 *         workspace  device, >= rl_bf16_delta_workspace_size(n_words) bytes (per 16,384-word
 *                    tile: counts, a 2 KB change bitmask and a 4 KB staging slot; ~0.38 B/word)
 *         Each snapshot read once; a tile's changes are staged compacted and copied to their
 *         sorted position (dense tiles: bitmask + gather from next); deterministic output.
 * apply:  base[idx[j]] = word[j] for j < min(*count, capacity); indices >= n_words are skipped and
 *         counted in *bad_index_count (device u64, added to).
 * Errors: RL_ERR_INVALID_ARGUMENT (sizes, NULL arrays), RL_ERR_ALIGNMENT, RL_ERR_WORKSPACE. */
size_t rl_bf16_delta_workspace_size(int64_t n_words);
rl_status rl_bf16_delta_encode(const void* prev, const void* next, int64_t n_words, uint32_t* idx_out,
                               uint16_t* word_out, int64_t capacity, unsigned long long* count_out,
                               void* workspace, size_t workspace_bytes, rl_stream stream);
rl_status rl_bf16_delta_apply(void* base, int64_t n_words, const uint32_t* idx, const uint16_t* words,
                              const unsigned long long* count, int64_t capacity,
                              unsigned long long* bad_index_count, rl_stream stream);

/* ---------------------------------------------------------------- (8) fused LM-head log-prob (NEXT 4)
 * SURVEY.md §8(f) NEXT 4 ("Fused LM-head GEMM + loss (tcgen05, logits never materialised) ... it
 * takes hidden states and W"), forward half: c3 of §8(c) on x = (h W^T) * inv_T without writing
 * the [n_tokens, vocab] logits (each 128 x 256 logits tile exists only in tensor memory).
 *   hidden     device bf16 [n_tokens, ld_hidden] row-major (the first d columns are h), 16-B aligned
 *   weight     device bf16 [vocab, ld_weight] row-major LM-head weight (the first d columns), 16-B aligned
 *   ld_*       row strides in elements, >= d, multiples of 8
 *   targets    device i32 [n_tokens]: y < 0 -> logp 0; y >= vocab -> logp NaN (as rl_token_logprob)
 *   logp_out   device f32 [n_tokens];  lse_out  device f32 [n_tokens] or NULL (natural log)
 *   workspace  device, >= rl_lmhead_workspace_size(n_tokens, d, vocab) bytes (per-vocabulary-split
 *              row records, 16 B per token per split; 0 when one split is used)
 * fp32 accumulation of bf16 products on the tensor cores (tcgen05.mma kind::f16), fp32 softmax.
 * Errors: RL_ERR_INVALID_ARGUMENT (sizes, NULL, inv_temperature <= 0), RL_ERR_ALIGNMENT,
 * RL_ERR_UNSUPPORTED (n_tokens, d or vocab >= 2^31), RL_ERR_WORKSPACE, RL_ERR_CUDA (tensor-map
 * encoding, launch).
 * Deterministic: fixed K order per tile, fixed tile order per row. */
size_t rl_lmhead_workspace_size(int64_t n_tokens, int64_t d, int64_t vocab);
rl_status rl_lmhead_logprob(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                            int64_t n_tokens, int64_t d, int64_t vocab, const int32_t* targets,
                            float inv_temperature, float* logp_out, float* lse_out, void* workspace,
                            size_t workspace_bytes, rl_stream stream);

/* ---------------------------------------------------------------- (8b) LM-head loss backward (NEXT 4)
 * The backward half of NEXT 4: the gradients of the policy loss through the LM head x = h W^T,
 *     G[t, v] = s_t (softmax(x_t inv_T)_v - [v == y_t])      (c7 of SURVEY.md §8(c); s_t from
 *                                                           rl_policy_loss_from_logp, lse_t from
 *                                                           rl_lmhead_logprob)
 *     dhidden = G W            [n_tokens, d]   (overwritten)
 *     dweight = G^T h          [vocab, d]      (overwritten, or added to with RL_F_STATS_ACCUMULATE)
 * without the logits ever existing in memory: per chunk of C tokens a tcgen05 kernel recomputes each
 * 128 x 256 logits tile in tensor memory and writes G in bf16 (one rounding) into the workspace, then
 * two GEMMs consume it (cuBLAS, bf16 x bf16 -> fp32 accumulate; plain library GEMMs).
 *   hidden, weight, ld_*, n_tokens, d, vocab, inv_temperature: as rl_lmhead_logprob
 *   targets    device i32 [n_tokens] (y outside [0, vocab): G row 0)
 *   lse        device f32 [n_tokens] natural-log lse of x_t inv_T (rl_lmhead_logprob's lse_out)
 *   scale      device f32 [n_tokens] s_t (rl_policy_loss_from_logp's scale_out; 0 -> G row 0)
 *   dhidden    device f32 [n_tokens, ld_dhidden] or NULL;  dweight  device f32 [vocab, ld_dweight] or NULL
 *   flags      RL_F_STATS_ACCUMULATE: dweight += (gradient accumulation over micro-batches)
 *   workspace  device, 16-B aligned; C = workspace_bytes / (2 * round_up(vocab, 8)) rounded down to a
 *              multiple of 128 tokens per chunk (>= min(n_tokens, 128)); see
 *              rl_lmhead_loss_bwd_workspace_size(chunk_tokens, vocab)
 * Errors: RL_ERR_INVALID_ARGUMENT (sizes, strides, NULL, neither output), RL_ERR_ALIGNMENT,
 * RL_ERR_WORKSPACE, RL_ERR_UNSUPPORTED (>= 2^31 sizes, not sm_100), RL_ERR_CUDA (tensor map, cuBLAS).
 * Deterministic (fixed chunk order; cuBLAS without atomics). */
size_t rl_lmhead_loss_bwd_workspace_size(int64_t chunk_tokens, int64_t vocab);
rl_status rl_lmhead_loss_bwd(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                             int64_t n_tokens, int64_t d, int64_t vocab, const int32_t* targets, const float* lse,
                             const float* scale, float inv_temperature, float* dhidden, int64_t ld_dhidden,
                             float* dweight, int64_t ld_dweight, uint32_t flags, void* workspace,
                             size_t workspace_bytes, rl_stream stream);

/* ---------------------------------------------------------------- (9) loss from log-probs
 * c4–c7 of SURVEY.md §8(c) (PPO clipped surrogate; with the NEXT 2 terms of
 * rl_loss_params) evaluated from per-token log-probs instead of logits: the loss statistics and
 * the per-token gradient scale s_t of dL/dlogits = s_t (softmax − onehot) (c7), no dlogits write.
 * Used after rl_lmhead_logprob (NEXT 4: the LM-head loss forward without logits) and by callers
 * that already hold log-probs.  Same per-token decisions as rl_policy_loss_fwd_bwd.
 *   logp       device f32 [n_tokens] (c3 log-probs; read for valid tokens only)
 *   vocab      V (a target >= V is a counted bad target, masked)
 *   targets, old_logp, loss_mask, token_seq, seq_adv, seq_version, seq_active, p: as
 *              rl_policy_loss_fwd_bwd (RL_F_ENTROPY is rejected: the entropy needs the logits)
 *   scale_out  device f32 [n_tokens] or NULL: s_t (0 for invalid / clipped / clamped tokens)
 *   clipped_out device u8 [n_tokens] or NULL;  stats  device rl_loss_stats
 *   workspace  device, >= rl_policy_loss_from_logp_workspace_size(n_tokens) bytes
 * Errors: as rl_policy_loss_fwd_bwd; RL_ERR_UNSUPPORTED for RL_F_ENTROPY.  Deterministic. */
size_t rl_policy_loss_from_logp_workspace_size(int64_t n_tokens);
rl_status rl_policy_loss_from_logp(const float* logp, int64_t n_tokens, int64_t vocab, const int32_t* targets,
                                   const float* old_logp, const uint8_t* loss_mask, const int32_t* token_seq,
                                   const float* seq_adv, const int32_t* seq_version, const int32_t* seq_active,
                                   const rl_loss_params* p, float* scale_out, uint8_t* clipped_out,
                                   rl_loss_stats* stats, void* workspace, size_t workspace_bytes,
                                   rl_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* RL_POLICY_H_ */
