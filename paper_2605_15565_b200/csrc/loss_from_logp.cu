// (9) The clipped-surrogate loss from log-probs alone (c4–c7 of DESIGN.md §3 without the
// gradient write): per token the same token_epilogue every fused loss kernel runs, giving the
// loss statistics and the per-token gradient scale s_t of dL/dlogits = s_t (softmax − onehot).
// With rl_lmhead_logprob (NEXT 4 forward) this is the whole LM-head loss forward without logits;
// (s_t, lse_t) are what a fused LM-head backward consumes.
#include "loss_common.cuh"

namespace rl {

rl_status launch_stats_reduce(const double* partials, int n_ctas, rl_loss_stats* stats, bool accumulate,
                              cudaStream_t s);

constexpr int kLfThreads = 256;

__global__ void __launch_bounds__(kLfThreads) loss_from_logp_kernel(
    const float* __restrict__ logp, int64_t n, int64_t vocab, const int32_t* __restrict__ targets,
    const float* __restrict__ old_logp, const uint8_t* __restrict__ mask, const int32_t* __restrict__ token_seq,
    const float* __restrict__ seq_adv, const int32_t* __restrict__ seq_version, const int32_t* __restrict__ seq_active,
    const Knobs kn, float* __restrict__ scale_out, uint8_t* __restrict__ clipped_out, double* __restrict__ partials) {
  __shared__ double red[kLfThreads / 32][RL_LOSS_STATS_N];
  const double inv_tm = token_mean_inv(kn);
  Acc acc;
  acc.zero();
  for (int64_t t = blockIdx.x * (int64_t)kLfThreads + threadIdx.x; t < n; t += (int64_t)gridDim.x * kLfThreads) {
    const RowMeta mt = row_meta(t, vocab, targets, mask, token_seq, seq_version, kn.trainer_version,
                                kn.max_staleness);
    const float A = mt.valid ? seq_adv[mt.seq] : 0.f;
    const float old = mt.valid ? old_logp[t] : 0.f;
    float prox, ref;
    token_extra(kn, t, old, prox, ref);
    const float s = token_epilogue(mt, mt.valid ? logp[t] : 0.f, old, A, seq_active, inv_tm, kn, acc,
                                   clipped_out ? clipped_out + t : nullptr, prox, ref);
    if (scale_out) scale_out[t] = s;
  }
  // fixed-order block reduction: lanes by shuffle tree, warps in index order
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < RL_LOSS_STATS_N; ++i) {
    double v = acc.v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < RL_LOSS_STATS_N) {
    double v = 0.0;
    for (int w = 0; w < kLfThreads / 32; ++w) v += red[w][threadIdx.x];
    partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + threadIdx.x] = v;
  }
}

}  // namespace rl

extern "C" size_t rl_policy_loss_from_logp_workspace_size(int64_t n_tokens) {
  (void)n_tokens;
  return (size_t)rl::kMaxStatCtas * RL_LOSS_STATS_N * sizeof(double);
}

extern "C" rl_status rl_policy_loss_from_logp(const float* logp, int64_t n_tokens, int64_t vocab,
                                              const int32_t* targets, const float* old_logp,
                                              const uint8_t* loss_mask, const int32_t* token_seq,
                                              const float* seq_adv, const int32_t* seq_version,
                                              const int32_t* seq_active, const rl_loss_params* p,
                                              float* scale_out, uint8_t* clipped_out, rl_loss_stats* stats,
                                              void* workspace, size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (!p) return fail(RL_ERR_INVALID_ARGUMENT, "NULL params");
  if (n_tokens < 0 || vocab < 1) return fail(RL_ERR_INVALID_ARGUMENT, "n_tokens < 0 or vocab < 1");
  if (!(p->inv_temperature > 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be > 0");
  if (!(p->log_ratio_clamp >= 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "log_ratio_clamp must be >= 0");
  if (!(p->clip_eps_low >= 0.f) || !(p->clip_eps_high >= 0.f))
    return fail(RL_ERR_INVALID_ARGUMENT, "clip eps must be >= 0");
  if (p->agg < RL_AGG_TOKEN_MEAN || p->agg > RL_AGG_SUM) return fail(RL_ERR_INVALID_ARGUMENT, "bad agg %d", p->agg);
  if (p->agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN && !seq_active)
    return fail(RL_ERR_INVALID_ARGUMENT, "SEQ_MEAN_TOKEN_MEAN needs seq_active");
  if (p->flags & RL_F_ENTROPY) return fail(RL_ERR_UNSUPPORTED, "entropy needs the logits (rl_policy_loss_fwd_bwd)");
  if (p->kl_coef != 0.f && !p->ref_logp) return fail(RL_ERR_INVALID_ARGUMENT, "kl_coef != 0 needs ref_logp");
  if (!(p->kl_coef == p->kl_coef)) return fail(RL_ERR_INVALID_ARGUMENT, "kl_coef is NaN");
  if (!stats) return fail(RL_ERR_INVALID_ARGUMENT, "NULL stats");
  if (!workspace || workspace_bytes < rl_policy_loss_from_logp_workspace_size(n_tokens))
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes", rl_policy_loss_from_logp_workspace_size(n_tokens));
  cudaStream_t s = (cudaStream_t)stream;
  const bool accumulate = (p->flags & RL_F_STATS_ACCUMULATE) != 0;
  if (n_tokens == 0) {
    if (!accumulate && cudaMemsetAsync(stats, 0, sizeof(rl_loss_stats), s) != cudaSuccess)
      return check_launch("memset stats");
    return RL_OK;
  }
  if (!logp || !targets || !old_logp || !token_seq || !seq_adv)
    return fail(RL_ERR_INVALID_ARGUMENT, "NULL logp/targets/old_logp/token_seq/seq_adv");
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  const int grid = (int)std::min<int64_t>((n_tokens + kLfThreads - 1) / kLfThreads, 148 * 4);
  double* partials = (double*)workspace;
  loss_from_logp_kernel<<<grid, kLfThreads, 0, s>>>(logp, n_tokens, vocab, targets, old_logp, loss_mask, token_seq,
                                                    seq_adv, seq_version, seq_active, make_knobs(p), scale_out,
                                                    clipped_out, partials);
  rl_status st = check_launch("loss_from_logp_kernel");
  if (st != RL_OK) return st;
  return launch_stats_reduce(partials, grid, stats, accumulate, s);
}
