// Host-buffer entry point of the fused loss (rl_policy_loss_fwd_bwd_host): streams the rows
// from host memory through two device staging slots carved from the caller's workspace,
// overlapping H2D of chunk c+1, the fused kernel on chunk c and D2H of chunk c-1 on three
// streams.  Every step of the math runs in the same kernels as rl_policy_loss_fwd_bwd.
#include <algorithm>

#include "common.cuh"

namespace rl {

struct HostLayout {
  size_t logits, tok_i32, tok_f32, tok_u8, partial, stats, seq, total;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static HostLayout host_layout(int64_t chunk, int64_t ld, int32_t dtype, int32_t n_seq) {
  HostLayout L;
  const size_t eb = dtype == RL_BF16 ? 2 : 4;
  L.logits = al((size_t)chunk * ld * eb);
  L.tok_i32 = al((size_t)chunk * 4);
  L.tok_f32 = al((size_t)chunk * 4);
  L.tok_u8 = al((size_t)chunk);
  L.partial = al(rl_policy_loss_workspace_size(chunk, 1, dtype));
  L.stats = al(sizeof(rl_loss_stats));
  L.seq = al((size_t)std::max(n_seq, 1) * 4);
  // per slot: logits, targets, token_seq, old_logp, logp, mask, partials
  const size_t slot = L.logits + 2 * L.tok_i32 + 2 * L.tok_f32 + L.tok_u8 + L.partial;
  L.total = 2 * slot + L.stats + 3 * L.seq;
  return L;
}

struct HostStreams {
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t ev[8] = {};
  int dev = -1;
};

static rl_status get_streams(HostStreams** out) {
  static thread_local HostStreams hs;
  int dev = 0;
  cudaGetDevice(&dev);
  if (hs.dev != dev) {
    if (cudaStreamCreateWithFlags(&hs.h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hs.comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hs.d2h, cudaStreamNonBlocking) != cudaSuccess)
      return check_launch("stream create");
    for (auto& e : hs.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return check_launch("event create");
    hs.dev = dev;
  }
  *out = &hs;
  return RL_OK;
}

#define RL_CK(x)                                        \
  do {                                                  \
    if ((x) != cudaSuccess) return check_launch(#x);    \
  } while (0)

}  // namespace rl

extern "C" size_t rl_policy_loss_host_workspace_size(int64_t chunk_tokens, int64_t vocab, int64_t ld,
                                                     int32_t dtype, int32_t n_seq) {
  (void)vocab;
  if (chunk_tokens < 1 || ld < 1) return 0;
  return rl::host_layout(chunk_tokens, ld, dtype, n_seq).total;
}

extern "C" rl_status rl_policy_loss_fwd_bwd_host(
    const void* logits_host, int32_t dtype, int64_t n_tokens, int64_t vocab, int64_t ld,
    const int32_t* targets_host, const float* old_logp_host, const uint8_t* loss_mask_host,
    const int32_t* token_seq_host, const float* seq_adv_host, const int32_t* seq_version_host,
    const int32_t* seq_active_host, int32_t n_seq, const rl_loss_params* p, void* dlogits_host,
    float* logp_out_host, rl_loss_stats* stats_host, int64_t chunk_tokens, void* workspace,
    size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (!p || !stats_host) return fail(RL_ERR_INVALID_ARGUMENT, "NULL params/stats_host");
  if (p->kl_coef != 0.f || p->prox_logp)  // per-token device arrays do not fit the host staging
    return fail(RL_ERR_UNSUPPORTED, "kl_coef / prox_logp are device-buffer options (rl_policy_loss_fwd_bwd)");
  if (n_tokens < 0 || vocab < 1 || ld < vocab || n_seq < 0 || chunk_tokens < 1)
    return fail(RL_ERR_INVALID_ARGUMENT, "bad sizes");
  if (dtype != RL_F32 && dtype != RL_BF16) return fail(RL_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  if (n_tokens > 0 && (!logits_host || !targets_host || !old_logp_host || !token_seq_host || !seq_adv_host))
    return fail(RL_ERR_INVALID_ARGUMENT, "NULL required host array");
  if (p->agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN && !seq_active_host)
    return fail(RL_ERR_INVALID_ARGUMENT, "SEQ_MEAN_TOKEN_MEAN needs seq_active");
  const HostLayout L = host_layout(chunk_tokens, ld, dtype, n_seq);
  if (!workspace || workspace_bytes < L.total)
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes", L.total);
  HostStreams* hs;
  rl_status st = get_streams(&hs);
  if (st != RL_OK) return st;
  cudaStream_t user = (cudaStream_t)stream;
  const size_t eb = dtype == RL_BF16 ? 2 : 4;
  char* w = (char*)workspace;
  char* slot_base[2];
  const size_t slot_bytes = L.logits + 2 * L.tok_i32 + 2 * L.tok_f32 + L.tok_u8 + L.partial;
  slot_base[0] = w;
  slot_base[1] = w + slot_bytes;
  char* tail = w + 2 * slot_bytes;
  rl_loss_stats* d_stats = (rl_loss_stats*)tail;
  float* d_adv = (float*)(tail + L.stats);
  int32_t* d_ver = (int32_t*)(tail + L.stats + L.seq);
  int32_t* d_act = (int32_t*)(tail + L.stats + 2 * L.seq);
  cudaEvent_t e_user = hs->ev[6], e_done = hs->ev[7];
  // order after prior work on the user's stream
  RL_CK(cudaEventRecord(e_user, user));
  RL_CK(cudaStreamWaitEvent(hs->h2d, e_user, 0));
  RL_CK(cudaStreamWaitEvent(hs->comp, e_user, 0));
  RL_CK(cudaStreamWaitEvent(hs->d2h, e_user, 0));
  if (n_seq > 0) {
    RL_CK(cudaMemcpyAsync(d_adv, seq_adv_host, (size_t)n_seq * 4, cudaMemcpyHostToDevice, hs->h2d));
    if (seq_version_host)
      RL_CK(cudaMemcpyAsync(d_ver, seq_version_host, (size_t)n_seq * 4, cudaMemcpyHostToDevice, hs->h2d));
    if (seq_active_host)
      RL_CK(cudaMemcpyAsync(d_act, seq_active_host, (size_t)n_seq * 4, cudaMemcpyHostToDevice, hs->h2d));
  }
  if (p->flags & RL_F_STATS_ACCUMULATE)  // seed the device accumulator with the caller's values
    RL_CK(cudaMemcpyAsync(d_stats, stats_host, sizeof(rl_loss_stats), cudaMemcpyHostToDevice, hs->comp));
  else
    RL_CK(cudaMemsetAsync(d_stats, 0, sizeof(rl_loss_stats), hs->comp));
  cudaEvent_t e_in[2] = {hs->ev[0], hs->ev[1]}, e_k[2] = {hs->ev[2], hs->ev[3]},
              e_out[2] = {hs->ev[4], hs->ev[5]};
  rl_loss_params pc = *p;
  pc.flags |= RL_F_STATS_ACCUMULATE;  // chunks accumulate into d_stats
  const int64_t nch = (n_tokens + chunk_tokens - 1) / chunk_tokens;
  for (int64_t c = 0; c < nch; ++c) {
    const int sl = (int)(c & 1);
    const int64_t t0 = c * chunk_tokens, n = std::min(chunk_tokens, n_tokens - t0);
    char* b = slot_base[sl];
    void* d_logits = b;
    int32_t* d_tgt = (int32_t*)(b + L.logits);
    int32_t* d_seq = (int32_t*)(b + L.logits + L.tok_i32);
    float* d_old = (float*)(b + L.logits + 2 * L.tok_i32);
    float* d_logp = (float*)(b + L.logits + 2 * L.tok_i32 + L.tok_f32);
    uint8_t* d_mask = (uint8_t*)(b + L.logits + 2 * L.tok_i32 + 2 * L.tok_f32);
    void* d_part = b + L.logits + 2 * L.tok_i32 + 2 * L.tok_f32 + L.tok_u8;
    if (c >= 2) RL_CK(cudaStreamWaitEvent(hs->h2d, e_out[sl], 0));  // slot drained
    RL_CK(cudaMemcpyAsync(d_logits, (const char*)logits_host + t0 * ld * eb, n * ld * eb,
                          cudaMemcpyHostToDevice, hs->h2d));
    RL_CK(cudaMemcpyAsync(d_tgt, targets_host + t0, n * 4, cudaMemcpyHostToDevice, hs->h2d));
    RL_CK(cudaMemcpyAsync(d_seq, token_seq_host + t0, n * 4, cudaMemcpyHostToDevice, hs->h2d));
    RL_CK(cudaMemcpyAsync(d_old, old_logp_host + t0, n * 4, cudaMemcpyHostToDevice, hs->h2d));
    if (loss_mask_host)
      RL_CK(cudaMemcpyAsync(d_mask, loss_mask_host + t0, n, cudaMemcpyHostToDevice, hs->h2d));
    RL_CK(cudaEventRecord(e_in[sl], hs->h2d));
    RL_CK(cudaStreamWaitEvent(hs->comp, e_in[sl], 0));
    st = rl_policy_loss_fwd_bwd(d_logits, dtype, n, vocab, ld, d_tgt, d_old,
                                loss_mask_host ? d_mask : nullptr, d_seq, d_adv,
                                seq_version_host ? d_ver : nullptr, seq_active_host ? d_act : nullptr,
                                &pc, d_logits /* in place */, d_logp, nullptr, d_stats, d_part,
                                L.partial, hs->comp);
    if (st != RL_OK) return st;
    RL_CK(cudaEventRecord(e_k[sl], hs->comp));
    RL_CK(cudaStreamWaitEvent(hs->d2h, e_k[sl], 0));
    if (dlogits_host)
      RL_CK(cudaMemcpyAsync((char*)dlogits_host + t0 * ld * eb, d_logits, n * ld * eb,
                            cudaMemcpyDeviceToHost, hs->d2h));
    if (logp_out_host)
      RL_CK(cudaMemcpyAsync(logp_out_host + t0, d_logp, n * 4, cudaMemcpyDeviceToHost, hs->d2h));
    RL_CK(cudaEventRecord(e_out[sl], hs->d2h));
  }
  RL_CK(cudaEventRecord(e_done, hs->comp));
  RL_CK(cudaStreamWaitEvent(hs->d2h, e_done, 0));
  RL_CK(cudaMemcpyAsync(stats_host, d_stats, sizeof(rl_loss_stats), cudaMemcpyDeviceToHost, hs->d2h));
  RL_CK(cudaStreamSynchronize(hs->d2h));
  RL_CK(cudaStreamSynchronize(hs->h2d));
  RL_CK(cudaStreamSynchronize(hs->comp));
  RL_CK(cudaEventRecord(e_done, hs->d2h));
  RL_CK(cudaStreamWaitEvent(user, e_done, 0));
  return RL_OK;
}
