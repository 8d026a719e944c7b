// Per-token epilogue of the clipped importance-ratio surrogate (c4–c7 of DESIGN.md §3) and the
// per-CTA statistics partials.  Shared by every loss kernel (two-pass, cluster row-resident,
// vocab-parallel) so all of them take bitwise-identical per-token decisions.
#pragma once
#include "common.cuh"

namespace rl {

struct Knobs {
  float lo_b, hi_b;  // 1 - eps_low, 1 + eps_high
  float inv_t, clamp_c, grad_scale;
  float kl_coef;     // beta of the k3 KL term (reading N1), 0 = off
  int32_t agg, trainer_version, max_staleness, global_num_seqs;
  uint32_t flags;
  double active_host;
  const double* active_dev;
  const float* ref_logp;   // [n] reference-policy log-probs (kl_coef != 0)
  const float* prox_logp;  // [n] proximal-policy log-probs or NULL (decoupled ratio, reading N2)
};

inline Knobs make_knobs(const rl_loss_params* p) {
  Knobs k;
  k.lo_b = 1.0f - p->clip_eps_low;
  k.hi_b = 1.0f + p->clip_eps_high;
  k.inv_t = p->inv_temperature;
  k.clamp_c = p->log_ratio_clamp;
  k.grad_scale = p->grad_scale;
  k.agg = p->agg;
  k.trainer_version = p->trainer_version;
  k.max_staleness = p->max_staleness;
  k.global_num_seqs = p->global_num_seqs;
  k.flags = p->flags;
  k.active_host = p->global_active_tokens;
  k.active_dev = p->active_tokens_dev;
  k.kl_coef = p->kl_coef;
  k.ref_logp = p->kl_coef != 0.f ? p->ref_logp : nullptr;
  k.prox_logp = p->prox_logp;
  return k;
}

// Statistics partials: indices follow rl_loss_stats field order.
enum {
  ST_LOSS = 0, ST_ACTIVE, ST_WSUM, ST_RSUM, ST_CLO, ST_CHI, ST_CLAMP, ST_STALE, ST_BAD, ST_NEG, ST_KL, ST_ENT
};
struct Acc {
  double v[RL_LOSS_STATS_N];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) v[i] = 0.0;
  }
};

// 1 / N_active (TOKEN_MEAN) read once per CTA.
__device__ __forceinline__ double token_mean_inv(const Knobs& kn) {
  const double d = kn.active_dev ? *kn.active_dev : kn.active_host;
  return d > 0.0 ? 1.0 / d : 0.0;
}

// Per-token ratio / clip decision (c4, c5), KL term (N1) and gradient scale (c7).  Shared by
// token_epilogue and the SV kernel's consumer threads, so the statistics and the written
// gradient take the same decisions from the same float operations.
//   base = prox (decoupled ratio, N2) or old;  rho = exp(clamp(prox - old)) or 1 (no gradient)
//   D = logp - base; Dc = clamp(D, +-c); r = exp(Dc); clipped: A>0 && r>hi -> 2, A<0 && r<lo -> 1
//   KL: Dk = clamp(ref - logp); kl = exp(Dk) - Dk - 1; dkl = dKL/dlogp = 1 - exp(Dk) (0 if clamped)
struct TokRatio {
  float r, rho, kl, dkl;
  uint8_t cl;
  bool clamp;
};
// prox / ref: the token's proximal / reference log-prob (ignored unless kn has them)
__device__ __forceinline__ TokRatio token_ratio(float logp, float old, float prox, float ref, float A,
                                                const Knobs& kn) {
  TokRatio t;
  const bool has_prox = kn.prox_logp != nullptr;
  const float base = has_prox ? prox : old;
  t.rho = has_prox ? expf(fminf(fmaxf(prox - old, -kn.clamp_c), kn.clamp_c)) : 1.f;
  const float D = logp - base;
  const float Dc = fminf(fmaxf(D, -kn.clamp_c), kn.clamp_c);
  t.clamp = Dc != D;
  t.r = expf(Dc);
  t.cl = 0;
  if (A > 0.f && t.r > kn.hi_b) t.cl = 2;
  else if (A < 0.f && t.r < kn.lo_b) t.cl = 1;
  t.kl = 0.f;
  t.dkl = 0.f;
  if (kn.kl_coef != 0.f) {
    const float Dk = ref - logp;
    const float Dkc = fminf(fmaxf(Dk, -kn.clamp_c), kn.clamp_c);
    const float e = expf(Dkc);
    t.kl = e - Dkc - 1.f;
    t.dkl = Dkc == Dk ? 1.f - e : 0.f;
  }
  return t;
}
// s = w (rho A r [unclipped and unclamped] - beta dKL/dlogp) inv_T grad_scale  (wf = (float) w)
__device__ __forceinline__ float token_scale(const TokRatio& t, float wf, float A, const Knobs& kn) {
  const float g = ((t.cl != 0 || t.clamp) ? 0.f : t.rho * A * t.r) - kn.kl_coef * t.dkl;
  return wf * g * kn.inv_t * kn.grad_scale;
}
// the clipped surrogate alone (no proximal ratio, no KL): the default path's per-token math
__device__ __forceinline__ TokRatio token_ratio_basic(float logp, float old, float A, const Knobs& kn) {
  TokRatio t;
  const float D = logp - old;
  const float Dc = fminf(fmaxf(D, -kn.clamp_c), kn.clamp_c);
  t.clamp = Dc != D;
  t.r = expf(Dc);
  t.rho = 1.f;
  t.kl = 0.f;
  t.dkl = 0.f;
  t.cl = 0;
  if (A > 0.f && t.r > kn.hi_b) t.cl = 2;
  else if (A < 0.f && t.r < kn.lo_b) t.cl = 1;
  return t;
}
__device__ __forceinline__ float token_scale_basic(const TokRatio& t, float wf, float A, const Knobs& kn) {
  return (t.cl != 0 || t.clamp) ? 0.f : wf * A * t.r * kn.inv_t * kn.grad_scale;
}
// w = 1/N | 1/(S L_i) | 1 (c6); Li = the token's sequence's active-token count
__device__ __forceinline__ double token_weight_li(int32_t Li, double inv_tm, const Knobs& kn) {
  if (kn.agg == RL_AGG_TOKEN_MEAN) return inv_tm;
  if (kn.agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN)
    return (Li > 0 && kn.global_num_seqs > 0) ? 1.0 / ((double)kn.global_num_seqs * (double)Li) : 0.0;
  return 1.0;
}
// L_i of a valid token, read only when the aggregation uses it
__device__ __forceinline__ int32_t token_li(const RowMeta& mt, const int32_t* seq_active, const Knobs& kn) {
  return (kn.agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN && seq_active) ? seq_active[mt.seq] : 0;
}
__device__ __forceinline__ double token_weight(const RowMeta& mt, const int32_t* seq_active, double inv_tm,
                                               const Knobs& kn) {
  return token_weight_li(token_li(mt, seq_active, kn), inv_tm, kn);
}
// the token's (prox, ref) inputs, loaded only when the knobs use them
__device__ __forceinline__ void token_extra(const Knobs& kn, int64_t row, float old, float& prox, float& ref) {
  prox = kn.prox_logp ? kn.prox_logp[row] : old;
  ref = kn.ref_logp ? kn.ref_logp[row] : 0.f;
}

// Per-token epilogue.  Returns the gradient scale s_t (0 for invalid tokens; clipped / clamped
// tokens keep only the KL part) and adds the token's contribution to `acc`.
//   L = -rho min(r A, clip(r, lo, hi) A) + beta KL
//   (token_epilogue_li: the same with the sequence's L_i already loaded)
__device__ __forceinline__ float token_epilogue_li(const RowMeta& mt, float logp, float old, float A, int32_t Li,
                                                   double inv_tm, const Knobs& kn, Acc& acc, uint8_t* clipped_out,
                                                   float prox, float ref) {
  acc.v[ST_BAD] += mt.bad ? 1.0 : 0.0;
  acc.v[ST_NEG] += mt.neg_stale ? 1.0 : 0.0;
  acc.v[ST_STALE] += mt.stale_drop ? 1.0 : 0.0;
  if (!mt.valid) {
    if (clipped_out) *clipped_out = 0;
    return 0.f;
  }
  const TokRatio t = token_ratio(logp, old, prox, ref, A, kn);
  const float u = t.r * A;
  const float kk = fminf(fmaxf(t.r, kn.lo_b), kn.hi_b) * A;
  const float L = -t.rho * fminf(u, kk) + kn.kl_coef * t.kl;
  const double w = token_weight_li(Li, inv_tm, kn);
  acc.v[ST_LOSS] += w * (double)L;
  acc.v[ST_ACTIVE] += 1.0;
  acc.v[ST_WSUM] += w;
  acc.v[ST_RSUM] += (double)t.r;
  acc.v[ST_CLO] += t.cl == 1 ? 1.0 : 0.0;
  acc.v[ST_CHI] += t.cl == 2 ? 1.0 : 0.0;
  acc.v[ST_CLAMP] += t.clamp ? 1.0 : 0.0;
  acc.v[ST_KL] += w * (double)t.kl;
  if (clipped_out) *clipped_out = t.cl;
  return token_scale(t, (float)w, A, kn);
}
__device__ __forceinline__ float token_epilogue(const RowMeta& mt, float logp, float old, float A,
                                                const int32_t* seq_active, double inv_tm,
                                                const Knobs& kn, Acc& acc, uint8_t* clipped_out,
                                                float prox = 0.f, float ref = 0.f) {
  const int32_t Li = mt.valid ? token_li(mt, seq_active, kn) : 0;
  return token_epilogue_li(mt, logp, old, A, Li, inv_tm, kn, acc, clipped_out, prox, ref);
}

// token_epilogue of the clipped surrogate alone (token_ratio_basic / token_scale_basic)
__device__ __forceinline__ float token_epilogue_basic(const RowMeta& mt, float logp, float old, float A,
                                                      const int32_t* seq_active, double inv_tm,
                                                      const Knobs& kn, Acc& acc, uint8_t* clipped_out) {
  acc.v[ST_BAD] += mt.bad ? 1.0 : 0.0;
  acc.v[ST_NEG] += mt.neg_stale ? 1.0 : 0.0;
  acc.v[ST_STALE] += mt.stale_drop ? 1.0 : 0.0;
  if (!mt.valid) {
    if (clipped_out) *clipped_out = 0;
    return 0.f;
  }
  const TokRatio t = token_ratio_basic(logp, old, A, kn);
  const float u = t.r * A;
  const float kk = fminf(fmaxf(t.r, kn.lo_b), kn.hi_b) * A;
  const float L = -fminf(u, kk);
  const double w = token_weight(mt, seq_active, inv_tm, kn);
  acc.v[ST_LOSS] += w * (double)L;
  acc.v[ST_ACTIVE] += 1.0;
  acc.v[ST_WSUM] += w;
  acc.v[ST_RSUM] += (double)t.r;
  acc.v[ST_CLO] += t.cl == 1 ? 1.0 : 0.0;
  acc.v[ST_CHI] += t.cl == 2 ? 1.0 : 0.0;
  acc.v[ST_CLAMP] += t.clamp ? 1.0 : 0.0;
  if (clipped_out) *clipped_out = t.cl;
  return token_scale_basic(t, (float)w, A, kn);
}

// log-prob from the log2-domain statistics: c2 = M + log2 S; logp = z_y - c2 ln2
__device__ __forceinline__ float logp_from(const RowMeta& mt, float zy, float c2) {
  if (mt.in_range) return zy - c2 * RL_LN2;
  if (mt.bad) return __int_as_float(0x7fc00000);
  return 0.f;
}

constexpr int kMaxStatCtas = 4096;  // upper bound of per-CTA partial rows in the workspace

}  // namespace rl
