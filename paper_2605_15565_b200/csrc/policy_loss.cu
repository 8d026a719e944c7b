// (4) Fused policy-loss forward + backward — c3–c7 of DESIGN.md §3 (north_star: the
// gather, ratio, clip, mask and gradient write fused into the streaming pass over the
// logits; dL/dlogits = scale*(softmax - onehot)).
//
// This file holds the entry point, the deterministic statistics reduction (K6) and the
// two-pass kernel "L": one CTA per row; pass 1 streams the row from HBM
// with an L2 evict_last policy and reduces (max, sum-exp2); pass 2 re-reads the row (L2
// hit) and writes dlogits with streaming stores.  The row-resident cluster kernel "R"
// (1 HBM read + 1 write, one MUFU.EX2 per element) lives in policy_loss_cluster.cu.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "loss_common.cuh"
#include "rowstats.cuh"

namespace rl {

constexpr int kL2Threads = 512;
constexpr int kL2Unroll = 4;

template <typename T>
__global__ void __launch_bounds__(kL2Threads) loss_two_pass_kernel(
    const void* __restrict__ logits, int64_t n_tokens, int64_t V, int64_t ld,
    const int32_t* __restrict__ targets, const float* __restrict__ old_logp,
    const uint8_t* __restrict__ loss_mask, const int32_t* __restrict__ token_seq,
    const float* __restrict__ seq_adv, const int32_t* __restrict__ seq_version,
    const int32_t* __restrict__ seq_active, Knobs kn, void* dlogits, float* __restrict__ logp_out,
    uint8_t* __restrict__ clipped_out, double* __restrict__ partials, const uint8_t* __restrict__ only) {
  constexpr int EPV = VecTraits<T>::EPV;
  __shared__ float red[64];
  __shared__ float s_row[3];  // s_t, c2, (unused)
  __shared__ uint32_t sel[kL2Threads / 32];
  const float k = kn.inv_t * RL_LOG2E;
  const uint64_t keep = policy_evict_last();
  const int64_t row_bytes = ld * elem_bytes<T>();
  const double inv_tm = token_mean_inv(kn);
  Acc acc;
  acc.zero();
  auto process = [&](int64_t row) {
    const char* rp = reinterpret_cast<const char*>(logits) + row * row_bytes;
    char* dp = reinterpret_cast<char*>(dlogits) + row * row_bytes;
    const RowMeta mt = row_meta(row, V, targets, loss_mask, token_seq, seq_version,
                                kn.trainer_version, kn.max_staleness);
    const bool skip = (kn.flags & RL_F_SKIP_MASKED_READS) && !mt.valid;
    float zy = 0.f;
    if (threadIdx.x == 0 && mt.in_range && !skip) zy = VecTraits<T>::load1(rp, mt.y) * kn.inv_t;
    MS st{-INFINITY, 0.f};
    if (!skip) st = row_stats_thread<T, kL2Threads, kL2Unroll>(rp, V, k, keep);
    st = block_reduce_ms<kL2Threads>(st, red);  // contains __syncthreads: row fully read
    if (threadIdx.x == 0) {
      const float c2 = st.m + fast_log2(st.s);
      const float lp = skip ? 0.f : logp_from(mt, zy, c2);
      if (logp_out) logp_out[row] = lp;
      const float A = mt.valid ? seq_adv[mt.seq] : 0.f;
      const float old = mt.valid ? old_logp[row] : 0.f;
      float prox_, ref_;
      token_extra(kn, row, old, prox_, ref_);
      const float s = token_epilogue(mt, lp, old, A, seq_active, inv_tm, kn, acc,
                                     clipped_out ? clipped_out + row : nullptr, prox_, ref_);
      s_row[0] = s;
      s_row[1] = c2;
    }
    __syncthreads();
    const float s = s_row[0], c2 = s_row[1];
    __syncthreads();  // s_row reusable by the next row
    // entropy (reading N3): H = lse - sum_v p_v z_v over the row, for valid tokens
    const bool ent = (kn.flags & RL_F_ENTROPY) && mt.valid;
    // pass 2: dlogits = s*(2^(t - c2) - [v == y]); exact zeros when s == 0
    const uint4* vrow = reinterpret_cast<const uint4*>(rp);
    uint4* vout = reinterpret_cast<uint4*>(dp);
    const int64_t nvec = V / EPV;
    if (s == 0.f && !ent) {
      for (int64_t i = threadIdx.x; i < nvec; i += kL2Threads) st_stream_v4(vout + i, make_uint4(0, 0, 0, 0));
      for (int64_t c = nvec * EPV + threadIdx.x; c < V; c += kL2Threads) VecTraits<T>::store1(dp, c, 0.f);
      return;
    }
    const uint64_t drop = policy_evict_first();
    const int32_t y = mt.y;
    float pz = 0.f;  // this thread's sum p_v x_v
    for (int64_t i = threadIdx.x; i < nvec; i += kL2Threads) {
      float f[EPV];
      VecTraits<T>::unpack(ld_hint_v4(vrow + i, drop), f);
#pragma unroll
      for (int j = 0; j < EPV; ++j) {
        const float pv = fast_exp2(fmaf(f[j], k, -c2));
        if (ent) pz = fmaf(pv, f[j], pz);
        f[j] = s * pv;
      }
      const int64_t c0 = i * EPV;
      onehot_sub(f, y - c0, s);  // static indices: f stays in registers
      RL_DCHECK(i < nvec);
      st_stream_v4(vout + i, VecTraits<T>::pack(f));
    }
    for (int64_t c = nvec * EPV + threadIdx.x; c < V; c += kL2Threads) {
      RL_DCHECK(c < V);
      const float x = VecTraits<T>::load1(rp, c);
      const float pv = fast_exp2(fmaf(x, k, -c2));
      if (ent) pz = fmaf(pv, x, pz);
      float v = s * pv;
      if (c == y) v -= s;
      VecTraits<T>::store1(dp, c, v);
    }
    if (ent) {  // block sum, then thread 0: H = c2 ln2 - inv_T sum p x
      pz = warp_sum(pz);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = pz;
      __syncthreads();
      if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < kL2Threads / 32; ++w) t += red[w];
        acc.v[ST_ENT] += (double)(c2 * RL_LN2 - kn.inv_t * t);
      }
      __syncthreads();  // red reusable
    }
  };
  if (!only) {
    for (int64_t row = blockIdx.x; row < n_tokens; row += gridDim.x) process(row);
  } else {
    // fixup launch after the single-visit kernel: only the rows it flagged, found 512 candidate
    // rows at a time by ballot and visited in ascending order (deterministic partial sums)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t base = 0; blockIdx.x + base * gridDim.x < n_tokens; base += kL2Threads) {
      const int64_t cand = blockIdx.x + (base + threadIdx.x) * gridDim.x;
      const uint32_t m = __ballot_sync(0xffffffffu, cand < n_tokens && only[cand] != 0);
      if (lane == 0) sel[warp] = m;
      __syncthreads();
      for (int w = 0; w < kL2Threads / 32; ++w) {
        uint32_t mw = sel[w];
        while (mw) {
          const int bit = __ffs(mw) - 1;
          mw &= mw - 1;
          process(blockIdx.x + (base + w * 32 + bit) * gridDim.x);
        }
      }
      __syncthreads();  // sel reusable
    }
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < RL_LOSS_STATS_N; ++i) partials[(int64_t)blockIdx.x * RL_LOSS_STATS_N + i] = acc.v[i];
  }
}

// K6: fixed-order fp64 reduction of the per-CTA partials (deterministic).
__global__ void stats_reduce_kernel(const double* __restrict__ partials, int n_ctas,
                                    rl_loss_stats* __restrict__ stats, int accumulate) {
  const int i = threadIdx.x;
  if (i >= RL_LOSS_STATS_N) return;
  double s = 0.0;
  for (int b = 0; b < n_ctas; ++b) s += partials[(int64_t)b * RL_LOSS_STATS_N + i];
  double* out = reinterpret_cast<double*>(stats);
  out[i] = accumulate ? out[i] + s : s;
}

rl_status launch_stats_reduce(const double* partials, int n_ctas, rl_loss_stats* stats,
                              bool accumulate, cudaStream_t s) {
  stats_reduce_kernel<<<1, 32, 0, s>>>(partials, n_ctas, stats, accumulate ? 1 : 0);
  return check_launch("stats_reduce_kernel");
}

static int two_pass_grid(int64_t n_tokens) {
  // one 297 KB row in flight per SM keeps ~44 MB resident in the 126 MB L2
  return (int)std::min<int64_t>(n_tokens, std::min(dev_info().sms, kMaxStatCtas));
}

rl_status launch_loss_two_pass(const void* logits, int32_t dtype, int64_t n, int64_t V, int64_t ld,
                               const int32_t* targets, const float* old_logp, const uint8_t* mask,
                               const int32_t* token_seq, const float* seq_adv,
                               const int32_t* seq_version, const int32_t* seq_active,
                               const Knobs& kn, void* dlogits, float* logp_out, uint8_t* clipped_out,
                               double* partials, int* n_ctas, cudaStream_t s, const uint8_t* only = nullptr) {
  // fixup launch (only != NULL): a fixed small grid, scanned rows are rare
  const int grid = only ? (int)std::min<int64_t>(n, 148) : two_pass_grid(n);
  *n_ctas = grid;
  if (dtype == RL_BF16)
    loss_two_pass_kernel<bf16_t><<<grid, kL2Threads, 0, s>>>(
        logits, n, V, ld, targets, old_logp, mask, token_seq, seq_adv, seq_version, seq_active, kn,
        dlogits, logp_out, clipped_out, partials, only);
  else
    loss_two_pass_kernel<float><<<grid, kL2Threads, 0, s>>>(
        logits, n, V, ld, targets, old_logp, mask, token_seq, seq_adv, seq_version, seq_active, kn,
        dlogits, logp_out, clipped_out, partials, only);
  return check_launch("loss_two_pass_kernel");
}

// Single-visit cluster kernel (policy_loss_sv.cu); rows it flags in `redo` are left to a
// two-pass fixup launch.
rl_status launch_loss_sv(const void* logits, int32_t dtype, int64_t n, int64_t V, int64_t ld,
                         const int32_t* targets, const float* old_logp, const uint8_t* mask,
                         const int32_t* token_seq, const float* seq_adv, const int32_t* seq_version,
                         const int32_t* seq_active, const Knobs& kn, void* dlogits, float* logp_out,
                         uint8_t* clipped_out, double* partials, uint8_t* redo, int* n_ctas,
                         cudaStream_t s);

// Kernel choice (development option RL_DEV_LOSS_KERNEL): 0 = single visit (default), 1 = two-pass.
enum { K_SV = 0, K_TWO_PASS = 1 };

}  // namespace rl

// per-CTA statistics partials (fast kernel + fixup) | per-row redo flags of the SV kernel
extern "C" size_t rl_policy_loss_workspace_size(int64_t n_tokens, int64_t vocab, int32_t dtype) {
  (void)vocab; (void)dtype;
  const size_t flags = n_tokens > 0 ? ((size_t)n_tokens + 255) & ~(size_t)255 : 0;
  return (size_t)rl::kMaxStatCtas * RL_LOSS_STATS_N * sizeof(double) + flags;
}

extern "C" rl_status rl_policy_loss_fwd_bwd(const void* logits, int32_t dtype, int64_t n_tokens,
                                            int64_t vocab, int64_t ld, const int32_t* targets,
                                            const float* old_logp, const uint8_t* loss_mask,
                                            const int32_t* token_seq, const float* seq_adv,
                                            const int32_t* seq_version, const int32_t* seq_active,
                                            const rl_loss_params* p, void* dlogits,
                                            float* logp_out, uint8_t* clipped_out,
                                            rl_loss_stats* stats, void* workspace,
                                            size_t workspace_bytes, rl_stream stream) {
  using namespace rl;
  if (!p) return fail(RL_ERR_INVALID_ARGUMENT, "NULL params");
  if (n_tokens < 0 || vocab < 1 || ld < vocab)
    return fail(RL_ERR_INVALID_ARGUMENT, "n_tokens < 0, vocab < 1 or ld < vocab");
  if (dtype != RL_F32 && dtype != RL_BF16) return fail(RL_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  if (!(p->inv_temperature > 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "inv_temperature must be > 0");
  if (!(p->log_ratio_clamp >= 0.f)) return fail(RL_ERR_INVALID_ARGUMENT, "log_ratio_clamp must be >= 0");
  if (!(p->clip_eps_low >= 0.f) || !(p->clip_eps_high >= 0.f))
    return fail(RL_ERR_INVALID_ARGUMENT, "clip eps must be >= 0");
  if (p->agg < RL_AGG_TOKEN_MEAN || p->agg > RL_AGG_SUM) return fail(RL_ERR_INVALID_ARGUMENT, "bad agg %d", p->agg);
  if (p->agg == RL_AGG_SEQ_MEAN_TOKEN_MEAN && !seq_active)
    return fail(RL_ERR_INVALID_ARGUMENT, "SEQ_MEAN_TOKEN_MEAN needs seq_active");
  if (!stats) return fail(RL_ERR_INVALID_ARGUMENT, "NULL stats");
  if (p->kl_coef != 0.f && !p->ref_logp) return fail(RL_ERR_INVALID_ARGUMENT, "kl_coef != 0 needs ref_logp");
  if (!(p->kl_coef == p->kl_coef)) return fail(RL_ERR_INVALID_ARGUMENT, "kl_coef is NaN");
  if (!workspace || workspace_bytes < rl_policy_loss_workspace_size(n_tokens, vocab, dtype))
    return fail(RL_ERR_WORKSPACE, "workspace must be >= %zu bytes",
                rl_policy_loss_workspace_size(n_tokens, vocab, dtype));
  cudaStream_t s = (cudaStream_t)stream;
  const bool acc = (p->flags & RL_F_STATS_ACCUMULATE) != 0;
  if (n_tokens == 0) {
    if (!acc && cudaMemsetAsync(stats, 0, sizeof(rl_loss_stats), s) != cudaSuccess)
      return check_launch("memset stats");
    return RL_OK;
  }
  if (!logits || !dlogits || !targets || !old_logp || !token_seq || !seq_adv)
    return fail(RL_ERR_INVALID_ARGUMENT, "NULL logits/dlogits/targets/old_logp/token_seq/seq_adv");
  const int64_t eb = dtype == RL_BF16 ? 2 : 4;
  if (((uintptr_t)logits & 15) || ((uintptr_t)dlogits & 15) || (ld * eb) % 16)
    return fail(RL_ERR_ALIGNMENT, "logits/dlogits must be 16-B aligned with ld*elem %% 16 == 0");
  if (dlogits != logits) {  // partial overlap is undefined: reject it when detectable
    const char* a = (const char*)logits;
    const char* b = (const char*)dlogits;
    const int64_t bytes = n_tokens * ld * eb;
    if (a < b + bytes && b < a + bytes)
      return fail(RL_ERR_INVALID_ARGUMENT, "dlogits partially overlaps logits");
  }
  if (rl_status e = require_sm100(); e != RL_OK) return e;  // RL_ERR_UNSUPPORTED off sm_100
  const Knobs kn = make_knobs(p);
  double* partials = (double*)workspace;
  int n_ctas = 0;
  rl_status st = RL_ERR_UNSUPPORTED;
  const int choice = dev_option(OPT_LOSS_KERNEL) == 1 ? K_TWO_PASS : K_SV;
  if (choice == K_SV) {
    uint8_t* redo = (uint8_t*)workspace + (size_t)kMaxStatCtas * RL_LOSS_STATS_N * sizeof(double);
    st = launch_loss_sv(logits, dtype, n_tokens, vocab, ld, targets, old_logp, loss_mask, token_seq,
                        seq_adv, seq_version, seq_active, kn, dlogits, logp_out, clipped_out, partials,
                        redo, &n_ctas, s);
    if (st == RL_OK) {  // rows the fast path flagged: exact two-pass, own partial slots
      int n_fix = 0;
      st = launch_loss_two_pass(logits, dtype, n_tokens, vocab, ld, targets, old_logp, loss_mask, token_seq, seq_adv, seq_version,
                                seq_active, kn, dlogits, logp_out, clipped_out,
                                partials + (size_t)n_ctas * RL_LOSS_STATS_N, &n_fix, s, redo);
      if (st != RL_OK) return st;
      n_ctas += n_fix;
    }
  }
  if (st == RL_ERR_UNSUPPORTED)
    st = launch_loss_two_pass(logits, dtype, n_tokens, vocab, ld, targets, old_logp, loss_mask,
                              token_seq, seq_adv, seq_version, seq_active, kn, dlogits, logp_out,
                              clipped_out, partials, &n_ctas, s);
  if (st != RL_OK) return st;
  return launch_stats_reduce(partials, n_ctas, stats, acc, s);
}
